// Standalone probe: LOP3 issue rate on the ALU pipe (and IMAD co-issue) on this B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NCHAIN, int WITH_IMAD>
__global__ void lop3_loop(uint32_t* out, uint32_t seed, int iters) {
  uint32_t v[NCHAIN];
  uint32_t a = seed ^ threadIdx.x, b = seed * 7u + blockIdx.x, m = seed | 1u;
#pragma unroll
  for (int i = 0; i < NCHAIN; i++) v[i] = a + i * 0x9E3779B9u;
  uint32_t acc = 0;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
#pragma unroll
      for (int i = 0; i < NCHAIN; i++) {
        uint32_t r;
        // immediates vary with (i,k) so nothing folds
        if ((k + i) & 1)
          asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(v[i]), "r"(a), "r"(b));
        else
          asm volatile("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(r) : "r"(v[i]), "r"(b), "r"(a));
        v[i] = r;
        if (WITH_IMAD) { asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(acc) : "r"(v[i]), "r"(m)); }
      }
    }
  }
  uint32_t x = acc;
#pragma unroll
  for (int i = 0; i < NCHAIN; i++) x ^= v[i];
  if (x == 0x12345678u) out[threadIdx.x] = x;
}

// Operand pattern of real circuits: 3 distinct register sources per lop3, drawn
// from a pool of P live registers (v[i] = f(v[i], v[i+O1], v[i+O2]) mod P), so the
// register-bank / operand-reuse behaviour of generated code is visible.
template <int P, int O1, int O2>
__global__ void lop3_pool(uint32_t* out, uint32_t seed, int iters) {
  uint32_t v[P];
#pragma unroll
  for (int i = 0; i < P; i++) v[i] = (seed ^ threadIdx.x) + i * 0x9E3779B9u + blockIdx.x;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < 2; k++) {
#pragma unroll
      for (int i = 0; i < P; i++) {
        uint32_t r;
        if ((k + i) & 1)
          asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(v[i]), "r"(v[(i + O1) % P]), "r"(v[(i + O2) % P]));
        else
          asm volatile("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(r) : "r"(v[i]), "r"(v[(i + O1) % P]), "r"(v[(i + O2) % P]));
        v[i] = r;
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < P; i++) x ^= v[i];
  if (x == 0x12345678u) out[threadIdx.x] = x;
}

template <int P, int O1, int O2>
void run_pool(int blocks, int threads, int iters) {
  uint32_t* d; cudaMalloc(&d, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; w++) lop3_pool<P, O1, O2><<<blocks, threads>>>(d, 1, iters);
  cudaEventRecord(e0);
  int reps = 5;
  for (int r = 0; r < reps; r++) lop3_pool<P, O1, O2><<<blocks, threads>>>(d, 1, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * iters * 2 * P * reps;
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("pool P=%d O=(%d,%d) blocks=%d threads=%d: %.3f ms  %.3e LOP3/s = %.2f /SM/clk\n", P, O1, O2, blocks,
         threads, ms, ops / (ms * 1e-3), ops / (ms * 1e-3) / 148 / (clk * 1e3));
  cudaFree(d);
}

template <int NCHAIN, int WITH_IMAD>
void run(int blocks, int threads, int iters) {
  uint32_t* d; cudaMalloc(&d, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; w++) lop3_loop<NCHAIN, WITH_IMAD><<<blocks, threads>>>(d, 1, iters);
  cudaEventRecord(e0);
  int reps = 5;
  for (int r = 0; r < reps; r++) lop3_loop<NCHAIN, WITH_IMAD><<<blocks, threads>>>(d, 1, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * iters * 16 * NCHAIN * reps;
  int dev; cudaGetDevice(&dev); int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("nchain=%d imad=%d blocks=%d threads=%d: %.3f ms  %.3e LOP3 thread-ops/s  = %.2f /SM/clk @%.0f MHz(attr)\n",
         NCHAIN, WITH_IMAD, blocks, threads, ms, ops / (ms * 1e-3), ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1e3);
  cudaFree(d);
}

int main() {
  run<4, 0>(148 * 4, 256, 2000);
  run<8, 0>(148 * 4, 256, 2000);
  run<8, 0>(148 * 2, 256, 2000);
  run<8, 0>(148 * 1, 128, 2000);
  run<2, 0>(148 * 1, 128, 2000);
  run<8, 1>(148 * 4, 256, 2000);
  run_pool<24, 8, 16>(148 * 4, 256, 1000);
  run_pool<24, 1, 2>(148 * 4, 256, 1000);
  run_pool<24, 5, 13>(148 * 4, 256, 1000);
  run_pool<32, 7, 19>(148 * 4, 256, 1000);
  run_pool<24, 8, 16>(148 * 9, 128, 1000);
  run_pool<24, 8, 16>(148 * 2, 128, 1000);
  run_pool<24, 8, 16>(148 * 1, 128, 1000);
  return 0;
}
