// Development probe: ALU-pipe efficiency of the generated table-MAC circuit
// with every operand in registers (no loads, no address arithmetic), i.e. the
// ceiling the conv kernel could reach with perfect operand delivery.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2007_06563_b200/csrc \
//        -I paper_2007_06563_b200/csrc/gen -o /tmp/mac_chain_probe tools/mac_chain_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#ifndef PROBE_FMT
#define PROBE_FMT F_e5m3_rne
#include "hobf_circuit_e5m3_rne.cuh"
#else
#include PROBE_HDR
#endif

using F = hobf_gen::PROBE_FMT;

// MODE 0: operands mutated in registers; 1: + EA/SX mutated too (no hoisting);
// 2: + table entry gathered from an L1-resident table every MAC (like the conv).
template <int NG, int MINB, int MODE>
__global__ void __launch_bounds__(128, MINB) chain(uint32_t* out, const uint32_t* in, int iters, uint32_t m) {
  const uint32_t m1 = m >> 24;  // 1 at run time (m = 0x01000193), opaque to the compiler
  __shared__ __align__(16) uint32_t stab[16 * 20];  // MODE 4/5: 16 table rows, 20-word (80 B) or 16-word stride
  if (MODE >= 4) {
    for (int i = threadIdx.x; i < 16 * 20; i += blockDim.x) stab[i] = in[i];
    __syncthreads();
  }
  const int32_t one = (int32_t)m1;
  uint32_t acc[NG][F::NOUT], T[F::NPT], EA[F::WE], SX[1];
  const uint32_t* p = in + (threadIdx.x & 31) * 64;
#pragma unroll
  for (int i = 0; i < NG; i++)
#pragma unroll
    for (int j = 0; j < F::NOUT; j++) acc[i][j] = 0;
#pragma unroll
  for (int j = 0; j < F::NPT; j++) T[j] = p[j];
#pragma unroll
  for (int j = 0; j < F::WE; j++) EA[j] = p[32 + j];
  SX[0] = p[40];
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < NG; i++) F::mac_tab(acc[i], T, EA, SX);
    if (MODE == 1 || MODE == 2 || MODE >= 4) {
#pragma unroll
      for (int j = 0; j < F::WE; j++) EA[j] = EA[j] * m + 0x7F4A7C15u;
      SX[0] = SX[0] * m + 1u;
    }
    if (MODE == 7) {
      // pre-broadcast records: 8 words per activation (EA planes, SX plane, row),
      // coalesced 2 x 128-bit loads per tap; table row gathered from shared memory
      const uint4* pr = reinterpret_cast<const uint4*>(in + 4096) + 2 * ((it * 37 + threadIdx.x) & 511);
      const uint4 r0 = __ldg(pr), r1 = __ldg(pr + 1);
      EA[0] = r0.x; EA[1] = r0.y; EA[2] = r0.z; EA[3] = r0.w; EA[4] = r1.x; SX[0] = r1.y;
      const uint32_t row = r1.z & 15u;
      const uint4* q = reinterpret_cast<const uint4*>(stab + row * 20);
#pragma unroll
      for (int j = 0; j < F::NPT / 4; j++) {
        const uint4 v = q[j];
        T[4 * j] = v.x; T[4 * j + 1] = v.y; T[4 * j + 2] = v.z; T[4 * j + 3] = v.w;
      }
    } else if (MODE == 6) {
      // the conv's per-tap work with the table in shared memory: record load,
      // IMAD/IMAD.HI broadcasts, row by IMAD.HI, 80-byte-stride row gather
      const uint32_t rec = __ldg(in + 4096 + ((it * 37 + threadIdx.x) & 1023));
#pragma unroll
      for (int j = 0; j < F::WE; j++) EA[j] = (uint32_t)__mulhi((int32_t)(rec * (1u << (31 - F::WF - j)) * m1), one);
      SX[0] = (uint32_t)__mulhi((int32_t)(rec * (1u << (31 - F::WF - F::WE)) * m1), one);
      const uint32_t row = __umulhi(rec, 16u * m1);
      const uint4* q = reinterpret_cast<const uint4*>(stab + row * 20);
#pragma unroll
      for (int j = 0; j < F::NPT / 4; j++) {
        const uint4 v = q[j];
        T[4 * j] = v.x; T[4 * j + 1] = v.y; T[4 * j + 2] = v.z; T[4 * j + 3] = v.w;
      }
    } else if (MODE == 3) {
      // like the conv: a per-tap record (L1-resident) -> exponent / sign planes by
      // IMAD + IMAD.HI broadcasts, table row by IMAD.HI, then the row gather
      const uint32_t rec = __ldg(in + 4096 + ((it * 37 + threadIdx.x) & 1023));
#pragma unroll
      for (int j = 0; j < F::WE; j++) EA[j] = (uint32_t)__mulhi((int32_t)(rec * (1u << (31 - F::WF - j)) * m1), one);
      SX[0] = (uint32_t)__mulhi((int32_t)(rec * (1u << (31 - F::WF - F::WE)) * m1), one);
      const uint32_t row = __umulhi(rec, 16u * m1);
      const uint4* q = reinterpret_cast<const uint4*>(in + row * 64);
#pragma unroll
      for (int j = 0; j < F::NPT / 4; j++) {
        const uint4 v = __ldg(q + j);
        T[4 * j] = v.x; T[4 * j + 1] = v.y; T[4 * j + 2] = v.z; T[4 * j + 3] = v.w;
      }
    } else if (MODE == 4 || MODE == 5) {
      const uint32_t r = (EA[0] * m) >> 28;
      const uint4* q = reinterpret_cast<const uint4*>(stab + r * (MODE == 4 ? 20 : 16));
#pragma unroll
      for (int j = 0; j < F::NPT / 4; j++) {
        const uint4 v = q[j];
        T[4 * j] = v.x; T[4 * j + 1] = v.y; T[4 * j + 2] = v.z; T[4 * j + 3] = v.w;
      }
    } else if (MODE == 2) {
      const uint4* q = reinterpret_cast<const uint4*>(in + ((EA[0] * m) >> 28) * 64);  // row from the "activation"
#pragma unroll
      for (int j = 0; j < F::NPT / 4; j++) {
        const uint4 v = __ldg(q + j);
        T[4 * j] = v.x; T[4 * j + 1] = v.y; T[4 * j + 2] = v.z; T[4 * j + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < F::NPT; j++) T[j] = T[j] * m + 0x9E3779B9u;  // FMA pipe: defeats hoisting
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < NG; i++)
#pragma unroll
    for (int j = 0; j < F::NOUT; j++) x ^= acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <int NG, int MINB, int MODE>
void run(int blocks, int iters, uint32_t* d, uint32_t* din) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  chain<NG, MINB, MODE><<<blocks, 128>>>(d, din, iters, 0x01000193u);
  cudaEventRecord(e0);
  chain<NG, MINB, MODE><<<blocks, 128>>>(d, din, iters, 0x01000193u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double lop3 = (double)blocks * 128 * iters * NG * F::G_TAB;
  printf("MODE=%d NG=%d MINB=%d blocks=%d (%.2f warps/SMSP): %.3f ms, %.1f lop3/SM/clk @1965 = %.3f of 64\n", MODE, NG, MINB,
         blocks, blocks * 4.0 / 592, ms, lop3 / (ms * 1e-3) / 148 / 1.965e9, lop3 / (ms * 1e-3) / 148 / 1.965e9 / 64);
}

int main() {
  uint32_t *d, *din;
  cudaMalloc(&d, 148 * 64 * 128 * 4);
  cudaMalloc(&din, 32 * 64 * 4 * 16 + 4096 * 4);
  static uint32_t h[32 * 64 * 16 + 1024];
  for (int i = 0; i < 32 * 64 * 16 + 1024; i++) h[i] = 0x9E3779B9u * (i + 1);
  cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
#ifdef PROBE_HDR  // wide formats: lone-warp ceiling of the circuit (no register cap)
  for (int b : {148, 296, 592}) run<1, 1, 1>(b, 500, d, din);
  for (int b : {148, 296, 592}) run<1, 1, 2>(b, 500, d, din);
  return 0;
#endif
  for (int b : {148, 1332}) run<1, 9, 1>(b, 2000, d, din);
  for (int b : {148, 296, 592, 1184}) run<1, 8, 4>(b, 2000, d, din);
  for (int b : {148, 296, 592, 1184}) run<1, 8, 6>(b, 2000, d, din);
  for (int b : {148, 296, 592, 1184}) run<1, 8, 7>(b, 2000, d, din);
  return 0;
}
