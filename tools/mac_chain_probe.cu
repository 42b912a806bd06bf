// Development probe: ALU-pipe efficiency of the generated table-MAC circuit
// with every operand in registers (no loads, no address arithmetic), i.e. the
// ceiling the conv kernel could reach with perfect operand delivery.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2007_06563_b200/csrc \
//        -I paper_2007_06563_b200/csrc/gen -o /tmp/mac_chain_probe tools/mac_chain_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "hobf_circuit_e5m3_rne.cuh"

using F = hobf_gen::F_e5m3_rne;

// MODE 0: operands mutated in registers; 1: + EA/SX mutated too (no hoisting);
// 2: + table entry gathered from an L1-resident table every MAC (like the conv).
template <int NG, int MINB, int MODE>
__global__ void __launch_bounds__(128, MINB) chain(uint32_t* out, const uint32_t* in, int iters, uint32_t m) {
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
    if (MODE >= 1) {
#pragma unroll
      for (int j = 0; j < F::WE; j++) EA[j] = EA[j] * m + 0x7F4A7C15u;
      SX[0] = SX[0] * m + 1u;
    }
    if (MODE == 2) {
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
  cudaMalloc(&din, 32 * 64 * 4 * 16);
  static uint32_t h[32 * 64 * 16];
  for (int i = 0; i < 32 * 64 * 16; i++) h[i] = 0x9E3779B9u * (i + 1);
  cudaMemcpy(din, h, sizeof(h), cudaMemcpyHostToDevice);
  for (int b : {148, 296, 592, 1332}) run<1, 9, 0>(b, 2000, d, din);
  for (int b : {148, 296, 592, 1332}) run<1, 9, 1>(b, 2000, d, din);
  for (int b : {148, 296, 592, 1332}) run<1, 9, 2>(b, 2000, d, din);
  for (int b : {148, 296, 592}) run<2, 4, 2>(b, 1000, d, din);
  return 0;
}
