// hobf_words.cuh -- per-element word helpers shared by the C-ABI kernels and the
// per-format conv kernels: activation records and the layer-epilogue
// re-rounding of a chained network.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hobf {

// Activation record (hobf_prepare_activations, hobf_conv2d_prepared): the
// canonical x word of F(we, wf) in bits [0, 20) and the weight-table row it
// selects in bits [20, 32): row = frac for a normal x, 2^wF + 0/1/2 for
// zero / inf / NaN (padding = +0 -> row 2^wF).
__device__ __forceinline__ uint32_t xrec_of(uint32_t x, int we, int wf) {
  const uint32_t exc = (x >> (wf + we + 1)) & 3u;
  const uint32_t row = exc == 1u ? (x & ((1u << wf) - 1u)) : ((1u << wf) + (exc == 0u ? 0u : exc - 1u));
  return x | (row << 20);
}

// Layer epilogue of a chained network ("rounding ... dealt with at the
// end of the layer in the activation function", P:265 layers kept in the
// custom format): a canonical word of F(we, wfi) re-rounded into the next
// layer's F(we, wfo), RNE (ties to even) or RTZ.  The exponent width is
// unchanged, so a normal stays normal unless rounding up leaves the top binade
// (-> inf, L5); widening (wfo >= wfi) is exact; zero / inf keep
// their sign, NaN stays the canonical NaN.
__device__ __forceinline__ uint32_t requant_word(uint32_t x, int we, int wfi, int wfo, int rnd) {
  const uint32_t exc = (x >> (wfi + we + 1)) & 3u;
  const uint32_t s = (x >> (wfi + we)) & 1u;
  const int top = wfo + we + 1;
  if (exc != 1u) return (exc << top) | ((exc == 3u ? 0u : s) << (wfo + we));
  uint32_t e = (x >> wfi) & ((1u << we) - 1u);
  uint32_t f = x & ((1u << wfi) - 1u);
  if (wfo >= wfi) {
    f <<= (wfo - wfi);
  } else {
    const int sh = wfi - wfo;
    const uint32_t rem = f & ((1u << sh) - 1u), half = 1u << (sh - 1);
    f >>= sh;
    if (rnd == 0 && (rem > half || (rem == half && (f & 1u)))) {
      if (++f == (1u << wfo)) {  // carried into the next binade
        f = 0u;
        if (++e == (1u << we)) return (2u << top) | (s << (wfo + we));  // overflow -> inf
      }
    }
  }
  return (1u << top) | (s << (wfo + we)) | (e << wfo) | f;
}

// Weight-table geometry (hobf_prepare_weights, hobf_conv2d_prepared).
// Entry planes NPT = roundup(wfo + (we + 2) + 3, 4); rows are stored with a
// stride of tab_stride(NPT, wf) words.  For the formats whose tables are staged
// in shared memory (wF <= 5) the stride is chosen so that stride / 4 is odd: the
// 16-byte segments of 8 consecutive rows then fall in 8 distinct bank quads,
// and a warp's 128-bit row gathers are (nearly) conflict-free.  Wider formats
// are served from L1/L2 and keep stride = NPT (their 2^wF + 3 rows make the
// tables large: C2's e5m10 tables must stay L2-resident).  Layout [ceil(cout/32)][cin][kh][kw][2^wF + 3 rows][stride]:
// everything one output-channel group needs for one input channel is one
// contiguous block (one bulk copy).
__host__ __device__ constexpr int tab_stride(int npt, int wf) {
  return (wf > 7 || ((npt / 4) & 1)) ? npt : npt + 4;
}

// F(we, wf) word -> float32 (exact for we <= 7, wf <= 23).  Branch-free: the
// four exception classes are selected, not branched on (no divergence).
__device__ __forceinline__ float decode_f32(uint32_t v, int we, int wf) {
  const uint32_t exc = (v >> (wf + we + 1)) & 3u;
  const uint32_t sbit = ((v >> (wf + we)) & 1u) << 31;
  const int E = (int)((v >> wf) & ((1u << we) - 1u)) - ((1 << (we - 1)) - 1);
  const uint32_t frac = v & ((1u << wf) - 1u);
  const uint32_t normal = sbit | ((uint32_t)(E + 127) << 23) | (frac << (23 - wf));
  const uint32_t special = exc == 3u ? 0x7FC00000u : (sbit | (exc == 2u ? 0x7F800000u : 0u));
  return __uint_as_float(exc == 1u ? normal : special);
}

// 32 x 32 bit-matrix transpose in registers (bit j of A[i] <-> bit i of A[j]):
// five rounds of block swaps, the s x s off-diagonal blocks of every 2s x 2s
// block exchanged with one shift and two xors per row pair.
__device__ __forceinline__ void transpose32(uint32_t (&A)[32]) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const uint32_t m = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u
                                                                                                   : 0x55555555u;
#pragma unroll
    for (int i = 0; i < 32; i++) {
      if (i & s) continue;
      const uint32_t t = ((A[i] >> s) ^ A[i + s]) & m;
      A[i + s] ^= t;
      A[i] ^= t << s;
    }
  }
}

}  // namespace hobf
