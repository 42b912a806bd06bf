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


// The same transpose with fewer ALU-pipe instructions (the kernels it serves are
// ALU-issue-bound): the 16- and 8-bit rounds are byte permutes (two PRMT per row
// pair instead of five shift / logic ops), and in the 4-, 2- and 1-bit rounds the
// shifts are multiplies on the FMA pipe (x << s = x * 2^s, x >> s = umulhi(x,
// 2^(32-s))) so only the three lop3 stay on the ALU pipe.  The powers of two
// must be run-time values (else ptxas turns the multiplies back into shifts):
// `one` is a kernel argument equal to 1.
__device__ __forceinline__ void transpose32_fma(uint32_t (&A)[32], uint32_t one) {
#pragma unroll
  for (int i = 0; i < 16; i++) {
    const uint32_t x = A[i], y = A[i + 16];
    A[i] = __byte_perm(x, y, 0x5410);
    A[i + 16] = __byte_perm(x, y, 0x7632);
  }
#pragma unroll
  for (int i = 0; i < 32; i++) {
    if (i & 8) continue;
    const uint32_t x = A[i], y = A[i + 8];
    A[i] = __byte_perm(x, y, 0x6240);
    A[i + 8] = __byte_perm(x, y, 0x7351);
  }
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const uint32_t m = s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u : 0x55555555u;
    const uint32_t up = one << s, down = one << (32 - s);  // 2^s, 2^(32-s)
#pragma unroll
    for (int i = 0; i < 32; i++) {
      if (i & s) continue;
      const uint32_t t = (__umulhi(A[i], down) ^ A[i + s]) & m;
      A[i + s] ^= t;
      A[i] ^= t * up;
    }
  }
}

// ---------------------------------------------------------------------------
// Bitsliced float32 <-> F(WE, WF) conversion on 32 lanes at once (the pack
// kernels and the conv's float32 epilogue): the conversion is done on bit
// planes with ~3 lop3 per output bit instead of ~20 scalar ops per element.
// Plane k of U = bit k of the 32 lanes' float32 words (after transpose32).

// Planes of (x + K) mod 2^NO for the NI-bit planes x and a constant K (ripple
// carry, the constant's bits folded: ~2 lop3 per bit).
template <int NI, int NO, unsigned K>
__device__ __forceinline__ void add_const_planes(const uint32_t* x, uint32_t* out) {
  uint32_t c = 0u;
#pragma unroll
  for (int i = 0; i < NO; i++) {
    const uint32_t xi = i < NI ? x[i] : 0u;
    const bool k = (K >> i) & 1u;
    out[i] = k ? ~(xi ^ c) : (xi ^ c);
    c = k ? (xi | c) : (xi & c);
  }
}

// float32 planes U[0..31] -> planes P[0..3+WE+WF-1] of F(WE, WF), rounded at the
// float's own binade (rnd 0: RNE, 1: RTZ) -- the same function as encode_f32_fast
// (WE <= 7: every float32 subnormal underflows to a signed zero; overflow -> inf
// with sign; NaN -> canonical NaN, L5/L6).
template <int WE, int WF>
__device__ __forceinline__ void encode_planes_f32(const uint32_t (&U)[32], int rnd, uint32_t* P) {
  static_assert(WE <= 7 && WF <= 22, "bitsliced encode: WE <= 7, WF <= 22");
  constexpr int SH = 23 - WF;  // mantissa bits dropped
  uint32_t sticky = 0u;
#pragma unroll
  for (int k = 0; k + 1 < SH; k++) sticky |= U[k];
  const uint32_t guard = U[SH - 1];
  const uint32_t inc = rnd == 0 ? (guard & (sticky | U[SH])) : 0u;
  // increment [kept mantissa (WF) | exponent (8)] by inc; R[WF..WF+7] = rounded exponent
  uint32_t R[WF + 8];
  uint32_t c = inc;
#pragma unroll
  for (int i = 0; i < WF + 8; i++) {
    R[i] = U[SH + i] ^ c;
    c = U[SH + i] & c;
  }
  // D = e8r - (127 - bias) as a 9-bit two's complement number: e8r + (512 - OFF)
  constexpr unsigned OFF = 127u - ((1u << (WE - 1)) - 1u);
  uint32_t D[9];
  add_const_planes<8, 9, (512u - OFF) & 511u>(R + WF, D);
  uint32_t hi = 0u;
#pragma unroll
  for (int i = WE; i < 8; i++) hi |= D[i];
  const uint32_t unf = D[8];
  const uint32_t ovf = ~D[8] & hi;
  uint32_t eand = U[23], eor = U[23], mor = 0u;
#pragma unroll
  for (int k = 24; k < 31; k++) { eand &= U[k]; eor |= U[k]; }
#pragma unroll
  for (int k = 0; k < 23; k++) mor |= U[k];
  const uint32_t nan = eand & mor;
  const uint32_t inf = (eand & ~mor) | (ovf & eor & ~eand);
  const uint32_t normal = eor & ~eand & ~ovf & ~unf;
#pragma unroll
  for (int j = 0; j < WF; j++) P[j] = R[j] & normal;
#pragma unroll
  for (int j = 0; j < WE; j++) P[WF + j] = D[j] & normal;
  P[WF + WE] = U[31] & ~nan;
  P[WF + WE + 1] = normal | nan;
  P[WF + WE + 2] = inf | nan;
}

// planes A[0..3+WE+WF-1] of canonical F(WE, WF) words -> float32 planes U[0..31]
// of their exact values (WE <= 7, WF <= 23): the same function as decode_f32
// (+-0, +-inf, NaN = 0x7FC00000).
template <int WE, int WF>
__device__ __forceinline__ void decode_planes_f32(const uint32_t* A, uint32_t (&U)[32]) {
  static_assert(WE <= 7 && WF <= 23, "bitsliced decode: WE <= 7, WF <= 23");
  const uint32_t c0 = A[WF + WE + 1], c1 = A[WF + WE + 2];
  const uint32_t normal = c0 & ~c1, nan = c0 & c1, spec = c1;  // spec: inf or NaN
#pragma unroll
  for (int k = 0; k < 23; k++) U[k] = 0u;
#pragma unroll
  for (int i = 0; i < WF; i++) U[23 - WF + i] = A[i] & normal;
  U[22] |= nan;
  constexpr unsigned OFF = 127u - ((1u << (WE - 1)) - 1u);
  uint32_t E[8];
  add_const_planes<WE, 8, OFF>(A + WF, E);
#pragma unroll
  for (int i = 0; i < 8; i++) U[23 + i] = (E[i] & normal) | spec;
  U[31] = A[WF + WE] & ~nan;
}
}  // namespace hobf
