// hobf_kernels.cuh -- format-templated CUDA kernels of the hot path (sm_100a).
//
// Instantiated once per generated circuit (csrc/gen/hobf_fmt_*.cu).  F is a
// generated struct (csrc/gen/hobf_circuit_*.cuh) holding the format constants
// and the straight-line lop3 MAC / ReLU bodies.
//
// Plane layout (L18): a tensor [rows][C] of NBITS-bit words is
// stored as planes[rows][ceil(C/32)][NP], NP = roundup(NBITS, 4); bit l of
// word (r, g, j) is field bit j of element (r, 32g + l).  Padding lanes and
// planes are zero (= canonical +0).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <set>
#include <utility>

#include "hobf_internal.h"
#include "hobf_words.cuh"

namespace hobf {

// Broadcast bit b of w to all 32 lanes (0 or ~0) without touching the ALU
// pipe, which the lop3 gates saturate: (w * 2^(31-b)) puts bit b in the sign
// position (IMAD), and the high word of (that * one) as a signed 64-bit
// product is its sign extension (IMAD.HI).  `one` is a runtime 1 so that
// ptxas cannot turn the IMAD.HI into an ALU shift.
// 2^(31-b) for b = 0..31, read from constant memory so that the multiply
// stays an IMAD (a visible power of two would become an ALU shift).
__constant__ uint32_t c_lift[32] = {
    1u << 31, 1u << 30, 1u << 29, 1u << 28, 1u << 27, 1u << 26, 1u << 25, 1u << 24,
    1u << 23, 1u << 22, 1u << 21, 1u << 20, 1u << 19, 1u << 18, 1u << 17, 1u << 16,
    1u << 15, 1u << 14, 1u << 13, 1u << 12, 1u << 11, 1u << 10, 1u << 9,  1u << 8,
    1u << 7,  1u << 6,  1u << 5,  1u << 4,  1u << 3,  1u << 2,  1u << 1,  1u << 0};

__device__ __forceinline__ uint32_t bcast_bit(uint32_t w, uint32_t lift, int32_t one) {
  const int32_t t = (int32_t)(w * lift);
  return (uint32_t)__mulhi(t, one);
}

// (c, kh, kw) tap counter in the order of the reduction (c outermost, L10).
struct TapIter {
  int c = 0, kh = 0, kw = 0;
  __device__ __forceinline__ void next(int KH, int KW) {
    if (++kw == KW) {
      kw = 0;
      if (++kh == KH) { kh = 0; ++c; }
    }
  }
};

// Bit b of w as 0/1, on the FMA pipe: high word of (w * 2^(31-b)) * two, two = 2.
__device__ __forceinline__ uint32_t bit01(uint32_t w, uint32_t lift, uint32_t two) {
  return __umulhi(w * lift, two);
}

// ---------------------------------------------------------------------------
// Output epilogue shared by the conv kernels.  acc holds the canonical (and,
// if requested, ReLU'd) accumulator planes of output pixel pix (image ni, row
// oy, column ox), channels 32g + lane.
//   out_mode 0: the planes as they are, F(we, wfo) (NPO words, uint4 stores);
//   out_mode 1: every lane re-rounded into the next layer's F(we, next_wf)
//               (requant_word) and bitsliced again: the next layer's
//               input planes, no unpack in between;
//   out_mode 2: the same words written as the next layer's activation
//               records (zero-padded by next_pad; the caller's buffer holds
//               the +0 border), one coalesced 4-byte store per channel.
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ uint32_t lane_word(const uint32_t* acc, int l) {
  uint32_t x = 0u;
#pragma unroll
  for (int j = 0; j < F::NOUT; j++) x |= ((acc[j] >> l) & 1u) << j;
  return x;
}

template <class F>
__device__ __forceinline__ void store_requant(const uint32_t* acc, const ConvArgs& a, int64_t pix, int g, int ni,
                                           int oy, int ox) {
  const int G = (a.cout + 31) >> 5;
  const int nbn = 3 + F::WE + a.next_wf;
  if (a.out_mode == 1) {
    uint32_t P[32];
#pragma unroll
    for (int j = 0; j < 32; j++) P[j] = 0u;
#pragma unroll 1
    for (int l = 0; l < 32; l++) {
      if (32 * g + l >= a.cout) break;  // padding lanes stay +0 (all planes zero)
      const uint32_t w = requant_word(lane_word<F>(acc, l), F::WE, F::WFO, a.next_wf, F::RND);
#pragma unroll
      for (int j = 0; j < 32; j++) P[j] |= ((w >> j) & 1u) << l;
    }
    const int npn = (nbn + 3) / 4 * 4;
    uint4* py = reinterpret_cast<uint4*>(a.y + (pix * G + g) * npn);
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if (4 * q >= npn) break;
      py[q] = make_uint4(P[4 * q], P[4 * q + 1], P[4 * q + 2], P[4 * q + 3]);
    }
  } else {
    const int Hn = a.ho + 2 * a.next_pad, Wn = a.wo + 2 * a.next_pad;
    uint32_t* base = a.y + (((int64_t)ni * a.cout + 32 * g) * Hn + oy + a.next_pad) * Wn + ox + a.next_pad;
#pragma unroll 1
    for (int l = 0; l < 32; l++) {
      if (32 * g + l >= a.cout) break;
      const uint32_t w = requant_word(lane_word<F>(acc, l), F::WE, F::WFO, a.next_wf, F::RND);
      base[(int64_t)l * Hn * Wn] = xrec_of(w, F::WE, a.next_wf);
    }
  }
}

// out_mode 3 (HOBF_OUT_F32, the last layer): the 32 lanes' words, by a
// register bit transpose of the NOUT planes, decoded to their exact float32
// values and stored NHWC -- the 32 channels of the group are 128 contiguous
// bytes (eight 16-byte stores when cout % 4 == 0).  No plane round trip.
template <class F>
__device__ __forceinline__ void store_f32(const uint32_t* acc, const ConvArgs& a, int64_t pix, int g) {
  uint32_t U[32];
  decode_planes_f32<F::WE, F::WFO>(acc, U);  // float32 bit planes of the 32 lanes (bitsliced decode)
  transpose32_fma(U, (uint32_t)a.one);       // U[l] = float32 bits of lane l
  float* base = reinterpret_cast<float*>(a.y) + pix * a.cout + 32 * g;
  const int nl = min(32, a.cout - 32 * g);
  if ((a.cout & 3) == 0) {
#pragma unroll
    for (int q = 0; q < 8; q++) {
      if (4 * q >= nl) break;
      reinterpret_cast<uint4*>(base)[q] = make_uint4(U[4 * q], U[4 * q + 1], U[4 * q + 2], U[4 * q + 3]);
    }
  } else {
#pragma unroll
    for (int l = 0; l < 32; l++)
      if (l < nl) reinterpret_cast<uint32_t*>(base)[l] = U[l];
  }
}

template <class F>
__device__ __forceinline__ void store_out(const uint32_t* acc, const ConvArgs& a, int64_t pix, int g, int ni, int oy,
                                          int ox) {
  if (a.out_mode == 3) {
    if constexpr (F::WE <= 7) store_f32<F>(acc, a, pix, g);
    return;
  }
  if (a.out_mode != 0) {
    store_requant<F>(acc, a, pix, g, ni, oy, ox);
    return;
  }
  const int G = (a.cout + 31) >> 5;
  uint4* py = reinterpret_cast<uint4*>(a.y + (pix * G + g) * F::NPO);
#pragma unroll
  for (int q = 0; q < F::NPO / 4; q++) {
    uint4 v;
    v.x = (4 * q + 0 < F::NOUT) ? acc[(4 * q + 0) % F::NOUT] : 0u;
    v.y = (4 * q + 1 < F::NOUT) ? acc[(4 * q + 1) % F::NOUT] : 0u;
    v.z = (4 * q + 2 < F::NOUT) ? acc[(4 * q + 2) % F::NOUT] : 0u;
    v.w = (4 * q + 3 < F::NOUT) ? acc[(4 * q + 3) % F::NOUT] : 0u;
    py[q] = v;
  }
}

// ---------------------------------------------------------------------------
// conv2d: one thread = one output pixel x one group of 32 output channels.
// Lanes of every register are the 32 output channels (the paper's tiling of
// the M kernels by LANES); the activation value is broadcast across
// the lanes.  The accumulator (NOUT registers) stays in registers for
// the whole serial (c, kh, kw) reduction (L10); ReLU is fused (L12).
// ---------------------------------------------------------------------------
template <class F, int MINB = 1, bool K33 = false>
__global__ void __launch_bounds__(128, MINB) conv_direct_kernel(ConvArgs a) {
  const int G = (a.cout + 31) >> 5;
  const int CG = (a.cin + 31) >> 5;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.items) return;
  const int g = (int)(t % G);
  const int64_t pix = t / G;
  const int ox = (int)(pix % a.wo);
  const int oy = (int)((pix / a.wo) % a.ho);
  const int64_t ni = pix / ((int64_t)a.wo * a.ho);

  uint32_t acc[F::NOUT];
#pragma unroll
  for (int j = 0; j < F::NOUT; j++) acc[j] = 0u;  // +0 (L9)

  const uint32_t* __restrict__ xbase = a.x + ni * (int64_t)a.h * a.w * CG * F::NPI;
  const uint32_t* __restrict__ wbase = a.wt + (int64_t)g * F::NPI;
  const int64_t wstride_c = (int64_t)G * F::NPI;  // next input channel
  // one tap: the activation's planes broadcast from lane bit (c mod 32), the weight's planes
  auto tap = [&](int c, int kh, int kw) {
    const int cg = c >> 5;
    const uint32_t lift = c_lift[c & 31];  // bit c%32 -> bit 31 (multiply on the FMA pipe)
    const int iy = oy * a.stride - a.pad + kh, ix = ox * a.stride - a.pad + kw;
    uint32_t X[F::NPI];
    if (iy >= 0 && iy < a.h && ix >= 0 && ix < a.w) {
      const uint4* px = reinterpret_cast<const uint4*>(xbase + (((int64_t)iy * a.w + ix) * CG + cg) * F::NPI);
#pragma unroll
      for (int q = 0; q < F::NPI / 4; q++) {
        const uint4 v = __ldg(px + q);
        X[4 * q + 0] = v.x; X[4 * q + 1] = v.y; X[4 * q + 2] = v.z; X[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < F::NPI; j++) X[j] = bcast_bit(X[j], lift, a.one);  // broadcast
    } else {
#pragma unroll
      for (int j = 0; j < F::NPI; j++) X[j] = 0u;  // zero padding = +0 (L11, L14)
    }
    uint32_t W[F::NPI];
    const uint4* pw = reinterpret_cast<const uint4*>(wbase + ((int64_t)(kh * a.kw + kw) * a.cin + c) * wstride_c);
#pragma unroll
    for (int q = 0; q < F::NPI / 4; q++) {
      const uint4 v = __ldg(pw + q);
      W[4 * q + 0] = v.x; W[4 * q + 1] = v.y; W[4 * q + 2] = v.z; W[4 * q + 3] = v.w;
    }
    F::mac(acc, X, W);
  };
  if constexpr (K33) {  // the channel's nine taps in one unrolled body (more independent work in view)
#pragma unroll 1
    for (int c = 0; c < a.cin; c++) {
#pragma unroll
      for (int kh = 0; kh < 3; kh++)
#pragma unroll
        for (int kw = 0; kw < 3; kw++) tap(c, kh, kw);
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < a.cin; c++) {
#pragma unroll 1
      for (int kh = 0; kh < a.kh; kh++) {
#pragma unroll 1
        for (int kw = 0; kw < a.kw; kw++) tap(c, kh, kw);
      }
    }
  }
  if (a.relu) F::relu(acc, acc);
  store_out<F>(acc, a, pix, g, (int)ni, oy, ox);
}

// ---------------------------------------------------------------------------
// Depthwise conv2d (MobileNets "Conv dw"):
// output channel m reads only input channel m, so the 32 lanes of a register
// are 32 channels of BOTH operands -- the activation is bitsliced like the
// weight (no broadcast) and every lane runs its own full MAC (F::mac: the
// (wF+1)^2 multiplier array and the adder).  One thread = one output pixel x
// one group of 32 channels; the serial (kh, kw) chain stays in registers.
// x planes [n][h][w][G][NPI], w planes [kh][kw][G][NPI], G = ceil(C/32).
// ---------------------------------------------------------------------------
template <class F, int MINB = 1, bool K33 = false>
__global__ void __launch_bounds__(128, MINB) conv_dw_kernel(ConvArgs a) {
  const int G = (a.cout + 31) >> 5;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.items) return;
  const int g = (int)(t % G);
  const int64_t pix = t / G;
  const int ox = (int)(pix % a.wo);
  const int oy = (int)((pix / a.wo) % a.ho);
  const int ni = (int)(pix / ((int64_t)a.wo * a.ho));

  uint32_t acc[F::NOUT];
#pragma unroll
  for (int j = 0; j < F::NOUT; j++) acc[j] = 0u;  // +0 (L9)
  const uint32_t* __restrict__ xbase = a.x + ((int64_t)ni * a.h * a.w * G + g) * F::NPI;
  const uint32_t* __restrict__ wbase = a.wt + (int64_t)g * F::NPI;
  auto tap = [&](int kh, int kw) {
    const int iy = oy * a.stride - a.pad + kh, ix = ox * a.stride - a.pad + kw;
    uint32_t X[F::NPI], W[F::NPI];
    const bool inside = iy >= 0 && iy < a.h && ix >= 0 && ix < a.w;
    const uint4* px = reinterpret_cast<const uint4*>(xbase + ((int64_t)iy * a.w + ix) * G * F::NPI);
    const uint4* pw = reinterpret_cast<const uint4*>(wbase + (int64_t)(kh * a.kw + kw) * G * F::NPI);
#pragma unroll
    for (int q = 0; q < F::NPI / 4; q++) {
      const uint4 v = inside ? __ldg(px + q) : make_uint4(0u, 0u, 0u, 0u);  // padding = +0 (L11, L14)
      X[4 * q + 0] = v.x; X[4 * q + 1] = v.y; X[4 * q + 2] = v.z; X[4 * q + 3] = v.w;
      const uint4 u = __ldg(pw + q);
      W[4 * q + 0] = u.x; W[4 * q + 1] = u.y; W[4 * q + 2] = u.z; W[4 * q + 3] = u.w;
    }
    F::mac(acc, X, W);
  };
  if constexpr (K33) {  // the nine taps in one body: the loads of later taps issue early
#pragma unroll
    for (int kh = 0; kh < 3; kh++)
#pragma unroll
      for (int kw = 0; kw < 3; kw++) tap(kh, kw);
  } else {
#pragma unroll 1
    for (int kh = 0; kh < a.kh; kh++) {
#pragma unroll 1
      for (int kw = 0; kw < a.kw; kw++) tap(kh, kw);
    }
  }
  if (a.relu) F::relu(acc, acc);
  store_out<F>(acc, a, pix, g, ni, oy, ox);
}

// ---------------------------------------------------------------------------
// conv2d with prepared weights and prepared activations.
//
// The activation x is one scalar per thread (broadcast across the 32
// output-channel lanes), so its class and fraction select a row of the
// per-weight table built by hobf_prepare_weights (row = frac for a normal x,
// 2^wF + {0,1,2} for x = zero / inf / NaN; the table holds, for every lane,
// the rounded significand product, eb - bias + carry, the weight sign and the
// product class).  The remaining multiplier gates (activation exponent add,
// overflow / underflow, sign) and the whole adder run as generated lop3 code
// (F::mac_tab).
//
// Activations come as records (hobf_prepare_activations): one uint32 per
// element in a zero-padded [n][c][h+2p][w+2p] layout, holding the x word in
// bits [0, 20) and its table row in bits [20, 32).  Per tap a thread does one
// coalesced 4-byte load (consecutive threads = consecutive output columns),
// no bounds check (padding records are +0), and FMA-pipe work only: the row
// is IMAD.HI(rec, 2^12), the exponent / sign bits are broadcast with
// IMAD (rec * 2^(31-j)) + IMAD.HI (by 1); the ALU pipe is left to the gates.
// grid = (ceil(npix / 128), ceil(cout / 32)); one CTA = one group of 32
// output channels, so every warp of the CTA reads the same table block.
// ---------------------------------------------------------------------------
// Per-tap operands of the table MAC: broadcast activation exponent / sign
// planes (FMA pipe) and the table entry the activation's row selects.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// The TAB_W live planes of a table entry: 128-bit loads for full quads, a 64-
// and / or 32-bit load for the tail -- never a load into a dead register.  (A
// 128-bit load whose last register is dead lets ptxas reuse that register at
// once; the reuse then waits on the load in flight, which cost the latency-bound
// schedule half its speed.)  Planes past TAB_W are never read by the circuit.
template <class F, bool GLOBAL = true>
__device__ __forceinline__ void load_entry(uint32_t (&T)[F::NPT], const uint32_t* __restrict__ p, int zero) {
  constexpr int W = F::TAB_W;
  const uint4* p4 = reinterpret_cast<const uint4*>(p);
#pragma unroll
  for (int q = 0; q < W / 4; q++) {
    const uint4 v = GLOBAL ? __ldg(p4 + q) : p4[q];
    T[4 * q + 0] = v.x; T[4 * q + 1] = v.y; T[4 * q + 2] = v.z; T[4 * q + 3] = v.w;
  }
  // the tail as separate narrower loads; the last word's address goes through a
  // run-time zero so that neither the compiler nor ptxas can prove the loads
  // adjacent and merge them back into one 128-bit load with a dead register
  constexpr int b = W / 4 * 4;
  if constexpr (W - b >= 2) {
    const uint2* p2 = reinterpret_cast<const uint2*>(p + b);
    const uint2 v = GLOBAL ? __ldg(p2) : *p2;
    T[b] = v.x; T[b + 1] = v.y;
  }
  if constexpr ((W - b) & 1) {
    const uint32_t* pl = p + W - 1 + zero;
    T[W - 1] = GLOBAL ? __ldg(pl) : *pl;
  }
#pragma unroll
  for (int j = W; j < F::NPT; j++) T[j] = 0u;
}

template <class F>
struct TabTap {
  uint32_t EA[F::WE], SX[1], T[F::NPT];
  __device__ __forceinline__ void load(uint32_t rec, const uint32_t* __restrict__ tblock, const ConvArgs& a) {
    constexpr int WF = F::WF, WE = F::WE;
#pragma unroll
    for (int j = 0; j < WE; j++) EA[j] = (uint32_t)__mulhi((int32_t)(rec * a.lift[WF + j]), a.one);
    SX[0] = (uint32_t)__mulhi((int32_t)(rec * a.lift[WF + WE]), a.one);
    const uint32_t row = __umulhi(rec, a.row_mul);  // rec >> 20
    load_entry<F>(T, tblock + (int64_t)row * tab_stride(F::NPT, F::WF), a.one - 1);
  }
};

// KW3: kernel width fixed at 3 (inner loop unrolled); RU kernel rows per
// unrolled loop body.  PD > 0: software pipeline -- the table entries of taps
// t+1..t+PD and the record of tap t+PD+1 are in flight while the MAC of tap t
// runs (latency-bound configs, large tables).
// THR (variant 14, the float32 epilogue): a progress throttle.  The CTAs of a Cout
// group gather from the same table blocks; left alone they spread over more taps
// than L2 holds (profiles/r02_c5_e5m10_one_wave.txt).  Here thread 0 of a CTA
// publishes the number of input channels it has finished (a token in its own
// float32 output word, overwritten by the output at the end), and each warp, once
// per input channel, reads the tokens of 32 CTAs of its group and sleeps (bounded:
// 16 x 250 ns) while it is more than THR_D channels ahead of the slowest of them.
// Waits are bounded and words that are not tokens (CTAs not started, finished) are
// ignored, so the schedule cannot deadlock and the results do not depend on it.
constexpr uint32_t THR_TOKEN = 0xA5A50000u;
constexpr int THR_D = 2;

// COOP (variant 15): warp-cooperative table gathers.  A warp's 32 row gathers
// cost the L1 tag stage 32 lines per 128-bit load instruction (6 instructions per
// tap at wF = 9, 10).  Here 8 lanes copy the 16-byte chunks of one row (4 rows per
// instruction: ~4-8 lines) with cp.async into a per-warp shared-memory slot, a tap
// ahead, double-buffered; each thread then reads its own row back with 128-bit
// shared loads (row stride NPT + 4 words: conflict-free quads).  No table registers
// are held across the MAC.  Every lane computes (a lane past the last pixel on
// pixel 0) so that the warp-wide shuffles and barriers see all 32 lanes.
template <class F, int NT, int MINB, bool KW3, int PD, int RU = 1, bool THR = false, bool COOP = false>
__global__ void __launch_bounds__(NT, MINB) conv_tab_kernel(ConvArgs a) {
  // linear grid, output-channel group fastest: the G groups of a pixel tile run
  // together, so each activation record comes from DRAM once and is reused from L2
  const int G = (a.cout + 31) >> 5;
  const int g = (int)(blockIdx.x % G);
  const int64_t pix_t = (int64_t)(blockIdx.x / G) * blockDim.x + threadIdx.x;
  const bool valid = pix_t < (int64_t)a.n * a.ho * a.wo;
  if (!COOP && !valid) return;
  const int64_t pix = valid ? pix_t : 0;
  const int ox = (int)(pix % a.wo);
  const int oy = (int)((pix / a.wo) % a.ho);
  const int ni = (int)(pix / ((int64_t)a.wo * a.ho));
  const int Hp = a.h + 2 * a.pad, Wp = a.w + 2 * a.pad;
  const int KW = KW3 ? 3 : a.kw;

  uint32_t acc[F::NOUT];
#pragma unroll
  for (int j = 0; j < F::NOUT; j++) acc[j] = 0u;  // +0 (L9)

  // record of (ni, c, oy*stride + kh, ox*stride + kw) = rbase[c*Hp*Wp + kh*Wp + kw]
  const uint32_t* __restrict__ rbase =
      a.x + ((int64_t)ni * a.cin * Hp + (int64_t)oy * a.stride) * Wp + (int64_t)ox * a.stride;
  // table block (c, kh, kw) of group g: [g][c][kh][kw] blocks of TAB_ROWS x stride words (hobf_words.cuh)
  const int64_t tstride = (int64_t)F::TAB_ROWS * tab_stride(F::NPT, F::WF);
  const uint32_t* __restrict__ tbase = a.wt + (int64_t)g * a.cin * a.kh * KW * tstride;
  const int64_t cstride = (int64_t)Hp * Wp;
  auto rec_at = [&](int c, int kh, int kw) { return __ldg(rbase + c * cstride + kh * Wp + kw); };
  auto tblock = [&](int c, int kh, int kw) { return tbase + ((int64_t)c * a.kh * KW + kh * KW + kw) * tstride; };

  if constexpr (COOP) {
    constexpr int CH = F::NPT / 4, RS = F::NPT + 4;  // 16-byte chunks per row; padded slot row (words)
    static_assert(CH <= 8 && F::NPT % 4 == 0, "8 lanes copy one row");
    __shared__ __align__(16) uint32_t cbuf[NT / 32][2][32][RS];
    const int lane = (int)(threadIdx.x & 31), wrp = (int)(threadIdx.x >> 5);
    constexpr int rstride = tab_stride(F::NPT, F::WF);
    // lane = 8 s + m copies chunk m of the rows of lanes 8 s + q, q = 0..7: the row comes
    // by a width-8 shuffle (source lane q of the own 8-lane segment: an immediate), the
    // slot address is a per-thread base plus immediates, the source a 32-bit word offset
    // (IMADs on the FMA pipe) on the tap's uniform block pointer -- no ALU-pipe work
    const uint32_t m4 = 4u * (uint32_t)(lane & 7);
    const bool copies = (lane & 7) < CH;
    const uint32_t dst0 = smem_addr(&cbuf[wrp][0][lane & 24][4 * (lane & 7)]);
    auto issue = [&](uint32_t rec, const uint32_t* __restrict__ tb, int b) {
      const uint32_t row = __umulhi(rec, a.row_mul);  // rec >> 20
      const uint32_t dstb = dst0 + (uint32_t)b * (uint32_t)(32 * RS * 4);
#pragma unroll
      for (int q = 0; q < 8; q++) {
        const uint32_t r = __shfl_sync(0xffffffffu, row, q, 8);
        if (copies) {
          const uint32_t* src = tb + (r * (uint32_t)rstride + m4);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dstb + (uint32_t)(q * RS * 4)), "l"(src)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    const int taps = a.cin * a.kh * KW;
    TapIter tt, tr;  // tap of the next table rows to copy (t + 1) / of the next record to load (t + 2)
    uint32_t rc = rec_at(0, 0, 0);
    issue(rc, tblock(0, 0, 0), 0);
    tt.next(a.kh, KW);
    uint32_t rn = tt.c < a.cin ? rec_at(tt.c, tt.kh, tt.kw) : 0u;
    tr = tt;
    tr.next(a.kh, KW);
#pragma unroll 1
    for (int t = 0; t < taps; t++) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncwarp();
      uint32_t T[F::NPT], EA[F::WE], SX[1];
      const uint4* p4 = reinterpret_cast<const uint4*>(&cbuf[wrp][t & 1][lane][0]);
#pragma unroll
      for (int q = 0; q < CH; q++) {
        const uint4 v = p4[q];
        T[4 * q + 0] = v.x; T[4 * q + 1] = v.y; T[4 * q + 2] = v.z; T[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < F::WE; j++) EA[j] = (uint32_t)__mulhi((int32_t)(rc * a.lift[F::WF + j]), a.one);
      SX[0] = (uint32_t)__mulhi((int32_t)(rc * a.lift[F::WF + F::WE]), a.one);
      if (tt.c < a.cin) issue(rn, tblock(tt.c, tt.kh, tt.kw), (t + 1) & 1);
      tt.next(a.kh, KW);
      rc = rn;
      rn = tr.c < a.cin ? rec_at(tr.c, tr.kh, tr.kw) : 0u;
      tr.next(a.kh, KW);
      F::mac_tab(acc, T, EA, SX);
    }
  } else if constexpr (PD == 0 && KW3) {
    // the 3 records of the next kernel row are loaded while this row's 3 MACs run
    uint32_t rn[3];
#pragma unroll
    for (int kw = 0; kw < 3; kw++) rn[kw] = rec_at(0, 0, kw);
    int nc = 0, nkh = 0;
#pragma unroll RU
    for (int row = 0; row < a.cin * a.kh; row++) {
      const int c = nc, kh = nkh;
      uint32_t rc[3];
#pragma unroll
      for (int kw = 0; kw < 3; kw++) rc[kw] = rn[kw];
      if (++nkh == a.kh) { nkh = 0; ++nc; }
      if (nc < a.cin) {
#pragma unroll
        for (int kw = 0; kw < 3; kw++) rn[kw] = rec_at(nc, nkh, kw);
      }
#pragma unroll
      for (int kw = 0; kw < 3; kw++) {
        TabTap<F> tp;
        tp.load(rc[kw], tblock(c, kh, kw), a);
        F::mac_tab(acc, tp.T, tp.EA, tp.SX);
      }
    }
  } else if constexpr (PD == 0) {
#pragma unroll 1
    for (int c = 0; c < a.cin; c++) {
#pragma unroll 1
      for (int kh = 0; kh < a.kh; kh++) {
#pragma unroll
        for (int kw = 0; kw < KW; kw++) {
          TabTap<F> tp;
          tp.load(rec_at(c, kh, kw), tblock(c, kh, kw), a);
          F::mac_tab(acc, tp.T, tp.EA, tp.SX);
        }
      }
    }
  } else {
    if constexpr (NT == 32) {  // latency-bound (one warp per CTA): static rings, no register rotation
      // ring of R = PD + 1 operand slots: the MAC of tap t reads slot t % R while
      // the table entry of tap t + PD is loaded into slot (t + PD) % R, and the
      // record of tap t + PD + R (which that load will need R taps later) into
      // record slot (t + PD) % R.  The loop is unrolled by R so every slot index
      // is static (modulo variable expansion): no register move rotates a ring --
      // a move of a slot still being loaded would wait for the load and defeat
      // the prefetch.
      constexpr int R = PD + 1;
      const int taps = a.cin * a.kh * KW;
      TabTap<F> q[R];
      uint32_t rq[R];
      TapIter tt, tr;  // tap of the next table entry to load / of the next record to load
#pragma unroll
      for (int i = 0; i < PD; i++) {
        if (tt.c < a.cin) q[i].load(rec_at(tt.c, tt.kh, tt.kw), tblock(tt.c, tt.kh, tt.kw), a);
        tt.next(a.kh, KW);
      }
      tr = tt;
#pragma unroll
      for (int i = 0; i < R; i++) {  // records of taps PD .. PD + R - 1 -> slots (PD + i) % R
        rq[(PD + i) % R] = tr.c < a.cin ? rec_at(tr.c, tr.kh, tr.kw) : 0u;
        tr.next(a.kh, KW);
      }
      auto step = [&](TabTap<F>& use, TabTap<F>& fill, uint32_t& rslot) {
        if (tt.c < a.cin) fill.load(rslot, tblock(tt.c, tt.kh, tt.kw), a);
        tt.next(a.kh, KW);
        rslot = tr.c < a.cin ? rec_at(tr.c, tr.kh, tr.kw) : 0u;
        tr.next(a.kh, KW);
        F::mac_tab(acc, use.T, use.EA, use.SX);
      };
      int t = 0;
#pragma unroll 1
      for (; t + R <= taps; t += R) {
#pragma unroll
        for (int i = 0; i < R; i++) step(q[i], q[(i + PD) % R], rq[(i + PD) % R]);
      }
#pragma unroll
      for (int i = 0; i < R; i++)
        if (t + i < taps) step(q[i], q[(i + PD) % R], rq[(i + PD) % R]);
    } else {  // throughput configs with large tables: rotating ring (measured faster there)
      // ring of PD taps whose operands are loaded; the record of tap t+PD is one further ahead
      const int taps = a.cin * a.kh * KW;
      TabTap<F> q[PD > 0 ? PD : 1];
      TapIter tt, tr;  // tap of the next table entry to load / of the next record to load
#pragma unroll
      for (int i = 0; i < PD; i++) {
        if (tt.c < a.cin) q[i].load(rec_at(tt.c, tt.kh, tt.kw), tblock(tt.c, tt.kh, tt.kw), a);
        tt.next(a.kh, KW);
      }
      tr = tt;
      uint32_t rn = tr.c < a.cin ? rec_at(tr.c, tr.kh, tr.kw) : 0u;
      tr.next(a.kh, KW);
      [[maybe_unused]] int left = a.kh * KW, cdone = 0;
#pragma unroll 1
      for (int t = 0; t < taps; t++) {
        TabTap<F> cur = q[0];
#pragma unroll
        for (int i = 0; i + 1 < PD; i++) q[i] = q[i + 1];
        if (tt.c < a.cin) q[PD - 1].load(rn, tblock(tt.c, tt.kh, tt.kw), a);
        tt.next(a.kh, KW);
        rn = tr.c < a.cin ? rec_at(tr.c, tr.kh, tr.kw) : 0u;
        tr.next(a.kh, KW);
        F::mac_tab(acc, cur.T, cur.EA, cur.SX);
        if constexpr (THR) {
          if (--left == 0) {  // an input channel done
            left = a.kh * KW;
            ++cdone;
            const int tile = (int)(blockIdx.x / G), ntiles = (int)(gridDim.x / G);
            volatile uint32_t* slots = a.y + 32 * g + 31;  // word 31 of (pixel, group g)'s 32 floats
            if (threadIdx.x == 0) slots[(int64_t)tile * NT * a.cout] = THR_TOKEN | (uint32_t)cdone;
            const unsigned m = __activemask();
            const int lane = (int)(threadIdx.x & 31);
            const int peer = (tile + 1 + lane * max(1, ntiles / 32)) % ntiles;
            for (int k = 0; k < 16; k++) {
              const uint32_t v = slots[(int64_t)peer * NT * a.cout];
              const int prog = (v >> 16) == (THR_TOKEN >> 16) ? (int)(v & 0xffffu) : 0x7fffffff;
              if (cdone <= __reduce_min_sync(m, prog) + THR_D) break;
              __nanosleep(250);
            }
          }
        }
      }
    }
  }
  F::canon(acc, acc);  // the chain keeps a relaxed accumulator (fpgen.build_mac_tab)
  if (a.relu) F::relu(acc, acc);
  if (valid) store_out<F>(acc, a, pix, g, ni, oy, ox);
}

// ---------------------------------------------------------------------------
// Fractional-wave schedule of the L1-served kernel (variant 12, the float32
// epilogue): U work units (CTA tiles of 128 pixels x one Cout group) on W < U
// co-resident workers.  Run as variant 4, the E = U - W units past the wave
// would form a second, nearly empty wave that takes a whole chain's time at a
// few warps per SM (C5, wF = 10: 784 units on 740 slots).  Here every worker
// runs one unit (unit b) and, for E * S of them, one of S consecutive tap
// segments of an extra unit: such a worker does its own taps [0, sL),
// then segment s of an extra unit of its own Cout group (taps [sL, (s+1)L), the
// last segment to the end), then its own taps [sL, taps).  Segment s - 1 is done by the time
// segment s starts (both workers have run sL taps), so the chain of every
// extra unit moves through the S workers in its serial (c, kh, kw) order
// (L10): the same chain, the same result as one thread running it.
// Hand-off: the segment's accumulator planes are stored in the producing
// thread's own float32 output slot of the extra unit (32 words; NOUT <= 31),
// then a token (segment index) in the slot's word 31 after a fence; the next
// segment's thread spins on that word (acquire) and reads the planes through
// L2.  The host zeroes the extra units' slots before the launch, and the last
// segment overwrites them with the unit's float32 outputs.  Each worker's own
// accumulator waits in its own output slot during the extra segment (one
// accumulator in registers).  The launch is cooperative (every worker
// resident), so a waiting worker never holds a slot its producer needs.
// ---------------------------------------------------------------------------
template <class F>
__device__ __forceinline__ void tab_span(uint32_t (&acc)[F::NOUT], const ConvArgs& a, const uint32_t* __restrict__ rbase,
                                         const uint32_t* __restrict__ tbase, int t0, int t1) {
  if (t0 >= t1) return;
  const int Wp = a.w + 2 * a.pad;
  const int64_t cstride = (int64_t)(a.h + 2 * a.pad) * Wp;
  const int64_t tstride = (int64_t)F::TAB_ROWS * tab_stride(F::NPT, F::WF);
  const int kk = a.kh * a.kw;
  auto at = [&](int t) {
    TapIter it;
    it.c = t / kk;
    const int r = t - it.c * kk;
    it.kh = r / a.kw;
    it.kw = r - it.kh * a.kw;
    return it;
  };
  // one tap's operands in flight while the previous tap's MAC runs (variant 4's ring, PD = 1).
  // The loads past the span's end are not skipped: the tap iterators stop at the last
  // tap, which is re-read (unconditional loads).  A skipped load compiles to "reg = 0;
  // branch over the load", and that zeroing waits for the previous iteration's load
  // into the same register (measured: 42% of the warp samples on it).
  auto rec_ptr = [&](const TapIter& i) { return rbase + i.c * cstride + i.kh * Wp + i.kw; };
  auto tblock = [&](const TapIter& i) { return tbase + ((int64_t)i.c * kk + i.kh * a.kw + i.kw) * tstride; };
  TapIter tt = at(t0);  // tap of the next table entry to load, min(t + 1, t1 - 1)
  TabTap<F> q;
  q.load(__ldg(rec_ptr(tt)), tblock(tt), a);
  if (t0 + 1 < t1) tt.next(a.kh, a.kw);
  TapIter tr = tt;      // tap of the next record to load, min(t + 2, t1 - 1)
  uint32_t rn = __ldg(rec_ptr(tr));
  if (t0 + 2 < t1) tr.next(a.kh, a.kw);
#pragma unroll 1
  for (int t = t0; t < t1; t++) {
    TabTap<F> cur = q;
    q.load(rn, tblock(tt), a);
    if (t + 2 < t1) tt.next(a.kh, a.kw);
    rn = __ldg(rec_ptr(tr));
    if (t + 3 < t1) tr.next(a.kh, a.kw);
    F::mac_tab(acc, cur.T, cur.EA, cur.SX);
  }
}

constexpr uint32_t SPLIT_TOKEN = 0xA5A50000u;

template <class F, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) conv_tab_split_kernel(ConvArgs a) {
  static_assert(F::NOUT <= 31, "the hand-off slot holds NOUT planes and a token in 32 words");
  const int G = (a.cout + 31) >> 5;
  const int64_t npix = (int64_t)a.n * a.ho * a.wo;
  const int W = (int)gridDim.x, E = a.split_e, S = a.split_s, L = a.split_l;
  const int taps = a.cin * a.kh * a.kw;
  const int b = (int)blockIdx.x;
  const int Hp = a.h + 2 * a.pad, Wp = a.w + 2 * a.pad;
  const int64_t tstride = (int64_t)F::TAB_ROWS * tab_stride(F::NPT, F::WF);
  struct Unit {
    int64_t pix;
    int g;
    bool valid;
    const uint32_t* rbase;
    const uint32_t* tbase;
    uint32_t* slot;
  };
  auto unit = [&](int u) {
    Unit r;
    r.g = u % G;
    r.pix = (int64_t)(u / G) * NT + threadIdx.x;
    r.valid = r.pix < npix;
    const int64_t p = r.valid ? r.pix : 0;
    const int ox = (int)(p % a.wo), oy = (int)((p / a.wo) % a.ho), ni = (int)(p / ((int64_t)a.wo * a.ho));
    r.rbase = a.x + ((int64_t)ni * a.cin * Hp + (int64_t)oy * a.stride) * Wp + (int64_t)ox * a.stride;
    r.tbase = a.wt + (int64_t)r.g * a.cin * a.kh * a.kw * tstride;
    r.slot = a.y + p * a.cout + 32 * r.g;  // float32 output words of (pixel, group): 32 x 4 bytes
    return r;
  };
  auto finish = [&](uint32_t (&acc)[F::NOUT], const Unit& u) {
    F::canon(acc, acc);  // the chain keeps a relaxed accumulator (fpgen.build_mac_tab)
    if (a.relu) F::relu(acc, acc);
    if constexpr (F::WE <= 7) store_f32<F>(acc, a, u.pix, u.g);
  };
  // phases: 0 = own taps [0, x0) then the accumulator parked in the own output slot;
  // 1 = segment s of the extra unit, taps [x0, x1); 2 = own taps [x0, taps).  One loop,
  // so the circuit is emitted once and nothing but the accumulator lives across phases.
  // a worker takes segments of extra units of its own Cout group only (the
  // table rows it gathers are the ones its SM's other CTAs keep in L1): of group
  // g's workers (b = g + G r), rank r takes segment r / c of the group's extra
  // unit number r % c (c extra units in group g: W + i0 + G k, k < c)
  const int g = b % G, r = b / G;
  const int i0 = ((g - W) % G + G) % G;
  const int c = i0 < E ? (E - i0 + G - 1) / G : 0;
  const bool has_x = r < c * S;
  const int s = has_x ? r / c : 0;
  const int xu = has_x ? W + i0 + G * (r % c) : 0;
  const int x0 = has_x ? s * L : 0, x1 = s == S - 1 ? taps : x0 + L;
  // Phases, one loop (the circuit is emitted once; only the accumulator lives across
  // phases): 0 = own taps [0, x0), then -- while segment s - 1 has not handed its
  // accumulator on -- further own taps a kernel window (kh x kw) at a time, so no
  // worker idles on a spin, then the own accumulator parked in the own output slot
  // (tm taps done); 1 = segment s of the extra unit, taps [x0, x1); 2 = own taps
  // [tm, taps).  Every lane computes (a lane past the last pixel on pixel 0) so
  // the warp-wide ready vote sees all 32; stores and waits are per valid lane.
  const int chunk = a.kh * a.kw;
  const uint32_t want = SPLIT_TOKEN | (uint32_t)s;
  uint32_t acc[F::NOUT];
#pragma unroll
  for (int j = 0; j < F::NOUT; j++) acc[j] = 0u;  // +0 (L9)
  int ph = has_x ? 0 : 2, tm = 0;
#pragma unroll 1
  while (true) {
    int t0, t1;
    if (ph == 0) {
      if (tm >= x0) {
        bool ready = s == 0 || tm >= taps;
        if (!ready) {
          const Unit ex = unit(xu);
          uint32_t v = want;
          if (ex.valid) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ex.slot + 31) : "memory");
          ready = __all_sync(0xffffffffu, v == want);
        }
        if (ready) {
          const Unit me = unit(b);
          if (me.valid && tm > 0) {
#pragma unroll
            for (int j = 0; j < F::NOUT; j++) me.slot[j] = acc[j];
          }
          ph = 1;
          continue;
        }
        t0 = tm;
        t1 = min(tm + chunk, taps);
      } else {
        t0 = 0;
        t1 = x0;
      }
    } else if (ph == 1) {
      const Unit ex = unit(xu);
      if (s > 0 && ex.valid) {  // (only when the own taps ran out first) wait for the hand-off
        uint32_t v, ns = 64;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ex.slot + 31) : "memory");
          if (v == want) break;
          __nanosleep(ns);
          ns = min(2 * ns, 4096u);
        }
#pragma unroll
        for (int j = 0; j < F::NOUT; j++) acc[j] = __ldcg(ex.slot + j);
      } else {
#pragma unroll
        for (int j = 0; j < F::NOUT; j++) acc[j] = 0u;
      }
      t0 = x0;
      t1 = x1;
    } else {
      const Unit me = unit(b);
#pragma unroll
      for (int j = 0; j < F::NOUT; j++) acc[j] = tm > 0 && me.valid ? me.slot[j] : 0u;
      t0 = tm;
      t1 = taps;
    }
    const Unit u = unit(ph == 1 ? xu : b);
    tab_span<F>(acc, a, u.rbase, u.tbase, t0, t1);
    if (ph == 0) {
      tm = t1;
    } else if (ph == 1) {
      if (u.valid) {
        if (s < S - 1) {
#pragma unroll
          for (int j = 0; j < F::NOUT; j++) __stcg(u.slot + j, acc[j]);
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(u.slot + 31),
                       "r"(SPLIT_TOKEN | (uint32_t)(s + 1))
                       : "memory");
        } else {
          finish(acc, u);
        }
      }
      ph = 2;
    } else {
      if (u.valid) finish(acc, u);
      break;
    }
  }
}

// ---------------------------------------------------------------------------
// conv2d_prepared with the weight tables staged in shared memory.
//
// The per-thread table-row gathers are the part of the inner loop that costs
// ALU issue efficiency when served by L1 (sector misses, wavefront
// serialisation of 32 scattered 16-byte reads).  Here one CTA = one group of
// 32 output channels x NT output pixels; for each input channel c the CTA's
// whole table block [kh][kw][rows][stride] (hobf_words.cuh layout: one
// contiguous block per (group, channel)) is brought into shared memory by one
// TMA bulk copy (cp.async.bulk, completion on an mbarrier), double-buffered:
// the copy of channel c+1 is in flight while channel c's kh*kw MACs run.  The
// row stride makes a warp's 128-bit row gathers (nearly) bank-conflict-free.
// Records stay in global memory (one coalesced 4-byte load per tap, the next
// kernel row's records prefetched).  Same circuit, same serial (c, kh, kw)
// order as conv_tab_kernel: identical results.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// TMA bulk copy global -> shared (this CTA), completing `bytes` on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

template <class F>
constexpr int tab_block_words(int khw) {
  return khw * F::TAB_ROWS * tab_stride(F::NPT, F::WF);
}

// One tap of the staged-table MAC: broadcast planes of the record (FMA pipe),
// the row gather from shared memory, the generated circuit.
template <class F>
__device__ __forceinline__ void smem_tap(uint32_t* acc, uint32_t rec, const uint32_t* __restrict__ tblk,
                                         const ConvArgs& a) {
  constexpr int S = tab_stride(F::NPT, F::WF), WF = F::WF, WE = F::WE;
  uint32_t EA[WE], SX[1], T[F::NPT];
#pragma unroll
  for (int j = 0; j < WE; j++) EA[j] = (uint32_t)__mulhi((int32_t)(rec * a.lift[WF + j]), a.one);
  SX[0] = (uint32_t)__mulhi((int32_t)(rec * a.lift[WF + WE]), a.one);
  const uint32_t row = __umulhi(rec, a.row_mul);  // rec >> 20
  load_entry<F, false>(T, tblk + (int)row * S, a.one - 1);
  F::mac_tab(acc, T, EA, SX);
}

// CC input channels per staged buffer (one TMA bulk copy of CC contiguous
// channel blocks); K33: kh = kw = 3, the channel's nine taps fully unrolled.
// UT > 0 (K33 only): UT taps of one channel per staged buffer -- 3 = one kernel
// row, 1 = one tap -- for the formats whose channel block pair does not fit
// (wF >= 6; wF = 5 of the extended class): the flat unit k = (9 c + 3 kh + kw) / UT is the contiguous slice
// of UT taps of the group's block.
template <class F, int NT, int MINB, int CC, bool K33, int UT = 0>
__global__ void __launch_bounds__(NT, MINB) conv_tab_smem_kernel(ConvArgs a) {
  extern __shared__ __align__(128) uint32_t smem_tab[];  // [2][CC][kh*kw][rows][stride]
  __shared__ __align__(8) uint64_t full[2];
  constexpr int S = tab_stride(F::NPT, F::WF), R = F::TAB_ROWS;
  const int G = (a.cout + 31) >> 5;
  const int g = (int)(blockIdx.x % G);  // linear grid, output-channel group fastest (see conv_tab_kernel)
  const int64_t npix = (int64_t)a.n * a.ho * a.wo;
  const int64_t pix_raw = (int64_t)(blockIdx.x / G) * NT + threadIdx.x;
  const bool valid = pix_raw < npix;
  const int64_t pix = valid ? pix_raw : npix - 1;  // idle threads still join the CTA barriers
  const int ox = (int)(pix % a.wo);
  const int oy = (int)((pix / a.wo) % a.ho);
  const int ni = (int)(pix / ((int64_t)a.wo * a.ho));
  const int Hp = a.h + 2 * a.pad, Wp = a.w + 2 * a.pad;
  const int KH = K33 ? 3 : a.kh, KW = K33 ? 3 : a.kw, KHW = KH * KW;
  const uint32_t blk = (uint32_t)(KHW * R * S);  // words per (group, channel) block
  const uint32_t* __restrict__ gsrc = a.wt + (int64_t)g * a.cin * blk;
  const int nchunks = (a.cin + CC - 1) / CC;
  constexpr uint32_t UBLK = (uint32_t)UT * R * S;  // UT > 0: words per staged unit

  uint32_t acc[F::NOUT];
#pragma unroll
  for (int j = 0; j < F::NOUT; j++) acc[j] = 0u;  // +0 (L9)

  const uint32_t* __restrict__ rbase =
      a.x + ((int64_t)ni * a.cin * Hp + (int64_t)oy * a.stride) * Wp + (int64_t)ox * a.stride;
  const int64_t cstride = (int64_t)Hp * Wp;

  if (threadIdx.x == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int k) {  // chunk k -> buffer k & 1
    if (UT > 0) {
      mbar_expect_tx(&full[k & 1], UBLK * 4u);
      bulk_g2s(smem_tab + (k & 1) * UBLK, gsrc + (int64_t)k * UBLK, UBLK * 4u, &full[k & 1]);
      return;
    }
    const int c0 = k * CC, cc = min(CC, a.cin - c0);
    const uint32_t bytes = (uint32_t)cc * blk * 4u;
    mbar_expect_tx(&full[k & 1], bytes);
    bulk_g2s(smem_tab + (k & 1) * CC * blk, gsrc + (int64_t)c0 * blk, bytes, &full[k & 1]);
  };
  if (threadIdx.x == 0) issue(0);
  uint32_t rn[3];  // K33: records of the next kernel row
  if (K33) {
#pragma unroll
    for (int kw = 0; kw < 3; kw++) rn[kw] = __ldg(rbase + kw);
  }
  if (UT > 0) {
    static_assert(UT == 0 || (K33 && (UT == 1 || UT == 3)), "unit staging: 3x3 kernels, a row or a tap per unit");
    const int nunits = a.cin * (9 / (UT > 0 ? UT : 1));
    // one staged unit: refill the other buffer, wait for this one, its taps, barrier
    auto unit = [&](int k, const uint32_t* rc) {
      if (threadIdx.x == 0 && k + 1 < nunits) {
        // buffer (k+1)&1 was last read in unit k-1, which ended with a CTA barrier
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(k + 1);
      }
      mbar_wait(&full[k & 1], (uint32_t)(k >> 1) & 1u);
      const uint32_t* __restrict__ tb = smem_tab + (k & 1) * UBLK;
#pragma unroll
      for (int t = 0; t < UT; t++) smem_tap<F>(acc, rc[t], tb + t * R * S, a);
      __syncthreads();  // buffer k&1 is refilled at unit k+2's issue
    };
#pragma unroll 1
    for (int c = 0; c < a.cin; c++) {
      const uint32_t* __restrict__ rc_base = rbase + c * cstride;
#pragma unroll
      for (int kh = 0; kh < 3; kh++) {
        uint32_t rc[3];
#pragma unroll
        for (int kw = 0; kw < 3; kw++) rc[kw] = rn[kw];
        if (kh < 2 || c + 1 < a.cin) {
          const uint32_t* nrow = kh < 2 ? rc_base + (kh + 1) * Wp : rc_base + cstride;
#pragma unroll
          for (int kw = 0; kw < 3; kw++) rn[kw] = __ldg(nrow + kw);
        }
        if (UT == 3) {
          unit(3 * c + kh, rc);
        } else {
#pragma unroll
          for (int kw = 0; kw < 3; kw++) unit(9 * c + 3 * kh + kw, rc + kw);
        }
      }
    }
  }
#pragma unroll 1
  for (int k = 0; k < (UT > 0 ? 0 : nchunks); k++) {
    if (threadIdx.x == 0 && k + 1 < nchunks) {
      // buffer (k+1)&1 was last read in chunk k-1, which ended with a CTA barrier
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + 1);
    }
    mbar_wait(&full[k & 1], (uint32_t)(k >> 1) & 1u);
    const uint32_t* __restrict__ tbuf = smem_tab + (k & 1) * CC * blk;
    const int c0 = k * CC, cc = min(CC, a.cin - c0);
#pragma unroll 1
    for (int ci = 0; ci < cc; ci++) {
      const int c = c0 + ci;
      const uint32_t* __restrict__ tb = tbuf + ci * blk;
      const uint32_t* __restrict__ rc_base = rbase + c * cstride;
      if (K33) {
#pragma unroll
        for (int kh = 0; kh < 3; kh++) {
          uint32_t rc[3];
#pragma unroll
          for (int kw = 0; kw < 3; kw++) rc[kw] = rn[kw];
          // next kernel row: same channel, or the next channel's first row
          if (kh < 2 || c + 1 < a.cin) {
            const uint32_t* nrow = kh < 2 ? rc_base + (kh + 1) * Wp : rc_base + cstride;
#pragma unroll
            for (int kw = 0; kw < 3; kw++) rn[kw] = __ldg(nrow + kw);
          }
#pragma unroll
          for (int kw = 0; kw < 3; kw++) smem_tap<F>(acc, rc[kw], tb + (kh * 3 + kw) * R * S, a);
        }
      } else {
#pragma unroll 1
        for (int kh = 0; kh < KH; kh++) {
#pragma unroll 1
          for (int kw = 0; kw < KW; kw++)
            smem_tap<F>(acc, __ldg(rc_base + kh * Wp + kw), tb + (kh * KW + kw) * R * S, a);
        }
      }
    }
    __syncthreads();  // buffer k&1 is refilled at chunk k+2's issue (iteration k+1)
  }
  if (!valid) return;
  F::canon(acc, acc);  // the chain keeps a relaxed accumulator (fpgen.build_mac_tab)
  if (a.relu) F::relu(acc, acc);
  store_out<F>(acc, a, pix, g, ni, oy, ox);
}

// mac_planes: acc[i] = add(acc[i], mul(a[i], b[i])) lane-wise on plane groups.
template <class F>
__global__ void __launch_bounds__(256) mac_planes_kernel(uint32_t* __restrict__ acc_p, const uint32_t* __restrict__ a_p,
                                                         const uint32_t* __restrict__ b_p, int64_t n_groups) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_groups; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t acc[F::NPO], x[F::NPI], w[F::NPI];
#pragma unroll
    for (int j = 0; j < F::NPO; j++) acc[j] = acc_p[i * F::NPO + j];
#pragma unroll
    for (int j = 0; j < F::NPI; j++) { x[j] = a_p[i * F::NPI + j]; w[j] = b_p[i * F::NPI + j]; }
    F::mac(acc, x, w);
#pragma unroll
    for (int j = 0; j < F::NPO; j++) acc_p[i * F::NPO + j] = (j < F::NOUT) ? acc[j] : 0u;
  }
}

// Opt a kernel in to up to 200 KB of dynamic shared memory, once per (kernel,
// device): the attribute is per function and per device, so a process that
// launches several instantiations or uses several GPUs sets each one.
inline void allow_big_smem(const void* kern) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({kern, dev}).second)
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
}

// Launch `kern`, or -- when a.info is set (hobf_conv_kernel_info) -- only record
// which kernel and launch shape the schedule chose.
template <class K>
cudaError_t run(const ConvArgs& a, K kern, dim3 grid, int threads, size_t smem, cudaStream_t s, int variant) {
  if (a.info) {
    a.info->func = (const void*)kern;
    a.info->variant = variant;
    a.info->threads = threads;
    a.info->smem = smem;
    a.info->blocks = (int64_t)grid.x * grid.y * grid.z;
    return cudaSuccess;
  }
  if (smem > 48 * 1024) allow_big_smem((const void*)kern);
  kern<<<grid, threads, smem, s>>>(a);
  return cudaGetLastError();
}

template <class F>
cudaError_t launch_conv(const ConvArgs& a, cudaStream_t s) {
  if (a.items == 0) return cudaSuccess;
  const int threads = 128;
  const int64_t blocks = (a.items + threads - 1) / threads;
  // 3x3: the channel's nine taps in one body; CTAs per SM (register budget) by
  // mantissa width, measured on C3's shape: wF <= 6 5 (<= 96 registers: e5m5 0.67 ->
  // 0.70 of the roof vs 6), wF = 7, 8 6 (<= 80), wF >= 9 4 (<= 128: e5m10 0.60 -> 0.66)
  constexpr int GM = F::WF >= 9 ? 4 : (F::WF >= 7 ? 6 : 5);
  if (a.kh == 3 && a.kw == 3)
    return run(a, conv_direct_kernel<F, GM, true>, dim3((unsigned)blocks), threads, 0, s, 0);
  else
    return run(a, conv_direct_kernel<F>, dim3((unsigned)blocks), threads, 0, s, 0);
}

// Warps on the busiest SM when CTAs of nt threads run at most 2 per SM (in rounds).
inline int64_t busiest_2per(int64_t npix, int64_t gy, int nt) {
  const int64_t blocks = (npix + nt - 1) / nt * gy;
  return (blocks + 147) / 148 * (nt / 32);
}
inline int64_t busiest352(int64_t npix, int64_t gy) { return busiest_2per(npix, gy, 352); }
inline int64_t busiest256(int64_t npix, int64_t gy) { return busiest_2per(npix, gy, 256); }

// Fractional-wave launch (conv_tab_split_kernel at MB CTAs per SM).  done = false: the
// shape does not call for it (no overhang, too few workers per extra unit) or the
// device cannot co-schedule the workers -- nothing ran, the caller launches variant 4.
template <class F, int MB>
cudaError_t launch_split(const ConvArgs& a, cudaStream_t s, int64_t npix, unsigned gy, bool& done) {
  done = false;
  auto kern = conv_tab_split_kernel<F, 128, MB>;
  int dev = 0, sms = 0, nb = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 128, 0) != cudaSuccess) {
    done = true;
    return cudaGetLastError();
  }
  const int64_t W = (int64_t)nb * sms, U = (npix + 127) / 128 * gy, E = U - W;
  const int taps = a.cin * a.kh * a.kw;
  // segments per extra unit: every group's workers cover its extra units S times
  int64_t S = E > 0 ? 16 : 0;
  for (int64_t g = 0; g < gy && E > 0; g++) {
    const int64_t i0 = ((g - W) % gy + gy) % gy, c = i0 < E ? (E - i0 + gy - 1) / gy : 0;
    if (c > 0) S = std::min<int64_t>(S, ((W - g + gy - 1) / gy) / c);
  }
  if (!(E > 0 && S >= 2 && taps >= S)) return cudaSuccess;
  done = true;
  if (a.info) return run(a, kern, dim3((unsigned)W), 128, 0, s, MB == 4 && a.variant != 12 ? 13 : 12);
  ConvArgs b = a;
  b.split_e = (int)E;
  b.split_s = (int)S;
  b.split_l = (int)(taps / S);
  // zero the extra units' output slots (the hand-off tokens start cleared)
  const int64_t p0 = W / gy * 128;
  cudaError_t err = cudaMemsetAsync(b.y + p0 * a.cout, 0, (size_t)((npix - p0) * a.cout) * 4, s);
  if (err != cudaSuccess) return err;
  void* args[] = {&b};
  err = cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)W), dim3(128), args, 0, s);
  // a device / context that cannot co-schedule the W workers (MPS partition, no
  // cooperative launch): nothing ran, fall back to variant 4 (same results)
  if (err != cudaErrorCooperativeLaunchTooLarge && err != cudaErrorNotSupported && err != cudaErrorNotPermitted)
    return err;
  (void)cudaGetLastError();
  if (a.variant == 12 || a.variant == 13) return err;  // forced by the caller: report it
  done = false;
  return cudaSuccess;
}

template <class F>
cudaError_t launch_conv_tab(const ConvArgs& a, cudaStream_t s) {
  const int64_t npix = (int64_t)a.n * a.ho * a.wo;
  if (npix == 0) return cudaSuccess;
  const unsigned gy = (unsigned)((a.cout + 31) / 32);
  auto grid = [&](int threads) { return dim3((unsigned)((npix + threads - 1) / threads * gy)); };
  const bool k3 = a.kw == 3;
  int variant = a.variant;
  const int64_t warps = (npix + 31) / 32 * gy;
  // shared-memory table staging (variant 7): one channel block per buffer, double-
  // buffered; the pair must fit 50 KB so that 4 (256-thread) CTAs share an SM
  const int64_t blk_bytes = (int64_t)tab_block_words<F>(a.kh * a.kw) * 4;
  const bool k33 = k3 && a.kh == 3;
  const bool smem_ok = 2 * blk_bytes <= 50 * 1024;
  // unit staging (variant 8, 3x3, wF >= 6, or 5 extended): a kernel row per buffer when the pair
  // fits 64 KB (wF = 6, 7), else one tap per buffer (pair <= 100 KB: wF = 8, 9)
  const int64_t row_bytes = blk_bytes / 3, tap_bytes = blk_bytes / 9;
  const int ut = 2 * row_bytes <= 64 * 1024 ? 3 : (2 * tap_bytes <= 100 * 1024 ? 1 : 0);
  const bool units_ok = k33 && F::WF >= 5 && F::WF <= 9 && ut > 0;  // (wF = 5: extended class)
  if (variant == 0) {
    // auto: with fewer warps than 2 per SMSP the reduction chains are latency-bound:
    // one-warp CTAs (so every SM gets work) running the software-pipelined kernel;
    // otherwise the tables staged in shared memory -- a channel block per buffer when
    // the pair fits (wF <= 5 for 3x3), a kernel row or a tap (wF = 6-9, 3x3) --, else
    // the L1-served kernels: prefetching one tap ahead when the table rows do not stay
    // L1 resident (wF >= 6, measured on C5), or three kernel rows per unrolled loop
    // body at <= 64 registers.
    // (measured on the strong-split shares of C3 / C4 / C5 / MOB, profiles/r02_shapes_*.txt:
    // with the tables staged, even 392 warps run better staged than latency-scheduled --
    // C5 e5m3 at 8 images 0.49 vs 0.35, C3 at 4 images 0.51 vs 0.41)
    variant = (smem_ok && warps >= 148) ? 7
              : warps < 148 * 4 * 2 ? 5 : smem_ok ? 7 : units_ok ? 8 : (F::WF >= 6 ? 4 : (k3 ? 6 : 3));
  }
  if constexpr (F::WF == 9 && F::NOUT >= 19 && F::NOUT <= 31 && F::WE <= 7) {
    // e6m9: its tap-staged kernel holds 2 CTAs / SM and measured 0.66 / 0.65 of the roof
    // (RNE / RTZ) on C5, the L1-served fractional wave at 4 CTAs / SM 0.69 / 0.68
    // (profiles/r02_c5_split13_wf89.txt; e4m9 / e5m9, NOUT = 17 / 18: staged 0.75 vs 0.62)
    if (a.variant == 0 && variant == 8 && ut == 1 && 6 * tap_bytes > 216 * 1024 && a.out_mode == 3 &&
        (a.cout & 31) == 0) {
      bool done = false;
      const cudaError_t err = launch_split<F, 4>(a, s, npix, gy, done);
      if (done) return err;
    }
  }
  int shape = 0;  // variants 10 / 11: variant 7 with the CTA shape forced (256 x 3 / 128 x 6)
  if (variant >= 10 && variant <= 11) {
    shape = variant;
    variant = 7;
  }
  if (variant == 8 && !units_ok) variant = 7;
  if (variant == 7 && !smem_ok) variant = 6;
  if (variant == 8) {
    if constexpr (F::WF >= 5 && F::WF <= 9) {
      const int64_t ub = ut == 3 ? row_bytes : tap_bytes;
      auto go = [&](auto kern) { return run(a, kern, grid(256), 256, (size_t)(2 * ub), s, 8); };
      // 256-thread CTAs, 3 per SM (80 registers; measured on C5: 4 per SM at 64
      // registers, 512-thread CTAs and per-channel staging at 2 CTAs / SM are slower)
      if (ut == 3) return go(conv_tab_smem_kernel<F, 256, 3, 1, true, 3>);
      if (6 * ub <= 216 * 1024) return go(conv_tab_smem_kernel<F, 256, 3, 1, true, 1>);
      // two CTAs per SM: 352-thread CTAs hold 22 warps per SM, so a layer of up to
      // 148 x 22 warps (C5: 3136) runs as one wave instead of 1.32 waves of 256-thread CTAs
      if (busiest352(npix, gy) < busiest256(npix, gy))
        return run(a, conv_tab_smem_kernel<F, 352, 2, 1, true, 1>, grid(352), 352, (size_t)(2 * ub), s, 8);
      return go(conv_tab_smem_kernel<F, 256, 2, 1, true, 1>);
    }
    return cudaGetLastError();
  }
  if (variant == 7) {
    // CTA shape: 128 threads x 6 per SM or 256 x 3 (both <= 80 registers, 24 warps per SM),
    // whichever puts fewer warps on the busiest SM (ceil(CTAs / 148) x warps per CTA),
    // ties to 256.  Measured (profiles/r02_shapes_*.txt): C3 (44 vs 48 warps) 0.84 vs 0.77,
    // C4 0.89, MOB / C5 (24 vs 24) 0.78 vs 0.76; strong-split shares: C3 at 8 images
    // (12 vs 16) 0.70 vs 0.55, C5 at 32 (12 vs 16) 0.74 vs 0.57.
    auto busiest = [&](int nt) { return ((npix + nt - 1) / nt * gy + 147) / 148 * (nt / 32); };
    int cfg = (busiest(128) < busiest(256) && 12 * blk_bytes <= 216 * 1024) ? 6 : 7;
    if (shape == 10) cfg = 7;
    if (shape == 11 && 12 * blk_bytes <= 216 * 1024) cfg = 6;
    auto go = [&](auto kern, int nt, int cc) { return run(a, kern, grid(nt), nt, (size_t)(2 * cc * blk_bytes), s, 7); };
    if (k33) {
      if (cfg == 6) {
        // two input channels per staged buffer when the pairs still fit 6 CTAs / SM:
        // one CTA barrier per two channels
        if (24 * blk_bytes <= 216 * 1024) return go(conv_tab_smem_kernel<F, 128, 6, 2, true>, 128, 2);
        return go(conv_tab_smem_kernel<F, 128, 6, 1, true>, 128, 1);
      }
      if (12 * blk_bytes <= 216 * 1024) return go(conv_tab_smem_kernel<F, 256, 3, 2, true>, 256, 2);
      return go(conv_tab_smem_kernel<F, 256, 3, 1, true>, 256, 1);
    }
    return go(conv_tab_smem_kernel<F, 256, 4, 1, false>, 256, 1);
  }
  if (variant == 6 && k3) {  // KW=3, 3 kernel rows (one input channel) per unrolled body, <= 64 registers
    return run(a, conv_tab_kernel<F, 128, 8, true, 0, 3>, grid(128), 128, 0, s, 6);
  } else if (variant == 5) {  // latency-bound: 32-thread CTAs spread over all SMs
    return run(a, conv_tab_kernel<F, 32, 1, false, 3>, grid(32), 32, 0, s, 5);
  } else if (variant == 4 || (variant >= 12 && variant <= 15)) {  // software-pipelined (large tables / latency-bound configs)
    constexpr int M4 = F::G_TAB > 400 ? 4 : 5;
    if constexpr (F::NOUT <= 31 && F::WE <= 7) {
      // variants 12 / 13 (the default for variant 4's launches with the float32 epilogue
      // when the units overhang one wave): the fractional-wave schedule,
      // conv_tab_split_kernel, at M4 (12) or 4 (13) CTAs / SM.  Automatic: 4 CTAs / SM
      // (128 registers) from NOUT = 19, where the 96-register kernel spills inside the
      // tap loop (C5 e6m10 0.63 -> 0.69, e5m10 0.67 -> 0.69, e6m9 0.66 -> 0.69 of the
      // roof; e4m10, NOUT = 18, no spills: 0.64 at 5 vs 0.625 at 4;
      // profiles/r02_c5_split13.txt)
      if ((variant == 12 || variant == 13 || a.variant == 0) && a.out_mode == 3 && (a.cout & 31) == 0) {
        bool done = false;
        bool four = variant == 13 || (a.variant == 0 && F::NOUT >= 19);
        if (four && a.variant == 0 && M4 > 4) {
          // units that fit one wave of variant 4's own M4 CTAs / SM run there (C5 e5m10 at
          // 60 images, 736 units on 740 slots: 0.73 of the roof vs 0.65 split over 592)
          int dev = 0, sms = 0, nb = 0;
          if (cudaGetDevice(&dev) == cudaSuccess &&
              cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess &&
              cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, conv_tab_kernel<F, 128, M4, false, 1>, 128, 0) ==
                  cudaSuccess &&
              (int64_t)(npix + 127) / 128 * gy <= (int64_t)nb * sms)
            four = false;  // (launch_split then finds no overhang and variant 4 runs)
        }
        const cudaError_t err = four ? launch_split<F, 4>(a, s, npix, gy, done)
                                     : launch_split<F, M4>(a, s, npix, gy, done);
        if (done) return err;
      }
    }
    if constexpr (F::NPT % 4 == 0 && F::NPT <= 32) {
      if (variant == 15) return run(a, conv_tab_kernel<F, 128, M4, false, 1, 1, false, true>, grid(128), 128, 0, s, 15);
    }
    if (variant == 14 && a.out_mode == 3 && (a.cout & 31) == 0 && a.cin < 65536)
      return run(a, conv_tab_kernel<F, 128, M4, false, 1, 1, true>, grid(128), 128, 0, s, 14);
    // <= 96 registers, 5 CTAs / SM (C3 e5m10 0.79 -> 0.81, C5 wF = 10 +0-3% vs 128 registers);
    // the extended class's largest circuits (> 400 lop3) get 128 (4 CTAs / SM)
    return run(a, conv_tab_kernel<F, 128, M4, false, 1>, grid(128), 128, 0, s, 4);
  } else if (k3) {     // kernel width 3 unrolled, <= 56 registers (9 CTAs / SM)
    return run(a, conv_tab_kernel<F, 128, 9, true, 0>, grid(128), 128, 0, s, 3);
  }
  return run(a, conv_tab_kernel<F, 128, 9, false, 0>, grid(128), 128, 0, s, 3);
}

template <class F>
cudaError_t launch_conv_dw(const ConvArgs& a, cudaStream_t s) {
  if (a.items == 0) return cudaSuccess;
  const int threads = 128;
  const unsigned blocks = (unsigned)((a.items + threads - 1) / threads);
  // 3x3: nine taps in one body at <= 128 registers (MOBDW conv 0.63 -> 0.65 of the roof;
  // 5 or 6 CTAs / SM at 96 / 80 registers: 0.62 / 0.63)
  if (a.kh == 3 && a.kw == 3) return run(a, conv_dw_kernel<F, 4, true>, dim3(blocks), threads, 0, s, 0);
  return run(a, conv_dw_kernel<F>, dim3(blocks), threads, 0, s, 0);
}

template <class F>
cudaError_t launch_mac(uint32_t* acc, const uint32_t* x, const uint32_t* w, int64_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  mac_planes_kernel<F><<<(unsigned)blocks, 256, 0, s>>>(acc, x, w, n);
  return cudaGetLastError();
}

}  // namespace hobf

#define HOBF_INSTANTIATE(TAG, WE, WF, RND)                                                                   \
  cudaError_t hobf_launch_conv_##TAG(const hobf::ConvArgs& a, cudaStream_t s) {                            \
    return hobf::launch_conv<hobf_gen::F_##TAG>(a, s);                                                      \
  }                                                                                                         \
  cudaError_t hobf_launch_mac_##TAG(uint32_t* acc, const uint32_t* x, const uint32_t* w, int64_t n,        \
                                    cudaStream_t s) {                                                       \
    return hobf::launch_mac<hobf_gen::F_##TAG>(acc, x, w, n, s);                                            \
  }                                                                                                         \
  cudaError_t hobf_launch_convtab_##TAG(const hobf::ConvArgs& a, cudaStream_t s) {                         \
    return hobf::launch_conv_tab<hobf_gen::F_##TAG>(a, s);                                                  \
  }                                                                                                         \
  cudaError_t hobf_launch_convdw_##TAG(const hobf::ConvArgs& a, cudaStream_t s) {                          \
    return hobf::launch_conv_dw<hobf_gen::F_##TAG>(a, s);                                                   \
  }
