// hobf_capi.cu -- the C ABI (include/hobf.h) and the format-generic kernels:
// bitslice pack / quantise+pack / unpack / unpack-to-float32, and the LOP3
// issue-rate microbenchmark.  Per-format conv / MAC kernels live in the
// generated translation units (csrc/gen/hobf_fmt_*.cu) and are reached
// through the dispatch table below.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>

#include "../../include/hobf.h"
#include "hobf_internal.h"
#include "hobf_words.cuh"

using hobf::ConvArgs;
using hobf::FormatEntry;
using hobf::xrec_of;
using hobf::decode_f32;
using hobf::transpose32;
using hobf::transpose32_fma;

#define HOBF_DECLARE(TAG)                                                                    \
  cudaError_t hobf_launch_conv_##TAG(const hobf::ConvArgs& a, cudaStream_t s);               \
  cudaError_t hobf_launch_mac_##TAG(uint32_t* acc, const uint32_t* x, const uint32_t* w, int64_t n, \
                                    cudaStream_t s);                                         \
  cudaError_t hobf_launch_convtab_##TAG(const hobf::ConvArgs& a, cudaStream_t s);            \
  cudaError_t hobf_launch_convdw_##TAG(const hobf::ConvArgs& a, cudaStream_t s);
#define HOBF_ENTRY(TAG, WE, WF, RND, EXT, GM, GMUL, GADD, GRELU, GTAB) \
  {WE, WF, RND, EXT, GM, GMUL, GADD, GRELU, GTAB, hobf_launch_conv_##TAG, hobf_launch_mac_##TAG, hobf_launch_convtab_##TAG, \
   hobf_launch_convdw_##TAG},
#include "gen/hobf_table.inc"

static const FormatEntry kFormats[] = {HOBF_TABLE_ENTRIES};
static const int kNumFormats = (int)(sizeof(kFormats) / sizeof(kFormats[0]));

static thread_local int32_t g_last_launches = 0;

static const FormatEntry* find_format(int we, int wf, int rnd, int ext) {
  for (int i = 0; i < kNumFormats; i++)
    if (kFormats[i].we == we && kFormats[i].wf == wf && kFormats[i].rnd == rnd && kFormats[i].ext == ext)
      return &kFormats[i];
  return nullptr;
}

static inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
static inline bool fmt_ok(int we, int wf) { return we >= 2 && we <= 8 && wf >= 1 && 3 + we + wf <= 32; }

// ----------------------------------------------------------------------------- device helpers

// Canonical form: mask to NBITS; exc != 01 -> exp = frac = 0; NaN -> sign 0.
__device__ __forceinline__ uint32_t canon_word(uint32_t v, int we, int wf) {
  const int nb = 3 + we + wf;
  v &= (nb >= 32) ? 0xffffffffu : ((1u << nb) - 1u);
  const uint32_t exc = (v >> (wf + we + 1)) & 3u;
  if (exc != 1u) v &= ~((1u << (wf + we)) - 1u);
  if (exc == 3u) v &= ~(1u << (wf + we));
  return v;
}

// float32 -> F(we, wf): exact value M*2^e of the float,
// rounded at its own binade (RNE ties-to-even or RTZ), then overflow -> inf,
// underflow (biased exponent < 0) -> zero keeping the sign (L5/L6).
__device__ __forceinline__ uint32_t encode_f32(float f, int we, int wf, int rnd) {
  // Branch-free (activations mix zeros, normals and the odd special within a
  // warp): the finite nonzero path is always computed and the special classes
  // are selected over it.
  const uint32_t u = __float_as_uint(f);
  const uint32_t sign = u >> 31;
  const int ex = (int)((u >> 23) & 0xFFu);
  const uint32_t man = u & 0x7FFFFFu;
  const int top = wf + we + 1;
  const uint32_t sfield = sign << (wf + we);
  const uint32_t M = ex ? (man | 0x800000u) : man;  // exact value M * 2^e
  const int e = ex ? ex - 150 : -149;
  const int k = 31 - __clz(M | 1u);                  // M = 1.xxx * 2^k (M = 0 is selected away below)
  const int sh = k - wf;                             // bits below the kept fraction
  const int shr = sh > 0 ? sh : 0;
  const uint32_t qd = M >> shr;
  const uint32_t rem = M & ((1u << shr) - 1u);
  const uint32_t half = sh > 0 ? 1u << (sh - 1) : 0u;
  const bool up = rnd == 0 && sh > 0 && (rem > half || (rem == half && (qd & 1u)));
  uint32_t q = sh > 0 ? qd + (up ? 1u : 0u) : (M << (-sh));
  int E = e + k + ((1 << (we - 1)) - 1);
  const bool carry = q == (2u << wf);
  q = carry ? q >> 1 : q;
  E += carry ? 1 : 0;
  const uint32_t inf = (2u << top) | sfield;
  const uint32_t normal = (1u << top) | sfield | ((uint32_t)E << wf) | (q - (1u << wf));
  const uint32_t finite = E > (1 << we) - 1 ? inf : (E < 0 ? sfield : normal);
  const uint32_t nonfinite = man ? (3u << top) : inf;
  return ex == 0xFF ? nonfinite : ((ex == 0 && man == 0) ? sfield : finite);
}

// float32 -> F(we, wf) for we <= 7, wf <= 22 (the activation quantiser's fast
// path; same results as encode_f32): the rounding to wf fraction bits is done on
// the float32 bit pattern itself (RNE: add half - 1 + lsb below the cut, then
// truncate -- a carry out of the mantissa moves into the float exponent, i.e.
// the value rounds up into the next binade), then the exponent is re-biased and
// range-checked (overflow -> inf, underflow -> zero keeping the sign; every
// float32 subnormal underflows because the format's emin >= -63 here).
__device__ __forceinline__ uint32_t encode_f32_fast(float f, int we, int wf, int rnd) {
  const uint32_t u = __float_as_uint(f);
  const int sh = 23 - wf;
  const uint32_t lsb = (u >> sh) & 1u;
  const uint32_t ur = rnd == 0 ? u + ((1u << (sh - 1)) - 1u) + lsb : u;
  const int ex = (int)((u >> 23) & 0xFFu);
  const int E = (int)((ur >> 23) & 0xFFu) - 127 + ((1 << (we - 1)) - 1);
  const int top = wf + we + 1;
  const uint32_t sfield = (u >> 31) << (wf + we);
  const uint32_t frac = (ur >> sh) & ((1u << wf) - 1u);
  const uint32_t inf = (2u << top) | sfield;
  const uint32_t finite = E > (1 << we) - 1 ? inf
                        : (E < 0 || ex == 0) ? sfield : (1u << top) | sfield | ((uint32_t)E << wf) | frac;
  const uint32_t nonfinite = (u & 0x7FFFFFu) ? (3u << top) : inf;
  return ex == 0xFF ? nonfinite : finite;
}

// ----------------------------------------------------------------------------- pack / unpack
// One warp per (row, 32-lane group): lane l holds element 32g+l; plane j is
// the warp ballot of bit j.  Coalesced 128-byte word reads and
// 4*NP-byte plane writes.

template <bool FROM_F32>
__global__ void __launch_bounds__(256) pack_kernel(const void* __restrict__ src, int64_t rows, int64_t C, int we,
                                                   int wf, int rnd, int np, uint32_t* __restrict__ planes) {
  const int lane = threadIdx.x & 31;
  const int64_t G = (C + 31) >> 5;
  const int64_t items = rows * G;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool dense = (C & 31) == 0;  // element (r, 32g + l) is then at it * 32 + l: no division
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items; it += nw) {
    int64_t idx;
    bool ok = true;
    if (dense) {
      idx = it * 32 + lane;
    } else {
      const int64_t r = it / G;
      const int64_t c = (it - r * G) * 32 + lane;
      ok = c < C;
      idx = r * C + c;
    }
    uint32_t v = 0u;
    if (ok) {
      if (FROM_F32) {
        const float xf = __ldg(reinterpret_cast<const float*>(src) + idx);
        v = we <= 7 ? encode_f32_fast(xf, we, wf, rnd) : encode_f32(xf, we, wf, rnd);
      }
      else
        v = canon_word(__ldg(reinterpret_cast<const uint32_t*>(src) + idx), we, wf);
    }
    uint32_t mine = 0u;
    for (int j = 0; j < np; j++) {
      const uint32_t bal = __ballot_sync(0xffffffffu, (v >> j) & 1u);
      if (lane == j) mine = bal;
    }
    if (lane < np) planes[it * np + lane] = mine;
  }
}

template <bool TO_F32>
__global__ void __launch_bounds__(256) unpack_kernel(const uint32_t* __restrict__ planes, int64_t rows, int64_t C,
                                                     int we, int wf, int np, void* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t G = (C + 31) >> 5;
  const int64_t items = rows * G;
  const int nb = 3 + we + wf;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool dense = (C & 31) == 0;  // element (r, 32g + l) is then at it * 32 + l: no division
  // UNR groups per warp iteration: their plane loads are all in flight before the
  // shuffles (the loop body is otherwise one dependent load -> shfl -> store chain).
  constexpr int UNR = 4;
  for (int64_t it0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * UNR; it0 < items; it0 += nw * UNR) {
    uint32_t mine[UNR];
#pragma unroll
    for (int u = 0; u < UNR; u++) mine[u] = (lane < np && it0 + u < items) ? __ldg(planes + (it0 + u) * np + lane) : 0u;
#pragma unroll
    for (int u = 0; u < UNR; u++) {
      const int64_t it = it0 + u;
      if (it >= items) break;
      uint32_t v = 0u;
      for (int j = nb - 1; j >= 0; j--) {  // bit j of v = bit `lane` of plane j
        const uint32_t pj = __shfl_sync(0xffffffffu, mine[u], j);
        v = (v << 1) | ((pj >> lane) & 1u);
      }
      int64_t idx;
      bool ok = true;
      if (dense) {
        idx = it * 32 + lane;
      } else {
        const int64_t r = it / G;
        const int64_t c = (it - r * G) * 32 + lane;
        ok = c < C;
        idx = r * C + c;
      }
      if (ok) {
        if (TO_F32)
          reinterpret_cast<float*>(dst)[idx] = decode_f32(v, we, wf);
        else
          reinterpret_cast<uint32_t*>(dst)[idx] = v;
      }
    }
  }
}

// Unpack, one thread per 32-lane group (the fast path): the group's NP plane
// words arrive by 128-bit loads (consecutive threads = consecutive groups:
// coalesced), a register transpose turns planes into the 32 lanes' words, and
// the 32 outputs leave as eight 128-bit stores.  No shuffles, no division.
// Used when C is a multiple of 32 (dense rows) and dst is 16-byte aligned.
template <bool TO_F32, int NP>
__global__ void __launch_bounds__(256) unpack_t_kernel(const uint32_t* __restrict__ planes, int64_t items, int we,
                                                       int wf, void* __restrict__ dst, uint32_t one) {
  const int nb = 3 + we + wf;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    uint32_t A[32];
    const uint4* src = reinterpret_cast<const uint4*>(planes + it * NP);
#pragma unroll
    for (int q = 0; q < NP / 4; q++) {
      const uint4 v = __ldg(src + q);
      A[4 * q] = v.x; A[4 * q + 1] = v.y; A[4 * q + 2] = v.z; A[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int j = NP; j < 32; j++) A[j] = 0u;
#pragma unroll
    for (int j = 0; j < NP; j++)
      if (j >= nb) A[j] = 0u;  // padding planes are zero anyway; keep the words exact
    transpose32_fma(A, one);
    uint4* out = reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(dst) + it * 32);
#pragma unroll
    for (int q = 0; q < 8; q++) {
      uint4 o;
      if (TO_F32) {
        o.x = __float_as_uint(decode_f32(A[4 * q], we, wf));
        o.y = __float_as_uint(decode_f32(A[4 * q + 1], we, wf));
        o.z = __float_as_uint(decode_f32(A[4 * q + 2], we, wf));
        o.w = __float_as_uint(decode_f32(A[4 * q + 3], we, wf));
      } else {
        o = make_uint4(A[4 * q], A[4 * q + 1], A[4 * q + 2], A[4 * q + 3]);
      }
      out[q] = o;
    }
  }
}

template <bool TO_F32>
static void launch_unpack_t(int np, const uint32_t* planes, int64_t items, int we, int wf, void* dst,
                            cudaStream_t s) {
  int64_t blocks = (items + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  const unsigned b = (unsigned)(blocks < 1 ? 1 : blocks);
  switch (np) {
    case 8: unpack_t_kernel<TO_F32, 8><<<b, 256, 0, s>>>(planes, items, we, wf, dst, 1u); break;
    case 12: unpack_t_kernel<TO_F32, 12><<<b, 256, 0, s>>>(planes, items, we, wf, dst, 1u); break;
    case 16: unpack_t_kernel<TO_F32, 16><<<b, 256, 0, s>>>(planes, items, we, wf, dst, 1u); break;
    case 20: unpack_t_kernel<TO_F32, 20><<<b, 256, 0, s>>>(planes, items, we, wf, dst, 1u); break;
    case 24: unpack_t_kernel<TO_F32, 24><<<b, 256, 0, s>>>(planes, items, we, wf, dst, 1u); break;
    case 28: unpack_t_kernel<TO_F32, 28><<<b, 256, 0, s>>>(planes, items, we, wf, dst, 1u); break;
    default: unpack_t_kernel<TO_F32, 32><<<b, 256, 0, s>>>(planes, items, we, wf, dst, 1u); break;
  }
}

// Pack, one thread per 32-lane group (the fast path for dense rows): the 32
// consecutive source elements arrive as eight 128-bit loads, are encoded /
// canonicalised in registers, and the register bit transpose turns the 32 words
// into the group's plane words, stored as NP / 4 128-bit stores.
template <bool FROM_F32, int NP>
__global__ void __launch_bounds__(256) pack_t_kernel(const void* __restrict__ src, int64_t items, int we, int wf,
                                                     int rnd, uint32_t* __restrict__ planes, uint32_t one) {
  const int nb = 3 + we + wf;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    uint32_t A[32];
    const uint4* in = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(src) + it * 32);
#pragma unroll
    for (int q = 0; q < 8; q++) {
      const uint4 v = __ldg(in + q);
      A[4 * q] = v.x; A[4 * q + 1] = v.y; A[4 * q + 2] = v.z; A[4 * q + 3] = v.w;
    }
#pragma unroll
    for (int l = 0; l < 32; l++) {
      if (FROM_F32) {
        const float xf = __uint_as_float(A[l]);
        A[l] = we <= 7 ? encode_f32_fast(xf, we, wf, rnd) : encode_f32(xf, we, wf, rnd);
      } else {
        A[l] = canon_word(A[l], we, wf);
      }
    }
    transpose32_fma(A, one);  // A[j] = plane j: bit l = field bit j of lane l
    uint4* out = reinterpret_cast<uint4*>(planes + it * NP);
#pragma unroll
    for (int q = 0; q < NP / 4; q++) {
      uint4 o;
      o.x = 4 * q < nb ? A[4 * q] : 0u;
      o.y = 4 * q + 1 < nb ? A[4 * q + 1] : 0u;
      o.z = 4 * q + 2 < nb ? A[4 * q + 2] : 0u;
      o.w = 4 * q + 3 < nb ? A[4 * q + 3] : 0u;
      out[q] = o;
    }
  }
}

// float32 -> planes for the formats of the generated table (we 4-6, wf 2-10): the
// 32 floats are transposed first and encoded in bitsliced form
// (hobf::encode_planes_f32: ~3 lop3 per output plane instead of ~20 scalar ops
// per element), so the kernel moves its bytes at close to HBM speed.
template <int WE, int WF>
__global__ void __launch_bounds__(256, 2) pack_f32_bs_kernel(const float* __restrict__ src, int64_t items, int rnd,
                                                             uint32_t* __restrict__ planes, uint32_t one) {
  constexpr int NB = 3 + WE + WF, NP = (NB + 3) / 4 * 4;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // software pipeline over the grid-stride loop: the next group's 128 bytes are in
  // flight while this group is transposed and encoded
  uint4 nx[8];
  auto load = [&](int64_t i) {
    const uint4* in = reinterpret_cast<const uint4*>(src + i * 32);
#pragma unroll
    for (int q = 0; q < 8; q++) nx[q] = __ldg(in + q);
  };
  // the warp's 32 groups are 4 KB of contiguous source: lane 0 also asks L2 for the
  // block two iterations ahead in one bulk prefetch (whole DRAM rows instead of the
  // scattered 16-byte pieces the per-lane loads request first)
  const int lane = threadIdx.x & 31;
  auto prefetch = [&](int64_t i0) {
    if (lane == 0 && i0 < items) {
      const int64_t bytes = std::min<int64_t>(32, items - i0) * 128;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + i0 * 32), "r"((uint32_t)bytes)
                   : "memory");
    }
  };
  const int64_t w0 = it - lane;  // first group of this warp
  prefetch(w0 + step);
  if (it < items) load(it);
  for (; it < items; it += step) {
    uint32_t U[32];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      U[4 * q] = nx[q].x; U[4 * q + 1] = nx[q].y; U[4 * q + 2] = nx[q].z; U[4 * q + 3] = nx[q].w;
    }
    prefetch(it - lane + 2 * step);
    if (it + step < items) load(it + step);
    transpose32_fma(U, one);  // U[k] = bit k of the 32 floats
    uint32_t P[NP];
#pragma unroll
    for (int j = NB; j < NP; j++) P[j] = 0u;
    hobf::encode_planes_f32<WE, WF>(U, rnd, P);
    uint4* out = reinterpret_cast<uint4*>(planes + it * NP);
#pragma unroll
    for (int q = 0; q < NP / 4; q++) out[q] = make_uint4(P[4 * q], P[4 * q + 1], P[4 * q + 2], P[4 * q + 3]);
  }
}

template <int WE, int WF>
static void go_pack_bs(unsigned, const void* src, int64_t items, int rnd, uint32_t* planes, cudaStream_t s) {
  // one wave of 2 CTAs per SM, every thread looping over several groups (pipelined)
  const int64_t b = std::min<int64_t>((items + 255) / 256, 148 * 2);
  pack_f32_bs_kernel<WE, WF><<<(unsigned)std::max<int64_t>(b, 1), 256, 0, s>>>(reinterpret_cast<const float*>(src),
                                                                               items, rnd, planes, 1u);
}

template <int WE>
static bool pack_bs_we(int wf, unsigned b, const void* src, int64_t items, int rnd, uint32_t* planes,
                       cudaStream_t s) {
  switch (wf) {
    case 2: go_pack_bs<WE, 2>(b, src, items, rnd, planes, s); return true;
    case 3: go_pack_bs<WE, 3>(b, src, items, rnd, planes, s); return true;
    case 4: go_pack_bs<WE, 4>(b, src, items, rnd, planes, s); return true;
    case 5: go_pack_bs<WE, 5>(b, src, items, rnd, planes, s); return true;
    case 6: go_pack_bs<WE, 6>(b, src, items, rnd, planes, s); return true;
    case 7: go_pack_bs<WE, 7>(b, src, items, rnd, planes, s); return true;
    case 8: go_pack_bs<WE, 8>(b, src, items, rnd, planes, s); return true;
    case 9: go_pack_bs<WE, 9>(b, src, items, rnd, planes, s); return true;
    case 10: go_pack_bs<WE, 10>(b, src, items, rnd, planes, s); return true;
  }
  return false;
}

static bool launch_pack_bs(int we, int wf, unsigned b, const void* src, int64_t items, int rnd, uint32_t* planes,
                           cudaStream_t s) {
  if (we == 4) return pack_bs_we<4>(wf, b, src, items, rnd, planes, s);
  if (we == 5) return pack_bs_we<5>(wf, b, src, items, rnd, planes, s);
  if (we == 6) return pack_bs_we<6>(wf, b, src, items, rnd, planes, s);
  return false;
}

template <bool FROM_F32>
static void launch_pack_t(int np, const void* src, int64_t items, int we, int wf, int rnd, uint32_t* planes,
                          cudaStream_t s) {
  int64_t blocks = (items + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  const unsigned b = (unsigned)(blocks < 1 ? 1 : blocks);
  if (FROM_F32 && launch_pack_bs(we, wf, b, src, items, rnd, planes, s)) return;
  switch (np) {
    case 8: pack_t_kernel<FROM_F32, 8><<<b, 256, 0, s>>>(src, items, we, wf, rnd, planes, 1u); break;
    case 12: pack_t_kernel<FROM_F32, 12><<<b, 256, 0, s>>>(src, items, we, wf, rnd, planes, 1u); break;
    case 16: pack_t_kernel<FROM_F32, 16><<<b, 256, 0, s>>>(src, items, we, wf, rnd, planes, 1u); break;
    case 20: pack_t_kernel<FROM_F32, 20><<<b, 256, 0, s>>>(src, items, we, wf, rnd, planes, 1u); break;
    case 24: pack_t_kernel<FROM_F32, 24><<<b, 256, 0, s>>>(src, items, we, wf, rnd, planes, 1u); break;
    case 28: pack_t_kernel<FROM_F32, 28><<<b, 256, 0, s>>>(src, items, we, wf, rnd, planes, 1u); break;
    default: pack_t_kernel<FROM_F32, 32><<<b, 256, 0, s>>>(src, items, we, wf, rnd, planes, 1u); break;
  }
}

static unsigned warp_grid(int64_t items) {
  int64_t blocks = (items + 7) / 8;  // 8 warps per 256-thread block
  const int64_t cap = 148 * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

// ----------------------------------------------------------------------------- weight tables
// Largest wF with a prepared-weights (table) kernel; the table has 2^wF + 3 rows.
static const int kTabMaxWf = 10;

// entry planes: product fraction (wfo = wF+1, or 2wF+1 extended) | Epart (wE+2) | S | K0 | K1
// Product-class encoding of an entry: one-hot flags (zero, normal, inf, NaN) when
// the two extra planes fit the 16-byte-rounded entry, else the 2-bit code K1 K0
// (gen/fpgen.tab_onehot states the same rule for the circuit that reads it).
__host__ __device__ static inline bool tab_onehot(int we, int wfo) {
  const int base = wfo + (we + 2) + 3;
  return (base + 2 + 3) / 4 == (base + 3) / 4;
}
__host__ __device__ static inline int tab_width(int we, int wfo) {
  return wfo + (we + 2) + (tab_onehot(we, wfo) ? 5 : 3);
}
__host__ __device__ static inline int tab_rows(int wf) { return (1 << wf) + 3; }

// One table entry for weight word w (canonical) and table row r (see
// conv_tab_kernel / gen/fpgen.product_from_table):
//   bits [0, wF+1)         rounded product fraction (round to wF+1 bits at the
//                          product's own binade, RNE ties-to-even or RTZ)
//   bits [wF+1, wF+wE+3)   Epart = eb - bias + (normalise carry + round carry),
//                          wE+2-bit two's complement; the conv adds ea
//   bit  wF+wE+3           weight sign (the conv XORs the activation sign)
//   bits wF+wE+4, +5       product class K0, K1 (00 zero, 01 normal, 10 inf,
//                          11 NaN), exception algebra of S:68 / SURVEY 8(c) mul;
//                          or (tab_onehot) bits +4..+7 = zero, normal, inf, NaN flags
// Rows: r < 2^wF: normal x with fraction r; 2^wF: x zero; +1: x inf; +2: x NaN.
// Extended class (wfo = 2wF+1): the product fraction is exact (no rounding).
__device__ uint32_t tab_entry(uint32_t w, int r, int we, int wf, int wfo, int rnd) {
  const int EW = we + 2;
  const uint32_t exc = (w >> (wf + we + 1)) & 3u;
  const uint32_t sw = (w >> (wf + we)) & 1u;
  const uint32_t eb = (w >> wf) & ((1u << we) - 1u);
  const uint32_t fb = w & ((1u << wf) - 1u);
  const int sbit = wfo + EW, k0 = sbit + 1, k1 = sbit + 2;
  const bool oh = tab_onehot(we, wfo);  // one-hot: Tzero sbit+1, Tnorm +2, Tinf +3, Tnan +4
  const uint32_t NAN_E = oh ? (1u << (sbit + 4)) : ((1u << k0) | (1u << k1));
  const uint32_t INF_E = (oh ? (1u << (sbit + 3)) : (1u << k1)) | (sw << sbit);
  const uint32_t ZERO_E = (oh ? (1u << (sbit + 1)) : 0u) | (sw << sbit);
  const uint32_t NORM_FLAG = oh ? (1u << (sbit + 2)) : (1u << k0);
  const int nrows = 1 << wf;
  if (r == nrows) return (exc & 2u) ? NAN_E : ZERO_E;                  // x = 0: 0*inf, 0*NaN = NaN
  if (r == nrows + 1) return (exc == 0u || exc == 3u) ? NAN_E : INF_E;  // x = inf: inf*0 = NaN
  if (r == nrows + 2) return NAN_E;                                    // x = NaN
  if (exc == 0u) return ZERO_E;
  if (exc == 2u) return INF_E;
  if (exc == 3u) return NAN_E;
  // both normal: exact significand product, normalise, round to wfo bits
  const uint32_t ma = (1u << wf) | (uint32_t)r, mb = (1u << wf) | fb;
  const uint32_t P = ma * mb;  // < 2^(2wf+2) <= 2^22 for wf <= 10
  const uint32_t top = (P >> (2 * wf + 1)) & 1u;
  const uint32_t N = top ? P : (P << 1);       // leading one at bit 2wf+1
  const int sh = 2 * wf + 1 - wfo;             // bits below the kept wfo+1 (0 if extended)
  uint32_t kept = N >> sh;
  if (sh > 0) {
    const uint32_t rem = N & ((1u << sh) - 1u);
    const uint32_t half = 1u << (sh - 1);
    if (rnd == 0 && (rem > half || (rem == half && (kept & 1u)))) kept += 1u;
  }
  uint32_t inc = top;
  if (kept == (2u << wfo)) { kept >>= 1; inc += 1u; }
  const uint32_t frac = kept - (1u << wfo);
  const int bias = (1 << (we - 1)) - 1;
  const uint32_t ep = (uint32_t)((int)eb - bias + (int)inc) & ((1u << EW) - 1u);
  return frac | (ep << wfo) | (sw << sbit) | NORM_FLAG;
}

// Activation records for hobf_conv2d_prepared: one uint32 per element in a
// zero-padded [n][c][h+2p][w+2p] layout: the canonical x word in bits [0, 20)
// and the weight-table row it selects in bits [20, 32) (row = frac if normal,
// 2^wF + 0/1/2 for zero/inf/NaN; padding = +0 -> row 2^wF).  One thread per
// padded pixel, looping over the channels; consecutive threads write
// consecutive columns (coalesced).

__global__ void __launch_bounds__(256) prepare_acts_kernel(const uint32_t* __restrict__ planes, int n, int h, int w,
                                                           int cin, int pad, int we, int wf,
                                                           uint32_t* __restrict__ rec) {
  const int Hp = h + 2 * pad, Wp = w + 2 * pad;
  const int64_t npix = (int64_t)n * Hp * Wp;
  const int CG = (cin + 31) >> 5;
  const int nb = 3 + we + wf, np = (nb + 3) / 4 * 4;
  const uint32_t zero_rec = xrec_of(0u, we, wf);
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix; p += (int64_t)gridDim.x * blockDim.x) {
    const int ixp = (int)(p % Wp);
    const int iyp = (int)((p / Wp) % Hp);
    const int ni = (int)(p / ((int64_t)Wp * Hp));
    const int iy = iyp - pad, ix = ixp - pad;
    const bool inside = iy >= 0 && iy < h && ix >= 0 && ix < w;
    uint32_t* out = rec + ((int64_t)ni * cin * Hp + iyp) * Wp + ixp;
    for (int cg = 0; cg < CG; cg++) {
      uint32_t P[32];
      if (inside) {
        const uint32_t* src = planes + ((((int64_t)ni * h + iy) * w + ix) * CG + cg) * np;
        for (int j = 0; j < nb; j++) P[j] = __ldg(src + j);
      }
      const int cmax = min(32, cin - cg * 32);
      for (int b = 0; b < cmax; b++) {
        uint32_t v = zero_rec;
        if (inside) {
          uint32_t x = 0u;
          for (int j = 0; j < nb; j++) x |= ((P[j] >> b) & 1u) << j;
          v = xrec_of(x, we, wf);
        }
        out[(int64_t)(cg * 32 + b) * Hp * Wp] = v;
      }
    }
  }
}

// float32 NHWC activations -> quantised records in the padded [n][c][h+2p][w+2p]
// layout in one pass (the first layer of a network: no bitslice round trip).
// CTA tile = 32 padded columns x 32 channels of one (n, padded row): coalesced
// float reads along c, smem transpose, coalesced record writes along columns.
__global__ void __launch_bounds__(256) quantize_acts_kernel(const float* __restrict__ x, int n, int h, int w, int cin,
                                                            int pad, int we, int wf, int rnd,
                                                            uint32_t* __restrict__ rec) {
  __shared__ uint32_t tile[32][33];
  const int Hp = h + 2 * pad, Wp = w + 2 * pad;
  const int xtiles = (Wp + 31) / 32, ctiles = (cin + 31) / 32;
  const int64_t ntiles = (int64_t)n * Hp * xtiles * ctiles;
  const uint32_t zero_rec = xrec_of(0u, we, wf);
  // flattened tiles (column tile fastest), grid-stride: no grid dimension limit
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
  const int xb = (int)(t % xtiles) * 32;   // first padded column of the tile
  const int cb = (int)((t / xtiles) % ctiles) * 32;  // first channel of the tile
  const int64_t rowi = t / ((int64_t)xtiles * ctiles);
  const int ni = (int)(rowi / Hp), iyp = (int)(rowi % Hp);
  const int iy = iyp - pad;
  // all of this thread's loads first (4 in flight per thread), then the encodes
  constexpr int K = 32 / 8;  // blockDim.y == 8
  float xv[K];
  bool in[K];
  const int c = cb + threadIdx.x;
  const bool row_in = iy >= 0 && iy < h && c < cin;
  const float* __restrict__ xrow = x + ((int64_t)ni * h + iy) * w * cin + c;
#pragma unroll
  for (int u = 0; u < K; u++) {  // column within the tile
    const int ix = xb + threadIdx.y + 8 * u - pad;
    in[u] = row_in && ix >= 0 && ix < w;
    xv[u] = in[u] ? __ldg(xrow + (int64_t)ix * cin) : 0.0f;
  }
#pragma unroll
  for (int u = 0; u < K; u++)
    tile[threadIdx.y + 8 * u][threadIdx.x] = in[u] ? xrec_of(encode_f32(xv[u], we, wf, rnd), we, wf) : zero_rec;
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {  // channel within the tile
    const int c = cb + k, ixp = xb + threadIdx.x;
    if (c < cin && ixp < Wp) rec[(((int64_t)ni * cin + c) * Hp + iyp) * Wp + ixp] = tile[threadIdx.x][k];
  }
  __syncthreads();  // the tile is refilled by the next iteration
  }
}

// Row-wise variant (the fast path when cin % 4 == 0 and x is 16-byte aligned):
// one CTA per (image, padded input row) and chunk of CC channels.  Phase 1
// reads the row's float4 channel quads (consecutive threads = consecutive
// 16-byte quads: coalesced), encodes them (branch-free encode_f32) and writes
// the records transposed into shared memory [c][stride]; phase 2 writes each
// channel's padded record row (Wp words, contiguous in the [n][c][Hp][Wp]
// layout) with coalesced stores, padding columns / rows as +0 records.
// One (image ni, padded row iyp, channel chunk c0) tile; srec = [cc][stride].
__device__ __forceinline__ void quantize_row_tile(const float* __restrict__ x, int n, int h, int w, int cin, int pad,
                                                  int we, int wf, int rnd, int cc, int stride,
                                                  uint32_t* __restrict__ rec, uint32_t* srec, int iyp, int ni,
                                                  int c0) {
  const int Hp = h + 2 * pad, Wp = w + 2 * pad;
  const uint32_t zero_rec = xrec_of(0u, we, wf);
  const int ncc = min(cc, cin - c0);
  const int iy = iyp - pad;
  if (iy >= 0 && iy < h) {
    // thread -> (pixel lane, channel quad) once; no division in the loops
    const int quads = ncc >> 2;
    const int ppt = blockDim.x / quads;  // pixels per pass (quads <= 64 when cc <= 256)
    const int qd = threadIdx.x % quads, ix0 = threadIdx.x / quads;
    const float4* __restrict__ src = reinterpret_cast<const float4*>(x + (((int64_t)ni * h + iy) * w) * cin + c0);
    if (ix0 < ppt) {
      // UNR float4 loads of this thread in flight before any encode (the loop is
      // otherwise one dependent HBM round trip per iteration)
      constexpr int UNR = 4;
      for (int ix = ix0; ix < w; ix += UNR * ppt) {
        float4 v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; u++) {
          const int xx = ix + u * ppt;
          v[u] = xx < w ? __ldg(src + (int64_t)xx * (cin >> 2) + qd) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < UNR; u++) {
          const int xx = ix + u * ppt;
          if (xx >= w) break;
          uint32_t* d = srec + (4 * qd) * stride + xx;
          if (we <= 7) {
            d[0] = xrec_of(encode_f32_fast(v[u].x, we, wf, rnd), we, wf);
            d[stride] = xrec_of(encode_f32_fast(v[u].y, we, wf, rnd), we, wf);
            d[2 * stride] = xrec_of(encode_f32_fast(v[u].z, we, wf, rnd), we, wf);
            d[3 * stride] = xrec_of(encode_f32_fast(v[u].w, we, wf, rnd), we, wf);
          } else {
            d[0] = xrec_of(encode_f32(v[u].x, we, wf, rnd), we, wf);
            d[stride] = xrec_of(encode_f32(v[u].y, we, wf, rnd), we, wf);
            d[2 * stride] = xrec_of(encode_f32(v[u].z, we, wf, rnd), we, wf);
            d[3 * stride] = xrec_of(encode_f32(v[u].w, we, wf, rnd), we, wf);
          }
        }
      }
    }
  }
  __syncthreads();
  const bool row_in = iy >= 0 && iy < h;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  uint32_t* __restrict__ dst = rec + (((int64_t)ni * cin + c0) * Hp + iyp) * Wp;
  for (int c = warp; c < ncc; c += nwarps) {  // one channel row per warp: coalesced stores
    uint32_t* __restrict__ drow = dst + (int64_t)c * Hp * Wp;
    const uint32_t* srow = srec + c * stride;
    for (int ixp = lane; ixp < Wp; ixp += 32) {
      const int ix = ixp - pad;
      drow[ixp] = (row_in && ix >= 0 && ix < w) ? srow[ix] : zero_rec;
    }
  }
}

__global__ void __launch_bounds__(256) quantize_acts_row_kernel(const float* __restrict__ x, int n, int h, int w,
                                                                int cin, int pad, int we, int wf, int rnd, int cc,
                                                                int stride, uint32_t* __restrict__ rec) {
  extern __shared__ uint32_t srec[];  // [cc][stride], stride odd
  quantize_row_tile(x, n, h, w, cin, pad, we, wf, rnd, cc, stride, rec, srec, blockIdx.x, blockIdx.y,
                    blockIdx.z * cc);
}

// Same tiles flattened (padded row fastest) with a grid-stride loop, for shapes
// past the grid's y / z limits (n or channel chunks > 65535).
__global__ void __launch_bounds__(256) quantize_acts_row_flat_kernel(const float* __restrict__ x, int n, int h,
                                                                     int w, int cin, int pad, int we, int wf,
                                                                     int rnd, int cc, int stride,
                                                                     uint32_t* __restrict__ rec) {
  extern __shared__ uint32_t srec[];
  const int Hp = h + 2 * pad;
  const int chunks = (cin + cc - 1) / cc;
  const uint64_t ntiles = (uint64_t)n * Hp * chunks;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t rest = t / Hp;
    quantize_row_tile(x, n, h, w, cin, pad, we, wf, rnd, cc, stride, rec, srec, (int)(t % Hp), (int)(rest % n),
                      (int)(rest / n) * cc);
    __syncthreads();  // srec is refilled by the next tile
  }
}

// float32 NHWC -> activation records, bitsliced (the fast path for the formats of
// the generated table when cin % 32 == 0): one thread per (image, padded row,
// 32-channel group, padded column), columns fastest.  The thread's 32 channel
// floats (128 contiguous bytes) are transposed into bit planes, encoded in
// bitsliced form (encode_planes_f32), the record's table-row field is formed on
// the planes too (row = frac for a normal x, 2^wF + {0, 1, 2} for zero / inf /
// NaN), and a second transpose gives the 32 records, stored one per channel row
// of the [n][c][h+2p][w+2p] layout (consecutive threads = consecutive columns:
// coalesced).  Padding positions store the +0 record.
template <int WE, int WF, typename IDX>
__global__ void __launch_bounds__(256, 2) quantize_acts_bs_kernel(const float* __restrict__ x, int n, int h, int w,
                                                                  int cin, int pad, int rnd,
                                                                  uint32_t* __restrict__ rec, uint32_t one) {
  constexpr int NB = 3 + WE + WF;
  static_assert(NB <= 20 && WF >= 2, "record layout: word in bits [0, 20), row in [20, 32)");
  const int Hp = h + 2 * pad, Wp = w + 2 * pad, CG = cin >> 5;
  const int64_t items = (int64_t)n * Hp * CG * Wp;
  const uint32_t zero_rec = (1u << WF) << 20;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  // item -> (image, padded row, channel group, padded column), columns fastest;
  // the next item's 128 bytes are loaded while this one is encoded (pipeline)
  struct Pos { int ni, iyp, cg, ixp; bool in; };
  // IDX = uint32_t whenever the item count fits (32-bit divisions are a few
  // instructions; 64-bit ones cost ~80 and were a quarter of the kernel's issue)
  auto pos = [&](int64_t it64) {
    Pos p;
    const IDX it = (IDX)it64;
    p.ixp = (int)(it % (IDX)Wp);
    const IDX r1 = it / (IDX)Wp;
    p.cg = (int)(r1 % (IDX)CG);
    const IDX r2 = r1 / (IDX)CG;
    p.iyp = (int)(r2 % (IDX)Hp);
    p.ni = (int)(r2 / (IDX)Hp);
    const int iy = p.iyp - pad, ix = p.ixp - pad;
    p.in = iy >= 0 && iy < h && ix >= 0 && ix < w;
    return p;
  };
  uint4 nx[8];
  auto load = [&](const Pos& p) {
    if (!p.in) return;
    const uint4* src =
        reinterpret_cast<const uint4*>(x + (((int64_t)p.ni * h + p.iyp - pad) * w + p.ixp - pad) * cin + 32 * p.cg);
#pragma unroll
    for (int q = 0; q < 8; q++) nx[q] = __ldg(src + q);
  };
  int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  Pos cur = pos(it < items ? it : 0);
  if (it < items) load(cur);
  for (; it < items; it += step) {
    uint32_t Q[32];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      Q[4 * q] = nx[q].x; Q[4 * q + 1] = nx[q].y; Q[4 * q + 2] = nx[q].z; Q[4 * q + 3] = nx[q].w;
    }
    const Pos p = cur;
    if (it + step < items) {
      cur = pos(it + step);
      load(cur);
    }
    if (p.in) {
      transpose32_fma(Q, one);  // Q[k] = bit k of the 32 floats
      uint32_t P[NB];
      hobf::encode_planes_f32<WE, WF>(Q, rnd, P);
      const uint32_t c0 = P[NB - 2], c1 = P[NB - 1];
#pragma unroll
      for (int j = 0; j < 32; j++) Q[j] = j < NB ? P[j % NB] : 0u;
      // table row: frac (normal; canonical specials have frac 0) | 2^wF + {0: zero, 1: inf, 2: NaN}
#pragma unroll
      for (int j = 0; j < WF; j++) Q[20 + j] = P[j];
      Q[20] |= c1 & ~c0;                // inf -> +1
      Q[21] |= c1 & c0;                 // NaN -> +2
      Q[20 + WF] = ~(c0 & ~c1);         // not normal -> 2^wF
      transpose32_fma(Q, one);          // Q[l] = record of channel 32 cg + l
    } else {
#pragma unroll
      for (int l = 0; l < 32; l++) Q[l] = zero_rec;
    }
    uint32_t* dst = rec + (((int64_t)p.ni * cin + 32 * p.cg) * Hp + p.iyp) * Wp + p.ixp;
    const int64_t cstride = (int64_t)Hp * Wp;
#pragma unroll
    for (int l = 0; l < 32; l++) dst[l * cstride] = Q[l];
  }
}

// float32 -> activation record of F(WE, WF) (word | table row << 20), scalar and
// with every width a compile-time constant (~20 integer ops): the same function
// as xrec_of(encode_f32_fast(..)).  The rounding to WF fraction bits is done on
// the float32 pattern (RNE: + half - 1 + lsb below the cut), so t = [e8 | frac]
// - (127 - bias) << WF is the format's [E | frac] when 0 <= t < 2^(WE+WF);
// t < 0 is an underflow (float32 zeros and subnormals included, since the
// format's emin >= -63 for WE <= 7) -> zero keeping the sign; t >= 2^(WE+WF)
// is an overflow or a float32 inf -> inf keeping the sign; NaN -> canonical NaN
// (L5/L6).
template <int WE, int WF, int RND>
__device__ __forceinline__ uint32_t qrec_f32(uint32_t u, uint32_t one) {
  static_assert(WE <= 7 && WF <= 17 && 3 + WE + WF <= 20, "record: word in bits [0, 20)");
  constexpr int SH = 23 - WF;
  constexpr int TOP = WE + WF + 1;
  constexpr uint32_t LO = (uint32_t)(127 - ((1 << (WE - 1)) - 1)) << WF;  // [e8 | frac] of the format's E = 0
  constexpr uint32_t HI = LO + (1u << (WE + WF));                       // first [e8 | frac] past its range
  constexpr uint32_t SGN = 1u << (WE + WF);
  // the shifts are multiplies by run-time powers of two (`one` == 1), so they
  // issue on the FMA pipe and leave the ALU pipe (the binding one) to the rest
  const uint32_t ur = RND == 0 ? u + ((1u << (SH - 1)) - 1u) + (__umulhi(u, one << (32 - SH)) & 1u) : u;
  const uint32_t m = __umulhi(ur * (one << 1), one << (31 - SH));  // (ur & 0x7fffffff) >> SH = [e8r | frac]
  const uint32_t tt = m + ((1u << TOP) - LO);                     // exc 01 | E | frac (when LO <= m < HI)
  const uint32_t us = __umulhi(u, one << (WE + WF + 1));         // the sign lands on bit WE + WF
  const uint32_t nrec = ((tt & ((1u << WF) - 1u)) * (one << 20) + tt) | (us & SGN);
  const uint32_t zrec = (us & SGN) | ((1u << WF) << 20);
  const uint32_t irec = (us & SGN) | (2u << TOP) | (((1u << WF) + 1u) << 20);
  constexpr uint32_t qnan = (3u << TOP) | (((1u << WF) + 2u) << 20);
  const uint32_t r = m < LO ? zrec : (m >= HI ? irec : nrec);
  return u * (one << 1) > 0xFF000000u ? qnan : r;
}

// float32 NHWC -> activation records (cin % 16 == 0, the generated formats), no
// shared memory: one CTA per (image, padded row); a warp's unit is 8 padded
// columns x 16 channels, lane = (column cl, channel quad q): one float4 load per
// lane (8 x 64 contiguous bytes per warp), 4 records encoded (qrec_f32), and 4
// stores -- for each j the warp writes 8 consecutive columns of the 4 channel rows
// 4q + j (32-byte segments of the [n][c][h+2p][w+2p] layout).  Padding columns /
// rows store the +0 record.  Up to 4 units' loads are in flight per thread.
// (A one-wave grid with the units spread over all warps, to remove the CTA tail
// wave, measured slower: C3 18.4 -> 21.0 us, C4 55 -> 86 us.)
template <int WE, int WF, int RND>
__global__ void __launch_bounds__(256, 6) quantize_acts_direct_kernel(const float* __restrict__ x, int h, int w,
                                                                      int cin, int pad, uint32_t* __restrict__ rec,
                                                                      uint32_t one) {
  constexpr int MAXU = 4;
  const int Hp = h + 2 * pad, Wp = w + 2 * pad;
  const int iyp = blockIdx.x % Hp, ni = blockIdx.x / Hp;
  const int iy = iyp - pad;
  const bool row_in = iy >= 0 && iy < h;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cl = lane & 7, q = lane >> 3;
  const int G16 = cin >> 4, XB = (Wp + 7) >> 3;
  const int units = G16 * XB;
  // u -> (column block, 16-channel group) by a multiply-high (exact: G16^2 * XB < 2^32)
  const uint32_t magic = G16 == 1 ? 0u : 0xFFFFFFFFu / (uint32_t)G16 + 1u;
  auto split = [&](int u, int& xb, int& g) {
    xb = G16 == 1 ? u : (int)__umulhi((uint32_t)u, magic);
    g = u - xb * G16;
  };
  const float* __restrict__ xrow = x + ((int64_t)ni * h + (row_in ? iy : 0)) * w * cin + 4 * q;
  uint32_t* __restrict__ dst = rec + ((int64_t)ni * cin * Hp + iyp) * Wp + cl;
  const int64_t cs = (int64_t)Hp * Wp;
  for (int u0 = warp; u0 < units; u0 += 8 * MAXU) {
    float4 v[MAXU];
#pragma unroll
    for (int k = 0; k < MAXU; k++) {
      const int u = u0 + 8 * k;
      int xb, g;
      split(u, xb, g);
      const int ix = 8 * xb + cl - pad;
      v[k] = (u < units && row_in && ix >= 0 && ix < w)
                 ? __ldg(reinterpret_cast<const float4*>(xrow + (int64_t)ix * cin + 16 * g))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < MAXU; k++) {
      const int u = u0 + 8 * k;
      int xb, g;
      split(u, xb, g);
      const int ixp = 8 * xb + cl;
      // padding positions hold +0.0f, whose record is the +0 record: no branch
      const uint32_t r0 = qrec_f32<WE, WF, RND>(__float_as_uint(v[k].x), one);
      const uint32_t r1 = qrec_f32<WE, WF, RND>(__float_as_uint(v[k].y), one);
      const uint32_t r2 = qrec_f32<WE, WF, RND>(__float_as_uint(v[k].z), one);
      const uint32_t r3 = qrec_f32<WE, WF, RND>(__float_as_uint(v[k].w), one);
      if (u < units && ixp < Wp) {
        uint32_t* d = dst + (16 * g + 4 * q) * cs + 8 * xb;
        d[0] = r0;
        d[cs] = r1;
        d[2 * cs] = r2;
        d[3 * cs] = r3;
      }
    }
  }
}

template <int WE, int WF, int RND>
static bool go_qa_tile(const float* x, int n, int h, int w, int cin, int pad, uint32_t* rec, cudaStream_t s) {
  const int64_t ctas = (int64_t)n * (h + 2 * pad);
  const int64_t g16 = cin >> 4, xb = (w + 2 * pad + 7) >> 3;
  if ((cin & 15) != 0 || ctas > 2147483647LL || g16 * g16 * xb >= (1LL << 32) || g16 * xb > 2147483647LL - 256)
    return false;
  quantize_acts_direct_kernel<WE, WF, RND><<<(unsigned)ctas, 256, 0, s>>>(x, h, w, cin, pad, rec, 1u);
  return true;
}

template <int WE, int WF>
static void go_qa_bs(const float* x, int n, int h, int w, int cin, int pad, int rnd, uint32_t* rec, cudaStream_t s) {
#ifndef HOBF_NO_QA_TILE  // (A/B builds of the development tools only)
  if (rnd == 0 ? go_qa_tile<WE, WF, 0>(x, n, h, w, cin, pad, rec, s) : go_qa_tile<WE, WF, 1>(x, n, h, w, cin, pad, rec, s))
    return;
#endif
  const int64_t items = (int64_t)n * (h + 2 * pad) * (cin >> 5) * (w + 2 * pad);
  const int64_t blocks = std::min<int64_t>((items + 255) / 256, 148 * 2);  // one wave, pipelined loop
  const unsigned b = (unsigned)(blocks < 1 ? 1 : blocks);
  if (items + (int64_t)b * 256 < (int64_t)UINT32_MAX)
    quantize_acts_bs_kernel<WE, WF, uint32_t><<<b, 256, 0, s>>>(x, n, h, w, cin, pad, rnd, rec, 1u);
  else
    quantize_acts_bs_kernel<WE, WF, uint64_t><<<b, 256, 0, s>>>(x, n, h, w, cin, pad, rnd, rec, 1u);
}

template <int WE>
static bool qa_bs_we(int wf, const float* x, int n, int h, int w, int cin, int pad, int rnd, uint32_t* rec,
                     cudaStream_t s) {
  switch (wf) {
    case 2: go_qa_bs<WE, 2>(x, n, h, w, cin, pad, rnd, rec, s); return true;
    case 3: go_qa_bs<WE, 3>(x, n, h, w, cin, pad, rnd, rec, s); return true;
    case 4: go_qa_bs<WE, 4>(x, n, h, w, cin, pad, rnd, rec, s); return true;
    case 5: go_qa_bs<WE, 5>(x, n, h, w, cin, pad, rnd, rec, s); return true;
    case 6: go_qa_bs<WE, 6>(x, n, h, w, cin, pad, rnd, rec, s); return true;
    case 7: go_qa_bs<WE, 7>(x, n, h, w, cin, pad, rnd, rec, s); return true;
    case 8: go_qa_bs<WE, 8>(x, n, h, w, cin, pad, rnd, rec, s); return true;
    case 9: go_qa_bs<WE, 9>(x, n, h, w, cin, pad, rnd, rec, s); return true;
    case 10: go_qa_bs<WE, 10>(x, n, h, w, cin, pad, rnd, rec, s); return true;
  }
  return false;
}

static bool launch_qa_bs(int we, int wf, const float* x, int n, int h, int w, int cin, int pad, int rnd,
                         uint32_t* rec, cudaStream_t s) {
  if ((cin & 31) != 0 || !aligned16(x) || 3 + we + wf > 20) return false;
  if (we == 4) return qa_bs_we<4>(wf, x, n, h, w, cin, pad, rnd, rec, s);
  if (we == 5) return qa_bs_we<5>(wf, x, n, h, w, cin, pad, rnd, rec, s);
  if (we == 6) return qa_bs_we<6>(wf, x, n, h, w, cin, pad, rnd, rec, s);
  return false;
}

// Warp per (weight row, output-channel group, table row): each lane decodes
// its weight from the planes (shfl transpose), computes its entry, and the
// entry bits are ballot-transposed back into NPT planes.
__global__ void __launch_bounds__(256) build_wtab_kernel(const uint32_t* __restrict__ wplanes, int64_t wrows, int G,
                                                         int cin, int khw, int we, int wf, int wfo, int rnd,
                                                         uint32_t* __restrict__ wtab) {
  const int lane = threadIdx.x & 31;
  const int npi = (3 + we + wf + 3) / 4 * 4;
  const int rows = tab_rows(wf);
  const int npt = (tab_width(we, wfo) + 3) / 4 * 4;
  const int S = hobf::tab_stride(npt, wf);
  // item = (weight row, group, chunk of 32 table rows): the weight is decoded once
  // per item and reused for the chunk's rows.
  const int chunks = (rows + 31) / 32;
  const int64_t items = wrows * G * chunks;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; it < items; it += nw) {
    const int r0 = (int)(it % chunks) * 32;
    const int64_t grp = it / chunks;  // (weight row, group)
    const uint32_t mine = lane < npi ? __ldg(wplanes + grp * npi + lane) : 0u;
    uint32_t w = 0u;
    for (int j = 0; j < 3 + we + wf; j++) w |= ((__shfl_sync(0xffffffffu, mine, j) >> lane) & 1u) << j;
    const int r1 = min(rows, r0 + 32);
    constexpr int U = 4;  // rows in flight (independent entry computations and ballots)
    for (int r = r0; r < r1; r += U) {
      uint32_t e[U], out[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        e[u] = r + u < r1 ? tab_entry(w, r + u, we, wf, wfo, rnd) : 0u;
        out[u] = 0u;
      }
      for (int j = 0; j < npt; j++) {
#pragma unroll
        for (int u = 0; u < U; u++) {
          const uint32_t bal = __ballot_sync(0xffffffffu, (e[u] >> j) & 1u);
          out[u] = lane == j ? bal : out[u];
        }
      }
      // weight row (tap, c) of group g -> table block [g][c][tap] (hobf_words.cuh);
      // the stride padding words stay zero
      const int64_t wrow = grp / G, g = grp % G;
      const int64_t blk = (g * cin + wrow % cin) * khw + wrow / cin;
#pragma unroll
      for (int u = 0; u < U; u++)
        if (lane < S && r + u < r1) wtab[(blk * rows + r + u) * S + lane] = lane < npt ? out[u] : 0u;
    }
  }
}

// ----------------------------------------------------------------------------- lop3 peak
__global__ void lop3_peak_kernel(uint32_t* sink, uint32_t seed, int iters) {
  uint32_t v[8];
  const uint32_t a = seed ^ threadIdx.x, b = seed * 7u + blockIdx.x;
#pragma unroll
  for (int i = 0; i < 8; i++) v[i] = a + i * 0x9E3779B9u;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int k = 0; k < 16; k++) {
#pragma unroll
      for (int i = 0; i < 8; i++) {
        uint32_t r;
        if ((k + i) & 1)
          asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(v[i]), "r"(a), "r"(b));
        else
          asm volatile("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(r) : "r"(v[i]), "r"(b), "r"(a));
        v[i] = r;
      }
    }
  }
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) x ^= v[i];
  if (x == 0x12345678u) sink[threadIdx.x & 1023] = x;
}

// ----------------------------------------------------------------------------- C ABI
extern "C" {

int32_t hobf_nbits(int32_t we, int32_t wf) { return 3 + we + wf; }

int32_t hobf_out_wf(hobf_fmt f) { return f.extended ? 2 * f.wf + 1 : f.wf + 1; }

int32_t hobf_nplanes(int32_t nbits) { return (nbits + 3) / 4 * 4; }

int64_t hobf_planes_words(int64_t rows, int64_t c, int32_t nbits) {
  if (rows < 0 || c < 0) return -1;
  return rows * ((c + 31) / 32) * hobf_nplanes(nbits);
}

int32_t hobf_last_launch_count(void) { return g_last_launches; }

const char* hobf_status_str(hobf_status s) {
  switch (s) {
    case HOBF_OK: return "ok";
    case HOBF_EINVAL: return "invalid argument";
    case HOBF_ESHAPE: return "inconsistent shapes";
    case HOBF_EUNSUPPORTED: return "unsupported format (no generated kernel)";
    case HOBF_ECUDA: return "CUDA launch error";
  }
  return "unknown status";
}

const char* hobf_version(void) { return "hobf-b200 0.1 (sm_100a)"; }

static hobf_status pack_common(bool f32, int32_t we, int32_t wf, int32_t rnd, const void* src, int64_t rows,
                               int64_t c, uint32_t* planes, hobf_stream stream) {
  g_last_launches = 0;
  if (!fmt_ok(we, wf) || (f32 && (we > 8 || wf > 23)) || (rnd != 0 && rnd != 1)) return HOBF_EINVAL;
  if (rows < 0 || c < 0) return HOBF_EINVAL;
  if (rows == 0 || c == 0) return HOBF_OK;
  if (!src || !planes || !aligned16(planes)) return HOBF_EINVAL;
  const int np = hobf_nplanes(3 + we + wf);
  const int64_t items = rows * ((c + 31) / 32);
  if ((c & 31) == 0 && aligned16(src) && np >= 8) {  // dense rows: thread-per-group transpose
    if (f32) launch_pack_t<true>(np, src, items, we, wf, rnd, planes, (cudaStream_t)stream);
    else launch_pack_t<false>(np, src, items, we, wf, 0, planes, (cudaStream_t)stream);
  } else if (f32) {
    pack_kernel<true><<<warp_grid(items), 256, 0, (cudaStream_t)stream>>>(src, rows, c, we, wf, rnd, np, planes);
  } else {
    pack_kernel<false><<<warp_grid(items), 256, 0, (cudaStream_t)stream>>>(src, rows, c, we, wf, 0, np, planes);
  }
  if (cudaGetLastError() != cudaSuccess) return HOBF_ECUDA;
  g_last_launches = 1;
  return HOBF_OK;
}

hobf_status hobf_pack(int32_t we, int32_t wf, const uint32_t* d_words, int64_t rows, int64_t c, uint32_t* d_planes,
                      hobf_stream stream) {
  return pack_common(false, we, wf, 0, d_words, rows, c, d_planes, stream);
}

hobf_status hobf_quantize_pack(int32_t we, int32_t wf, int32_t round, const float* d_x, int64_t rows, int64_t c,
                               uint32_t* d_planes, hobf_stream stream) {
  return pack_common(true, we, wf, round, d_x, rows, c, d_planes, stream);
}

static hobf_status unpack_common(bool f32, int32_t we, int32_t wf, const uint32_t* planes, int64_t rows, int64_t c,
                                 void* dst, hobf_stream stream) {
  g_last_launches = 0;
  if (!fmt_ok(we, wf) || (f32 && (we > 7 || wf > 23))) return HOBF_EINVAL;
  if (rows < 0 || c < 0) return HOBF_EINVAL;
  if (rows == 0 || c == 0) return HOBF_OK;
  if (!planes || !dst || !aligned16(planes)) return HOBF_EINVAL;
  const int np = hobf_nplanes(3 + we + wf);
  const int64_t items = rows * ((c + 31) / 32);
  if ((c & 31) == 0 && aligned16(dst) && np >= 8) {  // dense rows: thread-per-group transpose
    if (f32) launch_unpack_t<true>(np, planes, items, we, wf, dst, (cudaStream_t)stream);
    else launch_unpack_t<false>(np, planes, items, we, wf, dst, (cudaStream_t)stream);
  } else if (f32) {
    unpack_kernel<true><<<warp_grid(items), 256, 0, (cudaStream_t)stream>>>(planes, rows, c, we, wf, np, dst);
  } else {
    unpack_kernel<false><<<warp_grid(items), 256, 0, (cudaStream_t)stream>>>(planes, rows, c, we, wf, np, dst);
  }
  if (cudaGetLastError() != cudaSuccess) return HOBF_ECUDA;
  g_last_launches = 1;
  return HOBF_OK;
}

hobf_status hobf_unpack(int32_t we, int32_t wf, const uint32_t* d_planes, int64_t rows, int64_t c, uint32_t* d_words,
                        hobf_stream stream) {
  return unpack_common(false, we, wf, d_planes, rows, c, d_words, stream);
}

hobf_status hobf_unpack_f32(int32_t we, int32_t wf, const uint32_t* d_planes, int64_t rows, int64_t c, float* d_x,
                            hobf_stream stream) {
  return unpack_common(true, we, wf, d_planes, rows, c, d_x, stream);
}

// Epilogue arguments (hobf_epilogue) -> ConvArgs; HOBF_EINVAL if inconsistent.
static bool set_epilogue(ConvArgs& a, hobf_fmt f, hobf_epilogue ep, bool records_ok) {
  a.out_mode = ep.mode;
  a.next_wf = ep.next_wf;
  a.next_pad = ep.next_pad;
  if (ep.mode == HOBF_OUT_PLANES) return true;
  if (ep.mode == HOBF_OUT_F32) return f.we <= 7;  // float32 holds every F(we <= 7, wfo <= 23) value
  if (ep.next_wf < 1 || ep.next_pad < 0) return false;
  if (ep.mode == HOBF_OUT_NEXT_PLANES) return 3 + f.we + ep.next_wf <= 32;
  if (ep.mode == HOBF_OUT_NEXT_RECORDS) return records_ok && ep.next_wf <= kTabMaxWf && 3 + f.we + ep.next_wf <= 20;
  return false;
}

// largest (pixel, output-channel group) count a conv launch covers: grid.x < 2^31
// blocks of >= 32 threads
static const int64_t kMaxConvItems = 2147483647LL * 32;

enum { OP_CONV = 0, OP_PREPARED = 1, OP_DW = 2 };

static const FormatEntry* tab_format(hobf_fmt f);

// Shared argument checks of the conv entry points, in the order the header
// documents: format, sizes, shapes, format support, then (n > 0 and `launch`)
// pointers and alignment, the grid limits and the epilogue.  Fills `a` and `e`.
// *empty is set when n == 0 (nothing to launch).
static hobf_status conv_setup(int op, hobf_fmt f, const uint32_t* x, int32_t n, int32_t h, int32_t w, int32_t cin,
                              const uint32_t* wt, int32_t kh, int32_t kw, int32_t cout, int32_t stride, int32_t pad,
                              int32_t relu, hobf_epilogue ep, void* out, int32_t variant, bool launch, ConvArgs& a,
                              const FormatEntry*& e, bool* empty) {
  *empty = false;
  if (op == OP_PREPARED ? (variant != 0 && (variant < 3 || variant > 15 || variant == 9)) : variant != 0)
    return HOBF_EINVAL;
  if (!fmt_ok(f.we, f.wf) || (f.round != 0 && f.round != 1) || (f.extended != 0 && f.extended != 1))
    return HOBF_EINVAL;
  if (op == OP_DW) cout = cin;
  if (n < 0 || h < 0 || w < 0 || cin < 0 || kh < 0 || kw < 0 || cout < 0 || stride <= 0 || pad < 0)
    return HOBF_EINVAL;
  if (h == 0 || w == 0 || cin == 0 || kh == 0 || kw == 0 || cout == 0) return HOBF_ESHAPE;
  const int ho = (h + 2 * pad - kh) / stride + 1, wo = (w + 2 * pad - kw) / stride + 1;
  if (h + 2 * pad < kh || w + 2 * pad < kw || ho <= 0 || wo <= 0) return HOBF_ESHAPE;
  if (op == OP_PREPARED && (cout + 31) / 32 > 65535) return HOBF_ESHAPE;  // output-channel groups index grid.y
  e = op == OP_PREPARED ? tab_format(f) : find_format(f.we, f.wf, f.round, f.extended);
  if (!e) return HOBF_EUNSUPPORTED;
  if (n == 0) {
    *empty = true;
    return HOBF_OK;
  }
  if (launch) {
    if (!x || !wt || !out) return HOBF_EINVAL;
    if (!aligned16(x) || !aligned16(wt) || !aligned16(out)) return HOBF_EINVAL;
  }
  a = ConvArgs();
  a.x = x; a.wt = wt; a.y = reinterpret_cast<uint32_t*>(out);
  a.n = n; a.h = h; a.w = w; a.cin = cin; a.kh = kh; a.kw = kw; a.cout = cout;
  a.stride = stride; a.pad = pad; a.relu = relu ? 1 : 0; a.ho = ho; a.wo = wo;
  a.items = (int64_t)n * ho * wo * ((cout + 31) / 32);
  if (a.items > kMaxConvItems) return HOBF_ESHAPE;  // one grid.x block per <= 32 items
  a.variant = variant;
  if (!set_epilogue(a, f, ep, op != OP_CONV)) return HOBF_EINVAL;
  a.row_mul = 1u << 12;
  for (int j = 0; j < 32; j++) a.lift[j] = 1u << (31 - j);
  a.one = 1;
  a.two = 2u;
  a.split_e = a.split_s = a.split_l = 0;
  a.info = nullptr;
  return HOBF_OK;
}

static hobf_status conv_launch(int op, hobf_fmt f, const uint32_t* x, int32_t n, int32_t h, int32_t w, int32_t cin,
                               const uint32_t* wt, int32_t kh, int32_t kw, int32_t cout, int32_t stride, int32_t pad,
                               int32_t relu, hobf_epilogue ep, void* out, int32_t variant, hobf_stream stream) {
  g_last_launches = 0;
  ConvArgs a;
  const FormatEntry* e = nullptr;
  bool empty = false;
  const hobf_status st = conv_setup(op, f, x, n, h, w, cin, wt, kh, kw, cout, stride, pad, relu, ep, out, variant,
                                    true, a, e, &empty);
  if (st != HOBF_OK || empty) return st;
  const hobf::conv_launcher L = op == OP_CONV ? e->conv : op == OP_PREPARED ? e->conv_tab : e->conv_dw;
  if (L(a, (cudaStream_t)stream) != cudaSuccess) return HOBF_ECUDA;
  g_last_launches = 1;
  return HOBF_OK;
}

hobf_status hobf_conv2d(hobf_fmt f, const uint32_t* d_x_planes, int32_t n, int32_t h, int32_t w, int32_t cin,
                        const uint32_t* d_w_planes, int32_t kh, int32_t kw, int32_t cout, int32_t stride,
                        int32_t pad, int32_t relu, uint32_t* d_y_planes, hobf_stream stream) {
  const hobf_epilogue ep = {HOBF_OUT_PLANES, 0, 0};
  return conv_launch(OP_CONV, f, d_x_planes, n, h, w, cin, d_w_planes, kh, kw, cout, stride, pad, relu, ep,
                     d_y_planes, 0, stream);
}

hobf_status hobf_conv2d_ex(hobf_fmt f, const uint32_t* d_x_planes, int32_t n, int32_t h, int32_t w, int32_t cin,
                           const uint32_t* d_w_planes, int32_t kh, int32_t kw, int32_t cout, int32_t stride,
                           int32_t pad, int32_t relu, hobf_epilogue ep, uint32_t* d_out, hobf_stream stream) {
  return conv_launch(OP_CONV, f, d_x_planes, n, h, w, cin, d_w_planes, kh, kw, cout, stride, pad, relu, ep, d_out,
                     0, stream);
}

hobf_status hobf_conv2d_dw(hobf_fmt f, const uint32_t* d_x_planes, int32_t n, int32_t h, int32_t w, int32_t c,
                           const uint32_t* d_w_planes, int32_t kh, int32_t kw, int32_t stride, int32_t pad,
                           int32_t relu, hobf_epilogue ep, uint32_t* d_out, hobf_stream stream) {
  return conv_launch(OP_DW, f, d_x_planes, n, h, w, c, d_w_planes, kh, kw, c, stride, pad, relu, ep, d_out, 0,
                     stream);
}

hobf_status hobf_conv_kernel_info(int32_t op, hobf_fmt f, int32_t n, int32_t h, int32_t w, int32_t cin, int32_t kh,
                                  int32_t kw, int32_t cout, int32_t stride, int32_t pad, hobf_epilogue ep,
                                  int32_t variant, hobf_kernel_info* info) {
  if (!info || op < OP_CONV || op > OP_DW) return HOBF_EINVAL;
  *info = hobf_kernel_info();
  ConvArgs a;
  const FormatEntry* e = nullptr;
  bool empty = false;
  hobf_status st = conv_setup(op, f, nullptr, n, h, w, cin, nullptr, kh, kw, cout, stride, pad, 0, ep, nullptr,
                              variant, false, a, e, &empty);
  if (st != HOBF_OK || empty) return st;
  hobf::LaunchInfo li = {};
  a.info = &li;
  const hobf::conv_launcher L = op == OP_CONV ? e->conv : op == OP_PREPARED ? e->conv_tab : e->conv_dw;
  if (L(a, nullptr) != cudaSuccess || !li.func) return HOBF_ECUDA;
  info->variant = li.variant;
  info->threads = li.threads;
  info->dyn_smem = (int32_t)li.smem;
  info->blocks = li.blocks;
  const char* name = nullptr;
  if (cudaFuncGetName(&name, li.func) == cudaSuccess && name) {
    snprintf(info->name, sizeof(info->name), "%s", name);
  }
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, li.func) != cudaSuccess) return HOBF_ECUDA;
  info->regs = fa.numRegs;
  info->local_bytes = (int32_t)fa.localSizeBytes;
  info->static_smem = (int32_t)fa.sharedSizeBytes;
  if (li.smem > 48 * 1024)
    cudaFuncSetAttribute(li.func, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, li.func, li.threads, li.smem) != cudaSuccess)
    return HOBF_ECUDA;
  info->ctas_per_sm = nb;
  return HOBF_OK;
}

hobf_status hobf_mac_planes(hobf_fmt f, uint32_t* d_acc, const uint32_t* d_a, const uint32_t* d_b, int64_t n_groups,
                            hobf_stream stream) {
  g_last_launches = 0;
  if (!fmt_ok(f.we, f.wf) || (f.round != 0 && f.round != 1) || n_groups < 0) return HOBF_EINVAL;
  const FormatEntry* e = find_format(f.we, f.wf, f.round, f.extended);
  if (!e) return HOBF_EUNSUPPORTED;
  if (n_groups == 0) return HOBF_OK;
  if (!d_acc || !d_a || !d_b || !aligned16(d_acc) || !aligned16(d_a) || !aligned16(d_b)) return HOBF_EINVAL;
  if (e->mac(d_acc, d_a, d_b, n_groups, (cudaStream_t)stream) != cudaSuccess) return HOBF_ECUDA;
  g_last_launches = 1;
  return HOBF_OK;
}

hobf_status hobf_gate_count(hobf_fmt f, int32_t* mac, int32_t* mul, int32_t* add, int32_t* relu,
                            int32_t* mac_tab) {
  const FormatEntry* e = find_format(f.we, f.wf, f.round, f.extended);
  if (!e) return HOBF_EUNSUPPORTED;
  if (mac) *mac = e->g_mac;
  if (mul) *mul = e->g_mul;
  if (add) *add = e->g_add;
  if (relu) *relu = e->g_relu;
  if (mac_tab) *mac_tab = e->g_tab;
  return HOBF_OK;
}

static const FormatEntry* tab_format(hobf_fmt f) {
  if (f.wf > kTabMaxWf) return nullptr;
  return find_format(f.we, f.wf, f.round, f.extended);
}

int64_t hobf_wtab_words(hobf_fmt f, int32_t kh, int32_t kw, int32_t cin, int32_t cout) {
  if (!fmt_ok(f.we, f.wf) || kh <= 0 || kw <= 0 || cin <= 0 || cout <= 0) return -1;
  if (!tab_format(f)) return -1;
  const int64_t npt = (tab_width(f.we, hobf_out_wf(f)) + 3) / 4 * 4;
  return (int64_t)kh * kw * cin * ((cout + 31) / 32) * tab_rows(f.wf) * hobf::tab_stride((int)npt, f.wf);
}

hobf_status hobf_prepare_weights(hobf_fmt f, const uint32_t* d_w_planes, int32_t kh, int32_t kw, int32_t cin,
                                 int32_t cout, uint32_t* d_wtab, hobf_stream stream) {
  g_last_launches = 0;
  if (!fmt_ok(f.we, f.wf) || (f.round != 0 && f.round != 1) || kh < 0 || kw < 0 || cin < 0 || cout < 0)
    return HOBF_EINVAL;
  if (kh == 0 || kw == 0 || cin == 0 || cout == 0) return HOBF_ESHAPE;
  if (!tab_format(f)) return HOBF_EUNSUPPORTED;
  if (!d_w_planes || !d_wtab || !aligned16(d_w_planes) || !aligned16(d_wtab)) return HOBF_EINVAL;
  const int G = (cout + 31) / 32;
  const int64_t wrows = (int64_t)kh * kw * cin;
  const int64_t items = wrows * G * ((tab_rows(f.wf) + 31) / 32);
  build_wtab_kernel<<<warp_grid(items), 256, 0, (cudaStream_t)stream>>>(d_w_planes, wrows, G, cin, kh * kw, f.we,
                                                                          f.wf, hobf_out_wf(f), f.round, d_wtab);
  if (cudaGetLastError() != cudaSuccess) return HOBF_ECUDA;
  g_last_launches = 1;
  return HOBF_OK;
}

int64_t hobf_xrec_words(int32_t n, int32_t h, int32_t w, int32_t cin, int32_t pad) {
  if (n < 0 || h <= 0 || w <= 0 || cin <= 0 || pad < 0) return -1;
  return (int64_t)n * cin * (h + 2 * pad) * (w + 2 * pad);
}

hobf_status hobf_prepare_activations(hobf_fmt f, const uint32_t* d_x_planes, int32_t n, int32_t h, int32_t w,
                                     int32_t cin, int32_t pad, uint32_t* d_xrec, hobf_stream stream) {
  g_last_launches = 0;
  if (!fmt_ok(f.we, f.wf) || n < 0 || h < 0 || w < 0 || cin < 0 || pad < 0) return HOBF_EINVAL;
  if (h == 0 || w == 0 || cin == 0) return HOBF_ESHAPE;
  if (!tab_format(f)) return HOBF_EUNSUPPORTED;
  if (n == 0) return HOBF_OK;
  if (!d_x_planes || !d_xrec || !aligned16(d_x_planes)) return HOBF_EINVAL;
  const int64_t npix = (int64_t)n * (h + 2 * pad) * (w + 2 * pad);
  int64_t blocks = (npix + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  prepare_acts_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d_x_planes, n, h, w, cin, pad, f.we, f.wf,
                                                                            d_xrec);
  if (cudaGetLastError() != cudaSuccess) return HOBF_ECUDA;
  g_last_launches = 1;
  return HOBF_OK;
}

hobf_status hobf_quantize_activations(hobf_fmt f, const float* d_x, int32_t n, int32_t h, int32_t w, int32_t cin,
                                      int32_t pad, uint32_t* d_xrec, hobf_stream stream) {
  g_last_launches = 0;
  if (!fmt_ok(f.we, f.wf) || (f.round != 0 && f.round != 1) || n < 0 || h < 0 || w < 0 || cin < 0 || pad < 0)
    return HOBF_EINVAL;
  if (h == 0 || w == 0 || cin == 0) return HOBF_ESHAPE;
  if (!tab_format(f)) return HOBF_EUNSUPPORTED;
  if (n == 0) return HOBF_OK;
  if (!d_x || !d_xrec) return HOBF_EINVAL;
  const int Hp = h + 2 * pad, Wp = w + 2 * pad;
  if ((int64_t)n * Hp > 2147483647LL) return HOBF_EINVAL;
  if (launch_qa_bs(f.we, f.wf, d_x, n, h, w, cin, pad, f.round, d_xrec, (cudaStream_t)stream)) {
    if (cudaGetLastError() != cudaSuccess) return HOBF_ECUDA;
    g_last_launches = 1;
    return HOBF_OK;
  }
  const int stride = w | 1;  // odd smem row stride: the transposed writes spread over the banks
  const int cc = (int)std::min<int64_t>(std::min<int64_t>(cin, 256),
                                        std::max<int64_t>(4, (32 * 1024 / 4) / stride) / 4 * 4);
  const int64_t kMaxGrid = 2147483647LL;
  const size_t smem = (size_t)cc * stride * 4;
  // row kernels: float4 channel quads, the row's records transposed in at most the
  // default 48 KB of shared memory (w up to 3071); wider rows take the tile kernel
  if ((cin & 3) == 0 && aligned16(d_x) && smem <= 48 * 1024) {
    const int chunks = (cin + cc - 1) / cc;
    if (n <= 65535 && chunks <= 65535) {
      quantize_acts_row_kernel<<<dim3((unsigned)Hp, (unsigned)n, (unsigned)chunks), 256, smem,
                                 (cudaStream_t)stream>>>(d_x, n, h, w, cin, pad, f.we, f.wf, f.round, cc, stride,
                                                         d_xrec);
    } else {
      const int64_t tiles = (int64_t)n * Hp * chunks;
      quantize_acts_row_flat_kernel<<<(unsigned)std::min(tiles, kMaxGrid), 256, smem, (cudaStream_t)stream>>>(
          d_x, n, h, w, cin, pad, f.we, f.wf, f.round, cc, stride, d_xrec);
    }
  } else {
    const int64_t tiles = (int64_t)n * Hp * ((Wp + 31) / 32) * ((cin + 31) / 32);
    quantize_acts_kernel<<<(unsigned)std::min(tiles, kMaxGrid), dim3(32, 8), 0, (cudaStream_t)stream>>>(
        d_x, n, h, w, cin, pad, f.we, f.wf, f.round, d_xrec);
  }
  if (cudaGetLastError() != cudaSuccess) return HOBF_ECUDA;
  g_last_launches = 1;
  return HOBF_OK;
}

hobf_status hobf_conv2d_prepared(hobf_fmt f, const uint32_t* d_xrec, int32_t n, int32_t h, int32_t w, int32_t cin,
                                 const uint32_t* d_wtab, int32_t kh, int32_t kw, int32_t cout, int32_t stride,
                                 int32_t pad, int32_t relu, uint32_t* d_y_planes, hobf_stream stream) {
  const hobf_epilogue ep = {HOBF_OUT_PLANES, 0, 0};
  return hobf_conv2d_prepared_ex(f, d_xrec, n, h, w, cin, d_wtab, kh, kw, cout, stride, pad, relu, ep, d_y_planes,
                                 0, stream);
}

hobf_status hobf_conv2d_prepared_ex(hobf_fmt f, const uint32_t* d_xrec, int32_t n, int32_t h, int32_t w,
                                    int32_t cin, const uint32_t* d_wtab, int32_t kh, int32_t kw, int32_t cout,
                                    int32_t stride, int32_t pad, int32_t relu, hobf_epilogue ep, uint32_t* d_out,
                                    int32_t variant, hobf_stream stream) {
  return conv_launch(OP_PREPARED, f, d_xrec, n, h, w, cin, d_wtab, kh, kw, cout, stride, pad, relu, ep, d_out,
                     variant, stream);
}

hobf_status hobf_lop3_peak(int32_t blocks, int32_t threads, int32_t iters, uint32_t* d_sink, hobf_stream stream,
                           int64_t* lop3_per_launch) {
  g_last_launches = 0;
  if (blocks <= 0 || threads <= 0 || threads > 1024 || iters <= 0 || !d_sink) return HOBF_EINVAL;
  lop3_peak_kernel<<<blocks, threads, 0, (cudaStream_t)stream>>>(d_sink, 1u, iters);
  if (cudaGetLastError() != cudaSuccess) return HOBF_ECUDA;
  if (lop3_per_launch) *lop3_per_launch = (int64_t)blocks * threads * iters * 128;
  g_last_launches = 1;
  return HOBF_OK;
}

}  // extern "C"
