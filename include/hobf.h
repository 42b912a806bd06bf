/*
 * hobf.h -- C ABI of the B200-native HOBFLOPS hot path (arXiv 2007.06563):
 * bitslice-parallel custom-precision floating-point multiply-accumulate inside
 * a CNN convolution, on sm_100a.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n (the reference text).
 *
 * DATA FORMATS
 *   Word (one element, low NBITS bits of a uint32): FloPoCo encoding
 *     [exc:2 | sign:1 | exp:wE | frac:wF], MSB to LSB; exc 00 zero, 01 normal,
 *     10 inf, 11 NaN; significand 1.frac, bias 2^(wE-1)-1, every
 *     exponent code normal, no subnormals.  NBITS = 2+1+wE+wF.
 *   Planes (bitslice layout, Fig. 4a): a [rows][C] array of words
 *     is stored as uint32 planes[rows][ceil(C/32)][NP], NP = hobf_nplanes(NBITS)
 *     = roundup(NBITS, 4); bit l of plane word (r, g, j) is field bit j of
 *     element (r, 32g + l).  Padding lanes and planes are zero (+0).
 *   Conv tensors: activations NHWC (rows = n*h*w, C = cin); weights
 *     [kh][kw][cin][cout] (rows = kh*kw*cin, C = cout); outputs NHWC
 *     (rows = n*ho*wo, C = cout) in the MAC output format F(wE, hobf_out_wf(f)).
 *
 * MAC SEMANTICS
 *   single class: product and accumulator fraction width wF+1; RNE or RTZ in
 *   both the multiplier and the adder; overflow -> inf, underflow -> zero with
 *   sign, exact cancellation -> +0; each output is acc = +0 then
 *   acc = add(acc, mul(x, w)) serially over (c, kh, kw), c outermost, with
 *   zero padding taps included; optional ReLU.
 *
 * CONVENTIONS
 *   - The caller owns every buffer; device pointers must be 16-byte aligned.
 *     The library keeps no device allocation.  Its only mutable state is the
 *     per-thread launch counter (hobf_last_launch_count) and a mutex-guarded
 *     record of which kernels were already opted in to > 48 KB of dynamic
 *     shared memory on which device; nothing reads the environment.
 *   - Argument checks are synchronous and return HOBF_EINVAL (null pointer,
 *     negative size, misaligned pointer, format out of range) / HOBF_ESHAPE
 *     (inconsistent shapes; a conv with more than 65535 x 32 output channels or
 *     more than (2^31 - 1) x 32 (pixel, 32-channel group) items -- the launch
 *     grid's limits) / HOBF_EUNSUPPORTED (no generated kernel for the
 *     format) before anything is launched.  Work is enqueued asynchronously on
 *     `stream` (a cudaStream_t; NULL = legacy default stream); a launch failure
 *     returns HOBF_ECUDA.  Nothing aborts or throws across the ABI.
 *   - Words are not validated on the device: pack is total (masks to NBITS and
 *     canonicalises: exc != 01 -> exp = frac = 0, NaN sign 0).
 */
#ifndef HOBF_H
#define HOBF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HOBF_OK = 0,
  HOBF_EINVAL = 1,
  HOBF_ESHAPE = 2,
  HOBF_EUNSUPPORTED = 3,
  HOBF_ECUDA = 4
} hobf_status;

typedef enum { HOBF_RNE = 0, HOBF_RTZ = 1 } hobf_round;

/* Input format + MAC mode.  extended: 0 = single class (product and
 * accumulator fraction wF+1, rounded with `round`); 1 = extended class
 * (HOBFLOPSxxe: the product is exact at 2wF+1 fraction bits,
 * the accumulator is 2wF+1 bits wide and the adder rounds with `round`; RTZ is
 * the paper's cheaper adder).  Outputs are in F(we, hobf_out_wf(f)). */
typedef struct {
  int32_t we, wf, round, extended;
} hobf_fmt;

typedef void* hobf_stream; /* cudaStream_t */

/* NINBITS = 2+1+we+wf. */
int32_t hobf_nbits(int32_t we, int32_t wf);
/* Fraction width of the MAC output: wf+1 (single) or 2wf+1 (extended) (Table 4). */
int32_t hobf_out_wf(hobf_fmt f);
/* Words per 32-lane plane group: roundup(nbits, 4). */
int32_t hobf_nplanes(int32_t nbits);
/* rows * ceil(c/32) * hobf_nplanes(nbits): size of a plane buffer in uint32 words. */
int64_t hobf_planes_words(int64_t rows, int64_t c, int32_t nbits);

/* Bitslice transform: words[rows][c] (F(we,wf) words, device) ->
 * planes (device).  Masks to NBITS and canonicalises. */
hobf_status hobf_pack(int32_t we, int32_t wf, const uint32_t* d_words, int64_t rows, int64_t c,
                      uint32_t* d_planes, hobf_stream stream);

/* Quantise float32 values x[rows][c] (device) into F(we, wf) with `round`
 * (RNE/RTZ at the value's own binade; NaN -> NaN, +-inf -> +-inf, +-0 -> +-0,
 * overflow -> inf, underflow -> zero with sign)
 * and pack into planes (device), one kernel. */
hobf_status hobf_quantize_pack(int32_t we, int32_t wf, int32_t round, const float* d_x, int64_t rows,
                               int64_t c, uint32_t* d_planes, hobf_stream stream);

/* Inverse transform: planes -> words[rows][c] (device). */
hobf_status hobf_unpack(int32_t we, int32_t wf, const uint32_t* d_planes, int64_t rows, int64_t c,
                        uint32_t* d_words, hobf_stream stream);

/* planes -> float32 values (exact for we <= 7; "transformed ... to floats"). */
hobf_status hobf_unpack_f32(int32_t we, int32_t wf, const uint32_t* d_planes, int64_t rows, int64_t c,
                            float* d_x, hobf_stream stream);

/* HOBFLOPS convolution (Fig. 5): x planes (format f.we/f.wf),
 * weight planes (same format), output planes in F(f.we, hobf_out_wf(f)).
 * ho = (h + 2 pad - kh)/stride + 1, wo likewise; both must be >= 1. */
hobf_status hobf_conv2d(hobf_fmt f, const uint32_t* d_x_planes, int32_t n, int32_t h, int32_t w, int32_t cin,
                        const uint32_t* d_w_planes, int32_t kh, int32_t kw, int32_t cout, int32_t stride,
                        int32_t pad, int32_t relu, uint32_t* d_y_planes, hobf_stream stream);

/* Lane-wise MAC on plane groups: acc = add(acc, mul(a, b)).  acc: [n_groups][NP(NOUT)],
 * a, b: [n_groups][NP(NIN)] (device).  One step of the conv reduction. */
hobf_status hobf_mac_planes(hobf_fmt f, uint32_t* d_acc, const uint32_t* d_a, const uint32_t* d_b,
                            int64_t n_groups, hobf_stream stream);

/* Gate counts of the generated circuits (lop3 per 32 lanes; P:249 analogue):
 * mac = multiplier and adder mapped jointly (the hobf_conv2d inner loop body);
 * mac_tab = the hobf_conv2d_prepared inner loop body (multiplier significand
 * read from the weight table).  Any output pointer may be NULL. */
hobf_status hobf_gate_count(hobf_fmt f, int32_t* mac, int32_t* mul, int32_t* add, int32_t* relu,
                            int32_t* mac_tab);

/* Prepared weights ("kernel data pre-transformed").  In the paper's
 * tiling the 32 lanes of a register are 32 output channels and the activation
 * is broadcast across them, so inside the conv the activation is
 * one scalar per thread: for every weight the library precomputes, per lane,
 * the rounded significand product with each possible activation fraction
 * (plus the exception algebra for x = 0 / inf / NaN) once, and the conv reads
 * the row the activation selects instead of evaluating the multiplier array.
 * Results are identical to hobf_conv2d.
 *
 * hobf_wtab_words: size in uint32 words of the table buffer for these weights,
 * or -1 if the format has no table kernel (wf > 10).  Extended-class entries
 * hold the exact product (2wf+1 fraction bits).
 * Layout: [ceil(cout/32)][cin][kh][kw][2^wf + 3 rows][stride] uint32, where an
 * entry has NPT = roundup(wfo + we + 5, 4) planes and rows are padded to
 * stride = NPT + 4 words when wf <= 7 and NPT/4 is even (conflict-free 128-bit
 * row gathers from shared memory), else stride = NPT; everything one 32-channel output group needs
 * for one input channel is one contiguous block (one bulk copy). */
int64_t hobf_wtab_words(hobf_fmt f, int32_t kh, int32_t kw, int32_t cin, int32_t cout);

/* Build the weight table from weight planes (layout as for hobf_conv2d). */
hobf_status hobf_prepare_weights(hobf_fmt f, const uint32_t* d_w_planes, int32_t kh, int32_t kw, int32_t cin,
                                 int32_t cout, uint32_t* d_wtab, hobf_stream stream);

/* Prepared activations: because the activation is broadcast (one scalar per
 * thread), the conv reads it per element, not bitsliced.  Records are one
 * uint32 per element, zero-padded by `pad` on each spatial side, layout
 * [n][cin][h+2pad][w+2pad]: the canonical F(we,wf) word in bits [0,20) and the
 * weight-table row it selects in bits [20,32).  Formats as for
 * hobf_wtab_words.  hobf_xrec_words returns the buffer size in words. */
int64_t hobf_xrec_words(int32_t n, int32_t h, int32_t w, int32_t cin, int32_t pad);
hobf_status hobf_prepare_activations(hobf_fmt f, const uint32_t* d_x_planes, int32_t n, int32_t h, int32_t w,
                                     int32_t cin, int32_t pad, uint32_t* d_xrec, hobf_stream stream);
/* float32 NHWC activations (device) -> records directly, quantised with f.round
 * exactly as hobf_quantize_pack (first layer: no bitslice round trip). */
hobf_status hobf_quantize_activations(hobf_fmt f, const float* d_x, int32_t n, int32_t h, int32_t w, int32_t cin,
                                      int32_t pad, uint32_t* d_xrec, hobf_stream stream);

/* hobf_conv2d on prepared activations (built with the same pad) and prepared
 * weights; identical results.  Output planes as for hobf_conv2d. */
hobf_status hobf_conv2d_prepared(hobf_fmt f, const uint32_t* d_xrec, int32_t n, int32_t h, int32_t w,
                                 int32_t cin, const uint32_t* d_wtab, int32_t kh, int32_t kw, int32_t cout,
                                 int32_t stride, int32_t pad, int32_t relu, uint32_t* d_y_planes,
                                 hobf_stream stream);

/* ---- Conv with an explicit output epilogue / kernel schedule ----------------
 * Layer chaining ("the OFM stays in the bitsliced format between
 * layers"; with the extended class "rounding is dealt with at the end
 * of the layer in the activation function"): after the serial reduction (and
 * ReLU when relu != 0) every output word of F(we, wfo) is re-rounded into the
 * NEXT layer's input format F(we, next_wf) (RNE or RTZ as f.round; exact
 * when next_wf >= wfo; rounding up out of the top binade -> inf; zero / inf
 * keep their sign) and written in the layout the next layer consumes, so no
 * unpack / repack runs between layers.
 *   HOBF_OUT_PLANES        plain output planes F(we, wfo) (= hobf_conv2d[_prepared]);
 *   HOBF_OUT_NEXT_PLANES   planes of F(we, next_wf): [n*ho*wo][ceil(cout/32)]
 *                          [roundup(3+we+next_wf, 4)] = the next hobf_conv2d's x;
 *   HOBF_OUT_NEXT_RECORDS  activation records of F(we, next_wf), zero-padded by
 *                          next_pad: [n][cout][ho+2*next_pad][wo+2*next_pad]
 *                          (hobf_xrec_words(n, ho, wo, cout, next_pad) words) =
 *                          the next hobf_conv2d_prepared's x.  Only the interior
 *                          is written: the caller's buffer must hold +0 records
 *                          in the padding border (e.g. zero-filled once; the
 *                          +0 record of F(we, next_wf) is (2^next_wf) << 20).
 *                          Needs 3+we+next_wf <= 20 and next_wf <= 10
 *                          (hobf_conv2d_prepared_ex only).
 *   HOBF_OUT_F32           the last layer (floats only at the network's
 *                          edges): every output word of F(we, wfo) decoded to
 *                          its exact float32 value ((-1)^s 1.f 2^(E-bias); +-0,
 *                          +-inf, NaN = 0x7FC00000), written NHWC as float
 *                          [n][ho][wo][cout] (d_out is a float*, 16-byte
 *                          aligned) -- what hobf_unpack_f32 of the planes
 *                          gives, without the planes.  Needs we <= 7.
 * next_wf / next_pad are ignored for HOBF_OUT_PLANES / HOBF_OUT_F32; inconsistent
 * values -> HOBF_EINVAL.  The oracle's definition is ref_convert(relu(acc)). */
typedef enum {
  HOBF_OUT_PLANES = 0,
  HOBF_OUT_NEXT_PLANES = 1,
  HOBF_OUT_NEXT_RECORDS = 2,
  HOBF_OUT_F32 = 3
} hobf_out_mode;
typedef struct {
  int32_t mode;     /* hobf_out_mode */
  int32_t next_wf;  /* next layer's fraction width (same exponent width we) */
  int32_t next_pad; /* next layer's padding (records only) */
} hobf_epilogue;

hobf_status hobf_conv2d_ex(hobf_fmt f, const uint32_t* d_x_planes, int32_t n, int32_t h, int32_t w, int32_t cin,
                           const uint32_t* d_w_planes, int32_t kh, int32_t kw, int32_t cout, int32_t stride,
                           int32_t pad, int32_t relu, hobf_epilogue ep, uint32_t* d_out, hobf_stream stream);

/* Depthwise conv (MobileNets "Conv dw", the layer of P:255 / P:270; SURVEY
 * 8(f) row 4): output channel m = serial (kh, kw) chain over input channel m
 * only, acc = +0; acc = add(acc, mul(x[n, iy, ix, m] or +0, w[kh, kw, m])),
 * same MAC, rounding, padding and ReLU rules as hobf_conv2d (oracle:
 * ref_conv2d_dw).  The 32 lanes are 32 channels of both operands (no
 * broadcast), so every lane runs the full gate MAC (hobf_gate_count mac).
 * x planes: [n*h*w][ceil(c/32)][NP(NIN)]; w planes: [kh*kw][ceil(c/32)][NP(NIN)]
 * (words [kh][kw][c]); output per `ep` as for hobf_conv2d_ex with cout = c
 * (records: the next layer's prepared activations). */
hobf_status hobf_conv2d_dw(hobf_fmt f, const uint32_t* d_x_planes, int32_t n, int32_t h, int32_t w, int32_t c,
                           const uint32_t* d_w_planes, int32_t kh, int32_t kw, int32_t stride, int32_t pad,
                           int32_t relu, hobf_epilogue ep, uint32_t* d_out, hobf_stream stream);

/* hobf_conv2d_prepared with an epilogue (above) and an explicit kernel
 * schedule: variant 0 = automatic (what hobf_conv2d_prepared uses), 3 = one thread
 * per (pixel, 32-Cout group), kernel row of 3 taps unrolled, <= 56 registers;
 * 4 = table entry of the next tap prefetched (large tables); 5 = one-warp CTAs
 * with a 3-deep prefetch ring (fewer warps than SMSPs); 6 = three kernel rows
 * (one input channel) per unrolled loop body, <= 64 registers; 7 = the
 * weight-table block of each input channel staged in shared memory by TMA bulk
 * copies (double-buffered, mbarrier completion), 128/256-thread CTAs -- needs
 * 2 * kh*kw * (2^wf + 3) * stride * 4 bytes <= 50 KB (wf <= 5 for 3x3), else
 * it falls back to variant 6; 8 = as 7 with one kernel row (3 taps, wf = 6, 7)
 * or one tap (wf = 8, 9) of one input channel per staged buffer (3x3 only,
 * else it falls back to variant 7); 10 / 11 = variant 7 with its CTA shape
 * forced to 256 threads x 3 per SM / 128 x 6 (variant 7 picks the one that
 * puts fewer warps on the busiest SM); 12 = variant 4 on a fractional wave
 * (the float32 epilogue, cout % 32 == 0, more 128-pixel units than resident
 * CTAs but at most 1.5 waves): one cooperative CTA per resident slot, each
 * running its own unit plus one of S <= 16 consecutive tap segments of a unit
 * past the wave, the segment accumulators handed on through the units' own
 * float32 output slots (zeroed first, one cudaMemsetAsync) -- the automatic
 * choice where variant 4 would be; otherwise it runs as variant 4.  Variant 12
 * launches the conv through cudaLaunchCooperativeKernel (a device or context
 * that cannot co-schedule the workers: variant 4 runs instead, unless 12 / 13
 * was asked for explicitly, which returns HOBF_ECUDA); 13 = variant 12 at 4
 * CTAs per SM (128 registers); 14 = variant 4 with a progress throttle (the
 * float32 epilogue, cout % 32 == 0, else it runs as variant 4): every CTA
 * publishes the number of input channels it has finished as a token in one of
 * its own output words, and a warp more than two channels ahead of the slowest
 * of 32 CTAs of its Cout group sleeps (bounded) -- an experiment in keeping a
 * group's table gathers inside the L2 window; never the automatic choice;
 * 15 = variant 4 with warp-cooperative table gathers: 8 lanes copy the 16-byte
 * chunks of one table row (cp.async, 4 rows per instruction) into a per-warp
 * shared-memory slot a tap ahead, and each thread reads its own row back.
 * Variants 3 and 6 need kw == 3 (others fall back to the generic loop).  Every
 * variant
 * runs the same circuit over the same serial (c, kh, kw) order: identical
 * results.  Unknown variants -> HOBF_EINVAL. */
hobf_status hobf_conv2d_prepared_ex(hobf_fmt f, const uint32_t* d_xrec, int32_t n, int32_t h, int32_t w,
                                    int32_t cin, const uint32_t* d_wtab, int32_t kh, int32_t kw, int32_t cout,
                                    int32_t stride, int32_t pad, int32_t relu, hobf_epilogue ep, uint32_t* d_out,
                                    int32_t variant, hobf_stream stream);

/* ---- Which kernel a conv call runs (evidence for the measurements) ---------
 * Runs the argument checks and the schedule choice of hobf_conv2d_ex (op 0),
 * hobf_conv2d_prepared_ex (op 1; `variant` as there) or hobf_conv2d_dw (op 2;
 * cin = cout = c) for these shapes, launches nothing, and fills *info with the
 * kernel that call would launch: its symbol (mangled, cudaFuncGetName), the
 * schedule (variant; 0 for ops 0 and 2), CTA size, CTA count, dynamic and
 * static shared memory, registers and local (spill) bytes per thread
 * (cudaFuncGetAttributes) and resident CTAs per SM
 * (cudaOccupancyMaxActiveBlocksPerMultiprocessor).  Same statuses as the conv
 * call (pointers are not needed); n = 0 -> HOBF_OK with an empty name; needs
 * a CUDA device for the attribute queries (else HOBF_ECUDA). */
typedef struct {
  char name[256];
  int32_t variant, threads, dyn_smem, static_smem, regs, local_bytes, ctas_per_sm;
  int64_t blocks;
} hobf_kernel_info;

hobf_status hobf_conv_kernel_info(int32_t op, hobf_fmt f, int32_t n, int32_t h, int32_t w, int32_t cin, int32_t kh,
                                  int32_t kw, int32_t cout, int32_t stride, int32_t pad, hobf_epilogue ep,
                                  int32_t variant, hobf_kernel_info* info);

/* LOP3 issue-rate microbenchmark (roofline denominator): launches `blocks` x
 * `threads` threads, each issuing `iters` x 128 dependent-free lop3 ops;
 * *lop3_per_launch receives the thread-op count.  d_sink: >= 4 KiB device. */
hobf_status hobf_lop3_peak(int32_t blocks, int32_t threads, int32_t iters, uint32_t* d_sink,
                           hobf_stream stream, int64_t* lop3_per_launch);

/* Number of kernel launches the previous successful call on this thread enqueued. */
int32_t hobf_last_launch_count(void);

const char* hobf_status_str(hobf_status s);
const char* hobf_version(void);

#ifdef __cplusplus
}
#endif

#endif /* HOBF_H */
