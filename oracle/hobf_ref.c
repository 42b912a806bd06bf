/*
 * oracle/hobf_ref.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, scalar CPU emulation of the HOBFLOPS custom floating-point
 * format and MAC (arXiv 2007.06563), written from the paper and from SURVEY.md
 * section 8(c).  It exists to check the CUDA path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It shares no code, header, table or generator with the CUDA
 * path (paper_2007_06563_b200/), and neither side includes the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n.
 *
 * Arithmetic is exact: every finite value is held as (sign, integer
 * significand M, exponent e) meaning (-1)^sign * M * 2^e, with M in an
 * unsigned __int128, and rounded exactly once per operation (round_to).
 *
 * -------------------------------------------------------------------------
 * Readings of the paper (the ledger; DESIGN.md section "Readings" repeats it)
 * -------------------------------------------------------------------------
 * L1  Exponent codes: FloPoCo encoding -- every code 0..2^wE-1 is a
 *     normal binade; there are no subnormals.  emin = -bias, emax = 2^wE-1-bias.
 * L2  bias = 2^(wE-1) - 1 (the paper inherits FloPoCo's without stating it).
 * L3  Rounding of the configs: RNE primary; RTZ also supported.
 * L4  The rounding mode applies to both the multiplier and the adder.
 * L5  Overflow (biased exponent > 2^wE-1 after rounding) gives +-inf in BOTH
 *     modes.  PARITY UNPINNED (no external reference fixes RTZ overflow).
 * L6  Round at the value's own binade with an unbounded exponent first, then
 *     flush to zero if the biased exponent is < 0; the flushed zero keeps the
 *     exact result's sign.  PARITY UNPINNED (sign of an underflow flush).
 * L7  Zero signs in add (IEEE RNE/RTZ rule): x + (-x) -> +0; (+0)+(-0) -> +0;
 *     (-0)+(-0) -> -0; x + (+-0) -> x.
 * L8  Precision class of the configs: single (product/acc fraction wF+1,
 *     P:164-172).  Extended (2wF+1) is supported by mul.
 * L9  Accumulator format = multiplier-output format; initial value +0.
 * L10 Accumulation order (c, kh, kw), c outermost, strictly serial.
 * L11 Zero padding: padded taps are real MACs with a canonical +0 activation
 *     (so 0 * inf = NaN propagates); MACs counted dense.
 * L12 ReLU is a flag of conv2d; both relu=0 and relu=1 are checked.
 * L13 Quantisation: RNE from float32 ("any quantization method").
 * L14 Padding value is canonical +0; an input -0.0 encodes as -0.
 * L17 Non-canonical words (exc != 01 with nonzero exp/frac, NaN with sign 1)
 *     are accepted and read canonically; every output is canonical
 *     (exc != 01 -> exp = frac = 0; NaN sign 0).
 * L18 Lane l <-> bit l of a plane word; plane j <-> field bit j.
 *     (Layout matters only to the CUDA path; this file works on words.)
 * NaN has no payload and sign 0.  PARITY UNPINNED (canonical NaN sign).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

enum { CLS_ZERO = 0, CLS_NORMAL = 1, CLS_INF = 2, CLS_NAN = 3 };
enum { RND_RNE = 0, RND_RTZ = 1 };

/* A decoded value: cls, sign, and for CLS_NORMAL the exact value M * 2^e. */
typedef struct {
    int cls;
    int sign;
    u128 M;
    int e;
} val_t;

/* Encoded width NINBITS = EXC + SIGN + EXPO + MANT = 2 + 1 + wE + wF. */
int ref_nbits(int we, int wf) { return 3 + we + wf; }

static int bias_of(int we) { return (1 << (we - 1)) - 1; } /* L2 */

/* Field layout of a FloPoCo word: [exc:2 | sign:1 | exp:wE | frac:wF],
 * MSB to LSB, exc 00 zero / 01 normal / 10 inf / 11 NaN. */
static val_t decode(uint32_t w, int we, int wf) {
    val_t v;
    uint32_t frac = w & ((1u << wf) - 1u);
    uint32_t ex = (w >> wf) & ((1u << we) - 1u);
    int sign = (int)((w >> (wf + we)) & 1u);
    int exc = (int)((w >> (wf + we + 1)) & 3u);
    v.cls = exc;
    v.sign = sign;
    v.M = 0;
    v.e = 0;
    if (exc == CLS_NORMAL) {
        /* significand 1.ff..ff: M = 2^wF + frac, value M * 2^(E - bias - wF) */
        v.M = ((u128)1 << wf) + frac;
        v.e = (int)ex - bias_of(we) - wf;
    }
    if (exc == CLS_NAN) v.sign = 0; /* canonical NaN */
    return v;
}

static uint32_t enc_special(int cls, int sign, int we, int wf) {
    if (cls == CLS_NAN) sign = 0;
    return ((uint32_t)cls << (wf + we + 1)) | ((uint32_t)sign << (wf + we));
}

static uint32_t enc_normal(int sign, uint32_t ex, uint32_t frac, int we, int wf) {
    return ((uint32_t)CLS_NORMAL << (wf + we + 1)) | ((uint32_t)sign << (wf + we)) |
           (ex << wf) | frac;
}

static int bitlen128(u128 x) {
    int n = 0;
    while (x) { n++; x >>= 1; }
    return n;
}

/* round_to: round the exact nonzero value (-1)^sign * M * 2^e
 * into F(wE, wf_out) at its own binade (unbounded exponent), ties to even for
 * RNE, truncation for RTZ; then overflow -> inf (L5), underflow -> zero with
 * the exact result's sign (L6). */
static uint32_t round_to(int sign, u128 M, int e, int we, int wf_out, int mode) {
    int k = bitlen128(M) - 1;        /* value = 1.xxx * 2^(e+k) */
    int sh = k - wf_out;             /* bits below the kept fraction */
    u128 q;
    if (sh <= 0) {
        q = M << (-sh);              /* exact */
    } else {
        u128 rem = M & (((u128)1 << sh) - 1);
        u128 half = (u128)1 << (sh - 1);
        q = M >> sh;
        if (mode == RND_RNE) {
            if (rem > half || (rem == half && (q & 1))) q += 1;
        }
    }
    long E = (long)e + k + bias_of(we);
    if (q == ((u128)1 << (wf_out + 1))) { /* rounding carried into a new binade */
        q >>= 1;
        E += 1;
    }
    if (E > (long)((1 << we) - 1)) return enc_special(CLS_INF, sign, we, wf_out); /* L5 */
    if (E < 0) return enc_special(CLS_ZERO, sign, we, wf_out);                    /* L6 */
    return enc_normal(sign, (uint32_t)E, (uint32_t)(q - ((u128)1 << wf_out)), we, wf_out);
}

/* ref_mul (SURVEY 8(c) "mul"; Table 4 P:151-177 for the output width):
 * a, b in F(wE, wF); result in F(wE, wf_out), wf_out = wF+1 (single) or 2wF+1 (extended). */
uint32_t ref_mul(uint32_t a, uint32_t b, int we, int wf, int wf_out, int mode) {
    val_t x = decode(a, we, wf), y = decode(b, we, wf);
    if (x.cls == CLS_NAN || y.cls == CLS_NAN) return enc_special(CLS_NAN, 0, we, wf_out);
    if ((x.cls == CLS_INF && y.cls == CLS_ZERO) || (x.cls == CLS_ZERO && y.cls == CLS_INF))
        return enc_special(CLS_NAN, 0, we, wf_out);
    int s = x.sign ^ y.sign;
    if (x.cls == CLS_INF || y.cls == CLS_INF) return enc_special(CLS_INF, s, we, wf_out);
    if (x.cls == CLS_ZERO || y.cls == CLS_ZERO) return enc_special(CLS_ZERO, s, we, wf_out);
    /* exact product (2^wF + fa)(2^wF + fb) * 2^(ea + eb), then one rounding */
    return round_to(s, x.M * y.M, x.e + y.e, we, wf_out, mode);
}

/* ref_add (SURVEY 8(c) "add"): operands and result in F(wE, wf). */
uint32_t ref_add(uint32_t a, uint32_t b, int we, int wf, int mode) {
    val_t x = decode(a, we, wf), y = decode(b, we, wf);
    if (x.cls == CLS_NAN || y.cls == CLS_NAN) return enc_special(CLS_NAN, 0, we, wf);
    if (x.cls == CLS_INF && y.cls == CLS_INF) {
        if (x.sign == y.sign) return enc_special(CLS_INF, x.sign, we, wf);
        return enc_special(CLS_NAN, 0, we, wf); /* +inf + -inf */
    }
    if (x.cls == CLS_INF) return enc_special(CLS_INF, x.sign, we, wf);
    if (y.cls == CLS_INF) return enc_special(CLS_INF, y.sign, we, wf);
    if (x.cls == CLS_ZERO && y.cls == CLS_ZERO) /* L7: -0 only if both are -0 */
        return enc_special(CLS_ZERO, x.sign & y.sign, we, wf);
    if (x.cls == CLS_ZERO) return round_to(y.sign, y.M, y.e, we, wf, mode); /* exact: 0 + y = y */
    if (y.cls == CLS_ZERO) return round_to(x.sign, x.M, x.e, we, wf, mode); /* exact: x + 0 = x */
    /* normal + normal.  Far-apart operands first: let X be the operand with the
     * larger exponent (X = Mx 2^ex, Mx in [2^wf, 2^(wf+1))) and d = ex - ey.  If
     * d >= wf + 3 then 0 < |Y| < 2^(ey+wf+1) <= 2^(ex-2), so the exact sum lies
     * strictly between X and X +- 2^(ex-2), an open interval that holds no point
     * of the F(wE, wf) grid and no RNE midpoint (the grid spacing is 2^ex at X's
     * binade and 2^(ex-1) in the binade below).  Every rounding decision is then
     * fixed by X and the sign of Y alone, so Y may be replaced by any value of the
     * same sign in that interval -- here (-1)^sy 2^(ex-3) -- without changing the
     * result.  This keeps the alignment shift below wf + 3 bits (exponent gaps
     * reach 2^wE - 1 + wf, beyond the 128-bit integer for wE >= 7). */
    if (x.e - y.e >= wf + 3) { y.M = 1; y.e = x.e - 3; }
    else if (y.e - x.e >= wf + 3) { x.M = 1; x.e = y.e - 3; }
    /* exact sum over the common exponent min(ex, ey) */
    int e = x.e < y.e ? x.e : y.e;
    i128 sx = (i128)(x.M << (x.e - e));
    i128 sy = (i128)(y.M << (y.e - e));
    i128 S = (x.sign ? -sx : sx) + (y.sign ? -sy : sy);
    if (S == 0) return enc_special(CLS_ZERO, 0, we, wf); /* exact cancellation -> +0 */
    int s = S < 0;
    u128 mag = (u128)(S < 0 ? -S : S);
    return round_to(s, mag, e, we, wf, mode);
}

/* ref_relu: NaN stays NaN; zero or sign=1 (incl. -inf) -> +0; else unchanged. */
uint32_t ref_relu(uint32_t a, int we, int wf) {
    val_t x = decode(a, we, wf);
    if (x.cls == CLS_NAN) return enc_special(CLS_NAN, 0, we, wf);
    if (x.cls == CLS_ZERO || x.sign) return enc_special(CLS_ZERO, 0, we, wf);
    if (x.cls == CLS_INF) return enc_special(CLS_INF, 0, we, wf);
    return round_to(0, x.M, x.e, we, wf, RND_RNE); /* exact re-encode (canonical) */
}

/* Canonical form of a word: exc != 01 -> exp = frac = 0; NaN sign 0. */
uint32_t ref_canon(uint32_t a, int we, int wf) {
    val_t x = decode(a, we, wf);
    if (x.cls != CLS_NORMAL) return enc_special(x.cls, x.sign, we, wf);
    return round_to(x.sign, x.M, x.e, we, wf, RND_RNE);
}

/* ref_convert (with the extended class "rounding is dealt with at the end
 * of the layer in the activation function"; layers chained in the
 * bitsliced format): a word of F(wE, wf_in) re-rounded into
 * the next layer's F(wE, wf_out) -- round_to of its exact value (one rounding,
 * RNE or RTZ; widening is exact).  Zero / inf keep their sign, NaN stays NaN.
 * The exponent width is unchanged, so only rounding up to the next binade can
 * overflow (-> inf, L5); nothing underflows. */
uint32_t ref_convert(uint32_t a, int we, int wf_in, int wf_out, int mode) {
    val_t x = decode(a, we, wf_in);
    if (x.cls != CLS_NORMAL) return enc_special(x.cls, x.sign, we, wf_out);
    return round_to(x.sign, x.M, x.e, we, wf_out, mode);
}

/* from_binary32 (L13): exact rational of the float32 (IEEE
 * subnormals included), then round_to; NaN -> NaN, +-inf -> +-inf, +-0 -> +-0. */
uint32_t ref_encode_f32(float f, int we, int wf, int mode) {
    uint32_t u;
    memcpy(&u, &f, 4);
    int sign = (int)(u >> 31);
    int ex = (int)((u >> 23) & 0xFF);
    uint32_t man = u & 0x7FFFFFu;
    if (ex == 0xFF) return man ? enc_special(CLS_NAN, 0, we, wf) : enc_special(CLS_INF, sign, we, wf);
    if (ex == 0 && man == 0) return enc_special(CLS_ZERO, sign, we, wf);
    u128 M;
    int e;
    if (ex == 0) { M = man; e = -149; }                 /* binary32 subnormal */
    else { M = (u128)(0x800000u | man); e = ex - 150; } /* 1.m * 2^(ex-127) */
    return round_to(sign, M, e, we, wf, mode);
}

/* decode to a double (exact for wE <= 8, wF <= 52): (-1)^s (1 + f/2^wF) 2^(E-bias). */
double ref_decode_f64(uint32_t w, int we, int wf) {
    val_t x = decode(w, we, wf);
    if (x.cls == CLS_NAN) return __builtin_nan("");
    if (x.cls == CLS_INF) return x.sign ? -__builtin_inf() : __builtin_inf();
    if (x.cls == CLS_ZERO) return x.sign ? -0.0 : 0.0;
    double m = (double)(uint64_t)x.M;
    double v = __builtin_ldexp(m, x.e);
    return x.sign ? -v : v;
}

/* ---------------- batch helpers (vectorised calls from Python) ---------------- */

void ref_mul_batch(const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t n,
                   int we, int wf, int wf_out, int mode) {
    for (int64_t i = 0; i < n; i++) out[i] = ref_mul(a[i], b[i], we, wf, wf_out, mode);
}

void ref_add_batch(const uint32_t* a, const uint32_t* b, uint32_t* out, int64_t n,
                   int we, int wf, int mode) {
    for (int64_t i = 0; i < n; i++) out[i] = ref_add(a[i], b[i], we, wf, mode);
}

void ref_relu_batch(const uint32_t* a, uint32_t* out, int64_t n, int we, int wf) {
    for (int64_t i = 0; i < n; i++) out[i] = ref_relu(a[i], we, wf);
}

void ref_canon_batch(const uint32_t* a, uint32_t* out, int64_t n, int we, int wf) {
    for (int64_t i = 0; i < n; i++) out[i] = ref_canon(a[i], we, wf);
}

void ref_convert_batch(const uint32_t* a, uint32_t* out, int64_t n, int we, int wf_in, int wf_out, int mode) {
    for (int64_t i = 0; i < n; i++) out[i] = ref_convert(a[i], we, wf_in, wf_out, mode);
}

void ref_encode_f32_batch(const float* x, uint32_t* out, int64_t n, int we, int wf, int mode) {
    for (int64_t i = 0; i < n; i++) out[i] = ref_encode_f32(x[i], we, wf, mode);
}

void ref_decode_f64_batch(const uint32_t* w, double* out, int64_t n, int we, int wf) {
    for (int64_t i = 0; i < n; i++) out[i] = ref_decode_f64(w[i], we, wf);
}

/* Elementwise MAC on words: acc[i] = add(acc[i], mul(a[i], b[i])) -- one step of
 * the serial reduction; acc in F(wE, wf_out), a and b in F(wE, wF). */
void ref_mac_batch(uint32_t* acc, const uint32_t* a, const uint32_t* b, int64_t n,
                   int we, int wf, int wf_out, int mode) {
    for (int64_t i = 0; i < n; i++)
        acc[i] = ref_add(acc[i], ref_mul(a[i], b[i], we, wf, wf_out, mode), we, wf_out, mode);
}

/* ---------------- conv2d (SURVEY 8(c) "conv2d"; B.configs) ----------------
 * x: NHWC words in F(wE, wF); w: [kh][kw][cin][cout] words in F(wE, wF);
 * y: [n][ho][wo][cout] words in F(wE, wf_out).  For every output:
 *   acc = +0; for c, for kh, for kw (c outermost, L10):
 *     xv = x[n, oy*stride - pad + kh, ox*stride - pad + kw, c] or +0 outside (L11, L14)
 *     acc = add(acc, mul(xv, w[kh, kw, c, m]))
 *   y = relu ? relu(acc) : acc                                              */
typedef struct {
    const uint32_t* x; const uint32_t* w; uint32_t* y;
    int n, h, wd, cin, kh, kw, cout, stride, pad, relu, we, wf, wf_out, mode;
    int ho, wo;
    int64_t lo, hi; /* output pixel range [lo, hi) over n*ho*wo */
} conv_job_t;

static uint32_t conv_one(const conv_job_t* J, int ni, int oy, int ox, int m) {
    uint32_t acc = enc_special(CLS_ZERO, 0, J->we, J->wf_out); /* L9: +0 */
    const uint32_t pad_word = enc_special(CLS_ZERO, 0, J->we, J->wf); /* L14: +0 */
    for (int c = 0; c < J->cin; c++)
        for (int a = 0; a < J->kh; a++)
            for (int b = 0; b < J->kw; b++) {
                int iy = oy * J->stride - J->pad + a;
                int ix = ox * J->stride - J->pad + b;
                uint32_t xv = pad_word;
                if (iy >= 0 && iy < J->h && ix >= 0 && ix < J->wd)
                    xv = J->x[(((int64_t)ni * J->h + iy) * J->wd + ix) * J->cin + c];
                uint32_t wv = J->w[(((int64_t)a * J->kw + b) * J->cin + c) * J->cout + m];
                uint32_t p = ref_mul(xv, wv, J->we, J->wf, J->wf_out, J->mode);
                acc = ref_add(acc, p, J->we, J->wf_out, J->mode);
            }
    return J->relu ? ref_relu(acc, J->we, J->wf_out) : acc;
}

static void* conv_worker(void* arg) {
    conv_job_t* J = (conv_job_t*)arg;
    for (int64_t p = J->lo; p < J->hi; p++) {
        int ox = (int)(p % J->wo);
        int oy = (int)((p / J->wo) % J->ho);
        int ni = (int)(p / ((int64_t)J->wo * J->ho));
        for (int m = 0; m < J->cout; m++) J->y[p * J->cout + m] = conv_one(J, ni, oy, ox, m);
    }
    return NULL;
}

/* Returns 0 on success, -1 on bad arguments. Every output chain is computed
 * serially by one thread; threads only split the set of output pixels. */
int ref_conv2d(const uint32_t* x, int n, int h, int wd, int cin,
               const uint32_t* w, int kh, int kw, int cout,
               int stride, int pad, int relu, int we, int wf, int wf_out, int mode,
               uint32_t* y, int nthreads) {
    if (n < 0 || h <= 0 || wd <= 0 || cin <= 0 || kh <= 0 || kw <= 0 || cout <= 0 || stride <= 0 || pad < 0)
        return -1;
    int ho = (h + 2 * pad - kh) / stride + 1, wo = (wd + 2 * pad - kw) / stride + 1;
    if (ho <= 0 || wo <= 0) return -1;
    int64_t npix = (int64_t)n * ho * wo;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    conv_job_t jobs[256];
    pthread_t th[256];
    for (int t = 0; t < nthreads; t++) {
        conv_job_t J = {x, w, y, n, h, wd, cin, kh, kw, cout, stride, pad, relu, we, wf, wf_out, mode,
                        ho, wo, npix * t / nthreads, npix * (t + 1) / nthreads};
        jobs[t] = J;
    }
    if (nthreads == 1) { conv_worker(&jobs[0]); return 0; }
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, conv_worker, &jobs[t]);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* ---------------- depthwise conv2d (the MobileNets
 * "Conv dw / s2" layer of P:255 / P:270 in its depthwise form) ----------------
 * x: NHWC words, C channels; w: [kh][kw][C] words (one kh x kw filter per
 * channel); y: [n][ho][wo][C].  For every output (n, oy, ox, m):
 *   acc = +0; for kh, for kw: acc = add(acc, mul(x[n, iy, ix, m] or +0, w[kh, kw, m]))
 *   y = relu ? relu(acc) : acc            (same MAC, order and padding rules as conv2d) */
static uint32_t conv_dw_one(const conv_job_t* J, int ni, int oy, int ox, int m) {
    uint32_t acc = enc_special(CLS_ZERO, 0, J->we, J->wf_out);
    const uint32_t pad_word = enc_special(CLS_ZERO, 0, J->we, J->wf);
    for (int a = 0; a < J->kh; a++)
        for (int b = 0; b < J->kw; b++) {
            int iy = oy * J->stride - J->pad + a;
            int ix = ox * J->stride - J->pad + b;
            uint32_t xv = pad_word;
            if (iy >= 0 && iy < J->h && ix >= 0 && ix < J->wd)
                xv = J->x[(((int64_t)ni * J->h + iy) * J->wd + ix) * J->cin + m];
            uint32_t wv = J->w[((int64_t)a * J->kw + b) * J->cin + m];
            acc = ref_add(acc, ref_mul(xv, wv, J->we, J->wf, J->wf_out, J->mode), J->we, J->wf_out, J->mode);
        }
    return J->relu ? ref_relu(acc, J->we, J->wf_out) : acc;
}

static void* conv_dw_worker(void* arg) {
    conv_job_t* J = (conv_job_t*)arg;
    for (int64_t p = J->lo; p < J->hi; p++) {
        int ox = (int)(p % J->wo);
        int oy = (int)((p / J->wo) % J->ho);
        int ni = (int)(p / ((int64_t)J->wo * J->ho));
        for (int m = 0; m < J->cin; m++) J->y[p * J->cin + m] = conv_dw_one(J, ni, oy, ox, m);
    }
    return NULL;
}

int ref_conv2d_dw(const uint32_t* x, int n, int h, int wd, int c, const uint32_t* w, int kh, int kw,
                  int stride, int pad, int relu, int we, int wf, int wf_out, int mode,
                  uint32_t* y, int nthreads) {
    if (n < 0 || h <= 0 || wd <= 0 || c <= 0 || kh <= 0 || kw <= 0 || stride <= 0 || pad < 0) return -1;
    int ho = (h + 2 * pad - kh) / stride + 1, wo = (wd + 2 * pad - kw) / stride + 1;
    if (ho <= 0 || wo <= 0) return -1;
    int64_t npix = (int64_t)n * ho * wo;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    conv_job_t jobs[256];
    pthread_t th[256];
    for (int t = 0; t < nthreads; t++) {
        conv_job_t J = {x, w, y, n, h, wd, c, kh, kw, c, stride, pad, relu, we, wf, wf_out, mode,
                        ho, wo, npix * t / nthreads, npix * (t + 1) / nthreads};
        jobs[t] = J;
    }
    if (nthreads == 1) { conv_dw_worker(&jobs[0]); return 0; }
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, conv_dw_worker, &jobs[t]);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
    return 0;
}

/* Sampled outputs at full size: idx[i] = ((ni*ho + oy)*wo + ox)*cout + m. */
int ref_conv2d_sample(const uint32_t* x, int n, int h, int wd, int cin,
                      const uint32_t* w, int kh, int kw, int cout,
                      int stride, int pad, int relu, int we, int wf, int wf_out, int mode,
                      const int64_t* idx, int64_t nidx, uint32_t* y) {
    int ho = (h + 2 * pad - kh) / stride + 1, wo = (wd + 2 * pad - kw) / stride + 1;
    if (ho <= 0 || wo <= 0) return -1;
    conv_job_t J = {x, w, y, n, h, wd, cin, kh, kw, cout, stride, pad, relu, we, wf, wf_out, mode, ho, wo, 0, 0};
    for (int64_t i = 0; i < nidx; i++) {
        int64_t q = idx[i];
        int m = (int)(q % cout);
        int64_t p = q / cout;
        int ox = (int)(p % wo);
        int oy = (int)((p / wo) % ho);
        int ni = (int)(p / ((int64_t)wo * ho));
        y[i] = conv_one(&J, ni, oy, ox, m);
    }
    return 0;
}
