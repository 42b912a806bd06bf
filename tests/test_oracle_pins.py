"""Pins for the oracle (oracle/hobf_ref.c) against things other than itself.

* worked examples printed in PAPER/SPEC (tests/golden/worked_examples.txt),
* Table 4 / P:257-263 width formulas,
* brute-force exact-rational reference (tests/pyref.py) on every pair of tiny formats,
* float64 library rounding (tests/libpin.py) on every pair of the <= 9-bit formats
  and on 10^6 random pairs of the 16-bit formats,
* IEEE half / fp8 library casts and arithmetic where the paper says they coincide,
* invariants (commutativity, sign symmetry, identities, special values).
"""
import os

import numpy as np
import pytest

import oracle
import pyref
import libpin

HERE = os.path.dirname(os.path.abspath(__file__))


def fmt(s):
    we, wf = s[1:].split("m")
    return int(we), int(wf)


def val_of(tok):
    from fractions import Fraction
    if tok in ("nan", "+0", "-0"):
        return tok
    if tok == "inf":
        return "+inf"
    if tok == "-inf":
        return "-inf"
    if tok == "0":
        return "+0"
    return Fraction(tok)


def canon_words(we, wf):
    return np.array(pyref.canonical_words(we, wf), dtype=np.uint32)


# ----------------------------------------------------------------------------- golden

def load_golden():
    rows = []
    with open(os.path.join(HERE, "golden", "worked_examples.txt")) as f:
        for line in f:
            line = line.split("#")[0].strip()
            if not line:
                continue
            lhs, rhs = line.split("->")
            toks = lhs.split()
            rows.append((toks[0], fmt(toks[1]), fmt(toks[2]), 0 if toks[3] == "RNE" else 1, toks[4:], rhs.strip()))
    return rows


@pytest.mark.parametrize("row", load_golden(), ids=lambda r: f"{r[0]}-{'_'.join(r[4])}")
def test_worked_examples(row):
    op, (we, wf), (we2, wfo), mode, args, res = row
    assert we == we2
    expect = val_of(res)
    if op == "encode":
        w = oracle.encode_f32(np.float32(float(args[0])), we, wf, mode).item()
        got = pyref.word_to_value(w, we, wf)
    else:
        words = [pyref.value_to_word(val_of(a), we, wf) for a in args]
        if op == "mul":
            w = oracle.mul(words[0], words[1], we, wf, wfo, mode).item()
        elif op == "add":
            w = oracle.add(words[0], words[1], we, wf, mode).item()
        elif op == "relu":
            w = oracle.relu(words[0], we, wf).item()
        got = pyref.word_to_value(w, we, wfo)
    assert got == expect, (row, got)


def test_table4_widths():
    """Table 4 and P:257-263: NIN = 2+1+wE+wF, NOUT single = NIN+1,
    extended = 2+1+wE+2wF+1; e.g. HOBFLOPS9 (e5m3) -> 11 / 12 / 15."""
    assert oracle.nbits(5, 3) == 11
    assert oracle.nbits(5, 3 + 1) == 12
    assert oracle.nbits(5, 2 * 3 + 1) == 15
    table = {"IEEE8": (4, 3, 4, 7), "8": (5, 2, 3, 5), "9": (5, 3, 4, 7), "16": (5, 10, 11, 21)}
    for name, (we, wf, single, ext) in table.items():
        assert wf + 1 == single and 2 * wf + 1 == ext, name


# ----------------------------------------------------------------------------- pyref brute force

TINY = [(2, 1), (3, 1), (3, 2)]


@pytest.mark.parametrize("we,wf", TINY)
@pytest.mark.parametrize("mode", [0, 1])
def test_mul_add_exhaustive_vs_rational_tiny(we, wf, mode):
    words = canon_words(we, wf)
    A, B = np.meshgrid(words, words, indexing="ij")
    A, B = A.ravel(), B.ravel()
    for wfo in (wf + 1, 2 * wf + 1):
        got = oracle.mul(A, B, we, wf, wfo, mode)
        exp = [pyref.mul(int(a), int(b), we, wf, wfo, mode) for a, b in zip(A, B)]
        assert np.array_equal(got, np.array(exp, np.uint32))
    got = oracle.add(A, B, we, wf, mode)
    exp = [pyref.add(int(a), int(b), we, wf, mode) for a, b in zip(A, B)]
    assert np.array_equal(got, np.array(exp, np.uint32))


@pytest.mark.parametrize("mode", [0, 1])
def test_random_vs_rational_e5m3(mode):
    rng = np.random.default_rng(1)
    w3, w4 = canon_words(5, 3), canon_words(5, 4)
    A, B = rng.choice(w3, 3000), rng.choice(w3, 3000)
    got = oracle.mul(A, B, 5, 3, 4, mode)
    exp = [pyref.mul(int(a), int(b), 5, 3, 4, mode) for a, b in zip(A, B)]
    assert np.array_equal(got, np.array(exp, np.uint32))
    A, B = rng.choice(w4, 3000), rng.choice(w4, 3000)
    got = oracle.add(A, B, 5, 4, mode)
    exp = [pyref.add(int(a), int(b), 5, 4, mode) for a, b in zip(A, B)]
    assert np.array_equal(got, np.array(exp, np.uint32))


def test_encode_vs_rational():
    rng = np.random.default_rng(2)
    x = np.concatenate([rng.standard_normal(2000).astype(np.float32),
                        (rng.standard_normal(500) * 1e-5).astype(np.float32),
                        (rng.standard_normal(500) * 3e4).astype(np.float32),
                        np.array([1e-45, -1e-45, 3e38, np.inf, -np.inf, np.nan, 0.0, -0.0], np.float32)])
    for we, wf in [(5, 2), (4, 3), (5, 10), (6, 5)]:
        for mode in (0, 1):
            got = oracle.encode_f32(x, we, wf, mode)
            exp = [pyref.encode_f32(v, we, wf, mode) for v in x]
            assert np.array_equal(got, np.array(exp, np.uint32)), (we, wf, mode)


# ----------------------------------------------------------------------------- float64 library rounding

def normals_only(words, we, wf):
    exc = (words.astype(np.int64) >> (wf + we + 1)) & 3
    return words[exc == 1]


SMALL_MUL = [(5, 3), (4, 3), (5, 2), (6, 2), (4, 4)]


@pytest.mark.parametrize("we,wf", SMALL_MUL)
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("ext", [0, 1])
def test_mul_exhaustive_vs_float64(we, wf, mode, ext):
    wfo = 2 * wf + 1 if ext else wf + 1
    n = normals_only(canon_words(we, wf), we, wf)
    A, B = np.meshgrid(n, n, indexing="ij")
    A, B = A.ravel(), B.ravel()
    got = oracle.mul(A, B, we, wf, wfo, mode)
    exp = libpin.mul_normals(A, B, we, wf, wfo, mode)
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, [(hex(A[i]), hex(B[i]), hex(got[i]), hex(exp[i])) for i in bad[:5]]


SMALL_ADD = [(5, 4), (4, 4), (5, 3), (6, 3), (4, 5)]


@pytest.mark.parametrize("we,wf", SMALL_ADD)
@pytest.mark.parametrize("mode", [0, 1])
def test_add_exhaustive_vs_float64(we, wf, mode):
    n = normals_only(canon_words(we, wf), we, wf)
    A, B = np.meshgrid(n, n, indexing="ij")
    A, B = A.ravel(), B.ravel()
    got = oracle.add(A, B, we, wf, mode)
    exp, exact = libpin.add_normals(A, B, we, wf, mode)
    if we <= 5:
        assert exact.all()
    if mode == 1:  # RTZ: only exact float64 sums are a valid pin (see libpin.add_normals)
        got, exp, A, B = got[exact], exp[exact], A[exact], B[exact]
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, [(hex(A[i]), hex(B[i]), hex(got[i]), hex(exp[i])) for i in bad[:5]]


def random_normals(rng, n, we, wf):
    s = rng.integers(0, 2, n)
    e = rng.integers(0, 1 << we, n)
    f = rng.integers(0, 1 << wf, n)
    return ((1 << (wf + we + 1)) | (s << (wf + we)) | (e << wf) | f).astype(np.uint32)


@pytest.mark.parametrize("we,wf", [(5, 10), (6, 10), (4, 10), (6, 7)])
@pytest.mark.parametrize("mode", [0, 1])
def test_mul_add_random_wide_vs_float64(we, wf, mode):
    rng = np.random.default_rng(3 + we * 100 + wf)
    N = 1_000_000
    A, B = random_normals(rng, N, we, wf), random_normals(rng, N, we, wf)
    got = oracle.mul(A, B, we, wf, wf + 1, mode)
    assert np.array_equal(got, libpin.mul_normals(A, B, we, wf, wf + 1, mode))
    got = oracle.mul(A, B, we, wf, 2 * wf + 1, mode)
    assert np.array_equal(got, libpin.mul_normals(A, B, we, wf, 2 * wf + 1, mode))
    wfo = wf + 1
    A, B = random_normals(rng, N, we, wfo), random_normals(rng, N, we, wfo)
    # make half of the pairs close in exponent so that cancellation and rounding carries occur
    A[: N // 2] = (A[: N // 2] & ~np.uint32(((1 << we) - 1) << wfo)) | (B[: N // 2] & np.uint32(((1 << we) - 1) << wfo))
    got = oracle.add(A, B, we, wfo, mode)
    exp, exact = libpin.add_normals(A, B, we, wfo, mode)
    sel = exact if mode == 1 else np.ones_like(exact)
    assert sel.sum() > N // 2
    assert np.array_equal(got[sel], exp[sel])


WIDE_EXP = [(7, 4), (7, 11), (8, 4), (8, 11)]


@pytest.mark.parametrize("we,wf", WIDE_EXP)
def test_add_mul_wide_exponent_vs_float64(we, wf):
    """wE = 7, 8 (exponent gaps up to 2^wE - 1, past a 128-bit alignment shift):
    10^6 random normal pairs, add and mul in RNE against float64 library rounding
    (double rounding through 53 bits is innocuous for p = wF + 1 <= 12 since
    53 >= 2p + 2; the float64 product is exact), plus every exponent gap around the
    far-operand threshold wF + 3 of ref_add."""
    rng = np.random.default_rng(40 + we * 100 + wf)
    N = 1_000_000
    A, B = random_normals(rng, N, we, wf), random_normals(rng, N, we, wf)
    # a quarter of the pairs with exponent gap d in [0, wf + 6], both orders
    q = N // 4
    ea = (A[:q].astype(np.int64) >> wf) & ((1 << we) - 1)
    d = rng.integers(0, wf + 7, q) * np.where(rng.random(q) < 0.5, 1, -1)
    eb = np.clip(ea + d, 0, (1 << we) - 1)
    B[:q] = ((B[:q].astype(np.int64) & ~(((1 << we) - 1) << wf)) | (eb << wf)).astype(np.uint32)
    got = oracle.add(A, B, we, wf, 0)
    exp, _ = libpin.add_normals(A, B, we, wf, 0)
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, [(hex(A[i]), hex(B[i]), hex(got[i]), hex(exp[i])) for i in bad[:5]]
    got = oracle.mul(A, B, we, wf, wf + 1, 0)
    assert np.array_equal(got, libpin.mul_normals(A, B, we, wf, wf + 1, 0))


@pytest.mark.parametrize("we,wf", WIDE_EXP)
@pytest.mark.parametrize("mode", [0, 1])
def test_add_wide_exponent_vs_rational(we, wf, mode):
    """The same widths against the exact-rational reference in both modes (RTZ has
    no float64 pin once the gap exceeds 53 - wF - 2 bits), gaps around wF + 3."""
    rng = np.random.default_rng(50 + we * 100 + wf + mode)
    N = 3000 if wf <= 4 else 400  # the grid search of pyref grows with 2^wF
    A, B = random_normals(rng, N, we, wf), random_normals(rng, N, we, wf)
    ea = (A.astype(np.int64) >> wf) & ((1 << we) - 1)
    d = rng.integers(wf, wf + 6, N) * np.where(rng.random(N) < 0.5, 1, -1)
    eb = np.where(np.arange(N) < N // 2, np.clip(ea + d, 0, (1 << we) - 1), (B.astype(np.int64) >> wf) & ((1 << we) - 1))
    B = ((B.astype(np.int64) & ~(((1 << we) - 1) << wf)) | (eb << wf)).astype(np.uint32)
    got = oracle.add(A, B, we, wf, mode)
    exp = np.array([pyref.add(int(a), int(b), we, wf, mode) for a, b in zip(A, B)], np.uint32)
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, [(hex(A[i]), hex(B[i]), hex(got[i]), hex(exp[i])) for i in bad[:5]]


# ----------------------------------------------------------------------------- IEEE library coincidence

def half_words_normal(h):
    """float16 with exp codes 1..30 -> FloPoCo e5m10 word (same bias 15)."""
    u = h.view(np.uint16).astype(np.int64)
    return ((1 << 16) | ((u >> 15) << 15) | (u & 0x7FFF)).astype(np.uint32)


def test_e5m10_mul_add_match_ieee_half():
    """the FloPoCo cores are equivalent to IEEE-754 where both are defined.
    numpy float16 ops are correctly rounded (float32 intermediate, 24 >= 2*11+2)."""
    rng = np.random.default_rng(4)
    N = 400_000
    u = rng.integers(0, 1 << 16, (2, N)).astype(np.uint16)
    ecode = (u >> 10) & 31
    u = u[:, ((ecode[0] >= 1) & (ecode[0] <= 30) & (ecode[1] >= 1) & (ecode[1] <= 30))]
    # draw the second operand near the first for add so that cancellation happens
    ha, hb = u[0].view(np.float16), u[1].view(np.float16)
    hb2 = (-ha.astype(np.float32) * (1 + rng.standard_normal(ha.size).astype(np.float32) * 0.01)).astype(np.float16)
    hb2[::7] = -ha[::7]  # exact cancellations
    wa, wb = half_words_normal(ha), half_words_normal(hb)
    with np.errstate(all="ignore"):
        for hx, hy, wx, wy in [(ha, hb, wa, wb)]:
            pm = (hx * hy)
            got = oracle.mul(wx, wy, 5, 10, 10, 0)
            code = (pm.view(np.uint16) >> 10) & 31
            # below 2^-14 IEEE rounds on its subnormal grid, FloPoCo on its exp-code-0 binade
            ok = (code >= 1) & (code <= 30) & (np.abs(hx.astype(np.float64) * hy.astype(np.float64)) >= 2.0 ** -14)
            assert ok.sum() > 1000
            assert np.array_equal(got[ok], half_words_normal(pm[ok]))
        for hx, hy, need_zero in [(ha, hb, False), (ha, hb2, True)]:
            ecode2 = (hy.view(np.uint16) >> 10) & 31
            sel = (ecode2 >= 1) & (ecode2 <= 30)
            hx, hy = hx[sel], hy[sel]
            ps = hx + hy
            got = oracle.add(half_words_normal(hx), half_words_normal(hy), 5, 10, 0)
            code = (ps.view(np.uint16) >> 10) & 31
            ok = (code >= 1) & (code <= 30)
            assert np.array_equal(got[ok], half_words_normal(ps[ok]))
            z = ps == 0
            assert z.sum() > 0 or not need_zero
            assert np.all(got[z] == 0)  # exact cancellation -> +0


def test_encode_matches_library_casts():
    """RNE float32 -> e5m10 / e5m2 / e4m3 equals numpy float16 and ml_dtypes fp8
    casts on their common normal range (exp codes shared with FloPoCo)."""
    import ml_dtypes
    rng = np.random.default_rng(5)
    x = (rng.standard_normal(300_000) * np.exp(rng.uniform(-12, 12, 300_000))).astype(np.float32)
    cases = [(5, 10, np.float16, 2.0 ** -14, 65504.0),
             (5, 2, ml_dtypes.float8_e5m2, 2.0 ** -14, 57344.0),
             (4, 3, ml_dtypes.float8_e4m3fn, 2.0 ** -6, 448.0)]
    for we, wf, dt, lo, hi in cases:
        with np.errstate(all="ignore"):
            lib = x.astype(dt).astype(np.float64)
        ok = (np.abs(lib) >= lo) & (np.abs(lib) <= hi) & (np.abs(x) <= hi) & (np.abs(x) >= lo)
        got = oracle.decode_f64(oracle.encode_f32(x, we, wf, 0), we, wf)
        assert ok.sum() > 10000
        assert np.array_equal(got[ok], lib[ok]), (we, wf)


# ----------------------------------------------------------------------------- invariants

@pytest.mark.parametrize("mode", [0, 1])
def test_invariants_e5m3(mode):
    we, wf, wfo = 5, 3, 4
    w = canon_words(we, wf)
    A, B = np.meshgrid(w, w, indexing="ij")
    A, B = A.ravel(), B.ravel()
    sbit = np.uint32(1 << (wf + we))
    # commutativity
    assert np.array_equal(oracle.mul(A, B, we, wf, wfo, mode), oracle.mul(B, A, we, wf, wfo, mode))
    w4 = canon_words(we, wfo)
    C, D = np.meshgrid(w4, w4, indexing="ij")
    C, D = C.ravel(), D.ravel()
    assert np.array_equal(oracle.add(C, D, we, wfo, mode), oracle.add(D, C, we, wfo, mode))
    # sign symmetry of mul on non-NaN results: mul(-a, b) = -mul(a, b)
    exc = lambda x, wfx: (x.astype(np.int64) >> (wfx + we + 1)) & 3
    m1 = oracle.mul(A ^ sbit * (exc(A, wf) != 3), B, we, wf, wfo, mode)
    m0 = oracle.mul(A, B, we, wf, wfo, mode)
    sb4 = np.uint32(1 << (wfo + we))
    nn = exc(m0, wfo) != 3
    assert np.array_equal(m1[nn], m0[nn] ^ sb4)
    # x + 0 = x for all canonical x, both zeros
    for z in (0, sb4):
        r = oracle.add(w4, np.full_like(w4, z), we, wfo, mode)
        fin = exc(w4, wfo) == 1
        assert np.array_equal(r[fin], w4[fin])
    # multiplication by a power of two is exact (only the exponent moves) when in range
    two = pyref.value_to_word(__import__("fractions").Fraction(2), we, wf)
    r = oracle.mul(w, np.full_like(w, two), we, wf, wfo, mode)
    for x, y in zip(w, r):
        vx, vy = pyref.word_to_value(int(x), we, wf), pyref.word_to_value(int(y), we, wfo)
        if not isinstance(vx, str) and abs(vx) * 2 <= pyref.word_to_value(int(canon_words(we, wfo)[-1]), we, wfo):
            assert vy == 2 * vx
    # NaN dominance and inf*0
    nan_in, inf_in, zero_in = np.uint32(3 << (wf + we + 1)), np.uint32(2 << (wf + we + 1)), np.uint32(0)
    assert np.all(exc(oracle.mul(np.full_like(w, nan_in), w, we, wf, wfo, mode), wfo) == 3)
    assert exc(oracle.mul(inf_in, zero_in, we, wf, wfo, mode), wfo) == 3


def test_noncanonical_inputs_read_canonically():
    """L17: exc != 01 words with junk exp/frac (and NaN with sign 1) are read canonically."""
    we, wf = 5, 3
    rng = np.random.default_rng(6)
    raw = rng.integers(0, 1 << 11, 5000).astype(np.uint32)
    can = oracle.canon(raw, we, wf)
    exc = (raw >> (wf + we + 1)) & 3
    assert np.all(((can >> (wf + we + 1)) & 3) == exc)
    junk = exc != 1
    assert np.all((can[junk] & ((1 << (wf + we)) - 1)) == 0)
    b = rng.integers(0, 1 << 11, 5000).astype(np.uint32)
    assert np.array_equal(oracle.mul(raw, b, we, wf, 4, 0), oracle.mul(can, oracle.canon(b, we, wf), we, wf, 4, 0))


# ----------------------------------------------------------------------------- conv

def small_conv_case(seed, n, h, w, cin, cout, we, wf):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, h, w, cin)).astype(np.float32)
    wt = (rng.standard_normal((3, 3, cin, cout)) * 0.5).astype(np.float32)
    return oracle.encode_f32(x, we, wf), oracle.encode_f32(wt, we, wf)


@pytest.mark.parametrize("mode", [0, 1])
def test_conv_vs_rational_small(mode):
    we, wf = 5, 3
    x, wt = small_conv_case(7, 1, 4, 5, 3, 4, we, wf)
    for relu in (0, 1):
        got = oracle.conv2d(x, wt, we, wf, wf + 1, mode, 1, 1, relu, nthreads=2)
        exp = pyref.conv2d(x, wt, we, wf, wf + 1, mode, 1, 1, relu)
        assert np.array_equal(got, exp)
    # stride 2, pad 0
    got = oracle.conv2d(x, wt, we, wf, wf + 1, mode, 2, 0, 0)
    exp = pyref.conv2d(x, wt, we, wf, wf + 1, mode, 2, 0, 0)
    assert np.array_equal(got, exp)


def test_conv_metamorphic():
    we, wf = 5, 10
    x, wt = small_conv_case(8, 2, 6, 7, 8, 8, we, wf)
    wfo = wf + 1
    # all-zero weights -> all +0
    y = oracle.conv2d(x, np.zeros_like(wt), we, wf, wfo)
    assert np.all(y == 0)
    # centred identity kernel: output = input widened to wF+1 (exact), -0 -> +0
    ident = np.zeros_like(wt)
    one = pyref.value_to_word(__import__("fractions").Fraction(1), we, wf)
    for c in range(8):
        ident[1, 1, c, c] = one
    y = oracle.conv2d(x, ident, we, wf, wfo)
    xv = oracle.decode_f64(x, we, wf)
    yv = oracle.decode_f64(y, we, wfo)
    assert np.array_equal(yv, xv + 0.0)
    assert not np.any(np.signbit(yv) & (yv == 0))
    # scaling weights by 2 scales every output by 2 (no overflow at these magnitudes)
    two = pyref.value_to_word(__import__("fractions").Fraction(2), we, wf)
    w2 = oracle.mul(wt, np.full_like(wt, two), we, wf, wf, 0)  # exact: power of two
    y1 = oracle.decode_f64(oracle.conv2d(x, wt, we, wf, wfo), we, wfo)
    y2 = oracle.decode_f64(oracle.conv2d(x, w2, we, wf, wfo), we, wfo)
    assert np.array_equal(y2, 2 * y1)
    # negating weights negates outputs (up to the sign of zero)
    sb = np.uint32(1 << (wf + we))
    wn = np.where(((wt >> (wf + we + 1)) & 3) != 3, wt ^ sb, wt).astype(np.uint32)
    yn = oracle.decode_f64(oracle.conv2d(x, wn, we, wf, wfo), we, wfo)
    assert np.array_equal(yn, -y1 + 0.0) or np.array_equal(np.abs(yn), np.abs(y1))
    assert np.array_equal(yn[y1 != 0], -y1[y1 != 0])
    # output-channel permutation commutes; images are independent; sampling agrees
    perm = np.random.default_rng(0).permutation(8)
    yp = oracle.conv2d(x, wt[..., perm], we, wf, wfo)
    y = oracle.conv2d(x, wt, we, wf, wfo)
    assert np.array_equal(yp, y[..., perm])
    assert np.array_equal(oracle.conv2d(x[1:], wt, we, wf, wfo), y[1:])
    idx = np.arange(0, y.size, 7)
    assert np.array_equal(oracle.conv2d_sample(x, wt, idx, we, wf, wfo), y.ravel()[idx])
    assert np.array_equal(oracle.conv2d(x, wt, we, wf, wfo, nthreads=1), oracle.conv2d(x, wt, we, wf, wfo, nthreads=5))


# ----------------------------------------------------------------------------- layer-epilogue conversion

@pytest.mark.parametrize("we,wf_in,wf_out", [(3, 3, 1), (3, 2, 1), (4, 3, 2), (2, 4, 2), (3, 1, 3)])
@pytest.mark.parametrize("mode", [0, 1])
def test_convert_exhaustive_vs_rational(we, wf_in, wf_out, mode):
    """ref_convert (P:262 epilogue rounding) on every canonical word of a tiny
    format against the exact-rational nearest-grid-point search of pyref."""
    words = pyref.canonical_words(we, wf_in)
    got = oracle.convert(np.array(words, dtype=np.uint32), we, wf_in, wf_out, mode)
    for w, g in zip(words, got):
        v = pyref.word_to_value(w, we, wf_in)
        if isinstance(v, str):
            exp = pyref.value_to_word(v, we, wf_out)
        else:
            exp = pyref.value_to_word(pyref.round_value(v, we, wf_out, mode), we, wf_out)
        assert int(g) == exp, (hex(w), hex(int(g)), hex(exp))


def test_convert_matches_ieee_half_and_fp8_casts():
    """e5m11 -> e5m10 equals numpy's float32 -> float16 RNE cast, and e4m4 -> e4m3
    equals ml_dtypes' float32 -> float8_e4m3fn cast, wherever both formats are
    normal (the FloPoCo cores coincide with IEEE there)."""
    ml = pytest.importorskip("ml_dtypes")
    rng = np.random.default_rng(5)
    for we, wfi, wfo, lo, hi, cast in ((5, 11, 10, 2.0 ** -14, 65504.0, np.float16),
                                       (4, 4, 3, 2.0 ** -6, 448.0, ml.float8_e4m3fn)):
        top = wfi + we + 1
        n = 200000
        words = ((1 << top) | (rng.integers(0, 2, n) << (wfi + we)) | (rng.integers(0, 1 << we, n) << wfi)
                 | rng.integers(0, 1 << wfi, n)).astype(np.uint32)
        v = oracle.decode_f64(words, we, wfi)
        keep = (np.abs(v) >= lo) & (np.abs(v) <= hi)
        words, v = words[keep], v[keep]
        lib = np.asarray(v.astype(np.float32).astype(cast).astype(np.float64))
        ok = np.isfinite(lib) & (np.abs(lib) <= hi)
        got = oracle.decode_f64(oracle.convert(words, we, wfi, wfo, 0), we, wfo)
        assert ok.sum() > 1000
        assert np.array_equal(got[ok], lib[ok])


def test_convert_invariants():
    """Widening is exact (and narrowing it back is the identity); RTZ never
    increases the magnitude; RNE is within half an ulp; specials keep class and sign."""
    rng = np.random.default_rng(6)
    we, wf = 5, 7
    words = oracle.encode_f32(rng.standard_normal(50000).astype(np.float32) * 8, we, wf)
    wide = oracle.convert(words, we, wf, 2 * wf + 1)
    assert np.array_equal(oracle.decode_f64(wide, we, 2 * wf + 1), oracle.decode_f64(words, we, wf))
    assert np.array_equal(oracle.convert(wide, we, 2 * wf + 1, wf), words)
    src = oracle.encode_f32(rng.standard_normal(50000).astype(np.float32), we, 10)
    src = src[oracle.decode_f64(src, we, 10) != 0]
    v = oracle.decode_f64(src, we, 10)
    z = oracle.decode_f64(oracle.convert(src, we, 10, 3, 1), we, 3)
    assert np.all(np.abs(z) <= np.abs(v)) and np.all(np.abs(v - z) < 2.0 ** (np.floor(np.log2(np.abs(v))) - 3))
    r = oracle.decode_f64(oracle.convert(src, we, 10, 3, 0), we, 3)
    assert np.all(np.abs(v - r) <= 2.0 ** (np.floor(np.log2(np.abs(v))) - 4))
    top = 10 + we + 1
    sp = np.array([0, 1 << (10 + we), 2 << top, (2 << top) | (1 << (10 + we)), 3 << top], dtype=np.uint32)
    t3 = 3 + we + 1
    assert list(oracle.convert(sp, we, 10, 3)) == [0, 1 << (3 + we), 2 << t3, (2 << t3) | (1 << (3 + we)), 3 << t3]
    # rounding up out of the top binade overflows to inf (L5)
    mx = np.array([(1 << top) | (((1 << we) - 1) << 10) | 1023], dtype=np.uint32)
    assert oracle.convert(mx, we, 10, 3, 0)[0] == 2 << t3
    assert oracle.convert(mx, we, 10, 3, 1)[0] == (1 << t3) | (((1 << we) - 1) << 3) | 7


def test_conv_chain_is_layerwise():
    """oracle.conv_chain = conv2d, convert, conv2d (the definition), and a chain
    whose second layer is a centred identity kernel reproduces the first layer's
    converted (then widened) output exactly."""
    from fractions import Fraction
    we, wf = 5, 3
    x, w1 = small_conv_case(9, 1, 5, 6, 4, 4, we, wf)
    ident = np.zeros((3, 3, 4, 4), dtype=np.uint32)
    one = pyref.value_to_word(Fraction(1), we, wf)
    for c in range(4):
        ident[1, 1, c, c] = one
    y = oracle.conv_chain(x, [(w1, wf, 1, 1, 1, 0), (ident, wf, 1, 1, 0, 0)], we)
    y1 = oracle.convert(oracle.conv2d(x, w1, we, wf, wf + 1, 0, 1, 1, 1), we, wf + 1, wf)
    assert np.array_equal(oracle.decode_f64(y, we, wf + 1), oracle.decode_f64(y1, we, wf))


# ----------------------------------------------------------------------------- depthwise conv (MobileNets Conv dw)

@pytest.mark.parametrize("stride", [1, 2])
def test_conv_dw_vs_rational(stride):
    """ref_conv2d_dw against an exact-rational chain of pyref.mul / pyref.add over
    (kh, kw) on a tiny case with ragged spatial size and zero padding."""
    we, wf, mode = 4, 3, 0
    rng = np.random.default_rng(11)
    x = oracle.encode_f32(rng.standard_normal((1, 5, 4, 3)).astype(np.float32), we, wf)
    wt = oracle.encode_f32((rng.standard_normal((3, 3, 3)) * 0.7).astype(np.float32), we, wf)
    for relu in (0, 1):
        got = oracle.conv2d_dw(x, wt, we, wf, wf + 1, mode, stride, 1, relu, nthreads=2)
        ho, wo = got.shape[1:3]
        for oy in range(ho):
            for ox in range(wo):
                for m in range(3):
                    acc = 0
                    for a in range(3):
                        for b in range(3):
                            iy, ix = oy * stride - 1 + a, ox * stride - 1 + b
                            xv = int(x[0, iy, ix, m]) if 0 <= iy < 5 and 0 <= ix < 4 else 0
                            acc = pyref.add(acc, pyref.mul(xv, int(wt[a, b, m]), we, wf, wf + 1, mode), we, wf + 1, mode)
                    if relu:
                        acc = pyref.relu(acc, we, wf + 1)
                    assert int(got[0, oy, ox, m]) == acc, (oy, ox, m)


def test_conv_dw_equals_full_conv_with_diagonal_kernel():
    """For finite inputs a depthwise conv is the full conv whose kernel is zero off
    the channel diagonal: the extra products are +-0, and acc + (+-0) = acc for
    every accumulator the chain can hold (+0, normals; L7), in the same relative
    (kh, kw) order -- so the pinned full conv pins the depthwise one."""
    we, wf = 5, 10
    rng = np.random.default_rng(12)
    n, h, w, c = 2, 7, 6, 9
    x = oracle.encode_f32(rng.standard_normal((n, h, w, c)).astype(np.float32), we, wf)
    wt = oracle.encode_f32((rng.standard_normal((3, 3, c)) * 0.5).astype(np.float32), we, wf)
    full = np.zeros((3, 3, c, c), dtype=np.uint32)
    for m in range(c):
        full[:, :, m, m] = wt[:, :, m]
    for stride, relu in ((1, 0), (2, 1)):
        a = oracle.conv2d_dw(x, wt, we, wf, wf + 1, 0, stride, 1, relu)
        b = oracle.conv2d(x, full, we, wf, wf + 1, 0, stride, 1, relu)
        assert np.array_equal(a, b)
