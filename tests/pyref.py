"""Independent exact-rational pin reference for the oracle (tests only).

Written separately from ``oracle/hobf_ref.c`` and by a different method: a
value is a ``fractions.Fraction`` (or a special tag), and rounding is done by
brute-force search for the nearest point of the format's value grid, not by
shifting an integer significand.  The grid is the set of normal values
(1 + f/2^wF) * 2^E for every integer E (unbounded exponent), so
"nearest grid point" is rounding at the value's own binade (SURVEY 8(c)
round_to); overflow/underflow are then classified from E (ledger L5, L6).

Special values are the strings 'nan', '+inf', '-inf', '+0', '-0'.
"""
from __future__ import annotations

from fractions import Fraction
import math

NAN, PINF, NINF, PZ, NZ = "nan", "+inf", "-inf", "+0", "-0"


def bias(we):
    return (1 << (we - 1)) - 1


def word_to_value(w, we, wf):
    """Decode a FloPoCo word [exc:2|s|exp:we|frac:wf]."""
    frac = w & ((1 << wf) - 1)
    e = (w >> wf) & ((1 << we) - 1)
    s = (w >> (wf + we)) & 1
    exc = (w >> (wf + we + 1)) & 3
    if exc == 0:
        return NZ if s else PZ
    if exc == 2:
        return NINF if s else PINF
    if exc == 3:
        return NAN
    mag = (1 + Fraction(frac, 1 << wf)) * Fraction(2) ** (e - bias(we))
    return -mag if s else mag


def value_to_word(v, we, wf):
    """Encode a value that is already representable (or special) as the canonical word."""
    top = wf + we + 1
    if v == NAN:
        return 3 << top
    if v in (PINF, NINF):
        return (2 << top) | ((1 if v == NINF else 0) << (wf + we))
    if v in (PZ, NZ):
        return (1 if v == NZ else 0) << (wf + we)
    s = 1 if v < 0 else 0
    m = abs(v)
    E = math.floor(math.log2(m))
    # fix floating-point log error by exact comparison
    while Fraction(2) ** E > m:
        E -= 1
    while Fraction(2) ** (E + 1) <= m:
        E += 1
    f = (m / Fraction(2) ** E - 1) * (1 << wf)
    assert f.denominator == 1, "value not representable"
    Eb = E + bias(we)
    assert 0 <= Eb < (1 << we)
    return (1 << top) | (s << (wf + we)) | (Eb << wf) | int(f)


def _binade(m):
    E = math.floor(math.log2(m)) if m > 0 else 0
    while Fraction(2) ** E > m:
        E -= 1
    while Fraction(2) ** (E + 1) <= m:
        E += 1
    return E


def round_value(r, we, wf, mode):
    """Round an exact nonzero Fraction r into F(we, wf): nearest grid point
    (ties to the point with even fraction, RNE) or the grid point toward zero
    (RTZ), found by searching the candidate grid points around r."""
    assert r != 0
    s = r < 0
    m = abs(r)
    E = _binade(m)
    # candidate grid points: every point of binade E plus 2^(E+1)
    step = Fraction(2) ** E / (1 << wf)
    cands = [(Fraction(2) ** E + k * step, E, k) for k in range(1 << wf)]
    cands.append((Fraction(2) ** (E + 1), E + 1, 0))
    if mode == 1:  # RTZ: largest candidate <= m
        best = max((c for c in cands if c[0] <= m), key=lambda c: c[0])
    else:
        dmin = min(abs(c[0] - m) for c in cands)
        ties = [c for c in cands if abs(c[0] - m) == dmin]
        if len(ties) == 1:
            best = ties[0]
        else:
            even = [c for c in ties if c[2] % 2 == 0]
            assert len(even) == 1
            best = even[0]
    val, Eo, _ = best
    Eb = Eo + bias(we)
    if Eb > (1 << we) - 1:
        return NINF if s else PINF
    if Eb < 0:
        return NZ if s else PZ
    return -val if s else val


def _is_zero(v):
    return v in (PZ, NZ)


def _is_inf(v):
    return v in (PINF, NINF)


def _sign(v):
    if v in (NZ, NINF):
        return 1
    if v in (PZ, PINF, NAN):
        return 0
    return 1 if v < 0 else 0


def mul(a, b, we, wf, wf_out, mode):
    """Product of two F(we,wf) words as an F(we,wf_out) word (ledger in hobf_ref.c)."""
    x, y = word_to_value(a, we, wf), word_to_value(b, we, wf)
    if x == NAN or y == NAN:
        return value_to_word(NAN, we, wf_out)
    if (_is_inf(x) and _is_zero(y)) or (_is_zero(x) and _is_inf(y)):
        return value_to_word(NAN, we, wf_out)
    s = _sign(x) ^ _sign(y)
    if _is_inf(x) or _is_inf(y):
        return value_to_word(NINF if s else PINF, we, wf_out)
    if _is_zero(x) or _is_zero(y):
        return value_to_word(NZ if s else PZ, we, wf_out)
    return value_to_word(round_value(x * y, we, wf_out, mode), we, wf_out)


def add(a, b, we, wf, mode):
    """Sum of two F(we,wf) words (L7 zero signs)."""
    x, y = word_to_value(a, we, wf), word_to_value(b, we, wf)
    if x == NAN or y == NAN:
        return value_to_word(NAN, we, wf)
    if _is_inf(x) and _is_inf(y):
        return value_to_word(x if x == y else NAN, we, wf)
    if _is_inf(x):
        return value_to_word(x, we, wf)
    if _is_inf(y):
        return value_to_word(y, we, wf)
    if _is_zero(x) and _is_zero(y):
        return value_to_word(NZ if (x == NZ and y == NZ) else PZ, we, wf)
    if _is_zero(x):
        return value_to_word(y, we, wf)
    if _is_zero(y):
        return value_to_word(x, we, wf)
    r = x + y
    if r == 0:
        return value_to_word(PZ, we, wf)
    return value_to_word(round_value(r, we, wf, mode), we, wf)


def relu(a, we, wf):
    x = word_to_value(a, we, wf)
    if x == NAN:
        return value_to_word(NAN, we, wf)
    if _is_zero(x) or _sign(x):
        return value_to_word(PZ, we, wf)
    return value_to_word(x, we, wf)


def encode_f32(f, we, wf, mode=0):
    """float32 -> format: exact rational of the float, then round."""
    import numpy as np
    f = np.float32(f)
    if np.isnan(f):
        return value_to_word(NAN, we, wf)
    if np.isinf(f):
        return value_to_word(NINF if f < 0 else PINF, we, wf)
    if f == 0:
        return value_to_word(NZ if np.signbit(f) else PZ, we, wf)
    return value_to_word(round_value(Fraction(float(f)), we, wf, mode), we, wf)


def canonical_words(we, wf):
    """Every canonical word of F(we, wf): +-0, +-inf, NaN and all normals."""
    top = wf + we + 1
    out = [0, 1 << (wf + we), 2 << top, (2 << top) | (1 << (wf + we)), 3 << top]
    for s in (0, 1):
        for e in range(1 << we):
            for f in range(1 << wf):
                out.append((1 << top) | (s << (wf + we)) | (e << wf) | f)
    return out


def conv2d(x, w, we, wf, wf_out, mode, stride=1, pad=1, relu_flag=0):
    """Direct conv over nested lists / numpy words, order (c, kh, kw)."""
    n, h, wd, cin = x.shape
    kh, kw, _, cout = w.shape
    ho = (h + 2 * pad - kh) // stride + 1
    wo = (wd + 2 * pad - kw) // stride + 1
    import numpy as np
    y = np.zeros((n, ho, wo, cout), np.uint32)
    pz = value_to_word(PZ, we, wf)
    for ni in range(n):
        for oy in range(ho):
            for ox in range(wo):
                for m in range(cout):
                    acc = value_to_word(PZ, we, wf_out)
                    for c in range(cin):
                        for a in range(kh):
                            for b in range(kw):
                                iy, ix = oy * stride - pad + a, ox * stride - pad + b
                                xv = int(x[ni, iy, ix, c]) if (0 <= iy < h and 0 <= ix < wd) else pz
                                p = mul(xv, int(w[a, b, c, m]), we, wf, wf_out, mode)
                                acc = add(acc, p, we, wf_out, mode)
                    y[ni, oy, ox, m] = relu(acc, we, wf_out) if relu_flag else acc
    return y
