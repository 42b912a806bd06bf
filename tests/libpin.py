"""Library-rounding pins for the oracle (tests only).

An independent vectorised computation of the HOBFLOPS operations using IEEE
float64 hardware arithmetic plus numpy's ``frexp`` / ``rint`` (ties-to-even) /
``floor``: the exact product or sum is formed in float64 (exact for the widths
pinned here, see each function), then rounded to p = wF_out + 1 significant
bits at its own binade, then classified into overflow (inf, ledger L5),
underflow (zero with sign, L6) or normal.  It shares nothing with
``oracle/hobf_ref.c`` except the format definition.
"""
from __future__ import annotations

import numpy as np


def bias(we):
    return (1 << (we - 1)) - 1


def fields(w, we, wf):
    w = np.asarray(w, dtype=np.int64)
    frac = w & ((1 << wf) - 1)
    e = (w >> wf) & ((1 << we) - 1)
    s = (w >> (wf + we)) & 1
    exc = (w >> (wf + we + 1)) & 3
    return exc, s, e, frac


def to_f64(w, we, wf):
    """Normal words -> exact float64 value (1 + f/2^wF) 2^(E-bias)."""
    exc, s, e, frac = fields(w, we, wf)
    mag = np.ldexp(1.0 + frac.astype(np.float64) / (1 << wf), (e - bias(we)).astype(np.int32))
    v = np.where(s == 1, -mag, mag)
    v = np.where(exc == 0, np.where(s == 1, -0.0, 0.0), v)
    v = np.where(exc == 2, np.where(s == 1, -np.inf, np.inf), v)
    v = np.where(exc == 3, np.nan, v)
    return v


def words_from(v, we, wf_out, mode):
    """Round exact float64 values v (nonzero finite) into F(we, wf_out); return words.

    RNE: q = rint(m * 2^p) with numpy's ties-to-even rint; RTZ: floor.  m, E from
    frexp (|v| = m 2^E, m in [0.5, 1))."""
    v = np.asarray(v, dtype=np.float64)
    s = np.signbit(v).astype(np.int64)
    a = np.abs(v)
    p = wf_out + 1
    m, E = np.frexp(a)
    scaled = np.ldexp(m, p)
    q = np.rint(scaled) if mode == 0 else np.floor(scaled)
    r = np.ldexp(q, E - p)                      # rounded magnitude (exact in float64)
    m2, E2 = np.frexp(r)
    Eb = E2.astype(np.int64) - 1 + bias(we)     # biased exponent of the rounded value
    frac = (np.ldexp(m2, p) - (1 << wf_out)).astype(np.int64)  # m2 in [0.5,1) -> p-bit int
    top = wf_out + we + 1
    normal = (1 << top) | (s << (wf_out + we)) | (np.clip(Eb, 0, (1 << we) - 1) << wf_out) | frac
    inf = (2 << top) | (s << (wf_out + we))
    zero = s << (wf_out + we)
    out = np.where(Eb > (1 << we) - 1, inf, np.where(Eb < 0, zero, normal))
    return out.astype(np.uint32)


def mul_normals(a, b, we, wf, wf_out, mode):
    """Both operands normal.  The product of two (wF+1)-bit significands has at
    most 2wF+2 <= 53 bits, so the float64 product is exact."""
    assert 2 * wf + 2 <= 53
    v = to_f64(a, we, wf) * to_f64(b, we, wf)
    return words_from(v, we, wf_out, mode)


def add_normals(a, b, we, wf, mode):
    """Both operands normal.  Returns (words, exact_mask): the float64 sum is exact
    when the exponent difference d satisfies d + wF + 2 <= 53 (exact_mask).  For
    RNE, inexact float64 sums are still correctly rounded to p = wF+1 <= 25 bits
    because double rounding through a 53-bit format is innocuous for +
    (53 >= 2p + 2); for RTZ only exact_mask lanes are meaningful."""
    va, vb = to_f64(a, we, wf), to_f64(b, we, wf)
    _, _, ea, _ = fields(a, we, wf)
    _, _, eb, _ = fields(b, we, wf)
    exact = np.abs(ea - eb) + wf + 2 <= 53
    v = va + vb
    out = np.where(v == 0, np.uint32(0), words_from(np.where(v == 0, 1.0, v), we, wf, mode))
    return out.astype(np.uint32), exact
