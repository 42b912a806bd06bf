"""Weight-table entries for the prepared-weights MAC circuit (tests only).

Vectorised numpy statement of what one table entry holds (see
include/hobf.h hobf_wtab_words and gen/fpgen.product_from_table), used to
drive the generated ``mac_tab`` circuit on CPU so that circuit + table
semantics can be checked exhaustively against the oracle.
"""
from __future__ import annotations

import numpy as np


def row_of(x, we, wf):
    """Table row selected by activation word x: fraction if normal; 2^wf + 0/1/2 for zero/inf/NaN."""
    x = np.asarray(x, dtype=np.int64)
    exc = (x >> (wf + we + 1)) & 3
    fa = x & ((1 << wf) - 1)
    special = np.select([exc == 0, exc == 2, exc == 3], [0, 1, 2], 0)
    return np.where(exc == 1, fa, (1 << wf) + special)


def onehot(we, wfo):
    """Class encoding of an entry: one-hot (zero, normal, inf, NaN flags) when the
    two extra planes fit the 4-plane-rounded entry, else the 2-bit code K1 K0."""
    base = wfo + we + 5
    return -(-(base + 2) // 4) == -(-base // 4)


def entries(w, r, we, wf, rnd, wfo=None):
    """wfo = wF+1 (single class, rounded) or 2wF+1 (extended class, exact)."""
    w = np.asarray(w, dtype=np.int64)
    r = np.asarray(r, dtype=np.int64)
    wfo = wf + 1 if wfo is None else wfo
    EW = we + 2
    exc = (w >> (wf + we + 1)) & 3
    sw = (w >> (wf + we)) & 1
    eb = (w >> wf) & ((1 << we) - 1)
    fb = w & ((1 << wf) - 1)
    sbit = wfo + EW
    oh = onehot(we, wfo)
    NAN = (1 << (sbit + 4)) if oh else (1 << (sbit + 1)) | (1 << (sbit + 2))
    INF = (1 << (sbit + (3 if oh else 2))) | (sw << sbit)
    ZERO = ((1 << (sbit + 1)) if oh else 0) | (sw << sbit)
    NORM = 1 << (sbit + (2 if oh else 1))
    nrows = 1 << wf
    # both normal: exact product (1.fa)(1.fb), round to wfo fraction bits at its binade
    ma = (1 << wf) | np.minimum(r, nrows - 1)
    mb = (1 << wf) | fb
    P = ma * mb
    top = (P >> (2 * wf + 1)) & 1
    N = np.where(top == 1, P, P << 1)
    sh = 2 * wf + 1 - wfo
    kept = N >> sh
    if sh > 0 and rnd == 0:
        rem = N & ((1 << sh) - 1)
        half = 1 << (sh - 1)
        kept = kept + ((rem > half) | ((rem == half) & ((kept & 1) == 1)))
    inc = top.copy()
    carry = kept == (2 << wfo)
    kept = np.where(carry, kept >> 1, kept)
    inc = inc + carry
    frac = kept - (1 << wfo)
    bias = (1 << (we - 1)) - 1
    ep = (eb - bias + inc) & ((1 << EW) - 1)
    normal_e = frac | (ep << wfo) | (sw << sbit) | NORM
    out = np.select([exc == 0, exc == 2, exc == 3], [ZERO, INF, NAN], normal_e)
    out = np.where(r == nrows, np.where((exc & 2) != 0, NAN, ZERO), out)
    out = np.where(r == nrows + 1, np.where((exc == 0) | (exc == 3), NAN, INF), out)
    out = np.where(r == nrows + 2, NAN, out)
    return out.astype(np.uint32)


def circuit_inputs(acc, x, w, we, wf, rnd, wfo=None):
    """Arrays for build_mac_tab's inputs (acc, t, ea, sx) for lane-wise (acc, x, w)."""
    x = np.asarray(x, dtype=np.int64)
    t = entries(w, row_of(x, we, wf), we, wf, rnd, wfo)
    ea = ((x >> wf) & ((1 << we) - 1)).astype(np.uint32)
    sx = ((x >> (wf + we)) & 1).astype(np.uint32)
    return [np.asarray(acc, np.uint32), t, ea, sx]


def canon(words, we, wf):
    """Canonical form: exc != 01 -> exp = frac = 0; NaN -> sign 0."""
    v = np.asarray(words, dtype=np.int64)
    exc = (v >> (wf + we + 1)) & 3
    v = np.where(exc != 1, v & ~((1 << (wf + we)) - 1), v)
    v = np.where(exc == 3, v & ~(1 << (wf + we)), v)
    return v.astype(np.uint32)


def relax(words, we, wf, rng):
    """Scramble exp/frac of non-normal words (the chained accumulator's relaxed form)."""
    v = np.asarray(words, dtype=np.int64)
    exc = (v >> (wf + we + 1)) & 3
    junk = rng.integers(0, 1 << (wf + we), v.size)
    return np.where(exc != 1, v | junk, v).astype(np.uint32)
