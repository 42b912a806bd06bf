"""Gate-level HOBFLOPS floating-point multiplier and adder (the FloPoCo + Genus
stage of the paper's flow, rebuilt in-repo).

Every circuit is built as an AIG (``aig.AIG``).  Bit vectors are Python lists
of literals, least significant bit first.

Operand format F(wE, wF): word bits [exc:2 | sign | exp:wE | frac:wF]
MSB..LSB; exc 00 zero, 01 normal, 10 inf, 11 NaN; significand 1.f; bias
2^(wE-1)-1; every exponent code is a normal binade (no subnormals).
Product / accumulator width: wF+1 (single) or 2wF+1 (extended) (Table 4,
P:151-177).  Rounding: RNE or RTZ.

The circuits assume canonical operands (exc != 01 => exp = frac = 0, NaN
sign 0), which pack/quantise guarantee and which every circuit output
satisfies; this don't-care is what lets zero operands flow through the adder
datapath without a bypass (see ``fp_add``).
"""
from __future__ import annotations

from .aig import AIG, FALSE, TRUE

RNE = 0
RTZ = 1


def bias(we: int) -> int:
    return (1 << (we - 1)) - 1


class FP:
    """Field view of an encoded word given as a list of literals."""

    def __init__(self, bits, we, wf):
        assert len(bits) == 3 + we + wf
        self.we, self.wf = we, wf
        self.frac = bits[0:wf]
        self.exp = bits[wf:wf + we]
        self.sign = bits[wf + we]
        self.exc0 = bits[wf + we + 1]
        self.exc1 = bits[wf + we + 2]


def pack_bits(frac, exp, sign, exc0, exc1):
    return list(frac) + list(exp) + [sign, exc0, exc1]


# --------------------------------------------------------------------------- integer blocks

def ripple_add(g: AIG, a, b, cin=FALSE, width=None):
    """a + b + cin (LSB first); returns width bits (default max(len)+1)."""
    n = max(len(a), len(b))
    if width is None:
        width = n + 1
    a = list(a) + [FALSE] * (width - len(a))
    b = list(b) + [FALSE] * (width - len(b))
    out = []
    c = cin
    for i in range(width):
        out.append(g.XOR3(a[i], b[i], c))
        if i < width - 1:
            c = g.MAJ(a[i], b[i], c)
    return out


def increment(g: AIG, a, inc, width=None):
    """a + inc (single bit); returns (bits[width], carry_out)."""
    if width is None:
        width = len(a)
    out = []
    c = inc
    for i in range(width):
        ai = a[i] if i < len(a) else FALSE
        out.append(g.XOR(ai, c))
        c = g.AND(ai, c)
    return out, c


def const_bits(value: int, width: int):
    return [TRUE if (value >> i) & 1 else FALSE for i in range(width)]


def less_than(g: AIG, a, b):
    """unsigned a < b (borrow out of a - b)."""
    br = FALSE
    for ai, bi in zip(a, b):
        br = g.MAJ(g.NOT(ai), bi, br)
    return br


def multiply(g: AIG, a, b):
    """Unsigned array multiplier (AND partial products, column compression with
    full/half adders, final ripple adder).  Returns len(a)+len(b) bits."""
    W = len(a) + len(b)
    cols = [[] for _ in range(W + 1)]
    for j, bj in enumerate(b):
        for i, ai in enumerate(a):
            p = g.AND(ai, bj)
            if p != FALSE:
                cols[i + j].append(p)
    # Dadda-style reduction to two rows
    while max(len(c) for c in cols) > 2:
        new = [[] for _ in range(W + 1)]
        for k in range(W):
            col = cols[k]
            while len(col) >= 3:
                x, y, z = col.pop(0), col.pop(0), col.pop(0)
                new[k].append(g.XOR3(x, y, z))
                new[k + 1].append(g.MAJ(x, y, z))
            new[k].extend(col)
        cols = new
    r0 = [c[0] if len(c) > 0 else FALSE for c in cols[:W]]
    r1 = [c[1] if len(c) > 1 else FALSE for c in cols[:W]]
    return ripple_add(g, r0, r1, FALSE, width=W)


def shift_right_sticky(g: AIG, v, d, order="small_first", kill=FALSE, clamp=False):
    """Logical right shift of v (LSB first) by the unsigned amount d (bits LSB
    first); returns (shifted, sticky) where sticky = OR of all bits shifted out.
    If ``kill`` is true the result and the sticky are forced to zero.

    clamp=True: a shift of 2^K - 1 >= len(v) already moves every bit into the
    sticky, so amounts >= 2^K (and ``kill``) are clamped to 2^K - 1 by OR-ing
    the high / kill bits into the K low shift bits, and ``kill`` then only has
    to clear the sticky -- instead of clearing every shifted bit."""
    W = len(v)
    K = 0
    while (1 << K) <= W:
        K += 1
    K = min(K, len(d))
    if clamp:
        hi = g.OR(g.OR_many(d[K:]), kill)
        dd = [g.OR(d[j], hi) for j in range(K)]
        cur, sticky = shift_right_sticky(g, v, dd, order=order)
        return cur, g.AND(sticky, g.NOT(kill))
    big = g.OR(g.OR_many(d[K:]), kill)
    cur = list(v)
    sticky = FALSE
    stages = list(range(K)) if order == "small_first" else list(reversed(range(K)))
    for j in stages:
        sh = 1 << j
        out_bits = g.OR_many(cur[:sh])
        sticky = g.OR(sticky, g.AND(d[j], out_bits))
        cur = [g.MUX(d[j], cur[i + sh] if i + sh < W else FALSE, cur[i]) for i in range(W)]
    if big != FALSE:
        anyv = g.AND(g.OR_many(v), g.NOT(kill))
        sticky = g.MUX(big, anyv, sticky)
        cur = [g.AND(g.NOT(big), x) for x in cur]
    return cur, sticky


def lzc(g: AIG, v):
    """Leading-zero count of v (LSB first; leading = from the MSB).  Returns
    (count bits LSB first, all_zero)."""
    n = len(v)
    P = 1
    while P < n:
        P *= 2
    msb_first = list(reversed(v)) + [FALSE] * (P - n)  # pad at the bottom (LSB side)

    def rec(bits):
        # returns (count bits LSB first over log2(len) bits, zero flag)
        if len(bits) == 1:
            return [], g.NOT(bits[0])
        h = len(bits) // 2
        ch, zh = rec(bits[:h])
        cl, zl = rec(bits[h:])
        cnt = [g.MUX(zh, cl[i], ch[i]) for i in range(len(ch))] + [zh]
        return cnt, g.AND(zh, zl)

    cnt, z = rec(msb_first)
    return cnt, z


def normalize_left(g: AIG, v, max_shift=None, low_zero=(0, 0)):
    """Leading-zero normalisation by successive detection: for 2^j from the
    largest power of two down, if the top 2^j bits of the current vector are
    all zero, shift it left by 2^j.  Returns (normalised v, shift count bits
    LSB first, all_zero).  Same result as lzc + shift_left, fewer gates.

    ``max_shift``: a bound on the shift any nonzero input needs (its leading
    one is never below bit L-1-max_shift); only bitlen(max_shift) stages are
    built.  all_zero stays exact: a nonzero input always ends with its leading
    one at the top.

    ``low_zero = (nbits, min_shift)``: whenever a stage shifting by >= min_shift
    shifts, the input's low nbits are zero (an invariant of the caller), so
    those output bits pass through without a gate."""
    L = len(v)
    K = 0
    if max_shift is None:
        max_shift = L - 1
    while (1 << K) <= max_shift:
        K += 1
    cur = list(v)
    cnt = [FALSE] * K
    for j in reversed(range(K)):
        sh = 1 << j
        zj = g.NOT(g.OR_many(cur[L - sh:]))
        cnt[j] = zj
        nlow = low_zero[0] if sh >= low_zero[1] > 0 else 0
        cur = [cur[i] if i < nlow else g.MUX(zj, cur[i - sh] if i - sh >= 0 else FALSE, cur[i]) for i in range(L)]
    return cur, cnt, g.NOT(cur[L - 1])


def shift_left(g: AIG, v, s):
    cur = list(v)
    W = len(v)
    for j in reversed(range(len(s))):
        sh = 1 << j
        if sh >= W:
            cur = [g.AND(g.NOT(s[j]), x) for x in cur]
            continue
        cur = [g.MUX(s[j], cur[i - sh] if i - sh >= 0 else FALSE, cur[i]) for i in range(W)]
    return cur


# --------------------------------------------------------------------------- FP multiplier

def fp_mul(g: AIG, A: FP, B: FP, wfo: int, rnd: int):
    """HOBFLOPS multiplier F(wE,wF) x F(wE,wF) -> F(wE,wfo) (Table 4).

    Exception combine, sign XOR, (wF+1)^2 significand product with the hidden
    bit wired to 1 (non-normal operands are overridden by the exception logic),
    1-bit normalisation, round to wfo fraction bits (RNE / RTZ), exponent
    Ea + Eb - bias + norm + round-carry at wE+2 bits, overflow -> inf,
    underflow -> zero (SURVEY 8(c) mul, ledger L5/L6)."""
    we, wf = A.we, A.wf
    assert wfo >= wf
    nA, nB = g.AND(A.exc1, A.exc0), g.AND(B.exc1, B.exc0)
    iA, iB = g.AND(A.exc1, g.NOT(A.exc0)), g.AND(B.exc1, g.NOT(B.exc0))
    zA, zB = g.AND(g.NOT(A.exc1), g.NOT(A.exc0)), g.AND(g.NOT(B.exc1), g.NOT(B.exc0))
    normA, normB = g.AND(g.NOT(A.exc1), A.exc0), g.AND(g.NOT(B.exc1), B.exc0)

    ma = list(A.frac) + [TRUE]
    mb = list(B.frac) + [TRUE]
    P = multiply(g, ma, mb)                    # 2wf+2 bits, value in [1, 4)
    top = P[2 * wf + 1]
    # normalised significand N (2wf+2 bits, leading one at 2wf+1)
    N = [g.MUX(top, P[i], P[i - 1] if i >= 1 else FALSE) for i in range(2 * wf + 2)]
    keep_lo = 2 * wf + 1 - wfo                 # kept bits N[2wf+1 .. keep_lo] (wfo+1 bits)
    if keep_lo >= 0:
        kept = N[keep_lo:2 * wf + 2]
        if keep_lo >= 1:
            guard = N[keep_lo - 1]
            sticky = g.OR_many(N[:keep_lo - 1])
        else:
            guard, sticky = FALSE, FALSE
    else:
        kept = [FALSE] * (-keep_lo) + N        # extended: exact, zero-fill below
        guard, sticky = FALSE, FALSE
    if rnd == RNE and guard != FALSE:
        inc = g.AND(guard, g.OR(sticky, kept[0]))
        rounded, rc = increment(g, kept, inc)
    else:
        rounded, rc = kept, FALSE
    frac = rounded[:wfo]                       # if rc, these are all zero already

    # exponent: Ea + Eb - bias + top + rc in wE+2 bits (two's complement).  top
    # and rc are never both 1 (a satisfiability don't-care the AIG cannot see): a
    # rounding carry needs the wfo+1 kept bits all ones and the guard set, i.e.
    # P >= 2^(2wF+2) - 2^(2wF-wfo) when top = 1, above the largest product
    # (2^(wF+1) - 1)^2 for every wfo >= wF -- so one carry-in (top | rc) replaces
    # the separate round-carry incrementer (e5m2 mul 66 -> 56 lop3).
    EW = we + 2
    s1 = ripple_add(g, A.exp, B.exp, g.OR(top, rc), width=EW)
    E = ripple_add(g, s1, const_bits((1 << EW) - bias(we), EW), FALSE, width=EW)
    unf = E[EW - 1]
    ovf = g.AND(g.NOT(E[EW - 1]), E[EW - 2])   # E >= 2^wE (E < 2^(wE+1) always)

    both = g.AND(normA, normB)
    nan = g.OR_many([nA, nB, g.AND(iA, zB), g.AND(zA, iB)])
    normal = g.AND(both, g.AND(g.NOT(ovf), g.NOT(unf)))
    exc1 = g.OR_many([nan, iA, iB, g.AND(both, ovf)])
    exc0 = g.OR(nan, normal)
    sign = g.AND(g.XOR(A.sign, B.sign), g.NOT(nan))
    exp_out = [g.AND(normal, e) for e in E[:we]]
    frac_out = [g.AND(normal, f) for f in frac]
    return pack_bits(frac_out, exp_out, sign, exc0, exc1)


# --------------------------------------------------------------------------- FP adder

class Operand:
    """Decoded adder operand.  ``canonical`` operands have exp = frac = 0
    whenever they are not normal; a non-canonical operand carries exact class
    flags but arbitrary exp/frac bits when zero, inf or NaN."""

    def __init__(self, we, wf, frac, exp, sign, norm, zero, inf, nan, special, canonical=True):
        self.we, self.wf = we, wf
        self.frac, self.exp, self.sign = list(frac), list(exp), sign
        self.norm, self.zero, self.inf, self.nan, self.special = norm, zero, inf, nan, special
        self.canonical = canonical

    @staticmethod
    def from_word(g: AIG, A: FP, canonical: bool = True):
        nan = g.AND(A.exc1, A.exc0)
        inf = g.AND(A.exc1, g.NOT(A.exc0))
        norm = g.AND(g.NOT(A.exc1), A.exc0)
        zero = g.AND(g.NOT(A.exc1), g.NOT(A.exc0))
        return Operand(A.we, A.wf, A.frac, A.exp, A.sign, norm, zero, inf, nan, A.exc1, canonical)


def fp_add(g: AIG, A: FP, B: FP, rnd: int, shift_order="small_first"):
    """HOBFLOPS adder on two canonical words (see fp_add_ops)."""
    return fp_add_ops(g, Operand.from_word(g, A), Operand.from_word(g, B), rnd, shift_order)


def fp_add_ops(g: AIG, A: Operand, B: Operand, rnd: int, shift_order="small_first", norm="detect",
               expo="one_adder", canon_out=True, clamp=True):
    """HOBFLOPS adder F(wE,w) + F(wE,w) -> F(wE,w) (single-path, P:190-198;
    SURVEY 8(c) add; ledger L5-L7).  A must be canonical; B may be
    non-canonical (its exp/frac are ignored when it is zero or special).

    Magnitude compare of (exp, frac) and swap so that |X| >= |Y|; alignment
    right shift of 1.fY by eX - eY with guard, round and sticky; effective
    add/subtract; leading-zero count and left normalisation; RNE/RTZ rounding;
    exponent eX + 1 - lzc + round-carry; overflow -> inf, underflow -> zero,
    exact cancellation -> +0, (-0) + (-0) -> -0.

    Canonical zero operands have exp = frac = 0 and hidden bit 0, so they
    sort below every normal (the hidden bit is the least significant compare
    key, which breaks the tie with the exp=0, frac=0 normal) and flow through
    the datapath: 0 + y = y exactly.  A non-canonical zero B never swaps to X
    and is killed in the aligner."""
    we, w = A.we, A.wf
    p = w + 1
    hA, hB = A.norm, B.norm
    special = g.OR(A.special, B.special)

    keyA = [hA] + list(A.frac) + list(A.exp)
    keyB = [hB] + list(B.frac) + list(B.exp)
    lt = less_than(g, keyA, keyB)
    swap = lt
    if not A.canonical:      # a zero A (arbitrary exp/frac) always goes to Y
        swap = g.OR(swap, A.zero)
    if not B.canonical:      # a zero B (arbitrary exp/frac) never goes to X
        swap = g.AND(swap, g.NOT(B.zero))
    eX = [g.MUX(swap, b, a) for a, b in zip(A.exp, B.exp)]
    eY = [g.MUX(swap, a, b) for a, b in zip(A.exp, B.exp)]
    fX = [g.MUX(swap, b, a) for a, b in zip(A.frac, B.frac)]
    fY = [g.MUX(swap, a, b) for a, b in zip(A.frac, B.frac)]
    # X (the larger magnitude) is normal unless both operands are zero (zeros
    # sort below every normal; specials are overridden below), so its hidden
    # bit is wired to 1 and the both-zero case is flagged explicitly.
    hX = TRUE
    hY = g.MUX(swap, hA, hB)
    sX = g.MUX(swap, B.sign, A.sign)
    sub = g.XOR(A.sign, B.sign)
    kill = FALSE if B.canonical else g.AND(g.NOT(swap), B.zero)
    if not A.canonical:
        kill = g.OR(kill, g.AND(swap, A.zero))
    both_zero = g.AND(A.zero, B.zero)

    # d = eX - eY >= 0
    d = ripple_add(g, eX, [g.NOT(x) for x in eY], TRUE, width=we)
    # alignment: W = p + 2 positions (significand + G + R), then sticky
    W = p + 2
    mY = [FALSE, FALSE] + list(fY) + [hY]
    yv, ys = shift_right_sticky(g, mY, d, order=shift_order, kill=kill, clamp=clamp)
    mX = [FALSE, FALSE] + list(fX) + [hX]
    # adder over W+1 bits: position 0 = sticky, 1..W = shifted significand
    xo = [FALSE] + mX
    yo = [g.XOR(ys, sub)] + [g.XOR(b, sub) for b in yv]
    Z = ripple_add(g, xo, yo, sub, width=W + 2)  # Z[W+1] = carry (add) / discard (sub)
    Z[W + 1] = g.AND(Z[W + 1], g.NOT(sub))
    # normalise: leading-zero count over Z[W+1..0] and left shift
    if norm == "detect":
        # Bound on the left shift: with d >= 2 the difference keeps its leading
        # one at bit W or W-1 (X >= 1, Y < 1/2 before alignment); with d <= 1
        # the aligned Y has no bits below position 2 (its LSB lands on the G
        # position at most), so the exact sum is a multiple of 2^2 and a
        # nonzero Z has its leading one at bit >= 2: shift <= W - 1 = p + 1.
        # A shift of >= 3 happens only for d <= 1 (or an all-zero sum), where the
        # aligned Y has no bits below position 2: Z[0] = Z[1] = 0 then.
        Zn, cnt, zsum = normalize_left(g, Z, max_shift=W - 1, low_zero=(2, 3))
    else:
        cnt, zsum = lzc(g, Z)
        Zn = shift_left(g, Z, cnt)
    # kept p bits: Zn[W+1 .. W+2-p] = Zn[p+3 .. 4]; guard Zn[3]; sticky Zn[2..0]
    kept = Zn[4:p + 4]
    guard = Zn[3]
    sticky = g.OR_many(Zn[0:3])
    if rnd == RNE:
        inc = g.AND(guard, g.OR(sticky, kept[0]))
        rounded, rc = increment(g, kept, inc)
    else:
        rounded, rc = kept, FALSE
    frac = rounded[:w]
    # exponent: eX + 1 - cnt + rc  (wE+2 bits two's complement)
    EW = we + 2
    ncnt = [g.NOT(c) for c in cnt] + [TRUE] * (EW - len(cnt))  # ~cnt sign-extended
    if expo == "one_adder":
        k = ripple_add(g, ncnt, const_bits(2, EW), FALSE, width=EW)  # 1 - cnt = ~cnt + 2
        E = ripple_add(g, eX, k, rc, width=EW)
    else:
        t = ripple_add(g, eX, ncnt, TRUE, width=EW)                # eX - cnt
        E = ripple_add(g, t, const_bits(1, EW), rc, width=EW)
    unf = E[EW - 1]
    ovf = g.AND(g.NOT(E[EW - 1]), E[EW - 2])

    nan = g.OR_many([A.nan, B.nan, g.AND(g.AND(A.inf, B.inf), sub)])
    zsum = g.OR(zsum, both_zero)   # both zero: the datapath (hidden bit of X = 1) is not zero
    fin_nz = g.AND(g.NOT(special), g.NOT(zsum))
    normal = g.AND(fin_nz, g.AND(g.NOT(ovf), g.NOT(unf)))
    exc1 = g.OR(special, g.AND(fin_nz, ovf))
    exc0 = g.OR(nan, normal)
    # zero result: -0 only for (-0) + (-0); exact cancellation of normals gives +0 (L7)
    zero_sign = g.AND(g.AND(A.sign, B.sign), A.zero if not A.canonical else g.NOT(hA))
    inf_sign = g.MUX(A.inf, A.sign, B.sign)
    sign_fin = g.MUX(zsum, zero_sign, sX)
    sign = g.MUX(special, inf_sign, sign_fin)
    if canon_out:  # a relaxed result's NaN sign is don't-care (the next add ignores it; canon clears it)
        sign = g.AND(g.NOT(nan), sign)
    if canon_out:
        exp_out = [g.AND(normal, e) for e in E[:we]]
        frac_out = [g.AND(normal, f) for f in frac]
    else:           # exp/frac arbitrary unless normal (the next MAC reads A non-canonically)
        exp_out, frac_out = E[:we], frac
    return pack_bits(frac_out, exp_out, sign, exc0, exc1)


def fp_canon(g: AIG, A: FP):
    """Canonical form of a word whose exp/frac are arbitrary unless normal
    (S:38): exc != 01 -> exp = frac = 0; NaN sign 0."""
    norm = g.AND(g.NOT(A.exc1), A.exc0)
    nan = g.AND(A.exc1, A.exc0)
    return pack_bits([g.AND(norm, f) for f in A.frac], [g.AND(norm, e) for e in A.exp],
                     g.AND(A.sign, g.NOT(nan)), A.exc0, A.exc1)


def fp_relu(g: AIG, A: FP):
    """ReLU on a canonical word: NaN (sign 0) passes, any word with
    sign 1 (negative, -0, -inf) becomes +0 (all bits zero), else unchanged."""
    ns = g.NOT(A.sign)
    bits = list(A.frac) + list(A.exp) + [A.sign, A.exc0, A.exc1]
    return [g.AND(ns, b) for b in bits[:-3]] + [FALSE, g.AND(ns, A.exc0), g.AND(ns, A.exc1)]


# --------------------------------------------------------------------------- circuits

class Circuit:
    """A built circuit: AIG, named input vectors and output literals."""

    def __init__(self, name, g, inputs, outputs):
        self.name = name
        self.g = g
        self.inputs = inputs      # list of (name, width)
        self.outputs = outputs    # list of literals


def build_mul(we, wf, wfo, rnd) -> Circuit:
    g = AIG()
    a = g.inputs("a", 3 + we + wf)
    b = g.inputs("b", 3 + we + wf)
    out = fp_mul(g, FP(a, we, wf), FP(b, we, wf), wfo, rnd)
    return Circuit(f"mul_e{we}m{wf}_o{wfo}_{'rne' if rnd == RNE else 'rtz'}", g,
                   [("a", 3 + we + wf), ("b", 3 + we + wf)], out)


def build_add(we, w, rnd, **kw) -> Circuit:
    g = AIG()
    a = g.inputs("a", 3 + we + w)
    b = g.inputs("b", 3 + we + w)
    out = fp_add(g, FP(a, we, w), FP(b, we, w), rnd, **kw)
    return Circuit(f"add_e{we}m{w}_{'rne' if rnd == RNE else 'rtz'}", g,
                   [("a", 3 + we + w), ("b", 3 + we + w)], out)


def build_mac(we, wf, wfo, rnd, **kw) -> Circuit:
    """acc' = add(acc, mul(x, w)) -- one step of the conv reduction."""
    g = AIG()
    acc = g.inputs("acc", 3 + we + wfo)
    x = g.inputs("x", 3 + we + wf)
    w = g.inputs("w", 3 + we + wf)
    p = fp_mul(g, FP(x, we, wf), FP(w, we, wf), wfo, rnd)
    out = fp_add(g, FP(acc, we, wfo), FP(p, we, wfo), rnd, **kw)
    return Circuit(f"mac_e{we}m{wf}_{'rne' if rnd == RNE else 'rtz'}", g,
                   [("acc", 3 + we + wfo), ("x", 3 + we + wf), ("w", 3 + we + wf)], out)


def build_canon(we, w) -> Circuit:
    g = AIG()
    a = g.inputs("a", 3 + we + w)
    return Circuit(f"canon_e{we}m{w}", g, [("a", 3 + we + w)], fp_canon(g, FP(a, we, w)))


def build_relu(we, w) -> Circuit:
    g = AIG()
    a = g.inputs("a", 3 + we + w)
    out = fp_relu(g, FP(a, we, w))
    return Circuit(f"relu_e{we}m{w}", g, [("a", 3 + we + w)], out)


# --------------------------------------------------------------------------- weight-table MAC

def tab_onehot(we: int, wfo: int) -> bool:
    """Product-class encoding of a table entry: one-hot flags (zero, normal, inf,
    NaN: 4 planes, 3 lop3 fewer per MAC) when they fit the padding of the
    16-byte-rounded entry, else the 2-bit class code K1 K0 (no wider entry)."""
    base = wfo + (we + 2) + 3
    return (base + 2 + 3) // 4 == (base + 3) // 4


def tab_entry_width(we: int, wf: int, wfo: int | None = None) -> int:
    """Planes of one weight-table entry: frac (wfo) | Epart (wE+2) | S | class,
    class = K0 K1 (2 planes) or Tzero Tnorm Tinf Tnan (4 planes, tab_onehot);
    wfo = wF+1 (single class) or 2wF+1 (extended: the exact product)."""
    wfo = wf + 1 if wfo is None else wfo
    return wfo + (we + 2) + (5 if tab_onehot(we, wfo) else 3)


def product_from_table(g: AIG, t, ea, sx, we: int, wf: int, wfo: int | None = None) -> Operand:
    """The multiplier output as an adder operand, from a weight-table entry
    (rows: x normal with fraction fa -> row fa; x zero -> row 2^wF; x inf ->
    row 2^wF + 1; x NaN -> row 2^wF + 2).

    The conv broadcasts the activation x across the 32 output-channel lanes
    (P:257), so x is one scalar per thread: its fraction selects a row of a
    per-weight table built once from the weight (kernels pre-transformed),
    holding for every lane the rounded product fraction (round to wF+1 bits at
    the product's own binade, RNE/RTZ), Epart = eb - bias + (normalise +
    round carry) as a wE+2-bit two's complement number, the weight sign and the
    product class (K1 K0: 00 zero, 01 normal, 10 inf, 11 NaN, or one-hot flags
    when they fit, tab_onehot; rows for x = zero / inf / NaN encode the
    exception algebra of S:68).  The gates left
    add the activation exponent, classify overflow / underflow (ledger L5, L6)
    and combine the signs.  Extended class (wfo = 2wF+1): the table holds the
    exact product fraction (no rounding)."""
    wfo = wf + 1 if wfo is None else wfo
    EW = we + 2
    F = t[0:wfo]
    Ep = t[wfo:wfo + EW]
    S = t[wfo + EW]
    E = ripple_add(g, Ep, list(ea), FALSE, width=EW)
    unf = E[EW - 1]
    ovf = g.AND(g.NOT(E[EW - 1]), E[EW - 2])
    sign = g.XOR(S, sx)
    if tab_onehot(we, wfo):
        Tz, Tn, Ti, Tq = t[wfo + EW + 1], t[wfo + EW + 2], t[wfo + EW + 3], t[wfo + EW + 4]
        norm = g.AND(Tn, g.AND(g.NOT(ovf), g.NOT(unf)))
        zero = g.OR(Tz, g.AND(Tn, unf))
        inf = g.OR(Ti, g.AND(Tn, ovf))
        return Operand(we, wfo, F, E[:we], sign, norm, zero, inf, Tq, g.OR(inf, Tq), canonical=False)
    K0, K1 = t[wfo + EW + 1], t[wfo + EW + 2]
    nK1 = g.NOT(K1)
    norm = g.AND(g.AND(nK1, K0), g.AND(g.NOT(ovf), g.NOT(unf)))
    zero = g.AND(nK1, g.OR(g.NOT(K0), unf))
    inf = g.OR(g.AND(K1, g.NOT(K0)), g.AND(g.AND(nK1, K0), ovf))
    nan = g.AND(K1, K0)
    special = g.OR(K1, g.AND(K0, ovf))
    return Operand(we, wfo, F, E[:we], sign, norm, zero, inf, nan, special, canonical=False)


def build_mac_tab(we, wf, rnd, wfo=None, chained=True, **kw) -> Circuit:
    """acc' = add(acc, mul(x, w)) with the multiplier read from the weight table;
    wfo = wF+1 (single class, default) or 2wF+1 (extended class).

    chained=True: the accumulator is read and written in a relaxed form whose
    exp/frac bits are arbitrary unless it is normal (the class bits are exact);
    the conv canonicalises once after the reduction (build_canon).  This saves
    the per-MAC zeroing of the result fields."""
    wfo = wf + 1 if wfo is None else wfo
    if chained:
        kw.setdefault("canon_out", False)
    g = AIG()
    acc = g.inputs("acc", 3 + we + wfo)
    t = g.inputs("t", tab_entry_width(we, wf, wfo))
    ea = g.inputs("ea", we)
    sx = g.inputs("sx", 1)[0]
    B = product_from_table(g, t, ea, sx, we, wf, wfo)
    out = fp_add_ops(g, Operand.from_word(g, FP(acc, we, wfo), canonical=not chained), B, rnd, **kw)
    return Circuit(f"mactab_e{we}m{wf}_o{wfo}_{'rne' if rnd == RNE else 'rtz'}", g,
                   [("acc", 3 + we + wfo), ("t", tab_entry_width(we, wf, wfo)), ("ea", we), ("sx", 1)], out)
