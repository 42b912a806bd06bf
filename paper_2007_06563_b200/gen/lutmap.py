"""Technology mapping of an AIG onto the LOP3 "cell library".

The paper maps its FP cores onto a Liberty library whose cells are the target
ISA's bitwise instructions with unit area; for
AVX512 that library is all 256 three-input functions (``vpternlog``).  PTX
``lop3.b32`` is the same 256-function family with the same immediate
convention (a = 0xF0, b = 0xCC, c = 0xAA), so mapping onto it is K=3 LUT
mapping with unit cost per LUT:

1. enumerate all 3-feasible cuts of every AND node, each with its 8-bit truth
   table; leaves the function does not depend on are dropped,
2. choose a cover by area flow,
3. improve it by exact local area recovery (reference counting), a few passes.

Truth-table convention used throughout: for a cut with leaves (u0, u1, u2)
the table index is v0 + 2*v1 + 4*v2; the emitter passes a = u2, b = u1,
c = u0 to ``lop3``, which is exactly the PTX convention 4a + 2b + c.
"""
from __future__ import annotations

from functools import lru_cache

K = 3
VAR_TT = (0xAA, 0xCC, 0xF0)  # tt of leaf position 0, 1, 2 over 3 variables


@lru_cache(maxsize=None)
def _expand_map(sub: tuple, n_union: int) -> tuple:
    """For leaves at positions ``sub`` of a union cut: index map from union index -> sub index."""
    out = []
    for k in range(1 << n_union):
        j = 0
        for i, pos in enumerate(sub):
            if (k >> pos) & 1:
                j |= 1 << i
        out.append(j)
    return tuple(out)


def _expand(tt: int, sub: tuple, n_union: int) -> int:
    m = _expand_map(sub, n_union)
    r = 0
    for k, j in enumerate(m):
        if (tt >> j) & 1:
            r |= 1 << k
    return r


def _full(tt: int, n: int) -> int:
    """Replicate an n-variable table to 8 bits (variables >= n are don't-care)."""
    size = 1 << n
    tt &= (1 << size) - 1
    r = 0
    for k in range(8):
        if (tt >> (k % size)) & 1:
            r |= 1 << k
    return r


def _depends(tt: int, n: int, i: int) -> bool:
    for k in range(1 << n):
        if not (k >> i) & 1:
            if ((tt >> k) & 1) != ((tt >> (k | (1 << i))) & 1):
                return True
    return False


def _drop(tt: int, n: int, i: int) -> int:
    r = 0
    j = 0
    for k in range(1 << n):
        if not (k >> i) & 1:
            # compress index k (remove bit i)
            lo = k & ((1 << i) - 1)
            hi = (k >> (i + 1)) << i
            if (tt >> k) & 1:
                r |= 1 << (lo | hi)
            j += 1
    return r


class Cut:
    __slots__ = ("leaves", "tt")

    def __init__(self, leaves: tuple, tt: int):
        self.leaves = leaves  # sorted node ids
        self.tt = tt          # over len(leaves) variables (2^n bits)


def _merge(c0: Cut, neg0: int, c1: Cut, neg1: int):
    u = tuple(sorted(set(c0.leaves) | set(c1.leaves)))
    if len(u) > K:
        return None
    n = len(u)
    pos0 = tuple(u.index(x) for x in c0.leaves)
    pos1 = tuple(u.index(x) for x in c1.leaves)
    mask = (1 << (1 << n)) - 1
    t0 = _expand(c0.tt, pos0, n)
    t1 = _expand(c1.tt, pos1, n)
    if neg0:
        t0 ^= mask
    if neg1:
        t1 ^= mask
    tt = t0 & t1
    # drop vacuous leaves
    leaves = list(u)
    i = 0
    while i < len(leaves):
        if not _depends(tt, len(leaves), i):
            tt = _drop(tt, len(leaves), i)
            leaves.pop(i)
        else:
            i += 1
    return Cut(tuple(leaves), tt)


class Mapping:
    """Result: ``luts`` in topological order, each (node, leaves, tt8)."""

    def __init__(self, aig, outputs, luts, chosen):
        self.aig = aig
        self.outputs = outputs
        self.luts = luts
        self.chosen = chosen

    @property
    def n_luts(self) -> int:
        return len(self.luts)


def map_aig(aig, outputs: list[int], passes: int = 4, max_cuts: int = 24, resynth: bool = True) -> Mapping:
    """Map the AIG onto 3-input LUTs (cut enumeration, area flow, exact local area
    recovery, the absorb post-pass) and, with ``resynth``, restructure the LUT
    network across the cover (``lutopt.optimize``: exact window resynthesis)."""
    n = aig.n_nodes()
    kind = aig.kind
    cuts: list[list[Cut]] = [None] * n
    for v in range(n):
        triv = Cut((v,), 0b10)
        if kind[v] != "and":
            cuts[v] = [triv] if kind[v] == "input" else [Cut((), 0)]
            continue
        l0, l1 = aig.f0[v], aig.f1[v]
        u0, u1 = l0 >> 1, l1 >> 1
        found = {}
        for c0 in cuts[u0]:
            for c1 in cuts[u1]:
                c = _merge(c0, l0 & 1, c1, l1 & 1)
                if c is None:
                    continue
                key = c.leaves
                if key not in found:
                    found[key] = c
        cl = list(found.values())
        # remove dominated cuts (a strict subset exists)
        sets = [set(c.leaves) for c in cl]
        keep = []
        for i, c in enumerate(cl):
            dom = False
            for j, s in enumerate(sets):
                if j != i and len(s) < len(sets[i]) and s <= sets[i]:
                    dom = True
                    break
            if not dom:
                keep.append(c)
        keep.sort(key=lambda c: len(c.leaves))
        keep = keep[:max_cuts]
        cuts[v] = keep + [triv]

    # fanout estimate
    refs_est = [0] * n
    for v in range(n):
        if kind[v] == "and":
            refs_est[aig.f0[v] >> 1] += 1
            refs_est[aig.f1[v] >> 1] += 1
    for o in outputs:
        refs_est[o >> 1] += 1

    def mappable(c: Cut, v: int) -> bool:
        return not (len(c.leaves) == 1 and c.leaves[0] == v)

    # ---------------- area flow
    af = [0.0] * n
    best = [None] * n
    for v in range(n):
        if kind[v] != "and":
            continue
        bv, bc = None, None
        for c in cuts[v]:
            if not mappable(c, v):
                continue
            a = 1.0 + sum(af[l] / max(1, refs_est[l]) for l in c.leaves if kind[l] == "and")
            if bv is None or a < bv - 1e-9 or (abs(a - bv) < 1e-9 and len(c.leaves) < len(bc.leaves)):
                bv, bc = a, c
        af[v] = bv
        best[v] = bc

    chosen = list(best)
    refs = [0] * n

    def ref(v: int) -> int:
        """Reference node v's chosen cut recursively; return LUTs newly needed."""
        if kind[v] != "and":
            return 0
        refs[v] += 1
        if refs[v] > 1:
            return 0
        a = 1
        for l in chosen[v].leaves:
            a += ref(l)
        return a

    def deref(v: int) -> int:
        if kind[v] != "and":
            return 0
        refs[v] -= 1
        if refs[v] > 0:
            return 0
        a = 1
        for l in chosen[v].leaves:
            a += deref(l)
        return a

    for o in outputs:
        ref(o >> 1)

    # ---------------- exact local area recovery
    for _ in range(passes):
        changed = False
        for v in range(n):
            if kind[v] != "and" or refs[v] == 0:
                continue
            cur = chosen[v]
            # free v's current cone (v itself stays referenced)
            for l in cur.leaves:
                deref(l)
            best_c, best_a = None, None
            for c in cuts[v]:
                if not mappable(c, v):
                    continue
                a = 0
                for l in c.leaves:
                    a += ref(l)
                for l in c.leaves:
                    deref(l)
                if best_a is None or a < best_a or (a == best_a and len(c.leaves) < len(best_c.leaves)):
                    best_a, best_c = a, c
            if best_c is not cur:
                changed = True
            chosen[v] = best_c
            for l in best_c.leaves:
                ref(l)
        if not changed:
            break

    luts = []
    for v in range(n):
        if kind[v] == "and" and refs[v] > 0:
            c = chosen[v]
            luts.append((v, c.leaves, _full(c.tt, len(c.leaves))))
    luts = absorb_small_luts(luts, outputs)
    if resynth:
        from . import lutopt
        luts = absorb_small_luts(lutopt.optimize(luts, outputs, aig.input_nodes), outputs)
    return Mapping(aig, outputs, luts, chosen)


def _eval_tt(tt: int, vals) -> int:
    idx = 0
    for i, x in enumerate(vals):
        idx |= (x & 1) << i
    return (tt >> idx) & 1


def absorb_small_luts(luts, outputs):
    """Post-pass: a LUT f that is not an output and whose every consumer can take
    f's leaves directly (the consumer's other leaves plus f's leaves number at
    most 3) is folded into all its consumers and removed -- one lop3 fewer.
    Local area recovery cannot find this when f has several consumers (freeing
    f needs all of them to move at once).  Repeated until no LUT qualifies."""
    lut = {v: (tuple(leaves), tt) for v, leaves, tt in luts}
    order = [v for v, _, _ in luts]
    out_nodes = {o >> 1 for o in outputs}
    changed = True
    while changed:
        changed = False
        fan = {}
        for v in order:
            for l in lut[v][0]:
                if l in lut:
                    fan.setdefault(l, []).append(v)
        for f in order:
            if f in out_nodes or f not in fan:
                continue
            fl, ftt = lut[f]
            new = {}
            for g in fan[f]:
                gl, gtt = lut[g]
                nl = tuple(sorted(set(x for x in gl if x != f) | set(fl)))
                if len(nl) > 3:
                    new = None
                    break
                tt = 0
                for k in range(8):
                    val = {x: (k >> i) & 1 for i, x in enumerate(nl)}
                    fv = _eval_tt(ftt, [val[x] for x in fl])
                    if _eval_tt(gtt, [fv if x == f else val[x] for x in gl]):
                        tt |= 1 << k
                new[g] = (nl, tt)
            if not new:
                continue
            lut.update(new)
            del lut[f]
            order.remove(f)
            changed = True
            break
    return [(v, lut[v][0], lut[v][1]) for v in order]


def lop3_eval(imm: int, a, b, c, ones):
    """Evaluate lop3(a, b, c, imm) on numpy words (reference semantics of PTX lop3.b32)."""
    r = None
    for k in range(8):
        if (imm >> k) & 1:
            t = (a if k & 4 else a ^ ones) & (b if k & 2 else b ^ ones) & (c if k & 1 else c ^ ones)
            r = t if r is None else (r | t)
    if r is None:
        r = a & (a ^ ones)
    return r


def simulate_mapping(m: Mapping, input_words: dict, np):
    """Evaluate the mapped LUT network (checks the mapper against the AIG)."""
    aig = m.aig
    shape = next(iter(input_words.values())).shape
    zero = np.zeros(shape, dtype=np.uint64)
    ones = ~zero
    vals = {0: zero}
    for name, node in zip(aig.input_names, aig.input_nodes):
        vals[node] = input_words[name]
    for v, leaves, tt in m.luts:
        ops = [vals[l] for l in leaves] + [zero] * (3 - len(leaves))
        # leaves[0] -> c, leaves[1] -> b, leaves[2] -> a
        vals[v] = lop3_eval(tt, ops[2], ops[1], ops[0], ones)
    out = []
    for o in m.outputs:
        x = vals[o >> 1]
        out.append(x ^ ones if o & 1 else x)
    return out
