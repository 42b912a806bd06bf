"""Resynthesis of a mapped LUT network (the analogue of ABC's ``refactor`` /
``resub`` stage of the paper's flow, on the LOP3 network).

The mapper (``lutmap``) covers the AIG by 3-input cuts; the LUT count it
reaches is bounded by the AIG's structure.  This pass restructures across the
cover: for every LUT r (in topological order) it enumerates the cuts of the
LUT network rooted at r with up to ``kmax`` leaves, computes r's exact
function over each cut's leaves by simulating the window (no don't-cares, so
every rewrite is an equivalence), and looks for an implementation over those
leaves with fewer LUTs than the window's maximum fanout-free cone (the LUTs
the rewrite frees):

* one LUT when r depends on at most 3 of the leaves;
* otherwise a disjoint-support decomposition f = H(g(A), R): A a 3-leaf bound
  set, g one LUT, R the other leaves -- valid when every cofactor of f over
  an assignment of R is a constant, g or ~g (column multiplicity <= 2) --
  with H decomposed the same way, recursively, within the LUT budget.

Passes repeat until nothing improves.  ``check`` re-simulates the rewritten
network against the original on random vectors; the generator's exhaustive
tests (tests/test_generator.py, the GPU MAC tests) cover the emitted circuits.

LUT convention (lutmap): a LUT is (node, leaves, tt8) with leaves[i] the
variable of index bit i and tt8 an 8-bit table over 3 variables (replicated
over the unused ones).
"""
from __future__ import annotations

import itertools

import numpy as np

_PROJ = {}


def _proj(n: int):
    if n not in _PROJ:
        idx = np.arange(1 << n)
        _PROJ[n] = [((idx >> i) & 1).astype(bool) for i in range(n)]
    return _PROJ[n]


def lut_eval(tt8: int, ins):
    """8-bit LUT on bool arrays ins[0..k-1], k <= 3 (index = in0 + 2 in1 + 4 in2)."""
    k = np.zeros(ins[0].shape, dtype=np.int64)
    for i, x in enumerate(ins):
        k |= x.astype(np.int64) << i
    table = np.array([(tt8 >> j) & 1 for j in range(8)], dtype=bool)
    return table[k]


def support(f: np.ndarray, n: int):
    idx = np.arange(1 << n)
    return [i for i in range(n) if (f != f[idx ^ (1 << i)]).any()]


def tt8_of(f: np.ndarray, n: int, vars_):
    """8-bit table of f (which depends only on vars_, |vars_| <= 3), replicated."""
    idx = np.arange(1 << n)
    t = 0
    for k in range(8):
        # a row whose vars_ bits equal (k restricted to len(vars_) bits)
        want = k & ((1 << len(vars_)) - 1)
        code = np.zeros(1 << n, dtype=np.int64)
        for i, v in enumerate(vars_):
            code |= ((idx >> v) & 1) << i
        rows = np.nonzero(code == want)[0]
        if f[rows[0]]:
            t |= 1 << k
    return t


def _bound_set(f: np.ndarray, n: int, A, R):
    """Disjoint decomposition f = H(g(A), R), |A| = 3: returns (g as an 8-bit table
    over A, H as a bool array over 1 + |R| variables [g, R...]) or None."""
    idx = np.arange(1 << n)
    a = np.zeros(1 << n, dtype=np.int64)
    for i, v in enumerate(A):
        a |= ((idx >> v) & 1) << i
    r = np.zeros(1 << n, dtype=np.int64)
    for i, v in enumerate(R):
        r |= ((idx >> v) & 1) << i
    T = np.zeros((1 << len(R), 8), dtype=bool)
    T[r, a] = f
    h = None
    for row in T:
        if row.all() or not row.any():
            continue
        if h is None:
            h = row
        elif not ((row == h).all() or (row == ~h).all()):
            return None
    if h is None:
        return None
    g = sum(1 << k for k in range(8) if h[k])
    nH = 1 + len(R)
    H = np.zeros(1 << nH, dtype=bool)
    for rc in range(1 << len(R)):
        row = T[rc]
        for gv in (0, 1):
            if row.all():
                v = True
            elif not row.any():
                v = False
            else:
                same = (row == h).all()
                v = bool(gv) if same else not gv
            H[gv | (rc << 1)] = v
    return g, H


def decompose(f: np.ndarray, n: int, budget: int):
    """Fewest-LUT implementation of f (bool array over 2^n rows) within `budget`
    LUTs, as a list of (inputs, tt8) -- inputs ('v', i) = variable i, ('l', j) =
    the j-th LUT of the list; the last LUT computes f.  None if none found."""
    if budget < 1:
        return None
    sup = support(f, n)
    if len(sup) <= 3:
        return [([("v", i) for i in sup], tt8_of(f, n, sup))]
    if budget < 2 or len(sup) > 2 * budget + 1:
        return None
    best = None
    for A in itertools.combinations(sup, 3):
        R = [v for v in sup if v not in A]
        d = _bound_set(f, n, A, R)
        if d is None:
            continue
        g, H = d
        sub = decompose(H, 1 + len(R), budget - 1 if best is None else len(best) - 2)
        if sub is None:
            continue
        out = [([("v", v) for v in A], g)]
        for ins, tt in sub:
            new = []
            for kind, i in ins:
                if kind == "l":
                    new.append(("l", i + 1))
                elif i == 0:
                    new.append(("l", 0))
                else:
                    new.append(("v", R[i - 1]))
            out.append((new, tt))
        if best is None or len(out) < len(best):
            best = out
            if len(best) == 2:
                break
    return best


# --------------------------------------------------------------------------- network rewriting

class Net:
    def __init__(self, luts, outputs, inputs):
        self.lut = {v: (tuple(l), tt) for v, l, tt in luts}
        self.order = [v for v, _, _ in luts]
        self.out_nodes = {o >> 1 for o in outputs}
        self.inputs = set(inputs)
        self.next_id = max(list(self.lut) + list(self.inputs) + [0]) + 1

    def fanouts(self):
        fo = {}
        for v in self.order:
            for l in self.lut[v][0]:
                fo.setdefault(l, set()).add(v)
        return fo

    def as_list(self):
        return [(v, self.lut[v][0], self.lut[v][1]) for v in self.order]


def _merge_cuts(cut_lists, kmax, limit):
    res = {frozenset()}
    for cl in cut_lists:
        nxt = set()
        for a in res:
            for b in cl:
                u = a | b
                if len(u) <= kmax:
                    nxt.add(u)
        res = nxt
        if not res:
            break
    res = sorted(res, key=len)
    return res[:limit]


def _window(net, root, cut):
    """LUTs between `cut` and `root` in topological order, or None if the cone of
    root is not bounded by cut."""
    seen, stack = set(), [root]
    while stack:
        v = stack.pop()
        if v in seen or v in cut:
            continue
        if v not in net.lut:
            return None        # an input or the constant outside the cut
        seen.add(v)
        stack.extend(net.lut[v][0])
    pos = {v: i for i, v in enumerate(net.order)}
    return sorted(seen, key=lambda v: pos[v])


def _mffc(net, root, win, fo):
    """The window's LUTs that are freed when root is re-implemented over the cut:
    root plus every window LUT whose fanouts all lie in the freed set (and that is
    not an output)."""
    wset = set(win)
    freed = {root}
    changed = True
    while changed:
        changed = False
        for v in reversed(win):
            if v in freed or v in net.out_nodes:
                continue
            f = fo.get(v, set())
            if f and f <= freed and f <= wset:
                freed.add(v)
                changed = True
    return freed


def _simulate_window(net, win, cut):
    cut = sorted(cut)
    n = len(cut)
    P = _proj(n)
    val = {c: P[i] for i, c in enumerate(cut)}
    for v in win:
        leaves, tt = net.lut[v]
        val[v] = lut_eval(tt, [val[l] for l in leaves]) if leaves else np.full(1 << n, bool(tt & 1))
    return cut, val


def optimize(luts, outputs, inputs, kmax: int = 6, max_cuts: int = 40, passes: int = 4):
    """Rewrite the LUT list (topological) -> a new topological LUT list with the same
    output functions and no more LUTs."""
    net = Net(luts, outputs, inputs)
    for _ in range(passes):
        gained = 0
        cuts = {}
        for v in net.inputs | {0}:
            cuts[v] = [frozenset([v])]
        fo = net.fanouts()
        i = 0
        while i < len(net.order):
            r = net.order[i]
            leaves, tt = net.lut[r]
            own = _merge_cuts([cuts.get(l, [frozenset([l])]) for l in leaves], kmax, max_cuts)
            best = None
            for cut in own:
                if len(cut) <= 1 and cut == frozenset(leaves):
                    continue
                win = _window(net, r, cut)
                if win is None:
                    continue
                freed = _mffc(net, r, win, fo)
                if len(freed) <= 1:
                    continue
                cl, val = _simulate_window(net, win, cut)
                budget = len(freed) - 1 if best is None else best[0] - 1
                if budget < 1:
                    continue
                dec = decompose(val[r], len(cl), budget)
                if dec is not None and len(dec) < len(freed) and (best is None or len(freed) - len(dec) > best[0]):
                    best = (len(freed) - len(dec), cut, cl, freed, dec)
            if best is not None:
                gain, cut, cl, freed, dec = best
                # remove the freed LUTs (except r), add the new ones before r
                for v in freed:
                    if v != r:
                        del net.lut[v]
                net.order = [v for v in net.order if v == r or v not in freed]
                i = net.order.index(r)
                ids = []
                for j, (ins, tt8) in enumerate(dec):
                    nid = r if j == len(dec) - 1 else net.next_id
                    if nid != r:
                        net.next_id += 1
                    lv = tuple(cl[k] if kind == "v" else ids[k] for kind, k in ins)
                    net.lut[nid] = (lv, tt8)
                    ids.append(nid)
                    if nid != r:
                        net.order.insert(i, nid)
                        i += 1
                        cuts[nid] = _merge_cuts([cuts.get(l, [frozenset([l])]) for l in lv], kmax, max_cuts) + \
                            [frozenset([nid])]
                fo = net.fanouts()
                gained += gain
                leaves = net.lut[r][0]
                own = _merge_cuts([cuts.get(l, [frozenset([l])]) for l in leaves], kmax, max_cuts)
            cuts[r] = own + [frozenset([r])]
            i += 1
        if gained == 0:
            break
    return net.as_list()


def simulate(luts, inputs_vals: dict, n_rows: int):
    """Evaluate a LUT list: inputs_vals {node: bool array}; returns {node: array}."""
    val = dict(inputs_vals)
    val[0] = np.zeros(n_rows, dtype=bool)
    for v, leaves, tt in luts:
        val[v] = lut_eval(tt, [val[l] for l in leaves]) if leaves else np.full(n_rows, bool(tt & 1))
    return val


def check(luts_a, luts_b, outputs, inputs, n_rows: int = 1 << 14, seed: int = 0) -> bool:
    """Random-vector equivalence of two LUT networks on the output nodes."""
    rng = np.random.default_rng(seed)
    iv = {v: rng.random(n_rows) < 0.5 for v in inputs}
    va, vb = simulate(luts_a, iv, n_rows), simulate(luts_b, iv, n_rows)
    return all((va[o >> 1] == vb[o >> 1]).all() for o in outputs)
