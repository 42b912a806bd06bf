"""Functional reduction of an AIG under its satisfiability don't-cares, proved by
exhaustive simulation (the in-repo analogue of ABC's ``fraig``; the paper's flow
optimises its netlists with ABC).

A generated circuit only ever sees *valid* inputs: canonical operand words
(pack / quantise canonicalise), weight-table entries that ``build_wtab_kernel``
can write, an activation exponent / sign taken from the same canonical word that
selected the table row.  Nodes that are equal (or complementary, or constant)
on every valid input vector can be merged; structural hashing cannot see such
equivalences (e.g. the top plane of a table entry's partial exponent is always a
copy of the plane below it).

For the formats whose valid input space is small enough (<= ~1.2e9 vectors) the
space is enumerated completely, every AIG node is simulated over all of it
(numpy uint64 words, chunked), nodes are grouped by a 64-bit random-linear
signature of their full value vector, and the AIG is rebuilt with every node
replaced by the first node of its class.  The rebuilt circuit's outputs are
then compared with the original's on the whole valid space -- that comparison,
not the signatures, is the proof.  The merge lists are cached in
``sweep_cache.json`` (keyed by a structural hash of the AIG), so a build applies
them without re-simulating; ``python -m paper_2007_06563_b200.gen.sweep``
recomputes and re-proves the cache.  Entries marked ``"proved": "gpu-exhaustive"``
(the wider table MACs, up to ~3e14 vectors) were proved by ``tools/sweep_gpu.py``,
which runs the original and the swept networks on every valid input on the B200.
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from . import fpgen
from .aig import AIG, FALSE

ONES = np.uint64(0xFFFFFFFFFFFFFFFF)
ZERO = np.uint64(0)
_LOWPAT = [0xAAAAAAAAAAAAAAAA, 0xCCCCCCCCCCCCCCCC, 0xF0F0F0F0F0F0F0F0, 0xFF00FF00FF00FF00,
           0xFFFF0000FFFF0000, 0xFFFFFFFF00000000]
CACHE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sweep_cache.json")
MAX_SPACE = 1 << 31          # valid vectors enumerated per circuit (e5m3 table MAC: 1.1e9)


# --------------------------------------------------------------------------- valid operand sets

def canonical_words(we: int, wf: int) -> np.ndarray:
    """Every canonical word of F(we, wf): all normals, +-0, +-inf, NaN (sign 0)."""
    top = wf + we + 1
    n = np.arange(1 << (1 + we + wf), dtype=np.uint32)
    normals = (np.uint32(1) << np.uint32(top)) | n
    sp = [0, 1 << (wf + we), 2 << top, (2 << top) | (1 << (wf + we)), 3 << top]
    return np.concatenate([normals, np.array(sp, np.uint32)])


def tab_entry(w, r, we: int, wf: int, wfo: int, rnd: int):
    """The weight-table entry build_wtab_kernel writes (hobf_capi.cu tab_entry):
    row r = activation fraction (normal x) or 2^wF + 0/1/2 (x zero / inf / NaN);
    fields frac (wfo) | partial exponent eb - bias + carry (wE+2) | weight sign |
    class (one-hot zero/normal/inf/NaN flags, or the 2-bit code)."""
    w = np.asarray(w, dtype=np.int64)
    r = np.asarray(r, dtype=np.int64)
    EW = we + 2
    exc = (w >> (wf + we + 1)) & 3
    sw = (w >> (wf + we)) & 1
    eb = (w >> wf) & ((1 << we) - 1)
    fb = w & ((1 << wf) - 1)
    sbit = wfo + EW
    oh = fpgen.tab_onehot(we, wfo)
    NAN = (1 << (sbit + 4)) if oh else (1 << (sbit + 1)) | (1 << (sbit + 2))
    INF = (1 << (sbit + (3 if oh else 2))) | (sw << sbit)
    ZER = ((1 << (sbit + 1)) if oh else 0) | (sw << sbit)
    NORM = 1 << (sbit + (2 if oh else 1))
    nrows = 1 << wf
    P = ((1 << wf) | np.minimum(r, nrows - 1)) * ((1 << wf) | fb)
    top = (P >> (2 * wf + 1)) & 1
    N = np.where(top == 1, P, P << 1)
    sh = 2 * wf + 1 - wfo
    kept = N >> sh
    if sh > 0 and rnd == fpgen.RNE:
        rem = N & ((1 << sh) - 1)
        half = 1 << (sh - 1)
        kept = kept + ((rem > half) | ((rem == half) & ((kept & 1) == 1)))
    carry = kept == (2 << wfo)
    kept = np.where(carry, kept >> 1, kept)
    ep = (eb - ((1 << (we - 1)) - 1) + top + carry) & ((1 << EW) - 1)
    out = np.select([exc == 0, exc == 2, exc == 3], [ZER, INF, NAN], (kept - (1 << wfo)) | (ep << wfo) | (sw << sbit) | NORM)
    out = np.where(r == nrows, np.where((exc & 2) != 0, NAN, ZER), out)
    out = np.where(r == nrows + 1, np.where((exc == 0) | (exc == 3), NAN, INF), out)
    out = np.where(r == nrows + 2, NAN, out)
    return out.astype(np.uint64)


def tab_operands(we: int, wf: int, rnd: int, wfo: int):
    """Distinct (table entry, activation exponent, activation sign) triples over all
    canonical (x, w) pairs: the x word selects the row and supplies ea / sx."""
    xi = canonical_words(we, wf).astype(np.int64)
    X, W = np.meshgrid(xi, xi, indexing="ij")
    X, W = X.ravel(), W.ravel()
    exc = (X >> (wf + we + 1)) & 3
    r = np.where(exc == 1, X & ((1 << wf) - 1), (1 << wf) + np.select([exc == 2, exc == 3], [1, 2], 0))
    t = tab_entry(W, r, we, wf, wfo, rnd)
    ea = ((X >> wf) & ((1 << we) - 1)).astype(np.uint64)
    sx = ((X >> (wf + we)) & 1).astype(np.uint64)
    key = np.unique(t | (ea << np.uint64(40)) | (sx << np.uint64(50)))
    return {"t": key & np.uint64((1 << 40) - 1), "ea": (key >> np.uint64(40)) & np.uint64(0x3FF),
            "sx": key >> np.uint64(50)}


# --------------------------------------------------------------------------- enumeration

class Space:
    """The valid input space of a circuit as chunks of input bit planes: the
    `fast` operand (all its listed values, padded to whole 64-bit words) varies
    fastest; the `combos` operands (one value per combination) are constant over
    a block of words."""

    def __init__(self, circuit, fast_name: str, fast_vals, combos: dict):
        self.c = circuit
        self.fast_name = fast_name
        fv = np.asarray(fast_vals, dtype=np.uint64)
        width = dict(circuit.inputs)[fast_name]
        if fv.size == (1 << width) and width >= 6:   # every pattern: constant planes
            self.wpb = 1 << (width - 6)
            self.fast = []
            for i in range(width):
                if i < 6:
                    self.fast.append(np.full(self.wpb, np.uint64(_LOWPAT[i])))
                else:
                    self.fast.append(np.where((np.arange(self.wpb) >> (i - 6)) & 1, ONES, ZERO))
        else:
            pad = (-fv.size) % 64
            fv = np.concatenate([fv, np.repeat(fv[:1], pad)])    # duplicates are harmless
            self.wpb = fv.size // 64
            bits = [((fv >> np.uint64(i)) & np.uint64(1)).astype(np.uint8) for i in range(width)]
            self.fast = [np.packbits(b, bitorder="little").view(np.uint64) for b in bits]
        self.combos = combos
        self.n_combo = next(iter(combos.values())).size
        self.vectors = self.n_combo * self.wpb * 64

    def chunks(self, words: int = 1 << 17):
        k_per = max(1, words // self.wpb)
        widths = dict(self.c.inputs)
        for s in range(0, self.n_combo, k_per):
            k = min(k_per, self.n_combo - s)
            d = {}
            for i, p in enumerate(self.fast):
                d[f"{self.fast_name}[{i}]"] = np.tile(p, k)
            for name, vals in self.combos.items():
                v = vals[s:s + k]
                for i in range(widths[name]):
                    b = (v >> np.uint64(i)) & np.uint64(1)
                    d[f"{name}[{i}]"] = np.repeat(np.where(b == 1, ONES, ZERO), self.wpb)
            yield d


def space_of(kind: str, circuit, we: int, wf: int, rnd: int, wfo: int):
    """Valid input space of a generated circuit, or None when it is too large."""
    ncanon = lambda wa: (1 << (1 + we + wa)) + 5  # noqa: E731
    if ncanon(wf) ** 2 > MAX_SPACE:
        return None
    if kind == "mac_tab":       # relaxed accumulator: every pattern; (t, ea, sx) from (x, w)
        na = 3 + we + wfo
        if (1 << na) * ncanon(wf) > MAX_SPACE:   # (distinct triples <= pairs; cheap first test)
            return None
        ops = tab_operands(we, wf, rnd, wfo)
        if (1 << na) * ops["t"].size > MAX_SPACE:
            return None
        return Space(circuit, "acc", np.arange(1 << na, dtype=np.uint64), ops)
    if kind == "mac":           # canonical accumulator, x, w
        acc = canonical_words(we, wfo)
        xi = canonical_words(we, wf).astype(np.uint64)
        if acc.size * xi.size ** 2 > MAX_SPACE:
            return None
        X, W = np.meshgrid(xi, xi, indexing="ij")
        return Space(circuit, "acc", acc, {"x": X.ravel(), "w": W.ravel()})
    if kind in ("mul", "add"):  # canonical operand pairs
        wa = wf if kind == "mul" else wfo
        xi = canonical_words(we, wa)
        if xi.size ** 2 > MAX_SPACE:
            return None
        return Space(circuit, "a", xi, {"b": xi.astype(np.uint64)})
    return None


# --------------------------------------------------------------------------- sweep

def _node_values(g: AIG, d: dict):
    vals = [None] * g.n_nodes()
    vals[0] = np.zeros(next(iter(d.values())).shape, np.uint64)
    for name, node in zip(g.input_names, g.input_nodes):
        vals[node] = d[name]
    f0, f1, kind = g.f0, g.f1, g.kind
    for v in range(1, g.n_nodes()):
        if kind[v] == "and":
            a, b = f0[v], f1[v]
            va, vb = vals[a >> 1], vals[b >> 1]
            vals[v] = (~va if a & 1 else va) & (~vb if b & 1 else vb)
    return vals


def structure_key(circuit) -> str:
    g = circuit.g
    h = hashlib.sha256()
    h.update(json.dumps([circuit.name, g.input_names, g.f0, g.f1, g.kind, circuit.outputs]).encode())
    return h.hexdigest()[:32]


def find_merges(circuit, space: Space):
    """[(v, u, p)]: node v equals node u (u < v; 0 = constant false) complemented
    if p, on every vector of the space (candidates by signature; proved by
    ``prove``)."""
    g = circuit.g
    n = g.n_nodes()
    rng = np.random.default_rng(12345)
    H = np.zeros(n, np.uint64)
    Hc = np.zeros(n, np.uint64)
    M = np.uint64(1000003)
    with np.errstate(over="ignore"):
        for d in space.chunks():
            vals = _node_values(g, d)
            R = rng.integers(0, 1 << 62, vals[0].size, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
            s_ones = np.sum(R * ONES)
            for v in range(n):
                if vals[v] is None:
                    continue
                hv = np.sum(vals[v] * R)
                H[v] = H[v] * M + hv
                Hc[v] = Hc[v] * M + (s_ones - hv)
    first = {}
    merges = []
    for v in range(n):
        if g.kind[v] == "const":
            first[int(H[v])] = (v, 0)
            first[int(Hc[v])] = (v, 1)
            continue
        k = int(H[v])
        if k in first:    # an AND node, or an input plane that copies another (e.g. a table field)
            u, p = first[k]
            merges.append((v, u, p))
            continue
        if k not in first:
            first[k] = (v, 0)
        kc = int(Hc[v])
        if kc not in first:
            first[kc] = (v, 1)
    return merges


def apply_merges(circuit, merges):
    """Rebuild the AIG with every merged node replaced by its representative."""
    g = circuit.g
    m = {v: (u, p) for v, u, p in merges}
    ng = AIG()
    sub = [None] * g.n_nodes()
    sub[0] = FALSE
    for name in g.input_names:
        ng.input(name)
    for i, node in enumerate(g.input_nodes):
        sub[node] = 2 * ng.input_nodes[i]
    for v in range(1, g.n_nodes()):
        if g.kind[v] == "input" and v in m:
            u, p = m[v]
            sub[v] = sub[u] ^ p
        if g.kind[v] != "and":
            continue
        if v in m:
            u, p = m[v]
            sub[v] = sub[u] ^ p
            continue
        a, b = g.f0[v], g.f1[v]
        sub[v] = ng.AND(sub[a >> 1] ^ (a & 1), sub[b >> 1] ^ (b & 1))
    outs = [sub[o >> 1] ^ (o & 1) for o in circuit.outputs]
    return fpgen.Circuit(circuit.name, ng, circuit.inputs, outs)


def prove(old, new, space: Space) -> bool:
    """The two circuits' outputs agree on every vector of the space."""
    for d in space.chunks():
        a = old.g.simulate(d, old.outputs, np)
        b = new.g.simulate(d, new.outputs, np)
        if not all(np.array_equal(x, y) for x, y in zip(a, b)):
            return False
    return True


def load_cache():
    try:
        with open(CACHE) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def reduce(kind: str, circuit, we: int, wf: int, rnd: int, wfo: int, cache=None, compute: bool = True):
    """The swept circuit (merges from the cache when its structure key matches,
    else -- with ``compute`` -- found and proved here), or the circuit unchanged
    when its valid space is not enumerable."""
    cache = load_cache() if cache is None else cache
    key = structure_key(circuit)
    ent = cache.get(circuit.name)
    if ent is not None and ent.get("key") == key:
        return apply_merges(circuit, [tuple(m) for m in ent["merges"]])
    if not compute:
        return circuit
    space = space_of(kind, circuit, we, wf, rnd, wfo)
    if space is None:
        return circuit
    merges = find_merges(circuit, space)
    new = apply_merges(circuit, merges)
    assert prove(circuit, new, space), f"sweep of {circuit.name}: outputs differ on the valid space"
    return new


# --------------------------------------------------------------------------- cache tool

BUILDERS = {
    "mac_tab": lambda we, wf, rnd: fpgen.build_mac_tab(we, wf, rnd),
    "mac": lambda we, wf, rnd: fpgen.build_mac(we, wf, wf + 1, rnd),
    "mul": lambda we, wf, rnd: fpgen.build_mul(we, wf, wf + 1, rnd),
    "add": lambda we, wf, rnd: fpgen.build_add(we, wf + 1, rnd),
}


def _targets():
    from .emit import SWEEP
    for we, wf in SWEEP:
        for rnd in (fpgen.RNE, fpgen.RTZ):
            for kind in BUILDERS:
                yield kind, we, wf, rnd


def _one(args):
    kind, we, wf, rnd = args
    c = BUILDERS[kind](we, wf, rnd)
    space = space_of(kind, c, we, wf, rnd, wf + 1)
    if space is None:
        return None
    merges = find_merges(c, space)
    new = apply_merges(c, merges)
    ok = prove(c, new, space)
    return c.name, {"key": structure_key(c), "merges": [list(m) for m in merges], "vectors": int(space.vectors),
                    "proved": bool(ok)}


def main():
    import time
    from concurrent.futures import ProcessPoolExecutor
    t0 = time.time()
    jobs = list(_targets())
    # keep the GPU-proved entries (tools/sweep_gpu.py) whose circuit is unchanged
    cache = {k: v for k, v in load_cache().items() if v.get("proved") == "gpu-exhaustive"}
    with ProcessPoolExecutor() as ex:
        for r in ex.map(_one, jobs):
            if r is None:
                continue
            name, ent = r
            assert ent["proved"], name
            cache[name] = ent
            print(f"{name}: {len(ent['merges'])} merges, {ent['vectors']:.3g} vectors, proved", flush=True)
    with open(CACHE, "w") as f:
        json.dump(cache, f, indent=0, sort_keys=True)
    print(f"wrote {CACHE} ({len(cache)} circuits, {time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()
