"""The LOP3 circuit generator, checked on CPU (no GPU): the AIG and the mapped
LOP3 network are simulated word-parallel (numpy uint64 bit planes) and
compared bit-exactly with the oracle -- exhaustively for the <= 9-bit input
formats, on random + directed vectors above (SURVEY 4 ladder step 3)."""
import json
import os

import numpy as np
import pytest

import oracle
import pyref
from paper_2007_06563_b200.gen import aig as aigmod, bitsim, emit, fpgen, lutmap


def canon_words(we, wf):
    return np.array(pyref.canonical_words(we, wf), dtype=np.uint32)


# ----------------------------------------------------------------------------- paper pins for the mapper

def test_full_adder_maps_to_two_lop3():
    """P:119 / P:241-244: the full adder is two 3-input LUT cells on AVX512
    (LUT150 = xor3 sum, LUT232 = majority carry); lop3 is the same library."""
    g = aigmod.AIG()
    a, b, c = g.input("a"), g.input("b"), g.input("c")
    s, co = g.XOR3(a, b, c), g.MAJ(a, b, c)
    m = lutmap.map_aig(g, [s, co])
    assert m.n_luts == 2
    tt_of = {v: tt for v, _, tt in m.luts}
    tts = sorted(tt_of[o >> 1] ^ (0xFF if o & 1 else 0) for o in (s, co))
    assert tts == sorted([0x96, 0xE8])  # same immediates as LUT150 / LUT232


def test_two_bit_adder_maps_to_four_lop3():
    """Alg. 2: a 2-bit ripple adder with carry-in in 4 LUT3 ops."""
    g = aigmod.AIG()
    x = [g.input("x0"), g.input("x1")]
    y = [g.input("y0"), g.input("y1")]
    cin = g.input("cin")
    out = fpgen.ripple_add(g, x, y, cin, width=3)
    m = lutmap.map_aig(g, out)
    assert m.n_luts == 4
    # exhaustive check of the mapped network
    vals = np.arange(32, dtype=np.uint32)
    words = {}
    for i, name in enumerate(["x0", "x1", "y0", "y1", "cin"]):
        words[name] = np.array([sum(((int(v) >> i) & 1) << k for k, v in enumerate(vals))], dtype=np.uint64)
    outs = lutmap.simulate_mapping(m, words, np)
    for k, v in enumerate(vals):
        v = int(v)
        xv, yv, cv = (v & 1) | ((v >> 1) & 1) << 1, ((v >> 2) & 1) | ((v >> 3) & 1) << 1, (v >> 4) & 1
        s = xv + yv + cv
        got = sum((((int(o[0]) >> k) & 1) << i) for i, o in enumerate(outs))
        assert got == s


def test_lop3_truth_table_convention():
    """lop3 immediate index = 4a + 2b + c with a=0xF0, b=0xCC, c=0xAA (PTX; Table 2 LUTnnn)."""
    ones = np.uint64(0xFFFFFFFFFFFFFFFF)
    a, b, c = np.uint64(0xF0), np.uint64(0xCC), np.uint64(0xAA)
    for imm in (0x96, 0xE8, 0x01, 0xFE, 0x80, 0x2A):
        assert int(lutmap.lop3_eval(imm, a, b, c, ones)) & 0xFF == imm


# ----------------------------------------------------------------------------- circuits vs oracle

def _check(circuit, mapping, arrays, expected, post=None):
    """post: applied to the circuit outputs before comparing (e.g. canonicalisation)."""
    post = post or (lambda v: v)
    got_aig = post(bitsim.run_aig(circuit, arrays))
    assert np.array_equal(got_aig, expected), "AIG differs from oracle"
    got_map = post(bitsim.run_mapping(circuit, mapping, arrays))
    assert np.array_equal(got_map, expected), "LOP3 mapping differs from oracle"


@pytest.mark.parametrize("we,wf", [(5, 3), (4, 3), (5, 2), (6, 2), (4, 2)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_mul_exhaustive(we, wf, rnd):
    c = fpgen.build_mul(we, wf, wf + 1, rnd)
    m = lutmap.map_aig(c.g, c.outputs)
    w = canon_words(we, wf)
    A, B = np.meshgrid(w, w, indexing="ij")
    A, B = A.ravel(), B.ravel()
    _check(c, m, [A, B], oracle.mul(A, B, we, wf, wf + 1, rnd))


def test_mul_normalise_and_round_carries_exclusive():
    """fpgen.fp_mul adds the normalisation carry (product >= 2) and the rounding
    carry through ONE exponent carry-in (top | rc), which is exact only if they
    are never both 1.  Brute force over every significand pair for wF <= 7 and
    every rounding width wF <= wfo <= 2wF (RNE: the only mode with a carry), and
    the closed form (largest product (2^(wF+1) - 1)^2 below the carry threshold
    2^(2wF+2) - 2^(2wF-wfo)) for every wF <= 23."""
    for wf in range(1, 8):
        m = np.arange(1 << wf, 1 << (wf + 1), dtype=np.int64)
        P = np.multiply.outer(m, m).ravel()
        top = P >= (1 << (2 * wf + 1))
        for wfo in range(wf, 2 * wf + 1):
            N = np.where(top, P, P << 1)                       # leading one at bit 2wF+1
            lo = 2 * wf + 1 - wfo                              # bits below the kept wfo+1
            kept, rem = N >> lo, N & ((1 << lo) - 1)
            half = 1 << (lo - 1)
            up = (rem > half) | ((rem == half) & ((kept & 1) == 1))
            rc = (kept + up) >> (wfo + 1)                      # rounding carried out of the kept bits
            assert not np.any(top & (rc == 1)), (wf, wfo)
    for wf in range(1, 24):
        for wfo in range(wf, 2 * wf + 1):
            assert ((1 << (wf + 1)) - 1) ** 2 < (1 << (2 * wf + 2)) - (1 << (2 * wf - wfo))


@pytest.mark.parametrize("we,w", [(5, 4), (4, 4), (5, 3), (6, 3)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_add_exhaustive(we, w, rnd):
    c = fpgen.build_add(we, w, rnd)
    m = lutmap.map_aig(c.g, c.outputs)
    x = canon_words(we, w)
    A, B = np.meshgrid(x, x, indexing="ij")
    A, B = A.ravel(), B.ravel()
    _check(c, m, [A, B], oracle.add(A, B, we, w, rnd))


def _rand_words(rng, n, we, wf, special_frac=0.05):
    s = rng.integers(0, 2, n)
    e = rng.integers(0, 1 << we, n)
    f = rng.integers(0, 1 << wf, n)
    w = ((1 << (wf + we + 1)) | (s << (wf + we)) | (e << wf) | f).astype(np.uint32)
    sp = rng.random(n) < special_frac
    specials = np.array([0, 1 << (wf + we), 2 << (wf + we + 1), (2 << (wf + we + 1)) | (1 << (wf + we)),
                         3 << (wf + we + 1)], np.uint32)
    w[sp] = rng.choice(specials, int(sp.sum()))
    return w


@pytest.mark.parametrize("we,wf", [(5, 10), (6, 10), (4, 10), (4, 7), (6, 5)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_mac_random_wide(we, wf, rnd):
    rng = np.random.default_rng(we * 31 + wf * 7 + rnd)
    N = 200_000
    c = fpgen.build_mac(we, wf, wf + 1, rnd)
    m = lutmap.map_aig(c.g, c.outputs)
    acc = _rand_words(rng, N, we, wf + 1)
    x = _rand_words(rng, N, we, wf)
    w = _rand_words(rng, N, we, wf)
    half = N // 2
    p = oracle.mul(x[:half], w[:half], we, wf, wf + 1, rnd)
    acc[:half] = np.where(rng.random(half) < 0.5, p ^ np.uint32(1 << (wf + 1 + we)), acc[:half])
    _check(c, m, [acc, x, w], oracle.mac(acc, x, w, we, wf, wf + 1, rnd))


@pytest.mark.parametrize("rnd", [0, 1])
def test_mac_exhaustive_pairs_e4m3(rnd):
    """All (x, w) pairs of e4m3 against a spread of accumulators."""
    we, wf = 4, 3
    c = fpgen.build_mac(we, wf, wf + 1, rnd)
    m = lutmap.map_aig(c.g, c.outputs)
    xi = canon_words(we, wf)
    X, W = np.meshgrid(xi, xi, indexing="ij")
    X, W = X.ravel(), W.ravel()
    accs = canon_words(we, wf + 1)[::37]
    A = np.repeat(accs, X.size)
    XX, WW = np.tile(X, accs.size), np.tile(W, accs.size)
    _check(c, m, [A, XX, WW], oracle.mac(A, XX, WW, we, wf, wf + 1, rnd))


def test_relu_circuit():
    for we, w in [(5, 4), (4, 11)]:
        c = fpgen.build_relu(we, w)
        m = lutmap.map_aig(c.g, c.outputs)
        x = canon_words(we, w) if w < 6 else _rand_words(np.random.default_rng(0), 50000, we, w, 0.2)
        _check(c, m, [x], oracle.relu(x, we, w))


# ----------------------------------------------------------------------------- gate-count properties

def test_gate_count_properties():
    """RTZ adder < RNE adder for every format; counts
    non-decreasing in wF at fixed wE (Figs. 8/10/12 trend); the e5m2
    MAC is within the paper's AVX512 bar of 53 + 204 = 257."""
    counts = {}
    for we in (4, 5, 6):
        for wf in range(2, 11):
            for rnd in (0, 1):
                ca = fpgen.build_add(we, wf + 1, rnd)
                cm = fpgen.build_mul(we, wf, wf + 1, rnd)
                counts[(we, wf, rnd)] = (lutmap.map_aig(cm.g, cm.outputs).n_luts,
                                         lutmap.map_aig(ca.g, ca.outputs).n_luts)
    for we in (4, 5, 6):
        for wf in range(2, 11):
            assert counts[(we, wf, 1)][1] < counts[(we, wf, 0)][1]
            if wf > 2:
                for rnd in (0, 1):
                    assert sum(counts[(we, wf, rnd)]) >= sum(counts[(we, wf - 1, rnd)])
    assert sum(counts[(5, 2, 0)]) <= 257


# ----------------------------------------------------------------------------- emitted sources

def test_emitted_headers_up_to_date(tmp_path):
    """The committed csrc/gen/ sources are exactly what the generator emits."""
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    gen_dir = os.path.join(here, "paper_2007_06563_b200", "csrc", "gen")
    emit.write_all(str(tmp_path), formats=[(5, 3), (4, 10)])
    for name in ["hobf_circuit_e5m3_rne.cuh", "hobf_circuit_e4m10_rtz.cuh", "hobf_fmt_e5m3.cu"]:
        assert open(os.path.join(gen_dir, name)).read() == open(os.path.join(tmp_path, name)).read(), name
    counts = json.load(open(os.path.join(gen_dir, "gate_counts.json")))
    assert len(counts) == 108  # 27 formats x {RNE, RTZ} x {single, extended}


def test_emitted_mac_lop3_count_matches_mapping():
    r = emit.gen_format(5, 3, 0)
    n_canon = lutmap.map_aig(fpgen.build_canon(5, 4).g, fpgen.build_canon(5, 4).outputs).n_luts
    assert r["src"].count("hobf_lop3<") == r["g_mac"] + r["g_tab"] + r["g_relu"] + n_canon


def test_chained_relaxed_accumulator_over_many_steps():
    """A chain of MACs through the relaxed accumulator, canonicalised at the end,
    equals the oracle's chain step for step."""
    we, wf = 5, 3
    c = fpgen.build_mac_tab(we, wf, 0)
    m = lutmap.map_aig(c.g, c.outputs)
    rng = np.random.default_rng(0)
    xi = canon_words(we, wf)
    N = 100_000
    acc = np.zeros(N, np.uint32)
    ref = acc.copy()
    for _ in range(8):
        x, w = rng.choice(xi, N), rng.choice(xi, N)
        acc = bitsim.run_mapping(c, m, tabref.circuit_inputs(acc, x, w, we, wf, 0))
        ref = oracle.mac(ref, x, w, we, wf, wf + 1, 0)
        assert np.array_equal(tabref.canon(acc, we, wf + 1), ref)


# ----------------------------------------------------------------------------- prepared-weights (table) MAC

import tabref  # noqa: E402


@pytest.mark.parametrize("we,wf", [(5, 3), (4, 3), (5, 2), (6, 2)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_mac_tab_exhaustive_pairs(we, wf, rnd):
    """Table MAC circuit fed with table entries (tests/tabref.py) equals the
    oracle MAC for every (x, w) pair of canonical operands against a spread of
    accumulators (every 23rd canonical accumulator, plus all specials)."""
    c = fpgen.build_mac_tab(we, wf, rnd)
    m = lutmap.map_aig(c.g, c.outputs)
    xi = canon_words(we, wf)
    X, W = np.meshgrid(xi, xi, indexing="ij")
    X, W = X.ravel(), W.ravel()
    acc_all = canon_words(we, wf + 1)
    accs = np.concatenate([acc_all[:5], acc_all[5::23]])
    rng = np.random.default_rng(9)
    post = lambda v: tabref.canon(v, we, wf + 1)  # noqa: E731  (the chain canonicalises once)
    for s in range(0, accs.size, 8):
        a = accs[s:s + 8]
        A = np.repeat(a, X.size)
        XX, WW = np.tile(X, a.size), np.tile(W, a.size)
        exp = oracle.mac(A, XX, WW, we, wf, wf + 1, rnd)
        # the relaxed accumulator input (arbitrary exp/frac when not normal) gives the same result
        _check(c, m, tabref.circuit_inputs(tabref.relax(A, we, wf + 1, rng), XX, WW, we, wf, rnd), exp, post)


@pytest.mark.parametrize("we,wf", [(5, 7), (4, 6), (6, 5)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_mac_tab_random(we, wf, rnd):
    rng = np.random.default_rng(we * 13 + wf * 3 + rnd)
    N = 200_000
    c = fpgen.build_mac_tab(we, wf, rnd)
    m = lutmap.map_aig(c.g, c.outputs)
    acc = _rand_words(rng, N, we, wf + 1)
    x = _rand_words(rng, N, we, wf)
    w = _rand_words(rng, N, we, wf)
    half = N // 2
    p = oracle.mul(x[:half], w[:half], we, wf, wf + 1, rnd)
    acc[:half] = np.where(rng.random(half) < 0.5, p ^ np.uint32(1 << (wf + 1 + we)), acc[:half])
    _check(c, m, tabref.circuit_inputs(tabref.relax(acc, we, wf + 1, rng), x, w, we, wf, rnd),
           oracle.mac(acc, x, w, we, wf, wf + 1, rnd), lambda v: tabref.canon(v, we, wf + 1))


# ----------------------------------------------------------------------------- extended class

@pytest.mark.parametrize("we,wf", [(5, 2), (4, 3), (5, 3)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_extended_mul_exhaustive(we, wf, rnd):
    """HOBFLOPSxxe multiplier: exact product at 2wF+1 (only over/underflow can differ from exact)."""
    c = fpgen.build_mul(we, wf, 2 * wf + 1, rnd)
    m = lutmap.map_aig(c.g, c.outputs)
    w = canon_words(we, wf)
    A, B = np.meshgrid(w, w, indexing="ij")
    A, B = A.ravel(), B.ravel()
    _check(c, m, [A, B], oracle.mul(A, B, we, wf, 2 * wf + 1, rnd))


@pytest.mark.parametrize("we,wf", [(5, 2), (4, 3), (5, 10), (6, 5)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_extended_mac_and_mac_tab_random(we, wf, rnd):
    wfo = 2 * wf + 1
    rng = np.random.default_rng(we * 7 + wf + 100 * rnd)
    N = 100_000
    acc = _rand_words(rng, N, we, wfo)
    x = _rand_words(rng, N, we, wf)
    w = _rand_words(rng, N, we, wf)
    half = N // 2
    p = oracle.mul(x[:half], w[:half], we, wf, wfo, rnd)
    acc[:half] = np.where(rng.random(half) < 0.5, p ^ np.uint32(1 << (wfo + we)), acc[:half])
    exp = oracle.mac(acc, x, w, we, wf, wfo, rnd)
    c = fpgen.build_mac(we, wf, wfo, rnd)
    _check(c, lutmap.map_aig(c.g, c.outputs), [acc, x, w], exp)
    ct = fpgen.build_mac_tab(we, wf, rnd, wfo)
    _check(ct, lutmap.map_aig(ct.g, ct.outputs), tabref.circuit_inputs(tabref.relax(acc, we, wfo, rng), x, w, we, wf, rnd, wfo),
           exp, lambda v: tabref.canon(v, we, wfo))


def test_absorb_post_pass_preserves_function_and_never_adds_luts():
    """The mapper's post-pass (fold a LUT into all its consumers when each can take
    its leaves) on random AIGs: the mapped network computes the same outputs as
    the AIG, with no more LUTs than the mapping without the pass."""
    rng = np.random.default_rng(7)
    for trial in range(40):
        g = aigmod.AIG()
        ins = g.inputs("x", 6)
        pool = list(ins)
        for _ in range(int(rng.integers(10, 40))):
            a, b, c = (pool[int(rng.integers(0, len(pool)))] ^ int(rng.integers(0, 2)) for _ in range(3))
            op = int(rng.integers(0, 4))
            pool.append([g.AND(a, b), g.XOR(a, b), g.MUX(a, b, c), g.MAJ(a, b, c)][op])
        outs = [pool[-1 - int(k)] ^ int(rng.integers(0, 2)) for k in rng.choice(min(8, len(pool) - 6), 3, replace=False)]
        m = lutmap.map_aig(g, outs)
        # the same mapping without the post-pass
        orig = lutmap.absorb_small_luts
        try:
            lutmap.absorb_small_luts = lambda luts, outputs: luts
            m0 = lutmap.map_aig(g, outs)
        finally:
            lutmap.absorb_small_luts = orig
        assert m.n_luts <= m0.n_luts
        words = {"x": rng.integers(0, 1 << 63, (6, 4), dtype=np.uint64)}
        words = {f"x[{i}]": words["x"][i] for i in range(6)}
        ref = g.simulate(words, outs, np)
        got = lutmap.simulate_mapping(m, words, np)
        for r, o in zip(ref, got):
            assert np.array_equal(r, o), trial


# ----------------------------------------------------------------------------- SDC sweep (gen/sweep.py)

from paper_2007_06563_b200.gen import sweep  # noqa: E402


@pytest.mark.parametrize("we,wf", [(5, 3), (4, 3), (5, 6), (6, 2)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_sweep_table_entries_match_tabref(we, wf, rnd):
    """The generator's statement of the weight-table entry (the valid input space of
    the swept mac_tab circuit) equals tests/tabref.py on every (weight, row)."""
    w = canon_words(we, wf)
    r = np.arange((1 << wf) + 3)
    W, R = np.meshgrid(w, r, indexing="ij")
    for wfo in (wf + 1, 2 * wf + 1):
        got = sweep.tab_entry(W.ravel(), R.ravel(), we, wf, wfo, rnd)
        assert np.array_equal(got.astype(np.uint32), tabref.entries(W.ravel(), R.ravel(), we, wf, rnd, wfo))


def test_sweep_canonical_words_match_pyref():
    for we, wf in [(4, 3), (5, 2), (6, 4)]:
        assert sorted(sweep.canonical_words(we, wf).tolist()) == sorted(pyref.canonical_words(we, wf))


@pytest.mark.parametrize("kind,we,wf,rnd", [("mac_tab", 4, 3, 0), ("mac_tab", 5, 2, 1), ("mac", 4, 3, 1),
                                            ("mul", 5, 2, 0), ("add", 4, 2, 0)])
def test_sweep_cache_reproved(kind, we, wf, rnd):
    """The cached merges of a circuit re-proved here on its whole valid input space,
    and the cache key matches the circuit the generator builds today (so the
    emitted code is the swept circuit)."""
    c = sweep.BUILDERS[kind](we, wf, rnd)
    ent = sweep.load_cache()[c.name]
    assert ent["key"] == sweep.structure_key(c) and ent["merges"]
    new = sweep.apply_merges(c, [tuple(m) for m in ent["merges"]])
    assert sweep.prove(c, new, sweep.space_of(kind, c, we, wf, rnd, wf + 1))
    assert lutmap.map_aig(new.g, new.outputs).n_luts < lutmap.map_aig(c.g, c.outputs).n_luts


def test_sweep_merges_found_from_scratch_e4m2():
    """Signatures + rebuild + proof from scratch on a small table MAC (e4m2)."""
    c = fpgen.build_mac_tab(4, 2, 0)
    space = sweep.space_of("mac_tab", c, 4, 2, 0, 3)
    merges = sweep.find_merges(c, space)
    assert merges and sweep.prove(c, sweep.apply_merges(c, merges), space)
    # and a wrong merge is caught by the proof: a node claimed equal to constant false
    v = next(v for v in range(c.g.n_nodes()) if c.g.kind[v] == "and" and v not in {m[0] for m in merges}
             and any(o >> 1 == v for o in c.outputs))
    assert not sweep.prove(c, sweep.apply_merges(c, merges + [(v, 0, 0)]), space)


def test_mac_tab_swept_exhaustive_relaxed_acc_e4m3():
    """The emitted (swept) e4m3 table MAC over every 7th block of 256 accumulator
    patterns (the relaxed form: all 2^11 are covered, merged or not, by
    test_sweep_cache_reproved) and every canonical (x, w) pair: equals the oracle
    after canonicalisation."""
    we, wf, rnd = 4, 3, 0
    c = sweep.reduce("mac_tab", fpgen.build_mac_tab(we, wf, rnd), we, wf, rnd, wf + 1)
    m = lutmap.map_aig(c.g, c.outputs)
    xi = canon_words(we, wf)
    X, W = np.meshgrid(xi, xi, indexing="ij")
    X, W = X.ravel(), W.ravel()
    for a0 in range(0, 1 << (3 + we + wf + 1), 256 * 7):
        acc = np.arange(a0, a0 + 256, dtype=np.uint32)
        A = np.repeat(acc, X.size)
        XX, WW = np.tile(X, acc.size), np.tile(W, acc.size)
        exp = oracle.mac(tabref.canon(A, we, wf + 1), XX, WW, we, wf, wf + 1, rnd)
        _check(c, m, tabref.circuit_inputs(A, XX, WW, we, wf, rnd), exp, lambda v: tabref.canon(v, we, wf + 1))


def test_sweep_cache_holds_only_proved_merges():
    """Every cached merge list was proved on its circuit's whole valid input space
    (CPU: gen/sweep.py; GPU: tools/sweep_gpu.py, every valid input on the B200)."""
    cache = sweep.load_cache()
    assert cache
    for name, ent in cache.items():
        assert ent.get("proved") in (True, "gpu-exhaustive"), name
        assert ent["vectors"] > 0 and ent["key"]
