"""CUDA path vs oracle, bit-exact, through the C ABI (-m gpu).

Every comparison is on uint32 words: the GPU result is unpacked by the GPU
unpack kernel and compared element by element with the oracle's words.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import pyref
from gpu_util import hobf, to_dev_words, to_np_words, group_planes, ungroup_planes
from paper_2007_06563_b200 import inputs

pytestmark = pytest.mark.gpu

SWEEP = [(we, wf) for we in (4, 5, 6) for wf in range(2, 11)]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def special_floats():
    return np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, -1.0, 1e-45, -1e-45, 3.4e38, -3.4e38,
                     2.0 ** -15, 2.0 ** -16, 131008.0, 131072.0, 65504.0, 480.0, 464.0, 0.1, 2.1875],
                    dtype=np.float32)


# ----------------------------------------------------------------------------- quantise / pack / unpack

@pytest.mark.parametrize("we,wf", [(5, 10), (5, 3), (4, 3), (6, 2), (4, 10), (6, 9), (5, 2), (7, 12), (8, 7), (2, 1)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_quantize_pack_unpack_matches_oracle_encode(we, wf, rnd):
    """Both pack / unpack paths: ragged rows (warp-ballot kernels) and dense rows
    (C % 32 == 0: thread-per-group register transpose), the float32 fast
    quantiser (we <= 7) and the general one (we = 8)."""
    H = hobf()
    rng = np.random.default_rng(we * 100 + wf + rnd)
    x = (rng.standard_normal(50_000) * np.exp(rng.uniform(-25, 25, 50_000))).astype(np.float32)
    x = np.concatenate([x, special_floats()])
    for rows, c in [(x.size // 50, 50), (1, x.size), (x.size // 20, 20), (x.size // 64, 64), (x.size // 32, 32),
                    (1, x.size // 32 * 32)]:
        xx = x[: rows * c].reshape(rows, c)
        planes = H.quantize_pack(we, wf, torch.from_numpy(xx).cuda(), rnd)
        got = to_np_words(H.unpack(we, wf, planes, rows, c))
        exp = oracle.encode_f32(xx, we, wf, rnd)
        assert np.array_equal(got, exp)
        if we > 7:  # float32 holds every F(we <= 7, wf <= 23) value exactly; unpack_f32 refuses we = 8
            with pytest.raises(H.HobfError):
                H.unpack_f32(we, wf, planes, rows, c)
            continue
        # unpack to float32 is the exact decoded value
        f = H.unpack_f32(we, wf, planes, rows, c).cpu().numpy()
        dec = oracle.decode_f64(exp, we, wf)
        both_nan = np.isnan(f) & np.isnan(dec)
        assert np.array_equal(f[~both_nan].astype(np.float64), dec[~both_nan])
        assert np.array_equal(np.signbit(f[~both_nan]), np.signbit(dec[~both_nan]))


@pytest.mark.parametrize("we,wf", [(5, 3), (4, 10), (6, 5)])
def test_pack_canonicalises_dense_rows(we, wf):
    """The thread-per-group pack / unpack (C % 32 == 0) canonicalise like the ragged path."""
    H = hobf()
    rng = np.random.default_rng(12)
    rows, c = 257, 96
    raw = rng.integers(0, 1 << 32, (rows, c), dtype=np.uint64).astype(np.uint32)
    planes = H.pack(we, wf, to_dev_words(raw))
    got = to_np_words(H.unpack(we, wf, planes, rows, c))
    nb = 3 + we + wf
    assert np.array_equal(got, oracle.canon(raw & np.uint32((1 << nb) - 1), we, wf))
    assert np.all(to_np_words(planes)[:, :, nb:] == 0)


@pytest.mark.parametrize("we,wf", [(5, 3), (4, 10), (6, 5)])
def test_pack_canonicalises_and_round_trips(we, wf):
    H = hobf()
    rng = np.random.default_rng(11)
    rows, c = 333, 77  # ragged lanes
    raw = rng.integers(0, 1 << 32, (rows, c), dtype=np.uint64).astype(np.uint32)
    planes = H.pack(we, wf, to_dev_words(raw))
    assert tuple(planes.shape) == (rows, 3, H.nplanes(3 + we + wf))
    got = to_np_words(H.unpack(we, wf, planes, rows, c))
    nb = 3 + we + wf
    exp = oracle.canon(raw & np.uint32((1 << nb) - 1), we, wf)
    assert np.array_equal(got, exp)
    # padding lanes (c=77 -> lanes 13..31 of group 2) and padding planes are zero
    p = to_np_words(planes)
    assert np.all((p[:, 2, :] >> np.uint32(13)) == 0)
    assert np.all(p[:, :, nb:] == 0)
    # lane/bit layout (L18): bit l of plane j is bit j of element 32g+l
    canon = exp
    for (r, g, j, l) in [(0, 0, 0, 0), (5, 1, 3, 17), (332, 2, nb - 1, 12)]:
        assert ((p[r, g, j] >> l) & 1) == ((canon[r, 32 * g + l] >> j) & 1)


def test_empty_and_error_paths():
    H = hobf()
    f = H.Fmt(5, 3)
    z = torch.zeros((0, 5), dtype=torch.int32, device="cuda")
    out = H.pack(5, 3, z)
    assert out.numel() == 0
    with pytest.raises(H.HobfError) as e:
        H.gate_count(H.Fmt(7, 3))
    assert e.value.status == 3
    with pytest.raises(H.HobfError) as e:
        H.conv2d(H.Fmt(7, 3, extended=1), torch.zeros(64, dtype=torch.int32, device="cuda"), 1, 2, 2, 1,
                 torch.zeros(64, dtype=torch.int32, device="cuda"), 3, 3, 1)
    assert e.value.status == 3
    with pytest.raises(H.HobfError) as e:  # kernel larger than padded input
        H.conv2d(f, torch.zeros(64, dtype=torch.int32, device="cuda"), 1, 1, 1, 1,
                 torch.zeros(64, dtype=torch.int32, device="cuda"), 5, 5, 1, 1, 1)
    assert e.value.status == 2
    # n = 0 is a no-op
    y = H.conv2d(f, torch.zeros(64, dtype=torch.int32, device="cuda"), 0, 4, 4, 8,
                 torch.zeros(9 * 8 * 12, dtype=torch.int32, device="cuda"), 3, 3, 32)
    assert y.numel() == 0


# ----------------------------------------------------------------------------- MAC circuits

def canon_words(we, wf):
    return np.array(pyref.canonical_words(we, wf), dtype=np.uint32)


def run_mac(f, acc, a, b):
    """acc/a/b: 1-D words (same length, multiple of 32) -> GPU mac result words."""
    H = hobf()
    n = acc.size
    pa = group_planes(acc, f.we, f.wfo)
    pa = pa.contiguous()
    px = group_planes(a, f.we, f.wf)
    pw = group_planes(b, f.we, f.wf)
    H.mac_planes(f, pa, px, pw)
    return ungroup_planes(pa, f.we, f.wfo, n)


@pytest.mark.parametrize("rnd", [0, 1])
def test_mac_exhaustive_e5m3(rnd):
    """Every (acc, x, w) triple of canonical e5m3 operands / e5m4 accumulators:
    1029 x 517^2 = 2.75e8 MACs (ladder step 5)."""
    H = hobf()
    f = H.Fmt(5, 3, rnd)
    wi = canon_words(5, 3)
    wo = canon_words(5, 4)
    X, W = np.meshgrid(wi, wi, indexing="ij")
    X, W = X.ravel(), W.ravel()                     # 267,289 pairs
    pad = (-X.size) % 32
    X = np.concatenate([X, np.zeros(pad, np.uint32)])
    W = np.concatenate([W, np.zeros(pad, np.uint32)])
    chunk = 16
    for s in range(0, wo.size, chunk):
        accs = wo[s:s + chunk]
        A = np.repeat(accs, X.size)
        XX = np.tile(X, accs.size)
        WW = np.tile(W, accs.size)
        got = run_mac(f, A, XX, WW)
        exp = oracle.mac(A, XX, WW, 5, 3, 4, rnd)
        bad = np.nonzero(got != exp)[0]
        assert bad.size == 0, [(hex(A[i]), hex(XX[i]), hex(WW[i]), hex(got[i]), hex(exp[i])) for i in bad[:5]]


@pytest.mark.parametrize("we,wf", SWEEP)
@pytest.mark.parametrize("rnd", [0, 1])
def test_mac_random_all_formats(we, wf, rnd):
    H = hobf()
    f = H.Fmt(we, wf, rnd)
    rng = np.random.default_rng(we * 1000 + wf * 10 + rnd)
    N = 1 << 18

    def rand_words(wfx, n):
        s = rng.integers(0, 2, n)
        e = rng.integers(0, 1 << we, n)
        fr = rng.integers(0, 1 << wfx, n)
        w = ((1 << (wfx + we + 1)) | (s << (wfx + we)) | (e << wfx) | fr).astype(np.uint32)
        # sprinkle specials (zero, -0, inf, -inf, nan)
        sp = rng.random(n) < 0.05
        specials = np.array(pyref.canonical_words(we, 1)[:5], np.uint32)
        specials = np.array([0, 1 << (wfx + we), 2 << (wfx + we + 1), (2 << (wfx + we + 1)) | (1 << (wfx + we)),
                             3 << (wfx + we + 1)], np.uint32)
        w[sp] = rng.choice(specials, sp.sum())
        return w

    A = rand_words(wf + 1, N)
    X = rand_words(wf, N)
    Wt = rand_words(wf, N)
    # half the accumulators near the product magnitude so cancellation / rounding paths are hit
    half = N // 2
    prod = oracle.mul(X[:half], Wt[:half], we, wf, wf + 1, rnd)
    A[:half] = np.where(rng.random(half) < 0.5, prod ^ np.uint32(1 << (wf + 1 + we)), A[:half])
    got = run_mac(f, A, X, Wt)
    exp = oracle.mac(A, X, Wt, we, wf, wf + 1, rnd)
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, [(hex(A[i]), hex(X[i]), hex(Wt[i]), hex(got[i]), hex(exp[i])) for i in bad[:5]]


def test_gate_counts_reported():
    H = hobf()
    import json, os
    path = os.path.join(os.path.dirname(H.LIB_PATH), "csrc", "gen", "gate_counts.json")
    counts = json.load(open(path))
    for (we, wf) in SWEEP:
        for rnd, name in ((0, "rne"), (1, "rtz")):
            g = H.gate_count(H.Fmt(we, wf, rnd))
            assert g["mac"] == counts[f"e{we}m{wf}_{name}"]["g_mac"]
            assert g["mac_tab"] == counts[f"e{we}m{wf}_{name}"]["g_tab"]
            gx = H.gate_count(H.Fmt(we, wf, rnd, extended=1))
            assert gx["mac_tab"] == counts[f"e{we}m{wf}x_{name}"]["g_tab"]


# ----------------------------------------------------------------------------- conv

def gpu_conv(x_f32, w_f32, f, stride=1, pad=1, relu=0, prepared=False):
    """float32 NHWC x and KhKwCinCout w -> quantise+pack on GPU -> conv -> unpack words.
    prepared=True runs hobf_prepare_weights + hobf_conv2d_prepared (weight tables)."""
    H = hobf()
    n, h, w, cin = x_f32.shape
    kh, kw, _, cout = w_f32.shape
    xp = H.quantize_pack(f.we, f.wf, torch.from_numpy(x_f32.reshape(-1, cin)).cuda(), f.round)
    wp = H.quantize_pack(f.we, f.wf, torch.from_numpy(w_f32.reshape(-1, cout)).cuda(), f.round)
    if prepared:
        wt = H.prepare_weights(f, wp, kh, kw, cin, cout)
        xr = H.prepare_activations(f, xp, n, h, w, cin, pad)
        yp = H.conv2d_prepared(f, xr, n, h, w, cin, wt, kh, kw, cout, stride, pad, relu)
    else:
        yp = H.conv2d(f, xp, n, h, w, cin, wp, kh, kw, cout, stride, pad, relu)
    ho, wo = H.conv_out_hw(h, w, kh, kw, stride, pad)
    y = to_np_words(H.unpack(f.we, f.wfo, yp, n * ho * wo, cout)).reshape(n, ho, wo, cout)
    return y


def oracle_conv(x_f32, w_f32, f, stride=1, pad=1, relu=0):
    xq = oracle.encode_f32(x_f32, f.we, f.wf, f.round)
    wq = oracle.encode_f32(w_f32, f.we, f.wf, f.round)
    return oracle.conv2d(xq, wq, f.we, f.wf, f.wfo, f.round, stride, pad, relu)


def test_conv_C1_full():
    """configs[0] in full, both ReLU settings, both rounding modes."""
    H = hobf()
    cfg = inputs.CONFIGS["C1"]
    x, w = inputs.draw(cfg)
    for rnd in (0, 1):
        f = H.Fmt(5, 10, rnd)
        for relu in (0, 1):
            got = gpu_conv(x, w, f, relu=relu)
            exp = oracle_conv(x, w, f, relu=relu)
            assert np.array_equal(got, exp), (rnd, relu, np.argwhere(got != exp)[:5])


def test_conv_prepared_int64_indexing():
    """Maximum-size case: 7.5 M 1x1 images x 32 channels, so the zero-padded record
    buffer holds 2.16e9 words (indices past 2^31) and the output planes 9e7 words;
    the bench's launch shape (TMA-staged tables, 128 x 6 CTAs/SM).  Sampled outputs
    (the last images included) vs the oracle.  ~12 GB of device memory."""
    H = hobf()
    free, _ = torch.cuda.mem_get_info()
    if free < 40e9:
        pytest.skip("needs ~12 GB of free device memory (+ headroom)")
    n, h, w, cin, cout = 7_500_000, 1, 1, 32, 32
    f = H.Fmt(5, 3, 0)
    x, wt = inputs.small_case(511, n, h, w, cin, cout, "relu_normal", 0.2)
    assert n * cin * 3 * 3 > 2 ** 31
    xt = torch.from_numpy(x).cuda()
    wp = H.quantize_pack(5, 3, torch.from_numpy(wt.reshape(-1, cout)).cuda(), 0)
    tab = H.prepare_weights(f, wp, 3, 3, cin, cout)
    xr = H.quantize_activations(f, xt, 1)
    del xt
    yp = H.conv2d_prepared(f, xr, n, h, w, cin, tab, 3, 3, cout, 1, 1, 0)
    del xr
    got = to_np_words(H.unpack(5, f.wfo, yp, n * h * w, cout)).ravel()
    rng = np.random.default_rng(7)
    idx = np.unique(np.concatenate([rng.integers(0, got.size, 300), np.arange(got.size - 96, got.size)]))
    xq = oracle.encode_f32(x, 5, 3, 0)
    wq = oracle.encode_f32(wt, 5, 3, 0)
    exp = oracle.conv2d_sample(xq, wq, idx, 5, 3, f.wfo, 0)
    assert np.array_equal(got[idx], exp)


@pytest.mark.parametrize("we,wf", [(5, 3), (4, 3), (6, 2), (4, 7)])
def test_conv_prepared_full_vs_oracle(we, wf):
    """The weight-table path in full on a C1-shaped layer with every special class present."""
    H = hobf()
    x, w = inputs.small_case(77, 2, 8, 8, 48, 64)
    x[0, 0, :4, 0] = [np.inf, -np.inf, np.nan, -0.0]
    w[0, 0, 1, :3] = [np.inf, np.nan, 0.0]
    for rnd in (0, 1):
        f = H.Fmt(we, wf, rnd)
        for relu in (0, 1):
            got = gpu_conv(x, w, f, relu=relu, prepared=True)
            exp = oracle_conv(x, w, f, relu=relu)
            assert np.array_equal(got, exp), (rnd, relu, np.argwhere(got != exp)[:5])
            assert np.array_equal(got, gpu_conv(x, w, f, relu=relu, prepared=False))


@pytest.mark.parametrize("variant", [3, 4, 5, 6, 7, 8, 10, 11, 12, 13, 14, 15])  # 12-14 run as 4 here (planes out)
@pytest.mark.parametrize("we,wf,kh,kw", [(5, 3, 3, 3), (4, 6, 2, 3), (5, 10, 3, 3), (6, 2, 3, 2), (4, 6, 3, 3),
                                         (5, 7, 3, 3), (5, 8, 3, 3), (6, 9, 3, 3)])
def test_conv_prepared_every_schedule(variant, we, wf, kh, kw):
    """Every kernel schedule of hobf_conv2d_prepared_variant gives the oracle's words:
    several 128-pixel CTAs with a ragged tail, a ragged last Cout group, cin not a
    multiple of the 3-row unroll (kh = 2), stride 2, specials present."""
    H = hobf()
    n, h, w, cin, cout, stride, pad = 3, 11, 13, 5, 40, 1, 1
    x, wt = inputs.small_case(91 + variant, n, h, w, cin, cout, "normal", 0.4, kh=kh, kw=kw)
    x[0, 0, :3, 0] = [np.inf, np.nan, -0.0]
    wt[0, 0, 1, :2] = [np.inf, 0.0]
    for rnd in (0, 1):
        f = H.Fmt(we, wf, rnd)
        for s_ in (stride, 2):
            exp = oracle_conv(x, wt, f, stride=s_, pad=pad, relu=0)
            xp = H.quantize_pack(we, wf, torch.from_numpy(x.reshape(-1, cin)).cuda(), rnd)
            wp = H.quantize_pack(we, wf, torch.from_numpy(wt.reshape(-1, cout)).cuda(), rnd)
            tab = H.prepare_weights(f, wp, kh, kw, cin, cout)
            xr = H.prepare_activations(f, xp, n, h, w, cin, pad)
            yp = H.conv2d_prepared(f, xr, n, h, w, cin, tab, kh, kw, cout, s_, pad, 0, variant=variant)
            ho, wo = H.conv_out_hw(h, w, kh, kw, s_, pad)
            got = to_np_words(H.unpack(we, f.wfo, yp, n * ho * wo, cout)).reshape(exp.shape)
            assert np.array_equal(got, exp), (variant, rnd, s_, np.argwhere(got != exp)[:5])


@pytest.mark.parametrize("shape", [
    # n, h, w, cin, cout, kh, kw, stride, pad
    (2, 9, 7, 40, 50, 3, 3, 1, 1),     # ragged cin and cout, several tiles
    (1, 5, 6, 33, 64, 3, 3, 2, 0),     # stride 2, no padding
    (3, 4, 4, 1, 1, 3, 3, 1, 1),       # single channel in/out
    (1, 6, 5, 8, 96, 1, 1, 1, 0),      # 1x1 kernel
    (1, 7, 7, 5, 32, 5, 5, 1, 2),      # 5x5 kernel
    (1, 1, 1, 16, 32, 3, 3, 1, 1),     # 1x1 image: every tap but the centre is padding
])
@pytest.mark.parametrize("we,wf,prepared", [(5, 3, 0), (4, 3, 0), (5, 10, 0), (6, 7, 0),
                                             (5, 3, 1), (4, 3, 1), (6, 7, 1), (4, 2, 1), (5, 5, 1)])
def test_conv_small_shapes(shape, we, wf, prepared):
    H = hobf()
    n, h, w, cin, cout, kh, kw, stride, pad = shape
    x, wt = inputs.small_case(sum(shape) + we + wf, n, h, w, cin, cout, "normal", 0.5, kh, kw)
    for rnd in (0, 1):
        f = H.Fmt(we, wf, rnd)
        relu = rnd  # alternate
        got = gpu_conv(x, wt, f, stride, pad, relu, prepared=bool(prepared))
        exp = oracle_conv(x, wt, f, stride, pad, relu)
        assert np.array_equal(got, exp), np.argwhere(got != exp)[:5]


@pytest.mark.parametrize("prepared", [False, True])
def test_conv_specials_propagate(prepared):
    """inf / NaN / overflow inputs: 0*inf = NaN through padding taps, inf + -inf = NaN."""
    H = hobf()
    f = H.Fmt(5, 3, 0)
    rng = np.random.default_rng(3)
    x = rng.standard_normal((1, 5, 5, 8)).astype(np.float32)
    w = rng.standard_normal((3, 3, 8, 32)).astype(np.float32)
    x[0, 2, 2, 3] = np.inf
    x[0, 0, 0, 1] = np.nan
    x[0, 4, 4, 2] = 6e4       # near e5m3 max: products overflow
    w[1, 1, 0, :] = np.inf
    w[0, 2, 5, 7] = -np.inf
    w[2, 2, 6, :] = 3e4
    x[0, 1, 3, 4] = 1e-4      # tiny: products underflow to zero
    w[1, 0, 4, 3] = -2e-5
    for relu in (0, 1):
        got = gpu_conv(x, w, f, relu=relu, prepared=prepared)
        exp = oracle_conv(x, w, f, relu=relu)
        assert np.array_equal(got, exp)


@pytest.mark.parametrize("name,prepared", [("C2", 0), ("C3", 0), ("C4", 0), ("C3", 1), ("C4", 1)])
def test_conv_configs_sampled(name, prepared):
    """Full-size configs in the bench launch configuration, checked on sampled
    outputs the oracle computes one by one."""
    H = hobf()
    cfg = inputs.CONFIGS[name]
    x, w = inputs.draw(cfg)
    we, wf = cfg.formats[0]
    f = H.Fmt(we, wf, 0)
    got = gpu_conv(x, w, f, prepared=bool(prepared))
    xq = oracle.encode_f32(x, we, wf, 0)
    wq = oracle.encode_f32(w, we, wf, 0)
    rng = np.random.default_rng(5)
    total = got.size
    idx = np.unique(np.concatenate([rng.integers(0, total, 3000), np.arange(0, 64), np.arange(total - 64, total)]))
    exp = oracle.conv2d_sample(xq, wq, idx, we, wf, wf + 1, 0)
    assert np.array_equal(got.ravel()[idx], exp)


def test_conv_C5_sweep_sampled():
    H = hobf()
    cfg = inputs.CONFIGS["C5"]
    x, w = inputs.draw(cfg)  # full batch: the bench's launch configuration (staged schedules 7 / 8)
    rng = np.random.default_rng(6)
    for (we, wf) in cfg.formats:
        f = H.Fmt(we, wf, 0)
        got = gpu_conv(x, w, f, prepared=H.wtab_words(f, 3, 3, cfg.cin, cfg.cout) > 0)
        xq = oracle.encode_f32(x, we, wf, 0)
        wq = oracle.encode_f32(w, we, wf, 0)
        idx = rng.integers(0, got.size, 150)
        exp = oracle.conv2d_sample(xq, wq, idx, we, wf, wf + 1, 0)
        assert np.array_equal(got.ravel()[idx], exp), (we, wf)


def test_conv_public_api_float():
    """hobf.Conv2d (quantise+pack -> conv -> unpack to float32) equals the oracle's values."""
    H = hobf()
    x, w = inputs.small_case(21, 2, 10, 11, 24, 40)
    f = H.Fmt(5, 10, 0)
    layer = H.Conv2d(torch.from_numpy(w).cuda(), f, relu=True)
    y = layer(torch.from_numpy(x).cuda()).cpu().numpy()
    exp = oracle.decode_f64(oracle_conv(x, w, f, relu=1), 5, 11)
    assert np.array_equal(y.astype(np.float64), exp)


@pytest.mark.parametrize("we,wf,pad", [(5, 3, 1), (4, 3, 0), (5, 10, 2), (6, 7, 1)])
def test_activation_records_two_ways_agree(we, wf, pad):
    """quantize_activations(float32) == prepare_activations(quantize_pack(float32)), and the
    record's low bits are the oracle's encoding (padding = +0 with the zero row)."""
    H = hobf()
    rng = np.random.default_rng(we + wf + pad)
    n, h, w, cin = 2, 9, 37, 40
    x = (rng.standard_normal((n, h, w, cin)) * np.exp(rng.uniform(-8, 8, (n, h, w, cin)))).astype(np.float32)
    x.ravel()[:20] = special_floats()[:20]
    for rnd in (0, 1):
        f = H.Fmt(we, wf, rnd)
        xt = torch.from_numpy(x).cuda()
        r1 = to_np_words(H.quantize_activations(f, xt, pad))
        xp = H.quantize_pack(we, wf, xt.reshape(-1, cin), rnd)
        r2 = to_np_words(H.prepare_activations(f, xp, n, h, w, cin, pad))
        assert np.array_equal(r1, r2)
        rec = r1.reshape(n, cin, h + 2 * pad, w + 2 * pad)
        inner = rec[:, :, pad:pad + h, pad:pad + w] & np.uint32((1 << 20) - 1)
        assert np.array_equal(inner.transpose(0, 2, 3, 1), oracle.encode_f32(x, we, wf, rnd))
        if pad:
            assert np.all(rec[:, :, 0, :] == np.uint32((1 << wf) << 20))



@pytest.mark.parametrize("n,h,w,cin", [(70_000, 1, 1, 8), (70_000, 1, 2, 5)])
def test_activation_records_many_images(n, h, w, cin):
    """More images than a grid's y / z dimension holds (65535): the flattened-tile
    quantise kernels (row kernel for cin % 4 == 0, tile-transpose kernel otherwise)."""
    H = hobf()
    rng = np.random.default_rng(n + cin)
    x = rng.standard_normal((n, h, w, cin)).astype(np.float32)
    f = H.Fmt(5, 3, 0)
    pad = 1
    rec = to_np_words(H.quantize_activations(f, torch.from_numpy(x).cuda(), pad)).reshape(n, cin, h + 2, w + 2)
    inner = rec[:, :, pad:pad + h, pad:pad + w] & np.uint32((1 << 20) - 1)
    assert np.array_equal(inner.transpose(0, 2, 3, 1), oracle.encode_f32(x, 5, 3, 0))
    assert np.all(rec[:, :, 0, :] == np.uint32((1 << 3) << 20))


# ----------------------------------------------------------------------------- extended class

@pytest.mark.parametrize("we,wf", [(5, 2), (5, 3), (4, 3), (5, 10), (6, 6)])
@pytest.mark.parametrize("prepared", [False, True])
def test_conv_extended_class(we, wf, prepared):
    """HOBFLOPSxxe: exact products, accumulator at 2wF+1, both rounding modes."""
    H = hobf()
    x, wt = inputs.small_case(we * 10 + wf, 2, 7, 9, 40, 40, "normal", 0.5)
    for rnd in (0, 1):
        f = H.Fmt(we, wf, rnd, extended=1)
        assert f.wfo == 2 * wf + 1
        got = gpu_conv(x, wt, f, 1, 1, rnd, prepared=prepared)
        exp = oracle_conv(x, wt, f, 1, 1, rnd)
        assert np.array_equal(got, exp), np.argwhere(got != exp)[:5]


@pytest.mark.parametrize("variant", [4, 6, 7, 8, 10, 11, 15])
@pytest.mark.parametrize("we,wf", [(5, 3), (6, 5), (4, 6), (5, 7), (5, 8), (5, 9)])
def test_conv_extended_every_schedule(variant, we, wf):
    """Extended class through the explicit schedules (the auto schedule of the small
    cases above is the latency-bound one): staged channel blocks, kernel rows, taps,
    L1-served; ragged CTAs and Cout group, stride 1 and 2."""
    H = hobf()
    n, h, w, cin, cout, pad = 3, 11, 13, 5, 40, 1
    x, wt = inputs.small_case(300 + 10 * we + wf, n, h, w, cin, cout, "normal", 0.4)
    for rnd in (0, 1):
        f = H.Fmt(we, wf, rnd, extended=1)
        for s_ in (1, 2):
            exp = oracle_conv(x, wt, f, stride=s_, pad=pad, relu=0)
            xp = H.quantize_pack(we, wf, torch.from_numpy(x.reshape(-1, cin)).cuda(), rnd)
            wp = H.quantize_pack(we, wf, torch.from_numpy(wt.reshape(-1, cout)).cuda(), rnd)
            tab = H.prepare_weights(f, wp, 3, 3, cin, cout)
            xr = H.prepare_activations(f, xp, n, h, w, cin, pad)
            yp = H.conv2d_prepared(f, xr, n, h, w, cin, tab, 3, 3, cout, s_, pad, 0, variant=variant)
            ho, wo = H.conv_out_hw(h, w, 3, 3, s_, pad)
            got = to_np_words(H.unpack(we, f.wfo, yp, n * ho * wo, cout)).reshape(exp.shape)
            assert np.array_equal(got, exp), (variant, rnd, s_, np.argwhere(got != exp)[:5])


def test_staged_launch_shapes_same_format():
    """One format through both launch shapes of the staged schedule in one process
    (256 x 3 for a partial wave, then 128 x 6 for >= 8 warps per SMSP): each kernel
    instantiation needs its own > 48 KB shared-memory opt-in (a 49 KB table pair)."""
    H = hobf()
    f = H.Fmt(4, 5, 1, extended=1)
    rng = np.random.default_rng(17)
    for n, h, w, cin, cout in [(2, 11, 13, 3, 40), (26, 56, 56, 2, 64)]:
        x, wt = inputs.small_case(400 + n, n, h, w, cin, cout, "normal", 0.5)
        xp = H.quantize_pack(4, 5, torch.from_numpy(x.reshape(-1, cin)).cuda(), 1)
        wp = H.quantize_pack(4, 5, torch.from_numpy(wt.reshape(-1, cout)).cuda(), 1)
        tab = H.prepare_weights(f, wp, 3, 3, cin, cout)
        xr = H.prepare_activations(f, xp, n, h, w, cin, 1)
        yp = H.conv2d_prepared(f, xr, n, h, w, cin, tab, 3, 3, cout, 1, 1, 0, variant=7)
        got = to_np_words(H.unpack(4, f.wfo, yp, n * h * w, cout))
        idx = rng.integers(0, got.size, 400)
        xq = oracle.encode_f32(x, 4, 5, 1)
        wq = oracle.encode_f32(wt, 4, 5, 1)
        exp = oracle.conv2d_sample(xq, wq, idx, 4, 5, f.wfo, 1)
        assert np.array_equal(got.ravel()[idx], exp), (n, h, w)


@pytest.mark.parametrize("we,wf", [(5, 3), (4, 7), (6, 10)])
@pytest.mark.parametrize("rnd", [0, 1])
def test_mac_random_extended(we, wf, rnd):
    H = hobf()
    f = H.Fmt(we, wf, rnd, extended=1)
    rng = np.random.default_rng(we * 31 + wf * 3 + rnd)
    N = 1 << 16

    def rw(wfx):
        s = rng.integers(0, 2, N)
        e = rng.integers(0, 1 << we, N)
        fr = rng.integers(0, 1 << wfx, N)
        return ((1 << (wfx + we + 1)) | (s << (wfx + we)) | (e << wfx) | fr).astype(np.uint32)

    A, X, W = rw(f.wfo), rw(wf), rw(wf)
    got = run_mac(f, A, X, W)
    exp = oracle.mac(A, X, W, we, wf, f.wfo, rnd)
    assert np.array_equal(got, exp)


# ----------------------------------------------------------------------------- layer chaining

@pytest.mark.parametrize("prepared", [False, True])
@pytest.mark.parametrize("we,wf1,wf2,ext,rnd", [(5, 3, 3, 0, 0), (5, 10, 3, 0, 0), (4, 3, 3, 1, 0), (5, 3, 3, 0, 1),
                                                (6, 2, 5, 0, 0), (5, 4, 2, 1, 1)])
def test_two_layer_chain_vs_oracle(prepared, we, wf1, wf2, ext, rnd):
    """conv -> ReLU -> re-round into the next layer's format (fused epilogue) ->
    conv, with no unpack in between, equals oracle.conv_chain word for word; the
    intermediate (next-layer) tensor also equals oracle.convert of layer 1."""
    H = hobf()
    n, h, w, c0, c1, c2 = 2, 9, 11, 20, 40, 33
    x, w1 = inputs.small_case(61, n, h, w, c0, c1, "normal", 0.4)
    _, w2 = inputs.small_case(62, 1, 3, 3, c1, c2, "normal", 0.3)
    x[0, 0, :2, 0] = [np.inf, -0.0]
    f1, f2 = H.Fmt(we, wf1, rnd, extended=ext), H.Fmt(we, wf2, rnd)
    xq = oracle.encode_f32(x, we, wf1, rnd)
    w1q, w2q = oracle.encode_f32(w1, we, wf1, rnd), oracle.encode_f32(w2, we, wf2, rnd)
    exp = oracle.conv_chain(xq, [(w1q, wf1, 1, 1, 1, ext), (w2q, wf2, 2, 1, 0, 0)], we, rnd)
    mid = oracle.convert(oracle.conv2d(xq, w1q, we, wf1, f1.wfo, rnd, 1, 1, 1), we, f1.wfo, wf2, rnd)
    wp1 = H.quantize_pack(we, wf1, torch.from_numpy(w1.reshape(-1, c1)).cuda(), rnd)
    wp2 = H.quantize_pack(we, wf2, torch.from_numpy(w2.reshape(-1, c2)).cuda(), rnd)
    ho2, wo2 = H.conv_out_hw(h, w, 3, 3, 2, 1)
    if prepared and H.wtab_words(f1, 3, 3, c0, c1) > 0:
        xr = H.quantize_activations(f1, torch.from_numpy(x).cuda(), 1)
        t1, t2 = H.prepare_weights(f1, wp1, 3, 3, c0, c1), H.prepare_weights(f2, wp2, 3, 3, c1, c2)
        r2 = H.conv2d_prepared(f1, xr, n, h, w, c0, t1, 3, 3, c1, 1, 1, 1, nxt=H.Next(wf2, records=True, pad=1))
        # the records' words are the next layer's input: compare them with the oracle's conversion
        rec = to_np_words(r2).reshape(n, c1, h + 2, w + 2)
        got_mid = (rec[:, :, 1:-1, 1:-1] & 0xFFFFF).transpose(0, 2, 3, 1)
        assert np.array_equal(got_mid, mid)
        assert np.all((rec[:, :, 0, :] >> 20) == (1 << wf2)) and np.all((rec[:, :, :, 0] & 0xFFFFF) == 0)
        yp = H.conv2d_prepared(f2, r2, n, h, w, c1, t2, 3, 3, c2, 2, 1, 0)
    else:
        xp = H.quantize_pack(we, wf1, torch.from_numpy(x.reshape(-1, c0)).cuda(), rnd)
        p2 = H.conv2d(f1, xp, n, h, w, c0, wp1, 3, 3, c1, 1, 1, 1, nxt=H.Next(wf2, records=False))
        got_mid = to_np_words(H.unpack(we, wf2, p2, n * h * w, c1)).reshape(mid.shape)
        assert np.array_equal(got_mid, mid)
        yp = H.conv2d(f2, p2, n, h, w, c1, wp2, 3, 3, c2, 2, 1, 0)
    got = to_np_words(H.unpack(we, f2.wfo, yp, n * ho2 * wo2, c2)).reshape(exp.shape)
    assert np.array_equal(got, exp), np.argwhere(got != exp)[:5]


def test_chain_epilogue_argument_errors():
    H = hobf()
    f = H.Fmt(5, 3, 0)
    xr = torch.zeros(4096, dtype=torch.int32, device="cuda")
    t = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
    for nxt in (H.Next(0, True, 1), H.Next(3, True, -1), H.Next(12, True, 1), H.Next(30, False)):
        out = torch.zeros(4096, dtype=torch.int32, device="cuda") if nxt.records else None
        with pytest.raises(H.HobfError):
            H.conv2d_prepared(f, xr, 1, 4, 4, 4, t, 3, 3, 8, 1, 1, 0, out=out, nxt=nxt)


# ----------------------------------------------------------------------------- depthwise conv (MobileNets Conv dw)

def gpu_conv_dw(x_f32, w_f32, f, stride=1, pad=1, relu=0, nxt=None):
    H = hobf()
    n, h, w, c = x_f32.shape
    kh, kw, _ = w_f32.shape
    xp = H.quantize_pack(f.we, f.wf, torch.from_numpy(x_f32.reshape(-1, c)).cuda(), f.round)
    wp = H.quantize_pack(f.we, f.wf, torch.from_numpy(w_f32.reshape(-1, c)).cuda(), f.round)
    yp = H.conv2d_dw(f, xp, n, h, w, c, wp, kh, kw, stride, pad, relu, nxt=nxt)
    ho, wo = H.conv_out_hw(h, w, kh, kw, stride, pad)
    if nxt is not None:
        return yp, ho, wo
    return to_np_words(H.unpack(f.we, f.wfo, yp, n * ho * wo, c)).reshape(n, ho, wo, c)


@pytest.mark.parametrize("we,wf,ext", [(5, 3, 0), (4, 3, 0), (5, 10, 0), (6, 6, 0), (5, 3, 1), (4, 7, 1)])
@pytest.mark.parametrize("stride", [1, 2])
def test_conv_dw_vs_oracle(we, wf, ext, stride):
    """Depthwise conv: ragged channel count (several 32-lane groups + tail), ragged
    spatial tiles, specials, both rounding modes and ReLU settings."""
    H = hobf()
    x, w = inputs.small_case(71, 3, 13, 11, 75, 75, "normal", 0.5, dw=True)
    x[0, 0, :3, 0] = [np.inf, np.nan, -0.0]
    w[0, 1, :2] = [np.inf, 0.0]
    for rnd in (0, 1):
        f = H.Fmt(we, wf, rnd, extended=ext)
        xq, wq = oracle.encode_f32(x, we, wf, rnd), oracle.encode_f32(w, we, wf, rnd)
        for relu in (0, 1):
            exp = oracle.conv2d_dw(xq, wq, we, wf, f.wfo, rnd, stride, 1, relu)
            got = gpu_conv_dw(x, w, f, stride, 1, relu)
            assert np.array_equal(got, exp), (rnd, relu, np.argwhere(got != exp)[:5])


def test_conv_dw_chain_into_pointwise_records():
    """MobileNets block: depthwise 3x3 s2 -> ReLU -> re-round (fused epilogue) into
    activation records -> full 1x1 conv on the weight-table path; equals the oracle."""
    H = hobf()
    we, wf = 5, 3
    f = H.Fmt(we, wf, 0)
    n, h, w, c, m = 2, 14, 14, 64, 96
    x, wd = inputs.small_case(72, n, h, w, c, c, "relu_normal", 0.4, dw=True)
    _, wpw = inputs.small_case(73, 1, 1, 1, c, m, "normal", 0.2, kh=1, kw=1)
    rec, ho, wo = gpu_conv_dw(x, wd, f, 2, 1, 1, nxt=H.Next(wf, records=True, pad=0))
    wp = H.quantize_pack(we, wf, torch.from_numpy(wpw.reshape(-1, m)).cuda(), 0)
    tab = H.prepare_weights(f, wp, 1, 1, c, m)
    yp = H.conv2d_prepared(f, rec, n, ho, wo, c, tab, 1, 1, m, 1, 0, 0)
    got = to_np_words(H.unpack(we, f.wfo, yp, n * ho * wo, m)).reshape(n, ho, wo, m)
    xq, wdq, wpq = (oracle.encode_f32(a, we, wf) for a in (x, wd, wpw))
    mid = oracle.convert(oracle.conv2d_dw(xq, wdq, we, wf, wf + 1, 0, 2, 1, 1), we, wf + 1, wf)
    exp = oracle.conv2d(mid, wpq, we, wf, wf + 1, 0, 1, 0, 0)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("name", ["MOB", "MOBDW"])
def test_mobilenets_layer_sampled(name):
    """The paper's layer shape at full size: sampled outputs vs the oracle."""
    H = hobf()
    cfg = inputs.CONFIGS[name]
    we, wf = cfg.formats[0]
    f = H.Fmt(we, wf, 0)
    n = 2
    x, w = inputs.draw(cfg, n=n)
    if cfg.dw:
        y = gpu_conv_dw(x, w, f, cfg.stride, cfg.pad, 0)
    else:
        y = gpu_conv(x, w, f, stride=cfg.stride, pad=cfg.pad, prepared=True)
    xq, wq = oracle.encode_f32(x, we, wf), oracle.encode_f32(w, we, wf)
    if cfg.dw:
        exp = oracle.conv2d_dw(xq, wq, we, wf, wf + 1, 0, cfg.stride, cfg.pad, 0)
        assert np.array_equal(y, exp)
    else:
        idx = np.random.default_rng(3).integers(0, y.size, 512)
        exp = oracle.conv2d_sample(xq, wq, idx, we, wf, wf + 1, 0, cfg.stride, cfg.pad, 0)
        assert np.array_equal(y.ravel()[idx], exp)


# ----------------------------------------------------------------------------- float32 output epilogue (HOBF_OUT_F32)

def _f32_bits(t):
    return t.contiguous().cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("we,wf,ext", [(5, 3, 0), (4, 3, 0), (5, 10, 0), (6, 7, 0), (5, 3, 1), (6, 10, 1)])
@pytest.mark.parametrize("cout", [64, 40, 33])
def test_f32_epilogue_matches_oracle_decode(we, wf, ext, cout):
    """conv -> exact float32 NHWC in the conv's epilogue (no planes): every float's
    bits equal the oracle's words decoded (decode_f64 -> float32 is exact for
    we <= 7), for the gate kernel, every prepared schedule and the depthwise
    kernel; cout % 4 == 0 (16-byte stores) and ragged (scalar stores)."""
    H = hobf()
    n, h, w, cin = 2, 9, 11, 20
    x, wt = inputs.small_case(900 + cout + wf, n, h, w, cin, cout, "normal", 0.4)
    x[0, 0, :3, 0] = [np.inf, np.nan, -0.0]
    wt[0, 0, 1, :2] = [np.inf, 0.0]
    for rnd in (0, 1):
        f = H.Fmt(we, wf, rnd, extended=ext)
        for relu in (0, 1):
            exp_w = oracle_conv(x, wt, f, relu=relu).reshape(-1, cout)
            exp = oracle.decode_f64(exp_w, we, f.wfo).astype(np.float32).view(np.uint32)
            xp = H.quantize_pack(we, wf, torch.from_numpy(x.reshape(-1, cin)).cuda(), rnd)
            wp = H.quantize_pack(we, wf, torch.from_numpy(wt.reshape(-1, cout)).cuda(), rnd)
            got = _f32_bits(H.conv2d(f, xp, n, h, w, cin, wp, 3, 3, cout, 1, 1, relu, nxt=H.F32))
            assert np.array_equal(got, exp), ("gates", rnd, relu)
            if H.wtab_words(f, 3, 3, cin, cout) > 0:
                tab = H.prepare_weights(f, wp, 3, 3, cin, cout)
                xr = H.quantize_activations(f, torch.from_numpy(x).cuda(), 1)
                for variant in (0, 4, 5, 6, 7, 8, 12):
                    got = _f32_bits(H.conv2d_prepared(f, xr, n, h, w, cin, tab, 3, 3, cout, 1, 1, relu,
                                                      variant=variant, nxt=H.F32))
                    assert np.array_equal(got, exp), ("tables", variant, rnd, relu)
    # depthwise
    xd, wd = inputs.small_case(950 + cout, n, h, w, cout, cout, "normal", 0.5, dw=True)
    f = H.Fmt(we, wf, 0, extended=ext)
    exp_w = oracle.conv2d_dw(oracle.encode_f32(xd, we, wf), oracle.encode_f32(wd, we, wf), we, wf, f.wfo, 0, 2, 1, 1)
    exp = oracle.decode_f64(exp_w.reshape(-1, cout), we, f.wfo).astype(np.float32).view(np.uint32)
    xp = H.quantize_pack(we, wf, torch.from_numpy(xd.reshape(-1, cout)).cuda(), 0)
    wp = H.quantize_pack(we, wf, torch.from_numpy(wd.reshape(-1, cout)).cuda(), 0)
    got = _f32_bits(H.conv2d_dw(f, xp, n, h, w, cout, wp, 3, 3, 2, 1, 1, nxt=H.F32))
    assert np.array_equal(got, exp)


def test_f32_epilogue_rejects_wide_exponent():
    H = hobf()
    z = torch.zeros(1 << 12, dtype=torch.int32, device="cuda")
    with pytest.raises(H.HobfError) as e:
        H.conv2d(H.Fmt(8, 3), z, 1, 4, 4, 4, z, 3, 3, 32, 1, 1, 0, out=torch.zeros(512, device="cuda"), nxt=H.F32)
    assert e.value.status in (1, 3)


def test_quantize_activations_wide_rows():
    """Rows of >= 3072 columns with cin % 4 == 0: the row kernel's transposed records
    would need > 48 KB of shared memory, so the call takes the tile kernel."""
    H = hobf()
    rng = np.random.default_rng(33)
    for (n, h, w, cin) in [(1, 2, 4096, 8), (2, 3, 3071, 4), (1, 1, 5000, 12)]:
        x = rng.standard_normal((n, h, w, cin)).astype(np.float32)
        for pad in (0, 1):
            f = H.Fmt(5, 3, 0)
            rec = to_np_words(H.quantize_activations(f, torch.from_numpy(x).cuda(), pad))
            rec = rec.reshape(n, cin, h + 2 * pad, w + 2 * pad)
            inner = rec[:, :, pad:pad + h, pad:pad + w] & np.uint32((1 << 20) - 1)
            assert np.array_equal(inner.transpose(0, 2, 3, 1), oracle.encode_f32(x, 5, 3, 0))


def test_conv_kernel_info_reports_the_launch():
    """hobf_conv_kernel_info names the kernel the bench's launch runs (symbol, schedule,
    CTA shape, registers, no spills, resident CTAs) without launching anything."""
    H = hobf()
    c3 = inputs.CONFIGS["C3"]
    k = H.conv_kernel_info(H.OP_PREPARED, H.Fmt(5, 3, 0), c3.n, 56, 56, 64, 3, 3, 64, 1, 1, nxt=H.F32)
    assert k["variant"] == 7 and k["threads"] == 128 and "conv_tab_smem_kernel" in k["name"]
    assert k["ctas_per_sm"] == 6 and k["regs"] <= 80 and k["local_bytes"] == 0
    assert k["blocks"] == (c3.n * 56 * 56 + 127) // 128 * 2
    k2 = H.conv_kernel_info(H.OP_PREPARED, H.Fmt(5, 10, 0), 1, 56, 56, 64, 3, 3, 64, 1, 1)
    assert k2["variant"] == 5 and k2["threads"] == 32
    kd = H.conv_kernel_info(H.OP_DW, H.Fmt(5, 3, 0), 2, 14, 14, 512, 3, 3, 512, 2, 1)
    assert "conv_dw_kernel" in kd["name"] and kd["local_bytes"] == 0


@pytest.mark.parametrize("we,wf", SWEEP)
def test_bitsliced_quantisers_every_format(we, wf):
    """The bitsliced float32 encoders (pack_f32_bs_kernel for dense rows,
    quantize_acts_bs_kernel for cin % 32 == 0) on every format of the sweep, both
    rounding modes: values spread over the format's whole range and beyond
    (overflow, underflow, float32 subnormals), exact ties, values one float32 ulp
    either side of a tie, carries into the next binade, and the specials; words
    equal the oracle's encode_f32 and the records' row field is the table row."""
    H = hobf()
    rng = np.random.default_rng(7000 + we * 16 + wf)
    bias = (1 << (we - 1)) - 1
    n = 64 * 1024
    e = rng.integers(-bias - 4, (1 << we) - bias + 3, n)
    frac = rng.integers(0, 1 << 23, n)
    x = np.ldexp(1.0 + frac / 2.0 ** 23, e).astype(np.float32)
    # exact ties and their float32 neighbours: the bit below the kept fraction set, rest zero
    tie = np.ldexp(1.0 + (rng.integers(0, 1 << wf, n // 8) * 2 + 1) / 2.0 ** (wf + 1),
                   rng.integers(-bias, bias, n // 8)).astype(np.float32)
    x[: n // 8] = tie
    x[n // 8: n // 4] = np.nextafter(tie, np.float32(np.inf))
    x[n // 4: 3 * n // 8] = np.nextafter(tie, np.float32(0))
    x[3 * n // 8: n // 2] = -x[3 * n // 8: n // 2]
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-44, 3.4e38, -3.4e38], np.float32)
    x[n // 2: n // 2 + sp.size] = sp
    x = rng.permutation(x)
    for rnd in (0, 1):
        exp = oracle.encode_f32(x, we, wf, rnd)
        planes = H.quantize_pack(we, wf, torch.from_numpy(x.reshape(-1, 64)).cuda(), rnd)
        got = to_np_words(H.unpack(we, wf, planes, n // 64, 64)).ravel()
        assert np.array_equal(got, exp), ("pack", rnd, np.nonzero(got != exp)[0][:5])
        if 3 + we + wf > 20:
            continue  # records hold the word in 20 bits: no prepared path for this format
        f = H.Fmt(we, wf, rnd)
        xa = x.reshape(4, 16, 16, 64)
        rec = to_np_words(H.quantize_activations(f, torch.from_numpy(xa).cuda(), 1)).reshape(4, 64, 18, 18)
        inner = rec[:, :, 1:-1, 1:-1].transpose(0, 2, 3, 1).ravel()
        words = inner & np.uint32((1 << 20) - 1)
        assert np.array_equal(words, exp), ("records", rnd)
        exc = (words >> np.uint32(wf + we + 1)) & np.uint32(3)
        row = np.where(exc == 1, words & np.uint32((1 << wf) - 1), np.uint32(1 << wf) + np.where(exc == 0, 0, exc - 1))
        assert np.array_equal(inner >> np.uint32(20), row.astype(np.uint32))
        assert np.all(rec[:, :, 0, :] == np.uint32((1 << wf) << 20)) and np.all(rec[:, :, :, -1] == np.uint32((1 << wf) << 20))


@pytest.mark.parametrize("we,wfs,exts,rnd", [(5, (3, 3, 3), (0, 0, 0), 0), (5, (10, 3, 7), (0, 1, 0), 1),
                                             (4, (3, 5, 2), (0, 0, 1), 0)])
def test_chain_public_api_vs_oracle(we, wfs, exts, rnd):
    """hobf.Chain: three layers (stride 1, 2, 1; ReLU on the first two) kept in the
    custom format between layers (records epilogue), float32 out of the last;
    equals oracle.conv_chain decoded."""
    H = hobf()
    n, h, w, chans = 2, 13, 11, (24, 40, 33, 48)
    x, _ = inputs.small_case(170 + we, n, h, w, chans[0], chans[1], "normal", 0.5)
    ws = [inputs.small_case(180 + i, 1, 3, 3, chans[i], chans[i + 1], "normal", 0.3)[1] for i in range(3)]
    strides, relus = (1, 2, 1), (1, 1, 0)
    layers = [H.Conv2d(torch.from_numpy(ws[i]).cuda(), H.Fmt(we, wfs[i], rnd, extended=exts[i]), stride=strides[i],
                       pad=1, relu=bool(relus[i])) for i in range(3)]
    y = H.Chain(layers)(torch.from_numpy(x).cuda()).cpu().numpy()
    xq = oracle.encode_f32(x, we, wfs[0], rnd)
    spec = [(oracle.encode_f32(ws[i], we, wfs[i], rnd), wfs[i], strides[i], 1, relus[i], exts[i]) for i in range(3)]
    exp_w = oracle.conv_chain(xq, spec, we, rnd)
    wfo = 2 * wfs[2] + 1 if exts[2] else wfs[2] + 1
    exp = oracle.decode_f64(exp_w, we, wfo).astype(np.float32)
    assert y.shape == exp.shape
    assert np.array_equal(y.view(np.uint32), exp.view(np.uint32))


@pytest.mark.parametrize("we,wf,rnd,relu", [(5, 10, 0, 0), (5, 10, 1, 1), (6, 9, 0, 1), (4, 10, 0, 1)])
def test_fractional_wave_schedule(we, wf, rnd, relu):
    """Variant 12 (C5-like layer with a ragged last tile: 61 images of 14 x 14 -> 94
    tiles x 8 Cout groups = 752 units on 740 resident CTAs): every float32 output
    equals variant 4's (one thread per chain) and the automatic schedule's, and a
    sample -- most of it in the
    units whose chains were handed between CTAs (the last 12) -- equals the
    oracle's chains decoded."""
    H = hobf()
    n, h, w, cin, cout = 61, 14, 14, 32, 256
    x, wt = inputs.small_case(1200 + wf, n, h, w, cin, cout, "uniform4", 0.05)
    f = H.Fmt(we, wf, rnd)
    info = H.conv_kernel_info(H.OP_PREPARED, f, n, h, w, cin, 3, 3, cout, 1, 1, nxt=H.F32, variant=12)
    ctas = info["ctas_per_sm"] * torch.cuda.get_device_properties(0).multi_processor_count
    units = (n * h * w + 127) // 128 * (cout // 32)
    assert ctas < units <= ctas + ctas // 2 and info["variant"] == 12 and info["blocks"] == ctas, (info, units)
    wp = H.quantize_pack(we, wf, torch.from_numpy(wt.reshape(-1, cout)).cuda(), rnd)
    tab = H.prepare_weights(f, wp, 3, 3, cin, cout)
    xr = H.quantize_activations(f, torch.from_numpy(x).cuda(), 1)
    y = {}
    # 13 = the fractional wave at 4 CTAs / SM (592 workers, 160 extra units); 14 = variant 4 with the
    # progress throttle (tokens in the output words while the chains run)
    # 15 = variant 4 with warp-cooperative cp.async table gathers through shared memory
    for v in (0, 4, 12, 13, 14, 15):
        out = torch.full((n * h * w, cout), float("nan"), device="cuda")  # stale contents must not matter
        y[v] = _f32_bits(H.conv2d_prepared(f, xr, n, h, w, cin, tab, 3, 3, cout, 1, 1, relu, out=out,
                                           variant=v, nxt=H.F32))
    assert all(np.array_equal(y[v], y[4]) for v in (0, 12, 13, 14, 15))
    rng = np.random.default_rng(wf)
    npix = n * h * w
    last = (units - 12) // (cout // 32) * 128  # first pixel of the handed-off units (740 resident CTAs)
    pix = np.concatenate([rng.integers(last, npix, 600), rng.integers(0, npix, 200)])
    idx = pix * cout + rng.integers(0, cout, pix.size)
    xq = oracle.encode_f32(x, we, wf, rnd)
    wq = oracle.encode_f32(wt, we, wf, rnd)
    exp_w = oracle.conv2d_sample(xq, wq, idx, we, wf, wf + 1, rnd, relu=relu)
    exp = oracle.decode_f64(exp_w, we, wf + 1).astype(np.float32).view(np.uint32)
    assert np.array_equal(y[0].ravel()[idx], exp)
