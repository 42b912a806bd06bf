"""Full-size bit-exact parity on the BASELINE.json configs (-m gpu).

The north star's target is bit-exact agreement with the oracle on all five
configs.  Here EVERY output word of C1-C4 is compared with the threaded C
oracle (``oracle.conv2d``, one serial chain per output, threads only split
the output pixels), in both rounding modes, through the launch configuration
``bench.py`` times: ``quantize_activations`` (float32 -> records) +
``prepare_weights`` + ``conv2d_prepared`` (schedule chosen automatically for
the full batch) + ``unpack``.  ReLU is checked at full size on C3 (the GPU's
fused ReLU against ``oracle.relu`` of the oracle's chains, ledger L12), and
the full-gate kernel (``hobf_conv2d``) against the same words on C3; the
float32 epilogue the bench times (``HOBF_OUT_F32``) is compared bit for bit with
the oracle's words decoded, on every config.

C5 (27 formats x 7.4e9 MACs) is beyond the oracle's budget, so the GPU runs the
full batch of 64 images (the bench's launch shape) and two whole images --
the first and the last, 2 x 196 x 256 = 100,352 >= 2^16 complete chains --
are compared per format, in both rounding modes.  ("a seeded
sample of >= 2^16 complete output chains per format".)

Cost on a 16-core host: the oracle runs ~0.3e9 MAC/s, so C4 (2.96e10 MACs) is
~100 s per rounding mode; the whole file is a few minutes.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
from gpu_util import hobf, to_np_words
from paper_2007_06563_b200 import inputs

pytestmark = pytest.mark.gpu

CORES = os.cpu_count() or 1


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def gpu_bench_path(x, w, f, cfg, relu=0, n=None, f32=False):
    """The bench's step on the device: records, weight tables, conv, unpack to words
    (f32=True: the conv's float32 epilogue, as bench.py times it)."""
    H = hobf()
    n = x.shape[0] if n is None else n
    xt = torch.from_numpy(x).cuda()
    wp = H.quantize_pack(f.we, f.wf, torch.from_numpy(w.reshape(-1, cfg.cout)).cuda(), f.round)
    tab = H.prepare_weights(f, wp, cfg.kh, cfg.kw, cfg.cin, cfg.cout)
    xr = H.quantize_activations(f, xt, cfg.pad)
    if f32:
        y = H.conv2d_prepared(f, xr, n, cfg.h, cfg.w, cfg.cin, tab, cfg.kh, cfg.kw, cfg.cout, cfg.stride, cfg.pad,
                              relu, nxt=H.F32)
        return y.cpu().numpy().reshape(n, cfg.ho, cfg.wo, cfg.cout)
    yp = H.conv2d_prepared(f, xr, n, cfg.h, cfg.w, cfg.cin, tab, cfg.kh, cfg.kw, cfg.cout, cfg.stride, cfg.pad,
                           relu)
    rows = n * cfg.ho * cfg.wo
    y = to_np_words(H.unpack(f.we, f.wfo, yp, rows, cfg.cout)).reshape(n, cfg.ho, cfg.wo, cfg.cout)
    return y


def oracle_words(x, w, f, cfg, relu=0):
    xq = oracle.encode_f32(x, f.we, f.wf, f.round)
    wq = oracle.encode_f32(w, f.we, f.wf, f.round)
    return oracle.conv2d(xq, wq, f.we, f.wf, f.wfo, f.round, cfg.stride, cfg.pad, relu, nthreads=CORES)


def first_mismatches(got, exp, k=5):
    return [(tuple(int(v) for v in i), hex(int(got[tuple(i)])), hex(int(exp[tuple(i)])))
            for i in np.argwhere(got != exp)[:k]]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
@pytest.mark.parametrize("rnd", [0, 1])
def test_config_every_output(name, rnd):
    H = hobf()
    cfg = inputs.CONFIGS[name]
    x, w = inputs.draw(cfg)
    we, wf = cfg.formats[0]
    f = H.Fmt(we, wf, rnd)
    exp = oracle_words(x, w, f, cfg)
    got = gpu_bench_path(x, w, f, cfg)
    assert got.shape == exp.shape
    assert np.array_equal(got, exp), (name, rnd, int((got != exp).sum()), first_mismatches(got, exp))
    # the bench's own output: the float32 epilogue, every float's bits = the oracle's word decoded
    y32 = gpu_bench_path(x, w, f, cfg, f32=True)
    dec = oracle.decode_f64(exp, we, f.wfo).astype(np.float32)
    assert np.array_equal(y32.view(np.uint32), dec.view(np.uint32))
    if name == "C3":
        # fused ReLU at full size vs the oracle's ReLU of the same chains (L12)
        got_r = gpu_bench_path(x, w, f, cfg, relu=1)
        exp_r = oracle.relu(exp, we, f.wfo)
        assert np.array_equal(got_r, exp_r), first_mismatches(got_r, exp_r)
        # the paper-faithful full-gate MAC kernel gives the same words
        xp = H.quantize_pack(we, wf, torch.from_numpy(x.reshape(-1, cfg.cin)).cuda(), rnd)
        wp = H.quantize_pack(we, wf, torch.from_numpy(w.reshape(-1, cfg.cout)).cuda(), rnd)
        yp = H.conv2d(f, xp, cfg.n, cfg.h, cfg.w, cfg.cin, wp, cfg.kh, cfg.kw, cfg.cout, cfg.stride, cfg.pad, 0)
        got_g = to_np_words(H.unpack(we, f.wfo, yp, cfg.n * cfg.ho * cfg.wo, cfg.cout)).reshape(exp.shape)
        assert np.array_equal(got_g, exp), first_mismatches(got_g, exp)


@pytest.mark.parametrize("we,wf", list(inputs.SWEEP))
def test_C5_whole_images_every_format(we, wf):
    """Full batch on the GPU (bench launch shape); images 0 and 63 compared in full."""
    H = hobf()
    cfg = inputs.CONFIGS["C5"]
    x, w = _c5_inputs()
    for rnd, imgs in ((0, (0, cfg.n - 1)), (1, (0, cfg.n - 1))):
        f = H.Fmt(we, wf, rnd)
        got = gpu_bench_path(x, w, f, cfg)
        # the float32 epilogue the bench times (for wF = 10 and e6m9 the fractional-wave
        # schedule, variant 12: the last image's chains are handed between CTAs)
        y32 = gpu_bench_path(x, w, f, cfg, f32=True)
        for i in imgs:
            exp = oracle_words(x[i:i + 1], w, f, cfg)[0]
            assert np.array_equal(got[i], exp), ((we, wf, rnd, i), first_mismatches(got[i], exp))
            dec = oracle.decode_f64(exp, we, f.wfo).astype(np.float32)
            assert np.array_equal(y32[i].view(np.uint32), dec.view(np.uint32)), ("f32", we, wf, rnd, i)


_C5 = {}


def _c5_inputs():
    if not _C5:
        _C5["xw"] = inputs.draw(inputs.CONFIGS["C5"])
    return _C5["xw"]
