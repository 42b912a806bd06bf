"""Host-side checks of the synthetic workload definitions (no GPU): the configs
match BASELINE.json's shapes, the dense / valid-tap MAC counts match their
closed forms, and the seeded draws are deterministic."""
import numpy as np

from paper_2007_06563_b200 import inputs


def test_config_shapes_and_mac_counts():
    c = inputs.CONFIGS
    assert (c["C2"].n, c["C2"].h, c["C2"].cin, c["C2"].cout, c["C2"].formats) == (1, 56, 64, 64, ((5, 10),))
    assert (c["C3"].n, c["C3"].formats) == (32, ((5, 3),))
    assert (c["C4"].n, c["C4"].h, c["C4"].cin, c["C4"].formats) == (256, 28, 128, ((4, 3),))
    assert len(c["C5"].formats) == 27 and (c["C5"].n, c["C5"].h, c["C5"].cin) == (64, 14, 256)
    dense = {"C1": 294912, "C2": 115605504, "C3": 3699376128, "C4": 29595009024, "C5": 7398752256}
    valid = {"C1": 247808, "C2": 112869376, "C3": 3611820032, "C4": 28202500096, "C5": 6710886400}
    for k in dense:
        assert c[k].macs() == dense[k] == c[k].n * c[k].h * c[k].w * c[k].cin * c[k].cout * 9
        assert c[k].valid_macs() == valid[k]
        # padding taps: a 3x3 s1 p1 conv over h x w loses (3h - 2)(3w - 2) of 9hw taps per channel pair
        assert valid[k] == c[k].n * (3 * c[k].h - 2) * (3 * c[k].w - 2) * c[k].cin * c[k].cout
    mob, dw = c["MOB"], c["MOBDW"]
    assert (mob.ho, mob.wo, dw.ho, dw.wo) == (7, 7, 7, 7)
    assert dw.macs() == dw.n * 49 * 512 * 9


def test_draws_are_seeded_and_shaped():
    cfg = inputs.CONFIGS["C3"]
    x1, w1 = inputs.draw(cfg, n=2)
    x2, w2 = inputs.draw(cfg, n=2)
    assert x1.shape == (2, 56, 56, 64) and w1.shape == (3, 3, 64, 64) and x1.dtype == np.float32
    assert np.array_equal(x1, x2) and np.array_equal(w1, w2)
    assert (x1 >= 0).all() and 0.3 < (x1 == 0).mean() < 0.7          # ReLU(N(0,1))
    assert abs(float(w1.std()) - cfg.w_sigma) < 0.1 * cfg.w_sigma     # N(0, sigma), sigma a std (L15)
    xs, ws = inputs.draw(cfg, n=2, shard=1)
    assert not np.array_equal(xs, x1) and np.array_equal(ws, w1)      # weak-scaling shard: own data, same weights
    x5, _ = inputs.draw(inputs.CONFIGS["C5"], n=1)
    assert x5.min() >= 0 and x5.max() < 4                             # 4 * U[0, 1)
    _, wd = inputs.draw(inputs.CONFIGS["MOBDW"], n=1)
    assert wd.shape == (3, 3, 512)
