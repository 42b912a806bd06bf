"""Host-side partitioning of one conv layer over N ranks (no GPU).

paper_2007_06563_b200/shard.py splits the config's global layer by images, then
32-lane output-channel groups, then output rows; these tests check that every
plan tiles the output exactly once and that the per-rank slices, convolved by
the ORACLE and reassembled, give the N = 1 words -- for the BASELINE configs'
splits at N = 1/2/4/8 (shapes only) and for small layers (full values)."""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_2007_06563_b200 import inputs, shard


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5", "MOB", "MOBDW"])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_plans_tile_the_output_exactly_once(name, world):
    cfg = inputs.CONFIGS[name]
    shards = shard.all_shards(cfg.n, cfg.cout, cfg.ho, world)
    blocks = [np.full(shard.block_shape(s, cfg.wo), s.rank, np.uint32) for s in shards]
    y = shard.assemble(blocks, shards, cfg.n, cfg.ho, cfg.wo, cfg.cout)
    for s in shards:
        assert not s.empty()
        assert (y[s.n0:s.n1, s.oy0:s.oy1, :, s.c0:s.c1] == s.rank).all()
        assert s.c0 % 32 == 0          # channel splits fall on 32-lane group boundaries
    b, g, r = shards[0].factors
    assert b * g * r == world
    # the split the north star names: batch for C3/C4/C5, channel groups for C2
    if name in ("C3", "C4", "C5", "MOB", "MOBDW"):
        assert (b, g, r) == (world, 1, 1)
        assert [s.n for s in shards] == [cfg.n // world] * world if cfg.n % world == 0 else True
    if name == "C2" and world == 2:
        assert (b, g, r) == (1, 2, 1)
    if name == "C4" and world == 8:
        assert all(s.n == 32 for s in shards)


def test_assemble_detects_overlap():
    shards = shard.all_shards(2, 32, 4, 2)
    bad = [dataclasses.replace(s, n0=0, n1=2) for s in shards]
    with pytest.raises(AssertionError):
        shard.assemble([np.zeros((2, 4, 3, 32), np.uint32)] * 2, bad, 2, 4, 3, 32)


@pytest.mark.parametrize("n,h,w,cin,cout,stride,world", [
    (3, 5, 6, 7, 40, 1, 2),      # batch split, uneven (2 + 1 images)
    (1, 6, 5, 6, 64, 1, 2),      # channel groups
    (1, 7, 5, 4, 64, 1, 4),      # channel groups x rows
    (1, 9, 6, 5, 32, 2, 4),      # rows only, stride 2 (halo rows overlap)
    (2, 5, 5, 3, 96, 1, 8),      # images x groups x rows
    (1, 3, 4, 3, 33, 1, 3),      # rows, 3 ranks (uneven rows), ragged channel group
])
def test_slices_reassemble_to_the_n1_conv(n, h, w, cin, cout, stride, world):
    cfg = inputs.ConvConfig("t", n, h, w, cin, cout, ((5, 3),), "normal", 0.5, stride=stride)
    x, wt = inputs.draw(cfg, seed=n * 100 + world)
    x[0, 0, 0, 0] = np.inf      # specials cross the row boundaries too
    ref = oracle.conv2d(oracle.encode_f32(x, 5, 3), oracle.encode_f32(wt, 5, 3), 5, 3, 4, 0, stride, 1, 1)
    shards = shard.all_shards(n, cout, cfg.ho, world)
    blocks = []
    for s in shards:
        xs, ws, pad = shard.slice_inputs(x, wt, s, stride, 1)
        blocks.append(oracle.conv2d(oracle.encode_f32(xs, 5, 3), oracle.encode_f32(ws, 5, 3), 5, 3, 4, 0, stride,
                                    pad, 1))
    y = shard.assemble(blocks, shards, n, cfg.ho, cfg.wo, cout)
    assert np.array_equal(y, ref)
    assert shard.words_sha256(y) == shard.words_sha256(ref)
    macs = sum(b.shape[0] * b.shape[1] * b.shape[2] * b.shape[3] * cin * 9 for b in blocks)
    assert macs == cfg.macs()          # dense MACs are conserved (padding written out as +0 taps)


def test_depthwise_slices_reassemble():
    cfg = inputs.ConvConfig("d", 1, 9, 7, 64, 64, ((5, 3),), "normal", 0.5, stride=2, dw=True)
    x, wt = inputs.draw(cfg, seed=5)
    ref = oracle.conv2d_dw(oracle.encode_f32(x, 5, 3), oracle.encode_f32(wt, 5, 3), 5, 3, 4, 0, 2, 1, 0)
    for world in (2, 4):
        shards = shard.all_shards(1, 64, cfg.ho, world)
        blocks = []
        for s in shards:
            xs, ws, pad = shard.slice_inputs(x, wt, s, 2, 1, dw=True)
            blocks.append(oracle.conv2d_dw(oracle.encode_f32(xs, 5, 3), oracle.encode_f32(ws, 5, 3), 5, 3, 4, 0, 2,
                                           pad, 0))
        assert np.array_equal(shard.assemble(blocks, shards, 1, cfg.ho, cfg.wo, 64), ref)


def test_too_many_ranks_is_an_error():
    with pytest.raises(ValueError):
        shard.factors(1, 32, 2, 4)
