"""Multi-GPU partitioning of one conv layer.

Host-side plumbing only: it slices float32 inputs / weights into per-rank
pieces and reassembles per-rank output blocks.  It holds none of the method's
arithmetic (no encoding, no MAC), so the same code serves the CUDA path in
``bench.py`` and the oracle in the world-size-2 tests.

Every output chain acc = add(acc, mul(x, w)) over (c, kh, kw) is independent
(L10), so the layer splits with no exchange step:

* by images when the batch has at least one image per rank (C3, C4, C5);
* then by 32-lane output-channel groups (batch 1: C2 has 2 groups);
* then by output rows: the rank's input slab is the rows its outputs read
  (the halo rows replicated from the neighbours' share) with the zero padding
  written out as +0.0 rows / columns and the slab convolved with pad = 0 --
  the same chains, since a padding tap is a +0 activation (L11, L14) and
  float +0.0 encodes to the canonical +0.

The three factors multiply to the world size.  Splits are as even as the
counts allow (the first ranks take one more image / group / row).
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    n0: int
    n1: int          # images [n0, n1)
    c0: int
    c1: int          # output channels [c0, c1) (multiples of 32 except the last)
    oy0: int
    oy1: int         # output rows [oy0, oy1)
    factors: tuple   # (batch, group, row) split counts
    kind: str        # "batch" | "batch+cout" | "cout" | "cout+rows" | ...

    @property
    def n(self):
        return self.n1 - self.n0

    @property
    def cout(self):
        return self.c1 - self.c0

    @property
    def rows(self):
        return self.oy1 - self.oy0

    def empty(self):
        return self.n <= 0 or self.cout <= 0 or self.rows <= 0


def _even(total: int, parts: int, i: int):
    """[lo, hi) of part i when `total` items are split into `parts` nearly equal parts."""
    q, r = divmod(total, parts)
    lo = i * q + min(i, r)
    return lo, lo + q + (1 if i < r else 0)


def _largest_divisor_at_most(m: int, cap: int) -> int:
    best = 1
    for d in range(1, m + 1):
        if m % d == 0 and d <= cap:
            best = d
    return best


def factors(n: int, cout: int, ho: int, world: int):
    """(batch, group, row) split counts for a layer of n images, cout channels and
    ho output rows on `world` ranks."""
    if world < 1:
        raise ValueError("world must be >= 1")
    groups = (cout + 31) // 32
    if n >= world:
        return world, 1, 1
    b = _largest_divisor_at_most(world, n)
    g = _largest_divisor_at_most(world // b, groups)
    r = world // b // g
    if r > ho:
        raise ValueError(f"cannot split {n} image(s) x {groups} channel group(s) x {ho} rows over {world} ranks")
    return b, g, r


def plan(n: int, cout: int, ho: int, world: int, rank: int) -> Shard:
    b, g, r = factors(n, cout, ho, world)
    ib, rest = divmod(rank, g * r)
    ig, ir = divmod(rest, r)
    n0, n1 = _even(n, b, ib)
    groups = (cout + 31) // 32
    g0, g1 = _even(groups, g, ig)
    oy0, oy1 = _even(ho, r, ir)
    kind = "+".join(k for k, v in (("batch", b), ("cout", g), ("rows", r)) if v > 1) or "none"
    return Shard(rank, world, n0, n1, 32 * g0, min(cout, 32 * g1), oy0, oy1, (b, g, r), kind)


def all_shards(n: int, cout: int, ho: int, world: int):
    return [plan(n, cout, ho, world, r) for r in range(world)]


def slice_inputs(x: np.ndarray, w: np.ndarray, s: Shard, stride: int, pad: int, dw: bool = False):
    """The rank's conv problem: (x_slab, w_slab, pad_slab).

    x: float32 [n, h, w, cin] NHWC; w: [kh, kw, cin, cout] (or [kh, kw, c] for
    depthwise, where the channel split applies to both operands).  Without a row
    split the slab is x[n0:n1] with the layer's own padding; with one, the slab
    is the input rows output rows [oy0, oy1) read, the padding written out as
    zeros, and pad_slab = 0."""
    kh = w.shape[0]
    xs = x[s.n0:s.n1]
    if dw:
        xs = xs[..., s.c0:s.c1]
        ws = w[..., s.c0:s.c1]
    else:
        ws = w[..., s.c0:s.c1]
    if s.factors[2] == 1:
        return np.ascontiguousarray(xs), np.ascontiguousarray(ws), pad
    nimg, h, wd, cin = xs.shape
    iy0 = s.oy0 * stride - pad
    iy1 = (s.oy1 - 1) * stride - pad + kh          # exclusive
    slab = np.zeros((nimg, iy1 - iy0, wd + 2 * pad, cin), dtype=xs.dtype)
    lo, hi = max(iy0, 0), min(iy1, h)
    if hi > lo:
        slab[:, lo - iy0:hi - iy0, pad:pad + wd, :] = xs[:, lo:hi]
    return slab, np.ascontiguousarray(ws), 0


def block_shape(s: Shard, wo: int):
    return (s.n, s.rows, wo, s.cout)


def assemble(blocks, shards, n: int, ho: int, wo: int, cout: int, dtype=np.uint32):
    """Per-rank output blocks [n_r, rows_r, wo, cout_r] -> the layer's [n, ho, wo, cout]."""
    y = np.zeros((n, ho, wo, cout), dtype=dtype)
    covered = np.zeros((n, ho, 1, cout), dtype=np.int32)
    for blk, s in zip(blocks, shards):
        if s.empty():
            continue
        assert blk.shape == block_shape(s, wo), (blk.shape, block_shape(s, wo))
        y[s.n0:s.n1, s.oy0:s.oy1, :, s.c0:s.c1] = blk
        covered[s.n0:s.n1, s.oy0:s.oy1, :, s.c0:s.c1] += 1
    if not (covered == 1).all():
        raise AssertionError("shards do not tile the output exactly once")
    return y


def words_sha256(y: np.ndarray) -> str:
    """sha256 of the output words, C order, little-endian uint32."""
    return hashlib.sha256(np.ascontiguousarray(y, dtype="<u4").tobytes()).hexdigest()


def gather_to_rank0(dist_mod, block: np.ndarray, shards, wo: int, n: int, ho: int, cout: int, rank: int,
                    device=None):
    """Point-to-point gather of every rank's uint32 output block to rank 0 (off the
    clock): rank r > 0 sends its block, rank 0 receives each one into a buffer of
    the shape the plan gives and assembles the layer's output.  Returns the full
    output on rank 0, None elsewhere.  Works with gloo (CPU tensors) and NCCL
    (device tensors: pass `device`)."""
    import torch

    def to_t(a):
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32))
        return t.to(device) if device is not None else t

    if rank != 0:
        if not shards[rank].empty():
            dist_mod.send(to_t(block), dst=0)
        return None
    blocks = []
    for s in shards:
        if s.empty():
            blocks.append(None)
            continue
        if s.rank == 0:
            blocks.append(np.ascontiguousarray(block, dtype=np.uint32))
            continue
        buf = to_t(np.zeros(block_shape(s, wo), np.uint32))
        dist_mod.recv(buf, src=s.rank)
        blocks.append(buf.cpu().numpy().view(np.uint32))
    return assemble(blocks, shards, n, ho, wo, cout)
