"""CPU bit-plane simulation helpers for generated circuits (numpy uint64 words).

Word-parallel evaluation is the CPU analogue of the paper's bitslice execution
model (Fig. 4b): one 64-bit word holds one bit of 64 lanes.
"""
from __future__ import annotations

import numpy as np


def to_planes(vals, nbits):
    """vals: uint32 array (N,) -> list of nbits uint64 arrays of ceil(N/64) words."""
    vals = np.asarray(vals, dtype=np.uint32)
    N = vals.size
    pad = (-N) % 64
    v = np.concatenate([vals, np.zeros(pad, np.uint32)]) if pad else vals
    planes = []
    for i in range(nbits):
        bits = ((v >> np.uint32(i)) & np.uint32(1)).astype(np.uint8)
        planes.append(np.packbits(bits, bitorder="little").view(np.uint64))
    return planes


def from_planes(planes, N):
    out = np.zeros(((planes[0].size * 64) if planes else N,), np.uint32)
    for i, p in enumerate(planes):
        bits = np.unpackbits(p.view(np.uint8), bitorder="little").astype(np.uint32)
        out |= bits << np.uint32(i)
    return out[:N]


def input_dict(circuit, arrays):
    """arrays: list of uint32 arrays in circuit.inputs order -> {bitname: plane}."""
    d = {}
    for (name, width), vals in zip(circuit.inputs, arrays):
        for i, p in enumerate(to_planes(vals, width)):
            d[f"{name}[{i}]"] = p
    return d


def run_aig(circuit, arrays):
    N = np.asarray(arrays[0]).size
    outs = circuit.g.simulate(input_dict(circuit, arrays), circuit.outputs, np)
    return from_planes(outs, N)


def run_mapping(circuit, mapping, arrays):
    from .lutmap import simulate_mapping
    N = np.asarray(arrays[0]).size
    outs = simulate_mapping(mapping, input_dict(circuit, arrays), np)
    return from_planes(outs, N)
