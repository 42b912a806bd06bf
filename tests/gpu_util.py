"""Helpers for the -m gpu parity tests (tests only)."""
from __future__ import annotations

import numpy as np
import torch


def hobf():
    from paper_2007_06563_b200 import hobf as H
    return H


def to_dev_words(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint32))
    return torch.from_numpy(a.view(np.int32)).cuda()


def to_np_words(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def words_to_planes(words2d: np.ndarray, we: int, wf: int) -> torch.Tensor:
    H = hobf()
    return H.pack(we, wf, to_dev_words(words2d))


def planes_to_words(planes: torch.Tensor, we: int, wf: int, rows: int, c: int) -> np.ndarray:
    H = hobf()
    return to_np_words(H.unpack(we, wf, planes, rows, c))


def group_planes(words: np.ndarray, we: int, wf: int) -> torch.Tensor:
    """1-D words (len multiple of 32) -> [G, NP] planes (one row of c=len)."""
    H = hobf()
    return H.pack(we, wf, to_dev_words(words.reshape(1, -1))).reshape(-1, H.nplanes(3 + we + wf))


def ungroup_planes(planes: torch.Tensor, we: int, wf: int, n: int) -> np.ndarray:
    H = hobf()
    return to_np_words(H.unpack(we, wf, planes.contiguous(), 1, n)).reshape(-1)
