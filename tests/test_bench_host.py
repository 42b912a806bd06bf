"""Host-side logic of bench.py (no GPU): the roofline traffic lookup is keyed by
the exact (config, format, rounding, MAC class, kernel) its ncu capture measured."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_measured_traffic_keying():
    with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
        t = json.load(f)
    assert bench.measured_traffic("C3", 5, 3, True) == t["C3/e5m3/conv2d_prepared"]
    # a capture of the RNE single-class table kernel says nothing about other runs
    assert bench.measured_traffic("C3", 5, 3, True, rtz=True) is None
    assert bench.measured_traffic("C3", 5, 3, True, extended=True) is None
    assert bench.measured_traffic("C3", 5, 3, False) is None
    assert bench.measured_traffic("C4", 4, 3, True) == t.get("C4/e4m3/conv2d_prepared")
