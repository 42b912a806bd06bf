"""The GPU proof program of tools/sweep_gpu.py (which proves the wider SDC sweeps by
running the original and the swept LOP3 networks on every valid input) tells a
correct sweep from a wrong one: a CPU-proved sweep prints 0 differing words, the
same sweep with one output LUT's table corrupted does not."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.mark.gpu
@pytest.mark.parametrize("mutate", [False, True])
def test_sweep_proof_program(mutate, tmp_path):
    import sweep_gpu
    from paper_2007_06563_b200.gen import fpgen, sweep
    sweep_gpu.OUT = str(tmp_path)
    we, wf, rnd = 4, 3, 0
    c = fpgen.build_mac_tab(we, wf, rnd)
    new = sweep.reduce("mac_tab", c, we, wf, rnd, wf + 1)
    name = "prove_e4m3" + ("_mutant" if mutate else "")
    sweep_gpu.write_program(name, c, new, we, wf, rnd, mutate=mutate)
    out = subprocess.run([os.path.join(str(tmp_path), name)], capture_output=True, text=True, timeout=300).stdout
    f = out.split()
    assert f[0] == name and f[1] == "differing_words" and f[-1] == "ok", out
    assert (int(f[2]) > 0) == mutate, out
