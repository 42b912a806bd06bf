"""Multi-process (N>1) host logic on CPU with the gloo backend, world_size 2.

The hot path shards with no collective: the config's one
global input is split by images, then 32-lane output-channel groups, then output
rows (paper_2007_06563_b200/shard.py); what runs across ranks is the plumbing:
rendezvous, barrier, max-over-ranks timing, the per-rank slices, the gather of
the output words to rank 0 and their hash, and the reference arm printing on
rank 0 only.  The per-rank conv here is the oracle (no GPU on this host): the
test proves that the slices reassemble to the N = 1 result word for word."""
import json
import os
import socket
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def torchrun(args, nproc=2, timeout=600, env_extra=None):
    env = dict(os.environ)
    env["PYTHONPATH"] = ROOT + os.pathsep + env.get("PYTHONPATH", "")
    env["CUDA_VISIBLE_DEVICES"] = ""
    if env_extra:
        env.update(env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port())] + args
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


def test_dist_plumbing_gloo_world2(tmp_path):
    script = tmp_path / "w2.py"
    script.write_text(textwrap.dedent("""
        import json, os, sys
        import numpy as np
        sys.path.insert(0, os.environ["ROOT"])
        import bench
        from paper_2007_06563_b200 import inputs
        d = bench.Dist()
        d.init("gloo")
        assert d.world == 2
        d.barrier()
        # max over ranks
        m = d.max(float(d.rank + 1) * 1.5)
        cfg = inputs.CONFIGS["C1"]
        x, w = inputs.draw(cfg, shard=d.rank)
        x0, w0 = inputs.draw(cfg)
        out = {"rank": d.rank, "max": m, "x_sum": float(x.astype(np.float64).sum()),
               "same_w": bool((w == w0).all()), "x_is_cfg": bool((x == x0).all())}
        with open(os.path.join(os.environ["OUT"], f"r{d.rank}.json"), "w") as f:
            json.dump(out, f)
        d.barrier()
        d.done()
    """))
    r = torchrun([str(script)], env_extra={"ROOT": ROOT, "OUT": str(tmp_path)})
    assert r.returncode == 0, r.stderr[-3000:]
    res = [json.load(open(tmp_path / f"r{i}.json")) for i in range(2)]
    assert all(o["max"] == 3.0 for o in res)                 # max over ranks
    assert all(o["same_w"] for o in res)                      # weights replicated
    assert res[0]["x_is_cfg"] and not res[1]["x_is_cfg"]      # rank 0 = the config's own batch
    assert res[0]["x_sum"] != res[1]["x_sum"]                 # distinct shards (weak scaling)


def test_strong_split_gather_reassembles_n1_gloo_world2(tmp_path):
    """Each of 2 ranks takes its shard of the global layer (bench.Problem: images for
    a batch, rows for C1's single image and single channel group, channel groups for
    a 2-group batch-1 layer), runs the ORACLE conv on it, and the words are gathered
    to rank 0 over gloo: the assembled output and its sha256 equal the N = 1 conv."""
    script = tmp_path / "split.py"
    script.write_text(textwrap.dedent("""
        import dataclasses, json, os, sys
        import numpy as np
        sys.path.insert(0, os.environ["ROOT"])
        import bench, oracle
        from paper_2007_06563_b200 import inputs, shard
        d = bench.Dist()
        d.init("gloo")
        cases = {
            "C1": inputs.CONFIGS["C1"],
            "batch3": dataclasses.replace(inputs.CONFIGS["C1"], name="batch3", n=3, h=5, w=6, cin=7, cout=40),
            "groups2": dataclasses.replace(inputs.CONFIGS["C1"], name="groups2", n=1, h=6, w=5, cin=6, cout=64),
            "dw_s2": dataclasses.replace(inputs.CONFIGS["MOBDW"], name="dw_s2", n=1, h=9, w=7, cin=40, cout=40),
        }
        out = {}
        for name, cfg in cases.items():
            P = bench.Problem(cfg, d, weak=False)
            we, wf = 5, 3
            xq, wq = oracle.encode_f32(P.x, we, wf, 0), oracle.encode_f32(P.w, we, wf, 0)
            conv = oracle.conv2d_dw if cfg.dw else oracle.conv2d
            y = conv(xq, wq, we, wf, wf + 1, 0, cfg.stride, P.pad, 1, nthreads=2)
            shards = shard.all_shards(cfg.n, cfg.cout, cfg.ho, d.world)
            full = shard.gather_to_rank0(d.pg, y, shards, cfg.wo, cfg.n, cfg.ho, cfg.cout, d.rank)
            if d.rank == 0:
                xg, wg = inputs.draw(cfg)
                ref = conv(oracle.encode_f32(xg, we, wf, 0), oracle.encode_f32(wg, we, wf, 0), we, wf, wf + 1, 0,
                           cfg.stride, cfg.pad, 1, nthreads=2)
                out[name] = {"equal": bool(np.array_equal(full, ref)), "kind": P.shard.kind,
                             "sha": shard.words_sha256(full), "sha_n1": shard.words_sha256(ref),
                             "macs": P.macs()}
            else:
                out[name] = {"kind": P.shard.kind, "macs": P.macs()}
            out[name]["macs_total"] = d.sum(P.macs())
        with open(os.path.join(os.environ["OUT"], f"s{d.rank}.json"), "w") as f:
            json.dump(out, f)
        d.barrier()
        d.done()
    """))
    r = torchrun([str(script)], env_extra={"ROOT": ROOT, "OUT": str(tmp_path)})
    assert r.returncode == 0, r.stderr[-3000:]
    r0 = json.load(open(tmp_path / "s0.json"))
    r1 = json.load(open(tmp_path / "s1.json"))
    from paper_2007_06563_b200 import inputs
    import dataclasses
    for name, o in r0.items():
        assert o["equal"], name
        assert o["sha"] == o["sha_n1"], name
    assert r0["C1"]["kind"] == "rows" and r0["batch3"]["kind"] == "batch" and r0["groups2"]["kind"] == "cout"
    assert r0["dw_s2"]["kind"] == "cout"
    assert r0["C1"]["macs_total"] == inputs.CONFIGS["C1"].macs()   # dense MACs are conserved by the split
    assert r0["batch3"]["macs"] + r1["batch3"]["macs"] == r0["batch3"]["macs_total"]


def test_reference_arm_under_torchrun_rank0_only():
    r = torchrun(["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                  "--config", "C1"])
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                                     # only rank 0 prints
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["n_gpus"] == 2 and j["value"] > 0
    assert j["cpu_baseline"]["kind"] == "oracle" and j["e2e"]["h2d_bytes_per_step"] == 0


def test_shard_inputs_are_deterministic():
    from paper_2007_06563_b200 import inputs
    cfg = inputs.CONFIGS["C5"]
    a = inputs.draw(cfg, n=2, shard=3)[0]
    b = inputs.draw(cfg, n=2, shard=3)[0]
    assert (a == b).all()
    c = inputs.draw(cfg, n=2, shard=4)[0]
    assert not (a == c).all()
