"""The bench.py contract on CPU: the reference arm (the float64 oracle timed on the host) prints one JSON line
with the keys the driver reads; the GPU arm's pure helpers (algorithmic FLOPs / bytes, vs_baseline)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "pendulum", "--steps", "2",
                        "--warmup", "3"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "cpu_baseline", "e2e", "config"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "frames/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["vs_baseline"] is None  # pendulum: no paper number


def test_class_flops_and_vs_baseline():
    sys.path.insert(0, ROOT)
    import bench
    import synthdata
    # MFLOP per transition (critic + actor GEMMs; TD3 averaged over the policy delay)
    for name, ref in (("pendulum", 0.139), ("walker", 2.282), ("ant", 2.335), ("humanoid", 17.60),
                      ("humanoid_td3", 49.35)):
        w = synthdata.WORKLOADS[name]
        f = bench.class_flops(w, w.batch)
        per_t = sum(v for k, v in f.items() if not k.endswith("_mlp")) / w.batch
        assert abs(per_t / (ref * 1e6) - 1) < 0.02, (name, per_t)
    w = synthdata.WORKLOADS["walker"]
    assert bench.vs_baseline(w, 3.7e5) == 1.0
    assert bench.vs_baseline(synthdata.WORKLOADS["ant"], 1.0) is None


def test_class_flops_f4_variants():
    """SAC v1 drops the s2 actor pass and the target critics and adds the value net (V' and V forward over
    B rows each, V dgrad and wgrad over B rows); DDPG runs the TD3 kernels with no policy delay."""
    sys.path.insert(0, ROOT)
    import dataclasses
    import bench
    import synthdata
    w = synthdata.WORKLOADS["walker"]
    B, o, m, h, L = w.batch, w.obs_dim, w.act_dim, w.hidden, w.n_hidden
    total = lambda f: sum(v for k, v in f.items() if not k.endswith("_mlp"))
    sac = bench.class_flops(w, B)
    v1 = bench.class_flops(dataclasses.replace(w, algo="sacv1"), B)
    mlp = lambda rows, k_in: 2 * rows * (h * k_in + (L - 1) * h * h)
    dropped = mlp(B, o) + 2 * B * 2 * m * h + mlp(2 * B, o + m)  # actor on s2 (+ head), target critics
    added = mlp(2 * B, o) + B * 2 * (L - 1) * h * h + (2 * B * h * o + (L - 1) * 2 * B * h * h + 2 * B * h)
    assert abs(total(v1) - (total(sac) - dropped + added)) < 1e-6 * total(sac)
    assert v1["value_fwd_mlp"] == v1["value_fwd_gemm"] == mlp(2 * B, o)
    td3 = bench.class_flops(dataclasses.replace(w, algo="td3"), B)
    ddpg = bench.class_flops(dataclasses.replace(w, algo="ddpg"), B)
    assert total(ddpg) > total(td3)  # the delayed actor work every step
