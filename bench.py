"""Benchmark: SAC/TD3 update frames/s on B200 (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config walker] [--precision bf16]
    python bench.py --gpus 2 --dry-run        # the multi-GPU plan under gloo (no GPU needed)
    python bench.py --impl reference ...      # the float64 CPU oracle arm (host cores)

A "step" is one full update over one batch of B transitions sampled from a
device-resident ring filled with synthetic transitions (synthdata).  --gpus N > 1 without torchrun
re-launches itself under torch.distributed.run (one process per GPU); the world size must equal N.

Timing: W warm-up updates, then repetitions of EXACTLY K graph-replayed updates
(one spz_update(B, K) each), each bracketed by a barrier + synchronize and timed with CUDA events
on the learner's stream, max over ranks; repeated until at least --reps repetitions and
--min-time seconds of timed work.  value = frames per repetition / median repetition time
[frames/s = update frequency x B, P:465].  Modes for N > 1: dp = one row-sharded learner group
(NCCL gradient allreduce inside the step), split = actor/critic groups, replicas = N
independent learners; --scaling weak keeps B per GPU (global B x N), strong keeps the global B.

Extra keys: roofline (the dominant tensor-core kernel class vs the measured bf16 peak, plus the HBM
fractions of the gather and Adam + Polyak; per-class times from spz_learner_profile: gated, no host
gaps), fp32 (the same measurement in FP32 / 3xTF32 precision), cpu_baseline + parity (rank 0, one
GPU: K_o oracle updates from the same parameters, ring and seeds -- timed on the host cores -- and
the same K_o GPU updates checked against them, tests/parity.py), e2e (through the C ABI with host
buffers: each step pushes B fresh transitions from pinned host memory and reads the stats back),
clocks (nvidia-smi during the timed region), gpu_launches (our kernels in the timed region).
"""

import argparse
import dataclasses
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthdata  # noqa: E402

METRIC = "SAC update frames/s (transitions consumed) at 1/2/4/8 B200; % of GEMM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--config", default="walker", choices=list(synthdata.WORKLOADS))
    ap.add_argument("--precision", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--algo", default=None, choices=["sac", "td3", "ddpg", "sacv1"],
                    help="override the workload's algorithm (SURVEY.md §8(f) f4 variants on the same shapes)")
    ap.add_argument("--impl", default="spz", choices=["spz", "reference"])
    ap.add_argument("--batch", type=int, default=None, help="override the workload batch (B sweep)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sweep", action="store_true",
                    help="also run the batch-size adaptation (spz_tune_batch, §8(f) f3) over the §8(d) B ladder")
    ap.add_argument("--cpu-sample-steps", type=int, default=None)
    ap.add_argument("--mode", default="dp", choices=["dp", "split", "replicas"],
                    help="N > 1: dp = one row-sharded learner group (global batch B*N, NCCL gradient allreduce); "
                         "split = actor/critic model parallelism (critic group ranks [0, N*c), actor group the rest; "
                         "each group row-shards the global batch B*N/2); replicas = N independent learners")
    ap.add_argument("--critic-frac", type=float, default=0.5,
                    help="split mode: fraction of the ranks in the critic group (SAC critic:actor work ~1.7:1)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = B rows per GPU (global B x N); strong = the global batch B sharded over the group")
    ap.add_argument("--reps", type=int, default=5, help="minimum number of timed repetitions of K steps")
    ap.add_argument("--min-time", type=float, default=2.0, help="minimum seconds of timed work over all repetitions")
    ap.add_argument("--no-fp32", action="store_true", help="skip the FP32 (3xTF32) measurement key")
    ap.add_argument("--parity-steps", type=int, default=None, help="K_o (default: SURVEY.md §8(d) per config)")
    ap.add_argument("--dry-run", action="store_true", help="print the multi-GPU plan of every rank (gloo, no GPU)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the short device-resident measurement of the other BASELINE configs (the `configs` key)")
    return ap.parse_args()


# oracle updates K_o run beside the GPU in the same invocation (and checked)
PARITY_STEPS = {"pendulum": 200, "walker": 20, "ant": 5, "humanoid": 3, "humanoid_td3": 2}


def spawn_if_needed(a):
    """--gpus N > 1 outside torchrun: re-launch this command under torch.distributed.run, one rank per GPU."""
    if a.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def group_batch(mode, scaling, B, world):
    """Global batch one learner group consumes per update."""
    if world == 1 or mode == "replicas":
        return B
    if scaling == "strong":
        return B
    return B * world if mode == "dp" else B * world // 2


def split_critics(world, frac):
    return min(world - 1, max(1, int(round(world * frac))))


def dry_run(a, w, B):
    """The host-side plan (spz_plan_rank) of every rank under gloo: shard ranges, groups, exchange roots."""
    import torch.distributed as dist
    from paper_2312_06126_b200 import spz
    from paper_2312_06126_b200.dist import env_rank
    rank, world, _ = env_rank()
    if world > 1:
        dist.init_process_group("gloo")
    GB = group_batch(a.mode, a.scaling, B, world)
    kw = {}
    if a.mode == "split" and world > 1:
        nc = split_critics(world, a.critic_frac)
        kw = dict(role=spz.SPZ_ROLE_CRITIC if rank < nc else spz.SPZ_ROLE_ACTOR, n_critic_ranks=nc)
    if a.mode == "replicas":
        plan = spz.spz_plan_rank(GB, 1, 0)
    else:
        plan = spz.spz_plan_rank(GB, world, rank, **kw)
    plans = [None] * world
    if world > 1:
        dist.all_gather_object(plans, plan)
    else:
        plans = [plan]
    if rank == 0:
        groups = {}
        for p in plans:
            groups.setdefault(p["group_color"], []).append((p["row0"], p["rows"]))
        tiled = all(sorted(g)[0][0] == 0 and sum(n for _, n in g) == GB and
                    all(x[0] + x[1] == y[0] for x, y in zip(sorted(g), sorted(g)[1:])) for g in groups.values())
        if a.mode == "replicas":
            tiled = True
        print(json.dumps({"dry_run": True, "n_gpus": world, "mode": a.mode, "scaling": a.scaling,
                          "config": {"workload": w.name, "global_batch": GB * (world if a.mode == "replicas" else 1)},
                          "plans": plans, "partitions_tile_batch": tiled}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sust=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    src="measured")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sust=1400.0, src="fallback")


# ----------------------------------------------------------------------------- algorithmic work per kernel class

def class_flops(w, B):
    """Algorithmic GEMM FLOPs (2 * M * N * K over the true, unpadded dims) per step, by kernel class.

    SAC: actor on [s2; s], twin critics on every row kind.  TD3 (averaged over the policy delay): the
    target actor on s2 every step, the online actor and the actor rows of Q1 (its only critic for the
    actor loss) on delayed steps only (reading #18)."""
    o, m, h, L = w.obs_dim, w.act_dim, w.hidden, w.n_hidden
    td3 = w.algo in ("td3", "ddpg")  # DDPG: the TD3 kernels, twin tied to the first, no delay
    v1 = w.algo == "sacv1"           # SAC v1: actor on s only, V'(s2) + V(s) instead of the target critics
    dly = 1.0 / 2 if w.algo == "td3" else 1.0  # share of steps with actor work (TD3 policy delay 2)
    aout = m if td3 else 2 * m
    cin = o + m
    f = {}
    add = lambda k, v: f.__setitem__(k, f.get(k, 0) + v)
    mlp = lambda rows, k_in, out: 2 * rows * (h * k_in + (L - 1) * h * h + (h * out if out else 0))
    # actor forward: SAC [s2; s] every step; TD3 target actor on s2 + online actor on s when delayed
    Ma = (B if v1 else 2 * B) if not td3 else B * (1 + dly)
    add("actor_fwd_gemm", mlp(Ma, o, 0))
    add("actor_head_gemm", 2 * Ma * aout * h)
    # critics: targets (2 nets x B rows) and online loss rows (2 x B) every step; actor rows: both
    # critics (SAC) / Q1 on delayed steps (TD3)
    crit_rows = (0 if v1 else 2 * B) + 2 * B + (2 * B if not td3 else B * dly)
    add("critic_fwd_gemm", mlp(crit_rows, cin, 0))
    dgrad_rows = 2 * B + (2 * B if not td3 else B * dly)
    add("critic_dgrad_gemm", dgrad_rows * 2 * (L - 1) * h * h)
    if v1:  # value net: V' and V forward (B rows each), dgrad and wgrad over the B s rows
        add("value_fwd_gemm", mlp(2 * B, o, 0))
        add("critic_dgrad_gemm", B * 2 * (L - 1) * h * h)
        add("wgrad_gemm", 2 * B * h * o + (L - 1) * 2 * B * h * h + 2 * B * h)
    add("critic_input_dgrad_gemm", (2 * B if not td3 else B * dly) * 2 * h * m)
    add("wgrad_gemm", 2 * (2 * B * h * cin + (L - 1) * 2 * B * h * h))  # critics ...
    add("actor_dgrad_gemm", dly * (2 * B * aout * h + (L - 1) * 2 * B * h * h))
    add("wgrad_gemm", dly * (2 * B * h * o + (L - 1) * 2 * B * h * h + 2 * B * aout * h))  # ... and the actor
    add("wgrad_gemm", 2 * 2 * B * h)  # critic-head weight gradients (g_q as a one-row operand)
    # fused multi-layer forwards (h <= 256): every hidden layer (+ the actor head) in one launch
    f["actor_fwd_mlp"] = f["actor_fwd_gemm"] + f["actor_head_gemm"]
    f["critic_fwd_mlp"] = f["critic_fwd_gemm"]
    if v1:
        f["value_fwd_mlp"] = f["value_fwd_gemm"]
    return f


def class_bytes(w, B, n_actor, n_critic):
    """Algorithmic HBM bytes per step of the memory-bound classes.

    gather: the sampled records (R fp32 per row) + one 4-byte index per row.
    adam_polyak: per trained parameter read p, m, v, g and write p, m, v (28 B); per critic parameter
    the Polyak target read + write (8 B).  TD3 (policy delay 2): the actor's Adam and every Polyak
    only on delayed steps (averaged).  n_critic counts both critics (SAC v1: + V)."""
    R = (2 * w.obs_dim + w.act_dim + 2 + 3) // 4 * 4
    dly = 0.5 if w.algo == "td3" else 1.0
    td3 = w.algo in ("td3", "ddpg")
    adam = 28 * n_critic + dly * 28 * n_actor + dly * 8 * n_critic + (dly * 8 * n_actor if td3 else 0)
    return {"gather": B * (4 * R + 4), "adam_polyak": adam}


# the paper's network-update frame rate for Walker2D SAC at its default batch (~8192):
# 3.7E+5 Hz -- on a GTX 1060, network size unstated: context, not the target
PAPER_WALKER_HZ = 3.7e5


def vs_baseline(w, value):
    return value / PAPER_WALKER_HZ if w.name == "walker" else None


TRAFFIC_FILES = ("r02_traffic.json", "r01_traffic.json")  # newest first


def traffic(workload, kernel):
    """(DRAM bytes read + written per launch of kernel class `kernel`, source) from the committed
    ncu --set full capture, or (None, None)."""
    for f in TRAFFIC_FILES:
        p = os.path.join(ROOT, "profiles", f)
        try:
            e = json.load(open(p))[workload][kernel]
        except (OSError, KeyError, ValueError):
            continue
        return e["dram_read"] + e["dram_write"], f"profiles/{f} (ncu --set full, per launch)"
    return None, None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ----------------------------------------------------------------------------- clocks sampler

class Clocks:
    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- oracle (CPU baseline / reference arm)

def oracle_rate(w, B, steps):
    """Time `steps` float64 oracle updates of the workload on this host; returns (frames/s, cores, seconds)."""
    from oracle import ddpg as oddpg, ring as oring, sac as osac, sacv1 as osacv1, td3 as otd3
    cores = len(os.sched_getaffinity(0))
    n = min(w.capacity, 1_000_000)
    tr = synthdata.workload_transitions(w, n=n)
    r = oring.Ring(w.obs_dim, w.act_dim, n)
    r.push(**tr)
    p = synthdata.init_params(w.obs_dim, w.act_dim, w.hidden, w.n_hidden, algo=w.algo)
    cfg = osac.Config(obs_dim=w.obs_dim, act_dim=w.act_dim, hidden=w.hidden, n_hidden=w.n_hidden,
                      alpha_auto=w.algo == "sac")
    if w.algo == "sacv1":
        cfg.alpha_auto = False
        st = osacv1.State.create(p["actor"], p["q1"], p["q2"], p["v"], log_alpha=np.log(0.2))
    else:
        st = osac.State.create(p["actor"], p["q1"], p["q2"], log_alpha=np.log(0.2),
                               actor_targ=p["actor"] if w.algo in ("td3", "ddpg") else None)
    if w.algo == "ddpg":
        cfg.td3_policy_delay, cfg.td3_noise, cfg.td3_noise_clip = 1, 0.0, 0.0
    step = {"sac": osac.sac_step, "td3": otd3.td3_step, "ddpg": oddpg.ddpg_step, "sacv1": osacv1.sacv1_step}[w.algo]
    t0 = time.perf_counter()
    for _ in range(steps):
        st, _, _ = step(st, r, B, synthdata.SAMPLE_SEED, cfg)
    dt = time.perf_counter() - t0
    return B * steps / dt, cores, dt


def reference_arm(a, w, B):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps = a.steps
    # each reference step = one full float64 oracle update at the workload's batch; keep the run to minutes
    probe_rate, cores, probe_t = oracle_rate(w, B, 1)
    per_step = probe_t
    budget_s = 240.0
    steps = max(1, min(steps, int(budget_s / max(per_step, 1e-3))))
    warm = 0 if per_step > 5 else min(a.warmup, 3)
    if warm:
        oracle_rate(w, B, warm)
    rate, cores, dt = oracle_rate(w, B, steps)
    line = {"metric": METRIC, "value": rate, "unit": "frames/s", "impl": "reference", "n_gpus": a.gpus,
            "steps": steps, "warmup": warm, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": vs_baseline(w, rate), "dtype": "f64", "data": "synthetic",
            "config": {"workload": w.name, "global_batch": B, "algo": w.algo, "hidden": f"{w.n_hidden}x{w.hidden}",
                       "obs_dim": w.obs_dim, "act_dim": w.act_dim, "ring": min(w.capacity, 1_000_000)},
            "cpu_baseline": {"value": rate, "unit": "frames/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"{steps} full float64 oracle updates at B={B} ({w.name})"},
            "e2e": {"value": rate, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def timed_reps(lrn, GB, K, a, stream, world, dist, torch):
    """Repetitions of exactly K updates (one spz_update(GB, K) each), CUDA events on the learner's stream,
    barrier + synchronize on both sides, max over ranks; at least a.reps repetitions and a.min_time s."""
    reps, total = [], 0.0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = None
    while len(reps) < a.reps or total < a.min_time:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        stats = lrn.update(GB, K)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        reps.append(ms)
        total += ms / 1e3
        if len(reps) >= 20000:
            break
    return reps, stats


def roofline(w, B, prof, precision, pk, n_actor, n_critic):
    """Dominant tensor-core class (bench-timed, gated per-class CUDA events) against the measured peak, and
    the HBM fractions of the gather and the optimizer against their algorithmic bytes (§8(d))."""
    fl = class_flops(w, B)
    by = class_bytes(w, B, n_actor, n_critic)
    tens = {k: t for k, t in prof.items() if k in fl}
    dom = max(tens, key=tens.get)
    ach = fl[dom] / (prof[dom] * 1e-3) / 1e12
    if precision == "bf16":
        pkv, src = pk["bf16_sust"], f"{pk['src']} bf16 sustained (MEASURED_PEAKS.json)"
    else:  # 3xTF32: three tf32 MMAs per product; tf32 peak = bf16 x 1/2 (the guide's nominal ratio)
        pkv, src = pk["bf16_sust"] / 2.0 / 3.0, f"{pk['src']} bf16 sustained x 1/2 (tf32 nominal) / 3 (3xTF32 MMAs per product)"
    tr, tr_src = traffic(w.name, dom) if precision == "bf16" else (None, None)
    roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": pkv, "unit": "TFLOP/s", "frac": ach / pkv,
            "traffic": tr, "traffic_src": tr_src, "peak_src": src, "algorithmic_flop_per_launch": fl[dom],
            "launch_ms": prof[dom],
            "timing": "spz_learner_profile: each step queued whole behind a gate, CUDA events around every op (no host gaps, no PDL overlap)"}
    hbm = {}
    for k in ("gather", "adam_polyak"):
        if k in prof:
            gbs = by[k] / (prof[k] * 1e-3) / 1e9
            hbm[k] = {"achieved": gbs, "peak": pk["hbm"], "unit": "GB/s", "frac": gbs / pk["hbm"],
                      "algorithmic_bytes_per_launch": by[k], "launch_ms": prof[k]}
    roof["hbm"] = hbm
    gemm_f = sum(v for k, v in fl.items() if not k.endswith("_mlp"))
    return roof, gemm_f


def main():
    a = parse()
    spawn_if_needed(a)
    w = synthdata.WORKLOADS[a.config]
    if a.algo and a.algo != w.algo:
        w = dataclasses.replace(w, name=f"{w.name}_{a.algo}", algo=a.algo)
    B = a.batch or w.batch
    if a.impl == "reference":
        reference_arm(a, w, B)
        return
    if a.dry_run:
        dry_run(a, w, B)
        return
    import torch
    import torch.distributed as dist
    from paper_2312_06126_b200 import spz

    from paper_2312_06126_b200.dist import broadcast_bytes, env_rank
    rank, world, local = env_rank()
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE {world}: launch with torchrun --nproc-per-node {a.gpus} or without torchrun")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    assert a.warmup >= 3, "timing rules: at least 3 warm-up steps"
    dp = world > 1 and a.mode == "dp"
    split = world > 1 and a.mode == "split"
    GB = group_batch(a.mode, a.scaling, B, world)

    # ring filled to capacity with synthetic transitions (ring bytes > L2, so gathers hit HBM)
    C = w.capacity
    ring = spz.Replay(w.obs_dim, w.act_dim, C, device=local)
    chunk = 1_000_000
    chunks = []
    want_cpu = rank == 0 and world == 1 and not a.no_cpu_baseline
    for s0 in range(0, C, chunk):
        tr = synthdata.workload_transitions(w, n=min(chunk, C - s0), seed=synthdata.DATA_SEED + s0)
        ring.push(**tr)
        if want_cpu:
            chunks.append(tr)
    kw = {}
    if dp or split:
        kw = dict(world_size=world, rank=rank, nccl_unique_id=broadcast_bytes(spz.spz_nccl_unique_id() if rank == 0 else None))
    if split:
        nc = split_critics(world, a.critic_frac)
        kw.update(role=spz.SPZ_ROLE_CRITIC if rank < nc else spz.SPZ_ROLE_ACTOR, n_critic_ranks=nc,
                  n_actor_ranks=world - nc)
    stream = torch.cuda.Stream(device=local)
    # no fallback: a failing NCCL path is an error, not a silent switch to replicas
    lrn = spz.Learner(ring, algo=w.algo, precision=a.precision, hidden=w.hidden, n_hidden=w.n_hidden, max_batch=GB,
                      device=local, seed=synthdata.SAMPLE_SEED + (0 if (dp or split) else rank), **kw)
    lrn.set_stream(stream.cuda_stream)
    lrn.update(GB, a.warmup)  # warm-up (includes CUDA-graph capture)
    plan = spz.spz_plan_rank(GB, world if (dp or split) else 1, rank if (dp or split) else 0,
                             **({k: kw[k] for k in ("role", "n_critic_ranks")} if split else {}))
    with Clocks(local) as clk:
        time.sleep(0.3)
        reps, stats = timed_reps(lrn, GB, a.steps, a, stream, world, dist, torch)
    ms = statistics.median(reps)
    # transitions consumed per update: the group batch (counted once, though in split mode both groups read
    # it); replicas: N learners x B
    frames = GB * a.steps if (dp or split) else B * a.steps * world
    value = frames / (ms / 1e3)
    ms_per_step = ms / a.steps

    pk = peaks()
    n_actor = lrn.get("actor").size
    n_critic = sum(lrn.get(n).size for n in ("q1", "q2") + (("v",) if w.algo == "sacv1" else ()))
    prof = lrn.profile(GB, 5)
    fl = class_flops(w, plan["rows"] if (dp or split) else B)  # this rank's rows
    roof, gemm_f = roofline(w, plan["rows"] if (dp or split) else B, prof, a.precision, pk, n_actor, n_critic)
    roof["step_gemm_tflops"] = gemm_f / (ms_per_step * 1e-3) / 1e12
    roof["step_frac_of_bf16_sustained"] = roof["step_gemm_tflops"] / pk["bf16_sust"]
    kern = {k: {"ms": t, **({"tflops": fl[k] / (t * 1e-3) / 1e12} if k in fl else {})} for k, t in prof.items()}
    launches = lrn.launches_per_step(GB) * a.steps

    # the same measurement at the paper's implied precision (fp32 on a GTX 1060): FP32 = 3xTF32 tcgen05
    fp32 = None
    if not a.no_fp32 and a.precision == "bf16":
        lf = spz.Learner(ring, algo=w.algo, precision="fp32", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=GB,
                         device=local, seed=synthdata.SAMPLE_SEED + (0 if (dp or split) else rank), **kw)
        lf.set_stream(stream.cuda_stream)
        lf.update(GB, a.warmup)
        a_f = argparse.Namespace(**{**vars(a), "min_time": max(1.0, a.min_time / 2)})
        reps_f, _ = timed_reps(lf, GB, a.steps, a_f, stream, world, dist, torch)
        ms_f = statistics.median(reps_f)
        prof_f = lf.profile(GB, 3)
        roof_f, _ = roofline(w, plan["rows"] if (dp or split) else B, prof_f, "fp32", pk, n_actor, n_critic)
        fp32 = {"value": frames / (ms_f / 1e3), "unit": "frames/s", "dtype": "f32 (3xTF32 tcgen05)",
                "ms_per_step": ms_f / a.steps,
                "repetitions": {"n": len(reps_f), "median_ms": ms_f, "min_ms": min(reps_f), "max_ms": max(reps_f)},
                "roofline": roof_f}
        lf.close()

    # cpu_baseline + parity first: the e2e leg below pushes fresh transitions into the ring
    cpu, parity = None, None
    if want_cpu:
        cpu, parity = cpu_leg(a, w, B, ring, chunks)
        del chunks

    # e2e through the C ABI with host buffers
    e2e = None
    if not a.no_e2e:
        R_fields = 2 * w.obs_dim + w.act_dim + 2
        host = synthdata.workload_transitions(w, n=GB * 4, seed=synthdata.DATA_SEED + 99)
        pinned = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in host.items()}
        # each host-timed run covers >= 0.3 s of updates (host scheduling noise averages out; round 2's 200-step
        # runs of ~20 ms spread 51-59M frames/s on one box)
        K2 = max(3, a.steps, int(math.ceil(300.0 / max(ms_per_step, 1e-3))))
        sl = lambda k: slice((k % 4) * GB, (k % 4 + 1) * GB)  # dp: every rank's ring replica takes the global batch
        for k in range(3):  # warm: staging allocation on the first pinned push
            ring.push(**{n: v[sl(k)] for n, v in pinned.items()})
            lrn.update(GB, 1)
        torch.cuda.synchronize()
        runs = []
        for it in range(6):  # host-timed: a discarded warm run, then the median of five
            t0 = time.perf_counter()
            # step k: push its B fresh transitions (H2D from pinned host memory) while updates k-2 and k-1 run on
            # the GPU, read back update k-2's statistics (D2H), enqueue update k (spz_update_async / _wait,
            # two updates in flight)
            for k in range(K2):
                # push_async: the slice stays untouched until the next push returns (4 rotating slices)
                ring.push(**{n: v[sl(k)] for n, v in pinned.items()}, wait=False)
                if k >= 2:
                    lrn.wait()
                lrn.update_async(GB, 1)
            lrn.wait()
            lrn.wait()
            ring.sync()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([dt], device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = t.item()
            if it > 0:
                runs.append((GB if (dp or split) else B * world) * K2 / dt)
        e2e = {"value": statistics.median(runs), "unit": "frames/s",
               "h2d_bytes_per_step": GB * R_fields * 4 * world,
               "d2h_bytes_per_step": 9 * 8 + 8 * 8 + 16, "steps": K2, "runs": runs,  # the read-back block (stats, counters, flag)
               "note": "median of 5 host-timed runs of >= 0.3 s (after one discarded warm run); per step: spz_replay_push_async of B fresh host transitions (pinned, H2D) "
                       "overlapping the updates in flight, spz_update_wait (stats D2H of the oldest), spz_update_async(B, 1); "
                       "two updates in flight"}

    configs = None
    if world == 1 and not a.no_configs and a.precision == "bf16" and a.algo is None and a.batch is None:
        configs = other_configs(a, w.name, local, torch, dist)

    sweep = None
    if a.sweep and world == 1:
        ladder = [128, 512, 2048, 8192, 32768, 65536]
        tl = spz.Learner(ring, algo=w.algo, precision=a.precision, hidden=w.hidden, n_hidden=w.n_hidden,
                         max_batch=ladder[-1], device=local)
        best, pts = tl.tune_batch(ladder, warmup=5, steps=50, tol=1.0, restore=True)
        sweep = {"best_batch": best, "points": pts, "note": "spz_tune_batch, 50 timed updates per B (CUDA events)"}
        tl.close()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_per_step, "updates_per_s": 1e3 / ms_per_step, "higher_is_better": True,
            "repetitions": {"n": len(reps), "median_ms": ms, "min_ms": min(reps), "max_ms": max(reps),
                            "timed_s": sum(reps) / 1e3, "frames_per_rep": frames},
            "scaling": "weak" if (world == 1 or a.mode == "replicas" or a.scaling == "weak") else "strong",
            "vs_baseline": vs_baseline(w, value), "dtype": a.precision, "data": "synthetic",
            "config": {"workload": w.name, "global_batch": GB if (dp or split) else B * world,
                       "batch_per_gpu": plan["rows"] if (dp or split) else B, "algo": w.algo,
                       "mode": ("dp-nccl" if dp else "split-nccl" if split else "replicas") if world > 1 else "single",
                       "hidden": f"{w.n_hidden}x{w.hidden}", "obs_dim": w.obs_dim, "act_dim": w.act_dim,
                       "ring": C, "parallelism": (f"dp{world}" if dp else f"split{world}" if split else f"replicas{world}") if world > 1 else "single",
                       "l2": f"ring {C * ((2 * w.obs_dim + w.act_dim + 2 + 3) // 4 * 4) * 4 / 1e6:.0f} MB > 126 MB L2; fresh random indices each step (inputs larger than L2)"},
            "roofline": roof, "kernels": kern, "fp32": fp32, "cpu_baseline": cpu, "parity": parity, "e2e": e2e,
            "clocks": clk.summary(), "gpu_launches": launches, "last_stats": stats,
            **({"configs": configs} if configs else {}),
            **({"batch_sweep": sweep} if sweep else {}),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def other_configs(a, done, local, torch, dist):
    """The other BASELINE configs on this GPU, device-resident, bf16, K = a.steps updates per repetition (>= 3
    repetitions, >= 0.5 s): value, ms_per_step and the dominant tensor-core class against the peak -- so every
    config has a number in the driver's own bench line (parity for each: tests/test_gpu_parity.py)."""
    from paper_2312_06126_b200 import spz
    pk = peaks()
    out = {}
    for name in ("ant", "humanoid", "humanoid_td3"):
        if name == done:
            continue
        w = synthdata.WORKLOADS[name]
        ring = spz.Replay(w.obs_dim, w.act_dim, w.capacity, device=local)
        for s0 in range(0, w.capacity, 1_000_000):
            ring.push(**synthdata.workload_transitions(w, n=min(1_000_000, w.capacity - s0), seed=synthdata.DATA_SEED + s0))
        stream = torch.cuda.Stream(device=local)
        lrn = spz.Learner(ring, algo=w.algo, precision="bf16", hidden=w.hidden, n_hidden=w.n_hidden, max_batch=w.batch,
                          device=local, seed=synthdata.SAMPLE_SEED)
        lrn.set_stream(stream.cuda_stream)
        lrn.update(w.batch, a.warmup)
        K = max(3, min(a.steps, 20)) if w.batch > 8192 else a.steps
        reps, _ = timed_reps(lrn, w.batch, K, argparse.Namespace(reps=3, min_time=0.5), stream, 1, dist, torch)
        ms = statistics.median(reps)
        prof = lrn.profile(w.batch, 2)
        n_actor = lrn.get("actor").size
        n_critic = sum(lrn.get(n).size for n in ("q1", "q2"))
        roof, gemm_f = roofline(w, w.batch, prof, "bf16", pk, n_actor, n_critic)
        out[name] = {"value": w.batch * K / (ms / 1e3), "unit": "frames/s", "ms_per_step": ms / K, "steps": K,
                     "repetitions": len(reps), "global_batch": w.batch, "algo": w.algo,
                     "hidden": f"{w.n_hidden}x{w.hidden}", "dtype": "bf16",
                     "roofline": {**{k: roof[k] for k in ("kernel", "achieved", "peak", "unit", "frac")},
                                  "hbm": {k: {f: v[f] for f in ("achieved", "frac", "algorithmic_bytes_per_launch")}
                                          for k, v in roof.get("hbm", {}).items()}},
                     "step_gemm_tflops": gemm_f / (ms / K * 1e-3) / 1e12}
        lrn.close()
        ring.close()
        del stream
        torch.cuda.synchronize()
    return out


def cpu_leg(a, w, B, ring, chunks):
    """cpu_baseline + parity (rank 0, one GPU): K_o float64 oracle updates on the host cores from the
    same initial parameters, ring contents and seeds as K_o GPU updates, which are checked against them
    (tests/parity.py: statistics, raw gradients of every tensor, Adam moments, parameters); the oracle's
    update time is the baseline.  Plus a 1-thread oracle rate and the host CPU model (§8(d))."""
    from oracle import ring as oring
    from tests import parity as par
    r = oring.Ring(w.obs_dim, w.act_dim, w.capacity)
    for tr in chunks:
        r.push(**tr)
    K_o = a.parity_steps or PARITY_STEPS.get(w.name, 2)
    cores = len(os.sched_getaffinity(0))
    threads = None
    try:
        from threadpoolctl import threadpool_info
        threads = max((d.get("num_threads", 0) for d in threadpool_info()), default=None)
    except Exception:
        pass
    timing = {}
    parity = {"k_o": K_o, "precision": a.precision}
    if w.algo in ("sac", "td3"):
        try:
            res = par.run_parity(w.algo, a.precision, w.obs_dim, w.act_dim, w.hidden, w.n_hidden, B, w.capacity, K_o,
                                 rings=(ring, r), timing=timing, tag=f"bench-{w.name}")
            parity.update(ok=True, max_param_err=max(res["params"].values()),
                          max_grad_err=max(res["grads"].values()) if res["grads"] else None,
                          bar={"params": par.TOL[a.precision], "grads_net": par.grad_bar(a.precision, B),
                               "grads_tensor": par.GTOL_TENSOR[a.precision]})
        except AssertionError as e:
            parity.update(ok=False, error=str(e)[:500])
        oracle_s, steps = timing.get("oracle_s", 0.0), timing.get("oracle_steps", 0)
    else:
        parity.update(ok=None, note=f"{w.algo}: parity in tests/test_gpu_parity.py only")
        _, _, oracle_s = oracle_rate(w, B, K_o)
        steps = K_o
    rate = B * steps / oracle_s if oracle_s > 0 else None
    one = None
    try:
        from threadpoolctl import threadpool_limits
        n1 = 1 if w.name.startswith(("humanoid",)) else 2
        with threadpool_limits(1):
            r1, _, dt1 = oracle_rate(w, B, n1)
        one = {"value": r1, "steps": n1, "seconds": dt1}
    except Exception as e:  # threadpoolctl missing: report why
        one = {"error": str(e)[:200]}
    cpu = {"value": rate, "unit": "frames/s", "cores": cores, "threads": threads, "kind": "oracle", "cpu_model": cpu_model(),
           "sample": f"{steps} float64 oracle updates at B={B} ({w.name}), {oracle_s:.1f} s -- the same steps the parity check runs",
           "one_thread": one}
    return cpu, parity


if __name__ == "__main__":
    main()
