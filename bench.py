"""Benchmark: SAC/TD3 update frames/s on B200 (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config walker] [--precision bf16]
    python bench.py --impl reference ...      # the float64 CPU oracle arm (host cores)

A "step" is one full update over one batch of B transitions
sampled from a device-resident ring filled with synthetic transitions (synthdata).
value = B * K * N / (max over ranks of the CUDA-event time of K steps) [frames/s];
frames/s = update frequency x B.  With N > 1 (torchrun, one process per GPU) the
default --mode dp runs ONE row-sharded learner group over a global batch of B * N (each
GPU B rows; gradients all-reduced with NCCL inside the step; weak scaling); --mode
replicas runs N independent learners instead.

Extra keys: roofline (dominant kernel class vs the measured peak in
MEASURED_PEAKS.json), cpu_baseline (the oracle on this host's cores, bounded sample),
e2e (through the C ABI with host buffers: each step pushes B fresh transitions from
pinned host memory and reads the stats back), clocks (nvidia-smi during the timed
region), gpu_launches (our kernels launched in the timed region).
"""

import argparse
import dataclasses
import json
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
    return ap.parse_args()


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


def class_bytes(w, B, n_params):
    """Algorithmic HBM bytes per step for the memory-bound classes (§8(d))."""
    R = (2 * w.obs_dim + w.act_dim + 2 + 3) // 4 * 4
    return {"gather": B * (4 * R + 4),
            # Adam+Polyak: read p, m, v, g; write p, m, v (+ target read/write for critics) -- fp32
            "adam_polyak": n_params * 28 + n_params * 2 // 3 * 8}


# the paper's network-update frame rate for Walker2D SAC at its default batch (~8192):
# 3.7E+5 Hz -- on a GTX 1060, network size unstated: context, not the target
PAPER_WALKER_HZ = 3.7e5


def vs_baseline(w, value):
    return value / PAPER_WALKER_HZ if w.name == "walker" else None


def traffic(workload, kernel):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu --set full capture, or None."""
    p = os.path.join(ROOT, "profiles", "r01_traffic.json")
    try:
        e = json.load(open(p))[workload][kernel]
    except (OSError, KeyError, ValueError):
        return None
    return e["dram_read"] + e["dram_write"]


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
            "cpu_baseline": {"value": rate, "unit": "frames/s", "cores": cores, "kind": "oracle",
                             "sample": f"{steps} full float64 oracle updates at B={B} ({w.name})"},
            "e2e": {"value": rate, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm

def main():
    a = parse()
    w = synthdata.WORKLOADS[a.config]
    if a.algo and a.algo != w.algo:
        w = dataclasses.replace(w, name=f"{w.name}_{a.algo}", algo=a.algo)
    B = a.batch or w.batch
    if a.impl == "reference":
        reference_arm(a, w, B)
        return
    import torch
    import torch.distributed as dist
    from paper_2312_06126_b200 import spz

    from paper_2312_06126_b200.dist import broadcast_bytes, env_rank
    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    assert a.warmup >= 3, "timing rules: at least 3 warm-up steps"
    dp = world > 1 and a.mode == "dp"
    split = world > 1 and a.mode == "split"
    # the batch one learner group consumes per update: dp B*N; split B*N/2 (both groups read every row)
    GB = B * world if dp else (B * world // 2 if split else B)

    # ring filled to capacity with synthetic transitions (ring bytes > L2, so gathers hit HBM)
    C = w.capacity
    ring = spz.Replay(w.obs_dim, w.act_dim, C, device=local)
    chunk = 1_000_000
    for s0 in range(0, C, chunk):
        tr = synthdata.workload_transitions(w, n=min(chunk, C - s0), seed=synthdata.DATA_SEED + s0)
        ring.push(**tr)
    kw = {}
    if dp or split:
        kw = dict(world_size=world, rank=rank, nccl_unique_id=broadcast_bytes(spz.spz_nccl_unique_id() if rank == 0 else None))
    if split:
        nc = min(world - 1, max(1, int(round(world * a.critic_frac))))
        kw.update(role=spz.SPZ_ROLE_CRITIC if rank < nc else spz.SPZ_ROLE_ACTOR, n_critic_ranks=nc,
                  n_actor_ranks=world - nc)
    stream = torch.cuda.Stream(device=local)
    fallback = None
    try:
        lrn = spz.Learner(ring, algo=w.algo, precision=a.precision, hidden=w.hidden, n_hidden=w.n_hidden, max_batch=GB,
                          device=local, seed=synthdata.SAMPLE_SEED + (0 if (dp or split) else rank), **kw)
        lrn.set_stream(stream.cuda_stream)
        # warm-up (includes CUDA-graph capture)
        lrn.update(GB, a.warmup)
        ok, err = 1, ""
    except spz.SpzError as e:
        ok, err = 0, str(e)
    if world > 1:
        t = torch.tensor([ok], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok = int(t.item())
    if not ok:
        if not (dp or split):
            raise RuntimeError(err)
        # the NCCL path failed on some rank: measure independent replicas instead (no collective), and say so
        fallback = f"{a.mode} path failed ({err or 'on another rank'}); measured {world} independent replicas"
        dp = split = False
        GB = B
        lrn = spz.Learner(ring, algo=w.algo, precision=a.precision, hidden=w.hidden, n_hidden=w.n_hidden, max_batch=GB,
                          device=local, seed=synthdata.SAMPLE_SEED + rank)
        lrn.set_stream(stream.cuda_stream)
        lrn.update(GB, a.warmup)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        time.sleep(0.3)
        ev0.record(stream)
        stats = lrn.update(GB, a.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        dist.barrier()
    torch.cuda.synchronize()
    # transitions consumed: dp B*N per update; split B*N/2 per update (counted once, though both groups read it);
    # replicas N learners x B
    frames = GB * a.steps if (dp or split) else B * a.steps * world
    value = frames / (ms / 1e3)
    ms_per_step = ms / a.steps

    # per-class device time (event-bracketed, un-graphed, same learner and batch) -> roofline
    prof = lrn.profile(GB, 5)
    pk = peaks()
    fl = class_flops(w, B)  # per-GPU rows
    n_params = sum(lrn.get(n).size for n in ("actor", "q1", "q2") + (("v",) if w.algo == "sacv1" else ()))
    by = class_bytes(w, B, n_params)
    kern = {}
    for k, t in prof.items():
        e = {"ms": t}
        if k in fl:
            e["tflops"] = fl[k] / (t * 1e-3) / 1e12
        if k in by:
            e["gbs"] = by[k] / (t * 1e-3) / 1e9
        kern[k] = e
    dom = max(prof, key=prof.get)
    if dom in fl:
        ach = fl[dom] / (prof[dom] * 1e-3) / 1e12
        pkv = pk["bf16_sust"] if a.precision == "bf16" else pk["bf16_sust"] / 2.0  # tf32 = bf16 / 2 (nominal ratio)
        roof = {"bound": "tensor", "kernel": dom, "achieved": ach, "peak": pkv, "unit": "TFLOP/s", "frac": ach / pkv,
                "traffic": None, "peak_src": f"{pk['src']} bf16 sustained" + ("" if a.precision == "bf16" else " x 1/2 (tf32 nominal ratio)")}
    else:
        ach = by.get(dom, 0) / (prof[dom] * 1e-3) / 1e9
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": pk["hbm"], "unit": "GB/s", "frac": ach / pk["hbm"],
                "traffic": None, "peak_src": f"{pk['src']} hbm"}
    tr = traffic(w.name, roof["kernel"])
    if tr is not None:
        roof["traffic"] = tr
        roof["traffic_src"] = "profiles/r01_traffic.json (ncu --set full, per launch)"
    gemm_t = sum(t for k, t in prof.items() if k in fl)
    gemm_f = sum(v for k, v in fl.items() if not k.endswith("_mlp"))  # the fused classes repeat per-layer work
    roof["step_gemm_tflops"] = gemm_f / (ms_per_step * 1e-3) / 1e12
    roof["step_frac_of_bf16_sustained"] = roof["step_gemm_tflops"] / pk["bf16_sust"]
    roof["gemm_share_of_step"] = gemm_t / sum(prof.values())
    launches = lrn.launches_per_step(GB) * a.steps

    # e2e through the C ABI with host buffers
    e2e = None
    if not a.no_e2e:
        R_fields = 2 * w.obs_dim + w.act_dim + 2
        host = synthdata.workload_transitions(w, n=GB * 4, seed=synthdata.DATA_SEED + 99)
        pinned = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in host.items()}
        K2 = max(3, min(a.steps, 500))
        sl = lambda k: slice((k % 4) * GB, (k % 4 + 1) * GB)  # dp: every rank's ring replica takes the global batch
        for k in range(3):  # warm: staging allocation on the first pinned push
            ring.push(**{n: v[sl(k)] for n, v in pinned.items()})
            lrn.update(GB, 1)
        torch.cuda.synchronize()
        runs = []
        for _ in range(3):  # host-timed: the median of three runs (host scheduling noise)
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
            runs.append((GB if (dp or split) else B * world) * K2 / dt)
        e2e = {"value": statistics.median(runs), "unit": "frames/s",
               "h2d_bytes_per_step": GB * R_fields * 4 * world,
               "d2h_bytes_per_step": 9 * 8 + 8 * 8 + 16, "steps": K2, "runs": runs,  # the read-back block (stats, counters, flag)
               "note": "median of 3 host-timed runs; per step: spz_replay_push_async of B fresh host transitions (pinned, H2D) "
                       "overlapping the updates in flight, spz_update_wait (stats D2H of the oldest), spz_update_async(B, 1); "
                       "two updates in flight"}

    sweep = None
    if a.sweep and world == 1:
        ladder = [128, 512, 2048, 8192, 32768, 65536]
        tl = spz.Learner(ring, algo=w.algo, precision=a.precision, hidden=w.hidden, n_hidden=w.n_hidden,
                         max_batch=ladder[-1], device=local)
        best, pts = tl.tune_batch(ladder, warmup=5, steps=50, tol=1.0, restore=True)
        sweep = {"best_batch": best, "points": pts, "note": "spz_tune_batch, 50 timed updates per B (CUDA events)"}
        tl.close()

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        # bounded sample: ~15 s of oracle work (one probe update sizes it), at least one update
        if a.cpu_sample_steps:
            steps = a.cpu_sample_steps
        else:
            _, _, probe = oracle_rate(w, B, 1)
            steps = max(1, min(2000, int(15.0 / max(probe, 1e-3))))
        rate, cores, dt = oracle_rate(w, B, steps)
        cpu = {"value": rate, "unit": "frames/s", "cores": cores, "kind": "oracle",
               "sample": f"{steps} float64 oracle updates at B={B} ({w.name}), {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_per_step, "updates_per_s": 1e3 / ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": vs_baseline(w, value), "dtype": a.precision, "data": "synthetic",
            "config": {"workload": w.name, "global_batch": GB if (dp or split) else B * world,
                       "batch_per_gpu": B if not split else GB // max(1, (world // 2)), "algo": w.algo,
                       "mode": ("dp-nccl" if dp else "split-nccl" if split else "replicas") if world > 1 else "single",
                       "hidden": f"{w.n_hidden}x{w.hidden}", "obs_dim": w.obs_dim, "act_dim": w.act_dim,
                       "ring": C, "parallelism": (f"dp{world}" if dp else f"split{world}" if split else f"replicas{world}") if world > 1 else "single",
                       "l2": f"ring {C * ((2 * w.obs_dim + w.act_dim + 2 + 3) // 4 * 4) * 4 / 1e6:.0f} MB > 126 MB L2; fresh random indices each step"},
            "roofline": roof, "kernels": kern, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clk.summary(), "gpu_launches": launches, "last_stats": stats,
            **({"batch_sweep": sweep} if sweep else {}),
            **({"fallback": fallback} if fallback else {}),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
