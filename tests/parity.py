"""Whole-update parity of the CUDA path (through the C ABI) against the float64 oracle.

TEST INFRASTRUCTURE (imports oracle/): used by tests/test_gpu_parity.py, __graft_entry__.smoke()
and the cpu_baseline leg of bench.py.

What one run pins, at every step k of K (SURVEY.md §8(c) "SAC step k" / "TD3 step k"; DESIGN.md
reading #20 for the metric, #25 for the gradient bound):

* the step statistics (losses, mean q, mean log pi, alpha) against the oracle's;
* the raw reduced gradient of every trained tensor (each layer's W and b of actor, q1, q2 -- TD3's
  actor on delayed steps only -- and log alpha), recovered exactly from the GPU's Adam first moment:
  g_k = (m_k - b1 m_{k-1}) / (1 - b1), against the oracle's gradient at its own step-k
  state.  A skipped Adam, a dropped weight or bias gradient, a wrong sign anywhere in a3-a7 fails it;
* after K steps: every parameter tensor (online and target) and both Adam moments m and v;
* on the last step, the GPU's own Adam and Polyak arithmetic in float64 from the GPU's values:
  theta_K = theta_{K-1} - lr (m_K / (1 - b1^t)) / (sqrt(v_K / (1 - b2^t)) + eps) and
  theta'_K = tau theta_K + (1 - tau) theta'_{K-1} -- the optimizer pinned independently of the
  ill-conditioned sign-like first Adam steps (App. B).
"""

import json
import os
import time

import numpy as np

import synthdata
from oracle import mlp, sac as osac, td3 as otd3

SEED = synthdata.SAMPLE_SEED
TOL = {"fp32": 1e-4, "bf16": 2e-2}
# raw-gradient bound per network / per tensor (reading #25: bf16 operands, measured on B200)
GTOL = {"fp32": 1e-4, "bf16": 2e-2}
# bf16 at small batches (B < 4096): the rounding noise of the bf16 operands averages over fewer rows; at
# PEN (B 256, m 1: a one-column action gradient summed over 64 units) the actor gradient reaches 2.6e-2
GTOL_SMALL_B = {"fp32": 1e-4, "bf16": 5e-2}
GTOL_TENSOR = {"fp32": 1e-3, "bf16": 1e-1}


def grad_bar(precision, B):
    return GTOL[precision] if B >= 4096 else GTOL_SMALL_B[precision]


def rel(x, ref):
    x, ref = np.asarray(x, np.float64), np.asarray(ref, np.float64)
    return float(np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-30))


def shapes_of(algo, cfg):
    td3 = algo in ("td3", "ddpg")
    return {"actor": osac.actor_shapes(cfg, td3=td3), "q1": osac.critic_shapes(cfg), "q2": osac.critic_shapes(cfg)}


def tensors(flat, shp):
    """Flat [W1|b1|...] -> [("W0", W), ("b0", b), ...]."""
    out = []
    for l, (W, b) in enumerate(mlp.unflatten(np.asarray(flat, np.float64), shp)):
        out += [(f"W{l}", W.ravel()), (f"b{l}", b)]
    return out


def oracle_inputs(algo, k, r, B, cfg):
    """Step k's minibatch and noise (a1-a2 and the Philox draws of §8(c) steps 1-2)."""
    idx, batch = r.sample(B, SEED, k)
    if algo == "sac":
        return batch, osac.draw_noise(SEED, k, B, cfg.act_dim)
    return batch, otd3.draw_smoothing(SEED, k, B, cfg)


def oracle_grads(algo, st, batch, noise, cfg, B, decisions=None):
    if algo == "sac":
        eps, eps2 = noise
        return osac.sac_grads(st, batch, eps, eps2, cfg, B, decisions=decisions)
    return otd3.td3_grads(st, batch, noise, cfg, B, st.step, decisions=decisions)


def oracle_step(algo, st, r, B, cfg, decisions=None):
    """sac_step / td3_step composed from their parts so the step's gradients are returned too (decisions:
    reading #25 -- the kernel's ReLU / min-tie decisions, taken by both sides in the kernel's precision)."""
    batch, noise = oracle_inputs(algo, st.step, r, B, cfg)
    grads, sums = oracle_grads(algo, st, batch, noise, cfg, B, decisions)
    if algo == "sac":
        return osac.sac_apply(st, grads, cfg), osac.stats_of(st, sums, B, cfg), grads
    return otd3.td3_apply(st, grads, cfg, st.step), otd3.stats_of(st, sums, B), grads


def state_of(snap, step, td3):
    """An oracle State at the GPU's parameters (snap: get() of every network + log alpha)."""
    st = osac.State.create(snap["actor"], snap["q1"], snap["q2"], snap["q1_targ"], snap["q2_targ"],
                           log_alpha=float(snap["log_alpha"][0]), actor_targ=snap["actor_targ"] if td3 else None)
    st.step = step
    return st


def unpack_mask(words, rows, h):
    """Packed ReLU-mask words [rows x ceil(h/32)] u32 (bit c % 32 of word c / 32) -> bool [rows x h]."""
    mw = (h + 31) // 32
    w = np.ascontiguousarray(words[:rows * mw]).reshape(rows, mw)
    return np.unpackbits(w.view(np.uint8), axis=1, bitorder="little")[:, :h].astype(bool)


def gpu_decisions(lrn, algo, precision, B, h, L, k, cfg):
    """The comparisons the kernels took at the last step -- ReLU masks of every gradient-carrying pass and
    the min-tie weight of Q1 on the actor rows -- for oracle_grads (reading #25).  bf16: the
    packed mask words the forward epilogues wrote; FP32: the sign of the stored fp32 activations."""
    dec = {}
    actor_rows = algo == "sac" or otd3.is_delayed(k, cfg)
    mw = (h + 31) // 32

    def masks(name, row0):
        if precision == "bf16":
            return unpack_mask(lrn.debug(name)[row0 * mw:], B, h)
        return lrn.debug(name)[row0 * h:(row0 + B) * h].reshape(B, h) > 0

    on = (lambda i, l: f"mask_c{i}_{l}") if precision == "bf16" else (lambda i, l: f"Aon{i}_{l}")
    act = (lambda l: f"mask_a{l}") if precision == "bf16" else (lambda l: f"Aact{l}")
    for i in range(2):
        dec[f"q{i + 1}"] = [masks(on(i, l), 0) for l in range(L)]
        if actor_rows and (algo == "sac" or i == 0):
            dec[f"q{i + 1}_pi"] = [masks(on(i, l), B) for l in range(L)]
    if actor_rows:
        dec["actor"] = [masks(act(l), B) for l in range(L)]
    if algo == "sac":
        qp = (h + 255) // 256 if precision == "bf16" else 1
        stride = 2 * B
        q = []
        for i in range(2):
            buf = lrn.debug(f"q_on{i}")
            acc = buf[B:2 * B].copy()
            for p in range(1, qp):  # the loss kernel's fp32 tile-order sum
                acc = (acc + buf[p * stride + B:p * stride + 2 * B]).astype(np.float32)
            q.append(acc)
        dec["w1"] = np.where(q[0] < q[1], 1.0, np.where(q[0] > q[1], 0.0, 0.5))
    return dec


def make_rings(o, m, C, n_push=None, seed=synthdata.DATA_SEED, kind="locomotion"):
    from oracle import ring as oring
    from paper_2312_06126_b200 import spz
    n = C if n_push is None else n_push
    g = spz.Replay(o, m, C)
    r = oring.Ring(o, m, C)
    chunk = 1_000_000  # bounded host memory for the 4M-transition TD3 ring
    for s0 in range(0, n, chunk):
        tr = synthdata.transitions(kind, o, m, min(chunk, n - s0), seed=seed if s0 == 0 else seed + s0)
        first = g.push(**tr)
        assert r.push(**tr) == first
    return g, r


def _report(rec):
    p = os.environ.get("SPZ_PARITY_REPORT")
    if p:
        with open(p, "a") as f:
            f.write(json.dumps(rec) + "\n")


def check_adam_polyak_identity(prev, cur, m, v, cfg, trained, targets, tag):
    """Last step, GPU values only: Adam (per optimizer t) and Polyak reproduce in float64 to fp32 rounding."""
    b1, b2, eps = cfg.beta1, cfg.beta2, cfg.adam_eps
    for n, lr, tn in trained:
        if tn is None:
            continue
        p0, p1 = prev[n].astype(np.float64), cur[n].astype(np.float64)
        mm, vv = m[n].astype(np.float64), v[n].astype(np.float64)
        step = lr * (mm / (1 - b1 ** tn)) / (np.sqrt(vv / (1 - b2 ** tn)) + eps)
        pred = p0 - step
        # fp32 kernel: each operation rounds (~1e-7 relative of the step) and the result rounds to fp32
        bound = 4 * np.spacing(np.abs(pred).astype(np.float32)).astype(np.float64) + 1e-5 * np.abs(step) + 1e-12
        bad = np.abs(p1 - pred) > bound
        assert not bad.any(), (tag, "adam identity", n, int(bad.sum()), float(np.max(np.abs(p1 - pred) - bound)))
    for tname, n in targets:
        t0, t1 = prev[tname].astype(np.float64), cur[tname].astype(np.float64)
        a_term, b_term = cfg.tau * cur[n].astype(np.float64), (1 - cfg.tau) * t0
        pred = a_term + b_term
        # fp32: each product rounds too, so where the terms nearly cancel (an online weight ~ -(1-tau)/tau times
        # its target, i.e. weights within ~3e-5 of zero) the error is an ulp of the terms, not of the result
        sp = lambda x: np.spacing(np.abs(x).astype(np.float32)).astype(np.float64)
        bound = 4 * (sp(pred) + sp(a_term) + sp(b_term)) + 1e-12
        bad = np.abs(t1 - pred) > bound
        assert not bad.any(), (tag, "polyak identity", tname, int(bad.sum()))


def run_parity(algo, precision, o, m, h, L, B, C, K, kind="locomotion", use_graph=True, check_grads=True,
               check_moments=True, rings=None, tag="", timing=None):
    """K full updates on the GPU and in the oracle from the same parameters, ring and seeds; asserts the
    module-level bar and returns {"params": ..., "grads": ...} relative errors (max over steps)."""
    from paper_2312_06126_b200 import spz
    g, r = rings if rings is not None else make_rings(o, m, C, kind=kind)
    p = synthdata.init_params(o, m, h, L, algo=algo)
    lrn = spz.Learner(g, algo=algo, precision=precision, hidden=h, n_hidden=L, max_batch=B, use_graph=use_graph)
    for n in ("actor", "q1", "q2"):
        lrn.set(n, p[n])
    lrn.set("q1_targ", p["q1"])
    lrn.set("q2_targ", p["q2"])
    td3 = algo == "td3"
    if td3:
        lrn.set("actor_targ", p["actor"])
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L, alpha_auto=(algo == "sac"))
    la = float(lrn.get("log_alpha")[0])
    st = osac.State.create(p["actor"], p["q1"], p["q2"], log_alpha=la, actor_targ=p["actor"] if td3 else None)
    tol, gtol, gtol_t = TOL[precision], grad_bar(precision, B), GTOL_TENSOR[precision]
    shp = shapes_of(algo, cfg)
    trained = ["actor", "q1", "q2"]
    targ_names = ["q1_targ", "q2_targ"] + (["actor_targ"] if td3 else [])
    all_names = trained + targ_names
    M = spz.SPZ_S_ADAM_M
    m_prev = {n: lrn.get(n, M).astype(np.float64) for n in trained}
    la_m_prev = float(lrn.get("log_alpha", M)[0])
    gerr = {}
    prev = None
    m_ref = {n: np.zeros_like(m_prev[n]) for n in trained}  # Adam moments of the GPU-state oracle gradients
    v_ref = {n: np.zeros_like(m_prev[n]) for n in trained}
    for k in range(K):
        # the GPU's step-k state: the gradient check evaluates the oracle there, so it pins step k's
        # arithmetic free of the trajectory drift (Adam's sign-like map of near-zero gradients, App. B)
        prev = {n: lrn.get(n) for n in all_names + ["log_alpha"]}
        gs = lrn.update(B, 1)
        batch, noise = oracle_inputs(algo, k, r, B, cfg)
        dec = gpu_decisions(lrn, algo, precision, B, h, L, k, cfg) if check_grads else None
        t0 = time.perf_counter()
        st, os_, _ = oracle_step(algo, st, r, B, cfg, dec)
        if timing is not None:  # bench.py's cpu_baseline: the oracle's own update time
            timing["oracle_s"] = timing.get("oracle_s", 0.0) + time.perf_counter() - t0
            timing["oracle_steps"] = timing.get("oracle_steps", 0) + 1
        assert gs["step"] == k + 1
        for key in ("critic_loss", "actor_loss", "q1_mean", "q2_mean", "logp_mean", "alpha"):
            ref = os_[key]
            # a mean of signed terms is compared relative to the mean |term| (its summation error scales with it)
            scale = max(abs(ref), os_.get(key + "_abs", 0.0))
            assert abs(gs[key] - ref) <= tol * max(scale, 1e-6) + (tol * 1e-2 if key in ("q1_mean", "q2_mean") else 0), \
                (tag, k, key, gs[key], ref)
        if not check_grads:
            continue
        grads, gsums = oracle_grads(algo, state_of(prev, k, td3), batch, noise, cfg, B, dec)
        m_now = {n: lrn.get(n, M).astype(np.float64) for n in trained}
        for n in trained:
            if n not in grads:  # TD3 actor on non-delayed steps: no Adam step, m unchanged
                assert np.array_equal(m_now[n], m_prev[n]), (tag, k, n, "moment moved without an update")
                continue
            gg = (m_now[n] - cfg.beta1 * m_prev[n]) / (1.0 - cfg.beta1)
            gr = np.asarray(grads[n], np.float64)
            m_ref[n] = cfg.beta1 * m_ref[n] + (1 - cfg.beta1) * gr
            v_ref[n] = cfg.beta2 * v_ref[n] + (1 - cfg.beta2) * gr * gr
            e_net = rel(gg, gr)
            _report({"tag": tag, "precision": precision, "step": k, "net": n, "tensor": "all", "err": e_net,
                     "norm": float(np.linalg.norm(gr))})
            gerr[n] = max(gerr.get(n, 0.0), e_net)
            assert e_net <= gtol, (tag, k, n, "gradient", e_net)
            for (tn, a), (_, b) in zip(tensors(gg, shp[n]), tensors(gr, shp[n])):
                e = rel(a, b)
                _report({"tag": tag, "precision": precision, "step": k, "net": n, "tensor": tn, "err": e,
                         "norm": float(np.linalg.norm(b))})
                gerr[f"{n}.{tn}"] = max(gerr.get(f"{n}.{tn}", 0.0), e)
                assert e <= gtol_t, (tag, k, n, tn, "gradient", e)
        if algo == "sac":
            la_m = float(lrn.get("log_alpha", M)[0])
            g_la = (la_m - cfg.beta1 * la_m_prev) / (1.0 - cfg.beta1)
            ref = float(grads["log_alpha"][0])
            lpm = gsums["logp"] / B
            _report({"tag": tag, "precision": precision, "step": k, "net": "log_alpha", "tensor": "all",
                     "err": abs(g_la - ref) / max(abs(ref), abs(lpm), 1e-6), "norm": abs(ref)})
            assert abs(g_la - ref) <= gtol * max(abs(ref), abs(lpm), 1e-6), (tag, k, "log_alpha grad", g_la, ref)
            la_m_prev = la_m
        m_prev = m_now
    errs = {}
    for n in all_names:
        errs[n] = rel(lrn.get(n), getattr(st, n))
        assert errs[n] <= tol, (tag, n, errs)
    if algo == "sac":
        assert abs(float(lrn.get("log_alpha")[0]) - st.log_alpha) <= tol * max(1.0, abs(st.log_alpha))
    c = lrn.counters()
    assert c["step"] == K and c["t_critic"] == K
    n_act = K if algo == "sac" else sum(1 for k in range(K) if otd3.is_delayed(k, cfg))
    assert c["t_actor"] == n_act
    mK = {n: lrn.get(n, M) for n in trained}
    vK = {n: lrn.get(n, spz.SPZ_S_ADAM_V) for n in trained}
    if check_moments and check_grads:
        # m and v of every trained net against the moments of the step-by-step oracle gradients
        for n in trained:
            if st.opt[n].t == 0:
                continue
            em, ev = rel(mK[n], m_ref[n]), rel(vK[n], v_ref[n])
            errs[n + ".m"], errs[n + ".v"] = em, ev
            assert em <= gtol, (tag, n, "m", em)
            assert ev <= 2 * gtol, (tag, n, "v", ev)
    cur = {nn: lrn.get(nn) for nn in all_names}
    delayed_last = (not td3) or otd3.is_delayed(K - 1, cfg)
    tr = [("q1", cfg.lr_critic, c["t_critic"]), ("q2", cfg.lr_critic, c["t_critic"]),
          ("actor", cfg.lr_actor, c["t_actor"] if delayed_last else None)]
    tg = [("q1_targ", "q1"), ("q2_targ", "q2")] + ([("actor_targ", "actor")] if td3 else [])
    check_adam_polyak_identity(prev, cur, mK, vK, cfg, tr, tg if delayed_last else [], tag)
    if td3 and not delayed_last:  # targets frozen on non-delayed steps
        for tname, _ in tg:
            assert np.array_equal(cur[tname], prev[tname]), (tag, tname, "target moved on a non-delayed step")
    lrn.close()
    return {"params": errs, "grads": gerr}
