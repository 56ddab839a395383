"""Diagnosis: compare step-0 intermediates of the CUDA path with the oracle (test infrastructure)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synthdata
from oracle import ring as oring, sac as osac, mlp
from paper_2312_06126_b200 import spz

def run(o, m, h, L, B, C, precision):
    tr = synthdata.transitions("locomotion", o, m, C)
    g = spz.Replay(o, m, C); g.push(**tr)
    r = oring.Ring(o, m, C); r.push(**tr)
    p = synthdata.init_params(o, m, h, L)
    lrn = spz.Learner(g, precision=precision, hidden=h, n_hidden=L, max_batch=B)
    for n in ("actor", "q1", "q2"): lrn.set(n, p[n])
    lrn.set("q1_targ", p["q1"]); lrn.set("q2_targ", p["q2"])
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L)
    la = float(lrn.get("log_alpha")[0])
    st = osac.State.create(p["actor"], p["q1"], p["q2"], log_alpha=la)
    gs = lrn.update(B, 1)
    idx, b = r.sample(B, 6126, 0)
    eps, eps2 = osac.draw_noise(6126, 0, B, m)
    s, a, rr, s2, d = [np.asarray(b[k], np.float64) for k in ("obs", "act", "rew", "next_obs", "done")]
    A = mlp.unflatten(st.actor, osac.actor_shapes(cfg))
    H, _ = mlp.forward(A, np.concatenate([s2, s]))
    a2, lp2, _, _ = osac.policy_forward(A, s2, eps2, cfg)
    at, lp, _, _ = osac.policy_forward(A, s, eps, cfg)
    cs = osac.critic_shapes(cfg)
    q1 = osac.critic_q(mlp.unflatten(st.q1, cs), s, a)[0]
    qt1 = osac.critic_q(mlp.unflatten(st.q1_targ, cs), s2, a2)[0]
    def cmp(name, gpu, ref):
        gpu = np.asarray(gpu, np.float64).reshape(ref.shape)
        e = np.abs(gpu - ref).max() / max(np.abs(ref).max(), 1e-30)
        bad = np.argwhere(np.abs(gpu - ref) > 1e-3 * max(np.abs(ref).max(), 1e-30))
        print(f"{name:8s} maxrel {e:.3e}  first bad {bad[:3].tolist() if len(bad) else None}")
    gidx = lrn.debug("idx")[:B]
    print("idx equal", np.array_equal(gidx, idx))
    lda, ldc, ldh = (o + 7)//8*8, (o + m + 7)//8*8, (2*m + 7)//8*8
    Xa = lrn.debug("Xa")[:2*B*lda].reshape(2*B, lda)
    cmp("Xa", Xa[:, :o], np.concatenate([s2, s]))
    Xc = lrn.debug("Xc")[:3*B*ldc].reshape(3*B, ldc)
    cmp("Xc_sa", Xc[:B, :o+m], np.concatenate([s, a], 1))
    cmp("Xc_s2a2", Xc[2*B:, :o+m], np.concatenate([s2, a2], 1))
    cmp("Xc_sat", Xc[B:2*B, :o+m], np.concatenate([s, at], 1))
    Hg = lrn.debug("H")[:2*B*ldh].reshape(2*B, ldh)[:, :2*m]
    cmp("H", Hg, H)
    A0 = lrn.debug("Aact0")[:2*B*h].reshape(2*B, h)
    cmp("Aact0", A0, np.maximum(np.concatenate([s2, s]) @ A[0][0].T + A[0][1], 0))
    cmp("logp2", lrn.debug("logp2")[:B], lp2)
    cmp("logp", lrn.debug("logp")[:B], lp)
    cmp("q_on0", lrn.debug("q_on0")[:B], q1)
    cmp("q_tg0", lrn.debug("q_tg0")[:B], qt1)
    q2 = osac.critic_q(mlp.unflatten(st.q2, cs), s, a)[0]
    qt2 = osac.critic_q(mlp.unflatten(st.q2_targ, cs), s2, a2)[0]
    cmp("q_on1", lrn.debug("q_on1")[:B], q2)
    cmp("q_tg1", lrn.debug("q_tg1")[:B], qt2)
    y = rr + cfg.gamma * (1 - d) * (np.minimum(qt1, qt2) - np.exp(la) * lp2)
    cmp("y", lrn.debug("y")[:B], y)
    print("critic_loss gpu", gs["critic_loss"], "oracle", np.mean((q1 - y) ** 2 + (q2 - y) ** 2))
    gy = lrn.debug("y")[:B]; gq1 = lrn.debug("q_on0")[:B]; gq2 = lrn.debug("q_on1")[:B]
    print("critic_loss from gpu buffers", np.mean((gq1 - gy) ** 2 + (gq2 - gy) ** 2))
    # shadow of the target critics vs the oracle weights
    npc = mlp.n_params(cs); npa = mlp.n_params(osac.actor_shapes(cfg))
    r64 = lambda x: (x + 63)//64*64
    pb = {}; off = 0
    for nm, n in (("actor", npa), ("q1", npc), ("q2", npc), ("q1t", npc), ("q2t", npc)):
        pb[nm] = off; off += r64(n)
    P = lrn.debug("P")
    for nm, ref in (("q1t", st.q1_targ), ("q2t", st.q2_targ)):
        cmp("P_" + nm, P[pb[nm]:pb[nm] + npc], ref)
    S = lrn.debug("S")
    def ns_of(shapes):
        return sum(r64(o_ * ((i_ + 7)//8*8)) for o_, i_ in shapes)
    sb = {}; off = 0
    for nm, shp in (("actor", osac.actor_shapes(cfg)), ("q1", cs), ("q2", cs), ("q1t", cs), ("q2t", cs)):
        sb[nm] = off; off += ns_of(shp)
    for nm, flat in (("q1t", st.q1_targ), ("q2t", st.q2_targ)):
        Ws = mlp.unflatten(flat, cs)
        o2 = sb[nm]
        for l, (o_, i_) in enumerate(cs):
            ld = (i_ + 7)//8*8
            Wg = S[o2:o2 + o_*ld].reshape(o_, ld)[:, :i_]
            cmp(f"S_{nm}_{l}", Wg, Ws[l][0])
            o2 += r64(o_*ld)
    At = lrn.debug("Atg1_0")[:B*h].reshape(B, h)
    W0 = mlp.unflatten(st.q2_targ, cs)[0]
    cmp("Atg1_0", At, np.maximum(np.concatenate([s2, a2], 1) @ W0[0].T + W0[1], 0))
    cmp("r", lrn.debug("r")[:B], rr)
    cmp("d", lrn.debug("d")[:B], d)

for args in [(3, 1, 64, 2, 256, 10000), (22, 6, 256, 2, 256, 20000), (22, 6, 256, 2, 1000, 20000), (3, 1, 64, 2, 1000, 10000)]:
    print("==", args); run(*args, "fp32")
