"""Step-0 intermediates of the TD3 / SAC update on the GPU against the oracle (diagnosis of the bf16
critic-gradient error): target action a', target critics, y, online q, g_q."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synthdata  # noqa: E402
from oracle import mlp, sac as osac, td3 as otd3  # noqa: E402
from tests.parity import make_rings  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402


def rel(x, y):
    return float(np.linalg.norm(np.asarray(x, np.float64) - y) / max(np.linalg.norm(y), 1e-30))


def main(algo, prec, o, m, h, L, B):
    g, r = make_rings(o, m, 8000)
    p = synthdata.init_params(o, m, h, L, algo=algo)
    lrn = spz.Learner(g, algo=algo, precision=prec, hidden=h, n_hidden=L, max_batch=B)
    for n in ("actor", "q1", "q2"):
        lrn.set(n, p[n])
    lrn.set("q1_targ", p["q1"])
    lrn.set("q2_targ", p["q2"])
    if algo == "td3":
        lrn.set("actor_targ", p["actor"])
    lrn.update(B, 1)
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L, alpha_auto=algo == "sac")
    idx, batch = r.sample(B, synthdata.SAMPLE_SEED, 0)
    s, a, rr, s2, d = osac._batch_f64(batch)
    cs = osac.critic_shapes(cfg)
    if algo == "td3":
        xi = otd3.draw_smoothing(synthdata.SAMPLE_SEED, 0, B, cfg)
        z2, _ = mlp.forward(mlp.unflatten(p["actor"].astype(np.float64), osac.actor_shapes(cfg, td3=True)), s2)
        a2 = np.clip(np.tanh(z2) + xi, -1, 1)
        lp2 = np.zeros(B)
    else:
        eps, eps2 = osac.draw_noise(synthdata.SAMPLE_SEED, 0, B, m)
        a2, lp2, _, _ = osac.policy_forward(mlp.unflatten(p["actor"].astype(np.float64), osac.actor_shapes(cfg)), s2, eps2, cfg)
    qt1, _ = osac.critic_q(mlp.unflatten(p["q1"].astype(np.float64), cs), s2, a2)
    qt2, _ = osac.critic_q(mlp.unflatten(p["q2"].astype(np.float64), cs), s2, a2)
    alpha = 0.0 if algo == "td3" else 0.2
    y = rr + cfg.gamma * (1 - d) * (np.minimum(qt1, qt2) - alpha * lp2)
    q1, _ = osac.critic_q(mlp.unflatten(p["q1"].astype(np.float64), cs), s, a)
    ldc = lrn.debug("Xc").size // (3 * B)
    Xc = lrn.debug("Xc").reshape(3 * B, ldc) if lrn.debug("Xc").size == 3 * B * ldc else None
    dy = lrn.debug("y")[:B]
    print(algo, prec, "y rel", rel(dy, y), "y-r rel", rel(dy - rr, y - rr))
    qt_g = lrn.debug("q_tg0")
    print("  q_tg0 plane0 rel", rel(qt_g[:B], qt1), "q_tg1", rel(lrn.debug("q_tg1")[:B], qt2))
    print("  q_on0 rel", rel(lrn.debug("q_on0")[:B], q1))
    gq = lrn.debug("gq0")[:B]
    print("  gq0 rel", rel(gq, 2 * (q1 - y) / B))
    if Xc is not None:
        print("  Xc s2|a' block a' rel", rel(Xc[2 * B:3 * B, o:o + m], a2), "Xc s|a", rel(Xc[:B, :o], s))


if __name__ == "__main__":
    main("td3", "bf16", 44, 17, 128, 3, 600)
    main("td3", "fp32", 44, 17, 128, 3, 600)
    main("sac", "bf16", 44, 17, 128, 3, 600)
