"""Sampler-side policy: spz_policy_act against oracle/act.py on the actor a learner
publishes with spz_sync_actor; deterministic and stochastic, SAC and TD3, bf16 and 3xTF32."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthdata  # noqa: E402
from oracle import act as oact, sac as osac  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402

TOL = {"fp32": 1e-4, "bf16": 2e-2}


def rel(x, ref):
    return float(np.linalg.norm(np.asarray(x, np.float64) - ref) / max(np.linalg.norm(ref), 1e-30))


def publish(algo, precision, o, m, h, L, steps=2):
    g = spz.Replay(o, m, 4000)
    g.push(**synthdata.transitions("locomotion", o, m, 4000))
    lrn = spz.Learner(g, algo=algo, precision=precision, hidden=h, n_hidden=L, max_batch=512)
    if steps:
        lrn.update(512, steps)
    n = lrn.get("actor").size
    buf = torch.zeros(spz.sync_bytes(n), dtype=torch.uint8, device="cuda")
    v = spz.spz_sync_actor(lrn.h, 0, buf.data_ptr(), buf.numel())
    return lrn, buf, v


@pytest.mark.parametrize("algo,precision,o,m,h,L", [
    ("sac", "bf16", 22, 6, 256, 2), ("sac", "fp32", 22, 6, 256, 2), ("td3", "bf16", 44, 17, 128, 3),
    ("td3", "fp32", 44, 17, 128, 3), ("sac", "bf16", 3, 1, 64, 2), ("sac", "bf16", 44, 17, 512, 3)])
@pytest.mark.parametrize("deterministic", [True, False])
def test_policy_matches_oracle(algo, precision, o, m, h, L, deterministic):
    lrn, buf, v = publish(algo, precision, o, m, h, L)
    pol = spz.Policy(o, m, algo=algo, precision=precision, hidden=h, n_hidden=L, max_batch=1000)
    assert pol.load(buf.data_ptr(), buf.numel()) == v
    cfg = osac.Config(obs_dim=o, act_dim=m, hidden=h, n_hidden=L)
    actor = lrn.get("actor").astype(np.float64)
    for n, seed, step in ((1, 3, 0), (37, 5, 11), (1000, 7, 123456789)):
        s = np.clip(np.random.default_rng(n).normal(size=(n, o)), -5, 5).astype(np.float32)
        got = pol.act(s, deterministic=deterministic, seed=seed, step=step)
        ref = oact.act(actor, s, cfg, algo=algo, deterministic=deterministic, seed=seed, step=step)
        assert got.shape == (n, m)
        assert rel(got, ref) <= TOL[precision], (n, rel(got, ref))
        assert np.all(np.abs(got) <= 1.0)


def test_policy_device_buffers_and_versions():
    o, m, h, L = 22, 6, 64, 2
    g = spz.Replay(o, m, 3000)
    g.push(**synthdata.transitions("locomotion", o, m, 3000))
    lrn = spz.Learner(g, precision="bf16", hidden=h, n_hidden=L, max_batch=256)
    n = lrn.get("actor").size
    buf = torch.zeros(spz.sync_bytes(n), dtype=torch.uint8, device="cuda")
    pol = spz.Policy(o, m, hidden=h, n_hidden=L, max_batch=300)
    s = np.random.default_rng(0).normal(size=(300, o)).astype(np.float32)
    with pytest.raises(spz.SpzError) as e:
        pol.act(s)
    assert e.value.status == spz.SPZ_ESTATE
    with pytest.raises(spz.SpzError) as e:  # nothing published yet
        pol.load(buf.data_ptr(), buf.numel())
    assert e.value.status == spz.SPZ_ESTATE
    v1 = spz.spz_sync_actor(lrn.h, 0, buf.data_ptr(), buf.numel())
    assert pol.load(buf.data_ptr(), buf.numel()) == v1
    a1 = pol.act(s, deterministic=True)
    lrn.update(256, 3)
    v2 = spz.spz_sync_actor(lrn.h, 0, buf.data_ptr(), buf.numel())
    # a host copy of the payload loads the same way
    host = buf.cpu().numpy()
    assert pol.load(host.ctypes.data, host.nbytes) == v2 == v1 + 1
    a2 = pol.act(s, deterministic=True)
    assert not np.array_equal(a1, a2)  # the new actor is in use
    # device observations and device actions give the host result bit for bit
    sd = torch.from_numpy(s).cuda()
    ad = torch.empty(300, m, device="cuda")
    spz.spz_policy_act(pol.h, 300, sd, True, 0, 0, ad)
    assert np.array_equal(ad.cpu().numpy(), a2)
    # shape mismatch and oversize batches are rejected
    small = spz.Policy(o, m, hidden=32, n_hidden=L, max_batch=10)
    with pytest.raises(spz.SpzError) as e:
        small.load(buf.data_ptr(), buf.numel())
    assert e.value.status == spz.SPZ_EINVAL
    with pytest.raises(spz.SpzError):
        pol.act(np.zeros((301, o), np.float32))


def test_sync_actor_concurrent_publish_never_blends():
    """a10/f1 stress (S:259 never a blend, S:271 monotone): one thread publishes thousands of versions of a
    large actor (3x1024, 8.6 MB per slot), each version a constant vector of its own value, while another
    thread loads on its own stream; every load must be exactly one published version's payload, and the
    versions a reader sees never go backwards."""
    import threading
    o, m, h, L = 44, 17, 1024, 3
    g = spz.Replay(o, m, 1000)
    g.push(**synthdata.transitions("locomotion", o, m, 1000))
    lrn = spz.Learner(g, algo="td3", precision="bf16", hidden=h, n_hidden=L, max_batch=256)
    n = lrn.get("actor").size
    buf = torch.zeros(spz.sync_bytes(n), dtype=torch.uint8, device="cuda")
    pol = spz.Policy(o, m, algo="td3", hidden=h, n_hidden=L, max_batch=16)
    N = 2000
    pats = [np.full(n, float(i + 1), np.float32) for i in range(2)]
    ver_val = {}
    done = threading.Event()
    errors = []

    def writer():
        try:
            for i in range(N):
                val = float(i + 1)
                pats[i % 2].fill(val)
                lrn.set("actor", pats[i % 2])
                v = spz.spz_sync_actor(lrn.h, 0, buf.data_ptr(), buf.numel())
                ver_val[v] = val
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)
        finally:
            done.set()

    loads, last = [], 0
    t = threading.Thread(target=writer)
    t.start()
    while not done.is_set() or len(loads) < 20:
        try:
            v = pol.load(buf.data_ptr(), buf.numel())
        except spz.SpzError as e:
            if e.status == spz.SPZ_ESTATE:  # before the first publication
                continue
            raise
        p = pol.params(n)
        assert v >= last, (v, last)
        last = v
        loads.append((v, float(p[0]), bool(np.all(p == p[0]))))
        if done.is_set() and len(loads) >= 20:
            break
    t.join()
    assert not errors, errors
    assert len(ver_val) == N
    for v, first, uniform in loads:
        assert uniform, ("blend", v)
        assert first == ver_val[v], (v, first, ver_val[v])
    assert len({v for v, _, _ in loads}) > 10  # the reader really overlapped many publications
