"""Experience transmission loss on the device ring against the
oracle ring's tag model: exact integer counts, with pushes from host / pinned / device memory and the
learner's own sampling marking the tags."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synthdata  # noqa: E402
from oracle import ring as oring  # noqa: E402
from paper_2312_06126_b200 import spz  # noqa: E402


def test_loss_capacity_100_no_sampling():
    g = spz.Replay(2, 1, 100)
    g.track()
    for k in range(100):
        g.push(**synthdata.transitions("locomotion", 2, 1, 100, seed=k))
    assert g.loss() == (10_000, 9_900, 100)


@pytest.mark.parametrize("src", ["host", "pinned", "device"])
def test_loss_matches_oracle_with_learner_sampling(src):
    o, m, C, B = 22, 6, 3000, 512
    g = spz.Replay(o, m, C)
    r = oring.Ring(o, m, C)
    first = synthdata.transitions("locomotion", o, m, C)
    g.push(**first)
    r.push(**first)
    g.track()
    r.track()
    lrn = spz.Learner(g, precision="bf16", hidden=64, n_hidden=2, max_batch=B)
    rng = np.random.default_rng(0)
    for k in range(12):
        n = int(rng.integers(0, 2 * C))  # sometimes longer than the ring
        tr = synthdata.transitions("locomotion", o, m, n, seed=50 + k)
        r.push(**tr)
        if src == "pinned":
            tr = {a: torch.from_numpy(v).pin_memory().numpy() for a, v in tr.items()}
        if src == "device" and n:
            g.push(**{a: torch.from_numpy(v).cuda() for a, v in tr.items()}, src_on_device=True)
        else:
            g.push(**tr)
        lrn.update(B, 1)                      # samples spz_replay_sample(ring, B, seed, k)
        r.sample(B, synthdata.SAMPLE_SEED, k)  # the same indices mark the oracle's tags
    pushed, lost, resident, _ = r.loss_stats()
    assert g.loss() == (pushed, lost, resident)
    assert lost > 0 and resident > 0


def test_track_errors_and_restart():
    g = spz.Replay(3, 1, 50)
    with pytest.raises(spz.SpzError) as e:
        g.loss()
    assert e.value.status == spz.SPZ_ESTATE
    g.push(**synthdata.transitions("pendulum", 3, 1, 80))
    g.track()
    assert g.loss() == (0, 0, 0)  # records pushed before tracking are not accounted
    g.push(**synthdata.transitions("pendulum", 3, 1, 10))
    assert g.loss() == (10, 0, 10)
    g.track(False)
    with pytest.raises(spz.SpzError):
        g.loss()


def test_push_async_matches_sync_and_buffer_contract():
    """spz_replay_push_async: the same records as spz_replay_push (gathered rows bit-identical to the oracle
    ring); a pinned buffer may be overwritten once the NEXT push returns (two alternating sets suffice), and
    spz_replay_sync covers the last one."""
    torch = pytest.importorskip("torch")
    o, m, C, n = 5, 2, 4096, 700
    tr = [synthdata.transitions("locomotion", o, m, n, seed=100 + i) for i in range(6)]
    bufs = [{k: torch.from_numpy(v.copy()).pin_memory().numpy() for k, v in tr[0].items()} for _ in range(2)]
    g = spz.Replay(o, m, C)
    r = oring.Ring(o, m, C)
    for i in range(6):
        b = bufs[i % 2]
        for k in b:
            b[k][...] = tr[i][k]  # refill: the push that used this set two pushes ago has returned since
        first = g.push(**b, wait=False)
        assert first == r.push(**tr[i])
    g.sync()
    for b in bufs:  # after sync every buffer may change without touching the ring
        for k in b:
            b[k][...] = -7.0
    B = 512
    idx = torch.empty(B, dtype=torch.int32, device="cuda")
    obs = torch.empty(B, o, device="cuda")
    act = torch.empty(B, m, device="cuda")
    rew = torch.empty(B, device="cuda")
    nobs = torch.empty(B, o, device="cuda")
    done = torch.empty(B, device="cuda")
    spz.spz_replay_sample(g.h, B, synthdata.SAMPLE_SEED, 3, idx, obs, act, rew, nobs, done)
    ridx, rb = r.sample(B, synthdata.SAMPLE_SEED, 3)
    assert np.array_equal(idx.cpu().numpy(), ridx)
    for name, t in (("obs", obs), ("act", act), ("rew", rew), ("next_obs", nobs), ("done", done)):
        assert np.array_equal(t.cpu().numpy(), rb[name]), name


def test_update_with_async_pushes_bit_identical():
    """An update loop fed by spz_replay_push_async equals the same loop fed by spz_replay_push."""
    torch = pytest.importorskip("torch")
    o, m, B = 22, 6, 1024
    outs = []
    for wait in (True, False):
        g = spz.Replay(o, m, 20_000)
        g.push(**synthdata.transitions("locomotion", o, m, 8000))
        lrn = spz.Learner(g, precision="bf16", hidden=64, n_hidden=2, max_batch=B)
        host = synthdata.transitions("locomotion", o, m, 4 * B, seed=77)
        pinned = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in host.items()}
        for k in range(6):
            sl = slice((k % 4) * B, (k % 4 + 1) * B)
            g.push(**{n: v[sl] for n, v in pinned.items()}, wait=wait)
            if k >= 2:
                lrn.wait()
            lrn.update_async(B, 1)
        lrn.wait()
        lrn.wait()
        g.sync()
        outs.append([lrn.get(n) for n in ("actor", "q1", "q2")])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
