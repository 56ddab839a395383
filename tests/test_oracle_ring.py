"""Pins for oracle/ring.py (replay ring indexing and sampling)."""

import itertools

import numpy as np
import pytest

from oracle import ring as oring


def _tr(n, o=3, m=1, tag0=0):
    t = np.arange(tag0, tag0 + n, dtype=np.float32)
    return dict(obs=np.tile(t[:, None], (1, o)), act=np.tile(-t[:, None], (1, m)), rew=t,
                next_obs=np.tile(t[:, None] + 0.5, (1, o)), done=(t % 2).astype(np.float32))


def test_capacity_zero_is_error():
    with pytest.raises(ValueError):
        oring.Ring(3, 1, 0)


def test_record_layout_and_roundtrip():
    assert oring.record_floats(3, 1) == 12 and oring.record_floats(22, 6) == 52
    assert oring.record_floats(28, 8) == 68 and oring.record_floats(44, 17) == 108
    r = oring.Ring(3, 1, 10)
    tr = _tr(4)
    r.push(**tr)
    back = r.unpack(r.records[:4])
    for k in tr:
        assert np.array_equal(back[k], tr[k])


def test_first_push_and_wraparound():
    r = oring.Ring(3, 1, 5)
    assert r.push(**_tr(1)) == 0 and r.fill == 1
    r = oring.Ring(3, 1, 5)
    for i in range(6):  # C+1 pushes
        r.push(**_tr(1, tag0=i))
    assert r.fill == 5 and r.cursor == 6
    assert r.unpack(r.records[0:1])["rew"][0] == 5.0  # slot 0 holds record C


def test_brute_force_push_sequences():
    """All push-size sequences for small C: readable set == last min(cursor, C) records."""
    for C in range(1, 6):
        for seq in itertools.product(range(1, C + 2), repeat=3):
            r = oring.Ring(3, 1, C)
            log = []
            tag = 0
            for n in seq:
                first = r.push(**_tr(n, tag0=tag))
                assert first == tag
                log.extend(range(tag, tag + n))
                tag += n
            assert r.fill == min(len(log), C)
            live = log[-C:]
            for g in live:
                assert r.records[g % C][4] == float(g)  # reward column (o+m) carries the tag


def test_sample_fill_one_and_not_enough_data():
    r = oring.Ring(3, 1, 8)
    r.push(**_tr(1, tag0=42))
    idx, b = r.sample(1, 6126, 0)
    assert idx[0] == 0 and b["rew"][0] == 42
    with pytest.raises(oring.NotEnoughData):
        r.sample(2, 6126, 0)


def test_sample_repeatable_and_gathers_rows():
    r = oring.Ring(3, 1, 100)
    r.push(**_tr(100))
    i1, b1 = r.sample(64, 9, 3)
    i2, b2 = r.sample(64, 9, 3)
    assert np.array_equal(i1, i2) and np.array_equal(b1["obs"], b2["obs"])
    assert np.array_equal(b1["rew"], i1.astype(np.float32))  # row tag == slot here


# ----------------------------------------------------------------------------- transmission loss

def _trl(n, o=2, m=1, seed=0):
    import synthdata
    return synthdata.transitions("locomotion", o, m, n, seed=seed)


def test_loss_no_sampling_capacity_100_ten_thousand_pushes():
    # capacity-100 ring, 10^4 pushes, no sampling -> loss 9900 / 10^4 = 99 %
    r = oring.Ring(2, 1, 100)
    r.track()
    for k in range(100):
        r.push(**_trl(100, seed=k))
    pushed, lost, resident, sampled = r.loss_stats()
    assert (pushed, lost, resident, sampled) == (10_000, 9_900, 100, 0)


def test_loss_conservation_and_brute_force():
    # brute force over push sizes (including pushes longer than C) with interleaved sampling: a plain
    # per-record tag model (every pushed record's fate tracked individually) gives the same counts
    rng = np.random.default_rng(3)
    for C in (1, 3, 8):
        r = oring.Ring(2, 1, C)
        r.track()
        fate = {}          # global index -> "resident" | "lost" | "sampled"
        slot_owner = {}    # slot -> global index resident there
        g = 0
        for step in range(40):
            n = int(rng.integers(0, 3 * C + 1))
            r.push(**_trl(n, seed=step))
            for gi in range(g, g + n):
                s = gi % C
                prev = slot_owner.get(s)
                if prev is not None and fate[prev] == "resident":
                    fate[prev] = "lost"
                if prev is not None and fate[prev] == "sampled_resident":
                    fate[prev] = "sampled"
                slot_owner[s] = gi
                fate[gi] = "resident"
            g += n
            if r.fill and rng.random() < 0.5:
                B = int(rng.integers(1, r.fill + 1))
                idx, _ = r.sample(B, 7, step)
                for s in idx:
                    gi = slot_owner[int(s)]
                    if fate[gi] == "resident":
                        fate[gi] = "sampled_resident"
        pushed, lost, resident, sampled = r.loss_stats()
        assert pushed == g == lost + resident + sampled
        assert lost == sum(v == "lost" for v in fate.values())
        assert resident == sum(v == "resident" for v in fate.values())
