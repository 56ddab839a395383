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
