"""Replay ring model (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows SPEC ReplayRing: monotone 64-bit cursor, fill =
min(cursor, C), slot for global index i is i mod C; push returns the global
index of its first record ("push onto empty ring -> index 0");
capacity 0 is an error; sampling is uniform with replacement over the
valid slots using ``philox.sample_indices``; sampling with
fill < B signals "not enough data".

Record layout:  one fp32 record per transition,
``[s | a | r | d | s2 | pad]`` padded to a multiple of 4 floats (16 B).
Transition fields per P:243 ("state s, action a, next state s2, reward r, and
done flag d").
"""

import numpy as np

from . import philox


def record_floats(obs_dim, act_dim):
    """R = round_up(2*o + m + 2, 4) floats."""
    n = 2 * obs_dim + act_dim + 2
    return (n + 3) // 4 * 4


class NotEnoughData(Exception):
    pass


class Ring:
    def __init__(self, obs_dim, act_dim, capacity):
        if capacity <= 0:
            raise ValueError("capacity must be positive (S:193)")
        if obs_dim < 1 or act_dim < 1:
            raise ValueError("dims must be >= 1")
        self.o, self.m, self.C = obs_dim, act_dim, int(capacity)
        self.R = record_floats(obs_dim, act_dim)
        self.records = np.zeros((self.C, self.R), dtype=np.float32)
        self.cursor = 0

    @property
    def fill(self):
        return min(self.cursor, self.C)

    def pack(self, obs, act, rew, next_obs, done):
        o, m = self.o, self.m
        n = len(rew)
        rec = np.zeros((n, self.R), dtype=np.float32)
        rec[:, 0:o] = obs
        rec[:, o:o + m] = act
        rec[:, o + m] = rew
        rec[:, o + m + 1] = done
        rec[:, o + m + 2:2 * o + m + 2] = next_obs
        return rec

    def push(self, obs, act, rew, next_obs, done):
        """Append n transitions; returns the global index of the first one."""
        rec = self.pack(obs, act, rew, next_obs, done)
        first = self.cursor
        n = rec.shape[0]
        keep = min(n, self.C)  # only the last C records of a push survive
        g = np.arange(first + n - keep, first + n)  # their global indices
        self.records[g % self.C] = rec[n - keep:]
        self.cursor += n
        return first

    def unpack(self, rows):
        o, m = self.o, self.m
        return dict(
            obs=rows[:, 0:o],
            act=rows[:, o:o + m],
            rew=rows[:, o + m],
            done=rows[:, o + m + 1],
            next_obs=rows[:, o + m + 2:2 * o + m + 2],
        )

    def sample(self, batch, seed, step, row0=0, global_batch=None):
        """Indices and fp32 rows of global rows row0..row0+batch-1 at step k.

        ``global_batch`` (default ``batch``) is the B the fill is checked
        against ("fill count >= B").
        """
        F = self.fill
        gb = batch if global_batch is None else global_batch
        if F < gb:
            raise NotEnoughData(f"fill {F} < batch {gb}")
        idx = philox.sample_indices(seed, step, F, batch, row0=row0)
        return idx, self.unpack(self.records[idx])
