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
        self.tags = None  # transmission-loss accounting (track())

    # ---- experience transmission loss (Table 3 column): the share of
    #      pushed records overwritten before ever being sampled.  Every resident record carries a
    #      "sampled" tag; a landing record that overwrites an unsampled one counts it as lost, and so does
    #      a record that never lands (a push longer than C keeps only its last C records).
    def track(self):
        self.tags = np.zeros(self.C, dtype=bool)
        self.lost = 0
        self.pushed0 = self.cursor  # pushes before tracking started are not accounted

    def loss_stats(self):
        """(pushed, lost, resident_unsampled, sampled) since track(); pushed = lost + resident_unsampled + sampled."""
        pushed = self.cursor - self.pushed0
        occ = np.arange(self.C) < self.fill
        # resident records pushed before track() are not counted as pushed
        first_tracked = max(self.pushed0, self.cursor - self.C)
        g_slot = np.arange(self.C)
        resident = 0
        for s in g_slot[occ]:
            g = self._global_of_slot(s)
            if g >= first_tracked and not self.tags[s]:
                resident += 1
        return pushed, self.lost, resident, pushed - self.lost - resident

    def _global_of_slot(self, s):
        """Global index of the record resident in slot s (the most recent g with g mod C = s, g < cursor)."""
        c = self.cursor
        return (c - 1) - ((c - 1 - s) % self.C)

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
        if self.tags is not None:
            self.lost += n - keep  # never resident
            occupied = min(first, self.C)  # slots holding a record before this push
            for s in np.unique(g % self.C):
                if s < occupied:
                    old = (first - 1) - ((first - 1 - s) % self.C)  # the record about to be overwritten
                    if old >= self.pushed0 and not self.tags[s]:
                        self.lost += 1
            self.tags[g % self.C] = False
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
        if self.tags is not None:
            self.tags[idx] = True
        return idx, self.unpack(self.records[idx])
