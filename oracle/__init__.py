"""CPU float64 oracle for the Spreeze (arXiv 2312.06126) network-update hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2312_06126_b200``) never imports it and the
two share no code: no kernels, headers, helpers, constants or pre/post
processing.  The only module both sides consume is ``synthdata`` (seeded input
generators, none of the method's arithmetic).

What it computes (PAPER.md = ``P:n``, SPEC.md = ``S:n``):

* ``philox``   -- Philox4x32-10 counter-based generator (random numbers the method
                  draws: replay indices, reparameterisation noise, TD3 smoothing
                  noise).  Both sides implement the same generator independently.
* ``ring``     -- replay ring model: slot = i mod C, fill = min(cursor, C), uniform
                  sampling with replacement.
* ``mlp``      -- dense ReLU MLP forward and manual reverse-mode backward
                  (S:46-63).
* ``sac``      -- one SAC update step, Jacobi order, float64 (§8(c)).
* ``td3``      -- one TD3 update step (Fujimoto et al.), Jacobi order.
* ``ddpg``     -- one DDPG update step, single critic, Jacobi order.
* ``sacv1``    -- one SAC v1 update step (state-value network + target V; §8(f) f4), Jacobi order.
* ``optim``    -- Adam and Polyak averaging.
* ``act``      -- sampler-side action selection from a synced actor (
                  SURVEY.md §8(f) f1): deterministic tanh(mu) / stochastic reparameterised
                  sample (SAC), tanh + clipped Gaussian exploration (TD3).
* ``schedules``-- the actor/critic split schedule and the G-way row
                  sharded schedule, both reorganisations of the
                  single schedule.

Every function is pinned by a ``-m "not gpu"`` test in ``tests/test_oracle_*.py``
against something other than itself (Random123 KATs, closed forms, finite
differences, torch.autograd in float64, quadrature, brute force).  The paper's
own hyper-parameters and the tensor set of its missing Fig. 3 are
"parity unpinned" (the paper is silent).
"""

from . import philox, ring, mlp, optim, sac, td3, schedules  # noqa: F401
