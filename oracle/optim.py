"""Adam and Polyak averaging, float64 (oracle side).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Adam (reading #11): per-optimizer step counter t,
  m <- b1 m + (1-b1) g ;  v <- b2 v + (1-b2) g^2 ;
  theta <- theta - lr * (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps)
with eps added to sqrt(v_hat) (the PyTorch form), no weight decay, no
clipping.

Polyak ("target network"): theta' <- tau theta + (1-tau) theta'.

Pinned by tests/test_oracle_optim.py: zero gradient leaves parameters
unchanged and t+1; one step from a fresh state moves by
-lr g/(|g|+eps); constant gradient gives the same step every time;
1000 steps on x^2 at lr 1e-2 reach |x| < 0.05; tau = 0 / 1 and the
frozen-theta geometric decay (1-tau)^n.
"""

import numpy as np


class AdamState:
    def __init__(self, n):
        self.m = np.zeros(n, dtype=np.float64)
        self.v = np.zeros(n, dtype=np.float64)
        self.t = 0

    def copy(self):
        s = AdamState(0)
        s.m, s.v, s.t = self.m.copy(), self.v.copy(), self.t
        return s


def adam_step(theta, g, st, lr, b1=0.9, b2=0.999, eps=1e-8):
    """Returns the new parameter vector; updates ``st`` in place."""
    g = np.asarray(g, dtype=np.float64)
    st.t += 1
    st.m = b1 * st.m + (1.0 - b1) * g
    st.v = b2 * st.v + (1.0 - b2) * g * g
    m_hat = st.m / (1.0 - b1 ** st.t)
    v_hat = st.v / (1.0 - b2 ** st.t)
    return np.asarray(theta, dtype=np.float64) - lr * m_hat / (np.sqrt(v_hat) + eps)


def polyak(target, online, tau):
    return tau * np.asarray(online, dtype=np.float64) + (1.0 - tau) * np.asarray(target, dtype=np.float64)
