"""Fixtures restating proj/tests/testutil.hpp:21-84 on top of the oracle's RNG.

random_model / simulate_obs draw from the same counter streams as the
reference's test utilities, so model instances are reproducible by seed.
"""
from __future__ import annotations

import numpy as np

from oracle import pyoracle as O


def random_spd(s, d, scale=1.0):
    g = np.stack([O.normal_vec(s, d) for _ in range(d)])
    return scale * (g @ g.T / d + 0.2 * np.eye(d))


def random_mat(s, rows, cols, scale=1.0):
    return np.stack([scale * O.normal_vec(s, cols) for _ in range(rows)])


def random_model(s, T, dx, dy, time_varying=False, with_mask=False):
    """testutil.hpp:35-68"""
    m0 = O.normal_vec(s, dx)
    p0 = random_spd(s, dx)
    n_dyn = max(T, 1) if time_varying else 1
    n_obs = T + 1 if time_varying else 1
    F, b, Q, H, c, R = [], [], [], [], [], []
    for _ in range(n_dyn):
        F.append(random_mat(s, dx, dx, 0.6 / np.sqrt(dx)))
        b.append(0.3 * O.normal_vec(s, dx))
        Q.append(random_spd(s, dx, 0.5))
    for _ in range(n_obs):
        H.append(random_mat(s, dy, dx))
        c.append(0.3 * O.normal_vec(s, dy))
        R.append(random_spd(s, dy, 0.5))
    mask = None
    if with_mask:
        mask = np.ones(T + 1, np.uint8)
        for t in range(T + 1):
            if O.next_uniform(s) < 0.33:
                mask[t] = 0
        mask[0] = 1
    return O.Model(T, m0, p0, np.array(F), np.array(b), np.array(Q), np.array(H), np.array(c),
                   np.array(R), mask)


def simulate_obs(m, s0):
    """testutil.hpp:71-84"""
    s = O.derive(s0, O.L_SIMULATE, 0)
    obs = np.zeros((m.T + 1, m.dy))
    x = m.m0 + O.chol_psd(m.P0) @ O.normal_vec(s, m.dx)
    for t in range(m.T + 1):
        if t > 0:
            i = t - 1 if m.F.shape[0] > 1 else 0
            j = t - 1 if m.Q.shape[0] > 1 else 0
            k = t - 1 if m.b.shape[0] > 1 else 0
            x = m.F[i] @ x + m.b[k] + O.chol_psd(m.Q[j]) @ O.normal_vec(s, m.dx)
        h = t if m.H.shape[0] > 1 else 0
        obs[t] = m.H[h] @ x + m.c[t if m.c.shape[0] > 1 else 0] + \
            O.chol_psd(m.R[t if m.R.shape[0] > 1 else 0]) @ O.normal_vec(s, m.dy)
    return obs


def to_gpu_model(m, device="cuda"):
    from paper_2303_00301_b200 import lgssm
    return lgssm.Model(m.T, m.m0, m.P0, m.F, m.b, m.Q, m.H, m.c, m.R, m.mask, device=device)


def predrawn(rng, B, T, dx, n_bridge=0):
    """Independent pre-drawn variates per path (numpy generator; the parity
    contract is identical variates on both sides, not identical streams)."""
    term = rng.standard_normal((B, dx))
    back = rng.standard_normal((B, max(T, 1), dx))
    bridge = rng.standard_normal((B, n_bridge, dx)) if n_bridge else None
    return term, back, bridge
