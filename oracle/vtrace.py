"""V-trace and N-step returns, plain and slow.

TEST INFRASTRUCTURE ONLY: only tests/ and bench.py may import this module; the product path
never does.  Float64 numpy, one trajectory at a time, written from the paper in its notation
(PAPER.md P:760-851).  Arrays are time-major [T][B] like the kernel's; each function loops over
the B trajectories.

Terminal handling (R#33): the paper's equations have no terminals.  A terminal at
step t sets that step's discount to zero: gamma_t = gamma * (1 - done_t).  That truncates the
bootstrapped return at the terminal ("bootstrap replaced by 0"), and with no
terminals gamma_t = gamma reproduces the paper's gamma^(t - t0).
"""
from __future__ import annotations

import numpy as np


def nstep_return(rewards, bootstrap, gamma, dones):
    """R~_t = sum_{i<k} gamma^i r_{t+i} + gamma^k V(s_{t+k}) to the end of the window,
    stopping at a terminal: R~_t = r_t + gamma_t R~_{t+1} written out as an explicit sum."""
    r = np.asarray(rewards, np.float64)
    T, B = r.shape
    d = np.asarray(dones).astype(bool)
    out = np.zeros((T, B))
    for b in range(B):
        for t in range(T):
            total, disc = 0.0, 1.0
            ended = False
            for i in range(t, T):
                total += disc * r[i, b]
                if d[i, b]:
                    ended = True
                    break
                disc *= gamma
            if not ended:
                total += disc * float(bootstrap[b])
            out[t, b] = total
    return out


def _weights(log_mu, log_pi, rho_bar, c_bar):
    ratio = np.exp(np.asarray(log_pi, np.float64) - np.asarray(log_mu, np.float64))
    return np.minimum(rho_bar, ratio), np.minimum(c_bar, ratio)  # Eqs. rho, c


def vtrace_direct(rewards, values, bootstrap, log_mu, log_pi, dones, gamma, rho_bar, c_bar):
    """Eq. target.off by explicit double summation, for every start step s:
    v_s = V(s_s) + sum_{t=s}^{T-1} (prod_{i=s}^{t-1} gamma_i c_i) delta_t V,
    delta_t V = rho_t (r_t + gamma_t V(s_{t+1}) - V(s_t)),  V(s_T) = bootstrap.
    Returns (vs, rho, advantages r_t + gamma_t v_{t+1} - V(s_t), v_T = bootstrap)."""
    r = np.asarray(rewards, np.float64)
    V = np.asarray(values, np.float64)
    T, B = r.shape
    rho, c = _weights(log_mu, log_pi, rho_bar, c_bar)
    g = np.where(np.asarray(dones).astype(bool), 0.0, float(gamma))
    Vn = np.vstack([V[1:], np.asarray(bootstrap, np.float64)[None, :]])  # V(s_{t+1})
    vs = np.zeros((T, B))
    for b in range(B):
        for s in range(T):
            total = V[s, b]
            for t in range(s, T):
                prod = 1.0
                for i in range(s, t):
                    prod *= g[i, b] * c[i, b]
                delta = rho[t, b] * (r[t, b] + g[t, b] * Vn[t, b] - V[t, b])
                total += prod * delta
            vs[s, b] = total
    vnext = np.vstack([vs[1:], np.asarray(bootstrap, np.float64)[None, :]])
    adv = r + g * vnext - V  # policy-gradient advantage
    return vs, rho, adv


def vtrace_recursive(rewards, values, bootstrap, log_mu, log_pi, dones, gamma, rho_bar, c_bar):
    """The paper's recursive form: v_t = V(s_t) + delta_t V + gamma_t c_t (v_{t+1} -
    V(s_{t+1})), v_T = V(s_T) = bootstrap; same outputs as vtrace_direct."""
    r = np.asarray(rewards, np.float64)
    V = np.asarray(values, np.float64)
    T, B = r.shape
    rho, c = _weights(log_mu, log_pi, rho_bar, c_bar)
    g = np.where(np.asarray(dones).astype(bool), 0.0, float(gamma))
    vs = np.zeros((T, B))
    adv = np.zeros((T, B))
    for b in range(B):
        v_next = V_next = float(bootstrap[b])
        for t in range(T - 1, -1, -1):
            delta = rho[t, b] * (r[t, b] + g[t, b] * V_next - V[t, b])
            vs[t, b] = V[t, b] + delta + g[t, b] * c[t, b] * (v_next - V_next)
            adv[t, b] = r[t, b] + g[t, b] * v_next - V[t, b]
            v_next, V_next = vs[t, b], V[t, b]
    return vs, rho, adv
