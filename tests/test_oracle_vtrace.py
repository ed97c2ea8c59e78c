"""Pins for the V-trace / N-step oracle (oracle/vtrace.py): the SPEC's
worked examples, the paper's two forms against each other, the on-policy reduction to the
N-step return, the truncation clamps and monotonicity."""
import numpy as np

from oracle import vtrace as VT


def rand_traj(rng, T, B, p_done=0.1):
    return dict(rewards=rng.normal(size=(T, B)), values=rng.normal(size=(T, B)), bootstrap=rng.normal(size=B),
                log_mu=rng.normal(scale=0.5, size=(T, B)), log_pi=rng.normal(scale=0.5, size=(T, B)),
                dones=(rng.random((T, B)) < p_done).astype(np.uint8))


def test_spec_nstep_examples():
    # r=(1,2), V(s2)=10, gamma=0.5 -> 1 + 0.5*2 + 0.25*10 = 4.5
    R = VT.nstep_return([[1.0], [2.0]], [10.0], 0.5, [[0], [0]])
    assert R[0, 0] == 4.5 and R[1, 0] == 2.0 + 0.5 * 10.0
    # gamma = 1, zero rewards -> the bootstrap value
    assert (VT.nstep_return(np.zeros((5, 1)), [3.25], 1.0, np.zeros((5, 1))) == 3.25).all()
    # terminal at step 0 -> r_0
    assert VT.nstep_return([[1.5], [7.0]], [9.0], 0.9, [[1], [0]])[0, 0] == 1.5


def test_on_policy_reduces_to_nstep_return():
    rng = np.random.default_rng(1)
    tr = rand_traj(rng, 12, 6)
    tr["log_pi"] = tr["log_mu"].copy()  # mu = pi
    R = VT.nstep_return(tr["rewards"], tr["bootstrap"], 0.97, tr["dones"])
    for f in (VT.vtrace_direct, VT.vtrace_recursive):
        vs, rho, _ = f(**tr, gamma=0.97, rho_bar=1.0, c_bar=1.0)
        assert np.allclose(vs, R, rtol=0, atol=1e-12)
        assert (rho == 1.0).all()


def test_direct_equals_recursive():
    rng = np.random.default_rng(2)
    for T in (1, 3, 17, 64):
        tr = rand_traj(rng, T, 4)
        a = VT.vtrace_direct(**tr, gamma=0.99, rho_bar=1.3, c_bar=0.9)
        b = VT.vtrace_recursive(**tr, gamma=0.99, rho_bar=1.3, c_bar=0.9)
        for x, y in zip(a, b):
            assert np.allclose(x, y, rtol=0, atol=1e-12)


def test_truncation_clamps_and_monotone():
    rng = np.random.default_rng(3)
    tr = rand_traj(rng, 6, 5)
    tr["log_pi"] = tr["log_mu"] + np.log(2.0)  # pi / mu = 2 everywhere
    _, rho, _ = VT.vtrace_recursive(**tr, gamma=0.9, rho_bar=1.0, c_bar=1.0)
    assert np.allclose(rho, 1.0)
    tr = rand_traj(rng, 6, 5)
    _, r1, _ = VT.vtrace_recursive(**tr, gamma=0.9, rho_bar=0.8, c_bar=0.5)
    _, r2, _ = VT.vtrace_recursive(**tr, gamma=0.9, rho_bar=1.6, c_bar=0.5)
    assert (r2 >= r1).all() and (r1 <= 0.8).all() and (r1 > 0).all()


def test_single_step_closed_form():
    # T = 1: v_0 = V_0 + rho_0 (r_0 + gamma V_boot - V_0); adv_0 = r_0 + gamma V_boot - V_0
    vs, rho, adv = VT.vtrace_direct([[2.0]], [[0.5]], [4.0], [[0.0]], [[np.log(0.5)]], [[0]], 0.9, 1.0, 1.0)
    assert np.isclose(rho[0, 0], 0.5, atol=1e-15)
    assert np.isclose(vs[0, 0], 0.5 + 0.5 * (2.0 + 0.9 * 4.0 - 0.5), atol=1e-15)
    assert np.isclose(adv[0, 0], 2.0 + 0.9 * 4.0 - 0.5, atol=1e-15)
