"""GPU parity of the batched V-trace kernel (cule_vtrace) against the
float64 oracle (oracle/vtrace.py) on the same float32 inputs.

Tolerance (R#33): the kernel computes in float32; each backward step does about eight
rounded operations (<= 2^-24 relative each) on quantities bounded by M, and carries the
previous step's error with the factor gamma_t c_t <= c_bar <= 1.  Hence
|v_gpu - v_oracle| <= T * 8 * 2^-24 * M plus expf's error on the ratio, bounded here by
2e-6 * T * (1 + M) with M = max |r|, |V|, |v|.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1907_08467_b200 import build
    build.build()


def case(rng, T, B, p_done, scale=1.0):
    f = lambda *s: (rng.normal(size=s) * scale).astype(np.float32)  # noqa: E731
    return dict(rewards=f(T, B), values=f(T, B), bootstrap=f(B),
                log_mu=(rng.normal(size=(T, B)) * 0.5).astype(np.float32),
                log_pi=(rng.normal(size=(T, B)) * 0.5).astype(np.float32),
                dones=(rng.random((T, B)) < p_done).astype(np.uint8))


@pytest.mark.parametrize("T,B,p_done,gamma,rho_bar,c_bar", [
    (1, 1, 0.0, 0.99, 1.0, 1.0), (5, 37, 0.1, 0.99, 1.0, 1.0), (20, 4096 + 13, 0.05, 0.99, 1.0, 1.0),
    (64, 300, 0.02, 1.0, 2.0, 1.0), (20, 513, 1.0, 0.9, 1.5, 0.5), (33, 129, 0.0, 0.5, 10.0, 0.25)])
def test_vtrace_matches_oracle(T, B, p_done, gamma, rho_bar, c_bar):
    from oracle import vtrace as VT
    from paper_1907_08467_b200.vtrace import vtrace
    rng = np.random.default_rng(T * 1000 + B)
    tr = case(rng, T, B, p_done)
    dev = {k: torch.from_numpy(v).cuda() for k, v in tr.items()}
    vs, rho, adv = vtrace(**dev, gamma=gamma, rho_bar=rho_bar, c_bar=c_bar)
    ref = VT.vtrace_recursive(**{k: v.astype(np.float64) if v.dtype != np.uint8 else v for k, v in tr.items()},
                              gamma=np.float32(gamma).item(), rho_bar=np.float32(rho_bar).item(),
                              c_bar=np.float32(c_bar).item())
    M = max(np.abs(tr["rewards"]).max(), np.abs(tr["values"]).max(), np.abs(ref[0]).max())
    tol = 2e-6 * T * (1.0 + M)
    for got, want, name in zip((vs, rho, adv), ref, ("vs", "rho", "adv")):
        err = np.abs(got.cpu().numpy().astype(np.float64) - want).max()
        assert err <= tol, (name, err, tol)


def test_vtrace_on_policy_equals_nstep_return():
    from oracle import vtrace as VT
    from paper_1907_08467_b200.vtrace import vtrace
    rng = np.random.default_rng(9)
    tr = case(rng, 20, 1000, 0.05)
    tr["log_pi"] = tr["log_mu"].copy()
    dev = {k: torch.from_numpy(v).cuda() for k, v in tr.items()}
    vs, rho, _ = vtrace(**dev, gamma=0.99)
    R = VT.nstep_return(tr["rewards"].astype(np.float64), tr["bootstrap"].astype(np.float64),
                        np.float32(0.99).item(), tr["dones"])
    assert (rho.cpu().numpy() == 1.0).all()
    assert np.abs(vs.cpu().numpy() - R).max() <= 2e-6 * 20 * (1 + np.abs(R).max())


def test_vtrace_rejects_bad_arguments():
    from paper_1907_08467_b200 import _lib
    from paper_1907_08467_b200.vtrace import vtrace
    rng = np.random.default_rng(0)
    dev = {k: torch.from_numpy(v).cuda() for k, v in case(rng, 4, 8, 0.1).items()}
    with pytest.raises(_lib.CuleError):
        vtrace(**dev, gamma=0.9, rho_bar=0.5, c_bar=1.0)  # rho_bar < c_bar
    with pytest.raises(_lib.CuleError):
        vtrace(**dev, gamma=1.5)
    with pytest.raises(ValueError):
        vtrace(**{**dev, "dones": dev["dones"].float()}, gamma=0.9)


def test_vtrace_sampled_at_bench_size():
    """The bench's HBM-roofline shape (T=20, B=2^20, 64-thread blocks across every SM): 200
    sampled trajectories against the oracle."""
    from oracle import vtrace as VT
    from paper_1907_08467_b200.vtrace import vtrace
    T, B = 20, 1 << 20
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    tr = dict(rewards=torch.randn(T, B, device="cuda", generator=g), values=torch.randn(T, B, device="cuda", generator=g),
              bootstrap=torch.randn(B, device="cuda", generator=g),
              log_mu=torch.randn(T, B, device="cuda", generator=g) * 0.5,
              log_pi=torch.randn(T, B, device="cuda", generator=g) * 0.5,
              dones=(torch.rand(T, B, device="cuda", generator=g) < 0.05).to(torch.uint8))
    vs, rho, adv = vtrace(**tr, gamma=0.99)
    cols = np.random.default_rng(0).choice(B, 200, replace=False)
    sub = {k: (v[..., cols] if v.dim() == 2 else v[cols]).cpu().numpy() for k, v in tr.items()}
    ref = VT.vtrace_recursive(**{k: v.astype(np.float64) if v.dtype != np.uint8 else v for k, v in sub.items()},
                              gamma=np.float32(0.99).item(), rho_bar=1.0, c_bar=1.0)
    M = max(np.abs(sub["rewards"]).max(), np.abs(sub["values"]).max(), np.abs(ref[0]).max())
    for got, want in zip((vs, rho, adv), ref):
        assert np.abs(got[:, cols].cpu().numpy().astype(np.float64) - want).max() <= 2e-6 * T * (1 + M)
