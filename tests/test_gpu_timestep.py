"""NEXT-3 on the GPU: the generalized-alpha vector updates (fem_time_init / fem_time_effective /
fem_time_increment, Block C P:404-417, D-1 P:421-424, D-4 P:459-465) against oracle/timestep.py, and
whole timesteps (Block C + Newton sub-steps through assembly and solve) against the oracle's assembler.

Tolerances: the vector updates are the correctly rounded left-to-right evaluation of the paper's
expressions on both sides -> bit-exact.  Whole timesteps go through iterative solves with relative
residual 1e-13 on the GPU vs a direct solve in the oracle -> states agree to 1e-8 relative (error <=
κ(K)·1e-13 and the penalty-dominated κ(K) of these small systems is below 1e5)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from oracle import timestep as ot  # noqa: E402
from fem_inputs import make_config, make_state  # noqa: E402
from fem_inputs.configs import TimeScheme  # noqa: E402


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _ts_dict(t):
    return dict(dt=t.dt, b1=t.b1, b2=t.b2, c1=t.c1, c2=t.c2, c3=t.c3)


@pytest.mark.parametrize("nu_hat", [0, 1, 2])
@pytest.mark.parametrize("n", [1, 257, 3_000_017])
def test_time_updates_bit_exact(nu_hat, n):
    _need_gpu()
    from paper_2111_03541_b200 import fem
    t = TimeScheme("genalpha", nu_hat, dt=0.0137, b1=0.61, b2=0.47, c1=0.9, c2=0.8, c3=0.7)
    ts, T = _ts_dict(t), fem.make_time_scheme(t)
    rng = np.random.default_rng(nu_hat * 1000 + n % 1000)
    phi0 = rng.standard_normal((nu_hat + 1, n))
    incr = rng.standard_normal((nu_hat + 1, n))
    dsub = rng.standard_normal(n)
    g_phi0, g_incr = torch.from_numpy(phi0).cuda(), torch.from_numpy(incr).cuda()
    g_eff = torch.empty_like(g_phi0)
    # Block C (+ fused D-1)
    ot.time_init(ts, nu_hat, phi0, incr)
    eff = ot.time_effective(ts, nu_hat, phi0, incr)
    fem.fem_time_init(T, n, g_phi0, g_incr, g_eff)
    assert np.array_equal(g_phi0.cpu().numpy(), phi0)
    assert np.array_equal(g_incr.cpu().numpy(), incr)
    assert np.array_equal(g_eff.cpu().numpy(), eff)
    # D-4 (+ fused D-1), twice
    for _ in range(2):
        ot.time_increment(ts, nu_hat, dsub, incr)
        eff = ot.time_effective(ts, nu_hat, phi0, incr)
        fem.fem_time_increment(T, n, torch.from_numpy(dsub).cuda(), g_incr, g_phi0, g_eff)
        assert np.array_equal(g_incr.cpu().numpy(), incr)
        assert np.array_equal(g_eff.cpu().numpy(), eff)
    # D-1 alone, and D-4 without the fused D-1
    g_eff2 = torch.full_like(g_phi0, np.nan)
    fem.fem_time_effective(T, n, g_phi0, g_incr, g_eff2)
    assert np.array_equal(g_eff2.cpu().numpy(), eff)
    ot.time_increment(ts, nu_hat, dsub, incr)
    fem.fem_time_increment(T, n, torch.from_numpy(dsub).cuda(), g_incr)
    assert np.array_equal(g_incr.cpu().numpy(), incr)


def test_time_calls_reject_bad_schemes():
    _need_gpu()
    from paper_2111_03541_b200 import fem
    x = torch.zeros(2, 4, dtype=torch.float64, device="cuda")
    for bad in (TimeScheme("static", 0), TimeScheme("genalpha", 3, dt=0.1),
                TimeScheme("genalpha", 1, dt=0.0), TimeScheme("genalpha", 1, dt=0.1, b1=0.0)):
        with pytest.raises(fem.FemError):
            fem.fem_time_init(fem.make_time_scheme(bad), 4, x, x)
    fem.fem_time_init(fem.make_time_scheme(TimeScheme("genalpha", 1, dt=0.1)), 0, None, None)  # n = 0: no-op


def _oracle_timestep(m, p, ts, nu_hat, phi0, incr, n_sub, shape):
    """Blocks C/D with the oracle assembler and a direct sparse solve (D-4)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    ot.time_init(ts, nu_hat, phi0, incr)
    n = phi0.shape[1]
    for _ in range(n_sub):
        eff = ot.time_effective(ts, nu_hat, phi0, incr)
        o = oracle.assemble(m, p, np.ascontiguousarray(eff.reshape(shape)))
        K = sp.csr_matrix((o["values"], o["colidx"], o["rowptr"]), shape=(n, n))
        dsub = spla.spsolve(K.tocsc(), -o["rhs"])
        ot.time_increment(ts, nu_hat, dsub, incr)


@pytest.mark.parametrize("variant", ["structured", "perturbed"])
def test_transient_thermal_timesteps_match_oracle(variant):
    """ν̂ = 1 heat conduction -C(T,T_t) - k(∇T,∇T) + (T,s) with the FIX boundary: five
    timesteps of three Newton sub-steps each, GPU (assembly + BiCGStab + time kernels) vs oracle."""
    _need_gpu()
    from paper_2111_03541_b200 import FemSystem
    m, p = make_config("c2", variant, (5, 4, 3))
    # b1 = 0.8, c = 1: the θ-method with θ = 0.8 (damps the stiff penalty modes, ρ∞ = 0.25); the
    # trapezoidal member (b1 = 1/2) leaves them undamped and the rough random start then drives the T^4
    # Newton off.  General b/c values are covered bit-exactly by test_time_updates_bit_exact.
    p.time = TimeScheme("genalpha", 1, dt=0.02, b1=0.8, b2=0.5, c1=1.0, c2=1.0, c3=1.0)
    p.terms[0].params = dict(p.terms[0].params, C=3.0)
    st = make_state("c2", m, p)                     # [2][1][N]
    st[1] = 0.0                                     # start at rest (random T_t drives Newton off)
    n = st.shape[1] * st.shape[2]
    phi0 = st.reshape(2, n).copy()
    incr = np.zeros_like(phi0)
    S = FemSystem(m, p)
    g_phi0 = torch.from_numpy(phi0.reshape(st.shape)).cuda()
    g_incr = torch.zeros_like(g_phi0)
    ts = _ts_dict(p.time)
    for step in range(5):
        _oracle_timestep(m, p, ts, 1, phi0, incr, 3, st.shape)
        hist = S.time_step(g_phi0, g_incr, n_sub=3, method="bicgstab", rtol=1e-13, max_iter=200000)
        assert len(hist) == 3 and hist[2][0] < hist[0][0]   # Newton on the T^4 boundary term converging
        got = (g_phi0 + g_incr).reshape(2, n).cpu().numpy()
        want = ot.committed(1, phi0, incr)
        for nu in range(2):
            err = np.abs(got[nu] - want[nu]).max() / np.abs(want[nu]).max()
            assert err <= 1e-8, (step, nu, err)
    S.close()
