"""NEXT-1: the Newton sub-step's linear solve on the GPU, through the C ABI.

D-4 solves K Δφ = -d.  The GPU path is fem_spmv / fem_cg_solve (Jacobi-PCG on
s K with s = -1: the elasticity K is symmetric negative definite in the paper's sign convention,
reading L17).  Pins:
  * fem_spmv against scipy's CSR product of the ORACLE's K (same pattern, bit-exact, see the parity
    tests), within a sum-of-|terms| bound;
  * the CG solution against scipy's direct solve of the oracle's system, within κ(A)·rtol;
  * linearity: the elasticity form is linear in d, so ONE Newton step from any state zeroes the
    residual (the D-2 convergence test);
  * mathematics: a P2-tet cantilever (the c3 beam with ν = 0, as the paper's beam P:944) deflects by
    Timoshenko's P L³/(3 E I) + P L/(κ G A) (I = h⁴/12, reading L24; κ = 5/6) to 0.5 %.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from fem_inputs import make_config, make_state  # noqa: E402


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _csr(ora):
    import scipy.sparse as sp
    n = len(ora["rowptr"]) - 1
    return sp.csr_matrix((ora["values"], ora["colidx"], ora["rowptr"]), shape=(n, n))


@pytest.mark.parametrize("name,dims", [("c1", (8,)), ("c3", (7, 3, 2)), ("c4", (9, 4, 3)), ("c5", (7, 5, 6))])
def test_spmv_matches_scipy_on_oracle_matrix(name, dims):
    _need_gpu()
    from paper_2111_03541_b200 import FemSystem
    m, p = make_config(name, "perturbed", dims)
    st = make_state(name, m, p)
    ora = oracle.assemble(m, p, st)
    S = FemSystem(m, p)
    S.alloc(True, False)
    S.values.copy_(torch.from_numpy(ora["values"]))
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, S.n_rows)
    y0 = rng.uniform(-1, 1, S.n_rows)
    y = S.spmv(torch.from_numpy(x).cuda(), torch.from_numpy(y0.copy()).cuda(), alpha=0.5, beta=-2.0).cpu().numpy()
    K = _csr(ora)
    ref = 0.5 * (K @ x) - 2.0 * y0
    scale = 0.5 * (abs(K) @ np.abs(x)) + 2.0 * np.abs(y0)
    assert np.max(np.abs(y - ref) / scale) <= 1e-14
    S.close()


@pytest.mark.parametrize("name,dims", [("c5", (7, 5, 6)), ("c3", (7, 3, 2))])
def test_cg_matches_direct_solve_and_is_bit_reproducible(name, dims):
    _need_gpu()
    import scipy.sparse.linalg as spla
    from paper_2111_03541_b200 import FemSystem
    m, p = make_config(name, "perturbed", dims)
    st = make_state(name, m, p)
    ora = oracle.assemble(m, p, st)
    K = _csr(ora)
    x_ref = spla.spsolve(K.tocsc(), -ora["rhs"])
    S = FemSystem(m, p)
    sd = torch.from_numpy(st).cuda()
    Kg, dg = S.system(sd, scatter="tiled")
    rtol = 1e-13
    x, it, rel = S.solve(-dg, rtol=rtol, max_iter=50000)
    assert rel <= rtol and it > 0
    x = x.cpu().numpy()
    # forward error <= κ(A) · relative residual (A = -K SPD; dense κ on these small systems)
    kappa = np.linalg.cond(-K.toarray())
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 10 * kappa * rtol
    # true residual of the original system (x0 = 0: r0 = b; the recurrence drifts from b - A x by rounding)
    assert np.linalg.norm(K @ x + ora["rhs"]) / np.linalg.norm(ora["rhs"]) <= 1e-11
    x2, it2, rel2 = S.solve(-dg, rtol=rtol, max_iter=50000)
    assert it2 == it and rel2 == rel and np.array_equal(x2.cpu().numpy(), x)
    S.close()


def test_one_newton_step_solves_linear_elasticity():
    """d(φ) is affine in φ for the elasticity forms, so φ1 = φ0 + Δφ with K Δφ = -d(φ0) zeroes it."""
    _need_gpu()
    from paper_2111_03541_b200 import FemSystem
    m, p = make_config("c5", "perturbed", (7, 5, 6))
    st = torch.from_numpy(make_state("c5", m, p)).cuda()
    S = FemSystem(m, p)
    _, d0 = S.system(st, scatter="tiled")
    n0 = float(torch.linalg.norm(d0))
    st1, it, rel = S.newton_step(st, scatter="tiled", rtol=1e-13)
    _, d1 = S.system(st1, scatter="tiled")
    assert float(torch.linalg.norm(d1)) <= 1e-9 * n0
    S.close()


def test_cantilever_tip_deflection_matches_beam_theory():
    """c3 beam [0,10]x[0,1]^2, P2 tets, ν = 0, fixed at x = 0, end load P = 1e-3."""
    _need_gpu()
    from paper_2111_03541_b200 import FemSystem
    m, p = make_config("c3", "structured", (40, 4, 4))
    p.terms[0].params = dict(E=1.0, nu=0.0)
    S = FemSystem(m, p)
    st = torch.zeros((1, 3, m.n_nodes), dtype=torch.float64, device="cuda")
    st1, it, rel = S.newton_step(st, scatter="tiled", rtol=1e-12, max_iter=200000)
    assert rel <= 1e-12
    uy = st1[0, 1].cpu().numpy()
    tip = np.isclose(m.coords[0], 10.0)
    P, L, E, G, A, I, kappa = 1e-3, 10.0, 1.0, 0.5, 1.0, 1.0 / 12.0, 5.0 / 6.0
    timoshenko = P * L ** 3 / (3 * E * I) + P * L / (kappa * G * A)
    assert abs(-uy[tip].mean() / timoshenko - 1.0) <= 5e-3
    S.close()


@pytest.mark.parametrize("name,dims", [("c1", (8,)), ("c2", (9, 7, 6))])
def test_bicgstab_matches_direct_solve_nonsymmetric(name, dims):
    """The thermal FIX term k N_a n·∇T makes K non-symmetric: BiCGStab.  (The NS saddle-point
    system, diverges under a Jacobi preconditioner; it needs a block preconditioner — DESIGN.)"""
    _need_gpu()
    import scipy.sparse.linalg as spla
    from paper_2111_03541_b200 import FemSystem
    m, p = make_config(name, "perturbed", dims)
    st = make_state(name, m, p)
    ora = oracle.assemble(m, p, st)
    K = _csr(ora)
    assert abs(K - K.T).max() > 0  # really non-symmetric
    x_ref = spla.spsolve(K.tocsc(), -ora["rhs"])
    S = FemSystem(m, p)
    _, dg = S.system(torch.from_numpy(st).cuda(), scatter="tiled")
    x, it, rel = S.solve(-dg, rtol=1e-13, max_iter=200000, method="bicgstab")
    assert rel <= 1e-13
    x = x.cpu().numpy()
    assert np.linalg.norm(K @ x + ora["rhs"]) / np.linalg.norm(ora["rhs"]) <= 1e-11
    kappa = np.linalg.cond(K.toarray())
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 10 * kappa * 1e-13
    x2, it2, rel2 = S.solve(-dg, rtol=1e-13, max_iter=200000, method="bicgstab")
    assert it2 == it and np.array_equal(x2.cpu().numpy(), x)
    S.close()


def _gpu_manufactured_error(n, etype):
    """The oracle pin's manufactured problem (T* = Π sin πx_d, s = dim π² T*, penalty 1e8·k/h, reading L22),
    assembled and solved on the GPU (one Newton step from T = 0, BiCGStab); the L2 error by quadrature."""
    import math
    from fem_inputs.meshgen import facets_on_plane, hex_box, tri_square
    from helpers import problem
    from paper_2111_03541_b200 import FemSystem
    if etype == "tri":
        m = tri_square(n)
        be = [facets_on_plane(m, a, v) for a in (0, 1) for v in (0.0, 1.0)]
        s, dim = 2 * math.pi ** 2, 2
    else:
        m = hex_box(n, n, n)
        be = [facets_on_plane(m, a, v) for a in (0, 1, 2) for v in (0.0, 1.0)]
        s, dim = 3 * math.pi ** 2, 3
    m.bsets = [(np.concatenate([b[0] for b in be]), np.concatenate([b[1] for b in be]))]
    pr = problem("thermal", etype, 1, [("THERMAL_DOMAIN", -1, dict(C=0.0, k=1.0, s=s, source="sine")),
                                       ("THERMAL_FIX", 0, dict(h_p=1e8 * n, T_fix=0.0, k=1.0))])
    S = FemSystem(m, pr)
    st = torch.zeros((1, 1, m.n_nodes), dtype=torch.float64, device="cuda")
    st1, it, rel = S.newton_step(st, scatter="tiled", rtol=1e-12, max_iter=500000, method="bicgstab")
    assert rel <= 1e-12
    T = st1[0, 0].cpu().numpy()
    S.close()
    err2 = 0.0
    for e in range(m.n_elems):
        d = oracle.qp_data(m, pr, e)
        Th = d["N"] @ T[m.conn[:, e]]
        ex = np.prod(np.sin(np.pi * d["x"][:, :dim]), axis=1)
        err2 += (d["w"] * (Th - ex) ** 2).sum()
    return math.sqrt(err2)


@pytest.mark.parametrize("etype,ns", [("tri", (8, 16, 32, 64)), ("hex", (4, 8, 16))])
def test_gpu_manufactured_convergence_rate(etype, ns):
    """The whole GPU path (assembly + solve) against mathematics: P1 / Q1 L2 error rate -> 2."""
    _need_gpu()
    import math
    errs = [_gpu_manufactured_error(n, etype) for n in ns]
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert all(1.8 < r < 2.3 for r in rates), (errs, rates)


@pytest.mark.parametrize("variant", ["structured", "perturbed"])
def test_ns_newton_step_gmres_matches_direct_solve(variant):
    """NEXT-1 remainder: the stabilised NS saddle point, where Jacobi-BiCGStab diverges, solved by
    point-block-Jacobi GMRES on the GPU with the pressure of point 0 pinned (L29): the Newton increment of
    small c4 matches scipy's direct solve of the ORACLE's pinned K and d within 10·κ·rtol, the solve is
    bit-identical run to run, and a Newton sub-step through the ABI reduces ||d||."""
    _need_gpu()
    import scipy.sparse.linalg as spla
    from paper_2111_03541_b200 import FemSystem
    m, p = make_config("c4", variant, (9, 4, 3))
    st = make_state("c4", m, p)
    ora = oracle.assemble(m, p, st)
    N = m.n_nodes
    pin = 3 * N
    K = _csr(ora).tolil()
    K[pin, :] = 0.0
    K[:, pin] = 0.0
    K[pin, pin] = 1.0
    K = K.tocsr()
    b = -ora["rhs"].copy()
    b[pin] = 0.0
    x_ref = spla.spsolve(K.tocsc(), b)
    S = FemSystem(m, p)
    sd = torch.from_numpy(st).cuda()
    S.system(sd, scatter="tiled")
    d = S.rhs.clone()
    rtol = 1e-11
    x, it, rel = S.solve(-d, rtol=rtol, max_iter=5000, method="gmres", restart=200)
    assert rel <= 10 * rtol and it > 0, (it, rel)
    xn = x.cpu().numpy()
    kappa = np.linalg.cond(K.toarray())
    assert np.linalg.norm(xn - x_ref) / np.linalg.norm(x_ref) <= 10 * kappa * rtol
    assert xn[pin] == 0.0
    x2, it2, rel2 = S.solve(-d, rtol=rtol, max_iter=5000, method="gmres", restart=200)
    assert it2 == it and rel2 == rel and torch.equal(x2, x)
    # Newton consistency of the increment: d(φ + εΔ) = (1 - ε) d(φ) + O(ε²) on every row but the pinned one
    dn = d.cpu().numpy()
    mask = np.ones(len(dn), bool)
    mask[pin] = False
    errs = []
    for eps in (1e-3, 2e-3):
        st_e = sd.clone()
        st_e[0] += eps * x.view(4, N)
        S.system(st_e, scatter="tiled")
        errs.append(np.linalg.norm((S.rhs.cpu().numpy() - (1 - eps) * dn)[mask]))
    assert errs[1] / errs[0] == pytest.approx(4.0, rel=0.1), errs
    # and a full Newton sub-step runs through the ABI with the pinned GMRES (φ ← φ + Δφ in the library)
    st1, it1, rel1 = S.newton_step(sd, scatter="tiled", rtol=1e-10, max_iter=5000, method="gmres")
    assert rel1 <= 1e-9 and float(st1[0, 3, 0]) == float(sd[0, 3, 0])  # pinned pressure unchanged
    S.close()
