"""NEXT-2 pins of the oracle: quadratic cubes (27-node Lagrange Q2 and 20-node serendipity)
and the second-derivative tables behind μ u_i,kk.  Nothing here compares the oracle with itself:
closed-form element matrices (Kronecker products of the textbook 1D quadratic matrices), exact monomial
integrals, reproduction of polynomial fields, invariants, the manufactured-solution rate 3 and the paper's
cantilever against beam theory."""
import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
from fem_inputs import make_config
from fem_inputs.configs import TimeScheme
from fem_inputs.meshgen import facets_on_plane, hex_box_quadratic, quad_cube_ref_nodes
from helpers import problem

QUAD = [("hex", 27), ("hexs", 20)]


def _rect(mesh, seed=3, amp=0.25):
    """Rectilinear (affine elements) but non-uniform grid: every lattice line shifted by a random amount
    along its own axis, so each element is an axis-aligned box of its own size."""
    rng = np.random.default_rng(seed)
    c = mesh.coords.copy()
    for d in range(3):
        vals = np.unique(np.round(c[d], 12))
        h = vals[2] - vals[0] if len(vals) > 2 else 1.0
        shift = np.zeros(len(vals))
        shift[2:-2:2] = rng.uniform(-amp, amp, len(shift[2:-2:2])) * h / 2   # move vertex lines
        newv = vals + shift
        newv[1::2] = 0.5 * (newv[0:-1:2] + newv[2::2])                        # mid lines stay centred
        idx = np.searchsorted(vals, np.round(c[d], 12))
        c[d] = newv[idx]
    mesh.coords = np.ascontiguousarray(c)
    return mesh


def _curved(mesh, seed=4, amp=0.12):
    """Non-affine quadratic geometry: every interior node (vertices AND mid nodes) jittered, so edges curve
    and the isoparametric map has non-zero second derivatives."""
    rng = np.random.default_rng(seed)
    c = mesh.coords.copy()
    lo, hi = c.min(axis=1), c.max(axis=1)
    on = np.zeros(c.shape[1], bool)
    for d in range(3):
        on |= (np.abs(c[d] - lo[d]) < 1e-12) | (np.abs(c[d] - hi[d]) < 1e-12)
    h = (hi - lo) / np.array([len(np.unique(np.round(c[d], 12))) - 1 for d in range(3)])
    c[:, ~on] += rng.uniform(-amp, amp, (3, int((~on).sum()))) * h[:, None]
    mesh.coords = np.ascontiguousarray(c)
    return mesh


def _one_cube(etype, h):
    serend = etype == "hexs"
    m = hex_box_quadratic(1, 1, 1, h, h, h, serendipity=serend)
    return m


def _dense(m, pr, st=None):
    kh = pr.kappa_hat(m.dim)
    st = np.zeros((pr.time.nu_hat + 1, kh, m.n_nodes)) if st is None else st
    out = oracle.assemble(m, pr, st)
    assert out["status"] == 0, out
    return oracle.to_dense(out, kh * m.n_nodes), out


def _lap(etype, k=1.0, C=0.0, time=None):
    return problem("thermal", etype, 2, [("THERMAL_DOMAIN", -1, dict(C=C, k=k, s=0.0))], 3, time)


# ------------------------------------------------------------------ Q2: Kronecker closed forms
@pytest.mark.parametrize("h", [1.0, 0.37])
def test_q2_laplacian_and_mass_are_kronecker_products(h):
    """On the cube [0,h]³ the Q2 Laplacian is K1⊗M1⊗M1 + M1⊗K1⊗M1 + M1⊗M1⊗K1 and the mass M1⊗M1⊗M1 with
    the textbook 1D quadratic element (nodes 0, h/2, h): K1 = [[7,-8,1],[-8,16,-8],[1,-8,7]]/(3h),
    M1 = h[[4,2,-1],[2,16,2],[-1,2,4]]/30 — GL 3 is exact (degree ≤ 4 per axis).  Paper sign (L17):
    K = -k·Laplacian - C f1·mass (f1 = c2/(b1 Δt), Eq. gen_alpha)."""
    m = _one_cube("hex", h)
    K1 = np.array([[7, -8, 1], [-8, 16, -8], [1, -8, 7]]) / (3 * h)
    M1 = h * np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]) / 30
    r = quad_cube_ref_nodes(27)
    # the dense matrix rows/cols are in mesh node order; node of local a is conn[a, 0]
    perm = m.conn[:, 0]

    def kron_entry(A, B, Cm, a, b):
        i, j = r[a] + 1, r[b] + 1
        return A[i[0], j[0]] * B[i[1], j[1]] * Cm[i[2], j[2]]

    L = np.array([[kron_entry(K1, M1, M1, a, b) + kron_entry(M1, K1, M1, a, b) + kron_entry(M1, M1, K1, a, b)
                   for b in range(27)] for a in range(27)])
    Mm = np.array([[kron_entry(M1, M1, M1, a, b) for b in range(27)] for a in range(27)])
    K, _ = _dense(m, _lap("hex", k=1.7))
    np.testing.assert_allclose(K[np.ix_(perm, perm)], -1.7 * L, atol=1e-13 * np.abs(L).max())
    ts = TimeScheme("genalpha", 1, dt=0.5, b1=0.8, b2=0.5, c1=1.0, c2=0.6, c3=1.0)
    K, _ = _dense(m, _lap("hex", k=0.0, C=2.3, time=ts))
    f1 = 0.6 / (0.8 * 0.5)
    np.testing.assert_allclose(K[np.ix_(perm, perm)], -2.3 * f1 * Mm, atol=1e-13 * np.abs(Mm).max())


# ------------------------------------------------------------------ quadrature and reproduction
@pytest.mark.parametrize("etype,nl", QUAD)
def test_partition_of_unity_and_gl3_exactness(etype, nl):
    """Σ_a N_a = 1, Σ_a ∇N_a = 0, Σ_a ∇∇N_a = 0 at every point; Σ_q w x^p over the box [0,a]x[0,b]x[0,c]
    is exact for every monomial of degree ≤ 5 per axis (3-point Gauss-Legendre per axis, L9)."""
    m = hex_box_quadratic(1, 1, 1, 0.7, 1.3, 0.9, serendipity=(etype == "hexs"))
    pr = _lap(etype)
    d = oracle.qp_data(m, pr, 0)
    assert len(d["w"]) == 27
    np.testing.assert_allclose(d["N"].sum(axis=1), 1.0, atol=1e-14)
    np.testing.assert_allclose(d["G"].sum(axis=1), 0.0, atol=1e-13)
    np.testing.assert_allclose(d["H"].sum(axis=1), 0.0, atol=1e-12)
    L = np.array([0.7, 1.3, 0.9])
    for p in [(0, 0, 0), (5, 0, 0), (0, 4, 1), (3, 5, 2), (5, 5, 5), (2, 1, 4)]:
        got = (d["w"] * np.prod(d["x"] ** np.array(p), axis=1)).sum()
        exact = np.prod(L ** (np.array(p) + 1) / (np.array(p) + 1))
        assert got == pytest.approx(exact, rel=1e-13)


def _poly_fields():
    """A few quadratic polynomials (in every quadratic-cube space): (value, gradient, Hessian) callables."""
    Q = np.array([[0.6, 0.2, -0.3], [0.2, -0.4, 0.5], [-0.3, 0.5, 0.8]])
    g0 = np.array([0.3, -1.1, 0.7])
    f = lambda x: 0.5 + g0 @ x + 0.5 * np.einsum("in,ij,jn->n", x, Q, x)  # noqa: E731
    return f, Q


@pytest.mark.parametrize("etype,nl", QUAD)
def test_second_derivatives_reproduce_quadratics(etype, nl):
    """Σ_a f(x_a) ∂²N_a/∂x_i∂x_j (x_q) = ∂²f/∂x_i∂x_j exactly for quadratic f on affine (rectilinear)
    elements, and Σ_a x_ak ∂²N_a = 0 for the linear fields on CURVED elements (the geometric term
    −Σ_i G_i ∂²x_i/∂ξ² of the chain rule; dropping it fails here)."""
    m = _rect(hex_box_quadratic(2, 2, 2, 1.0, 0.8, 1.2, serendipity=(etype == "hexs")))
    pr = _lap(etype)
    f, Q = _poly_fields()
    for e in range(m.n_elems):
        d = oracle.qp_data(m, pr, e)
        fv = f(m.coords[:, m.conn[:, e]])
        Hf = np.einsum("a,qaij->qij", fv, d["H"])
        np.testing.assert_allclose(Hf, np.broadcast_to(Q, Hf.shape), atol=1e-11)
        gv = np.einsum("a,qai->qi", fv, d["G"])
        np.testing.assert_allclose(gv, (np.array([0.3, -1.1, 0.7])[:, None] + Q @ d["x"].T).T, atol=1e-11)
    mc = _curved(hex_box_quadratic(2, 2, 2, serendipity=(etype == "hexs")))
    for e in range(mc.n_elems):
        d = oracle.qp_data(mc, pr, e)
        X = mc.coords[:, mc.conn[:, e]]
        for k in range(3):
            assert np.abs(np.einsum("a,qaij->qij", X[k], d["H"])).max() < 1e-10
            np.testing.assert_allclose(np.einsum("a,qai->qi", X[k], d["G"]), np.eye(3)[k][None, :].repeat(27, 0),
                                       atol=1e-12)


@pytest.mark.parametrize("etype,nl", QUAD)
def test_laplacian_weak_form_of_quadratic_fields(etype, nl):
    """Residual d(T) = -k ∫∇N_a·∇T of the thermal domain form for a quadratic T on a rectilinear mesh of the
    box B = [0,1]x[0,0.8]x[0,1.2]: test functions 1, x_k and x_k x_l lie in both spaces, so
    Σ_a c_a d_a = -k ∫_B ∇v·∇T with v = 1, x_k, x_k x_l — closed-form integrals of polynomials
    (a wrong serendipity basis function breaks the reproduction)."""
    m = _rect(hex_box_quadratic(2, 3, 2, 1.0, 0.8, 1.2, serendipity=(etype == "hexs")))
    k = 1.3
    pr = problem("thermal", etype, 2, [("THERMAL_DOMAIN", -1, dict(C=0.0, k=k, s=0.0))], 3)
    f, Q = _poly_fields()
    g0 = np.array([0.3, -1.1, 0.7])
    st = np.zeros((1, 1, m.n_nodes))
    st[0, 0] = f(m.coords)
    d = oracle.assemble(m, pr, st, matrix=False)["rhs"]
    Lb = np.array([1.0, 0.8, 1.2])
    vol = Lb.prod()
    mean = Lb / 2
    mxx = np.outer(mean, mean) + np.diag(Lb ** 2 / 12)  # E[x xᵀ] over the box
    # ∇T = g0 + Q x
    assert abs(d.sum()) < 1e-12 * np.abs(d).max() * m.n_nodes
    x = m.coords
    for kk in range(3):
        assert (x[kk] * d).sum() == pytest.approx(-k * vol * (g0[kk] + Q[kk] @ mean), rel=1e-12)
    for a in range(3):
        for b in range(3):
            # ∇(x_a x_b) = e_a x_b + e_b x_a;  ∫ ∇v·∇T = ∫ x_b (∇T)_a + x_a (∇T)_b
            E = lambda i, j: vol * (g0[i] * mean[j] + Q[i] @ mxx[:, j])  # noqa: E731  ∫ (∇T)_i x_j
            exact = -k * (E(a, b) + E(b, a))
            assert (x[a] * x[b] * d).sum() == pytest.approx(exact, rel=1e-11, abs=1e-12)


@pytest.mark.parametrize("etype,nl", QUAD)
def test_quadratic_elasticity_invariants(etype, nl):
    """Rigid modes in the kernel, symmetry, −K PSD with exactly 6 zero eigenvalues on a curved mesh."""
    m = _curved(hex_box_quadratic(2, 1, 1, serendipity=(etype == "hexs")))
    pr = problem("elasticity", etype, 2, [("ELAST_DOMAIN", -1, dict(E=1.0, nu=0.3))], 3)
    K, _ = _dense(m, pr)
    scale = np.abs(K).max()
    N = m.n_nodes
    x = m.coords
    modes = []
    for i in range(3):
        r = np.zeros((3, N)); r[i] = 1.0; modes.append(r.ravel())
    for (i, j) in ((0, 1), (1, 2), (0, 2)):
        r = np.zeros((3, N)); r[i] = -x[j]; r[j] = x[i]; modes.append(r.ravel())
    for r in modes:
        assert np.abs(K @ r).max() < 1e-12 * scale * np.abs(r).max()
    np.testing.assert_allclose(K, K.T, atol=1e-14 * scale)
    ev = np.linalg.eigvalsh(-K)
    assert ev.min() > -1e-12 * scale
    assert np.sum(ev < 1e-10 * scale) == 6


# ------------------------------------------------------------------ NS with μ u_i,kk
@pytest.mark.parametrize("etype,nl", QUAD)
def test_ns_pspg_residual_carries_viscous_laplacian(etype, nl):
    """u = (a y², b x z, 0), p = p0 + g·x on the rectilinear box [0,Lx]x[0,Ly]x[0,Lz]: Rc = div u = 0,
    Δu = (2a, 0, 0), u·∇u = (2ab xyz, ab y² z, 0), so Rm = (2ρab xyz + g1 − 2μa, ρab y²z + g2, g3).
    The pressure rows give Σ_a d_(a,p) = ∫Rc = 0 and Σ_a x_ak d_(a,p) = ∫ x_k Rc + τ_m Rm_k = τ_m ∫Rm_k —
    cubic integrands, exact under GL 3 on affine elements; the −μ u_i,kk term is visible with its sign."""
    Lb = np.array([1.0, 0.8, 1.2])
    m = _rect(hex_box_quadratic(2, 2, 3, *Lb, serendipity=(etype == "hexs")))
    a, b, rho, mu, tm = 0.7, -0.4, 2.0, 0.9, 0.37
    g, p0 = np.array([0.5, -1.0, 2.0]), 0.3
    x = m.coords
    st = np.zeros((1, 4, m.n_nodes))
    st[0, 0] = a * x[1] ** 2
    st[0, 1] = b * x[0] * x[2]
    st[0, 3] = p0 + g @ x
    pr = problem("ns", etype, 2, [("NS_DOMAIN", -1, dict(rho=rho, mu=mu, tau_m=tm, tau_c=0.0))], 3)
    d = oracle.assemble(m, pr, st, matrix=False)["rhs"].reshape(4, -1)
    vol = Lb.prod()
    I_xyz = (Lb[0] ** 2 / 2) * (Lb[1] ** 2 / 2) * (Lb[2] ** 2 / 2)
    I_y2z = Lb[0] * (Lb[1] ** 3 / 3) * (Lb[2] ** 2 / 2)
    ERm = np.array([2 * rho * a * b * I_xyz + (g[0] - 2 * mu * a) * vol, rho * a * b * I_y2z + g[1] * vol, g[2] * vol])
    assert abs(d[3].sum()) < 1e-12 * np.abs(d[3]).max() * m.n_nodes
    for k in range(3):
        assert (x[k] * d[3]).sum() == pytest.approx(tm * ERm[k], rel=1e-11)


@pytest.mark.parametrize("etype,nl", QUAD)
def test_ns_quadratic_fd_tangent(etype, nl):
    """Central FD of the NS residual (domain with τ ≠ 0 and every boundary group) vs the K columns on a
    curved quadratic mesh: the tangent carries −μ N_b,kk in dRm."""
    from test_oracle_pins import _fd_check
    m, p = make_config("q2ns", "perturbed", (2, 1, 1))
    if etype == "hexs":
        from fem_inputs.meshgen import hex_box_quadratic as hq
        m2 = hq(2, 1, 1, 2.5, 0.41, 0.41, serendipity=True)
        m2.bsets = [facets_on_plane(m2, 0, 0.0), facets_on_plane(m2, 0, 2.5),
                    facets_on_plane(m2, 1, 0.0)]
        m = _curved(m2)
        p.etype = "hexs"
    m = _curved(m) if etype == "hex" else m
    from fem_inputs import make_state
    st = make_state("q2ns", m, p)
    for t in p.terms:
        if t.form == "NS_DOMAIN":
            t.params = dict(t.params, tau_m=1e-3, tau_c=0.5)
    assert _fd_check(m, p, st, cols=range(0, 4 * m.n_nodes, 5)) < 1e-6


# ------------------------------------------------------------------ end to end
def _manufactured_error_q(n, etype):
    m = hex_box_quadratic(n, n, n, serendipity=(etype == "hexs"))
    be = [facets_on_plane(m, a, v) for a in (0, 1, 2) for v in (0.0, 1.0)]
    m.bsets = [(np.concatenate([b[0] for b in be]), np.concatenate([b[1] for b in be]))]
    terms = [("THERMAL_DOMAIN", -1, dict(C=0.0, k=1.0, s=3 * math.pi ** 2, source="sine")),
             ("THERMAL_FIX", 0, dict(h_p=1e8 * n, T_fix=0.0, k=1.0))]   # L22 penalty 1e8·k/h
    pr = problem("thermal", etype, 2, terms, 3)
    out = oracle.assemble(m, pr, np.zeros((1, 1, m.n_nodes)))
    K = sp.csr_matrix((out["values"], out["colidx"], out["rowptr"]), shape=(m.n_nodes,) * 2)
    T = spla.spsolve(K.tocsc(), -out["rhs"])
    err2 = 0.0
    for e in range(m.n_elems):
        d = oracle.qp_data(m, pr, e)
        Th = d["N"] @ T[m.conn[:, e]]
        ex = np.sin(np.pi * d["x"][:, 0]) * np.sin(np.pi * d["x"][:, 1]) * np.sin(np.pi * d["x"][:, 2])
        err2 += (d["w"] * (Th - ex) ** 2).sum()
    return math.sqrt(err2)


@pytest.mark.parametrize("etype,nl", QUAD)
def test_manufactured_convergence_rate_three(etype, nl):
    """T* = sin πx sin πy sin πz, s = 3π² T*: the L2 error of quadratic cubes falls at rate 3."""
    errs = [_manufactured_error_q(n, etype) for n in (2, 4, 8)]
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert rates[-1] > 2.7 and all(r < 3.4 for r in rates), (errs, rates)


@pytest.mark.parametrize("name", ["q2", "s2"])
def test_quadratic_cube_cantilever_beam_theory(name):
    """The paper's cantilever (ν = 0) on 10x4x4 quadratic cubes with the end load
    P = 1e-3 deflects by Timoshenko's P L³/(3EI) + P L/(κGA) (I = h⁴/12, reading L24, κ = 5/6) to 1%."""
    m, p = make_config(name, "structured", (10, 4, 4))
    p.terms[0].params = dict(E=1.0, nu=0.0)
    out = oracle.assemble(m, p, np.zeros((1, 3, m.n_nodes)))
    n = len(out["rowptr"]) - 1
    K = sp.csr_matrix((out["values"], out["colidx"], out["rowptr"]), shape=(n, n))
    x = spla.spsolve(K.tocsc(), -out["rhs"])
    uy = x[m.n_nodes:2 * m.n_nodes]
    tip = np.isclose(m.coords[0], 10.0)
    P, L, E, G, A, I, kappa = 1e-3, 10.0, 1.0, 0.5, 1.0, 1.0 / 12.0, 5.0 / 6.0
    assert abs(-uy[tip].mean() / (P * L ** 3 / (3 * E * I) + P * L / (kappa * G * A)) - 1.0) <= 1e-2
