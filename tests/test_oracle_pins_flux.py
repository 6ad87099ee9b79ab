"""Closed-form pins of the oracle's boundary and stabilisation *residuals* (VERDICT r1 "parity
unpinned" families): thermal conv-rad and FIX flux balances, the NS SUPG/PSPG/τ_c domain residual with
τ ≠ 0, and the NS BASE/OUTFLOW/FIX/INFLOW boundary residuals.

Method.  For a residual d_(a,κ) = ∫ v_a r(…) the weighted sum Σ_a c_a d_(a,κ) is the weak form evaluated
at the test function v = Σ_a c_a N_a.  With c_a = 1 (Σ_a N_a = 1, Σ_a ∇N_a = 0) or c_a = x_{a,k}
(Σ_a x_ak N_a = x_k, Σ_a x_ak ∇N_a = e_k — the isoparametric map reproduces linear functions) the sum is
a plain integral of a polynomial over a box face or the box, written out below in closed form.  States
are linear fields, which every element space here reproduces exactly, so the fields at the quadrature
points are exact.  Where the integrand has degree ≤ the rule's exactness the pin is exact to rounding;
where it does not (the inflow profile of P:1050 is degree 4), the pin is the closed-form integral
approached at the rule's convergence rate under refinement.

Meshes are the configs' boxes with *every* node jittered: interior nodes in all coordinates, boundary
nodes only tangentially (in the coordinates whose boundary planes they are not on), so boundary faces
stay planar (closed forms hold) but their facets are irregular (a wrong surface Jacobian or normal
fails).  Nothing here compares the oracle with itself.
"""
import math

import numpy as np
import pytest

import oracle
from fem_inputs import make_config as make_config_, make_state as make_state_
from fem_inputs.meshgen import facets_on_plane, hex_box, tet_box, tri_square
from helpers import problem

SIGMA_B = 5.670e-8


def jitter_all(mesh, amp, seed=5):
    """Jitter every node by U(-amp, amp)·h per coordinate, except along the normals of the box planes it
    lies on (boundary faces stay planar; facets become irregular)."""
    rng = np.random.default_rng(seed)
    c = mesh.coords.copy()
    lo, hi = c.min(axis=1), c.max(axis=1)
    n_per = [len(np.unique(np.round(c[d], 12))) - 1 for d in range(mesh.dim)]
    for d in range(mesh.dim):
        h = (hi[d] - lo[d]) / n_per[d]
        on = (np.abs(c[d] - lo[d]) <= 1e-12) | (np.abs(c[d] - hi[d]) <= 1e-12)
        c[d] += np.where(on, 0.0, rng.uniform(-amp, amp, c.shape[1]) * h)
    mesh.coords = np.ascontiguousarray(c)
    return mesh


def linear_state(mesh, kh, A, b):
    """state[0][κ] = b_κ + Σ_j A_κj x_j (linear fields, exactly reproduced by P1/Q1/P2)."""
    st = np.zeros((1, kh, mesh.n_nodes))
    st[0] = np.asarray(b)[:, None] + np.asarray(A) @ mesh.coords
    return st


def rhs(mesh, prob, st):
    out = oracle.assemble(mesh, prob, st, matrix=False)
    assert out["status"] == 0, out
    return out["rhs"].reshape(prob.kappa_hat(mesh.dim), mesh.n_nodes)


def face_moments(axis, value, lo, hi):
    """Closed-form ∫ 1, ∫ x_k, ∫ x_k x_l over the box face {x_axis = value} (a rectangle)."""
    dim = len(lo)
    t = [d for d in range(dim) if d != axis]
    area = float(np.prod([hi[d] - lo[d] for d in t]))
    m1 = np.zeros(dim)
    m2 = np.zeros((dim, dim))
    mean = np.array([(lo[d] + hi[d]) / 2 if d != axis else value for d in range(dim)])
    sq = np.array([(hi[d] ** 3 - lo[d] ** 3) / (3 * (hi[d] - lo[d])) if d != axis else value ** 2
                   for d in range(dim)])
    m1 = area * mean
    m2 = area * np.outer(mean, mean)
    for d in range(dim):
        m2[d, d] = area * sq[d]
    return area, m1, m2


# ------------------------------------------------------------------ meshes with single-face sets
def _mesh(etype):
    if etype == "hex":
        m = hex_box(4, 3, 5)
        lo, hi = np.zeros(3), np.ones(3)
    elif etype == "tet":
        m = tet_box(4, 3, 3, 2.5, 0.41, 0.41, order=1)
        lo, hi = np.zeros(3), np.array([2.5, 0.41, 0.41])
    else:
        m = tri_square(6)
        lo, hi = np.zeros(2), np.ones(2)
    return jitter_all(m, 0.2 if etype != "tet" else 0.12), lo, hi


FACES = [(0, "lo"), (0, "hi"), (1, "lo"), (2, "hi")]


def _face(m, lo, hi, axis, side):
    val = lo[axis] if side == "lo" else hi[axis]
    m.bsets = [facets_on_plane(m, axis, val)]
    assert len(m.bsets[0][0]) > 0
    n = np.zeros(m.dim)
    n[axis] = -1.0 if side == "lo" else 1.0
    return val, n


# ------------------------------------------------------------------ thermal conv-rad
@pytest.mark.parametrize("etype", ["hex", "tet", "tri"])
def test_conv_rad_flux_balance_constant_T(etype):
    """At constant T̃ = T0 the conv-rad integrand h(T_env − T) + e_m σ^b (T_env⁴ − T⁴) is a
    constant f, so Σ_a d_a = f·A and Σ_a x_ak d_a = f·∫x_k dA on every face (SPEC S:534 flux balance).
    The convective and radiative parts are pinned separately (h = 0 or e_m = 0) so a dropped e_m, a
    T − T_env sign or a missing σ^b fails."""
    m, lo, hi = _mesh(etype)
    for axis, side in FACES[: (2 * m.dim - 1)]:
        if axis >= m.dim:
            continue
        val, _ = _face(m, lo, hi, axis, side)
        A, m1, _ = face_moments(axis, val, lo, hi)
        T0, Te = 650.0, 293.15
        for h, em in ((25.0, 0.0), (0.0, 0.7), (25.0, 0.7)):
            pr = problem("thermal", etype, 1, [("THERMAL_CONV_RAD", 0,
                                                dict(h=h, T_env=Te, e_m=em, sigma_b=SIGMA_B))])
            st = np.full((1, 1, m.n_nodes), T0)
            d = rhs(m, pr, st)[0]
            f = h * (Te - T0) + em * SIGMA_B * (Te ** 4 - T0 ** 4)
            assert d.sum() == pytest.approx(f * A, rel=1e-12)
            for k in range(m.dim):
                assert (m.coords[k] * d).sum() == pytest.approx(f * m1[k], rel=1e-12, abs=1e-12 * abs(f) * A)


@pytest.mark.parametrize("etype", ["hex", "tet", "tri"])
def test_conv_linear_T_exact(etype):
    """Convection only (e_m = 0) with linear T = T0 + g·x: Σ_a d_a = h(T_env A − T0 A − g·∫x dA) and the
    x_k moments h(T_env ∫x_k − T0 ∫x_k − Σ_l g_l ∫x_k x_l) — degree-2 integrands, exact under the rules."""
    m, lo, hi = _mesh(etype)
    g = np.array([3.0, -5.0, 2.0])[: m.dim]
    T0, Te, h = 700.0, 293.15, 25.0
    for axis, side in FACES[:3]:
        val, _ = _face(m, lo, hi, axis, side)
        A, m1, m2 = face_moments(axis, val, lo, hi)
        pr = problem("thermal", etype, 1, [("THERMAL_CONV_RAD", 0,
                                            dict(h=h, T_env=Te, e_m=0.0, sigma_b=SIGMA_B))])
        d = rhs(m, pr, linear_state(m, 1, [g], [T0]))[0]
        assert d.sum() == pytest.approx(h * ((Te - T0) * A - g @ m1), rel=1e-12)
        for k in range(m.dim):
            ex = h * ((Te - T0) * m1[k] - g @ m2[k])
            assert (m.coords[k] * d).sum() == pytest.approx(ex, rel=1e-11, abs=1e-11 * h * Te * A)


# ------------------------------------------------------------------ thermal FIX
@pytest.mark.parametrize("etype", ["hex", "tet", "tri"])
def test_fix_flux_linear_T(etype):
    """FIX form h_p(T, T_fix − T) + k(T, n_i T_,i) with T = T0 + g·x: ∇T = g exactly (evaluated in
    the owning element from all its nodes, L18), so Σ_a d_a = h_p(T_fix A − T0 A − g·∫x) + k (g·n) A and
    Σ_a x_ak d_a = h_p(T_fix ∫x_k − T0 ∫x_k − g·∫x_k x) + k (g·n) ∫x_k, per single face.  A wrong normal
    sign, a dropped flux term or T=0-only testing (the r1 gap) fails here."""
    m, lo, hi = _mesh(etype)
    g = np.array([4.0, -3.0, 1.5])[: m.dim]
    T0, Tf, hp, k = 500.0, 1173.15, 7.0, 0.6
    for axis, side in FACES[:3]:
        val, n = _face(m, lo, hi, axis, side)
        A, m1, m2 = face_moments(axis, val, lo, hi)
        pr = problem("thermal", etype, 1, [("THERMAL_FIX", 0, dict(h_p=hp, T_fix=Tf, k=k))])
        d = rhs(m, pr, linear_state(m, 1, [g], [T0]))[0]
        flux = k * (g @ n)
        assert d.sum() == pytest.approx(hp * ((Tf - T0) * A - g @ m1) + flux * A, rel=1e-12)
        for kk in range(m.dim):
            ex = hp * ((Tf - T0) * m1[kk] - g @ m2[kk]) + flux * m1[kk]
            assert (m.coords[kk] * d).sum() == pytest.approx(ex, rel=1e-11, abs=1e-11 * hp * Tf * A)
        # the flux term alone (h_p = 0): k (g·n) A — nonzero only through ∇T at the facet points
        pr = problem("thermal", etype, 1, [("THERMAL_FIX", 0, dict(h_p=0.0, T_fix=Tf, k=k))])
        d = rhs(m, pr, linear_state(m, 1, [g], [T0]))[0]
        assert d.sum() == pytest.approx(flux * A, rel=1e-12)


# ------------------------------------------------------------------ NS domain with τ ≠ 0
def _box_moments(lo, hi):
    L = hi - lo
    vol = float(np.prod(L))
    mean = (lo + hi) / 2
    mxx = np.outer(mean, mean)
    for d in range(3):
        mxx[d, d] = (hi[d] ** 3 - lo[d] ** 3) / (3 * L[d])
    return vol, mean, mxx


def _E_lin_lin(vol, mean, mxx, a0, A, b0, B):
    """∫ (a0 + A x)_i (b0 + B x)_k over the box, as a matrix [i, k]."""
    return vol * (np.outer(a0, b0) + np.outer(a0, B @ mean) + np.outer(A @ mean, b0) + A @ mxx @ B.T)


def test_ns_domain_moments_with_stabilisation():
    """Linear u = u0 + A x, p = p0 + g·x and τ_m, τ_c ≠ 0.  Rm_i = ρ u_k u_i,k + p_,i = ρ (A u)_i + g_i
    (linear; μ u_i,kk = 0, L10), Rc = u_k,k = tr A.  Test functions x_k and 1 give
      Σ_a x_ak d_(a,i) = ∫ −ρ u_i u_k − δ_ik p + μ A_ik + τ_m ρ u_k Rm_i + τ_c δ_ik Rc,
      Σ_a d_(a,p)      = ∫ Rc,        Σ_a x_ak d_(a,p) = ∫ x_k Rc + τ_m Rm_k,
    all of degree ≤ 2, exact under the degree-2 tet rule on affine tets.  A transposed SUPG product
    (Rm_j u_i for Rm_i u_j) or a wrong τ_c placement fails."""
    m = jitter_all(tet_box(5, 3, 3, 2.5, 0.41, 0.41, order=1), 0.12)
    lo, hi = np.zeros(3), np.array([2.5, 0.41, 0.41])
    vol, mean, mxx = _box_moments(lo, hi)
    A = np.array([[0.3, -0.2, 0.5], [0.1, 0.4, -0.3], [-0.6, 0.2, 0.1]])
    u0 = np.array([0.2, -0.1, 0.3])
    g, p0 = np.array([0.5, -1.0, 2.0]), 0.7
    rho, mu, tm, tc = 2.0, 0.9, 0.37, 1.3
    st = linear_state(m, 4, np.vstack([A, g]), np.concatenate([u0, [p0]]))
    pr = problem("ns", "tet", 1, [("NS_DOMAIN", -1, dict(rho=rho, mu=mu, tau_m=tm, tau_c=tc))])
    d = rhs(m, pr, st)
    x = m.coords
    c, B = rho * A @ u0 + g, rho * A @ A          # Rm = c + B x
    Euu = _E_lin_lin(vol, mean, mxx, u0, A, u0, A)      # [i,k] ∫u_i u_k
    ERu = _E_lin_lin(vol, mean, mxx, c, B, u0, A)       # [i,k] ∫Rm_i u_k
    Ep = vol * (p0 + g @ mean)
    Rc = np.trace(A)
    scale = np.abs(d[:3]).max() * m.n_nodes
    for i in range(3):
        assert abs(d[i].sum()) <= 1e-12 * scale          # Σ_a ∇N_a = 0 kills every row-(a,i) term
        for k in range(3):
            ex = -rho * Euu[i, k] - (Ep if i == k else 0.0) + mu * A[i, k] * vol \
                + tm * rho * ERu[i, k] + (tc * Rc * vol if i == k else 0.0)
            assert (x[k] * d[i]).sum() == pytest.approx(ex, rel=1e-11, abs=1e-12 * scale)
    assert d[3].sum() == pytest.approx(Rc * vol, rel=1e-12)
    ERm = vol * (c + B @ mean)
    for k in range(3):
        assert (x[k] * d[3]).sum() == pytest.approx(Rc * vol * mean[k] + tm * ERm[k], rel=1e-11)


# ------------------------------------------------------------------ NS boundary
def _ns_channel(ny=3, seed=5):
    m = jitter_all(tet_box(3, ny, ny, 2.5, 0.41, 0.41, order=1), 0.12, seed)
    return m, np.zeros(3), np.array([2.5, 0.41, 0.41])


NSP = dict(rho=2.0, mu=0.9)
A_U = np.array([[0.3, -0.2, 0.5], [0.1, 0.4, -0.3], [-0.6, 0.2, 0.1]])
U0, G_P, P0 = np.array([0.2, -0.1, 0.3]), np.array([0.5, -1.0, 2.0]), 0.7


def _lin_ns_state(m):
    return linear_state(m, 4, np.vstack([A_U, G_P]), np.concatenate([U0, [P0]]))


def _face_E(axis, val, lo, hi):
    """Face moments as a 3D 'box' with zero thickness: ∫1, ∫x, ∫x xᵀ."""
    A, m1, m2 = face_moments(axis, val, lo, hi)
    return A, m1, m2


def _base_expected(A, m1, m2, n, mu):
    """BASE (every boundary group): row (a,i) N_a (p n_i − μ u_i,j n_j).
    Returns (Σ_a d_(a,i), Σ_a x_ak d_(a,i)) as (3,), (3,3)[i,k]."""
    Ip = P0 * A + G_P @ m1                       # ∫ p
    Ixp = P0 * m1 + m2 @ G_P                     # ∫ x_k p
    s = Ip * n - mu * (A_U @ n) * A
    mom = np.outer(n, Ixp) - mu * np.outer(A_U @ n, m1)
    return s, mom


def test_ns_outflow_residual_closed_form():
    """OUTFLOW = BASE + ρ(u_i, u_i u_j n_j) on x = 2.5 (n = +x̂): Σ_a d_(a,i) = ∫ p n_i − μ A_ij n_j +
    ρ u_i (u·n); pressure rows get nothing.  Degree ≤ 2, exact."""
    m, lo, hi = _ns_channel()
    val, n = _face(m, lo, hi, 0, "hi")
    A, m1, m2 = _face_E(0, val, lo, hi)
    pr = problem("ns", "tet", 1, [("NS_BND_OUTFLOW", 0, dict(NSP))])
    d = rhs(m, pr, _lin_ns_state(m))
    s, _ = _base_expected(A, m1, m2, n, NSP["mu"])
    Iuu = A * np.outer(U0, U0) + np.outer(U0, A_U @ m1) + np.outer(A_U @ m1, U0) + A_U @ m2 @ A_U.T
    ex = s + NSP["rho"] * Iuu @ n
    np.testing.assert_allclose(d[:3].sum(axis=1), ex, rtol=1e-12, atol=1e-13 * np.abs(ex).max())
    assert np.abs(d[3]).max() == 0.0


@pytest.mark.parametrize("form", ["NS_BND_FIX", "NS_BND_INFLOW"])
def test_ns_fix_and_zero_inflow_residual_closed_form(form):
    """FIX = BASE + μ(u_i,j, −u_i n_j) + τ_b ρ(u_i, u_i), pressure row (p, −u·n).
    INFLOW with U = 0 has u^w = 0 and reduces to the same expression.  On the wall y = 0
    (n = −ŷ) with linear u, p: Σ_a d_(a,i) = ∫ p n_i − μ A_ij n_j + τ_b ρ u_i (Σ_a ∇N_a = 0),
    Σ_a x_ak d_(a,i) adds −μ n_k ∫u_i (Σ_a x_ak ∇N_a = e_k), Σ_a d_(a,p) = −∫u·n,
    Σ_a x_ak d_(a,p) = −∫x_k u·n.  Degree ≤ 2, exact."""
    m, lo, hi = _ns_channel()
    val, n = _face(m, lo, hi, 1, "lo")
    A, m1, m2 = _face_E(1, val, lo, hi)
    tb = 3.1
    prm = dict(NSP, tau_b=tb) if form == "NS_BND_FIX" else dict(NSP, tau_b=tb, U=0.0, H=0.41)
    pr = problem("ns", "tet", 1, [(form, 0, prm)])
    d = rhs(m, pr, _lin_ns_state(m))
    rho, mu = NSP["rho"], NSP["mu"]
    s, mom = _base_expected(A, m1, m2, n, mu)
    Iu = U0 * A + A_U @ m1                               # ∫ u_i
    Ixu = np.outer(U0, m1) + A_U @ m2                    # [i,k] ∫ u_i x_k
    ex = s + tb * rho * Iu
    exm = mom - mu * np.outer(Iu, n) + tb * rho * Ixu
    x = m.coords
    sc = np.abs(ex).max() + np.abs(exm).max()
    np.testing.assert_allclose(d[:3].sum(axis=1), ex, rtol=1e-11, atol=1e-12 * sc)
    for k in range(3):
        np.testing.assert_allclose((x[k] * d[:3]).sum(axis=1), exm[:, k], rtol=1e-11, atol=1e-12 * sc)
    assert d[3].sum() == pytest.approx(-(Iu @ n), rel=1e-12)
    for k in range(3):
        assert (x[k] * d[3]).sum() == pytest.approx(-(Ixu[:, k] @ n), rel=1e-11, abs=1e-13)


def test_ns_inflow_profile_converges_to_closed_form():
    """INFLOW with the profile u^w = (16U(H−y)(H−z)yz/H⁴, 0, 0) at u = 0, p = 0 on x = 0 (n = −x̂):
      Σ_a d_(a,1) = −ρ∫u^w₁² − τ_b ρ ∫u^w₁ = −ρ·256U²H²/900 − τ_b ρ·4UH²/9,
      Σ_a d_(a,p) = ∫u^w·n = −4UH²/9,   Σ_a x_a1 d_(a,1) = μ n₁∫u^w₁ = −μ·4UH²/9,
    (∫₀ᴴ(H−y)y dy = H³/6, ∫₀ᴴ(H−y)²y² dy = H⁵/30).  The integrand is degree 4 (8 for u^w²) and the facet
    rule has degree 2, so the pin is convergence to the closed form at the composite rule's rate
    (≥ 2.5 observed; the theory gives 3 on uniform refinements)."""
    U, H, rho, mu, tb = 0.45, 0.41, 2.0, 0.9, 3.1
    ex = np.array([-rho * 256 * U * U * H * H / 900 - tb * rho * 4 * U * H * H / 9,
                   -4 * U * H * H / 9, -mu * 4 * U * H * H / 9])
    errs = []
    for ny in (2, 4, 8, 16):
        m = tet_box(1, ny, ny, 2.5, H, H, order=1)
        m.bsets = [facets_on_plane(m, 0, 0.0)]
        pr = problem("ns", "tet", 1, [("NS_BND_INFLOW", 0, dict(rho=rho, mu=mu, tau_b=tb, U=U, H=H))])
        d = rhs(m, pr, np.zeros((1, 4, m.n_nodes)))
        got = np.array([d[0].sum(), d[3].sum(), (m.coords[0] * d[0]).sum()])
        assert np.abs(d[1:3]).max() == 0.0
        errs.append(np.abs(got - ex) / np.abs(ex))
    errs = np.array(errs)
    assert errs[-1].max() < 2e-3, errs
    rates = np.log2(errs[:-1] / errs[1:])
    assert rates[1:].min() >= 2.5, (errs, rates)


def test_ns_jacobian_has_the_constant_pressure_null_vector():
    """Reading L29 (pinned on the oracle): with NS_boundary_BASE on every boundary group a constant
    pressure drops out of every row: K·[0; 1] = 0 to rounding, so the Newton system needs a pressure gauge."""
    m, p = make_config_("c4", "perturbed", (6, 3, 3))
    st = make_state_("c4", m, p)
    ora = oracle.assemble(m, p, st)
    import scipy.sparse as sp
    n = len(ora["rowptr"]) - 1
    K = sp.csr_matrix((ora["values"], ora["colidx"], ora["rowptr"]), shape=(n, n))
    N = m.n_nodes
    e = np.zeros(4 * N)
    e[3 * N:] = 1.0
    assert np.abs(K @ e).max() <= 1e-10 * abs(K).max()
