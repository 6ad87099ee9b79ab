"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every test here runs on CPU (`-m "not gpu"`).  None of them compares the oracle with itself:
they use closed-form element matrices (tests/golden), exact integrals of polynomials,
invariants (row sums, rigid modes, symmetry, definiteness), brute-force pattern enumeration,
finite differences of the residual, and a manufactured-solution convergence rate.
"""
import itertools
import math

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
from fem_inputs import make_config, make_state
from fem_inputs.configs import TimeScheme, ns_tau
from fem_inputs.meshgen import facets_on_plane, hex_box, perturb_and_permute, tet_box, tri_square
from helpers import (HEX_CORNERS, REF_TET, REF_TRI, frac, golden, one_element, p2_tet_coords,
                     problem)

G = golden("element_matrices.json")


def dense_K(m, prob, state=None, **kw):
    kh = prob.kappa_hat(m.dim)
    st = np.zeros((prob.time.nu_hat + 1, kh, m.n_nodes)) if state is None else state
    out = oracle.assemble(m, prob, st, **kw)
    assert out["status"] == 0, out
    return oracle.to_dense(out, kh * m.n_nodes), out


def lap(etype, order, k=1.0, q=2):
    return problem("thermal", etype, order, [("THERMAL_DOMAIN", -1, dict(C=0.0, k=k, s=0.0))], q)


# ----------------------------------------------------------------- quadrature and geometry
@pytest.mark.parametrize("name,dims,measure", [
    ("c1", (5,), 1.0), ("c2", (3, 4, 5), 1.0), ("c3", (7, 2, 3), 10.0),
    ("c4", (6, 3, 2), 2.5 * 0.41 ** 2), ("c5", (4, 3, 2), 1.0)])
@pytest.mark.parametrize("variant", ["structured", "perturbed"])
def test_measure_partition_of_unity(name, dims, measure, variant):
    """Σ_e Σ_q w = |Ω| (L1: physical weight); Σ_a N_a = 1, Σ_a ∇N_a = 0 at every qp."""
    m, p = make_config(name, variant, dims)
    tot = 0.0
    for e in range(m.n_elems):
        d = oracle.qp_data(m, p, e)
        tot += d["w"].sum()
        np.testing.assert_allclose(d["N"].sum(axis=1), 1.0, atol=1e-13)
        np.testing.assert_allclose(d["G"].sum(axis=1), 0.0, atol=1e-10)
    assert abs(tot - measure) <= 1e-13 * measure * 10


def _exact_monomial(etype, p):
    """Exact ∫ x^p0 y^p1 (z^p2) over the reference triangle / tet (Dirichlet formula) or [-1,1]^3."""
    if etype == "hex":
        return np.prod([0.0 if k % 2 else 2.0 / (k + 1) for k in p])
    n = len(p)
    return math.prod(math.factorial(k) for k in p) / math.factorial(sum(p) + n)


@pytest.mark.parametrize("etype,coords,deg", [
    ("tri", REF_TRI, 2), ("tet", REF_TET, 2), ("hex", 2 * HEX_CORNERS - 1, 3)])
def test_quadrature_exactness(etype, coords, deg):
    """The volume rule integrates every monomial of total degree <= deg exactly."""
    m = one_element(etype, 1, coords)
    d = oracle.qp_data(m, lap(etype, 1), 0)
    dim = coords.shape[0]
    for p in itertools.product(range(deg + 1), repeat=dim):
        if sum(p) > deg and etype != "hex":
            continue
        if etype == "hex" and max(p) > deg:
            continue
        val = (d["w"] * np.prod(d["x"][:, :dim] ** np.array(p), axis=1)).sum()
        assert abs(val - _exact_monomial(etype, p)) < 1e-14, p


@pytest.mark.parametrize("name,dims", [("c1", (4,)), ("c2", (3, 3, 3)), ("c3", (5, 2, 2)),
                                       ("c4", (5, 2, 2)), ("c5", (3, 3, 3))])
@pytest.mark.parametrize("variant", ["structured", "perturbed"])
def test_facet_measure_and_normals(name, dims, variant):
    """Facet weights sum to the face area; the unit normal is the outward plane normal."""
    m, p = make_config(name, variant, dims)
    lo, hi = m.coords.min(axis=1), m.coords.max(axis=1)
    for axis in range(m.dim):
        for side, val in ((-1.0, lo[axis]), (1.0, hi[axis])):
            be, bf = facets_on_plane(m, axis, val)
            area = 0.0
            for e, f in zip(be, bf):
                d = oracle.qp_data(m, p, int(e), int(f))
                area += d["w"].sum()
                expect = np.zeros(3)
                expect[axis] = side
                np.testing.assert_allclose(d["n"], np.tile(expect, (len(d["w"]), 1)), atol=1e-13)
                np.testing.assert_allclose(d["x"][:, axis], val, atol=1e-13)
            other = [hi[k] - lo[k] for k in range(m.dim) if k != axis]
            assert abs(area - np.prod(other)) < 1e-12 * max(1.0, np.prod(other))


# ----------------------------------------------------------------- closed-form element matrices
@pytest.mark.parametrize("h", [1.0, 0.25, 3.0])
def test_p1_triangle_laplacian_and_mass(h):
    g = G["p1_tri_laplacian_right_angle"]
    m = one_element("tri", 1, REF_TRI * h)
    K, _ = dense_K(m, lap("tri", 1, k=1.7))
    np.testing.assert_allclose(K, -1.7 * np.vectorize(frac)(np.array(g["K"])), atol=1e-14)
    # transient: -C(T, T_t) -> K = -C f1 M with f1 = c2/(b1 dt)  (Eq. gen_alpha)
    ts = TimeScheme("genalpha", 1, dt=0.1, b1=0.5, b2=0.5, c1=0.8, c2=0.6, c3=1.0)
    pr = problem("thermal", "tri", 1, [("THERMAL_DOMAIN", -1, dict(C=2.0, k=0.0, s=0.0))], time=ts)
    K, _ = dense_K(m, pr)
    f1 = 0.6 / (0.5 * 0.1)
    M = np.vectorize(frac)(np.array(G["p1_tri_mass_leg_h_over_h2"]["M"])) * h * h
    np.testing.assert_allclose(K, -2.0 * f1 * M, rtol=1e-13, atol=1e-15)


def test_c1_interior_stencil():
    """Pin P1: the assembled c1 Laplacian interior row is -k·(4,-1,-1,-1,-1) (5-point stencil)
    with the two diagonal neighbours present in the pattern and 0 (up to quadrature rounding)."""
    m, p = make_config("c1")
    K, out = dense_K(m, p)
    n = 8
    for i, j in [(1, 1), (4, 4), (3, 6), (7, 7)]:
        r = i + (n + 1) * j
        cols = out["colidx"][out["rowptr"][r]:out["rowptr"][r + 1]]
        assert len(cols) == 7
        expect = {r: -4.0, r - 1: 1.0, r + 1: 1.0, r - 9: 1.0, r + 9: 1.0, r - 10: 0.0, r + 10: 0.0}
        assert set(cols.tolist()) == set(expect)
        for c, v in expect.items():
            assert K[r, c] == pytest.approx(v, abs=1e-13)


@pytest.mark.parametrize("h", [1.0, 0.5])
def test_q1_hex_mass_and_laplacian_rows(h):
    m = one_element("hex", 1, HEX_CORNERS * h)
    K, _ = dense_K(m, lap("hex", 1, k=1.0))
    row = np.array([frac(x) for x in G["q1_hex_laplacian_row0_over_h"]["row"]]) * h
    np.testing.assert_allclose(K[0], -row, atol=1e-15)
    assert K[0, 1] == 0.0 or abs(K[0, 1]) < 1e-16
    ts = TimeScheme("genalpha", 1, dt=1.0, b1=1.0, b2=1.0, c1=1.0, c2=1.0, c3=1.0)
    pr = problem("thermal", "hex", 1, [("THERMAL_DOMAIN", -1, dict(C=1.0, k=0.0, s=0.0))], time=ts)
    K, _ = dense_K(m, pr)
    mrow = np.array([frac(x) for x in G["q1_hex_mass_row0_over_h3"]["row"]]) * h ** 3
    np.testing.assert_allclose(K[0], -mrow, rtol=1e-13)


def test_c2_assembled_interior_row():
    """Pin P3 (assembled): centre 8h/3, face 0, edge -h/6, corner -h/12 (times -k)."""
    n = 6
    m = hex_box(n, n, n)
    h, k = 1.0 / n, 0.6
    K, _ = dense_K(m, lap("hex", 1, k=k))
    g = G["q1_hex_laplacian_assembled_interior_over_h"]
    nid = lambda i, j, l: i + (n + 1) * (j + (n + 1) * l)  # noqa: E731
    r = nid(3, 2, 4)
    for di, dj, dl in itertools.product((-1, 0, 1), repeat=3):
        c = nid(3 + di, 2 + dj, 4 + dl)
        kind = {0: "centre", 1: "face", 2: "edge", 3: "corner"}[abs(di) + abs(dj) + abs(dl)]
        assert K[r, c] == pytest.approx(-k * h * frac(g[kind]), abs=1e-14)


def test_tet_laplacians_reference():
    m = one_element("tet", 1, REF_TET)
    K, _ = dense_K(m, lap("tet", 1))
    np.testing.assert_allclose(K, -np.vectorize(frac)(np.array(G["p1_tet_laplacian_reference"]["K"])),
                               atol=1e-15)
    m2 = one_element("tet", 2, p2_tet_coords(REF_TET))
    K2, _ = dense_K(m2, lap("tet", 2))
    g = G["p2_tet_laplacian_reference"]
    np.testing.assert_allclose(K2[0], -np.array([frac(x) for x in g["row0"]]), atol=1e-14)
    np.testing.assert_allclose(K2[4], -np.array([frac(x) for x in g["row4"]]), atol=1e-14)
    np.testing.assert_allclose(K2.sum(axis=1), 0.0, atol=1e-14)


@pytest.mark.parametrize("h", [1.0, 2.0])
def test_q1_hex_elasticity_entries(h):
    E, nu = 1.3, 0.27
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    m = one_element("hex", 1, HEX_CORNERS * h)
    pr = problem("elasticity", "hex", 1, [("ELAST_DOMAIN", -1, dict(E=E, nu=nu))])
    K, _ = dense_K(m, pr)
    N = 8
    for ent in G["q1_hex_elasticity_over_h"]["entries"]:
        r = ent["i"] * N + ent["a"]
        c = ent["m"] * N + ent["b"]
        expect = h * (frac(ent["lam"]) * lam + frac(ent["mu"]) * mu)
        assert K[r, c] == pytest.approx(-expect, rel=1e-13)


# ----------------------------------------------------------------- invariants
@pytest.mark.parametrize("name,dims", [("c1", (6,)), ("c2", (3, 4, 2)), ("c3", (4, 2, 2)),
                                       ("c4", (4, 2, 3))])
def test_laplacian_row_sums_zero_perturbed(name, dims):
    m, p = make_config(name, "perturbed", dims)
    K, _ = dense_K(m, lap(m.etype, m.order))
    np.testing.assert_allclose(K.sum(axis=1), 0.0, atol=1e-12 * np.abs(K).max())


def _rigid_modes(x):
    N = x.shape[1]
    modes = []
    for i in range(3):
        r = np.zeros((3, N))
        r[i] = 1.0
        modes.append(r.ravel())
    for (i, j) in [(0, 1), (1, 2), (0, 2)]:
        r = np.zeros((3, N))
        r[i] = -x[j]
        r[j] = x[i]
        modes.append(r.ravel())
    return modes


@pytest.mark.parametrize("name,dims", [("c3", (3, 2, 2)), ("c5", (3, 2, 2))])
def test_elasticity_rigid_modes_symmetry_definiteness(name, dims):
    m, p = make_config(name, "perturbed", dims)
    dom = problem("elasticity", m.etype, m.order, [("ELAST_DOMAIN", -1, dict(E=1.0, nu=0.3))])
    K, _ = dense_K(m, dom)
    scale = np.abs(K).max()
    for r in _rigid_modes(m.coords):
        assert np.abs(K @ r).max() < 1e-12 * scale * np.abs(r).max()
    np.testing.assert_allclose(K, K.T, atol=1e-14 * scale)
    ev = np.linalg.eigvalsh(-K)
    assert ev.min() > -1e-12 * scale
    assert np.sum(ev < 1e-10 * scale) == 6  # exactly the 6 rigid modes are in the kernel


def test_ns_stokes_special_case():
    """At u = 0, p = 0, τ = 0: uu = μ·(vector Laplacian), up = -Bᵀ-type, pu = +B (B_ab,m = ∫N_a G_bm);
    with τ_m > 0, pp = τ_m·Laplacian (SURVEY §8(c) NS special case)."""
    m, _ = make_config("c4", "perturbed", (2, 2, 2))
    N = m.n_nodes
    mu = 1.7
    pr = problem("ns", "tet", 1, [("NS_DOMAIN", -1, dict(rho=3.0, mu=mu, tau_m=0.0, tau_c=0.0))])
    K, _ = dense_K(m, pr)
    L, _ = dense_K(m, lap("tet", 1))  # L = -∫∇N_a·∇N_b
    for i in range(3):
        np.testing.assert_allclose(K[i * N:(i + 1) * N, i * N:(i + 1) * N], -mu * L, atol=1e-12)
        for j in range(3):
            if j != i:
                assert np.abs(K[i * N:(i + 1) * N, j * N:(j + 1) * N]).max() < 1e-12
    # B_ab,m = ∫ N_a G_bm via an independent route: sum over elements of qp data
    B = np.zeros((3, N, N))
    for e in range(m.n_elems):
        d = oracle.qp_data(m, pr, e)
        nodes = m.conn[:, e]
        for q in range(len(d["w"])):
            for i in range(3):
                B[i][np.ix_(nodes, nodes)] += d["w"][q] * np.outer(d["N"][q], d["G"][q][:, i])
    for i in range(3):
        np.testing.assert_allclose(K[3 * N:, i * N:(i + 1) * N], B[i], atol=1e-12)      # pu = +B
        np.testing.assert_allclose(K[i * N:(i + 1) * N, 3 * N:], -B[i].T, atol=1e-12)   # up = -Bᵀ
    assert np.abs(K[3 * N:, 3 * N:]).max() == 0.0
    tm = 0.37
    pr2 = problem("ns", "tet", 1, [("NS_DOMAIN", -1, dict(rho=3.0, mu=mu, tau_m=tm, tau_c=0.0))])
    K2, _ = dense_K(m, pr2)
    np.testing.assert_allclose(K2[3 * N:, 3 * N:], -tm * L, atol=1e-12)


def test_ns_residual_moments_linear_fields():
    """For linear u, p and τ = 0, Σ_a x_{a,k} d_(a,i) = ∫(-ρ u_i u_k - δ_ik p + μ u_i,k) and
    Σ_a d_(a,p) = ∫ div u (Σ_a N_a = 1, Σ_a x_ak G_aj = δ_kj; degree-2 rule exact on P1)."""
    m, _ = make_config("c4", "perturbed", (3, 2, 2))
    x = m.coords
    N = m.n_nodes
    A = np.array([[0.3, -0.2, 0.5], [0.1, 0.4, -0.3], [-0.6, 0.2, 0.1]])
    u0 = np.array([0.2, -0.1, 0.3])
    pg, p0 = np.array([0.5, -1.0, 2.0]), 0.7
    st = np.zeros((1, 4, N))
    st[0, :3] = u0[:, None] + A @ x
    st[0, 3] = p0 + pg @ x
    rho, mu = 2.0, 0.9
    pr = problem("ns", "tet", 1, [("NS_DOMAIN", -1, dict(rho=rho, mu=mu, tau_m=0.0, tau_c=0.0))])
    out = oracle.assemble(m, pr, st, matrix=False)
    d = out["rhs"].reshape(4, N)
    # exact integrals over the box [0,2.5]x[0,.41]^2 of polynomials of degree <= 2
    Lb = np.array([2.5, 0.41, 0.41])
    vol = Lb.prod()
    mean_x = Lb / 2
    mean_xx = np.outer(Lb, Lb) / 4 + np.diag(Lb ** 2 / 12)
    # ∫ u_i u_k = ∫ (u0 + A x)_i (u0 + A x)_k
    Euu = vol * (np.outer(u0, u0) + np.outer(u0, A @ mean_x) + np.outer(A @ mean_x, u0) + A @ mean_xx @ A.T)
    Ep = vol * (p0 + pg @ mean_x)
    for i in range(3):
        for k in range(3):
            got = (x[k] * d[i]).sum()
            expect = -rho * Euu[i, k] - (Ep if i == k else 0.0) + mu * A[i, k] * vol
            assert got == pytest.approx(expect, rel=1e-11, abs=1e-12)
    assert d[3].sum() == pytest.approx(np.trace(A) * vol, rel=1e-12)


# ----------------------------------------------------------------- residual vs matrix
def test_linear_consistency_thermal_and_elasticity():
    """For forms linear in φ: d(φ) - d(0) = K φ (pins the residual against the matrix)."""
    for name, dims in [("c1", (5,)), ("c3", (3, 2, 2)), ("c5", (3, 2, 2))]:
        m, p = make_config(name, "perturbed", dims)
        st = make_state(name, m, p)
        K, out1 = dense_K(m, p, st)
        out0 = oracle.assemble(m, p, np.zeros_like(st))
        lhs = out1["rhs"] - out0["rhs"]
        rhs = K @ st[0].ravel()
        assert np.abs(lhs - rhs).max() < 1e-12 * max(np.abs(out1["abs_d"]).max(), 1e-30)


def _fd_check(m, p, st, eps_rel=1e-6, cols=None, f=None):
    """Central FD of the residual along the Newton direction vs K columns."""
    K, _ = dense_K(m, p, st)
    kh = p.kappa_hat(m.dim)
    n = kh * m.n_nodes
    cols = range(n) if cols is None else cols
    f = f or [1.0]
    worst = 0.0
    for c in cols:
        k, a = divmod(c, m.n_nodes)
        h = eps_rel * max(1.0, abs(st[0, k, a]))
        sp_, sm_ = st.copy(), st.copy()
        for lev, fl in enumerate(f):
            sp_[lev, k, a] += fl * h
            sm_[lev, k, a] -= fl * h
        dp = oracle.assemble(m, p, sp_, matrix=False)["rhs"]
        dm = oracle.assemble(m, p, sm_, matrix=False)["rhs"]
        fd = (dp - dm) / (2 * h)
        scale = max(np.abs(K[:, c]).max(), np.abs(fd).max(), 1e-30)
        worst = max(worst, np.abs(fd - K[:, c]).max() / scale)
    return worst


def test_fd_tangent_radiation():
    m, p = make_config("c2", "perturbed", (2, 2, 2))
    st = make_state("c2", m, p)
    assert _fd_check(m, p, st) < 1e-6


def test_fd_tangent_ns_all_terms():
    m, p = make_config("c4", "perturbed", (2, 2, 2))
    st = make_state("c4", m, p)
    # make the nonlinear/stabilisation terms significant at this tiny size
    for t in p.terms:
        if t.form == "NS_DOMAIN":
            t.params = dict(t.params, tau_m=1e-3, tau_c=0.5)
    assert _fd_check(m, p, st, cols=range(0, 4 * m.n_nodes, 3)) < 1e-6


def test_fd_tangent_genalpha_time_factor():
    """K = c1 ∂d/∂T̃ + c2/(b1Δt) ∂d/∂Ṫ̃ (Eq. gen_alpha): FD along (c1, f1) in (T̃, Ṫ̃)."""
    m, p = make_config("c2", "perturbed", (2, 2, 2))
    ts = TimeScheme("genalpha", 1, dt=0.05, b1=0.6, b2=0.5, c1=0.7, c2=0.8, c3=1.0)
    p.time = ts
    p.terms[0].params = dict(p.terms[0].params, C=3.0)
    st = make_state("c2", m, p)
    f = [0.7, 0.8 / (0.6 * 0.05)]
    assert _fd_check(m, p, st, f=f) < 1e-6


# ----------------------------------------------------------------- boundary forms
def test_penalty_and_load_totals():
    """Σ_a d_a of the fix form at T = 0, T_fix = 1 equals h_p·|∂Ω| (Σ N_a = 1); the elasticity load
    sums to the traction × area; fix-d1 acts on component 1 only."""
    m, _ = make_config("c1", "perturbed", (6,))
    pr = problem("thermal", "tri", 1, [("THERMAL_FIX", 0, dict(h_p=7.0, T_fix=1.0, k=1.0))])
    out = oracle.assemble(m, pr, np.zeros((1, 1, m.n_nodes)))
    assert out["rhs"].sum() == pytest.approx(7.0 * 4.0, rel=1e-13)
    m, p = make_config("c5", "perturbed", (3, 3, 2))
    out = oracle.assemble(m, p, np.zeros((1, 3, m.n_nodes)))
    d = out["rhs"].reshape(3, -1)
    np.testing.assert_allclose(d.sum(axis=1), [0.0, 0.0, -1e-3], atol=1e-16)
    pr = problem("elasticity", "hex", 1, [("ELAST_FIX_D1", 0, dict(tau=5.0, dw=(2.0,)))])
    out = oracle.assemble(m, pr, np.zeros((1, 3, m.n_nodes)))
    d = out["rhs"].reshape(3, -1)
    assert d[0].sum() == pytest.approx(5.0 * 2.0 * 1.0, rel=1e-13)
    assert np.abs(d[1:]).max() == 0.0


# ----------------------------------------------------------------- pattern
def _brute_pattern(m, kh):
    pairs = set()
    for e in range(m.n_elems):
        nodes = m.conn[:, e].tolist()
        for a in nodes:
            for b in nodes:
                pairs.add((a, b))
    rows = {}
    for a, b in pairs:
        rows.setdefault(a, []).append(b)
    N = m.n_nodes
    rowptr, col = [0], []
    for k0 in range(kh):
        for a in range(N):
            r = sorted(rows.get(a, []))
            for kl in range(kh):
                col += [kl * N + b for b in r]
            rowptr.append(len(col))
    return np.array(rowptr), np.array(col)


@pytest.mark.parametrize("name,dims", [("c1", (8,)), ("c2", (3, 2, 2)), ("c3", (2, 2, 1)),
                                       ("c4", (3, 2, 2)), ("c5", (2, 2, 2))])
def test_pattern_brute_force_and_slot_definition(name, dims):
    m, p = make_config(name, "perturbed", dims)
    kh = p.kappa_hat(m.dim)
    out = oracle.assemble(m, p, make_state(name, m, p), slot=True)
    rp, ci = _brute_pattern(m, kh)
    np.testing.assert_array_equal(out["rowptr"], rp)
    np.testing.assert_array_equal(out["colidx"], ci)
    # slot definition: colidx_s[slot_s[a*n+b][e]] == α(e,b) within scalar row α(e,a)
    n = m.n_loc
    for a in range(n):
        for b in range(n):
            s = out["slot_s"][a * n + b]
            np.testing.assert_array_equal(out["colidx_s"][s], m.conn[b])
            rows = np.searchsorted(out["rowptr_s"], s, side="right") - 1
            np.testing.assert_array_equal(rows, m.conn[a])
    if name == "c1":
        assert out["values"].size == 497


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_q1_scalar_nnz_closed_form(n):
    m = hex_box(n, n, n)
    out = oracle.assemble(m, lap("hex", 1), np.zeros((1, 1, m.n_nodes)), matrix=True, residual=False)
    assert out["colidx_s"].size == (3 * n + 1) ** 3


def test_row_subset_equals_full():
    """Row-window mode (used for full-size sampled parity) returns exactly the selected full rows."""
    m, p = make_config("c4", "perturbed", (3, 2, 2))
    st = make_state("c4", m, p)
    full = oracle.assemble(m, p, st)
    rng = np.random.default_rng(0)
    mask = rng.random(m.n_nodes) < 0.3
    sub = oracle.assemble(m, p, st, row_mask=mask)
    Ff = oracle.to_dense(full, 4 * m.n_nodes)
    Fs = oracle.to_dense(sub, 4 * m.n_nodes)
    np.testing.assert_array_equal(Fs, Ff[sub["rows"]])
    np.testing.assert_array_equal(sub["rhs"], full["rhs"][sub["rows"]])


def test_inverted_element_reported():
    m = one_element("tet", 1, REF_TET[:, [0, 2, 1, 3]])
    out = oracle.assemble(m, lap("tet", 1), np.zeros((1, 1, 4)))
    assert out["status"] == -4 and out["bad_elem"] == 0


# ----------------------------------------------------------------- end to end
def _manufactured_error(n, etype):
    if etype == "tri":
        m = tri_square(n)
        be = [facets_on_plane(m, a, v) for a in (0, 1) for v in (0.0, 1.0)]
        terms = [("THERMAL_DOMAIN", -1, dict(C=0.0, k=1.0, s=2 * math.pi ** 2, source="sine"))]
        exact = lambda x: np.sin(np.pi * x[0]) * np.sin(np.pi * x[1])  # noqa: E731
        dim = 2
    else:
        m = hex_box(n, n, n)
        be = [facets_on_plane(m, a, v) for a in (0, 1, 2) for v in (0.0, 1.0)]
        terms = [("THERMAL_DOMAIN", -1, dict(C=0.0, k=1.0, s=3 * math.pi ** 2, source="sine"))]
        exact = lambda x: np.sin(np.pi * x[0]) * np.sin(np.pi * x[1]) * np.sin(np.pi * x[2])  # noqa: E731
        dim = 3
    m.bsets = [(np.concatenate([b[0] for b in be]), np.concatenate([b[1] for b in be]))]
    terms.append(("THERMAL_FIX", 0, dict(h_p=1e8 * n, T_fix=0.0, k=1.0)))  # L22 penalty 1e8·k/h
    pr = problem("thermal", etype, 1, terms)
    out = oracle.assemble(m, pr, np.zeros((1, 1, m.n_nodes)))
    K = sp.csr_matrix((out["values"], out["colidx"], out["rowptr"]), shape=(m.n_nodes,) * 2)
    T = spla.spsolve(K.tocsc(), -out["rhs"])  # Newton from T = 0: K ΔT = -d
    # L2 error by the element quadrature (mass-weighted nodal error is enough for the rate)
    err2 = 0.0
    for e in range(0, m.n_elems):
        d = oracle.qp_data(m, pr, e)
        Th = d["N"] @ T[m.conn[:, e]]
        err2 += (d["w"] * (Th - exact(d["x"][:, :dim].T)) ** 2).sum()
    return math.sqrt(err2)


@pytest.mark.parametrize("etype,ns", [("tri", (8, 16, 32)), ("hex", (4, 8))])
def test_manufactured_convergence_rate(etype, ns):
    errs = [_manufactured_error(n, etype) for n in ns]
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert all(1.8 < r < 2.3 for r in rates), (errs, rates)


def test_ns_tau_reading_L11():
    tm, tc, tb = ns_tau()
    assert tm == pytest.approx(4.802068e-6, rel=1e-6)
    assert tc == pytest.approx(1.246622, rel=1e-6)
    assert tb == pytest.approx(18.0488, rel=1e-5)


def test_cantilever_deflection_timoshenko():
    """NEXT-1 pin of the oracle: the c3 beam (P2 tets, ν = 0 as the paper's beam P:944) under the end load
    P = 1e-3 deflects by P L³/(3 E I) + P L/(κ G A), I = h⁴/12 (reading L24), κ = 5/6."""
    import scipy.sparse as sp
    m, p = make_config("c3", "structured", (20, 2, 2))
    p.terms[0].params = dict(E=1.0, nu=0.0)
    out = oracle.assemble(m, p, np.zeros((1, 3, m.n_nodes)))
    n = len(out["rowptr"]) - 1
    K = sp.csr_matrix((out["values"], out["colidx"], out["rowptr"]), shape=(n, n))
    x = spla.spsolve(K.tocsc(), -out["rhs"])
    uy = x[m.n_nodes:2 * m.n_nodes]
    tip = np.isclose(m.coords[0], 10.0)
    P, L, E, G, A, I, kappa = 1e-3, 10.0, 1.0, 0.5, 1.0, 1.0 / 12.0, 5.0 / 6.0
    assert abs(-uy[tip].mean() / (P * L ** 3 / (3 * E * I) + P * L / (kappa * G * A)) - 1.0) <= 5e-3


@pytest.mark.parametrize("name,dims", [("c1", (4,)), ("c3", (2, 1, 1)), ("c4", (2, 2, 1))])
def test_coo_view_is_the_csr_in_sparse_id_order(name, dims):
    """NEXT-4 pin of the COO view (reading L4): a bijection onto the CSR's entries, ordered
    lexicographically by (κ₀, κ_λ, α₁, α₂), carrying the CSR values; workpiece offsets shift I and J."""
    m, p = make_config(name, "perturbed", dims)
    st = make_state(name, m, p)
    out = oracle.assemble(m, p, st)
    kh, N = p.kappa_hat(m.dim), m.n_nodes
    coo = oracle.coo_view(out, N, kh)
    rp, ci = out["rowptr"], out["colidx"]
    csr = {(int(r), int(c)): out["values"][k] for r in range(len(rp) - 1) for k, c in zip(range(rp[r], rp[r + 1]), ci[rp[r]:rp[r + 1]])}
    pairs = list(zip(coo["I"].tolist(), coo["J"].tolist()))
    assert len(pairs) == len(csr) == len(set(pairs)) and set(pairs) == set(csr)
    key = [(i // N, j // N, i % N, j % N) for i, j in pairs]
    assert key == sorted(key)
    assert all(csr[pq] == v for pq, v in zip(pairs, coo["values"]))
    off = oracle.coo_view(out, N, kh, row_offset=1000)
    assert np.array_equal(off["I"], coo["I"] + 1000) and np.array_equal(off["J"], coo["J"] + 1000)
