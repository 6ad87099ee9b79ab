"""CPU pins of the NEXT-3 oracle (oracle/timestep.py): Blocks C/D of the generalized-alpha scheme
 against closed forms and invariants, never against itself."""
import numpy as np
import pytest

from oracle import timestep as ot


def _ts(dt, **k):
    d = dict(dt=dt, b1=0.5, b2=0.5, c1=1.0, c2=1.0, c3=1.0)
    d.update(k)
    return d


def _run(ts, nu_hat, mats, f, init, steps, n_sub=1):
    phi0 = np.array(init, dtype=np.float64)
    incr = np.zeros_like(phi0)
    hist = [phi0.copy()]
    for _ in range(steps):
        ot.step_linear(ts, nu_hat, mats, f, phi0, incr, n_sub=n_sub)
        hist.append(ot.committed(nu_hat, phi0, incr))
    return hist


def test_trapezoid_amplification_first_order():
    """ν̂ = 1, φ' = -λφ (d = -(u + λφ)), b1 = 1/2, c = 1: Eq. time_constraints becomes the trapezoidal
    rule, amplification (1 - λΔt/2)/(1 + λΔt/2) per step (closed form)."""
    lam, dt, n = 3.0, 0.1, 25
    mats = [np.array([[lam]]), np.array([[1.0]])]
    hist = _run(_ts(dt), 1, mats, np.zeros(1), [[1.0], [-lam]], n)
    g = (1 - lam * dt / 2) / (1 + lam * dt / 2)
    for m, s in enumerate(hist):
        assert s[0, 0] == pytest.approx(g ** m, rel=1e-13, abs=1e-300)
        assert s[1, 0] == pytest.approx(-lam * g ** m, rel=1e-13)   # u = -λφ holds at every step


def test_average_acceleration_conserves_energy():
    """ν̂ = 2 undamped oscillator φ'' + ω²φ = 0 with b1 = b2 = 1/2, c = 1 (Newmark average
    acceleration): the discrete energy ½u² + ½ω²φ² is conserved exactly for linear systems."""
    w, dt = 2.0, 0.07
    mats = [np.array([[w * w]]), np.zeros((1, 1)), np.array([[1.0]])]
    hist = _run(_ts(dt), 2, mats, np.zeros(1), [[1.0], [0.0], [-w * w]], 300)
    E0 = 0.5 * w * w
    for s in hist:
        assert 0.5 * s[1, 0] ** 2 + 0.5 * w * w * s[0, 0] ** 2 == pytest.approx(E0, rel=1e-12)
    # and the phase is not exact (it is a discretisation): the final value differs from cos(ωT)
    assert abs(hist[-1][0, 0] - np.cos(w * dt * 300)) > 1e-6


def test_genalpha_second_order_rho08():
    """SPEC S:410 / S:535: observed order >= 1.9 in Δt at ρ∞ = 0.8 against cos(ωt)."""
    w, T = 2.0 * np.pi, 1.0
    mats = [np.array([[w * w]]), np.zeros((1, 1)), np.array([[1.0]])]
    errs = []
    for n in (20, 40, 80, 160):
        ts = dict(dt=T / n, **ot.genalpha_rho(0.8))
        hist = _run(ts, 2, mats, np.zeros(1), [[1.0], [0.0], [-w * w]], n)
        errs.append(abs(hist[-1][0, 0] - np.cos(w * T)))
    orders = [np.log2(errs[i] / errs[i + 1]) for i in range(len(errs) - 1)]
    assert min(orders) >= 1.9, (errs, orders)


def test_constraints_hold_under_substeps():
    """Eq. time_constraints: after Block C and any number of D-4 updates,
    Δφ - b1Δt Δu = Δt u⁰ and Δu - b2Δt Δa = Δt a⁰.  A multiplying D-4 (P:463 as printed) or the
    printed C-3 seeding breaks this (readings L13, L14)."""
    rng = np.random.default_rng(7)
    ts = dict(dt=0.013, b1=0.61, b2=0.47, c1=0.9, c2=0.8, c3=0.7)
    n = 57
    phi0 = rng.standard_normal((3, n))
    incr = rng.standard_normal((3, n))
    ot.time_init(ts, 2, phi0, incr)
    for _ in range(5):
        ot.time_increment(ts, 2, rng.standard_normal(n), incr)
        dt = ts["dt"]
        np.testing.assert_allclose(incr[0] - ts["b1"] * dt * incr[1], dt * phi0[1], rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(incr[1] - ts["b2"] * dt * incr[2], dt * phi0[2], rtol=1e-10, atol=1e-12)


def test_time_init_commits_and_seeds():
    """C-1 adds the increments, C-2 clears the top one, C-3 seeds from Eq. time_constraints."""
    ts = dict(dt=0.5, b1=0.25, b2=0.5, c1=1, c2=1, c3=1)
    phi0 = np.array([[1.0], [2.0], [4.0]])
    incr = np.array([[0.5], [1.0], [3.0]])
    ot.time_init(ts, 2, phi0, incr)
    assert phi0[:, 0].tolist() == [1.5, 3.0, 7.0]
    assert incr[2, 0] == 0.0
    assert incr[1, 0] == 0.5 * 7.0                       # Δu = Δt a⁰
    assert incr[0, 0] == 0.5 * (3.0 + 0.25 * 3.5)        # Δφ = Δt(u⁰ + b1 Δu)


def test_linear_problem_converges_in_one_substep():
    """For a linear residual the Newton tangent of Eq. gen_alpha is exact: one sub-step drives d to
    rounding (a wrong time factor f_ν would leave a residual)."""
    rng = np.random.default_rng(3)
    n = 12
    mats = []
    for _ in range(3):
        X = rng.standard_normal((n, n))
        mats.append(X @ X.T + n * np.eye(n))
    f = rng.standard_normal(n)
    ts = dict(dt=0.02, b1=0.55, b2=0.6, c1=0.8, c2=0.7, c3=0.9)
    phi0 = rng.standard_normal((3, n))
    incr = rng.standard_normal((3, n))
    r = ot.step_linear(ts, 2, mats, f, phi0, incr, n_sub=1)
    scale = max(np.linalg.norm(m, 2) for m in mats) * np.abs(phi0).max() / ts["dt"] ** 2
    assert r <= 1e-11 * scale


def _hf_amplitude_ratio(ts, w=1e4, steps=40):
    mats = [np.array([[w * w]]), np.zeros((1, 1)), np.array([[1.0]])]
    phi0 = np.array([[1.0], [0.0], [-w * w]])
    incr = np.zeros_like(phi0)
    E = []
    for _ in range(steps):
        ot.step_linear(ts, 2, mats, np.zeros(1), phi0, incr)
        s = ot.committed(2, phi0, incr)
        E.append(0.5 * s[1, 0] ** 2 + 0.5 * w * w * s[0, 0] ** 2)
    return (E[-1] / E[0]) ** (1.0 / (2 * (steps - 1)))


def test_genalpha_rho_damps_high_frequencies_only_below_one():
    """SPEC S:535 (reading L26): with the ρ∞ mapping of S:412 the per-step high-frequency amplitude
    (ωΔt = 1e4) is < 1 at ρ∞ = 0 (visible numerical damping) and exactly 1 at ρ∞ = 1 (the average-
    acceleration member: α_m = ½, α_f = ½, γ = ½, c = ½), and it decreases monotonically with ρ∞."""
    amp = {r: _hf_amplitude_ratio(dict(dt=1.0, **ot.genalpha_rho(r))) for r in (0.0, 0.5, 0.8, 1.0)}
    assert amp[0.0] < 0.9
    assert amp[1.0] == pytest.approx(1.0, abs=1e-6)
    assert amp[0.0] < amp[0.5] < amp[0.8] < amp[1.0]
    # and the mapping is second order at every ρ∞ (γ = ½ − α_m + α_f), measured off the extrema of cos
    w, T = 2.0 * np.pi, 1.15
    mats = [np.array([[w * w]]), np.zeros((1, 1)), np.array([[1.0]])]
    for r in (0.0, 0.5, 1.0):
        errs = []
        for n in (80, 160, 320, 640):
            hist = _run(dict(dt=T / n, **ot.genalpha_rho(r)), 2, mats, np.zeros(1), [[1.0], [0.0], [-w * w]], n)
            errs.append(abs(hist[-1][0, 0] - np.cos(w * T)))
        assert min(np.log2(errs[i] / errs[i + 1]) for i in range(3)) >= 1.9, (r, errs)
