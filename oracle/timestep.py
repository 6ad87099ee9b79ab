"""oracle.timestep — TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py).

NEXT-3: the paper's generalized-alpha time stepping around the assembly, written out step by step in
the paper's order and notation, in fp64 numpy.  Shares nothing with the CUDA path.

Arrays: ``phi0[nu][n]`` = committed values ∂_t^ν φ, ``incr[nu][n]`` = increments
Δ∂_t^ν φ, ``eff[nu][n]`` = effective values ∂_t^ν φ̃, nu = 0..ν̂.
Scheme parameters follow fem_time_scheme: dt, b = (b1, b2), c = (c1, c2, c3).

Readings:
* L13 — D-4 prints Δ∂^ν φ += Δ_sub φ · Π(b Δt); Eq. gen_alpha and the
  constraints Eq. time_constraints require the division Δ_sub φ / Π_{β'≤ν}(b_β' Δt).
* L14 — C-3 as printed, Δ∂^ν φ = (b_{ν+1}Δt) ∂^{ν+1}φ + Δ∂^{ν+1}φ, contradicts Eq.
  time_constraints; we seed from Eq. time_constraints itself: Δ∂^ν φ = Δt(∂^{ν+1}φ + b_{ν+1} Δ∂^{ν+1}φ),
  ν = ν̂-1, ..., 0, after C-2 cleared Δ∂^ν̂ φ.

Pins (tests/test_oracle_pins.py): trapezoidal amplification factor for φ' = -λφ (closed form),
exact energy conservation of the average-acceleration member for the undamped oscillator, observed
order >= 1.9 against cos(ωt) at ρ∞ = 0.8 and high-frequency damping at ρ∞ = 0 but none at ρ∞ = 1
(reading L26), the constraint invariant of Eq.
time_constraints under repeated D-4 updates, and one-sub-step convergence for linear problems.
"""
from __future__ import annotations

import numpy as np


def _b(ts, k):   # b_k, k = 1, 2
    return (ts["b1"], ts["b2"])[k - 1]


def _c(ts, k):   # c_k, k = 1, 2, 3
    return (ts["c1"], ts["c2"], ts["c3"])[k - 1]


def prod_b_dt(ts, nu):
    """Π_{β'=1}^{ν} (b_β' Δt), empty product = 1 (Eq. gen_alpha)."""
    p = 1.0
    for k in range(1, nu + 1):
        p = p * (_b(ts, k) * ts["dt"])
    return p


def time_init(ts, nu_hat, phi0, incr):
    """Block C.  C-1: ∂^ν φ += Δ∂^ν φ.  C-2: Δ∂^ν̂ φ := 0.  C-3 (reading L14):
    Δ∂^ν φ = Δt(∂^{ν+1}φ + b_{ν+1} Δ∂^{ν+1}φ) for ν = ν̂-1 … 0.  In place."""
    for nu in range(nu_hat + 1):                       # C-1
        phi0[nu] = phi0[nu] + incr[nu]
    incr[nu_hat] = 0.0                                 # C-2
    for nu in range(nu_hat - 1, -1, -1):               # C-3
        incr[nu] = ts["dt"] * (phi0[nu + 1] + _b(ts, nu + 1) * incr[nu + 1])


def time_effective(ts, nu_hat, phi0, incr):
    """D-1: ∂^ν φ̃ = c_{ν+1} Δ∂^ν φ + ∂^ν φ."""
    eff = np.empty_like(phi0)
    for nu in range(nu_hat + 1):
        eff[nu] = _c(ts, nu + 1) * incr[nu] + phi0[nu]
    return eff


def time_increment(ts, nu_hat, delta_sub, incr):
    """D-4 (reading L13): Δ∂^ν φ += Δ_sub φ / Π_{β'≤ν}(b_β' Δt).  In place."""
    for nu in range(nu_hat + 1):
        incr[nu] = incr[nu] + delta_sub / prod_b_dt(ts, nu)


def tangent_factor(ts, nu):
    """f_ν = c_{ν+1} / Π_{β'≤ν}(b_β' Δt) (Eq. gen_alpha, D-3 P:452)."""
    return _c(ts, nu + 1) / prod_b_dt(ts, nu)


def step_linear(ts, nu_hat, mats, f, phi0, incr, n_sub=1):
    """One timestep of Blocks C, D for the linear residual d(φ̃, ũ, ã) = f - Σ_ν A_ν ∂^ν φ̃ with
    mats = [A_0, …, A_ν̂] (dense).  K = ∂d/∂φ = -Σ_ν f_ν A_ν (Eq. gen_alpha); D-4 solves K Δ_sub = -d
    with a dense direct solve.  Returns the residual norm after the last sub-step."""
    time_init(ts, nu_hat, phi0, incr)                                 # Block C
    K = -sum(tangent_factor(ts, nu) * mats[nu] for nu in range(nu_hat + 1))
    for _ in range(n_sub):
        eff = time_effective(ts, nu_hat, phi0, incr)                  # D-1
        d = f - sum(mats[nu] @ eff[nu] for nu in range(nu_hat + 1))   # D-2
        delta = np.linalg.solve(K, -d)                                # D-3, D-4
        time_increment(ts, nu_hat, delta, incr)
    eff = time_effective(ts, nu_hat, phi0, incr)
    d = f - sum(mats[nu] @ eff[nu] for nu in range(nu_hat + 1))
    return float(np.linalg.norm(d))


def committed(nu_hat, phi0, incr):
    """Values at the end of the timestep, {φ_{m+1}^0, …} := {φ_m^{n_m}, …}."""
    return np.array([phi0[nu] + incr[nu] for nu in range(nu_hat + 1)])


def genalpha_rho(rho_inf):
    """Scheme parameters from the spectral-radius knob ρ∞ (reading L26; the paper cites generalized-α
    but lists no values, SPEC S:412 fixes the mapping): α_m = (2ρ∞−1)/(ρ∞+1), α_f = ρ∞/(ρ∞+1),
    γ = ½ − α_m + α_f (the generalized-α second-order condition); b1 = ½, b2 = γ, c1 = c2 = 1 − α_f,
    c3 = 1 − α_m.  With b1 = ½ Eq. time_constraints is a Newmark update with β = γ/2."""
    a_m = (2.0 * rho_inf - 1.0) / (rho_inf + 1.0)
    a_f = rho_inf / (rho_inf + 1.0)
    gamma = 0.5 - a_m + a_f
    return dict(b1=0.5, b2=gamma, c1=1.0 - a_f, c2=1.0 - a_f, c3=1.0 - a_m)
