"""The five BASELINE.json configs as seeded synthetic workloads.

A Problem is the paper's statement of the linear system: weak forms (terms), element
type/order, quadrature order, temporal scheme; the numbering is fixed by both implementations
(P:370 κ-major).  Parameters are kept *named* here; each implementation maps them to its own
positional layout.  Seeds: 2111035410 + 100*cfg + stream (stream 0: mesh perturbation,
stream 1: state).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .meshgen import Mesh, facets_on_plane, hex_box, hex_box_quadratic, perturb_and_permute, tet_box, tri_square

SIGMA_B = 5.670e-8  # Stefan-Boltzmann constant as printed at P:827


@dataclass
class Term:
    form: str  # e.g. "THERMAL_DOMAIN"; see DESIGN.md §4 for the list
    region: int  # -1 = domain, k >= 0 = boundary set k
    params: dict


@dataclass
class TimeScheme:
    """Generalized-alpha parameters; static = nu_hat 0, c1 = 1 (reading L12)."""
    kind: str = "static"  # "static" | "genalpha"
    nu_hat: int = 0
    dt: float = 1.0
    b1: float = 1.0
    b2: float = 1.0
    c1: float = 1.0
    c2: float = 1.0
    c3: float = 1.0


@dataclass
class Problem:
    physics: str  # "thermal" | "elasticity" | "ns"
    etype: str
    order: int
    quad_order: int  # GL points/axis (hex) or exactness degree (tri/tet)
    terms: list
    time: TimeScheme = field(default_factory=TimeScheme)

    def kappa_hat(self, dim: int) -> int:
        return {"thermal": 1, "elasticity": dim, "ns": dim + 1}[self.physics]


@dataclass
class ConfigSpec:
    name: str
    index: int
    full_dims: tuple
    desc: str


CONFIGS = {
    "c1": ConfigSpec("c1", 1, (8,), "2D thermal (Poisson), unit square, 8x8 -> 128 P1 triangles"),
    "c2": ConfigSpec("c2", 2, (64, 64, 64), "3D steady heat, unit cube, 64^3 Q1 hex"),
    "c3": ConfigSpec("c3", 3, (230, 23, 23), "3D elasticity cantilever [0,10]x[0,1]^2, Kuhn P2 tets"),
    "c4": ConfigSpec("c4", 4, (451, 74, 74), "3D SUPG/PSPG Navier-Stokes channel, Kuhn P1/P1 tets"),
    "c5": ConfigSpec("c5", 5, (256, 256, 256), "3D elasticity, 256^3 Q1 hex"),
    # NEXT-2: the quadratic cubes of the paper's experiments
    "q2": ConfigSpec("q2", 6, (160, 16, 16), "3D elasticity cantilever [0,10]x[0,1]^2, 27-node Q2 hex"),
    "s2": ConfigSpec("s2", 7, (160, 16, 16), "3D elasticity cantilever [0,10]x[0,1]^2, 20-node serendipity hex"),
    "q2ns": ConfigSpec("q2ns", 8, (60, 10, 10), "3D SUPG/PSPG Navier-Stokes channel, 27-node Q2 hex"),
}


def seed(cfg_index: int, stream: int) -> int:
    return 2111035410 + 100 * cfg_index + stream


def ns_tau(rho=1000.0, mu=1.0, U=0.45, h_e=0.41 / 74):
    """Reading L11: tau_m = tau_SUPG / rho with tau_SUPG = ((2U/h_e)^2 + (4 nu/h_e^2)^2)^-1/2,
    tau_c = rho U h_e / 2, tau_b = 100 mu / (rho h_e)."""
    nu = mu / rho
    tau_supg = ((2 * U / h_e) ** 2 + (4 * nu / h_e ** 2) ** 2) ** -0.5
    return tau_supg / rho, rho * U * h_e / 2.0, 100.0 * mu / (rho * h_e)


def _problem_and_mesh(name: str, dims):
    if name == "c1":
        (n,) = dims
        mesh = tri_square(n)
        sets = [facets_on_plane(mesh, 0, 0.0), facets_on_plane(mesh, 0, 1.0),
                facets_on_plane(mesh, 1, 0.0), facets_on_plane(mesh, 1, 1.0)]
        be = np.concatenate([s[0] for s in sets])
        bf = np.concatenate([s[1] for s in sets])
        o = np.lexsort((bf, be))
        mesh.bsets = [(np.ascontiguousarray(be[o]), np.ascontiguousarray(bf[o]))]
        mesh.bset_names = ["all_sides"]
        k = 1.0
        terms = [Term("THERMAL_DOMAIN", -1, dict(C=0.0, k=k, s=2 * math.pi ** 2 * k, source="sine")),
                 Term("THERMAL_FIX", 0, dict(h_p=1e4, T_fix=0.0, k=k))]
        prob = Problem("thermal", "tri", 1, 2, terms)
        h = 1.0 / n
    elif name == "c2":
        nx, ny, nz = dims
        mesh = hex_box(nx, ny, nz)
        fix = [facets_on_plane(mesh, 0, 0.0), facets_on_plane(mesh, 0, 1.0)]
        cr = [facets_on_plane(mesh, 1, 0.0), facets_on_plane(mesh, 1, 1.0),
              facets_on_plane(mesh, 2, 0.0), facets_on_plane(mesh, 2, 1.0)]
        mesh.bsets = [_merge(fix), _merge(cr)]
        mesh.bset_names = ["x_faces_fix", "yz_faces_conv_rad"]
        k = 0.6
        terms = [Term("THERMAL_DOMAIN", -1, dict(C=0.0, k=k, s=1.6e3, source="const")),
                 Term("THERMAL_FIX", 0, dict(h_p=1e4, T_fix=1173.15, k=k)),
                 Term("THERMAL_CONV_RAD", 1, dict(h=25.0, T_env=293.15, e_m=0.7, sigma_b=SIGMA_B))]
        prob = Problem("thermal", "hex", 1, 2, terms)
        h = (1.0 / nx, 1.0 / ny, 1.0 / nz)
    elif name == "c3":
        nx, ny, nz = dims
        L, hh = 10.0, 1.0
        mesh = tet_box(nx, ny, nz, L, hh, hh, order=2)
        mesh.bsets = [facets_on_plane(mesh, 0, 0.0), facets_on_plane(mesh, 0, L)]
        mesh.bset_names = ["x0_fix", "xL_load"]
        P = 1e-3
        sl = [0.0] * 9
        sl[3 * 1 + 0] = -P / hh ** 2  # sigma^l_21 (P:923 load (d_i, sigma^l_ij n_j))
        terms = [Term("ELAST_DOMAIN", -1, dict(E=1.0, nu=0.3)),
                 Term("ELAST_FIX_ALL", 0, dict(tau=1e3, dw=(0.0, 0.0, 0.0))),
                 Term("ELAST_LOAD", 1, dict(sigma_l=tuple(sl)))]
        prob = Problem("elasticity", "tet", 2, 2, terms)
        h = (L / nx, hh / ny, hh / nz)
    elif name == "c4":
        nx, ny, nz = dims
        L, H = 2.5, 0.41
        mesh = tet_box(nx, ny, nz, L, H, H, order=1)
        walls = _merge([facets_on_plane(mesh, 1, 0.0), facets_on_plane(mesh, 1, H),
                        facets_on_plane(mesh, 2, 0.0), facets_on_plane(mesh, 2, H)])
        mesh.bsets = [facets_on_plane(mesh, 0, 0.0), facets_on_plane(mesh, 0, L), walls]
        mesh.bset_names = ["inflow", "outflow", "walls"]
        rho, mu, U = 1000.0, 1.0, 0.45
        tau_m, tau_c, tau_b = ns_tau(rho, mu, U, H / ny)
        terms = [Term("NS_DOMAIN", -1, dict(rho=rho, mu=mu, tau_m=tau_m, tau_c=tau_c)),
                 Term("NS_BND_INFLOW", 0, dict(rho=rho, mu=mu, tau_b=tau_b, U=U, H=H)),
                 Term("NS_BND_OUTFLOW", 1, dict(rho=rho, mu=mu)),
                 Term("NS_BND_FIX", 2, dict(rho=rho, mu=mu, tau_b=tau_b))]
        prob = Problem("ns", "tet", 1, 2, terms)
        h = (L / nx, H / ny, H / nz)
    elif name == "c5":
        nx, ny, nz = dims
        mesh = hex_box(nx, ny, nz)
        mesh.bsets = [facets_on_plane(mesh, 2, 0.0), facets_on_plane(mesh, 2, 1.0)]
        mesh.bset_names = ["z0_fix", "z1_load"]
        sl = [0.0] * 9
        sl[3 * 2 + 2] = -1e-3  # traction (0,0,-1e-3) on the z = 1 face (normal +z)
        terms = [Term("ELAST_DOMAIN", -1, dict(E=1.0, nu=0.3)),
                 Term("ELAST_FIX_ALL", 0, dict(tau=1e3, dw=(0.0, 0.0, 0.0))),
                 Term("ELAST_LOAD", 1, dict(sigma_l=tuple(sl)))]
        prob = Problem("elasticity", "hex", 1, 2, terms)
        h = (1.0 / nx, 1.0 / ny, 1.0 / nz)
    elif name in ("q2", "s2"):
        nx, ny, nz = dims
        L, hh = 10.0, 1.0
        mesh = hex_box_quadratic(nx, ny, nz, L, hh, hh, serendipity=(name == "s2"))
        mesh.bsets = [facets_on_plane(mesh, 0, 0.0), facets_on_plane(mesh, 0, L)]
        mesh.bset_names = ["x0_fix", "xL_load"]
        P = 1e-3
        sl = [0.0] * 9
        sl[3 * 1 + 0] = -P / hh ** 2
        terms = [Term("ELAST_DOMAIN", -1, dict(E=1.0, nu=0.3)),
                 Term("ELAST_FIX_ALL", 0, dict(tau=1e3, dw=(0.0, 0.0, 0.0))),
                 Term("ELAST_LOAD", 1, dict(sigma_l=tuple(sl)))]
        prob = Problem("elasticity", mesh.etype, 2, 3, terms)
        h = (L / nx, hh / ny, hh / nz)
    elif name == "q2ns":
        nx, ny, nz = dims
        L, H = 2.5, 0.41
        mesh = hex_box_quadratic(nx, ny, nz, L, H, H)
        walls = _merge([facets_on_plane(mesh, 1, 0.0), facets_on_plane(mesh, 1, H),
                        facets_on_plane(mesh, 2, 0.0), facets_on_plane(mesh, 2, H)])
        mesh.bsets = [facets_on_plane(mesh, 0, 0.0), facets_on_plane(mesh, 0, L), walls]
        mesh.bset_names = ["inflow", "outflow", "walls"]
        rho, mu, U = 1000.0, 1.0, 0.45
        tau_m, tau_c, tau_b = ns_tau(rho, mu, U, H / ny)
        terms = [Term("NS_DOMAIN", -1, dict(rho=rho, mu=mu, tau_m=tau_m, tau_c=tau_c)),
                 Term("NS_BND_INFLOW", 0, dict(rho=rho, mu=mu, tau_b=tau_b, U=U, H=H)),
                 Term("NS_BND_OUTFLOW", 1, dict(rho=rho, mu=mu)),
                 Term("NS_BND_FIX", 2, dict(rho=rho, mu=mu, tau_b=tau_b))]
        prob = Problem("ns", "hex", 2, 3, terms)
        h = (L / nx, H / ny, H / nz)
    else:
        raise KeyError(name)
    return mesh, prob, h


def _merge(sets):
    be = np.concatenate([s[0] for s in sets])
    bf = np.concatenate([s[1] for s in sets])
    o = np.lexsort((bf, be))
    return np.ascontiguousarray(be[o]), np.ascontiguousarray(bf[o])


def make_config(name: str, variant: str = "structured", dims=None):
    """Return (mesh, problem) for config `name` at `dims` (default: the BASELINE.json size).
    variant: "structured" or "perturbed" (jitter + random node/element permutation)."""
    spec = CONFIGS[name]
    dims = tuple(dims) if dims is not None else spec.full_dims
    mesh, prob, h = _problem_and_mesh(name, dims)
    if variant == "perturbed":
        rng = np.random.default_rng(seed(spec.index, 0))
        amp = 0.2 if mesh.etype in ("hex", "hexs", "tri") else 0.12
        mesh = perturb_and_permute(mesh, rng, h, amp)
    elif variant != "structured":
        raise ValueError(variant)
    return mesh, prob


def make_state(name: str, mesh: Mesh, prob: Problem, kind: str = "random"):
    """Effective state, float64 [nu_hat+1][kappa_hat][N] (SURVEY §8(d) 'State' column)."""
    spec = CONFIGS[name]
    rng = np.random.default_rng(seed(spec.index, 1))
    N = mesh.n_nodes
    kh = prob.kappa_hat(mesh.dim)
    levels = prob.time.nu_hat + 1
    st = np.zeros((levels, kh, N))
    x = mesh.coords
    if kind == "zero":
        return st
    if name == "c1":
        st[0, 0] = rng.uniform(0.0, 1.0, N)
    elif name == "c2":
        st[0, 0] = rng.uniform(300.0, 1200.0, N)
    elif name in ("c3", "c5", "q2", "s2"):
        st[0] = rng.uniform(-1e-3, 1e-3, (kh, N))
    elif name in ("c4", "q2ns"):
        U, H = 0.45, 0.41
        y, z = x[1], x[2]
        uw = 16 * U * (H - y) * (H - z) * y * z / H ** 4  # P:1050 inflow profile
        xi = rng.uniform(-1.0, 1.0, (3, N))
        st[0, 0] = uw * (1 + 0.01 * xi[0])
        st[0, 1] = uw * 0.01 * xi[1]
        st[0, 2] = uw * 0.01 * xi[2]
        st[0, 3] = 10.0 * (1 - x[0] / 2.5) + rng.uniform(-0.1, 0.1, N)
    if levels > 1:
        st[1:] = rng.uniform(-1.0, 1.0, st[1:].shape) * (np.abs(st[0]).max() + 1.0)
    return np.ascontiguousarray(st)
