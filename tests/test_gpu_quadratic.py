"""NEXT-2 on the GPU: quadratic cubes (27-node Q2, 20-node serendipity) and the NS strong
residual with μ u_i,kk on every element that carries second derivatives, through the C ABI,
against the oracle (pattern and slot map bit-exact, values within reading L20's 1e-12)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from fem_inputs import make_config, make_state  # noqa: E402
from fem_inputs.meshgen import facets_on_plane, hex_box, perturb_and_permute, tet_box  # noqa: E402
from helpers import csr_row_scaled_err, rhs_err  # noqa: E402

TOL = 1e-12


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _check(m, p, st, scatters=("atomic", "coloured", "stored")):
    from helpers import poisoned_system
    ora = oracle.assemble(m, p, st, slot=True)
    assert ora["status"] == 0
    S = poisoned_system(m, p)
    pat = S.export_pattern()
    for k in ("rowptr", "colidx", "rowptr_s", "colidx_s", "slot_s"):
        np.testing.assert_array_equal(pat[k].cpu().numpy(), ora[k])
    sd = torch.from_numpy(st).cuda()
    for sc in scatters:
        v, r = S.system(sd, scatter=sc)
        torch.cuda.synchronize()
        ek = csr_row_scaled_err(ora["rowptr"], v.cpu().numpy(), ora["values"])
        ed = rhs_err(r.cpu().numpy(), ora["rhs"], ora["abs_d"])
        assert ek <= TOL and ed <= TOL, (sc, ek, ed)
        r2 = S.residual(sd, scatter=sc).clone()
        assert rhs_err(r2.cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL
    assert S.status() == (0, -1)
    if "coloured" in scatters:  # deterministic: bit-identical repeats
        v0, r0 = [x.clone() for x in S.system(sd, scatter="coloured")]
        v1, r1 = S.system(sd, scatter="coloured")
        assert torch.equal(v0, v1) and torch.equal(r0, r1)
    S.close()


@pytest.mark.parametrize("name,dims", [("q2", (5, 2, 3)), ("s2", (5, 2, 3)), ("q2ns", (3, 2, 2))])
@pytest.mark.parametrize("variant", ["structured", "perturbed"])
def test_quadratic_cube_parity(name, dims, variant):
    _need_gpu()
    m, p = make_config(name, variant, dims)
    _check(m, p, make_state(name, m, p))


def test_quadratic_cube_two_point_rule_and_thermal():
    """quad_order 2 (2x2x2 Gauss points, reduced integration) and the thermal forms on both cubes."""
    _need_gpu()
    from helpers import problem
    for name in ("q2", "s2"):
        m, _ = make_config(name, "perturbed", (3, 2, 2))
        terms = [("THERMAL_DOMAIN", -1, dict(C=0.0, k=0.6, s=1.6e3)),
                 ("THERMAL_FIX", 0, dict(h_p=1e4, T_fix=1173.15, k=0.6)),
                 ("THERMAL_CONV_RAD", 1, dict(h=25.0, T_env=293.15, e_m=0.7, sigma_b=5.67e-8))]
        for q in (2, 3):
            p = problem("thermal", m.etype, 2, terms, q)
            st = np.random.default_rng(5).uniform(300.0, 1200.0, (1, 1, m.n_nodes))
            _check(m, p, st)


@pytest.mark.parametrize("etype", ["tet2", "hex1"])
def test_ns_on_elements_with_second_derivatives(etype):
    """NS (SUPG/PSPG, all boundary groups) on P2 tets and Q1 hexes: the μ u_i,kk term is non-zero on both
    (P2: constant Hessians; Q1 on perturbed cubes: mixed second derivatives of the trilinear map)."""
    _need_gpu()
    from fem_inputs.configs import ns_tau
    from helpers import problem
    L, H = 2.5, 0.41
    if etype == "tet2":
        m = tet_box(4, 2, 2, L, H, H, order=2)
        et, order = "tet", 2
    else:
        m = hex_box(4, 3, 3, L, H, H)
        et, order = "hex", 1
    walls = [facets_on_plane(m, 1, 0.0), facets_on_plane(m, 2, H)]
    m.bsets = [facets_on_plane(m, 0, 0.0), facets_on_plane(m, 0, L),
               (np.concatenate([w[0] for w in walls]), np.concatenate([w[1] for w in walls]))]
    m = perturb_and_permute(m, np.random.default_rng(3), (L / 4, H / 3, H / 3), 0.1)
    tm, tc, tb = ns_tau(1000.0, 1.0, 0.45, H / 3)
    terms = [("NS_DOMAIN", -1, dict(rho=1000.0, mu=1.0, tau_m=tm, tau_c=tc)),
             ("NS_BND_INFLOW", 0, dict(rho=1000.0, mu=1.0, tau_b=tb, U=0.45, H=H)),
             ("NS_BND_OUTFLOW", 1, dict(rho=1000.0, mu=1.0)),
             ("NS_BND_FIX", 2, dict(rho=1000.0, mu=1.0, tau_b=tb))]
    p = problem("ns", et, order, terms, 2)
    st = make_state("c4", m, p)
    _check(m, p, st)


def test_tiled_on_quadratic_cubes_is_explicitly_unsupported():
    """No silent fallback: the tile scatter has no quadratic-cube kernel and says so."""
    _need_gpu()
    from paper_2111_03541_b200 import FemSystem
    from paper_2111_03541_b200.fem import FemError
    m, p = make_config("q2", "structured", (3, 2, 2))
    S = FemSystem(m, p)
    with pytest.raises(FemError) as ei:
        S.system(torch.zeros((1, 3, m.n_nodes), dtype=torch.float64, device="cuda"), scatter="tiled")
    assert ei.value.code == -2
    S.close()
