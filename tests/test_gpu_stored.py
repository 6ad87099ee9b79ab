"""FEM_SCATTER_STORED (element-stored blocks + per-slot gather in element order, csrc/stored.cu) through
the C ABI: its contract (prepare first, no accumulate), that every call rewrites every element block (outputs
poisoned, the state changes between calls), and the inverted-element report of the P2-tet element pass.
Oracle parity and bit-identity of the mode on c1-c5 run in test_gpu_parity.py (SCATTERS)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from fem_inputs import make_config, make_state  # noqa: E402
from helpers import csr_row_scaled_err, rhs_err  # noqa: E402

TOL = 1e-12


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_stored_needs_prepare_and_rejects_accumulate():
    _need_gpu()
    from paper_2111_03541_b200 import fem
    from paper_2111_03541_b200.fem import FemError
    m, p = make_config("c3", "structured", (3, 2, 2))
    from paper_2111_03541_b200 import FemSystem
    S = FemSystem(m, p)
    S.alloc(True, True)
    sd = torch.from_numpy(make_state("c3", m, p)).cuda()
    with pytest.raises(FemError) as ei:  # no fem_pattern_stored_prepare yet
        fem.fem_assemble_system(S.mesh_h, S.pat_h, S.problem, sd, S.values, S.rhs, 0, "stored", P=S.P)
    assert ei.value.code == -1
    fem.fem_pattern_stored_prepare(S.pat_h, with_matrix=False)
    with pytest.raises(FemError):  # residual scratch only: a matrix call still refuses
        fem.fem_assemble_matrix(S.mesh_h, S.pat_h, S.problem, sd, S.values, 0, "stored")
    fem.fem_assemble_residual(S.mesh_h, S.pat_h, S.problem, sd, S.rhs, 0, "stored")
    fem.fem_pattern_stored_prepare(S.pat_h, with_matrix=True)
    with pytest.raises(FemError):
        fem.fem_assemble_system(S.mesh_h, S.pat_h, S.problem, sd, S.values, S.rhs, 1, "stored", P=S.P)
    fem.fem_assemble_system(S.mesh_h, S.pat_h, S.problem, sd, S.values, S.rhs, 0, "stored", P=S.P)
    S.close()


@pytest.mark.parametrize("name,dims", [("c3", (7, 3, 2)), ("c4", (9, 4, 3)), ("c5", (7, 5, 6)), ("c2", (9, 7, 6))])
def test_stored_parity_with_changing_state(name, dims):
    """Two different states in a row: the second call must not reuse any element block of the first
    (the oracle is evaluated at each state); system, matrix-only and residual-only calls."""
    _need_gpu()
    from helpers import poisoned_system
    m, p = make_config(name, "perturbed", dims)
    S = poisoned_system(m, p)
    for seed in (0, 1):
        st = make_state(name, m, p)
        if seed:
            st = st * 1.7 + np.random.default_rng(9).uniform(-1e-3, 1e-3, st.shape) * np.abs(st).max()
        ora = oracle.assemble(m, p, st)
        sd = torch.from_numpy(st).cuda()
        for v, r in [S.system(sd, scatter="stored"),
                     (S.matrix(sd, scatter="stored").clone(), S.residual(sd, scatter="stored").clone())]:
            assert csr_row_scaled_err(ora["rowptr"], v.cpu().numpy(), ora["values"]) <= TOL
            assert rhs_err(r.cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL
    assert S.status() == (0, -1)
    S.close()


def test_stored_inverted_element_reported():
    _need_gpu()
    from helpers import REF_TET, one_element, p2_tet_coords, problem
    from paper_2111_03541_b200 import FemSystem
    pr = problem("elasticity", "tet", 2, [("ELAST_DOMAIN", -1, dict(E=1.0, nu=0.3))])
    m = one_element("tet", 2, p2_tet_coords(REF_TET[:, [0, 2, 1, 3]]))
    S = FemSystem(m, pr)
    S.system(torch.zeros((1, 3, 10), dtype=torch.float64, device="cuda"), scatter="stored")
    rc, bad = S.status()
    assert rc == -4 and bad == 0
    S.close()


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_stored_through_the_host_entry_points(name):
    """fem_linearize_host / _async (host state in, norms out) with FEM_SCATTER_STORED: the same matrix,
    residual and norms as the device call, bit for bit, call after call."""
    _need_gpu()
    from paper_2111_03541_b200 import fem
    m, p = make_config(name, "perturbed", {"c3": (7, 3, 2), "c4": (9, 4, 3)}[name])
    st = make_state(name, m, p)
    from paper_2111_03541_b200 import FemSystem
    S = FemSystem(m, p)
    v_dev, r_dev = [x.clone() for x in S.system(torch.from_numpy(st).cuda(), scatter="stored")]
    n_dev = torch.zeros(2, dtype=torch.float64, device="cuda")
    fem.fem_residual_norms(S.mesh_h, r_dev, n_dev)
    hs = torch.from_numpy(st).pin_memory()
    n_sync = torch.zeros(2, dtype=torch.float64).pin_memory()
    fem.fem_linearize_host(S.mesh_h, S.pat_h, p, hs, S.values, S.rhs, n_sync, "stored", P=S.P)
    assert torch.equal(S.values, v_dev) and torch.equal(S.rhs, r_dev)
    assert torch.equal(n_sync, n_dev.cpu())
    n_async = torch.zeros(2, dtype=torch.float64).pin_memory()
    for _ in range(3):
        fem.fem_linearize_host_async(S.mesh_h, S.pat_h, p, hs, S.values, S.rhs, n_async, "stored", P=S.P)
    torch.cuda.synchronize()
    assert torch.equal(S.values, v_dev) and torch.equal(S.rhs, r_dev) and torch.equal(n_async, n_sync)
    S.close()
