"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Tolerance (BASELINE.json north_star, reading L20 in DESIGN.md §4):
  * pattern (rowptr, colidx, rowptr_s, colidx_s) and slot map: bit-exact;
  * K: max_ij |K_gpu - K_ora| / max_j |K_ora_ij| <= 1e-12 (row-scaled);
  * d: max_i |d_gpu - d_ora| / max(|d_ora_i|, A_d[i]) <= 1e-12, A_d = Σ|qp contributions|;
  * coloured / tiled scatter: bit-identical run to run.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from fem_inputs import make_config, make_state  # noqa: E402
from fem_inputs.configs import TimeScheme  # noqa: E402
from helpers import csr_row_scaled_err, rhs_err  # noqa: E402

TOL = 1e-12

SMALL = {  # sizes the oracle finishes in seconds; several CTA batches / tiles and a ragged tail
    "c1": (8,), "c2": (9, 7, 6), "c3": (7, 3, 2), "c4": (9, 4, 3), "c5": (7, 5, 6)}


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _gpu_system(m, p, own=None):
    from helpers import poisoned_system
    return poisoned_system(m, p, own=own)


def _to_dev(st):
    return torch.from_numpy(st).cuda()


SCATTERS = os.environ.get("FEM_SCATTERS", "atomic,coloured,tiled,stored").split(",")


@pytest.mark.parametrize("name", list(SMALL))
@pytest.mark.parametrize("variant", ["structured", "perturbed"])
def test_small_parity_all_modes(name, variant):
    _need_gpu()
    m, p = make_config(name, variant, SMALL[name])
    st = make_state(name, m, p)
    ora = oracle.assemble(m, p, st, slot=True)
    assert ora["status"] == 0
    S = _gpu_system(m, p)
    pat = S.export_pattern()
    np.testing.assert_array_equal(pat["rowptr"].cpu().numpy(), ora["rowptr"])
    np.testing.assert_array_equal(pat["colidx"].cpu().numpy(), ora["colidx"])
    np.testing.assert_array_equal(pat["rowptr_s"].cpu().numpy(), ora["rowptr_s"])
    np.testing.assert_array_equal(pat["colidx_s"].cpu().numpy(), ora["colidx_s"])
    np.testing.assert_array_equal(pat["slot_s"].cpu().numpy(), ora["slot_s"])
    sd = _to_dev(st)
    for sc in SCATTERS:
        vals, rhs = S.system(sd, scatter=sc)
        torch.cuda.synchronize()
        ek = csr_row_scaled_err(ora["rowptr"], vals.cpu().numpy(), ora["values"])
        ed = rhs_err(rhs.cpu().numpy(), ora["rhs"], ora["abs_d"])
        assert ek <= TOL, (sc, ek)
        assert ed <= TOL, (sc, ed)
        # matrix-only and residual-only calls agree with the fused call
        v2 = S.matrix(sd, scatter=sc).clone()
        r2 = S.residual(sd, scatter=sc).clone()
        assert csr_row_scaled_err(ora["rowptr"], v2.cpu().numpy(), ora["values"]) <= TOL
        assert rhs_err(r2.cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL
    assert S.status() == (0, -1)
    S.close()


@pytest.mark.parametrize("name,sc", [(n, sc) for n in ("c1", "c2", "c3", "c4", "c5") for sc in ("coloured", "tiled", "stored")])
def test_deterministic_modes_bit_exact(name, sc):
    """FEM_SCATTER_COLOURED, FEM_SCATTER_TILED and FEM_SCATTER_STORED are deterministic by contract (libfem.h)
    on every element type: hex (sweep / ordered tiles), P1 NS tets (ordered turns), P2 tets (ordered turns),
    triangles (colour runs); stored: element-order sums per CSR entry.
    Matrix, residual and the system call are bit-identical call after call."""
    _need_gpu()
    m, p = make_config(name, "perturbed", SMALL[name])
    st = _to_dev(make_state(name, m, p))
    S = _gpu_system(m, p)
    if name == "c5":
        assert S.info()["schedule"] == 1  # the z-sweep
    ref_v, ref_r = [x.clone() for x in S.system(st, scatter=sc)]
    ref_m = S.matrix(st, scatter=sc).clone()
    ref_res = S.residual(st, scatter=sc).clone()
    for _ in range(3):
        v, r = S.system(st, scatter=sc)
        assert torch.equal(v, ref_v) and torch.equal(r, ref_r)
        assert torch.equal(S.matrix(st, scatter=sc), ref_m)
        assert torch.equal(S.residual(st, scatter=sc), ref_res)
    S.close()


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_tiled_unordered_parity(name):
    """FEM_SCATTER_TILED_UNORDERED (shared-memory atomics where the kernels have them) agrees with the oracle."""
    _need_gpu()
    m, p = make_config(name, "perturbed", SMALL[name])
    st = make_state(name, m, p)
    ora = oracle.assemble(m, p, st)
    S = _gpu_system(m, p)
    sd = _to_dev(st)
    for v, r in [S.system(sd, scatter="tiled_unordered"),
                 (S.matrix(sd, scatter="tiled_unordered").clone(), S.residual(sd, scatter="tiled_unordered").clone())]:
        assert csr_row_scaled_err(ora["rowptr"], v.cpu().numpy(), ora["values"]) <= TOL
        assert rhs_err(r.cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL
    S.close()


def test_accumulate_and_residual_without_pattern():
    _need_gpu()
    from paper_2111_03541_b200 import fem
    m, p = make_config("c3", "perturbed", SMALL["c3"])
    st = make_state("c3", m, p)
    ora = oracle.assemble(m, p, st)
    S = _gpu_system(m, p)
    sd = _to_dev(st)
    v, r = S.system(sd, scatter="atomic")
    v, r = S.system(sd, scatter="coloured", accumulate=True)
    assert csr_row_scaled_err(ora["rowptr"], v.cpu().numpy(), 2 * ora["values"]) <= TOL
    assert rhs_err(r.cpu().numpy(), 2 * ora["rhs"], 2 * ora["abs_d"]) <= TOL
    rhs = torch.zeros(S.n_rows, dtype=torch.float64, device="cuda")
    fem.fem_assemble_residual(S.mesh_h, None, p, sd, rhs, 0, "atomic")
    assert rhs_err(rhs.cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL
    S.close()


def test_genalpha_thermal_transient_term():
    _need_gpu()
    m, p = make_config("c2", "perturbed", (5, 4, 3))
    p.time = TimeScheme("genalpha", 1, dt=0.05, b1=0.6, b2=0.5, c1=0.7, c2=0.8, c3=1.0)
    p.terms[0].params = dict(p.terms[0].params, C=3.0)
    st = make_state("c2", m, p)
    ora = oracle.assemble(m, p, st)
    S = _gpu_system(m, p)
    for sc in SCATTERS:
        v, r = S.system(_to_dev(st), scatter=sc)
        assert csr_row_scaled_err(ora["rowptr"], v.cpu().numpy(), ora["values"]) <= TOL
        assert rhs_err(r.cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL
    S.close()


@pytest.mark.parametrize("name", ["c5", "c3"])
def test_genalpha_elasticity_f0(name):
    """Gen-α factor f0 = c1 != 1 (reading L13) scales the tangent but not the residual: the hex
    kernel cannot fuse r = K'd into the scatter and takes its stress-GEMM residual instead."""
    _need_gpu()
    m, p = make_config(name, "perturbed", SMALL[name])
    p.time = TimeScheme("genalpha", 1, dt=0.05, b1=0.6, b2=0.5, c1=0.7, c2=0.8, c3=1.0)
    st = make_state(name, m, p)
    ora = oracle.assemble(m, p, st)
    assert ora["status"] == 0
    S = _gpu_system(m, p)
    sd = _to_dev(st)
    for sc in SCATTERS:
        for v, r in [S.system(sd, scatter=sc), (S.matrix(sd, scatter=sc).clone(), S.residual(sd, scatter=sc).clone())]:
            assert csr_row_scaled_err(ora["rowptr"], v.cpu().numpy(), ora["values"]) <= TOL, sc
            assert rhs_err(r.cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL, sc
    S.close()


@pytest.mark.parametrize("variant", ["structured", "perturbed"])
def test_hex_elasticity_boundary_terms_every_face(variant):
    """Q1 hex elasticity with FIX_D1 / FIX_ALL (non-zero dʷ) / LOAD (full σˡ) on faces of every axis and
    both sides, an element with two boundary faces in one set, and two terms on one set:
    the tiled kernels (sweep and node tiles) integrate them inside the element visits; the atomic /
    coloured paths must agree with the oracle."""
    _need_gpu()
    from fem_inputs.configs import Term
    from fem_inputs.meshgen import facets_on_plane
    m, p = make_config("c5", variant, SMALL["c5"])
    xm, xp, ym, zp = (facets_on_plane(m, 0, 0.0), facets_on_plane(m, 0, 1.0), facets_on_plane(m, 1, 0.0),
                      facets_on_plane(m, 2, 1.0))
    both = (np.concatenate([xp[0], zp[0]]).astype(np.int32), np.concatenate([xp[1], zp[1]]).astype(np.int8))
    m.bsets = [xm, ym, both]
    m.bset_names = ["x0", "y0", "x1_z1"]
    sl = (1e-3, -2e-4, 3e-4, -2e-4, 5e-4, 1e-4, 3e-4, 1e-4, -7e-4)
    p.terms = [p.terms[0],
               Term("ELAST_FIX_D1", 0, dict(tau=2e3, dw=(1e-3,))),
               Term("ELAST_FIX_ALL", 1, dict(tau=1e3, dw=(1e-3, -2e-3, 5e-4))),
               Term("ELAST_LOAD", 2, dict(sigma_l=sl)),
               Term("ELAST_FIX_ALL", 2, dict(tau=5e2, dw=(0.0, 1e-3, 0.0)))]
    st = make_state("c5", m, p)
    ora = oracle.assemble(m, p, st)
    assert ora["status"] == 0
    S = _gpu_system(m, p)
    sd = _to_dev(st)
    for sc in SCATTERS:
        for v, r in [S.system(sd, scatter=sc), (S.matrix(sd, scatter=sc).clone(), S.residual(sd, scatter=sc).clone())]:
            assert csr_row_scaled_err(ora["rowptr"], v.cpu().numpy(), ora["values"]) <= TOL, sc
            assert rhs_err(r.cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL, sc
    S.close()


def test_inverted_element_reported_and_edge_cases():
    _need_gpu()
    from helpers import REF_TET, one_element, problem
    from paper_2111_03541_b200 import FemSystem
    pr = problem("thermal", "tet", 1, [("THERMAL_DOMAIN", -1, dict(C=0.0, k=1.0, s=1.0))])
    m = one_element("tet", 1, REF_TET[:, [0, 2, 1, 3]])
    S = FemSystem(m, pr)
    S.system(torch.zeros((1, 1, 4), dtype=torch.float64, device="cuda"))
    rc, bad = S.status()
    assert rc == -4 and bad == 0
    assert S.status() == (0, -1)  # the error word is reset after reading
    S.close()
    # single element, right orientation: matches the oracle
    m = one_element("tet", 1, REF_TET)
    ora = oracle.assemble(m, pr, np.zeros((1, 1, 4)))
    S = FemSystem(m, pr)
    v, r = S.system(torch.zeros((1, 1, 4), dtype=torch.float64, device="cuda"), scatter="tiled")
    assert csr_row_scaled_err(ora["rowptr"], v.cpu().numpy(), ora["values"]) <= TOL
    S.close()


@pytest.mark.parametrize("name,variant", [("c2", "structured"), ("c4", "perturbed"), ("c5", "structured"),
                                          ("c5", "perturbed")])
def test_partitioned_owned_rows_equal_single(name, variant):
    """Each RCB part (local relabelling: owned points, then halo points; partition.py) assembles only its
    owned rows (owner computes, one ghost element layer) from its LOCAL coordinates and state; mapped back
    through node_ids the parts reproduce the single-GPU pattern bit-exactly and values within L20."""
    _need_gpu()
    from helpers import part_csr_to_global, scatter_rows_into
    from paper_2111_03541_b200 import FemSystem
    from paper_2111_03541_b200.partition import partition_nodes
    m, p = make_config(name, variant, SMALL[name])
    st = make_state(name, m, p)
    ora = oracle.assemble(m, p, st)
    parts = partition_nodes(m, 3)
    kh = p.kappa_hat(m.dim)
    for sc in SCATTERS:
        got_v = np.full(len(ora["values"]), np.nan)
        got_r = np.full(len(ora["rhs"]), np.nan)
        for part in parts:
            S = _gpu_system(part.mesh, p, own=part.own)
            v, r = S.system(_to_dev(part.local_state(st)), scatter=sc)
            pp = S.export_pattern(slot=False)
            rows, rp, cols, vals = part_csr_to_global(part, pp["rowptr"].cpu().numpy(), pp["colidx"].cpu().numpy(),
                                                      v.cpu().numpy(), kh, m.n_nodes)
            scatter_rows_into(ora["rowptr"], ora["colidx"], rows, rp, cols, vals, got_v)
            got_r[rows] = r.cpu().numpy()
            assert S.status() == (0, -1)
            S.close()
        assert not np.isnan(got_v).any() and not np.isnan(got_r).any()
        assert csr_row_scaled_err(ora["rowptr"], got_v, ora["values"]) <= TOL, sc
        assert rhs_err(got_r, ora["rhs"], ora["abs_d"]) <= TOL, sc


FULL_SAMPLES = 160


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5"])
def test_full_size_sampled_rows(name):
    """BASELINE.json full sizes, in the launch configuration bench.py times (fused system call):
    the oracle computes a random sample of rows (plus boundary-touching rows) one by one."""
    _need_gpu()
    m, p = make_config(name, "structured")
    st = make_state(name, m, p)
    rng = np.random.default_rng(7)
    sel = np.zeros(m.n_nodes, dtype=bool)
    sel[rng.choice(m.n_nodes, FULL_SAMPLES, replace=False)] = True
    for be, _bf in m.bsets:  # rows touched by boundary terms
        ids = np.unique(m.conn[:, be[rng.choice(len(be), min(8, len(be)), replace=False)]])
        sel[ids[:24]] = True
    sel[[0, m.n_nodes - 1]] = True
    ora = oracle.assemble(m, p, st, row_mask=sel)
    assert ora["status"] == 0
    from paper_2111_03541_b200 import FemSystem
    S = FemSystem(m, p)
    pat = S.export_pattern(slot=False)
    rowptr = pat["rowptr"]
    rows = torch.from_numpy(ora["rows"]).cuda()
    starts, ends = rowptr[rows], rowptr[rows + 1]
    lens = (ends - starts).cpu().numpy()
    np.testing.assert_array_equal(lens, np.diff(ora["rowptr"]))
    idx = torch.cat([torch.arange(int(a), int(b), device="cuda") for a, b in zip(starts.tolist(), ends.tolist())])
    np.testing.assert_array_equal(pat["colidx"][idx].cpu().numpy(), ora["colidx"])
    del pat
    sd = _to_dev(st)
    for sc in ["tiled", "atomic"] + (["stored"] if name in ("c3", "c4") else []):
        v, r = S.system(sd, scatter=sc)
        assert csr_row_scaled_err(ora["rowptr"], v[idx].cpu().numpy(), ora["values"]) <= TOL, sc
        assert rhs_err(r[rows].cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL, sc
    S.close()


def test_linearize_host_sync_and_pipelined_agree():
    """fem_linearize_host (synchronous) and fem_linearize_host_async (double-buffered staging, copy stream)
    give bit-identical matrices, residuals and norms in the ordered tiled mode, call after call."""
    _need_gpu()
    from paper_2111_03541_b200 import fem
    m, p = make_config("c5", "perturbed", SMALL["c5"])
    st = make_state("c5", m, p)
    S = _gpu_system(m, p)
    S.alloc(True, True)
    hs = torch.from_numpy(st).pin_memory()
    n_sync = torch.zeros(2, dtype=torch.float64).pin_memory()
    fem.fem_linearize_host(S.mesh_h, S.pat_h, p, hs, S.values, S.rhs, n_sync, "tiled", P=S.P)
    v_ref, r_ref, n_ref = S.values.clone(), S.rhs.clone(), n_sync.clone()
    n_async = torch.zeros(2, dtype=torch.float64).pin_memory()
    for _ in range(5):
        fem.fem_linearize_host_async(S.mesh_h, S.pat_h, p, hs, S.values, S.rhs, n_async, "tiled", P=S.P)
    torch.cuda.synchronize()
    assert torch.equal(S.values, v_ref) and torch.equal(S.rhs, r_ref) and torch.equal(n_async, n_ref)
    ora = oracle.assemble(m, p, st)
    assert csr_row_scaled_err(ora["rowptr"], S.values.cpu().numpy(), ora["values"]) <= TOL
    S.close()


@pytest.mark.parametrize("name,dims", [("c1", (5,)), ("c3", (3, 2, 1)), ("c4", (3, 2, 2)), ("c5", (3, 2, 2))])
def test_coo_export_matches_oracle_view(name, dims):
    """NEXT-4: the paper's COO (sparse-ID order, reading L4) exported on the GPU equals the
    oracle's coo_view bit-exactly (I, J), and the gathered values are the CSR values."""
    _need_gpu()
    m, p = make_config(name, "perturbed", dims)
    st = make_state(name, m, p)
    ora = oracle.assemble(m, p, st)
    ref = oracle.coo_view(ora, m.n_nodes, p.kappa_hat(m.dim), row_offset=7)
    S = _gpu_system(m, p)
    S.system(_to_dev(st), scatter="coloured")
    coo = S.export_coo(row_offset=7)
    assert np.array_equal(coo["I"].cpu().numpy(), ref["I"]) and np.array_equal(coo["J"].cpu().numpy(), ref["J"])
    assert np.array_equal(coo["values"].cpu().numpy(), S.values.cpu().numpy()[coo["csr_index"].cpu().numpy()])
    rp = ora["rowptr"]
    scale = np.repeat(np.maximum.reduceat(np.abs(ora["values"]), rp[:-1]), np.diff(rp))
    err = np.abs(coo["values"].cpu().numpy() - ref["values"]) / scale[coo["csr_index"].cpu().numpy()]
    assert err.max() <= TOL
    S.close()


def test_two_workpieces_block_diagonal_coo():
    """Two workpieces: their COO blocks at offsets n^dense (rows) and n^sp (sparse IDs) form
    the block-diagonal system; rows of workpiece 1 never couple to workpiece 0."""
    _need_gpu()
    parts = []
    off_rows = off_sp = 0
    for name, dims in [("c1", (4,)), ("c5", (2, 2, 2))]:
        m, p = make_config(name, "perturbed", dims)
        st = make_state(name, m, p)
        S = _gpu_system(m, p)
        S.system(_to_dev(st), scatter="tiled")
        coo = S.export_coo(row_offset=off_rows)
        ref = oracle.coo_view(oracle.assemble(m, p, st), m.n_nodes, p.kappa_hat(m.dim), row_offset=off_rows)
        assert np.array_equal(coo["I"].cpu().numpy(), ref["I"])
        parts.append((off_sp, coo["I"].cpu().numpy(), coo["J"].cpu().numpy()))
        off_rows += S.n_rows
        off_sp += S.nnz
        S.close()
    (s0, I0, J0), (s1, I1, J1) = parts
    assert s1 == len(I0) and I1.min() >= I0.max() + 1 and J1.min() >= J0.max() + 1


@pytest.mark.parametrize("sc", ["tiled", "tiled_unordered"])
def test_hex_elasticity_node_tiles_on_rotated_mesh(sc):
    """A Q1-hex elasticity mesh that does not bin onto an axis-aligned lattice (c5 rotated by 30° about z
    and 20° about x) keeps the node-tile schedule (k_hex_rec) instead of the z-sweep: parity with the
    oracle and, for FEM_SCATTER_TILED, bit-identical repeats."""
    _need_gpu()
    m, p = make_config("c5", "perturbed", SMALL["c5"])
    a, b = np.radians(30.0), np.radians(20.0)
    Rz = np.array([[np.cos(a), -np.sin(a), 0], [np.sin(a), np.cos(a), 0], [0, 0, 1]])
    Rx = np.array([[1, 0, 0], [0, np.cos(b), -np.sin(b)], [0, np.sin(b), np.cos(b)]])
    m.coords = np.ascontiguousarray(Rx @ Rz @ m.coords)
    st = make_state("c5", m, p)
    ora = oracle.assemble(m, p, st)
    assert ora["status"] == 0
    S = _gpu_system(m, p)
    assert S.info()["schedule"] == 0  # node tiles
    sd = _to_dev(st)
    v, r = [x.clone() for x in S.system(sd, scatter=sc)]
    assert csr_row_scaled_err(ora["rowptr"], v.cpu().numpy(), ora["values"]) <= TOL
    assert rhs_err(r.cpu().numpy(), ora["rhs"], ora["abs_d"]) <= TOL
    if sc == "tiled":
        v2, r2 = S.system(sd, scatter=sc)
        assert torch.equal(v, v2) and torch.equal(r, r2)
    S.close()
