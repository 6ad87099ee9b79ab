"""A10: the residual norms of the D-2 convergence test — fem_residual_norms against the oracle's
‖d‖ on the configs, NaN propagation, bit-identity at c5 full size, and the multi-rank reduction of norms
the GPU computed (gloo all-reduce of per-part device norms, exactly as bench.py reduces them over NCCL)."""
import math
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from fem_inputs import make_config, make_state  # noqa: E402

SMALL = {"c2": (9, 7, 6), "c3": (7, 3, 2), "c4": (9, 4, 3), "c5": (7, 5, 6)}


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("name", list(SMALL))
def test_norms_match_oracle(name):
    """‖d‖₂ and ‖d‖∞ of the tiled system call vs the oracle's d.  Since |Δd_i| ≤ 1e-12·max(|d_i|, A_d[i])
    (reading L20), |‖d_gpu‖ − ‖d_ora‖| ≤ ‖Δd‖ ≤ 1e-12·‖|d_ora| + A_d‖ for both norms."""
    _need_gpu()
    from paper_2111_03541_b200 import FemSystem
    m, p = make_config(name, "perturbed", SMALL[name])
    st = make_state(name, m, p)
    ora = oracle.assemble(m, p, st)
    S = FemSystem(m, p)
    S.system(torch.from_numpy(st).cuda(), scatter="tiled")
    nrm = S.norms().cpu().numpy()
    d, A = ora["rhs"], ora["abs_d"]
    bound2 = 1e-12 * np.linalg.norm(np.abs(d) + A)
    boundi = 1e-12 * (np.abs(d) + A).max()
    assert abs(math.sqrt(nrm[0]) - np.linalg.norm(d)) <= bound2 + 1e-15 * np.linalg.norm(d)
    assert abs(nrm[1] - np.abs(d).max()) <= boundi
    # and the norms of the GPU's own residual: Σd² to summation-order rounding, max exactly
    r = S.rhs.cpu().numpy()
    assert nrm[0] == pytest.approx(float((r * r).sum()), rel=1e-13)
    assert nrm[1] == float(np.abs(r).max())
    S.close()


def test_norms_nan_and_empty():
    _need_gpu()
    from paper_2111_03541_b200 import FemSystem
    m, p = make_config("c5", "structured", (3, 3, 3))
    S = FemSystem(m, p, build_pattern=False)
    n = S.kh * S.N
    d = torch.ones(n, dtype=torch.float64, device="cuda")
    d[n // 2] = float("nan")
    nrm = S.norms(d).cpu().numpy()
    assert math.isnan(nrm[0]) and math.isnan(nrm[1])
    d.fill_(float("nan"))
    nrm = S.norms(d).cpu().numpy()
    assert math.isnan(nrm[0]) and math.isnan(nrm[1])   # fmax would have returned 0 here
    d = torch.linspace(-3.0, 2.0, n, dtype=torch.float64, device="cuda")
    nrm = S.norms(d).cpu().numpy()
    assert nrm[1] == 3.0
    assert nrm[0] == pytest.approx(float((d.cpu().numpy() ** 2).sum()), rel=1e-13)
    S.close()


def test_norms_bit_identical_full_c5():
    """c5 full size: 50.9 M rows (κ̂N of the 256³ mesh); repeated calls give bit-identical norms (the
    round-1 kernel combined blocks with a global atomicAdd).  The norm depends on κ̂·N only, so the
    mesh here carries the full node set and a single element."""
    _need_gpu()
    from fem_inputs.meshgen import Mesh
    from paper_2111_03541_b200 import FemSystem
    _, p = make_config("c5", "structured", (2, 2, 2))
    n1 = 257
    N = n1 ** 3
    coords = np.zeros((3, N))
    i = np.arange(N)
    coords[0], coords[1], coords[2] = (i % n1) / 256.0, (i // n1 % n1) / 256.0, (i // (n1 * n1)) / 256.0
    conn = np.array([[0], [1], [1 + n1], [n1], [n1 * n1], [1 + n1 * n1], [1 + n1 + n1 * n1], [n1 + n1 * n1]],
                    dtype=np.int32)
    m = Mesh(3, "hex", 1, coords, conn)
    m.bsets = [(np.zeros(0, np.int32), np.zeros(0, np.int8))] * 2
    S = FemSystem(m, p, build_pattern=False)
    g = torch.Generator(device="cuda").manual_seed(7)
    d = torch.rand(3 * N, dtype=torch.float64, device="cuda", generator=g) * 2e-3 - 1e-3
    ref = S.norms(d).clone()
    for _ in range(5):
        assert torch.equal(S.norms(d), ref)
    dh = d.cpu().numpy()
    assert ref[0].item() == pytest.approx(float((dh * dh).sum()), rel=1e-12)
    assert ref[1].item() == float(np.abs(dh).max())
    S.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _norm_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from fem_inputs import make_config, make_state
    from paper_2111_03541_b200 import FemSystem
    from paper_2111_03541_b200.partition import part_for_rank
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, p = make_config("c5", "perturbed", (5, 4, 9))
    st = make_state("c5", m, p)
    part = part_for_rank(m, world, rank)
    S = FemSystem(part.mesh, p, own=part.own)
    S.system(torch.from_numpy(part.local_state(st)).cuda(), scatter="tiled")
    nrm = S.norms().cpu()
    sq, mx = nrm[:1].clone(), nrm[1:].clone()
    dist.all_reduce(sq)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    np.save(os.path.join(out_dir, f"n{rank}.npy"), np.array([sq.item(), mx.item()]))
    S.close()
    dist.destroy_process_group()


def test_two_rank_norms_reduce_to_global(tmp_path):
    """Two ranks (sequential kernels on one GPU, gloo on host tensors; the kernels do not wait on each
    other) each compute fem_residual_norms over their owned rows; the all-reduced norms equal the norms of
    the oracle's global d within the L20 bound."""
    _need_gpu()
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_norm_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    m, p = make_config("c5", "perturbed", (5, 4, 9))
    st = make_state("c5", m, p)
    ora = oracle.assemble(m, p, st)
    d, A = ora["rhs"], ora["abs_d"]
    for r in range(world):
        sq, mx = np.load(tmp_path / f"n{r}.npy")
        assert abs(math.sqrt(sq) - np.linalg.norm(d)) <= 1e-12 * np.linalg.norm(np.abs(d) + A) + 1e-15 * np.linalg.norm(d)
        assert abs(mx - np.abs(d).max()) <= 1e-12 * (np.abs(d) + A).max()
