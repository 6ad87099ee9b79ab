"""World-size-2 gloo test of the multi-GPU host path, run on CPU.

Each rank takes its owner-computes part from paper_2111_03541_b200.partition (RCB of the points, local
relabelling: owned points then halo points), assembles its owned rows with the oracle on the LOCAL mesh
(no GPU here), and the residual norms are all-reduced exactly as bench.py does over NCCL.  The parts,
mapped back through node_ids, must equal the single-process rows (pattern exact, values to rounding), the
reduced norms the global norms, and every rank must hold about 1/N of the elements and points.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, dims, variant, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from fem_inputs import make_config, make_state
    from paper_2111_03541_b200.partition import part_for_rank
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m, p = make_config(name, variant, dims)
    st = make_state(name, m, p)
    part = part_for_rank(m, world, rank)
    mask = np.zeros(part.mesh.n_nodes, dtype=bool)
    mask[: part.n_owned] = True
    out = oracle.assemble(part.mesh, p, part.local_state(st), row_mask=mask)
    assert out["status"] == 0
    d = torch.from_numpy(out["rhs"])
    sq = torch.tensor([float((d * d).sum())], dtype=torch.float64)
    mx = torch.tensor([float(d.abs().max()) if d.numel() else 0.0], dtype=torch.float64)
    dist.all_reduce(sq)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)  # max-over-ranks timing reduction
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), rowptr=out["rowptr"], colidx=out["colidx"],
             values=out["values"], rhs=out["rhs"], sq=sq.numpy(), mx=mx.numpy(), t=t.numpy(),
             n_elems=part.mesh.n_elems, n_local=part.mesh.n_nodes, n_owned=part.n_owned)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,dims", [("c2", (5, 4, 6)), ("c4", (6, 3, 3)), ("c5", (4, 3, 5))])
@pytest.mark.parametrize("variant", ["structured", "perturbed"])
def test_two_rank_partition_reproduces_global_rows(tmp_path, name, dims, variant):
    import oracle
    from fem_inputs import make_config, make_state
    from helpers import part_csr_to_global, scatter_rows_into
    from paper_2111_03541_b200.partition import part_for_rank
    oracle.build()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, dims, variant, str(tmp_path)), nprocs=world, join=True)
    m, p = make_config(name, variant, dims)
    st = make_state(name, m, p)
    kh = p.kappa_hat(m.dim)
    full = oracle.assemble(m, p, st)
    got_v = np.full(len(full["values"]), np.nan)
    got_r = np.full(len(full["rhs"]), np.nan)
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        part = part_for_rank(m, world, r)
        rows, rp, cols, vals = part_csr_to_global(part, z["rowptr"], z["colidx"], z["values"], kh, m.n_nodes)
        scatter_rows_into(full["rowptr"], full["colidx"], rows, rp, cols, vals, got_v)
        got_r[rows] = z["rhs"]
        assert z["t"][0] == world
    assert not np.isnan(got_v).any() and not np.isnan(got_r).any()   # every row owned exactly once
    np.testing.assert_allclose(got_v, full["values"], rtol=0, atol=1e-13 * np.abs(full["values"]).max())
    np.testing.assert_allclose(got_r, full["rhs"], rtol=1e-13, atol=1e-300)
    z = np.load(tmp_path / "r0.npz")
    assert z["sq"][0] == pytest.approx(float((full["rhs"] ** 2).sum()), rel=1e-12)
    assert z["mx"][0] == pytest.approx(float(np.abs(full["rhs"]).max()), rel=0, abs=0)


@pytest.mark.parametrize("variant", ["structured", "perturbed"])
@pytest.mark.parametrize("nparts", [2, 4, 8])
def test_rcb_parts_are_balanced_and_compact(variant, nparts):
    """on the perturbed variant (random node and element numbering) RCB still gives
    box-like parts: points balanced to one; elements within 10% of E/N for 2 ranks ((4,4,40): 20 layers +
    one ghost layer, ragged by the jitter), within 20% for 4 and 8 ranks on cubes (several cut faces of
    a 24³/32³ mesh); a rank's local arrays (coordinates, state) are owned + halo points only."""
    from fem_inputs import make_config
    from paper_2111_03541_b200.partition import partition_nodes
    dims = {2: (4, 4, 40), 4: (24, 24, 24), 8: (32, 32, 32)}[nparts]
    m, _ = make_config("c5", variant, dims)
    parts = partition_nodes(m, nparts)
    own = [p.n_owned for p in parts]
    assert sum(own) == m.n_nodes and max(own) - min(own) <= 1
    allown = np.concatenate([p.node_ids[: p.n_owned] for p in parts])
    assert np.array_equal(np.sort(allown), np.arange(m.n_nodes))
    E, N = m.n_elems, m.n_nodes
    ghost = {2: 1.1, 4: 1.2, 8: 1.2}[nparts]   # one ghost element layer on each cut face
    for p in parts:
        assert p.mesh.n_elems <= ghost * E / nparts, (p.rank, p.mesh.n_elems, E / nparts)
        assert p.mesh.n_nodes <= (ghost + 0.15) * N / nparts   # owned + the halo points of the ghost layer
        assert p.mesh.conn.max() < p.mesh.n_nodes
