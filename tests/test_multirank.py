"""World-size-2 gloo test of the multi-GPU host path, run on CPU.

Each rank takes its owner-computes part (contiguous control-point range + ghost element layer) from
paper_2111_03541_b200.partition, assembles its owned rows with the oracle (no GPU here), and the
residual norms are all-reduced exactly as bench.py does over NCCL.  The union of the parts must equal
the single-process rows, and the reduced norms the global norms.
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
    lo, hi = part.own
    mask = np.zeros(m.n_nodes, dtype=bool)
    mask[lo:hi] = True
    out = oracle.assemble(part.mesh, p, st, row_mask=mask)
    assert out["status"] == 0
    d = torch.from_numpy(out["rhs"])
    sq = torch.tensor([float((d * d).sum())], dtype=torch.float64)
    mx = torch.tensor([float(d.abs().max()) if d.numel() else 0.0], dtype=torch.float64)
    dist.all_reduce(sq)
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)  # max-over-ranks timing reduction
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), rows=out["rows"], rowptr=out["rowptr"], colidx=out["colidx"],
             values=out["values"], rhs=out["rhs"], sq=sq.numpy(), mx=mx.numpy(), t=t.numpy(),
             n_elems=part.mesh.n_elems)
    dist.destroy_process_group()


@pytest.mark.parametrize("name,dims", [("c2", (5, 4, 6)), ("c4", (6, 3, 3)), ("c5", (4, 3, 5))])
@pytest.mark.parametrize("variant", ["structured", "perturbed"])
def test_two_rank_partition_reproduces_global_rows(tmp_path, name, dims, variant):
    import oracle
    from fem_inputs import make_config, make_state
    oracle.build()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, dims, variant, str(tmp_path)), nprocs=world, join=True)
    m, p = make_config(name, variant, dims)
    st = make_state(name, m, p)
    full = oracle.assemble(m, p, st)
    K = oracle.to_dense(full, len(full["rows"]))
    got_rows = []
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        part = {k: z[k] for k in ("rows", "rowptr", "colidx", "values")}
        Kp = oracle.to_dense(part, len(full["rows"]))
        np.testing.assert_allclose(Kp, K[z["rows"]], rtol=0, atol=1e-13 * np.abs(K).max())
        np.testing.assert_allclose(z["rhs"], full["rhs"][z["rows"]], rtol=1e-13, atol=1e-300)
        got_rows.append(z["rows"])
        assert z["t"][0] == world
        if variant == "structured":  # z-slab ranges: a part holds its elements + one ghost layer
            assert z["n_elems"] < m.n_elems
    rows = np.sort(np.concatenate(got_rows))
    np.testing.assert_array_equal(rows, np.arange(len(full["rows"])))
    z = np.load(tmp_path / "r0.npz")
    assert z["sq"][0] == pytest.approx(float((full["rhs"] ** 2).sum()), rel=1e-12)
    assert z["mx"][0] == pytest.approx(float(np.abs(full["rhs"]).max()), rel=0, abs=0)
