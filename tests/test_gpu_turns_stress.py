"""Stress of the hand-rolled synchronisation (compute-sanitizer is closed on this GPU pool):
the ordered per-row turns (ld.acquire / st.release on shared memory), the sweep's ring lives, first-touch
stores and last-toucher TMA write-outs, and the stored mode's fixed-order gathers.  A missed or wrong
hand-off shows up as a value that changes between repeats (a lost update or a read of a half-written row)
or as a hang (caught by the pytest timeout).  Meshes sized so that many tiles / columns run concurrently
and every warp of a CTA is busy; 60 repeats each, bit-identical to the first, the first checked against
the oracle on sampled rows."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from fem_inputs import make_config, make_state  # noqa: E402
from helpers import csr_row_scaled_err, rhs_err  # noqa: E402

REPEATS = 60
CASES = [("c5", (40, 36, 70), "tiled"), ("c3", (40, 8, 8), "tiled"), ("c4", (40, 16, 12), "tiled"),
         ("c3", (40, 8, 8), "stored"), ("c2", (40, 30, 20), "tiled")]


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name,dims,sc", CASES)
def test_ordered_modes_bit_identical_under_load(name, dims, sc):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from helpers import poisoned_system
    m, p = make_config(name, "perturbed", dims)
    st = make_state(name, m, p)
    S = poisoned_system(m, p)
    sd = torch.from_numpy(st).cuda()
    v0, r0 = [x.clone() for x in S.system(sd, scatter=sc)]
    assert S.status() == (0, -1)
    assert torch.isfinite(v0).all() and torch.isfinite(r0).all()
    for _ in range(REPEATS):
        v, r = S.system(sd, scatter=sc)
        assert torch.equal(v, v0) and torch.equal(r, r0)
    # the first result is also right: sampled rows against the oracle (rows of a random node sample)
    rng = np.random.default_rng(7)
    sel = np.zeros(m.n_nodes, dtype=bool)
    sel[rng.choice(m.n_nodes, 64, replace=False)] = True
    ora = oracle.assemble(m, p, st, row_mask=sel)
    assert ora["status"] == 0
    pat = S.export_pattern(slot=False)
    rowptr = pat["rowptr"]
    rows = torch.from_numpy(ora["rows"]).cuda()
    idx = torch.cat([torch.arange(int(a), int(b), device="cuda")
                     for a, b in zip(rowptr[rows].tolist(), rowptr[rows + 1].tolist())])
    np.testing.assert_array_equal(pat["colidx"][idx].cpu().numpy(), ora["colidx"])
    assert csr_row_scaled_err(ora["rowptr"], v0[idx].cpu().numpy(), ora["values"]) <= 1e-12
    assert rhs_err(r0[rows].cpu().numpy(), ora["rhs"], ora["abs_d"]) <= 1e-12
    S.close()
