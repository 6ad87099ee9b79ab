"""NEXT-1 measurement: SpMV and Jacobi-PCG iteration on an assembled config (default c5, full size).
python tools/bench_solve.py [config] [dims...] -> one JSON line (CUDA events on the current stream)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fem_inputs import make_config, make_state  # noqa: E402
from paper_2111_03541_b200 import FemSystem, fem  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
dims = tuple(int(x) for x in sys.argv[2:]) or None
m, p = make_config(name, "structured", dims)
S = FemSystem(m, p)
st = torch.from_numpy(make_state(name, m, p)).cuda()
K, d = S.system(st, scatter="tiled")
n, nnz = S.n_rows, S.nnz
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.zeros(n, dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    S.spmv(x, y)
torch.cuda.synchronize()
reps = 10
ev[0].record()
for _ in range(reps):
    S.spmv(x, y)
ev[1].record()
torch.cuda.synchronize()
spmv_ms = ev[0].elapsed_time(ev[1]) / reps
spmv_bytes = 12 * nnz + 8 * (n + 1) + 8 * n + 8 * n  # values+colidx, rowptr, y, x (each element once)
peak = 6547.2
try:
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f).get("hbm_gbs", peak))
except Exception:
    pass
# CG: a fixed number of iterations (rtol = 0), timed end to end (3 launches per iteration + the checks)
iters = 40
S.solve(-d, rtol=0.0, max_iter=4, check_every=4)
torch.cuda.synchronize()
ev[0].record()
_, it, rel = S.solve(-d, rtol=0.0, max_iter=iters, check_every=iters)
ev[1].record()
torch.cuda.synchronize()
cg_ms = ev[0].elapsed_time(ev[1]) / iters
cg_bytes = spmv_bytes + 8 * n * 10  # + update (x, p, q, r, dinv read; x, r, z write) + direction (z, p read; p write)
print(json.dumps({
    "workload": f"{name} {m.n_elems} elements", "rows": n, "nnz": nnz,
    "spmv": {"ms": spmv_ms, "algorithmic_bytes": spmv_bytes, "achieved_gbs": spmv_bytes / spmv_ms / 1e6,
             "peak_gbs": peak, "frac": spmv_bytes / spmv_ms / 1e6 / peak},
    "cg_iteration": {"ms": cg_ms, "algorithmic_bytes": cg_bytes, "achieved_gbs": cg_bytes / cg_ms / 1e6,
                     "frac": cg_bytes / cg_ms / 1e6 / peak, "iterations_timed": it},
    "note": "values/colidx (49 GB on c5) exceed L2: every pass streams HBM"}))
