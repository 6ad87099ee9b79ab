"""NEXT-3 measurement: generalized-alpha timesteps of transient heat conduction (ν̂ = 1) on c2 full size
(64^3 Q1 hex, 274,625 rows) through FemSystem.time_step: Block C + n_sub x (assembly, BiCGStab, D-4).
CUDA events on the current stream; the component kernels are timed separately for the breakdown.
python tools/bench_transient.py [steps] [n_sub] -> one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fem_inputs import make_config, make_state  # noqa: E402
from fem_inputs.configs import TimeScheme  # noqa: E402
from paper_2111_03541_b200 import FemSystem, fem  # noqa: E402


def ev_time(fn, reps=5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    n_sub = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    m, p = make_config("c2", "structured")
    p.time = TimeScheme("genalpha", 1, dt=0.02, b1=0.8, b2=0.5, c1=1.0, c2=1.0, c3=1.0)
    p.terms[0].params = dict(p.terms[0].params, C=3.0)
    st = make_state("c2", m, p)
    st[1] = 0.0
    S = FemSystem(m, p)
    phi0 = torch.from_numpy(st).cuda()
    incr = torch.zeros_like(phi0)
    S.time_step(phi0, incr, n_sub=n_sub, rtol=1e-10)          # warm-up (allocations, first launches)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = []
    e0.record()
    for _ in range(steps):
        iters.append([h[1] for h in S.time_step(phi0, incr, n_sub=n_sub, rtol=1e-10)])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    n = S.n_rows
    ts = fem.make_time_scheme(p.time)
    eff = S._eff
    asm_ms = ev_time(lambda: S.system(eff, scatter="tiled"))
    dsub = torch.zeros(n, dtype=torch.float64, device="cuda")
    init_ms = ev_time(lambda: fem.fem_time_init(ts, n, phi0.clone(), incr.clone(), eff))
    inc_ms = ev_time(lambda: fem.fem_time_increment(ts, n, dsub, incr, phi0, eff))
    print(json.dumps({
        "workload": "c2 transient heat, 64^3 Q1 hex, genalpha nu_hat=1 (b1=0.8, c=1), BiCGStab rtol 1e-10",
        "rows": n, "nnz": S.nnz, "steps_timed": steps, "n_sub": n_sub, "ms_per_timestep": ms,
        "timesteps_per_s": 1e3 / ms, "bicgstab_iterations": iters,
        "breakdown_ms": {"assembly_system": asm_ms, "time_init+D1_incl_clones": init_ms, "increment+D1": inc_ms},
        "note": "rest of each timestep = the BiCGStab solves + residual norms (host sync per sub-step)"}))


if __name__ == "__main__":
    main()
