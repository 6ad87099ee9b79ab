"""Time the NEXT-3 vector updates (fem_time_init / _effective / _increment) at c5's system size
(n = κ̂N = 50,923,779, ν̂ = 2) with CUDA events on the launching stream; report GB/s of algorithmic
traffic (doubles per row moved once: C+D-1 5(ν̂+1), D-1 3(ν̂+1), D-4+D-1 1+4(ν̂+1)) against MEASURED_PEAKS.json."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fem_inputs.configs import TimeScheme  # noqa: E402
from paper_2111_03541_b200 import fem  # noqa: E402


def main():
    n, nu = int(os.environ.get("TS_N", 50_923_779)), int(os.environ.get("TS_NU", 2))
    L = nu + 1
    T = fem.make_time_scheme(TimeScheme("genalpha", nu, dt=0.01, b1=0.5, b2=0.5, c1=0.9, c2=0.9, c3=0.9))
    g = torch.Generator(device="cuda").manual_seed(0)
    phi0 = torch.randn(L, n, dtype=torch.float64, device="cuda", generator=g)
    incr = torch.randn(L, n, dtype=torch.float64, device="cuda", generator=g)
    eff = torch.empty_like(phi0)
    dsub = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    s = torch.cuda.current_stream()
    calls = {  # name: (fn, algorithmic bytes)
        "init+D1": (lambda: fem.fem_time_init(T, n, phi0, incr, eff), 8 * n * (2 * L + 3 * L)),
        "effective": (lambda: fem.fem_time_effective(T, n, phi0, incr, eff), 8 * n * 3 * L),
        "increment+D1": (lambda: fem.fem_time_increment(T, n, dsub, incr, phi0, eff), 8 * n * (1 + 4 * L)),
    }
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))
    hbm = peak["hbm_gbs"]
    out = {"n": n, "nu_hat": nu, "hbm_peak_gbs": hbm}
    for name, (fn, nbytes) in calls.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(20):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        out[name] = {"ms": ms, "GB/s": nbytes / ms / 1e6, "frac": nbytes / ms / 1e6 / hbm}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
