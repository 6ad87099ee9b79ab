#!/usr/bin/env python3
"""bench.py — BASELINE.json metric: assembled elements/s and CSR nnz/s (fp64), % of HBM roofline.

One *step* = one Newton linearisation of the hot path: D-3 matrix + D-2 residual of
every weak-form term (fem_assemble_system) over the whole mesh, through the
C ABI, with the pattern + slot map prebuilt (one-time Block B, reported separately).

Default workload: c5 = 256^3 Q1 hex linear elasticity (16,777,216 elements, 4,092,809,481 nnz),
the config BASELINE.json quotes at 1/2/4/8 B200.  `--config cN` selects another config.
Multi-GPU (torchrun): owner-computes RCB partition of the control points (local numbering, owned + halo)
with a ghost element layer; each rank writes its owned rows; the residual norms are all-reduced
over NCCL (the D-2 convergence test); time = max over ranks (strong scaling: the mesh is fixed).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--scatter tiled]
  python bench.py --impl reference ...   # the CPU oracle (the reference arm of this tier)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from fem_inputs import CONFIGS, make_config, make_state  # noqa: E402

METRIC = "assembled elements/s (fp64, matrix + residual per step)"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


FP64_PEAK_TFLOPS = 33.0  # measured DFMA peak on this pool's B200 (profiles/r01_m0_microbench.txt)
# Algorithmic fp64 flops per element of one matrix+residual step, counted once per element:
# c5 Q1 hex elasticity, 8 points: J (8·9·8·2 = 1152) + det/J^-1 (8·60 = 480) + G = J^-T ∇̂N (8·8·9·2 = 1152)
# + Gram M^jk_ab (9·64·8·2 = 9216) + K entries (576·4 = 2304) + r = K'd (576·2 = 1152) = 15456.
FLOPS_PER_ELEM = {"c5": 15456}
DMMA_PEAK_TFLOPS = 36.0  # measured fp64 DMMA m8n8k4 peak (profiles/r01_m0b_dmma_smem.txt)

# the record-driven kernel the tiled path launches per configuration (csrc/tiled.cu launch_tiled)
TILED_KERNEL = {"c1": "k_gen_rec<TRI,P1,DET>", "c2": "k_hex_rec<1,DET>", "c3": "k_p2_rec<ORD>",
                "c4": "k_ns_rec<DET> + coloured facet pass", "c5": "k_hex_sweep (z-sweep schedule)"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _oracle_worker(args):
    name, steps = args
    r = run_oracle_steps(name, steps, 0)
    return r["elements"] * steps, r["s_per_step"] * steps


def oracle_all_cores(name, seconds_per_core=8.0):
    """The same serial oracle, unmodified, run as one process per host core on the bounded sample
    (throughput of the CPU reference on the whole host: elements/s summed over the concurrent runs)."""
    import multiprocessing as mp
    cores = os.cpu_count() or 1
    one = run_oracle_steps(name, 1, 0)
    steps = max(1, int(seconds_per_core / max(one["s_per_step"], 1e-6)))
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_oracle_worker, [(name, steps)] * cores)
    wall = time.perf_counter() - t0
    elems = sum(r[0] for r in res)
    return {"value": elems / wall, "unit": "elements/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{cores} concurrent serial-oracle processes x {steps} step(s) on the {name} sub-box "
                      f"({one['elements']} elements each), wall {wall:.1f} s"}


def extra_entry(name, variant, scatter, steps, warmup):
    """One keyed entry of the reported matrix: ms per step (matrix + residual), elements/s,
    nnz/s and the HBM fraction of the algorithmic bytes, for another config / variant, same timing rules."""
    import torch
    from paper_2111_03541_b200 import FemSystem, fem
    peaks, _ = _peaks()
    mesh, prob = make_config(name, variant)
    state = make_state(name, mesh, prob)
    t0 = time.perf_counter()
    S = FemSystem(mesh, prob)
    torch.cuda.synchronize()
    t_pat = time.perf_counter() - t0
    S.alloc(True, True)
    sd = torch.from_numpy(state).cuda()
    out = {}
    for sc in scatter:
        if sc == "stored":  # one-time setup of FEM_SCATTER_STORED (contribution lists, element scratch)
            fem.fem_pattern_stored_prepare(S.pat_h, with_matrix=True)
        def step():
            fem.fem_assemble_system(S.mesh_h, S.pat_h, prob, sd, S.values, S.rhs, 0, sc, P=S.P)
        for _ in range(warmup):
            step()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / steps
        ab = algorithmic_bytes(mesh, prob, S.nnz, S.kh * mesh.n_nodes)
        out[sc] = {"ms_per_step": ms, "elements_per_s": mesh.n_elems / (ms * 1e-3), "nnz_per_s": S.nnz / (ms * 1e-3),
                   "hbm_frac": ab / (ms * 1e-3) / 1e9 / float(peaks.get("hbm_gbs", 6650.0)),
                   "kernel": (TILED_KERNEL.get(name) if sc == "tiled" else
                              "k_p2_el + k_st_gather (element-stored, per-slot gather)" if sc == "stored" and name == "c3" else
                              "k_ns_el + k_st_gather (element-stored, per-slot gather)" if sc == "stored" and name == "c4" else
                              f"{sc} path"),
                   "deterministic": sc in ("tiled", "coloured", "stored")}
    status = S.status()
    res = {"workload": f"{name}: {CONFIGS[name].desc}", "variant": variant, "elements": mesh.n_elems,
           "nnz": S.nnz, "pattern_build_s": t_pat, "status": list(status), "by_scatter": out}
    S.close()
    del sd
    torch.cuda.empty_cache()
    return res


def _traffic(name, variant, scatter):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel from the committed
    `ncu --set full` capture (profiles/traffic.json, written by tools/ncu_traffic.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)[f"{name}/{variant}/{scatter}"]
        return float(t["dram_bytes"]), t["source"]
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._thr = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._thr:
            self._thr.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def algorithmic_bytes(mesh, prob, nnz, n_rows):
    """Bytes the method must move per step: each nnz written once, the residual rows,
    the connectivity, the node data (coords + state) and the 1-byte local slot offsets."""
    kh = prob.kappa_hat(mesh.dim)
    E, N, nl = mesh.n_elems, mesh.n_nodes, mesh.n_loc
    return 8 * nnz + 8 * n_rows + 4 * nl * E + 8 * (mesh.dim + kh) * N + nl * nl * E


def cpu_sample(name):
    """A bounded sample of the workload for the oracle: a sub-box with the config's element size,
    element type, physics and boundary terms."""
    dims = {"c1": (8,), "c2": (64, 64, 32), "c3": (60, 10, 10), "c4": (60, 20, 20), "c5": (64, 64, 12)}[name]
    m, p = make_config(name, "structured", dims)
    full = CONFIGS[name].full_dims
    # rescale to the full config's spacing so the sample has the workload's element size
    if name != "c1":
        lengths = {"c2": (1, 1, 1), "c3": (10, 1, 1), "c4": (2.5, .41, .41), "c5": (1, 1, 1)}[name]
        for d in range(3):
            m.coords[d] *= (lengths[d] / full[d] * dims[d]) / max(m.coords[d].max(), 1e-300)
    return m, p, make_state(name, m, p)


def run_oracle_steps(name, steps, warmup):
    import oracle
    oracle.build()
    m, p, st = cpu_sample(name)
    for _ in range(warmup):
        oracle.assemble(m, p, st)
    times = []
    nnz = 0
    for _ in range(steps):
        t0 = time.perf_counter()
        o = oracle.assemble(m, p, st)
        times.append(time.perf_counter() - t0)
        nnz = len(o["values"])
    t = sum(times) / len(times)
    return {"elements": m.n_elems, "nnz": nnz, "s_per_step": t, "value": m.n_elems / t, "nnz_per_s": nnz / t,
            "sample": f"{name} sub-box {m.n_elems} elements at the full config's spacing, matrix+residual, "
                      f"serial C oracle, {steps} step(s)"}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    r = run_oracle_steps(args.config, args.steps, args.warmup)
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": "elements/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["s_per_step"] * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {CONFIGS[args.config].desc} (oracle sample)",
                       "sample_elements": r["elements"]},
            "nnz_per_s": r["nnz_per_s"],
            "cpu_baseline": {"value": r["value"], "unit": "elements/s", "cores": 1, "kind": "oracle",
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=list(CONFIGS))
    ap.add_argument("--variant", default="structured", choices=["structured", "perturbed"])
    ap.add_argument("--scatter", default="tiled", choices=["tiled", "atomic", "coloured"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the keyed c2-c4 / perturbed-c5 entries")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)
    args.warmup = max(args.warmup, 3)

    import torch
    import torch.distributed as dist

    from paper_2111_03541_b200 import FemSystem, fem
    from paper_2111_03541_b200.partition import part_for_rank

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    name = args.config
    mesh, prob = make_config(name, args.variant)
    state = make_state(name, mesh, prob)
    E_total = mesh.n_elems
    if world > 1:  # RCB part in local numbering: only owned + halo points travel to this GPU
        part = part_for_rank(mesh, world, rank)
        local_mesh, own = part.mesh, part.own
        state = part.local_state(state)
    else:
        local_mesh, own = mesh, (0, mesh.n_nodes)
    t0 = time.perf_counter()
    S = FemSystem(local_mesh, prob, own=own)
    torch.cuda.synchronize()
    t_pattern = time.perf_counter() - t0
    nnz_local = S.nnz
    S.alloc(True, True)
    sd = torch.from_numpy(state).cuda()
    stream = torch.cuda.current_stream()
    norms = torch.zeros(2, dtype=torch.float64, device="cuda")

    def step():
        fem.fem_assemble_system(S.mesh_h, S.pat_h, prob, sd, S.values, S.rhs, 0, args.scatter, P=S.P)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    # residual norms (the D-2 convergence check) reduced over ranks: the one collective of the path
    fem.fem_residual_norms(S.mesh_h, S.rhs, norms)
    if world > 1:
        sq = norms[:1].clone()
        mx = norms[1:].clone()
        dist.all_reduce(sq)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        nz = torch.tensor([nnz_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(nz)
        nnz_total = int(nz.item())
    else:
        nnz_total = nnz_local
    status = S.status()
    # ---- end to end through the C ABI with HOST buffers (pinned state in, norms out, per step)
    host_state = torch.from_numpy(state).pin_memory()
    host_norms = torch.zeros(2, dtype=torch.float64).pin_memory()
    # fem_linearize_host_async: the H2D of step k+1 (library copy stream, double-buffered staging)
    # overlaps the assembly of step k; every step still copies its full state in and its norms out
    for _ in range(2):
        fem.fem_linearize_host_async(S.mesh_h, S.pat_h, prob, host_state, S.values, S.rhs, host_norms,
                                     args.scatter, P=S.P)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(e2e_steps):
        fem.fem_linearize_host_async(S.mesh_h, S.pat_h, prob, host_state, S.values, S.rhs, host_norms,
                                     args.scatter, P=S.P)
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    # ---- dominant kernel timing on its own stream (one launch per step for the tiled path)
    kern_ms = ms
    if rank == 0:
        peaks, peak_kind = _peaks()
        hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
        alg_bytes = algorithmic_bytes(mesh, prob, nnz_total, S.kh * mesh.n_nodes)
        achieved = alg_bytes / (kern_ms * 1e-3) / 1e9 / world
        traffic, traffic_src = _traffic(name, args.variant, args.scatter) if world == 1 else (None, None)
        cpu = cpu_all = None
        if not args.no_cpu_baseline and world == 1:
            r = run_oracle_steps(name, 1, 0)
            cpu = {"value": r["value"], "unit": "elements/s", "cores": 1, "kind": "oracle", "sample": r["sample"],
                   "cpu_model": cpu_model()}
            cpu_all = oracle_all_cores(name)
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": E_total / (ms * 1e-3), "unit": "elements/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{name}: {CONFIGS[name].desc}", "variant": args.variant,
                       "elements": E_total, "nodes": mesh.n_nodes, "nnz": nnz_total, "scatter": args.scatter,
                       "parallelism": f"owner-computes node partition x{world}" if world > 1 else "single GPU",
                       "l2": f"inputs larger than L2 (values {8 * nnz_total / 1e9:.1f} GB)"},
            "nnz_per_s": nnz_total / (ms * 1e-3),
            "pattern_build_s": t_pattern,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "peak_kind": f"{peak_kind} hbm_gbs", "algorithmic_bytes_per_step": alg_bytes,
                         "kernel": (TILED_KERNEL[name] if args.scatter == "tiled" else f"{args.scatter} kernels")
                         + " (fem_assemble_system)"},
            "fp64": {"peak_tflops": FP64_PEAK_TFLOPS, "peak_kind": "measured DFMA (tools/m0)",
                     "dmma_peak_tflops": DMMA_PEAK_TFLOPS,
                     "algorithmic_flops_per_element": FLOPS_PER_ELEM.get(name),
                     "achieved_tflops": (FLOPS_PER_ELEM[name] * E_total / (ms * 1e-3) / 1e12
                                         if name in FLOPS_PER_ELEM else None),
                     "frac": (FLOPS_PER_ELEM[name] * E_total / (ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS
                              if name in FLOPS_PER_ELEM else None)},
            "cpu_baseline": cpu,
            "cpu_baseline_all_cores": cpu_all,
            "e2e": {"value": E_total / (e2e_ms * 1e-3), "unit": "elements/s",
                    "h2d_bytes_per_step": int(state.nbytes), "d2h_bytes_per_step": 16,
                    "ms_per_step": e2e_ms, "call": "fem_linearize_host_async (pipelined H2D)",
                    "result": "K and d stay in device memory for the device solver (D-4); the host reads back "
                              "the residual norms (||d||_2, ||d||_inf: 16 bytes) each step"},
            "gpu_launches": args.steps * (1 if args.scatter == "tiled" else 1 + len(prob.terms) * 8),
            "clocks": clocks,
            "status": list(status),
        }
    S.close()
    if rank == 0 and world == 1 and not args.no_extras and args.config == "c5":
        # the rest of the reported matrix, measured in the same run (not the headline): c2-c4 structured
        # and the perturbed-unstructured c5, TILED (deterministic) and for c3/c4 also TILED_UNORDERED; c3 also
        # STORED (deterministic element-stored gather, its fastest deterministic mode)
        del sd
        import gc
        gc.collect()
        torch.cuda.empty_cache()
        extras = {}
        for nm, var, scs in [("c2", "structured", ["tiled"]), ("c3", "structured", ["tiled", "tiled_unordered", "stored"]),
                             ("c4", "structured", ["tiled", "tiled_unordered", "stored"]), ("c5", "perturbed", ["tiled"])]:
            try:
                extras[f"{nm}/{var}"] = extra_entry(nm, var, scs, max(3, min(args.steps, 10)), 3)
            except Exception as exc:  # reported, never hidden
                extras[f"{nm}/{var}"] = {"error": repr(exc)}
        line["extra"] = extras
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
