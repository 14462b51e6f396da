"""Benchmark of the B200 2F block J-Jacobi hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--no-cpu-baseline]

One "step" is one whole eigensolve (parallel_jacobi, variant 2F, round-robin,
orth_tol = n*eps) of the BASELINE configuration.  N=1 runs configs[1] (cfg2:
complex128 2048x2048, b=64, p=16), the config the metric is quoted on.  For
N>1 (torchrun, one process per GPU) the same solve is split over the GPUs by
ring rank with NCCL block exchange (strong scaling).  Rank 0 prints ONE JSON
line.  ``--impl reference`` times the reference's CPU algorithm (the oracle
restatement, pinned bit-exact to the reference) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(ROOT, ".numba_cache"))

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
FP64_DATASHEET_TFLOPS = 40.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def measure_dgemm(torch, dev):
    """cuBLAS DGEMM 8192^3: the measured FP64 roofline denominator
    (MEASURED_PEAKS.json has no FP64 entry)."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn_like(a)
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * n ** 3 / (best * 1e-3) / 1e12


def flops_of(stats, w, cx):
    from paper_1008_4166_b200 import workloads
    b = w.b
    gram = (4.0 if cx else 1.0) * 2.0 * w.m * b * b * (stats["pairs_visited"] + stats["prepass_visited"])
    upd = (4.0 if cx else 1.0) * (8.0 * w.m * b * b * stats["pairs_updated"]
                                  + 2.0 * w.m * b * b * stats["prepass_updated"])
    total = workloads.algorithmic_flops(w.m, b, cx, stats["pairs_updated"], stats["pairs_visited"],
                                        stats["prepass_updated"], stats["prepass_visited"])
    # inner level: a dot product (2N real flops, x4 complex) per examined 2x2
    # pivot, and 14N real flops (x4 complex) per applied rotation on R and W
    N = 2 * b
    c = 4.0 if cx else 1.0
    piv = c * (2.0 * N * stats["inner_pair_visits"] + 14.0 * N * stats["rotations"])
    return total, gram, upd, piv


def cpu_profile():
    p = os.path.join(ROOT, "oracle", "cpu_profile.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def run_cpu_sample(w, threads):
    """The reference's algorithm (oracle restatement, pinned bit-exact) on
    the host: first sweep of the workload, extrapolated to the full solve
    with the per-sweep profile measured in the build container."""
    import oracle
    oracle.parallel_jacobi_2f(w.G[:128, :128], w.J[:128], 2, "round_robin", orth_tol=w.orth_tol)  # JIT warm
    t0 = time.perf_counter()
    oracle.parallel_jacobi_2f(w.G, w.J, w.p, "round_robin", orth_tol=w.orth_tol, threads=threads,
                              sweep_limit=1)
    t1 = time.perf_counter() - t0
    prof = cpu_profile().get(w.name, {})
    ratio = prof.get("t_total", None) and prof["t_total"] / prof["t_sweep1"]
    est = t1 * ratio if ratio else None
    return t1, est, ratio


def reference_arm(args, w):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    threads = max(1, min(os.cpu_count() or 1, w.p))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    for _ in range(max(0, min(args.warmup, 1))):
        run_cpu_sample(w, threads)
    vals = []
    for _ in range(args.steps):
        t1, est, ratio = run_cpu_sample(w, threads)
        vals.append(est if est else t1)
    v = statistics.mean(vals)
    sample = (f"first outer sweep of {w.name} ({w.description}) with the oracle "
              f"(numpy+numba restatement pinned bit-exact to the reference), p={w.p} worker threads; "
              f"extrapolated x{ratio:.2f} (full/first-sweep time ratio measured in the build container)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128" if np.iscomplexobj(w.G) else "f64",
            "data": "synthetic (seeded, BASELINE.json generators)",
            "config": {"workload": w.name, "n": w.n, "b": w.b, "p": w.p, "strategy": "round_robin",
                       "orth_tol": "n*eps"},
            "cpu_baseline": {"value": v, "unit": "s", "cores": threads, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    from paper_1008_4166_b200 import workloads
    w = workloads.make(args.config)
    if args.impl == "reference":
        return reference_arm(args, w)

    import torch
    import paper_1008_4166_b200 as P
    from paper_1008_4166_b200 import parallel as par
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    pg = None
    if world > 1 or "LOCAL_RANK" in os.environ:  # torchrun: NCCL ring comm even at N=1
        import torch.distributed as dist
        dist.init_process_group("gloo", init_method="env://")
        pg = dist
        from paper_1008_4166_b200 import distributed
        comm = distributed.Comm.create(rank, world, local)
    cx = np.iscomplexobj(w.G)
    cfg = P.SolverConfig(variant="2F", strategy="round_robin", p=w.p, tol=P.Tolerances(orth_tol=w.orth_tol),
                         comm=comm)
    cfg_pt = P.SolverConfig(variant="2F", strategy="round_robin", p=w.p,
                            tol=P.Tolerances(orth_tol=w.orth_tol), comm=comm, phase_times=True)
    signs = np.ascontiguousarray(w.J, np.int8)
    G0 = torch.from_numpy(np.ascontiguousarray(w.G.T)).to(dev).t()  # column-major, resident
    Gw = torch.empty_like(G0.t()).t()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize(dev)
        if pg is not None:
            pg.barrier()

    for _ in range(max(3, args.warmup)):
        res = par.solve_device(G0, signs, cfg, out=Gw)
    barrier()
    times = []
    last = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between timed steps (not timed)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            last = par.solve_device(G0, signs, cfg, out=Gw)
            e1.record(stream)
            barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
    t_local = statistics.mean(times)
    if pg is not None:
        tt = torch.tensor([t_local])
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        t_max = float(tt[0])
    else:
        t_max = t_local
    stats = {k: getattr(last, k) for k, _ in P._lib.Result._fields_}
    # phase split (separate, untimed run with per-phase events)
    pt = par.solve_device(G0, signs, cfg_pt, out=Gw)
    phase = {"gram_ms": pt.t_gram_ms, "pivot_ms": pt.t_pivot_ms, "update_ms": pt.t_update_ms,
             "exchange_ms": pt.t_exchange_ms}
    total_f, gram_f, upd_f, piv_f = flops_of(stats, w, cx)
    if pg is not None:  # every rank counts its own pairs: sum
        ft = torch.tensor([total_f, gram_f, upd_f, piv_f], dtype=torch.float64)
        pg.all_reduce(ft)
        total_f, gram_f, upd_f, piv_f = [float(x) for x in ft]
    peak = measure_dgemm(torch, dev)
    gflops = total_f / t_max / 1e9
    steps_per_sweep = P.steps_per_sweep("round_robin", w.p)
    launches = args.steps * stats["sweeps"] * (1 + steps_per_sweep) * 3
    kern = {"gram": (pt.t_gram_ms, gram_f), "pivot": (pt.t_pivot_ms, piv_f), "update": (pt.t_update_ms, upd_f)}
    dom = max(kern, key=lambda k: kern[k][0])
    nl = stats["sweeps"] * (1 + steps_per_sweep)
    ach = kern[dom][1] / (kern[dom][0] * 1e-3) / 1e12 if kern[dom][0] > 0 else 0.0
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):  # DRAM bytes per launch of this kernel from the committed ncu capture
        traffic = json.load(open(tp)).get(w.name, {}).get(dom)
    roofline = {"kernel": dom, "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak if peak else None, "traffic": traffic,
                "per_launch": {"launches": nl, "avg_ms": kern[dom][0] / nl, "flops": kern[dom][1] / nl},
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 tensor/CUDA-core; "
                               "MEASURED_PEAKS.json has no FP64 entry)"}
    e2e = None
    if not args.no_e2e and world == 1:
        Gh = torch.from_numpy(np.ascontiguousarray(w.G.T)).pin_memory()  # pinned host, column-major
        Gh_np = Gh.numpy().T
        et = []
        for k in range(args.steps + 1):
            t0 = time.perf_counter()
            Gout, info = P.parallel_jacobi(Gh_np, signs, cfg)
            if k:
                et.append(time.perf_counter() - t0)
        e2e = {"value": statistics.mean(et), "unit": "s", "h2d_bytes_per_step": int(w.G.nbytes + w.n),
               "d2h_bytes_per_step": int(w.G.nbytes)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = max(1, min(os.cpu_count() or 1, w.p))
        t1, est, ratio = run_cpu_sample(w, threads)
        cpu = {"value": est if est else t1, "unit": "s", "cores": threads, "kind": "port",
               "sample": f"first outer sweep of {w.name} with the oracle (numpy+numba restatement pinned "
                         f"bit-exact to the reference), {threads} threads, {t1:.2f}s, extrapolated "
                         f"x{ratio:.2f} to the full solve (per-sweep profile measured in the build container)"
               if ratio else f"first outer sweep only ({t1:.2f}s)"}
    clocks = clk.summary()
    if rank == 0:
        line = {"metric": METRIC, "value": t_max, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": t_max * 1e3, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "c128" if cx else "f64",
                "data": "synthetic (seeded, BASELINE.json generators)",
                "config": {"workload": w.name, "m": w.m, "n": w.n, "b": w.b, "p": w.p,
                           "strategy": "round_robin", "orth_tol": "n*eps",
                           "l2": "flushed (256 MiB write) between timed steps",
                           "parallelism": f"ring p={w.p} over {world} GPU(s)"},
                "fp64_gflops": gflops, "fp64_frac_of_peak": gflops / (peak * 1e3) if peak else None,
                "fp64_peak_tflops_measured": peak, "fp64_peak_tflops_datasheet": FP64_DATASHEET_TFLOPS,
                "sweeps": stats["sweeps"], "converged": bool(stats["converged"]),
                "rotations": stats["rotations"], "phase_ms": phase,
                "exchange_ms_per_sweep": pt.t_exchange_ms / max(1, pt.sweeps),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "cluster_size": stats["cluster_size"], "gram_splits": stats["gram_splits"]}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
