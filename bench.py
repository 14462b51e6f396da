"""Benchmark of the B200 2F block J-Jacobi hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg5r] [--no-cpu-baseline] [--no-e2e]

Metric: time-to-eigensolve (s, lower is better) with FP64 GFLOP/s and its
fraction of peak.  The default workload is the n = 32768 real config of
BASELINE.json's scaling line (``cfg5r``: float64 32768 x 32768, seed 5, J
half/half, b = 128, p = 128 ring workers, round-robin, orth_tol = n eps) --
the configuration the metric's 1/2/4/8-GPU series and the north-star target
are quoted on; it fits one B200 (8 GiB).

Steps.  For cfg4/cfg5 one step is ONE OUTER SWEEP of the solve (a whole
solve takes 15-20 sweeps): the timed region runs K consecutive sweeps,
starting a fresh solve from the resident input (device copy included) at the
first timed step and again whenever a solve converges.  ``value`` is the
device time of the first COMPLETE solve inside the timed region (the sum of
its sweep steps); ``ms_per_step`` is the mean step (sweep) time.  If K is
smaller than the solve's sweep count, the solve is finished after the timed
region (same timing) and the line says so.  For cfg1-cfg3 one step is one
whole solve.  N > 1 (torchrun, one process per GPU) splits the ring workers
over the GPUs with NCCL block exchange (strong scaling).

``--impl reference`` times the reference's CPU algorithm (the oracle: a
restatement pinned bit-exact to the reference, run as the reference runs it,
p worker threads coupled through ring channels) on the host cores.
"""

from __future__ import annotations

import os

# The reference pins BLAS to one thread per ring worker; this
# must be in the environment BEFORE numpy loads OpenBLAS, or the p worker
# threads of the CPU baseline oversubscribe the cores (measured: cfg1 7.0 s
# instead of 1.8 s).
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse
import json
import platform
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
SWEEP_STEP_CONFIGS = ("cfg4", "cfg5r", "cfg5c")
EPS = float(np.finfo(np.float64).eps)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5r")
    ap.add_argument("--variant", default="2F", choices=["2F", "3F", "2B", "3B"],
                    help="ring variant (parallel.py:43); the metric's line is 2F")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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


STAT_KEYS = ("pairs_visited", "pairs_updated", "prepass_visited", "prepass_updated", "rotations",
             "big_rotations", "inner_sweeps", "inner_pair_visits", "fallbacks")


def add_stats(acc, res):
    for k in STAT_KEYS:
        acc[k] = acc.get(k, 0) + getattr(res, k)
    for k in ("t_gram_ms", "t_pivot_ms", "t_update_ms", "t_exchange_ms"):
        acc[k] = acc.get(k, 0.0) + getattr(res, k)
    acc["exchange_bytes"] = acc.get("exchange_bytes", 0) + res.exchange_bytes
    acc["cluster_size"], acc["gram_splits"] = res.cluster_size, res.gram_splits
    return acc


def flops_of(stats, w, cx, variant="2F"):
    """SURVEY.md 8(d) algorithmic FLOPs (Gram + update, the headline) and
    the inner-level (pivot) flops reported separately.  B variants: three Gram
    products per pair (A_ii, A_jj, A_ij of the dense pair Gram), no pre-pass."""
    from paper_1008_4166_b200 import workloads
    b = w.b
    c = 4.0 if cx else 1.0
    gpp = 3.0 if variant.endswith("B") else 1.0
    gram = c * 2.0 * w.m * b * b * (gpp * stats["pairs_visited"] + stats["prepass_visited"])
    upd = c * (8.0 * w.m * b * b * stats["pairs_updated"] + 2.0 * w.m * b * b * stats["prepass_updated"])
    total = workloads.algorithmic_flops(w.m, b, cx, stats["pairs_updated"], stats["pairs_visited"],
                                        stats["prepass_updated"], stats["prepass_visited"])
    total += c * 2.0 * w.m * b * b * (gpp - 1.0) * stats["pairs_visited"]
    # inner level: a dot product (2N real flops, x4 complex) per examined 2x2
    # pivot and 6N (x4 complex) per applied rotation on R (W is formed once)
    N = 2 * b
    piv = c * (2.0 * N * stats["inner_pair_visits"] + 6.0 * N * stats["rotations"])
    return total, gram, upd, piv


# ----------------------------------------------------------------- reference arm

def cpu_profile():
    p = os.path.join(ROOT, "oracle", "cpu_profile.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def cpu_sample(w, full):
    """The reference's algorithm on the host (oracle restatement pinned
    bit-exact to the reference).  full=True: one whole solve, run as the
    reference runs it (p worker threads on ring channels).  full=False: a
    bounded sample extrapolated to the whole solve, labelled an ESTIMATE:
    cfg2 / cfg3 -- the first outer sweep, times the whole-solve / first-sweep
    ratio of the reference algorithm measured in the build container
    (oracle/cpu_profile.json, cfg2: 59.0 s / 8.9 s over 14 sweeps, scaled by
    the sweep count for cfg3); cfg4 / cfg5 -- the first F pre-pass and the
    first ring step of sweep 1 (p pairs, p threads), times the cost profile of
    the same-generator proxy (SURVEY.md 8(d) item iv)."""
    import oracle
    threads = w.p
    oracle.parallel_jacobi_2f(w.G[:128, :128], w.J[:128], 2, "round_robin", orth_tol=w.orth_tol)  # JIT warm
    prof = cpu_profile()
    t0 = time.perf_counter()
    if full:
        _, info = oracle.parallel_jacobi_2f(w.G, w.J, w.p, "round_robin", orth_tol=w.orth_tol, threads="ring")
        t = time.perf_counter() - t0
        return t, t, f"one whole {w.name} solve ({info.sweeps} sweeps), p={w.p} ring worker threads"
    if w.name in ("cfg2", "cfg3"):
        _, info = oracle.parallel_jacobi_2f(w.G, w.J, w.p, "round_robin", orth_tol=w.orth_tol, threads=threads,
                                            sweep_limit=1)
        t = time.perf_counter() - t0
        c2 = prof.get("cfg2", {})
        ratio = c2.get("t_total", 59.0) / c2.get("t_sweep1", 8.86)
        sweeps_ref = {"cfg2": 14, "cfg3": 15}[w.name]
        factor = ratio * sweeps_ref / 14.0
        return t, t * factor, (f"first outer sweep of {w.name} ({threads} threads), {t:.2f} s; whole-solve ESTIMATE "
                               f"x{factor:.2f} (whole/first-sweep ratio of the cfg2 reference run, "
                               f"{sweeps_ref} sweeps)")
    _, info = oracle.parallel_jacobi_2f(w.G, w.J, w.p, "round_robin", orth_tol=w.orth_tol, threads=threads,
                                        sweep_limit=1, step_limit=1)
    t = time.perf_counter() - t0
    ex = prof.get(w.name + "_extrapolation", {})
    factor = ex.get("factor")
    est = t * factor if factor else None
    desc = (f"F pre-pass + first ring step of sweep 1 of {w.name} ({w.p} pairs, {threads} threads), "
            f"{t:.2f} s; whole-solve ESTIMATE x{factor:.0f} ({ex.get('how', '')})" if factor else
            f"F pre-pass + first ring step of sweep 1 ({t:.2f} s), no extrapolation profile")
    return t, est, desc


def reference_arm(args, w):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    full = w.name == "cfg1"   # the others: bounded samples (cpu_sample), so K steps end within minutes
    cores = os.cpu_count() or 1
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_sample(w, full)
    samples, ests = [], []
    desc = ""
    for _ in range(args.steps):
        t, est, desc = cpu_sample(w, full)
        samples.append(t)
        ests.append(est if est else t)
    v = statistics.mean(ests)
    ms = statistics.mean(samples) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128" if np.iscomplexobj(w.G) else "f64",
            "data": "synthetic (seeded, BASELINE.json generators)",
            "config": {"workload": w.name, "n": w.n, "b": w.b, "p": w.p, "strategy": "round_robin",
                       "orth_tol": "n*eps", "step": "whole solve" if full else "bounded sample (see cpu_baseline)"},
            "cpu_baseline": {"value": v, "unit": "s", "cores": min(cores, w.p), "kind": "port",
                             "sample": desc, "cpu_model": cpu_model(), "nproc": cores,
                             "extrapolated": not full},
            "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- parity of the bench's own solve

def parity_check(torch, w, Gout, sweeps, P):
    """Size-independent checks of the solve the bench timed (outside the
    timed region): the reference's golden eigenvalues where one exists
    (cfg1-cfg3 at full size), else residual on sampled columns and the full
    column orthogonality (SURVEY.md 8(d) cfg5 items ii/iii)."""
    out = {}
    n = w.n
    res = P.extract_eigen(Gout, w.J)
    lam, U = res.eigenvalues, res.eigenvectors
    out["orthogonality"] = P.orthogonality(U)
    out["orth_bound"] = 64 * n * EPS
    # residual on 256 sampled columns: H u = G0 (J (G0^H u)), ||H||_2 = max|lam|
    idx = torch.from_numpy(np.random.default_rng(0).choice(n, min(n, 256), replace=False)).to(U.device)
    G0 = torch.from_numpy(np.ascontiguousarray(w.G.T)).to(U.device).t()
    Jd = torch.from_numpy(w.J.astype(np.float64)).to(U.device)
    Us = U[:, idx]
    HU = G0 @ (Jd[:, None].to(G0.dtype) * (G0.conj().T @ Us))
    R = HU - Us * lam[idx].to(Us.dtype)[None, :]
    out["residual"] = float((torch.linalg.vector_norm(R, dim=0)
                             / (lam.abs().max() * torch.linalg.vector_norm(Us, dim=0))).max())
    out["residual_bound"] = 64 * n * EPS
    ok = out["orthogonality"] <= out["orth_bound"] and out["residual"] <= out["residual_bound"]
    key = f"{w.name}_n{w.n}_b{w.b}"
    gp = os.path.join(ROOT, "tests", "golden", f"fullsize_{key}.npz")
    if os.path.exists(gp):
        z = np.load(gp)
        info = z[key + "_info"]
        ref = np.sort(z[key + "_lam"])
        kappa = float(info[6])
        got = np.sort(lam.cpu().numpy())
        rel = np.abs(got - ref) / np.abs(ref)
        out.update(max_rel_eig_vs_reference=float(rel.max()), eig_bound=64 * n * EPS * kappa,
                   sweeps_reference=int(info[0]))
        ok = ok and rel.max() <= 64 * n * EPS * kappa and abs(sweeps - int(info[0])) <= 1
    del G0
    out["status"] = "pass" if ok else "fail"
    return out


# ----------------------------------------------------------------- our arm

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
    sweep_mode = w.name in SWEEP_STEP_CONFIGS
    tol = P.Tolerances(orth_tol=w.orth_tol)
    cfg_solve = P.SolverConfig(variant=args.variant, strategy="round_robin", p=w.p, tol=tol, comm=comm)
    signs = np.ascontiguousarray(w.J, np.int8)
    G0 = torch.from_numpy(np.ascontiguousarray(w.G.T)).to(dev).t()  # column-major, resident
    Gw = torch.empty_like(G0.t()).t()
    big = G0.numel() * G0.element_size() > 2 * 126 * 2 ** 20
    flush = None if big else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    max_sw = tol.max_sweeps

    def barrier():
        torch.cuda.synchronize(dev)
        if pg is not None:
            pg.barrier()

    state = {"k": 1}

    def sweep_step():
        """One outer sweep of the running solve; returns its result."""
        if state["k"] == 1:
            Gw.copy_(G0)
        cfg = P.SolverConfig(variant=args.variant, strategy="round_robin", p=w.p, tol=tol, comm=comm,
                             phase_times=True, first_sweep=state["k"], sweep_count=1)
        r = par.solve_device(Gw, signs, cfg, out=Gw)
        done = bool(r.converged) or state["k"] >= max_sw
        state["k"] = 1 if done else state["k"] + 1
        return r, done

    def solve_step():
        return par.solve_device(G0, signs, cfg_solve, out=Gw), True

    step_fn = sweep_step if sweep_mode else solve_step
    for _ in range(max(3, args.warmup)):
        step_fn()
    state["k"] = 1
    barrier()
    times, results, done_flags = [], [], []
    Gsave = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            if flush is not None:
                flush.zero_()  # L2 flush between timed steps (not timed)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r, done = step_fn()
            e1.record(stream)
            barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
            results.append(r)
            done_flags.append(done)
            if sweep_mode and done and Gsave is None:  # keep the first complete solve for the parity check
                Gsave = Gw.clone()
    clocks = clk.summary()
    # per-step max over ranks
    if pg is not None:
        tt = torch.tensor(times, dtype=torch.float64)
        pg.all_reduce(tt, op=pg.ReduceOp.MAX)
        times = [float(x) for x in tt]
    # the first complete solve inside the timed region
    solve_t, solve_res, finished_inside = 0.0, [], True
    for t, r, d in zip(times, results, done_flags):
        solve_t += t
        solve_res.append(r)
        if d:
            break
    else:
        finished_inside = False
        while True:  # finish it after the timed region (same per-step timing)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r, d = step_fn()
            e1.record(stream)
            barrier()
            t = e0.elapsed_time(e1) / 1e3
            if pg is not None:
                tt = torch.tensor([t], dtype=torch.float64)
                pg.all_reduce(tt, op=pg.ReduceOp.MAX)
                t = float(tt[0])
            solve_t += t
            solve_res.append(r)
            if d:
                break
    last = solve_res[-1]
    sweeps = last.sweeps
    stats = {}
    for r in solve_res:
        add_stats(stats, r)
    if not sweep_mode:
        # phase split from a separate untimed run with per-phase events
        pt = par.solve_device(G0, signs, P.SolverConfig(variant=args.variant, strategy="round_robin", p=w.p,
                                                        tol=tol, comm=comm, phase_times=True), out=Gw)
        stats = add_stats({}, pt)
    elif Gsave is not None:
        Gw.copy_(Gsave)
        del Gsave
    phase = {"gram_ms": stats["t_gram_ms"], "pivot_ms": stats["t_pivot_ms"], "update_ms": stats["t_update_ms"],
             "exchange_ms": stats["t_exchange_ms"]}
    total_f, gram_f, upd_f, piv_f = flops_of(stats, w, cx, args.variant)
    if pg is not None:  # every rank counts its own pairs: sum
        ft = torch.tensor([total_f, gram_f, upd_f, piv_f], dtype=torch.float64)
        pg.all_reduce(ft)
        total_f, gram_f, upd_f, piv_f = [float(x) for x in ft]
    parity = None
    if rank == 0 and not args.no_parity:
        parity = parity_check(torch, w, Gw, sweeps, P)
    peak = measure_dgemm(torch, dev)
    gflops = total_f / solve_t / 1e9
    steps_per_sweep = P.steps_per_sweep("round_robin", w.p)
    # kernels this library launched inside the timed region (hjb_result.kernel_launches)
    launches = int(sum(r.kernel_launches for r in results))
    nl = sweeps * (1 + steps_per_sweep)  # launches of each phase per solve
    kern = {"gram": (phase["gram_ms"], gram_f, "tensor"), "pivot": (phase["pivot_ms"], piv_f, "latency"),
            "update": (phase["update_ms"], upd_f, "tensor")}
    fracs = {}
    for k, (ms, fl, _) in kern.items():
        a = fl / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
        fracs[k] = {"ms": ms, "tflops": a, "frac_of_dgemm": a / peak if peak else None}
    dom = max(kern, key=lambda k: kern[k][0])
    ach = fracs[dom]["tflops"]
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):  # DRAM bytes per launch of this kernel from the committed ncu capture
        traffic = json.load(open(tp)).get(w.name, {}).get(dom)
    roofline = {"kernel": dom, "bound": kern[dom][2], "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak if peak else None, "traffic": traffic,
                "per_launch": {"launches": nl, "avg_ms": kern[dom][0] / nl, "flops": kern[dom][1] / nl},
                "peak_source": "cuBLAS DGEMM 8192^3 measured in this run (FP64 tensor/CUDA-core; "
                               "MEASURED_PEAKS.json has no FP64 entry)",
                "kernels": fracs}
    e2e = None
    if not args.no_e2e and world == 1:
        Gh = torch.from_numpy(np.ascontiguousarray(w.G.T)).pin_memory()  # pinned host, column-major
        Gh_np = Gh.numpy().T
        et = []
        if sweep_mode:  # warm the page-locked result allocator (cfg1-3 do it with their untimed first solve)
            from paper_1008_4166_b200 import _device
            _warm = _device.pinned_host_colmajor(w.m, w.n, w.G.dtype)
            del _warm
        reps = 1 if sweep_mode else args.steps + 1
        for k in range(reps):
            t0 = time.perf_counter()
            Gout, info = P.parallel_jacobi(Gh_np, signs, cfg_solve)
            if k or sweep_mode:
                et.append(time.perf_counter() - t0)
            del Gout
        e2e = {"value": statistics.mean(et), "unit": "s", "h2d_bytes_per_step": int(w.G.nbytes + w.n),
               "d2h_bytes_per_step": int(w.G.nbytes),
               "note": "one whole solve through parallel_jacobi from pinned host G (H2D + D2H inside)"}
        del Gh
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
        t, est, desc = cpu_sample(w, full=w.name == "cfg1")
        cpu = {"value": est if est else t, "unit": "s", "cores": min(os.cpu_count() or 1, w.p), "kind": "port",
               "sample": desc, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
               "extrapolated": w.name != "cfg1"}
    if rank == 0:
        step_desc = ("one outer sweep of the solve (value = first complete solve in the timed region"
                     + ("" if finished_inside else ", finished after the timed region") + ")") \
            if sweep_mode else "one whole solve"
        line = {"metric": METRIC, "value": solve_t, "unit": "s", "n_gpus": world, "steps": args.steps,
                "warmup": max(3, args.warmup), "ms_per_step": statistics.mean(times) * 1e3,
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
                "dtype": "c128" if cx else "f64", "data": "synthetic (seeded, BASELINE.json generators)",
                "config": {"workload": w.name, "m": w.m, "n": w.n, "b": w.b, "p": w.p,
                           "variant": args.variant, "strategy": "round_robin", "orth_tol": "n*eps", "step": step_desc,
                           "l2": ("inputs larger than L2 (no flush)" if flush is None
                                  else "flushed (256 MiB write) between timed steps"),
                           "parallelism": f"ring p={w.p} over {world} GPU(s)"},
                "fp64_gflops": gflops, "fp64_frac_of_peak": gflops / (peak * 1e3) if peak else None,
                "fp64_peak_tflops_measured": peak, "fp64_peak_tflops_datasheet": FP64_DATASHEET_TFLOPS,
                "sweeps": sweeps, "converged": bool(last.converged), "rotations": stats["rotations"],
                "phase_ms": phase, "exchange_ms_per_sweep": phase["exchange_ms"] / max(1, sweeps),
                "exchange_bytes_per_sweep": stats.get("exchange_bytes", 0) / max(1, sweeps),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "parity": parity, "cluster_size": stats["cluster_size"],
                "gram_splits": stats["gram_splits"]}
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
