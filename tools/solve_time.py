"""One or more timed solves of a BASELINE config from device-resident G
(device time from the solver's CUDA events), for A/B runs under tuning
environment variables.
    python tools/solve_time.py cfg5r [--variant 2F] [--reps 1]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1008_4166_b200 as P
from paper_1008_4166_b200 import parallel as par, workloads
ap = argparse.ArgumentParser()
ap.add_argument("config"); ap.add_argument("--variant", default="2F"); ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--strategy", default="round_robin")
a = ap.parse_args()
w = workloads.make(a.config)
G0 = torch.from_numpy(np.ascontiguousarray(w.G.T)).cuda().t()
Gw = torch.empty_like(G0.t()).t()
signs = np.ascontiguousarray(w.J, np.int8)
cfg = P.SolverConfig(variant=a.variant, strategy=a.strategy, p=w.p, tol=P.Tolerances(orth_tol=w.orth_tol), phase_times=True)
for r in range(a.reps + (0 if w.n >= 16384 else 1)):
    res = par.solve_device(G0, signs, cfg, out=Gw)
    if r or w.n >= 16384:
        lam = (Gw.real ** 2 + Gw.imag ** 2).sum(0) if Gw.is_complex() else (Gw * Gw).sum(0)
        print(json.dumps({"workload": a.config, "variant": a.variant, "env": {k: v for k, v in os.environ.items() if k.startswith("HJB_")},
                          "sweeps": res.sweeps, "converged": bool(res.converged), "rotations": res.rotations,
                          "inner_sweeps": res.inner_sweeps, "t_total_ms": res.t_total_ms, "gram_ms": res.t_gram_ms,
                          "pivot_ms": res.t_pivot_ms, "update_ms": res.t_update_ms,
                          "lam_abs_sum": float(lam.sum())}), flush=True)
