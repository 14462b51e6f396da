"""Variants (F / B) x outer orderings (modulus / round-robin) under timing
(strategies.py:58-92, parallel.py:150-174): one
warm-up solve then 3 timed solves each, device time from the solver's own
CUDA events (hjb_result.t_total_ms).

    python tools/strategy_time.py [cfg1 cfg2 cfg3] > gpurun_out/strategy_time.jsonl
"""
import json
import sys

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_1008_4166_b200 as P  # noqa: E402
from paper_1008_4166_b200 import workloads  # noqa: E402

for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]:
    w = workloads.make(name)
    for variant, strat in [("2F", "round_robin"), ("2F", "modulus"), ("2B", "round_robin"), ("2B", "modulus")]:
        cfg = P.SolverConfig(variant=variant, strategy=strat, p=w.p, tol=P.Tolerances(orth_tol=w.orth_tol))
        P.parallel_jacobi(w.G, w.J, cfg)  # warm-up
        ts, lam = [], None
        for _ in range(3):
            Gout, info = P.parallel_jacobi(w.G, w.J, cfg)
            ts.append(info.stats["t_total_ms"])
        lam = np.sort(w.J * (np.abs(Gout) ** 2).sum(0))
        print(json.dumps({"workload": name, "variant": variant, "strategy": strat, "steps_per_sweep": P.steps_per_sweep(strat, w.p),
                          "sweeps": info.sweeps, "converged": bool(info.converged), "rotations": info.rotations,
                          "device_ms": ts, "device_ms_min": min(ts),
                          "lam_sum": float(lam.sum()), "lam_min": float(lam[0]), "lam_max": float(lam[-1])}),
              flush=True)
