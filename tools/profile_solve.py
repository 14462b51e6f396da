"""One solve of a BASELINE config (for ncu / launch lists).
    python tools/profile_solve.py cfg2 [--sweeps S] [--n N --b B]
--sweeps S runs only the first S outer sweeps (sweep_count; the inner cap stays 30)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1008_4166_b200 as P
from paper_1008_4166_b200 import workloads
ap = argparse.ArgumentParser()
ap.add_argument("config"); ap.add_argument("--sweeps", type=int, default=30)
ap.add_argument("--n", type=int); ap.add_argument("--b", type=int)
a = ap.parse_args()
kw = {k: v for k, v in (("n", a.n), ("b", a.b)) if v}
w = workloads.make(a.config, **kw)
cfg = P.SolverConfig(variant="2F", strategy="round_robin", p=w.p, tol=P.Tolerances(orth_tol=w.orth_tol),
                     sweep_count=0 if a.sweeps >= 30 else a.sweeps)
G, info = P.parallel_jacobi(w.G, w.J, cfg)
print(w.name, "sweeps", info.sweeps, "converged", info.converged, "t_total_ms", info.stats["t_total_ms"])
