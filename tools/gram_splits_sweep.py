"""cfg2/cfg3 solve with the Gram split-K capped by HJB_GRAM_SPLITS_MAX (set by
the caller); prints device and phase times.  Experiment helper."""
import json
import os
import sys

sys.path.insert(0, "/root/repo")
import paper_1008_4166_b200 as P  # noqa: E402
from paper_1008_4166_b200 import workloads  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    w = workloads.make(name)
    cfg = P.SolverConfig(variant="2F", strategy="round_robin", p=w.p, tol=P.Tolerances(orth_tol=w.orth_tol),
                         phase_times=True)
    P.parallel_jacobi(w.G, w.J, cfg)
    cfg2 = P.SolverConfig(variant="2F", strategy="round_robin", p=w.p, tol=P.Tolerances(orth_tol=w.orth_tol))
    ts = []
    for _ in range(3):
        _, info = P.parallel_jacobi(w.G, w.J, cfg2)
        ts.append(info.stats["t_total_ms"])
    _, ip = P.parallel_jacobi(w.G, w.J, cfg)
    s = ip.stats
    print(json.dumps({"workload": name, "splits_max": os.environ.get("HJB_GRAM_SPLITS_MAX", "16"),
                      "splits": s["gram_splits"], "sweeps": info.sweeps, "device_ms_min": min(ts),
                      "gram_ms": s["t_gram_ms"], "pivot_ms": s["t_pivot_ms"], "update_ms": s["t_update_ms"]}),
          flush=True)
