import time, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1008_4166_b200 as P
from paper_1008_4166_b200 import workloads
import torch
for name in ["cfg1", "cfg2", "cfg3"]:
    w = workloads.make(name)
    cfg = P.SolverConfig(variant="2F", strategy="round_robin", p=w.p, tol=P.Tolerances(orth_tol=w.orth_tol), phase_times=True)
    t = time.perf_counter(); Gout, info = P.parallel_jacobi(w.G, w.J, cfg); dt = time.perf_counter() - t
    s = info.stats
    print(name, "wall %.3fs dev %.1fms sweeps %d conv %s rot %d gram %.1f pivot %.1f update %.1f cluster %d splits %d inner_sweeps %d" % (dt, s["t_total_ms"], info.sweeps, info.converged, info.rotations, s["t_gram_ms"], s["t_pivot_ms"], s["t_update_ms"], s["cluster_size"], s["gram_splits"], s["inner_sweeps"]), flush=True)
    if name == "cfg2":
        np.save("gpurun_out/cfg2_lam_gpu.npy", w.J * (np.abs(Gout)**2).sum(0))
a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda"); b = torch.randn_like(a)
for _ in range(2): c = a @ b
torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(5): c = a @ b
e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/5
print("cuBLAS DGEMM 8192^3: %.2f TFLOP/s" % (2*8192**3/ms/1e9))
