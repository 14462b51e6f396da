"""Time the pivot kernel on one realistic step batch (sweep-2 state of a
BASELINE config) for several cluster sizes, with per-CTA phase clocks.
    python tools/pivot_bench.py cfg2 [--n N --b B] [--clusters 4,8,16]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1008_4166_b200 as P
from paper_1008_4166_b200 import workloads, strategies, _lib
ap = argparse.ArgumentParser()
ap.add_argument("config"); ap.add_argument("--n", type=int); ap.add_argument("--b", type=int)
ap.add_argument("--clusters", default="4"); ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--threads", default="0")
ap.add_argument("--count", type=int, default=0, help="limit the number of pivots")
ap.add_argument("--dup", type=int, default=1, help="tile the pivot list (co-scheduling experiments)")
ap.add_argument("--sweep", type=int, default=1, help="sweeps run before the timed step")
a = ap.parse_args()
kw = {k: v for k, v in (("n", a.n), ("b", a.b)) if v}
w = workloads.make(a.config, **kw)
cx = np.iscomplexobj(w.G)
L = _lib.lib()
cfg = P.SolverConfig(variant="2F", strategy="round_robin", p=w.p, tol=P.Tolerances(orth_tol=w.orth_tol, max_sweeps=max(1, a.sweep)))
G1 = P.parallel_jacobi(w.G, w.J, cfg)[0] if a.sweep > 0 else np.asfortranarray(w.G)
Gd = torch.from_numpy(np.ascontiguousarray(G1.T)).cuda().t()
m, n, b = w.m, w.n, w.b
sd = torch.from_numpy(np.ascontiguousarray(w.J, np.int8)).cuda()
dt = 1 if cx else 0
nmax = L.hjb_pivot_ld(b)
def phase(items, cluster=0, prof=None, time_it=False):
    cnt = items.shape[0]
    A = torch.zeros(cnt * b * b, dtype=Gd.dtype, device="cuda")
    D = torch.zeros(cnt * 2 * b, dtype=torch.float64, device="cuda")
    _lib.check(L.hjb_gram(dt, m, Gd.data_ptr(), m, items.ctypes.data, cnt, b, A.data_ptr(), D.data_ptr(), None))
    W = torch.zeros(cnt * nmax * nmax, dtype=Gd.dtype, device="cuda")
    st = torch.zeros(cnt * 8, dtype=torch.int64, device="cuda")
    L.hjb_pivot_set_profile(prof.data_ptr() if prof is not None else None)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    _lib.check(L.hjb_pivot(dt, m, Gd.data_ptr(), m, items.ctypes.data, cnt, b, A.data_ptr(), D.data_ptr(), sd.data_ptr(),
                           w.orth_tol, -1.0, 30, W.data_ptr(), st.data_ptr(), None, cluster, None))
    e1.record(); torch.cuda.synchronize()
    L.hjb_pivot_set_profile(None)
    return W, st, e0.elapsed_time(e1)
# pre-pass of the next sweep so the blocks are orthogonal (parallel.py:138-148)
lay, _ = strategies.schedule_arrays("round_robin", w.p, a.sweep + 1)
steps = strategies.steps_per_sweep("round_robin", w.p)
first = lay[a.sweep * steps]
off = lambda k: (k - 1) * b
pre = np.array([[off(k), b, 0, 0] for pr in first for k in pr], np.int32)
W, st, _ = phase(pre)
_lib.check(L.hjb_update(dt, m, Gd.data_ptr(), m, pre.ctypes.data, pre.shape[0], b, W.data_ptr(), st.data_ptr(), None))
items = np.array([[off(i), b, off(j), b] for i, j in first], np.int32)
if a.dup > 1:
    items = np.ascontiguousarray(np.tile(items, (a.dup, 1)))
if a.count:
    items = np.ascontiguousarray(items[:a.count])
import itertools
for c, nt in itertools.product([int(x) for x in a.clusters.split(",")], [int(x) for x in a.threads.split(",")]):
    L.hjb_tune(nt, 0)
    prof = torch.zeros(2 * items.shape[0] * 16 * 8, dtype=torch.int64, device="cuda")
    ts = []
    for r in range(a.reps):
        Wt, stt, ms = phase(items, c, prof)
        ts.append(ms)
    nct = items.shape[0] * c
    allp = prof.cpu().numpy()
    pf = allp[:nct * 8].reshape(-1, 8)
    ph = allp[nct * 8: 2 * nct * 8].reshape(-1, 8)
    keep = pf[:, 3] > 0
    pf, ph = pf[keep], ph[keep]
    s = stt.cpu().numpy().reshape(-1, 8)
    print(f"{w.name} b={b} cluster={c} threads={nt}: {min(ts):.3f} ms  pivots={items.shape[0]} inner sweeps avg {s[:,3].mean():.2f} max {s[:,3].max()} "
          f"rounds max {pf[:,3].max()}  chol kcyc avg {pf[:,0].mean()/1e3:.1f} max {pf[:,0].max()/1e3:.1f}  "
          f"[Rij {pf[:,6].mean()/1e3:.1f} S {pf[:,7].mean()/1e3:.1f}] jacobi kcyc max {pf[:,1].max()/1e3:.1f}  cyc/round {pf[:,1].max()/max(1,pf[:,3].max()):.0f}  out kcyc {pf[:,2].max()/1e3:.1f}", flush=True)
    R = max(1, pf[:, 3].max())
    names = ["dot+push", "mbar wait", "sum", "rot+apply", "ring", "recv", "blkxchg", "gramchk"]
    print("   per-round cycles (thread 0):", "  ".join(f"{nm} {ph[:, i].mean()/R:.0f}" for i, nm in enumerate(names)), flush=True)
