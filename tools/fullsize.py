"""Full-size single-solve timing + size-independent checks (cfg3/cfg4/cfg5).

    python tools/fullsize.py cfg5c [--phases] [--kappa]

One eigensolve of the BASELINE.json configuration at its full size on one
GPU (G resident in HBM, timed with CUDA events on the solve stream), then
checks that need no CPU oracle (SURVEY.md 8(d) "cfg5 oracle"):

* converged, sweep count;
* residual max_i ||H u_i - lam_i u_i|| / (||H|| ||u_i||) over 256 sampled
  columns, H u = G0 (J (G0^H u)) formed on the GPU, ||H|| = max |lam|;
* J-orthogonality loss off(G_out) = max_{i != j} |g_i^H g_j| / (||g_i|| ||g_j||)
  for the sampled columns against all columns, and the reference's
  max |U^H U - I| over all columns (hjb_orthogonality);
* cfg4: eigenvalues against the prescribed spectrum, bound 64 n eps kappa(G_s)
  with kappa from the scaled Gram (--kappa, GPU eigvalsh).

Prints one JSON line.  Not a bench line (one timed solve, one warm-up on a
small instance) -- DESIGN.md section 8 quotes these numbers.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

EPS = float(np.finfo(np.float64).eps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--phases", action="store_true")
    ap.add_argument("--kappa", action="store_true")
    ap.add_argument("--samples", type=int, default=256)
    args = ap.parse_args()

    import torch
    import paper_1008_4166_b200 as P
    from paper_1008_4166_b200 import parallel as par, workloads

    t0 = time.perf_counter()
    w = workloads.make(args.config, **({"n": args.n} if args.n else {}))
    t_gen = time.perf_counter() - t0
    dev = torch.device("cuda", 0)
    cx = np.iscomplexobj(w.G)
    signs = np.ascontiguousarray(w.J, np.int8)
    cfg = P.SolverConfig(variant="2F", strategy="round_robin", p=w.p, tol=P.Tolerances(orth_tol=w.orth_tol))

    # warm the library/driver on a small instance of the same dtype and b
    ws = workloads.make(args.config, n=4 * w.b)
    Gs = torch.from_numpy(np.ascontiguousarray(ws.G.T)).to(dev).t()
    par.solve_device(Gs, np.ascontiguousarray(ws.J, np.int8),
                     P.SolverConfig(variant="2F", strategy="round_robin", p=ws.p,
                                    tol=P.Tolerances(orth_tol=ws.orth_tol)), out=torch.empty_like(Gs.t()).t())
    del Gs

    G0 = torch.from_numpy(np.ascontiguousarray(w.G.T)).to(dev).t()
    lam_ref = getattr(w, "lam", None)
    m, n = w.m, w.n
    del w.G
    Gw = torch.empty_like(G0.t()).t()
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    res = par.solve_device(G0, signs, cfg, out=Gw)
    e1.record(stream)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    stats = {k: getattr(res, k) for k, _ in P._lib.Result._fields_}
    flops = workloads.algorithmic_flops(m, w.b, cx, stats["pairs_updated"], stats["pairs_visited"],
                                        stats["prepass_updated"], stats["prepass_visited"])
    out = {"workload": args.config, "m": m, "n": n, "b": w.b, "p": w.p, "dtype": "c128" if cx else "f64",
           "time_to_eigensolve_s": t, "fp64_gflops": flops / t / 1e9, "sweeps": res.sweeps,
           "converged": bool(res.converged), "rotations": res.rotations, "gen_s": t_gen,
           "pairs_updated": stats["pairs_updated"], "pairs_visited": stats["pairs_visited"],
           "cluster_size": stats["cluster_size"], "gram_splits": stats["gram_splits"]}

    print(json.dumps(out), file=sys.stderr, flush=True)  # survives a failing check
    # size-independent checks on the GPU
    Jd = torch.from_numpy(signs.astype(np.float64)).to(dev)
    nrm2 = (Gw.real ** 2 + Gw.imag ** 2).sum(0) if cx else (Gw ** 2).sum(0)
    lam = Jd * nrm2
    hn = float(lam.abs().max())
    g = torch.Generator().manual_seed(0)
    idx = torch.randperm(n, generator=g)[: args.samples].to(dev)
    U = Gw[:, idx] / nrm2[idx].sqrt()
    HU = G0 @ (Jd[:, None] * (G0.conj().t() @ U) if cx else Jd[:, None] * (G0.t() @ U))
    R = HU - U * lam[idx]
    out["residual_sampled"] = float((R.abs().pow(2).sum(0).sqrt() / (hn * U.abs().pow(2).sum(0).sqrt())).max())
    out["residual_bound"] = 64 * n * EPS
    Un = Gw / nrm2.sqrt()
    C = (Un[:, idx].conj().t() @ Un).abs() if cx else (Un[:, idx].t() @ Un).abs()
    C[torch.arange(len(idx), device=dev), idx] = 0
    out["orth_loss_sampled"] = float(C.max())
    out["orth_bound"] = 64 * n * EPS
    # the reference's metric over ALL columns (solve.py:108-110) on the GPU
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out["orthogonality_full"] = P.orthogonality(Un)
    out["orthogonality_full_s"] = time.perf_counter() - t0
    del C, Un, HU, R, U
    if lam_ref is not None:
        ls = np.sort(lam.cpu().numpy())
        rel = np.abs(ls - lam_ref) / np.abs(lam_ref)
        out["eig_rel_err_max"] = float(rel.max())
        if args.kappa:
            A = G0.conj().t() @ G0 if cx else G0.t() @ G0
            s = A.diagonal().real.rsqrt()
            As = A * s[:, None] * s[None, :]
            ev = torch.linalg.eigvalsh((As + As.conj().t()) / 2)
            kappa = math.sqrt(float(ev[-1] / ev[0]))
            out["kappa_Gs"] = kappa
            out["eig_bound"] = 64 * n * EPS * kappa
            out["eig_ok"] = bool(np.all(np.abs(ls - lam_ref) <= 64 * n * EPS * kappa * np.abs(lam_ref)))
            del A, As
    if args.phases:
        cfg_pt = P.SolverConfig(variant="2F", strategy="round_robin", p=w.p,
                                tol=cfg.tol, phase_times=True)
        pt = par.solve_device(G0, signs, cfg_pt, out=Gw)
        out["phase_ms"] = {"gram_ms": pt.t_gram_ms, "pivot_ms": pt.t_pivot_ms, "update_ms": pt.t_update_ms}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
