"""Inner-level micro-benchmark: hjb_pivot (prologue -> Jacobi -> epilogue,
or the round-1 single kernel with HJB_PIVOT_V1=1) on a batch of block pairs
shaped like one step of a BASELINE config (p pairs of b-column blocks with
internally orthogonal columns, as after the F pre-pass).

    python tools/jac_bench.py cfg2 [cfg5r ...] [--reps 5]

With a profiling build (HJB_NVCC_FLAGS=-DHJB_JAC_PROF=1, loaded through
HJB_LIB) it also prints the Jacobi kernel's per-warp phase clocks.
"""

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {"cfg1": (32, False, 8, 512), "cfg2": (64, True, 16, 2048), "cfg3": (64, False, 32, 4096),
          "cfg4": (64, True, 64, 8192), "cfg5r": (128, False, 128, 32768), "cfg5c": (128, True, 64, 16384)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--m", type=int, default=0, help="rows (default 4b: the pivot does not depend on m)")
    args = ap.parse_args()
    import torch
    import paper_1008_4166_b200 as P
    L = P._lib.lib()
    for name in args.configs:
        b, cx, count, n_full = SHAPES[name]
        m = args.m or 4 * b
        rng = np.random.default_rng(1)
        blocks = []
        for _ in range(2 * count):
            X = rng.standard_normal((m, b)) + (1j * rng.standard_normal((m, b)) if cx else 0)
            Q, _ = np.linalg.qr(X)
            blocks.append(Q * rng.uniform(0.5, 3.0, b)[None, :])
        G = np.asfortranarray(np.concatenate(blocks, axis=1))
        J = np.array(([1] * (b // 2) + [-1] * (b - b // 2)) * (2 * count), np.int8)
        Gd = torch.from_numpy(np.ascontiguousarray(G.T)).cuda().t()
        items = np.ascontiguousarray(np.array([[2 * q * b, b, (2 * q + 1) * b, b] for q in range(count)], np.int32))
        nmax = L.hjb_pivot_ld(b)
        dt = Gd.dtype
        A = torch.zeros(count * b * b, dtype=dt, device="cuda")
        D = torch.zeros(count * 2 * b, dtype=torch.float64, device="cuda")
        W = torch.zeros(count * nmax * nmax, dtype=dt, device="cuda")
        stats = torch.zeros(count * 8, dtype=torch.int64, device="cuda")
        sd = torch.from_numpy(J).cuda()
        desc = np.zeros(5, np.int32)
        P._lib.check(L.hjb_inner_order(1 if cx else 0, b, count, 0, desc.ctypes.data))
        prof = None
        if desc[0] == 2:
            prof = torch.zeros(count * desc[2] * desc[3] * 8, dtype=torch.int64, device="cuda")
            L.hjb_pivot_set_profile(prof.data_ptr())
        st = torch.cuda.current_stream().cuda_stream
        times = []
        for r in range(args.reps + 1):
            P._lib.check(L.hjb_gram(1 if cx else 0, m, Gd.data_ptr(), m, items.ctypes.data, count, b, A.data_ptr(),
                                    D.data_ptr(), st))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P._lib.check(L.hjb_pivot(1 if cx else 0, m, Gd.data_ptr(), m, items.ctypes.data, count, b, A.data_ptr(),
                                     D.data_ptr(), sd.data_ptr(), n_full * 2.220446049250313e-16, -1.0, 30,
                                     W.data_ptr(), stats.data_ptr(), None, 0, st))
            e1.record()
            torch.cuda.synchronize()
            if r:
                times.append(e0.elapsed_time(e1))
        L.hjb_pivot_set_profile(None)
        s = stats.cpu().numpy().reshape(count, 8)
        out = {"config": name, "b": b, "count": count, "order": desc.tolist(), "ms": float(np.median(times)),
               "inner_sweeps_avg": float(s[:, 3].mean()), "inner_sweeps_max": int(s[:, 3].max()),
               "rotations": int(s[:, 0].sum()), "status": int(s[:, 4].max())}
        if prof is not None and int(prof.abs().sum()) > 0:
            pf = prof.cpu().numpy().reshape(-1, 8).astype(float)
            rounds = pf[:, 6].mean()
            names = ["round", "empty_wait", "send", "full_wait", "recv", "sweep_end", "rounds", "total"]
            out["clocks_per_warp_mean"] = {k: float(pf[:, i].mean()) for i, k in enumerate(names)}
            out["cycles_per_round"] = {k: float(pf[:, i].mean() / max(rounds, 1)) for i, k in enumerate(names) if i != 6}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
