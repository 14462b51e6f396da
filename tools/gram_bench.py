"""Time the Gram kernel alone on config-shaped batches and check it against
torch (fp64 X^H Y).  The tile shape / DFMA variant comes from the environment
(HJB_GRAM_CFG, HJB_GRAM_FFMA, HJB_GRAM_SPLITS), so run one process per variant:

    HJB_GRAM_CFG=2 python tools/gram_bench.py [--shapes cfg5r,cfg5c,...]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_1008_4166_b200 import _lib  # noqa: E402

SHAPES = {  # name: (complex, m, b, pairs per step)
    "cfg1": (False, 512, 32, 8),
    "cfg2": (True, 2048, 64, 16),
    "cfg3": (False, 4096, 64, 32),
    "cfg4": (True, 8192, 64, 64),
    "cfg5c": (True, 16384, 128, 64),
    "cfg5r": (False, 32768, 128, 128),
}
ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="cfg5r,cfg5c,cfg4,cfg3,cfg2")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dense", action="store_true", help="pre-pass shape: 2 x count single-block items")
a = ap.parse_args()
L = _lib.lib()
for name in a.shapes.split(","):
    cx, m, b, cnt = SHAPES[name]
    if cx and os.environ.get("HJB_GRAM_FFMA"):
        continue
    dt = torch.complex128 if cx else torch.float64
    g = torch.Generator(device="cuda").manual_seed(1)
    G = torch.randn(2 * b * cnt, m, dtype=dt, device="cuda", generator=g).t()  # column-major m x n
    if a.dense:
        items = np.array([[k * b, b, 0, 0] for k in range(2 * cnt)], np.int32)
    else:
        items = np.array([[2 * k * b, b, (2 * k + 1) * b, b] for k in range(cnt)], np.int32)
    n_it = len(items)
    A = torch.zeros(n_it * b * b, dtype=dt, device="cuda")
    D = torch.zeros(n_it * 2 * b, dtype=torch.float64, device="cuda")
    ts = []
    for r in range(a.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.hjb_gram(1 if cx else 0, m, G.data_ptr(), m, items.ctypes.data, n_it, b, A.data_ptr(),
                              D.data_ptr(), None))
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    # check a few items against torch
    err = 0.0
    derr = 0.0
    for k in sorted({0, n_it // 2, n_it - 1}):
        oi, ni, oj, nj = items[k]
        X = G[:, oi:oi + ni]
        Y = X if nj == 0 else G[:, oj:oj + nj]
        ref = X.conj().t() @ Y
        got = A[k * b * b:(k + 1) * b * b].reshape(b, b).t()[:ni, :Y.shape[1]]
        err = max(err, float((got - ref).abs().max() / ref.abs().max()))
        if nj:
            dref = torch.cat([(X.abs() ** 2).sum(0), (Y.abs() ** 2).sum(0)])
            dgot = D[k * 2 * b:(k + 1) * 2 * b]
            derr = max(derr, float(((dgot - dref).abs() / dref).max()))
    c = 4 if cx else 1
    fl = c * 2.0 * m * b * b * n_it
    print(json.dumps({"shape": name, "dense": a.dense, "variant": os.environ.get("HJB_GRAM_CFG", "0"),
                      "ffma": os.environ.get("HJB_GRAM_FFMA", "0"), "splits_forced": os.environ.get("HJB_GRAM_SPLITS", "auto"),
                      "ms": min(ts), "tflops": fl / min(ts) / 1e9, "rel_err": err, "norm_rel_err": derr}), flush=True)
    del G, A, D
