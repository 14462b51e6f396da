"""Time the block-update kernel alone on a cfg-shaped batch (all items rotated).
    python tools/upd_bench.py [--cx] --m 32768 --b 128 --count 128"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1008_4166_b200 import _lib
ap = argparse.ArgumentParser()
ap.add_argument("--cx", action="store_true"); ap.add_argument("--m", type=int, default=32768)
ap.add_argument("--b", type=int, default=128); ap.add_argument("--count", type=int, default=128)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
L = _lib.lib()
m, b, cnt = a.m, a.b, a.count
dt = torch.complex128 if a.cx else torch.float64
G = torch.randn(2 * b * cnt, m, dtype=dt, device="cuda").t()  # column-major m x n
nmax = L.hjb_pivot_ld(b)
W = torch.randn(cnt * nmax * nmax, dtype=dt, device="cuda") * 0.05
st = torch.ones(cnt * 8, dtype=torch.int64, device="cuda")
items = np.array([[2 * k * b, b, (2 * k + 1) * b, b] for k in range(cnt)], np.int32)
ts = []
for r in range(a.reps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(L.hjb_update(1 if a.cx else 0, m, G.data_ptr(), m, items.ctypes.data, cnt, b, W.data_ptr(),
                            st.data_ptr(), None))
    e1.record(); torch.cuda.synchronize()
    if r: ts.append(e0.elapsed_time(e1))
c = 4 if a.cx else 1
fl = c * 2.0 * m * (2 * b) ** 2 * cnt
print(f"update {'c128' if a.cx else 'f64'} m={m} b={b} count={cnt}: {min(ts):.3f} ms  {fl / min(ts) / 1e9:.1f} TFLOP/s", flush=True)
