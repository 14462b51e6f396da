import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1008_4166_b200 import _lib
L = _lib.lib()
for dt, name in ((0, "f64"), (1, "c128")):
    for b in (32, 64, 128):
        for c in (1, 2, 4, 8, 16):
            for nt in (256, 512):
                r = L.hjb_pivot_occupancy(dt, b, c, nt)
                if r > 0:
                    print(f"{name} b={b} C={c} NT={nt}: max active clusters {r} ({r*c} CTAs)")
