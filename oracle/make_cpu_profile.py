"""Cost profile of the reference algorithm on the build container's CPU, used
by bench.py to extrapolate bounded CPU-baseline samples (cpu_sample) to a
whole solve.  TEST/BENCH INFRASTRUCTURE (oracle/): not part of the product.

    OPENBLAS_NUM_THREADS=1 NUMBA_CACHE_DIR=/tmp/nc python oracle/make_cpu_profile.py

Measures (oracle restatement, pinned bit-exact to the reference):
  * cfg2 at full size: the first outer sweep alone and the whole solve;
  * the cfg5r proxy (n = 4096, b = 128, same generator): first F pre-pass +
    first ring step, and the whole solve -- the ratio scales to cfg4 / cfg5c /
    cfg5r by (steps per sweep x sweeps) (SURVEY.md 8(d) item iv: an ESTIMATE).
Writes oracle/cpu_profile.json.
"""
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(ROOT, ".numba_cache"))
import oracle  # noqa: E402
from paper_1008_4166_b200 import workloads  # noqa: E402


def cpu_model():
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            return line.split(":", 1)[1].strip()
    return "unknown"


out = {"host": {"cpu_model": cpu_model(), "nproc": os.cpu_count(),
                "OPENBLAS_NUM_THREADS": os.environ["OPENBLAS_NUM_THREADS"]}}
w = workloads.make("cfg2")
oracle.parallel_jacobi_2f(w.G[:128, :128], w.J[:128], 2, "round_robin", orth_tol=w.orth_tol)  # JIT warm
t0 = time.perf_counter()
oracle.parallel_jacobi_2f(w.G, w.J, w.p, "round_robin", orth_tol=w.orth_tol, threads=w.p, sweep_limit=1)
t_sweep1 = time.perf_counter() - t0
t0 = time.perf_counter()
_, info = oracle.parallel_jacobi_2f(w.G, w.J, w.p, "round_robin", orth_tol=w.orth_tol, threads="ring")
t_total = time.perf_counter() - t0
out["cfg2"] = {"t_sweep1": t_sweep1, "t_total": t_total, "sweeps": info.sweeps, "rotations": info.rotations,
               "threads": w.p, "note": "first sweep: p-thread pool, step synchronous; whole solve: p ring worker "
                                       "threads as the reference runs it"}
print("cfg2", out["cfg2"], flush=True)

pw = workloads.make("cfg5r", n=4096, b=128)
t0 = time.perf_counter()
oracle.parallel_jacobi_2f(pw.G, pw.J, pw.p, "round_robin", orth_tol=pw.orth_tol, threads=pw.p, sweep_limit=1,
                          step_limit=1)
t_first = time.perf_counter() - t0
t0 = time.perf_counter()
_, pinfo = oracle.parallel_jacobi_2f(pw.G, pw.J, pw.p, "round_robin", orth_tol=pw.orth_tol, threads="ring")
t_ptotal = time.perf_counter() - t0
ratio = t_ptotal / t_first
psteps = 2 * pw.p - 1
proxy = {"name": "cfg5r", "kw": {"n": 4096, "b": 128}, "threads": pw.p, "t_total": t_ptotal, "sweeps": pinfo.sweeps,
         "rotations": pinfo.rotations, "t_prepass1_step1": t_first}
print("proxy", proxy, flush=True)
for name, steps, sweeps in (("cfg5r", 255, 18), ("cfg5c", 127, 17), ("cfg4", 127, 20)):
    f = ratio * (steps * sweeps) / (psteps * pinfo.sweeps)
    out[name + "_extrapolation"] = {
        "factor": f,
        "how": (f"proxy cfg5r n=4096 b=128 (p={pw.p}, {psteps} steps x {pinfo.sweeps} sweeps) measured in the build "
                f"container: whole solve {t_ptotal:.1f} s = {ratio:.0f} x (first pre-pass + first step); scaled by "
                f"({steps} steps x {sweeps} sweeps)/({psteps} x {pinfo.sweeps}); an ESTIMATE (SURVEY 8(d) item iv)"),
        "proxy": proxy}
json.dump(out, open(os.path.join(ROOT, "oracle", "cpu_profile.json"), "w"), indent=1)
print("written", flush=True)
