#!/bin/bash
# One GPU measurement pass: tests, smoke, bench, launch list, ncu captures.
# Usage (under gpurun): bash tools/gpu_round.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "rc=$?" >> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
for c in cfg1 cfg3; do timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline >> gpurun_out/bench_cfgs_$TAG.json 2>> gpurun_out/bench_cfgs_$TAG.err; done
# launch list of one full cfg2 solve (same kernels as one bench step)
python tools/profile_solve.py cfg2 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2_$TAG.csv python tools/profile_solve.py cfg2 > gpurun_out/ncu_list_$TAG.log 2>&1
# one full capture of each kernel (sweep-1 step launches)
python tools/profile_solve.py cfg2 --sweeps 1 > gpurun_out/plain1_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pivot_kernel|gram_kernel|update_kernel" -s 6 -c 3 -o gpurun_out/prof_cfg2_$TAG python tools/profile_solve.py cfg2 --sweeps 1 > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
