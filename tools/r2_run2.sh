#!/bin/bash
# round-2 pass 2: fixed tests, Jacobi phase clocks, v1/v2 inner micro-bench, cfg2 launch list
cd "$(dirname "$0")/.."
export NUMBA_CACHE_DIR=/tmp/nc
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -k "not cfg5c" > $O/t3.log 2>&1; echo "rc=$?" >> $O/t3.log
HJB_LIB=$PWD/paper_1008_4166_b200/libhjb200_prof.so timeout 600 python tools/jac_bench.py cfg1 cfg2 cfg3 cfg5r cfg5c > $O/jac_prof.jsonl 2> $O/jac_prof.err
timeout 600 python tools/jac_bench.py cfg1 cfg2 cfg3 cfg5r cfg5c > $O/jac_v2.jsonl 2> $O/jac_v2.err
HJB_PIVOT_V1=1 timeout 600 python tools/jac_bench.py cfg1 cfg2 cfg3 cfg5r cfg5c > $O/jac_v1.jsonl 2> $O/jac_v1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/launches_jac_cfg2.csv python tools/jac_bench.py cfg2 --reps 2 > $O/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:jacobi_kernel -c 1 -o $O/jac_cfg2 python tools/jac_bench.py cfg2 --reps 1 > $O/ncu_f.log 2>&1
echo done
