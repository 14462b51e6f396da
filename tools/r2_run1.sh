#!/bin/bash
# round-2 first GPU pass: new Jacobi kernel parity, GPU suite, cfg2 v1/v2 timing
cd "$(dirname "$0")/.."
export NUMBA_CACHE_DIR=/tmp/nc
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "pivot_kernel or dense_prepass" > $O/t1.log 2>&1; echo "rc=$?" >> $O/t1.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > $O/t2.log 2>&1; echo "rc=$?" >> $O/t2.log
timeout 300 python bench.py --config cfg2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/b_v2.json 2> $O/b_v2.err
HJB_PIVOT_V1=1 timeout 300 python bench.py --config cfg2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/b_v1.json 2> $O/b_v1.err
timeout 300 python bench.py --config cfg3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/b3_v2.json 2> $O/b3_v2.err
echo done
