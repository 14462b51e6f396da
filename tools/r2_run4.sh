#!/bin/bash
cd "$(dirname "$0")/.."
export NUMBA_CACHE_DIR=/tmp/nc
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "pivot or jacobi or cluster or small_solves" > $O/t5.log 2>&1; echo "rc=$?" >> $O/t5.log
HJB_LIB=$PWD/paper_1008_4166_b200/libhjb200_prof.so timeout 600 python tools/jac_bench.py cfg1 cfg2 cfg3 cfg5r cfg5c > $O/jac_prof4.jsonl 2> $O/jac_prof4.err
timeout 600 python tools/jac_bench.py cfg1 cfg2 cfg3 cfg5r cfg5c > $O/jac_v2_4.jsonl 2> $O/jac_v2_4.err
for sh in "4,8,2" "4,4,4"; do HJB_JAC_SHAPE=$sh timeout 300 python tools/jac_bench.py cfg2 cfg3 >> $O/jac_shapes4.jsonl 2>> $O/jac_shapes4.err; done
for sh in "4,8,4" "16,4,2"; do HJB_JAC_SHAPE=$sh timeout 300 python tools/jac_bench.py cfg5r cfg5c >> $O/jac_shapes4.jsonl 2>> $O/jac_shapes4.err; done
for sh in "4,4,2"; do HJB_JAC_SHAPE=$sh timeout 300 python tools/jac_bench.py cfg1 >> $O/jac_shapes4.jsonl 2>> $O/jac_shapes4.err; done
echo done
