#!/bin/bash
cd "$(dirname "$0")/.."
export NUMBA_CACHE_DIR=/tmp/nc
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > $O/t4.log 2>&1; echo "rc=$?" >> $O/t4.log
HJB_LIB=$PWD/paper_1008_4166_b200/libhjb200_prof.so timeout 600 python tools/jac_bench.py cfg1 cfg2 cfg3 cfg5r cfg5c > $O/jac_prof3.jsonl 2> $O/jac_prof3.err
timeout 600 python tools/jac_bench.py cfg1 cfg2 cfg3 cfg5r cfg5c > $O/jac_v2_3.jsonl 2> $O/jac_v2_3.err
for sh in "4,8,2" "4,4,4"; do HJB_JAC_SHAPE=$sh timeout 300 python tools/jac_bench.py cfg2 cfg3 >> $O/jac_shapes3.jsonl 2>> $O/jac_shapes3.err; done
for sh in "4,8,4" "16,4,2"; do HJB_JAC_SHAPE=$sh timeout 300 python tools/jac_bench.py cfg5r cfg5c >> $O/jac_shapes3.jsonl 2>> $O/jac_shapes3.err; done
for sh in "4,4,2"; do HJB_JAC_SHAPE=$sh timeout 300 python tools/jac_bench.py cfg1 >> $O/jac_shapes3.jsonl 2>> $O/jac_shapes3.err; done
timeout 300 python bench.py --config cfg2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/b_v2_3.json 2> $O/b_v2_3.err
echo done
