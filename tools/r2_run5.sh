#!/bin/bash
cd "$(dirname "$0")/.."
export NUMBA_CACHE_DIR=/tmp/nc
O=gpurun_out
L=$PWD/paper_1008_4166_b200
rm -f $O/jac5_*.jsonl
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k "pivot or jacobi or cluster or small_solves" > $O/t6.log 2>&1; echo "rc=$?" >> $O/t6.log
for v in f0p f1p; do HJB_LIB=$L/libhjb200_$v.so timeout 600 python tools/jac_bench.py cfg1 cfg2 cfg3 cfg5r cfg5c > $O/jac5_$v.jsonl 2>> $O/jac5.err; done
for v in f0 ""; do
  lib=$L/libhjb200${v:+_$v}.so
  for sh in "8,4,2" "4,8,2"; do HJB_LIB=$lib HJB_JAC_SHAPE=$sh timeout 300 python tools/jac_bench.py cfg2 cfg3 >> $O/jac5_shapes_${v:-f1}.jsonl 2>> $O/jac5.err; done
  for sh in "8,8,2" "4,8,4" "16,4,2"; do HJB_LIB=$lib HJB_JAC_SHAPE=$sh timeout 300 python tools/jac_bench.py cfg5r cfg5c >> $O/jac5_shapes_${v:-f1}.jsonl 2>> $O/jac5.err; done
  for sh in "2,4,4" "4,4,2"; do HJB_LIB=$lib HJB_JAC_SHAPE=$sh timeout 300 python tools/jac_bench.py cfg1 >> $O/jac5_shapes_${v:-f1}.jsonl 2>> $O/jac5.err; done
done
echo done
