#!/bin/bash
# Build ablation / profiling variants of libhjb200 into build/ (dev instance table).
# Usage: tools/build_variants.sh "name:FLAGS ..."   e.g. "a16:-DHJB_ABL=16 nb:-DHJB_PASS_NAMED=1"
cd "$(dirname "$0")/.."
for spec in $1; do
  name=${spec%%:*}; fl=${spec#*:}; fl=${fl//,/ }
  HJB_NVCC_FLAGS="-DHJB_PIVOT_DEV -DHJB_ROUND_PROFILE=1 $fl" HJB_LIB=$PWD/build/v_$name.so HJB_OBJ_TAG=_v$name \
    python -m paper_1008_4166_b200.build > build/v_$name.log 2>&1 &
done
wait
for spec in $1; do name=${spec%%:*}; ls build/v_$name.so >/dev/null 2>&1 || tail -5 build/v_$name.log; done
ls -la build/v_*.so
