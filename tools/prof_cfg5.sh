#!/bin/bash
# cfg5-scale evidence: ncu --set full of one step (Gram, pivot, update) of cfg5c and
# cfg5r (first outer sweep), then a full cfg5r solve with the phase split.
TAG=${1:-r1_v7}
mkdir -p gpurun_out
for c in cfg5c cfg5r; do
  timeout 300 python tools/profile_solve.py $c --sweeps 1 > gpurun_out/plain_${c}_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pivot_kernel|gram_kernel|update_kernel" -s 6 -c 3 \
    -o gpurun_out/prof_${c}_$TAG python tools/profile_solve.py $c --sweeps 1 > gpurun_out/ncu_${c}_$TAG.log 2>&1
done
timeout 1200 python tools/fullsize.py cfg5r --phases > gpurun_out/fullsize_cfg5r_$TAG.json 2> gpurun_out/fullsize_cfg5r_$TAG.log
