#!/bin/bash
# cfg5-scale evidence: ncu --set full of one step (Gram, pivot, update) of cfg5c and
# cfg5r (first outer sweep; the .ncu-rep stays in /tmp, its raw metric page comes back
# as CSV), then full-size solves with the phase split.
TAG=${1:-r1_v8}
mkdir -p gpurun_out
for c in cfg5c cfg5r; do
  timeout 300 python tools/profile_solve.py $c --sweeps 1 > gpurun_out/plain_${c}_$TAG.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:"pivot_kernel|gram_kernel|update_kernel" -s 6 -c 3 \
    -o /tmp/prof_${c}_$TAG python tools/profile_solve.py $c --sweeps 1 > gpurun_out/ncu_${c}_$TAG.log 2>&1
  ncu -i /tmp/prof_${c}_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_${c}_$TAG.csv 2>&1
  ncu -i /tmp/prof_${c}_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_details_${c}_$TAG.csv 2>&1
done
for c in cfg4 cfg5c cfg5r; do
  timeout 1200 python tools/fullsize.py $c --phases $([ $c = cfg4 ] && echo --kappa) >> gpurun_out/fullsize_$TAG.json 2>> gpurun_out/fullsize_$TAG.log
done
