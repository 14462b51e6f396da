#!/bin/bash
# final round-1 measurement pass: tests, smoke, bench lines, launch list, ncu, full-size solves
TAG=${1:-r1_v9}
bash tools/gpu_round.sh $TAG
for c in cfg4 cfg5c cfg5r; do
  timeout 1200 python tools/fullsize.py $c --phases $([ $c = cfg4 ] && echo --kappa) >> gpurun_out/fullsize_$TAG.json 2>> gpurun_out/fullsize_$TAG.log
done
