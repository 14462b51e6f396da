#!/bin/bash
TAG=${1:-r1_v10}
bash tools/gpu_round.sh $TAG
timeout 1200 python tools/fullsize.py cfg4 --phases --kappa >> gpurun_out/fullsize_$TAG.json 2>> gpurun_out/fullsize_$TAG.log
