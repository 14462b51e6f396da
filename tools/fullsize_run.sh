#!/bin/bash
# Full-size timings (one solve each) under gpurun: bash tools/fullsize_run.sh TAG
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/fullsize_$TAG.log
nproc >> gpurun_out/fullsize_$TAG.log
timeout 300 python tools/fullsize.py cfg3 --phases >> gpurun_out/fullsize_$TAG.json 2>> gpurun_out/fullsize_$TAG.log
timeout 900 python tools/fullsize.py cfg4 --phases --kappa >> gpurun_out/fullsize_$TAG.json 2>> gpurun_out/fullsize_$TAG.log
timeout 900 python tools/fullsize.py cfg5c --phases >> gpurun_out/fullsize_$TAG.json 2>> gpurun_out/fullsize_$TAG.log
timeout 900 python tools/fullsize.py cfg5r >> gpurun_out/fullsize_$TAG.json 2>> gpurun_out/fullsize_$TAG.log
echo done >> gpurun_out/fullsize_$TAG.log
