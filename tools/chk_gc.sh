#!/bin/bash
# quick check of a pivot change: GPU parity, cfg2 bench, cfg5c full size
TAG=${1:-gc}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python tools/fullsize.py ${2:-cfg5c} --phases > gpurun_out/fullsize_$TAG.json 2> gpurun_out/fullsize_$TAG.log
