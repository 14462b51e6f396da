#!/bin/bash
TAG=${1:-div}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
HJB_LIB=$PWD/build/v_wbp.so timeout 200 python tools/pivot_bench.py cfg2 --sweep 2 --clusters 8,4 --threads 128,256 > gpurun_out/pivbench_$TAG.log 2>&1
