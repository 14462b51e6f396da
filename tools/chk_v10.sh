#!/bin/bash
TAG=${1:-v10}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$TAG.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 120 python tools/upd_bench.py --cx --m 2048 --b 64 --count 16 > gpurun_out/upd_$TAG.log 2>&1
timeout 120 python tools/upd_bench.py --cx --m 8192 --b 64 --count 64 >> gpurun_out/upd_$TAG.log 2>&1
timeout 120 python tools/upd_bench.py --m 32768 --b 128 --count 128 >> gpurun_out/upd_$TAG.log 2>&1
timeout 120 python tools/upd_bench.py --cx --m 16384 --b 128 --count 64 >> gpurun_out/upd_$TAG.log 2>&1
