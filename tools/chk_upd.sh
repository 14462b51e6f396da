#!/bin/bash
mkdir -p gpurun_out
for v in base upd; do
  lib=$PWD/paper_1008_4166_b200/libhjb200.so; [ $v = upd ] && lib=$PWD/build/v_upd.so
  HJB_LIB=$lib timeout 120 python tools/upd_bench.py --m 32768 --b 128 --count 128 >> gpurun_out/upd_bench.log 2>&1
  HJB_LIB=$lib timeout 120 python tools/upd_bench.py --cx --m 16384 --b 128 --count 64 >> gpurun_out/upd_bench.log 2>&1
done
HJB_LIB=$PWD/build/v_wbp.so timeout 200 python tools/pivot_bench.py cfg2 --sweep 2 --clusters 8,4 --threads 128,256 > gpurun_out/pivbench_wbp2.log 2>&1
