mkdir -p gpurun_out
for v in base wr; do
  HJB_LIB=$PWD/build/v_$v.so timeout 200 python tools/pivot_bench.py cfg2 --sweep 2 --clusters 8,4 --threads 128,256 2>&1 | sed "s/^/$v /" >> gpurun_out/abl_wr.log
done
