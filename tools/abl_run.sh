# usage: bash tools/abl_run.sh "base a16 ..." [clusters] [threads] [config]
for v in $1; do
  HJB_LIB=$PWD/build/v_$v.so timeout 120 python tools/pivot_bench.py ${4:-cfg2} --sweep 0 --clusters ${2:-4,8} --threads ${3:-128,256} --count 15 2>&1 | grep -v "per-round" | sed "s/^/$v /"
done
