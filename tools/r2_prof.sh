#!/bin/bash
# round-2 profile pass: launch lists (one cfg2 solve, one cfg5r sweep) and
# ncu --set full captures of the Jacobi / update / Gram / pivot kernels,
# exported to text on the box (the .ncu-rep files are too large to bring back)
cd "$(dirname "$0")/.."
export NUMBA_CACHE_DIR=/tmp/nc
O=gpurun_out
T=${1:-r2}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2_$T.csv \
  python tools/profile_solve.py cfg2 > $O/ncu_l2_$T.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5r_$T.csv \
  python tools/profile_solve.py cfg5r --sweeps 1 > $O/ncu_l5_$T.log 2>&1
export_rep() {
  ncu -i $1.ncu-rep --page details > $1_details.txt 2>&1
  ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>&1
  ncu -i $1.ncu-rep --page source --csv --print-source sass -k regex:jacobi_kernel > $1_jac_sass.csv 2>&1
  gzip -f $1_raw.csv $1_jac_sass.csv
  rm -f $1.ncu-rep
}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"jacobi_kernel|update_kernel|gram_kernel|gram_reduce|factor_" -s 14 -c 7 \
  -o /tmp/full_cfg5r_$T python tools/profile_solve.py cfg5r --sweeps 1 > $O/ncu_f5_$T.log 2>&1
export_rep /tmp/full_cfg5r_$T; mv /tmp/full_cfg5r_${T}_* $O/
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"jacobi_kernel|factor_|gram_kernel|gram_reduce|update_kernel" -s 24 -c 7 \
  -o /tmp/full_cfg2_$T python tools/profile_solve.py cfg2 > $O/ncu_f2_$T.log 2>&1
export_rep /tmp/full_cfg2_$T; mv /tmp/full_cfg2_${T}_* $O/
du -sh $O
echo done
