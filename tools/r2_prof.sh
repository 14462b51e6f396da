#!/bin/bash
# round-2 profile pass: launch lists (one cfg2 solve, one cfg5r sweep) and
# ncu --set full captures of the Jacobi / update / Gram kernels
cd "$(dirname "$0")/.."
export NUMBA_CACHE_DIR=/tmp/nc
O=gpurun_out
T=${1:-r2}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg2_$T.csv \
  python tools/profile_solve.py cfg2 > $O/ncu_l2_$T.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg5r_$T.csv \
  python tools/profile_solve.py cfg5r --sweeps 1 > $O/ncu_l5_$T.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"jacobi_kernel|update_kernel|gram_kernel|pivot_kernel" -s 12 -c 5 \
  -o $O/full_cfg5r_$T python tools/profile_solve.py cfg5r --sweeps 1 > $O/ncu_f5_$T.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"jacobi_kernel|pivot_kernel|gram_kernel|update_kernel" -s 20 -c 5 \
  -o $O/full_cfg2_$T python tools/profile_solve.py cfg2 > $O/ncu_f2_$T.log 2>&1
echo done
