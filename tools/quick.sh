# quick GPU iteration: pivot parity subset, pivot_bench, bench (dev instance table)
export HJB_LIB=$PWD/build/dev.so
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "test_pivot_kernel_matches_oracle and (64-4 or 64-0 or 32-0) or test_pivot_dense or test_cfg1_full or test_config_proxies and (cfg2 or cfg3)" 2>&1 | tail -2
HJB_LIB=$PWD/build/libhjb200_prof.so timeout 200 python tools/pivot_bench.py cfg2 --sweep 4 --clusters ${1:-4,8} --threads ${2:-128,256} 2>&1 | grep -v per-round
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['sweeps'], d['phase_ms'], d['cluster_size'])"
