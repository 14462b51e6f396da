for n in 16; do timeout 120 python tools/pivot_bench.py cfg2 --sweep 0 --clusters 4,8,16 --threads 128,256 --dup 2 --count $n 2>&1 | grep -v per-round; done
timeout 120 python tools/pivot_bench.py cfg3 --sweep 0 --clusters 2,4 --threads 256 --dup 2 --count 32 2>&1 | grep -v per-round
