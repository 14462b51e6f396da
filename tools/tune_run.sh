# whole-solve time for forced pivot (cluster, threads) pairs: bash tools/tune_run.sh cfg2 "4:256 8:128 8:256"
for ct in $2; do
  c=${ct%%:*}; t=${ct#*:}
  HJB_PIVOT_CLUSTER=$c HJB_PIVOT_THREADS=$t timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 C=$c NT=$t', round(d['value'],4), {k: round(v,1) for k,v in d['phase_ms'].items()}, d['cluster_size'])"
done
