for v in k0 k1 k4 k16 k64; do
  echo "== $v"; HJB_LIB=$PWD/build/v_$v.so timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['sweeps'], d['rotations'], d['phase_ms']['pivot_ms'])"
  HJB_LIB=$PWD/build/v_$v.so timeout 300 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['sweeps'], d['rotations'], d['phase_ms']['pivot_ms'])"
done
