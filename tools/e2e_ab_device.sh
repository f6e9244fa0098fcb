# e2e with small uploads pinned (current) vs pageable (SIMDEX_SMALL_PAGEABLE=1)
for i in 1 2; do
  for v in A B; do
    if [ $v = B ]; then export SIMDEX_SMALL_PAGEABLE=1; else unset SIMDEX_SMALL_PAGEABLE; fi
    echo -n "$v "; python bench.py --no-cpu --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); e=d['e2e']; print(round(e['value']/1e6,2), {k: round(v*1e3,2) for k,v in e['stage_seconds'].items()}, e.get('pass_ms'))"
  done
done
