for cfg in "cfg2 --k 10" "cfg2 --k 1" "cfg2 --k 5" "cfg2 --k 50" "cfg4 --k 10"; do
  for o in list score; do
    for e in off on; do
      echo -n "$o "; SIMDEX_PREFIX_ORDER=$o python tools/ab_kernels.py --config $cfg --prefix-exit $e --steps 10 2>&1 | tail -1
    done
  done
done
