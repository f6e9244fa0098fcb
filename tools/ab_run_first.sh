# list-order exit prefix (cfg4): first chunk stored whole (default) vs threshold-filtered stores
for k in 10 1; do
  for v in A B A B; do
    if [ $v = B ]; then export SIMDEX_FIRST_FILTERED=1; else unset SIMDEX_FIRST_FILTERED; fi
    echo -n "$v cfg4 k=$k: "; python tools/ab_kernels.py --config cfg4 --k $k --steps 20 2>&1 | tail -1
  done
done
unset SIMDEX_FIRST_FILTERED
