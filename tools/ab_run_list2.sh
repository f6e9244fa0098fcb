# stage 2 over each cluster's own list (default) vs the norm-sorted catalogue (SIMDEX_NO_LIST_STAGE2=1)
for cfg in "cfg2 --k 10" "cfg2 --k 5" "cfg2 --k 1" "cfg2 --k 50"; do
  for v in A B A B; do
    if [ $v = B ]; then export SIMDEX_NO_LIST_STAGE2=1; else unset SIMDEX_NO_LIST_STAGE2; fi
    echo -n "$v $cfg: "; python tools/ab_kernels.py --config $cfg --steps 20 2>&1 | tail -1
  done
done
unset SIMDEX_NO_LIST_STAGE2
