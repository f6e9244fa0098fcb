for r in 1 2; do
for cfg in "cfg4 --k 10" "cfg4 --k 1" "cfg2 --k 1" "cfg2 --k 5" "cfg2 --k 10 --prefix-exit on"; do
  for st in 0 3 2; do echo -n "st=$st "; SIMDEX_EXIT_STAGES=$st python tools/ab_kernels.py --config $cfg --steps 10 2>&1 | tail -1; done
done
done
