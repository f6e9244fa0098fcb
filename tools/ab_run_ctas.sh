for r in 1 2; do
for cfg in "cfg2 --k 10" "cfg2 --k 1" "cfg2 --k 50" "cfg4 --k 10" "cfg3"; do
  for v in A B D; do echo -n "$v "; SIMDEX_LIB_PATH=build/ab/lib$v.so python tools/ab_kernels.py --config $cfg --steps 10 2>&1 | tail -1; done
done
done
