# finalize variants: A = previous, B = two-per-lane + vector rank loop (48 regs), C = B at 40 regs, D = C without two-per-lane
for cfg in "cfg2 --k 10" "cfg2 --k 5" "cfg2 --k 50" "cfg4 --k 10" "cfg3"; do
  for v in A B C D; do
    echo -n "$cfg $v: "; SIMDEX_LIB_PATH=build/ab/lib$v.so python tools/ab_kernels.py --config $cfg --steps 20 2>&1 | tail -1
  done
done
