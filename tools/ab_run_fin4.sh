# finalize rescoring: A = exact float32 item rows (converted per factor), B = float64 item rows (twice the bytes, no conversions)
for cfg in "cfg2 --k 10" "cfg4 --k 10" "cfg3"; do
  for v in A B A B; do
    echo -n "$cfg $v: "; SIMDEX_LIB_PATH=build/ab/lib$v.so python tools/ab_kernels.py --config $cfg --steps 20 2>&1 | tail -1
  done
done
