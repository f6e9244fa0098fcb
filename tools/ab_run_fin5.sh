# finalize rescoring: A = a lane per candidate (two per lane at 9..16 survivors), B = the row's 8 lanes share each candidate's item row
for cfg in "cfg2 --k 10" "cfg2 --k 5" "cfg2 --k 1" "cfg2 --k 50" "cfg4 --k 10" "cfg4 --k 1"; do
  for v in A B; do
    echo -n "$cfg $v: "; SIMDEX_LIB_PATH=build/ab/lib$v.so python tools/ab_kernels.py --config $cfg --steps 20 2>&1 | tail -1
  done
done
