for cfg in "cfg2 --k 10" "cfg2 --k 1" "cfg4 --k 10" "cfg3"; do
  for v in 0 1; do
    echo -n "coop=$v "; SIMDEX_FIN_COOP=$v python tools/ab_kernels.py --config $cfg --steps 10 2>&1 | tail -1
  done
done
for lib in Old New; do
  for c in "cfg2 10" "cfg4 10"; do SIMDEX_LIB_PATH=build/ab/lib$lib.so python tools/walk_bench.py $c 2>&1 | tail -1; done
done
