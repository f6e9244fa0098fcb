# timing only: E = certified band x 0.001 (NOT exact), F = band x 0.5 (NOT exact); A = shipped
for cfg in "cfg2 --k 10" "cfg4 --k 10" "cfg3"; do
  for v in A F E; do echo -n "$v "; SIMDEX_LIB_PATH=build/ab/lib$v.so python tools/ab_kernels.py --config $cfg --steps 10 2>&1 | tail -1; done
done
