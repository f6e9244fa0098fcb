# finalize v1 (lane per candidate) vs v2 (warp per row), same library
for cfg in "cfg2 --k 10" "cfg2 --k 1" "cfg2 --k 50" "cfg4 --k 10" "cfg3" "cfg5 --scale 0.25"; do
  for v in V1 V2; do
    if [ $v = V1 ]; then export SIMDEX_FINALIZE_V1=1; else unset SIMDEX_FINALIZE_V1; fi
    echo -n "$v "; python tools/ab_kernels.py --config $cfg --steps 10 2>&1 | tail -1
  done
done
