for k in 10 5; do
  for h in 128 256 384; do
    echo -n "hyb$h k=$k: "; SIMDEX_PREFIX_HEAD=$h python tools/ab_kernels.py --config cfg2 --k $k --steps 20 2>&1 | tail -1
  done
done
