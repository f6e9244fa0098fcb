# prefix: centroid order without exit (default) vs list order + exit vs hybrid head H + exit
for k in 10 50 5 1; do
  echo -n "off k=$k: "; python tools/ab_kernels.py --config cfg2 --k $k --steps 20 --prefix-exit off 2>&1 | tail -1
  echo -n "list k=$k: "; SIMDEX_PREFIX_HEAD=0 python tools/ab_kernels.py --config cfg2 --k $k --steps 20 --prefix-exit on 2>&1 | tail -1
  for h in 256 512 1024; do
    echo -n "hyb$h k=$k: "; SIMDEX_PREFIX_HEAD=$h python tools/ab_kernels.py --config cfg2 --k $k --steps 20 --prefix-exit on 2>&1 | tail -1
  done
done
for h in 0 256 512; do
  echo -n "cfg4 hyb$h k=10: "; SIMDEX_PREFIX_HEAD=$h python tools/ab_kernels.py --config cfg4 --k 10 --steps 20 2>&1 | tail -1
done
