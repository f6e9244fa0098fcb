for k in 1 5 10 50; do for e in off on; do python tools/ab_kernels.py --config cfg2 --k $k --prefix-exit $e --steps 10 2>&1 | tail -1; done; done
for e in off on; do python tools/ab_kernels.py --config cfg4 --k 10 --prefix-exit $e --steps 10 2>&1 | tail -1; done
