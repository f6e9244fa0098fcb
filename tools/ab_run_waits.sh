set -x
for r in 1 2; do
for v in A B C D; do SIMDEX_LIB_PATH=build/ab/lib$v.so python tools/ab_kernels.py --config cfg2 --k 10 --steps 30 2>&1 | tail -1; done
done
for v in A B D; do SIMDEX_LIB_PATH=build/ab/lib$v.so python tools/ab_kernels.py --config cfg3 --steps 10 2>&1 | tail -1; done
for v in A B D; do SIMDEX_LIB_PATH=build/ab/lib$v.so python tools/ab_kernels.py --config cfg2 --k 50 --steps 10 2>&1 | tail -1; done
for v in A B D; do SIMDEX_LIB_PATH=build/ab/lib$v.so python tools/ab_kernels.py --config cfg4 --k 10 --steps 10 2>&1 | tail -1; done
