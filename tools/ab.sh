#!/bin/bash
# A/B timing of two builds of the library on the same box:
#   tools/ab.sh ROUNDS cmd...   (build/ab/libA.so vs build/ab/libB.so, alternating)
n=$1; shift
for i in $(seq 1 $n); do
  for v in A B; do
    echo -n "$v: "; SIMDEX_LIB_PATH=build/ab/lib$v.so "$@" 2>&1 | tail -1
  done
done
