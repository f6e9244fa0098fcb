# stage-2 catalogue segments + pruning: target 2 (default) / 4 / 8 units per CTA slot, and no split
for n in 1 2 4 8; do
  for v in T2 T4 T8 NS; do
    case $v in T2) L=paper_1706_01449_b200/lib/libsimdex_b200.so;; NS) L=paper_1706_01449_b200/lib/libsimdex_b200.so;; *) L=build/ab/lib${v}.so;; esac
    if [ $v = NS ]; then export SIMDEX_NO_SPLIT=1; else unset SIMDEX_NO_SPLIT; fi
    echo -n "$v "; SIMDEX_LIB_PATH=$L python tools/shard_kernels.py cfg2 $n 0 2>&1 | tail -1
  done
done
unset SIMDEX_NO_SPLIT
for v in T2 NS; do
  if [ $v = NS ]; then export SIMDEX_NO_SPLIT=1; else unset SIMDEX_NO_SPLIT; fi
  echo -n "$v cfg4 "; python tools/shard_kernels.py cfg4 1 0 2>&1 | tail -1
done
