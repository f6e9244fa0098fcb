# round profile, part B: the bench lines (cfg2 with e2e and cpu_baseline, the reference arm, cfg3/4/5), shard scaling, e2e timeline
set -x
python bench.py > gpurun_out/r02h_bench_cfg2.json 2> gpurun_out/r02h_bench_cfg2.err
python bench.py --impl reference > gpurun_out/r02h_bench_reference_arm.json 2> gpurun_out/r02h_ref.err
for c in cfg3 cfg4 cfg5; do python bench.py --config $c --no-e2e --no-cpu > gpurun_out/r02h_bench_$c.json 2> gpurun_out/r02h_bench_$c.err; done
for c in cfg2 cfg3 cfg4; do python tools/shard_scaling.py $c --graph; done > gpurun_out/r02h_shard_scaling.jsonl 2>gpurun_out/r02h_scal.err
python tools/kprof_e2e.py cfg2 > gpurun_out/r02h_kprof_e2e.txt 2>&1
for k in 1 5 50; do python bench.py --k $k --no-e2e --no-cpu > gpurun_out/r02h_bench_cfg2_k$k.json 2> gpurun_out/r02h_bench_cfg2_k$k.err; done
