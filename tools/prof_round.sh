set -x
python bench.py > gpurun_out/r02h_bench_cfg2.json 2> gpurun_out/r02h_bench_cfg2.err
python bench.py --impl reference > gpurun_out/r02h_bench_reference_arm.json 2> gpurun_out/r02h_ref.err
for c in cfg3 cfg4 cfg5; do python bench.py --config $c --no-e2e --no-cpu > gpurun_out/r02h_bench_$c.json 2> gpurun_out/r02h_bench_$c.err; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02h_ncu_launch.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_topk_kernel -o gpurun_out/r02h_gemm python tools/ncu_step.py --config cfg2 --k 10 > gpurun_out/r02h_ncu_gemm.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:finalize_kernel -o gpurun_out/r02h_fin python tools/ncu_step.py --config cfg2 --k 10 > gpurun_out/r02h_ncu_fin.log 2>&1
for c in cfg2 cfg3 cfg4; do python tools/shard_scaling.py $c --graph; done > gpurun_out/r02h_shard_scaling.jsonl 2>gpurun_out/r02h_scal.err
python tools/kprof_e2e.py cfg2 > gpurun_out/r02h_kprof_e2e.txt 2>&1
