# round profile, part A: GPU tests, then the ncu captures (launch list, gemm_topk and finalize --set full)
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02h_gputest.log 2>&1
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/r02h_pre.json 2> gpurun_out/r02h_pre.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches_bench.csv python bench.py --steps 2 --warmup 3 --eager --no-e2e --no-cpu > gpurun_out/r02h_ncu_launch.log 2>&1
ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:gemm_topk_kernel -o gpurun_out/r02h_gemm python tools/ncu_step.py --config cfg2 --k 10 > gpurun_out/r02h_ncu_gemm.log 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:finalize_kernel -o gpurun_out/r02h_fin python tools/ncu_step.py --config cfg2 --k 10 > gpurun_out/r02h_ncu_fin.log 2>&1
