set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/gemm_bench.py 768 > gpurun_out/gemm_bench_768.log 2>&1
timeout 300 python tools/gemm_bench.py 1024 > gpurun_out/gemm_bench_1024.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01c.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r01c.csv python bench.py --steps 2 --warmup 1 --profile --no-baselines --no-cpu-baseline > gpurun_out/bench_under_ncu2.log 2>&1
tail -3 gpurun_out/bench_r01c.log
