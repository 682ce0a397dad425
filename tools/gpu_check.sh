timeout 1500 python -m pytest tests/ -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_all.log 2>&1
grep -E "passed|failed|FAILED|Error |error:" gpurun_out/pytest_gpu_all.log | head -30
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fa_fwd_tc -s 30 -c 1 -o gpurun_out/prof_fa_fwd -f python bench.py --steps 1 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/ncu_fa_fwd.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fa_bwd_dkv_tc -s 30 -c 1 -o gpurun_out/prof_fa_dkv -f python bench.py --steps 1 --warmup 3 --no-baselines --no-cpu-baseline > gpurun_out/ncu_fa_dkv.log 2>&1
tail -3 gpurun_out/ncu_fa_fwd.log
