# End-of-round refresh on one B200 (dev tool): smoke, the -m gpu suite, the interactive bench
# line and every BASELINE config, on the final tree (the ncu captures come from round_profiles.sh).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python tools/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err
timeout 600 python tools/time_kd.py 512 1024 > gpurun_out/time_kd.txt 2>&1
