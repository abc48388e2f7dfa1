# End-of-round refresh on one B200 (dev tool): smoke, the -m gpu suite, the interactive bench
# line and every BASELINE config, on the final tree (the ncu captures come from round_profiles.sh).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python tools/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err
timeout 600 python tools/time_kd.py 512 1024 > gpurun_out/time_kd.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_classify_pack|k_levels" -c 3 -o gpurun_out/kd_1024 \
  python tools/prof_kd.py 1024 hybrid 0.6 1 > /dev/null 2>&1
python tools/round_summaries.py ${ROUND:-r02} gpurun_out/summaries > gpurun_out/summaries.log 2>&1
rm -f gpurun_out/*.ncu-rep
