# Round evidence on one B200 (dev tool; run under gpurun).  Everything lands in gpurun_out/:
#   bench*.json        bench.py lines (interactive frame; 4-channel frame)
#   configs.json       tools/bench_configs.py (every BASELINE config)
#   launches_*.csv     ncu launch lists (gpu__time_duration.sum, cold + serialised)
#   *.ncu-rep          ncu --set full captures of the kernels named in DESIGN.md
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python bench.py --channels 4 > gpurun_out/bench_mc4.json 2> gpurun_out/bench_mc4.err
timeout 900 python tools/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_interactive_frame.csv python bench.py --steps 2 --warmup 3 --no-cpu --frame-only > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_mc4.csv python bench.py --channels 4 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_hybrid_1024.csv python tools/prof_kd.py 1024 hybrid 0.3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_kd_deep_512.csv python tools/prof_kd.py 512 kd-deep-mls32 0.3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_classify_pack|k_spans_rows|k_decide" -c 4 -o gpurun_out/kd_1024 \
  python tools/prof_kd.py 1024 hybrid 0.6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_brick_summary|k_segments|k_integrate_segments" -s 3 -c 3 -o gpurun_out/frame_1024 \
  python bench.py --steps 2 --warmup 3 --no-cpu --frame-only > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_integrate_multi" -c 1 -o gpurun_out/multi_1024 \
  python bench.py --channels 4 --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out
