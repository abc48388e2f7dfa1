# Round evidence on one B200 (dev tool; run under gpurun).  Everything lands in gpurun_out/:
#   smoke.log, pytest_gpu.log     smoke() and the full -m gpu suite
#   bench*.json                   bench.py lines (interactive frame; reference arm; 4-channel)
#   configs.json                  tools/bench_configs.py (every BASELINE config)
#   launches_*.csv                ncu launch lists (gpu__time_duration.sum, cold + serialised)
#   *.ncu-rep                     ncu --set full captures of the kernels named in DESIGN.md
set -x
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --channels 4 > gpurun_out/bench_mc4.json 2> gpurun_out/bench_mc4.err
timeout 900 python tools/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_interactive_frame.csv python bench.py --steps 4 --warmup 3 --no-cpu --frame-only > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_mc4.csv python bench.py --channels 4 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_hybrid_1024.csv python tools/prof_kd.py 1024 hybrid 0.3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_kd_deep_512.csv python tools/prof_kd.py 512 kd-deep-mls32 0.3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_brick_summary" -s 2 -c 1 -o gpurun_out/summary_1024 \
  python bench.py --steps 2 --warmup 3 --no-cpu --frame-only > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_segments_brick|k_integrate_segments|k_flags_tiles|k_tree_chunk|k_leaves_coop|k_presence" -s 12 -c 8 -o gpurun_out/frame_1024 \
  python bench.py --steps 2 --warmup 3 --no-cpu --frame-only > /dev/null 2>&1
for t in 0.6 0.3 0.0; do
  timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"k_segments_brick|k_integrate_segments" -c 2 -o gpurun_out/render_t$t \
    python tools/prof_render.py 1024 lbvh $t 32 > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_classify_pack|k_levels" -c 3 -o gpurun_out/kd_1024 \
  python tools/prof_kd.py 1024 hybrid 0.6 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"k_integrate_multi" -c 1 -o gpurun_out/multi_1024 \
  python bench.py --channels 4 --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
# summaries on the box (the .ncu-rep files exceed what gpurun copies back)
python tools/round_summaries.py ${ROUND:-r02} gpurun_out/summaries > gpurun_out/summaries.log 2>&1
mkdir -p gpurun_out/keep; mv gpurun_out/summary_1024.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out gpurun_out/summaries
