# full GPU suite + bench + launch list of the interactive frame (dev tool)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_frame.csv python bench.py --steps 2 --warmup 3 --no-cpu --frame-only > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_frame.csv > gpurun_out/launches_frame.txt
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cat gpurun_out/launches_frame.txt; tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['build'], d['render_by_t'], d['lbvh_height'], d['parity_index_vs_public_api'])"
