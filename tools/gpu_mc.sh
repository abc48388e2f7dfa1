cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multichannel.py tests/test_gpu_render.py tests/test_gpu_scale.py -k "multi or channel or config4 or render or frame" -m gpu -q -p no:cacheprovider > gpurun_out/pytest_mc.log 2>&1
tail -3 gpurun_out/pytest_mc.log
timeout 400 python bench.py --channels 4 --no-cpu 2>/dev/null > gpurun_out/bench_mc4.json; python -c "import json; d=json.load(open('gpurun_out/bench_mc4.json')); print(d['value'], d['e2e']['value'], d['render'])"
