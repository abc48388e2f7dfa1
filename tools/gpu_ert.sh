cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scale.py -k "early_ray or lbvh_1024" tests/test_gpu_render.py tests/test_gpu_build.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_ert.log 2>&1
tail -3 gpurun_out/pytest_ert.log
timeout 400 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['e2e']['value'], d['ert'], {k: v for k, v in d['build'].items() if not isinstance(v, str)}, d['rebuild_ms_by_kind'])"
