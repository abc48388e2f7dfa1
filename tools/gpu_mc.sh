# 4-channel: parity tests (default build) + bench per variant (dev tool)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multichannel.py tests/test_gpu_scale.py -k "multi or channel or config4" -m gpu -q -p no:cacheprovider > gpurun_out/pytest_mc.log 2>&1
tail -2 gpurun_out/pytest_mc.log
for f in variants/lib_*.so; do
  echo "== $f"
  VSB200_LIB=$PWD/$f timeout 400 python bench.py --channels 4 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['render'])"
done
