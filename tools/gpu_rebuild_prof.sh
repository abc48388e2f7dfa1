# rebuild kernels: lbvh parity tests, bench frame-only numbers, ncu --set full of the warm and
# cold rebuild kernels (dev tool)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_scale.py -k "lbvh or random or blobs64 or config3_1024_indices" -m gpu -q -p no:cacheprovider > gpurun_out/pytest_lbvh.log 2>&1
tail -2 gpurun_out/pytest_lbvh.log
timeout 400 python bench.py --no-cpu --frame-only > gpurun_out/bench_fo.json 2> gpurun_out/bench_fo.err
python -c "import json; d=json.load(open('gpurun_out/bench_fo.json')); print(d['value'], d['e2e']['value'], {k: v for k, v in d['build'].items() if not isinstance(v, str)})"
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"k_flags_tiles|k_tree_chunk|k_leaves_coop|k_tile_scan|k_tree_cross|k_brick_summary" -s 40 -c 12 \
  -o gpurun_out/rebuild_full python bench.py --steps 2 --warmup 3 --no-cpu --frame-only > /dev/null 2>&1
ls -la gpurun_out/rebuild_full.ncu-rep
