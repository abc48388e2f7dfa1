# render A/B: parity tests with the default build + timing and launch lists per variant (dev tool)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_render.py tests/test_gpu_scale.py -k "render or frame or brick or 1080p" -m gpu -q -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1
tail -2 gpurun_out/pytest_ab.log
KINDS=${KINDS:-lbvh,grid} TS=${TS:-0.6,0.3,0.0} bash tools/tune_variants.sh
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  VSB200_LIB=$PWD/$f timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:"k_segments|k_integrate" --log-file gpurun_out/launch_$n.csv python tools/prof_render.py 1024 lbvh 0.3 32 > /dev/null 2>&1
  echo "== $n"; python tools/launch_summary.py gpurun_out/launch_$n.csv | head -4
done
