# k_classify_pack A/B on one B200 (dev tool): parity tests, then per-variant kernel times.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_build.py tests/test_gpu_kdtree.py tests/ref_suite/test_ref_volume.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/cp_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -m gpu -p no:cacheprovider -k "config3" 2>&1 | tail -3 >> gpurun_out/cp_tests.log
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/cp_time.txt
  for t in 0.6 0.0; do
    VSB200_LIB=$PWD/$f timeout 300 python tools/kd_breakdown.py 1024 hybrid $t 0 2>&1 | grep -E "wall|classify" >> gpurun_out/cp_time.txt
  done
  KINDS="kd-shallow hybrid" VSB200_LIB=$PWD/$f timeout 300 python tools/time_kd.py 1024 >> gpurun_out/cp_time.txt 2>&1
done
