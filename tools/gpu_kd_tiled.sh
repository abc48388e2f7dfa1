# k-d device level loop A/B on one B200 (dev tool): parity tests, then per-variant timings.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kdtree.py tests/ref_suite/test_ref_kdtree.py tests/ref_suite/test_ref_hybrid.py tests/test_gpu_build.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/tiled_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -m gpu -p no:cacheprovider -k "config2 or config3" 2>&1 | tail -5 >> gpurun_out/tiled_tests.log
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/tiled_time.txt
  KINDS="kd-shallow kd-deep-mls32 kd-deep-mls128 hybrid" VSB200_LIB=$PWD/$f timeout 300 python tools/time_kd.py 512 1024 >> gpurun_out/tiled_time.txt 2>&1
done
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/tiled_prof.txt
  VSB200_LIB=$PWD/$f VSB200_KD_PROFILE=1 timeout 300 python tools/prof_kd.py 1024 hybrid 0.6 2>&1 | grep "k_levels" >> gpurun_out/tiled_prof.txt
  VSB200_LIB=$PWD/$f VSB200_KD_PROFILE=1 timeout 300 python tools/prof_kd.py 512 kd-deep-mls32 0.3 2>&1 | grep "k_levels" >> gpurun_out/tiled_prof.txt
done
