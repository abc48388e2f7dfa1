# k_leaf_shrink A/B on one B200 (dev tool): k-d parity tests (default build), per-variant timings.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kdtree.py tests/ref_suite/test_ref_kdtree.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/sh_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -m gpu -p no:cacheprovider -k "config2 or config3" 2>&1 | tail -3 >> gpurun_out/sh_tests.log
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/sh_time.txt
  KINDS="kd-binned-mls32" VSB200_LIB=$PWD/$f timeout 300 python tools/time_kd.py 512 1024 >> gpurun_out/sh_time.txt 2>&1
  VSB200_LIB=$PWD/$f timeout 300 python tools/kd_breakdown.py 1024 kd-binned-mls32 0.0 0 2>&1 | grep -E "shrink" >> gpurun_out/sh_time.txt
done
