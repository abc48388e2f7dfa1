# Binned k-d check on one B200 (dev tool): parity tests, then per-variant build timings / breakdowns.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kdtree.py tests/ref_suite/test_ref_kdtree.py tests/test_gpu_build.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/binned_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -m gpu -p no:cacheprovider -k "config2 or config3" 2>&1 | tail -5 >> gpurun_out/binned_tests.log
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/binned_time.txt
  KINDS=kd-binned-mls32 VSB200_LIB=$PWD/$f timeout 300 python tools/time_kd.py 512 1024 >> gpurun_out/binned_time.txt 2>&1
done
N=1024 KINDS=kd-binned-mls32 TS="0.6 0.0" TOP=10 bash tools/kd_variants.sh > gpurun_out/binned_variants.txt 2>&1
