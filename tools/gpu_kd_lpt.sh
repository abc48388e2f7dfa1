# k_subtrees launch order A/B on one B200 (dev tool): parity tests, then per-variant timings.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kdtree.py tests/ref_suite/test_ref_kdtree.py tests/test_gpu_build.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/lpt_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -m gpu -p no:cacheprovider -k "config2" 2>&1 | tail -5 >> gpurun_out/lpt_tests.log
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/lpt_time.txt
  KINDS="kd-deep-mls32 kd-deep-mls128" VSB200_LIB=$PWD/$f timeout 300 python tools/time_kd.py 512 >> gpurun_out/lpt_time.txt 2>&1
  for t in 0.6 0.3 0.0; do
    VSB200_LIB=$PWD/$f VSB200_KD_PROFILE=1 timeout 300 python tools/prof_kd.py 512 kd-deep-mls32 $t 2>&1 | grep "k_subtrees\|k_levels" >> gpurun_out/lpt_time.txt
  done
done
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/lpt_breakdown.txt
  VSB200_LIB=$PWD/$f timeout 300 python tools/kd_breakdown.py 512 kd-deep-mls32 0.0 0 2>&1 | grep -v -i warn | head -8 >> gpurun_out/lpt_breakdown.txt
done
