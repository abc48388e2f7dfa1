# k-d builder check on one B200 (dev tool): tests, then rebuild timings per variant.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kdtree.py tests/test_gpu_build.py tests/ref_suite/test_ref_kdtree.py tests/ref_suite/test_ref_acceptance.py -q -x -m gpu 2>&1 | tail -30 > gpurun_out/kd_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -m gpu -k "config2 or config3_1024_indices" 2>&1 | tail -5 >> gpurun_out/kd_tests.log
for c in "512 kd-deep-mls32 0.6" "512 kd-deep-mls32 0.0" "1024 kd-shallow 0.6" "1024 kd-shallow 0.3"; do
  echo "== $c" >> gpurun_out/kd_prof.txt
  VSB200_KD_PROFILE=1 timeout 300 python tools/prof_kd.py $c >> gpurun_out/kd_prof.txt 2>&1
done
timeout 600 python tools/time_kd.py 512 1024 > gpurun_out/time_kd_dev.txt 2>&1
