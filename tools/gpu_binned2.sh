# Binned level loop check on one B200 (dev tool): k-d parity tests, timings, one timeline.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kdtree.py tests/ref_suite/test_ref_kdtree.py tests/test_gpu_build.py -q -x -m gpu -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/b2_tests.log
timeout 900 python -m pytest tests/test_gpu_scale.py -q -x -m gpu -p no:cacheprovider -k "config2 or config3" 2>&1 | tail -3 >> gpurun_out/b2_tests.log
KINDS="kd-binned-mls32" timeout 300 python tools/time_kd.py 512 1024 > gpurun_out/b2_time.txt 2>&1
timeout 300 python tools/kd_breakdown.py 1024 kd-binned-mls32 0.6 80 > gpurun_out/b2_timeline.txt 2>&1
