# full GPU test suite + smoke + k-d timings (dev tool)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/time_kd.py 512 1024 > gpurun_out/time_kd_dev.txt 2>&1
