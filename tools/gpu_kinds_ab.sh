cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
KINDS=lbvh,grid,hybrid,naive,kd-binned-mls32 TS=0.3,0.0 bash tools/tune_variants.sh
