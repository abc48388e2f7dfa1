# Binned narrow-level decision width A/B on one B200 (dev tool): parity of each variant, timings.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/wpn_time.txt
  VSB200_LIB=$PWD/$f timeout 600 python -m pytest tests/test_gpu_kdtree.py -q -x -m gpu -p no:cacheprovider -k binned 2>&1 | tail -1 >> gpurun_out/wpn_time.txt
  KINDS="kd-binned-mls32" VSB200_LIB=$PWD/$f timeout 300 python tools/time_kd.py 512 1024 >> gpurun_out/wpn_time.txt 2>&1
done
