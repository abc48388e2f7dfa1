# Packed cell-slab pass depth A/B on one B200 (dev tool).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/cu_time.txt
  KINDS="kd-binned-mls32" VSB200_LIB=$PWD/$f timeout 300 python tools/time_kd.py 512 1024 >> gpurun_out/cu_time.txt 2>&1
  VSB200_LIB=$PWD/$f timeout 300 python tools/kd_breakdown.py 1024 kd-binned-mls32 0.6 0 2>&1 | grep -E "wall|span|slabs" >> gpurun_out/cu_time.txt
done
