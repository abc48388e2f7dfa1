# k_subtrees hand-off size A/B on one B200 (dev tool): per-variant k-d timings and subtree stats.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in variants/lib_*.so; do
  echo "== $f" >> gpurun_out/sw_time.txt
  KINDS="kd-deep-mls32 kd-deep-mls128 kd-shallow" VSB200_LIB=$PWD/$f timeout 300 python tools/time_kd.py 512 >> gpurun_out/sw_time.txt 2>&1
  for t in 0.6 0.0; do
    VSB200_LIB=$PWD/$f VSB200_KD_PROFILE=1 timeout 300 python tools/prof_kd.py 512 kd-deep-mls32 $t 2>&1 | grep "k_subtrees\|k_levels" >> gpurun_out/sw_time.txt
  done
done
