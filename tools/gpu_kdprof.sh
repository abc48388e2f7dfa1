# k_levels phase profile (dev tool): VSB200_KD_PROFILE=1 prints per-phase device timestamps.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; rm -f gpurun_out/kd_prof.txt
for c in "512 kd-deep-mls32 0.6" "1024 kd-shallow 0.6" ${EXTRA_CONFIGS}; do
  echo "== $c" >> gpurun_out/kd_prof.txt
  VSB200_KD_PROFILE=1 timeout 300 python tools/prof_kd.py $c >> gpurun_out/kd_prof.txt 2>&1
done
