# k-d / hybrid build diagnostics on one B200 (dev tool): per-kernel breakdowns and k_levels phase profiles.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in "1024 kd-binned-mls32 0.0" "1024 kd-binned-mls32 0.6" "1024 hybrid 0.6" "512 kd-deep-mls32 0.0" "512 kd-deep-mls32 0.3"; do
  echo "== $c" >> gpurun_out/kd_breakdown.txt
  timeout 300 python tools/kd_breakdown.py $c 60 >> gpurun_out/kd_breakdown.txt 2>&1
done
for c in "1024 hybrid 0.6" "512 kd-deep-mls32 0.0" "512 kd-deep-mls32 0.3"; do
  echo "== $c" >> gpurun_out/kd_prof.txt
  VSB200_KD_PROFILE=1 timeout 300 python tools/prof_kd.py $c >> gpurun_out/kd_prof.txt 2>&1
done
