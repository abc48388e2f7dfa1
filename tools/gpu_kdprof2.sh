# k-d builder breakdown (dev tool): device-loop phase profile + launch lists
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in "512 kd-deep-mls32 0.3" "512 kd-deep-mls32 0.0" "1024 hybrid 0.6" "1024 kd-binned-mls32 0.3"; do
  set -- $cfg
  echo "== $cfg" >> gpurun_out/kdprof.txt
  VSB200_KD_PROFILE=1 timeout 300 python tools/prof_kd.py $1 $2 $3 >> gpurun_out/kdprof.txt 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_kd_$1_$2_$3.csv python tools/prof_kd.py $1 $2 $3 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/launches_kd_$1_$2_$3.csv >> gpurun_out/kdprof.txt
done
cat gpurun_out/kdprof.txt
