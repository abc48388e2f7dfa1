cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu_kdprof.sh
for c in "512 kd-deep-mls32 0.6" "512 kd-deep-mls32 0.0" "1024 hybrid 0.6"; do
  n=$(echo $c | tr ' ' '_')
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_$n.csv python tools/prof_kd.py $c > /dev/null 2>&1
done
