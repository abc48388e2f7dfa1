# launch lists of k-d builds (dev tool): bash tools/kdprof.sh "N kind t" ...
i=0
for a in "$@"; do
  i=$((i+1))
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kd_launch_$i.csv python tools/prof_kd.py $a > gpurun_out/kd_launch_$i.log 2>&1
done
