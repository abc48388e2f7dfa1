set -x
for a in "1024 kd-shallow 0.6" "512 kd-deep-mls32 0.3" "512 kd-binned-mls32 0.6" "512 kd-binned-mls32 0.3" "1024 hybrid 0.3"; do
  python tools/prof_kd.py $a
  python tools/prof_kd.py $a
done > gpurun_out/kd_wall.log 2>&1
i=0
for a in "1024 kd-shallow 0.6" "512 kd-deep-mls32 0.3" "512 kd-binned-mls32 0.6"; do
  i=$((i+1))
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kd_launch_$i.csv python tools/prof_kd.py $a > /dev/null 2>&1
done
