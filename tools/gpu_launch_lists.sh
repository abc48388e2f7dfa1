# Refresh the k-d launch lists on the final tree (dev tool).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_hybrid_1024.csv python tools/prof_kd.py 1024 hybrid 0.3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_kd_deep_512.csv python tools/prof_kd.py 512 kd-deep-mls32 0.3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_kd_binned_1024.csv python tools/prof_kd.py 1024 kd-binned-mls32 0.6 > /dev/null 2>&1
python tools/round_summaries.py ${ROUND:-r02} gpurun_out/summaries > gpurun_out/summaries.log 2>&1
python tools/launch_summary.py gpurun_out/launches_kd_binned_1024.csv > gpurun_out/summaries/r02_launches_kd_binned_mls32_1024.txt 2>&1
cp gpurun_out/launches_kd_binned_1024.csv gpurun_out/summaries/r02_launches_kd_binned_mls32_1024.csv
