cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"k_integrate_multi" -c 1 -o gpurun_out/multi_src \
  python bench.py --channels 4 --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
ls -la gpurun_out/multi_src.ncu-rep
