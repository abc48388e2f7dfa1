# render variants: timing (median of 5 x 10 frames) + ncu launch list per variant (dev tool)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
KINDS=${KINDS:-lbvh,grid} TS=${TS:-0.6,0.3,0.0} bash tools/tune_variants.sh > gpurun_out/variants.txt 2>&1
for f in variants/lib_*.so; do
  n=$(basename $f .so)
  VSB200_LIB=$PWD/$f timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k regex:"k_segments|k_integrate" --log-file gpurun_out/launch_$n.csv python tools/prof_render.py 1024 ${PKIND:-lbvh} 0.3 32 > /dev/null 2>&1
  echo "== $n"; python tools/launch_summary.py gpurun_out/launch_$n.csv | head -5
done >> gpurun_out/variants.txt
cat gpurun_out/variants.txt
