cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"${KRE:-k_integrate_segments}" -c ${NCAP:-1} -o gpurun_out/integ_src python tools/prof_render.py 1024 ${KIND:-lbvh} 0.3 32 > /dev/null 2>&1
ls -la gpurun_out/integ_src.ncu-rep
