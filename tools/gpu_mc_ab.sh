cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in variants/lib_*.so; do echo "== $f"; VSB200_LIB=$PWD/$f timeout 300 python tools/time_mc.py 2>&1 | tail -3; done
