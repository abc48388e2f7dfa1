cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in variants/lib_*.so; do echo "== $f"; VSB200_LIB=$PWD/$f timeout 600 python tools/time_kd.py ${SIZES:-512 1024} 2>&1 | grep -v "^$"; done
