#!/bin/bash
# Time the renderer with several build variants of libvsb200.so (dev tool).
for f in variants/lib_*.so; do
  echo "== $f"
  VSB200_LIB=$PWD/$f timeout 300 python tools/time_render.py 1024 ${KINDS:-lbvh,grid} ${TS:-0.6,0.3,0.0} 1 2>&1
done
