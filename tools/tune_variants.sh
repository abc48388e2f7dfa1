#!/bin/bash
# Time the renderer with several launch-bound variants of libvsb200.so (dev tool).
for f in variants/lib_*.so; do
  echo "== $f"
  VSB200_LIB=$PWD/$f timeout 300 python tools/tune_render2.py 1024 lbvh,grid 0.3,0.0 2>&1 | grep -v "^{"
done
