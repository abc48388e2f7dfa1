#!/bin/bash
# k-d / hybrid build breakdown with several build variants of libvsb200.so (dev tool).
# env: N (1024), KINDS ("kd-binned-mls32"), TS ("0.6 0.0"), TOP (6)
for f in variants/lib_*.so; do
  echo "== $f"
  for kind in ${KINDS:-kd-binned-mls32}; do
    for t in ${TS:-0.6 0.0}; do
      VSB200_LIB=$PWD/$f timeout 300 python tools/kd_breakdown.py ${N:-1024} $kind $t 0 2>&1 | grep -v -i warn | head -${TOP:-6}
    done
  done
done
