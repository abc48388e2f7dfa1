# LBVH rebuild variants: warm / cold rebuild ms via bench --frame-only (dev tool)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for f in variants/lib_*.so; do echo "== $f"; VSB200_LIB=$PWD/$f timeout 400 python bench.py --no-cpu --frame-only --steps 32 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['build']; print(d['value'], b['warm_ms'], b['cold_ms'], b['roofline_frac_cold'], d['parity_index_vs_public_api'], d['roofline_warm_vote']['ms'], d['roofline_warm_vote']['frac'])"; done
