cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; cat gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -2 gpurun_out/bench.err
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
for k in ['value','ms_per_step','e2e','build','render_by_t','ert','roofline','roofline_warm_vote','clocks']: print(k, json.dumps(d.get(k))[:400])
"
