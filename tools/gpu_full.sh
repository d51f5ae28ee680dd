python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/gputest.log
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench rc=$? $(( $(date +%s) - t0 ))s
python -c "
import json;d=json.load(open('gpurun_out/bench_full.json'))
print(d['value'], d['ms_per_step'], d['config']['passes_per_step'], d['roofline']['frac'], d['roofline_fp64'], d['e2e'], d['check'], d['clocks'], d['compile'])
print(json.dumps(d.get('incremental'))[:1500])"
