set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo bench rc=$?
tail -3 gpurun_out/bench_r2a.err
python -c "
import json;d=json.load(open('gpurun_out/bench_r2a.json'))
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('roofline_fp64'), d.get('interpreted'))"
