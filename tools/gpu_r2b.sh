set -x
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
for ring in 1 0; do
QTB_JIT_RING=$ring timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ring$ring.json 2> gpurun_out/bench_ring$ring.err; echo bench rc=$?
tail -3 gpurun_out/bench_ring$ring.err
python -c "
import json;d=json.load(open('gpurun_out/bench_ring$ring.json'))
print('ring$ring', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline_fp64']['frac'], d['e2e']['value'])"
done
QTB_JIT=1 python tools/prof_pass.py --reps 2 2>&1 | tail -3
