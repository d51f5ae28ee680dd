python tools/ring_check.py 24 28 > gpurun_out/rc.log 2>&1; tail -2 gpurun_out/rc.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --incremental-mods 0 > gpurun_out/b.json 2> gpurun_out/b.err
python -c "
import json;d=json.load(open('gpurun_out/b.json'))
print('c3', d['value'], d['ms_per_step'], d['config']['passes_per_step'], d['roofline']['frac'], d['roofline_fp64']['frac'], d['check'], d['clocks']['sm_mhz'])"
QTB_JIT=1 python tools/prof_pass.py --workload c5 --n 28 --reps 2 | tail -2 | cut -c1-200
python tools/c5_hybrid.py --mods 16 --modes 0 | cut -c1-500
