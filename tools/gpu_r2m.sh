# default path after the two-phase plan search: parity + bench
timeout 900 python -m pytest tests/test_jit.py tests/test_gpu_state.py tests/test_gpu_golden.py -x -q -m gpu 2>&1 | tail -2
python tools/ring_check.py 24 30 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --incremental-mods 0 > gpurun_out/b_default.json 2> gpurun_out/b_default.err
python -c "
import json;d=json.load(open('gpurun_out/b_default.json'))
print('c3', d['value'], d['ms_per_step'], d['config']['passes_per_step'], d['roofline']['frac'], d['roofline_fp64']['frac'], d['check'], d['clocks'], d['compile'])"
QTB_JIT=1 python tools/prof_pass.py --workload c5 --n 28 --reps 3 2>&1 | tail -2 | cut -c1-200
QTB_JIT=1 python tools/prof_pass.py --workload c4 --n 30 --reps 3 2>&1 | tail -2 | cut -c1-300
