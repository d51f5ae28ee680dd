# kernel experiments: tile shrinking (smaller tiles for passes whose low bits are idle)
run() {
  tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --incremental-mods 0 > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err
  python -c "
import json;d=json.load(open('gpurun_out/b_$tag.json'))
print('$tag c3', d['ms_per_step'], d['config']['passes_per_step'], d['roofline']['frac'], d['roofline_fp64']['frac'], d['check'], d['clocks']['sm_mhz'])"
  env "$@" QTB_JIT=1 python tools/prof_pass.py --reps 3 | tail -2 | cut -c1-400
  env "$@" QTB_JIT=1 python tools/prof_pass.py --workload c5 --n 28 --reps 3 | tail -2 | cut -c1-700
}
run s10r2 QTB_SHRINK_MIN=10 QTB_SHRINK_RUN=2
run s10r3 QTB_SHRINK_MIN=10 QTB_SHRINK_RUN=3
run s11r2 QTB_SHRINK_MIN=11 QTB_SHRINK_RUN=2
run s9r1 QTB_SHRINK_MIN=9 QTB_SHRINK_RUN=1
QTB_SHRINK_MIN=10 timeout 900 python -m pytest tests/test_jit.py tests/test_gpu_state.py tests/test_gpu_sim.py -x -q -m gpu 2>&1 | tail -5
