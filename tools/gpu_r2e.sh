# kernel experiments: early refill of the ring buffers, 2^11 tiles (2 CTAs per SM)
run() {
  tag=$1; shift
  env "$@" timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --incremental-mods 0 > gpurun_out/b_$tag.json 2> gpurun_out/b_$tag.err
  python -c "
import json;d=json.load(open('gpurun_out/b_$tag.json'))
print('$tag c3', d['ms_per_step'], d['config']['passes_per_step'], d['roofline']['frac'], d['roofline_fp64']['frac'], d['check'], d['clocks']['sm_mhz'])"
  env "$@" QTB_JIT=1 python tools/prof_pass.py --reps 3 | tail -2 | cut -c1-400
  env "$@" QTB_JIT=1 python tools/prof_pass.py --workload c5 --n 28 --reps 3 | tail -2 | cut -c1-700
}
run base QTB_JIT_EARLY=0
run early QTB_JIT_EARLY=1
run k11 QTB_JIT_EARLY=1 QTB_TILE_BITS=11
