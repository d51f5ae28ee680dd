# Compiled-pass (QTB_JIT=1) correctness + C3 timing sweep.
# usage: bash tools/gpu_jit_sweep.sh [--no-tests] ["ENV=.. ENV=.." ...]
mkdir -p gpurun_out
if [ "$1" = "--no-tests" ]; then shift; else
  QTB_JIT=1 QTB_PIPE=1 QTB_TILE_BITS=11 QTB_LOW_BITS=3 timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
fi
run() {
  tag=$(echo "$*" | tr ' =' '_-')
  env QTB_JIT=1 $* timeout 600 python tools/prof_pass.py --workload c3 --n 30 --reps 3 > gpurun_out/sweep_$tag.log 2>&1
  echo "$* : $(grep -E '"rep": (0|2)' gpurun_out/sweep_$tag.log | cut -c1-48 | tr '\n' ' ')"
}
if [ $# -eq 0 ]; then set -- \
  "QTB_TILE_BITS=11 QTB_LOW_BITS=3 QTB_PIPE=1" \
  "QTB_TILE_BITS=10 QTB_LOW_BITS=3 QTB_PIPE=1" \
  "QTB_TILE_BITS=12 QTB_LOW_BITS=3 QTB_PIPE=1" \
  "QTB_TILE_BITS=11 QTB_LOW_BITS=3 QTB_REG_BITS=4 QTB_PIPE=1" \
  "QTB_TILE_BITS=12 QTB_LOW_BITS=3 QTB_REG_BITS=4 QTB_JIT_MINB=3" \
  "QTB_TILE_BITS=12 QTB_LOW_BITS=3 QTB_REG_BITS=4 QTB_PF=1" \
  "QTB_TILE_BITS=11 QTB_LOW_BITS=3 QTB_PF=1" \
  "QTB_TILE_BITS=12 QTB_LOW_BITS=3 QTB_REG_BITS=4"; fi
for cfg in "$@"; do run $cfg; done
