# Correctness (pytest -m gpu) then an A/B sweep of tile-pass settings on C3
# (30 q). usage: bash tools/gpu_pipe_sweep.sh ["ENV=.. ENV2=.." ...]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
run() { echo "$* : $(env $* timeout 300 python tools/prof_pass.py --workload c3 --n 30 --reps 3 2>&1 | grep '"rep": 2' | cut -c1-60)"; }
if [ $# -eq 0 ]; then set -- "QTB_X=0" "QTB_PF=1" "QTB_PIPE=1" "QTB_TILE_BITS=12 QTB_LOW_BITS=3" \
  "QTB_TILE_BITS=11 QTB_LOW_BITS=3" "QTB_TILE_BITS=13 QTB_LOW_BITS=3 QTB_REG_BITS=4" \
  "QTB_TILE_BITS=12 QTB_LOW_BITS=3 QTB_REG_BITS=4" "QTB_TILE_BITS=11 QTB_LOW_BITS=3 QTB_REG_BITS=4 QTB_PIPE=1"; fi
for cfg in "$@"; do run $cfg; done
