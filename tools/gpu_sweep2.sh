# Timing sweep on the GPU box (prof_pass wall ms of one full simulation, 3rd rep).
# usage: bash tools/gpu_sweep2.sh ["ENV=.. wl n" ...]; default: c3 / c5 / c4
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
run() { echo "$1 $2 n=$3: $(env $2 timeout 300 python tools/prof_pass.py --workload $1 --n $3 --reps 3 2>&1 | grep '"rep": 2' | cut -c1-48)"; }
if [ $# -eq 0 ]; then set -- "c3 QTB_X=0 30" "c5 QTB_X=0 28" "c4 QTB_X=0 30"; fi
for cfg in "$@"; do run $cfg; done
