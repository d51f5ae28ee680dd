# A/B timing on the GPU box: merged layer ops (default) vs QTB_NOLAYER=1,
# on the C3 / C5 / C4 workloads (prof_pass wall ms of one full simulation).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for wl in "c3 30" "c5 28" "c4 30"; do
  set -- $wl
  for env in "" "QTB_NOLAYER=1"; do
    echo "$1 n=$2 [$env] $(env $env timeout 300 python tools/prof_pass.py --workload $1 --n $2 --reps 3 2>&1 | grep '"rep": 2' | cut -c1-48)"
  done
done
