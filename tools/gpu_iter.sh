# One iteration on the GPU box: gpu tests, C3 timing, a tile/reg sweep, and
# an ncu capture of one mid-circuit pass (prof_iter.ncu-rep).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python tools/prof_pass.py --reps 2 2>&1 | tail -2
for cfg in "3 11" "3 12" "4 12"; do
  set -- $cfg
  echo "R=$1 K=$2 $(QTB_REG_BITS=$1 QTB_TILE_BITS=$2 timeout 300 python tools/prof_pass.py --reps 2 2>&1 | tail -2 | head -1 | cut -c1-60)"
done
QTB_REG_BITS=3 QTB_TILE_BITS=10 timeout 300 python tools/microbench.py 2>&1 | tail -3
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_pass -s 8 -c 1 \
    -o gpurun_out/prof_iter -f python tools/prof_pass.py --reps 1 > gpurun_out/ncu_iter.log 2>&1
  echo ncu rc=$?
fi
