# ncu --set full of one mid-circuit tile pass (skip $SKIP launches) of workload
# $WL (default c3) at $N qubits -> gpurun_out/prof_iter.ncu-rep
set -x
mkdir -p gpurun_out
WL=${WL:-c3}; N=${N:-30}
python tools/prof_pass.py --workload $WL --n $N --reps 2 2>&1 | tail -2 | cut -c1-200
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_pass -s ${SKIP:-8} -c 1 \
  -o gpurun_out/prof_iter -f python tools/prof_pass.py --workload $WL --n $N --reps 1 > gpurun_out/ncu_iter.log 2>&1
echo ncu rc=$?
