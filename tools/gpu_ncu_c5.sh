# ncu --set full of one C5 (28 q, 5000 gates) interpreter pass
mkdir -p gpurun_out
python tools/prof_pass.py --workload c5 --n 28 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_pass -s 40 -c 1 \
  -o gpurun_out/prof_c5 -f python tools/prof_pass.py --workload c5 --n 28 --reps 1 > gpurun_out/ncu_c5.log 2>&1
echo ncu rc=$?
