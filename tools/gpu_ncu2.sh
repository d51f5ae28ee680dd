mkdir -p gpurun_out
python tools/prof_pass.py --workload c3 --n 30 --reps 2 2>&1 | tail -1 | cut -c1-100
for S in 0 8; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_pass -s $S -c 1 \
  -o gpurun_out/prof_s$S -f python tools/prof_pass.py --workload c3 --n 30 --reps 1 > gpurun_out/ncu_s$S.log 2>&1
echo ncu $S rc=$?
done
