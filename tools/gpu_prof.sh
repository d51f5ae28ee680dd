set -x
python tools/prof_pass.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_pass -s 22 -c 2 -o gpurun_out/prof_c3 -f python tools/prof_pass.py --reps 2 > gpurun_out/ncu_c3.log 2>&1
echo ncu rc=$?
tail -5 gpurun_out/ncu_c3.log
cat gpurun_out/prof_plain.log
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
