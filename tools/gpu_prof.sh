python tools/prof_pass.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_pass -s 40 -c 1 -o gpurun_out/prof_c3_v7 -f python tools/prof_pass.py --reps 2 > gpurun_out/ncu_c3.log 2>&1
echo ncu rc=$?
