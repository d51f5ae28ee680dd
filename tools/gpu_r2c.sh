python tools/tilebits_bench.py > gpurun_out/tilebits.log 2>&1
QTB_JIT=1 python tools/prof_pass.py --reps 2 > gpurun_out/pp.log 2>&1 && \
QTB_JIT=1 ncu --set full --clock-control none --import-source on -k regex:qtjit -s 22 -c 1 -o gpurun_out/r2_pass0 python tools/prof_pass.py --reps 2 > gpurun_out/ncu0.log 2>&1
QTB_JIT=1 ncu --set full --clock-control none --import-source on -k regex:qtjit -s 38 -c 1 -o gpurun_out/r2_pass16 python tools/prof_pass.py --reps 2 > gpurun_out/ncu16.log 2>&1
ls -la gpurun_out
