# ncu of one heavy pass of the default C3 plan: as is, and arithmetic only (no loads / stores)
QTB_JIT=1 python tools/prof_pass.py --reps 2 > gpurun_out/prof_plain2.log 2>&1
QTB_JIT=1 ncu --set full --clock-control none --import-source on -k regex:qtjit -s 14 -c 1 -o gpurun_out/prof_heavy -f python tools/prof_pass.py --reps 2 > gpurun_out/ncu_heavy.log 2>&1; echo rc=$?
QTB_JIT=1 QTB_JIT_DEBUG=12 QTB_JIT_CACHE_DIR=off ncu --set full --clock-control none --import-source on -k regex:qtjit -s 14 -c 1 -o gpurun_out/prof_heavy_compute -f python tools/prof_pass.py --reps 2 > gpurun_out/ncu_heavy_c.log 2>&1; echo rc=$?
cat gpurun_out/prof_plain2.log | cut -c1-300
