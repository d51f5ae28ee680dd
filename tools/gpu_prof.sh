export QTB_REG_BITS=3 QTB_TILE_BITS=10
python tools/microbench.py > gpurun_out/mb_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tile_pass -s 2 -c 1 -o gpurun_out/prof_mb -f python tools/microbench.py > gpurun_out/ncu_mb.log 2>&1
echo ncu rc=$?
