# C5 incremental latency: where does a modifier's time go (trace), hybrid R = 3 vs R = 4
QTB_SIM_TRACE=1 python tools/c5_hybrid.py --mods 8 --modes 0 2> gpurun_out/c5_trace.err | cut -c1-700
grep -c segment gpurun_out/c5_trace.err
tail -60 gpurun_out/c5_trace.err | cut -c1-200
python tools/c5_hybrid.py --mods 24 --modes 0 2>/dev/null | cut -c1-600
QTB_REG_BITS=4 python tools/c5_hybrid.py --mods 24 --modes 0 2>/dev/null | cut -c1-600
