# bench line + launch list + one ncu --set full of a compiled C3 pass
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -2 gpurun_out/bench.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --incremental-mods 0 > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --incremental-mods 0 > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
QTB_JIT=1 python tools/prof_pass.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
QTB_JIT=1 ncu --set full --clock-control none --import-source on -k regex:qtjit -s 28 -c 1 -o gpurun_out/prof_full -f python tools/prof_pass.py --reps 2 > gpurun_out/ncu_full.log 2>&1; echo ncufull rc=$?
