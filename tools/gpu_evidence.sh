# Round evidence refresh (GPU box): tests, smoke, bench (+reference arm),
# supplementary configs, QASM + incremental-harness tools, launch list and
# one ncu --set full capture. Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 1200 python tools/bench_configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; echo configs rc=$?
timeout 600 python tools/bench_qasm.py > gpurun_out/qasm.json 2> gpurun_out/qasm.err; echo qasm rc=$?
timeout 900 python tools/bench_incremental.py > gpurun_out/incremental.json 2> gpurun_out/incremental.err; echo incr rc=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
# one compiled pass of C3 (the bench's dominant kernel): the 2nd rep's pass 5 of 10
QTB_JIT=1 python tools/prof_pass.py --reps 2 > gpurun_out/prof_plain.log 2>&1 && \
QTB_JIT=1 ncu --set full --clock-control none --import-source on -k regex:qtjit -s 14 -c 1 -o gpurun_out/prof_full -f python tools/prof_pass.py --reps 2 > gpurun_out/ncu_full.log 2>&1; echo ncufull rc=$?
