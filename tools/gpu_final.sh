# final check of the round: the whole GPU suite, smoke, the bench (both arms), a torchrun launch with one rank
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline --incremental-mods 0 > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err; echo torchrun rc=$?
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-hbm-bound --incremental-mods 0 > gpurun_out/bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-hbm-bound --incremental-mods 0 > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
