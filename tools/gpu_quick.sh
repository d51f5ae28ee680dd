set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python tools/prof_pass.py --reps 2 2>&1 | tail -3
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench rc=$?
tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
