python tools/prof_pass.py --reps 3 2>&1 | tail -2 | cut -c1-300
python tools/prof_pass.py --workload c5 --n 28 --reps 2 2>&1 | tail -2 | cut -c1-100
timeout 900 python -m pytest tests/test_gpu_state.py tests/test_gpu_golden.py tests/test_gpu_group.py -x -q -m gpu 2>&1 | tail -2
python tools/ring_check.py 24 26 2>&1 | tail -2
