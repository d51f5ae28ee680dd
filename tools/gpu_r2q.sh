timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_topk.py tests/test_jit.py -x -q -m gpu 2>&1 | tail -5
