timeout 1200 python -m pytest tests/test_gpu_group.py -x -q -m gpu 2>&1 | tail -8
python tools/c4_group_check.py --compiled 1 --worlds 8 --n 30 2>&1 | cut -c1-600 | tail -3
QTB_FUSE_EXCHANGE=0 python tools/c4_group_check.py --compiled 1 --worlds 8 --n 30 2>&1 | cut -c1-600 | tail -1
