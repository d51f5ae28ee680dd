python tools/fused_exchange_bench.py --n 30 --world 8 2>&1 | tail -2
python tools/fused_exchange_bench.py --n 30 --world 2 2>&1 | tail -2
