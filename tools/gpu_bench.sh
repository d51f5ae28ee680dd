for cfg in "3 10" "3 11" "4 11" "4 12" "3 9"; do set -- $cfg; echo "R=$1 K=$2 $(QTB_REG_BITS=$1 QTB_TILE_BITS=$2 python tools/prof_pass.py --reps 2 2>&1 | tail -2 | head -1 | cut -c1-50)"; done
QTB_REG_BITS=3 QTB_TILE_BITS=10 python tools/microbench.py 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
