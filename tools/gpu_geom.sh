# C5 full simulation (28 q) per geometry: interpreter R3/R4, compiled R3/R4 (ring)
run() { echo "$* : $(env $* timeout 600 python tools/prof_pass.py --workload c5 --n 28 --reps 3 2>&1 | grep '"rep": 2' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["passes"], round(d["wall_ms"],1), round(sum(d["pass_ms"])/len(d["pass_ms"]),3))')"; }
run QTB_JIT=0 QTB_TILE_BITS=12 QTB_REG_BITS=3 QTB_LOW_BITS=3
run QTB_JIT=0 QTB_TILE_BITS=12 QTB_REG_BITS=4 QTB_LOW_BITS=4
run QTB_JIT=0 QTB_TILE_BITS=12 QTB_REG_BITS=4 QTB_LOW_BITS=3
run QTB_JIT=1 QTB_TILE_BITS=12 QTB_REG_BITS=3 QTB_LOW_BITS=3
run QTB_JIT=1 QTB_TILE_BITS=12 QTB_REG_BITS=4 QTB_LOW_BITS=3
run QTB_JIT=1 QTB_TILE_BITS=12 QTB_REG_BITS=4 QTB_LOW_BITS=4
run QTB_JIT=1 QTB_TILE_BITS=12 QTB_REG_BITS=4 QTB_LOW_BITS=4 QTB_PLAN_SEARCH=0
