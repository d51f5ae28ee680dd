# C5 (28 q, 5000 gates) full-simulation time through StateVector under tile settings
run() { echo "$* : $(env $* timeout 600 python tools/prof_pass.py --workload c5 --n 28 --reps 3 2>&1 | grep '"rep": 2' | cut -c1-60)"; }
if [ $# -eq 0 ]; then set -- "QTB_X=0" "QTB_TILE_BITS=12 QTB_LOW_BITS=3" "QTB_TILE_BITS=11 QTB_LOW_BITS=3" \
  "QTB_TILE_BITS=12" "QTB_TILE_BITS=13 QTB_REG_BITS=4 QTB_LOW_BITS=3" "QTB_TILE_BITS=11" "QTB_TILE_BITS=12 QTB_LOW_BITS=2"; fi
for cfg in "$@"; do run $cfg; done
