# planner variants on C3: beam width and reserved low bits (run length), compiled mode
run() {
  tag=$1; shift
  env "$@" QTB_JIT=1 python tools/prof_pass.py --reps 4 2>&1 | tail -2 | cut -c1-330 | sed "s/^/$tag /"
}
run base QTB_WINDOW_SEARCH=1
run beam16 QTB_WINDOW_SEARCH=1 QTB_WINDOW_BEAM=16
run beam64 QTB_WINDOW_SEARCH=1 QTB_WINDOW_BEAM=64
run low3 QTB_WINDOW_SEARCH=1 QTB_LOW_BITS=3
run low3b16 QTB_WINDOW_SEARCH=1 QTB_LOW_BITS=3 QTB_WINDOW_BEAM=16
run low2 QTB_WINDOW_SEARCH=1 QTB_LOW_BITS=2
run low2b16 QTB_WINDOW_SEARCH=1 QTB_LOW_BITS=2 QTB_WINDOW_BEAM=16
run low2b16tma QTB_WINDOW_SEARCH=1 QTB_LOW_BITS=2 QTB_WINDOW_BEAM=16 QTB_JIT_TMA=2
run base QTB_WINDOW_SEARCH=1
