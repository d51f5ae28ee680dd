# window search in the planner (fewer, heavier passes on layered circuits)
run() {
  tag=$1; shift
  env "$@" QTB_JIT=1 python tools/prof_pass.py --reps 3 2>&1 | tail -2 | cut -c1-400 | sed "s/^/$tag /"
}
run base QTB_WINDOW_SEARCH=0
run win QTB_WINDOW_SEARCH=1
run win_tma2 QTB_WINDOW_SEARCH=1 QTB_JIT_TMA=2
run win_tma1 QTB_WINDOW_SEARCH=1 QTB_JIT_TMA=1
QTB_WINDOW_SEARCH=1 python tools/ring_check.py 22 26 2>&1 | tail -2
QTB_WINDOW_SEARCH=1 timeout 900 python -m pytest tests/test_jit.py tests/test_gpu_state.py -x -q -m gpu 2>&1 | tail -3
