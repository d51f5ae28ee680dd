# TMA bulk stores in the ring kernel: parity first, then timing against the st.global path
QTB_JIT_TMA=2 python tools/ring_check.py 20 24 26 2>&1 | tail -4
QTB_JIT_TMA=2 timeout 900 python -m pytest tests/test_jit.py tests/test_gpu_state.py -x -q -m gpu 2>&1 | tail -3
run() {
  tag=$1; shift
  env "$@" QTB_JIT=1 python tools/prof_pass.py --reps 3 2>&1 | tail -2 | cut -c1-400 | sed "s/^/$tag /"
  env "$@" QTB_JIT=1 python tools/prof_pass.py --workload c5 --n 28 --reps 3 2>&1 | tail -2 | head -1 | cut -c1-120 | sed "s/^/$tag /"
}
run base QTB_JIT_TMA=0
run tma QTB_JIT_TMA=2
run base QTB_JIT_TMA=0
run tma QTB_JIT_TMA=2
