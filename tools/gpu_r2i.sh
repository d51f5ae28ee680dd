# L2 policy experiments for the ring kernel's stores / loads
run() {
  tag=$1; shift
  env "$@" QTB_JIT=1 python tools/prof_pass.py --reps 3 2>&1 | tail -2 | cut -c1-400 | sed "s/^/$tag /"
  env "$@" QTB_JIT=1 python tools/prof_pass.py --workload c5 --n 28 --reps 3 2>&1 | tail -2 | head -1 | cut -c1-120 | sed "s/^/$tag /"
}
run base QTB_JIT_STPOL=0 QTB_JIT_LDPOL=0
run st1 QTB_JIT_STPOL=1 QTB_JIT_LDPOL=0
run ld1 QTB_JIT_STPOL=0 QTB_JIT_LDPOL=1
run st1ld1 QTB_JIT_STPOL=1 QTB_JIT_LDPOL=1
run st2ld1 QTB_JIT_STPOL=2 QTB_JIT_LDPOL=1
run base QTB_JIT_STPOL=0 QTB_JIT_LDPOL=0
