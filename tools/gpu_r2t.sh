# direct-store eligibility: how many low physical bits must stay thread bits for the last round to store straight to HBM
run() {
  tag=$1; shift
  env "$@" QTB_JIT=1 python tools/prof_pass.py --reps 4 2>&1 | tail -2 | head -1 | cut -c1-110 | sed "s/^/$tag c3 /"
  env "$@" QTB_JIT=1 python tools/prof_pass.py --workload c5 --n 28 --reps 3 2>&1 | tail -2 | head -1 | cut -c1-110 | sed "s/^/$tag c5 /"
  env "$@" QTB_JIT=1 python tools/prof_pass.py --workload c4 --n 30 --reps 3 2>&1 | tail -2 | head -1 | cut -c1-110 | sed "s/^/$tag c4 /"
}
run d3 QTB_DIRECT_BITS=3
run d2 QTB_DIRECT_BITS=2
run d1 QTB_DIRECT_BITS=1
run d4 QTB_DIRECT_BITS=4
run d3 QTB_DIRECT_BITS=3
