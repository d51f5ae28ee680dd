# timing ablations of the ring kernel on C3 (results are garbage by design): what do
# the stores / loads / arithmetic cost, alone and together?
run() {
  tag=$1; shift
  env "$@" QTB_JIT=1 QTB_JIT_CACHE_DIR=off python tools/prof_pass.py --reps 3 2>&1 | tail -2 | head -1 | cut -c1-400 | sed "s/^/$tag /"
}
run base QTB_JIT_DEBUG=0
run nost QTB_JIT_DEBUG=4
run nold QTB_JIT_DEBUG=8
run nofp QTB_JIT_DEBUG=16
run nost_nold QTB_JIT_DEBUG=12
run nofp_nost QTB_JIT_DEBUG=20
run nofp_nold QTB_JIT_DEBUG=24
run base2 QTB_JIT_DEBUG=0
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv
