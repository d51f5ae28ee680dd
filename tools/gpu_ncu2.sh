# ncu --set full of tile passes of C3 under env settings: usage
#   bash tools/gpu_ncu2.sh TAG SKIP "ENV=.. ENV=.." [TAG SKIP "ENV" ...]
# (kernel regex: tile_pass or, with QTB_JIT=1, the compiled qtjit passes)
mkdir -p gpurun_out
while [ $# -ge 3 ]; do
  TAG=$1; S=$2; E=$3; shift 3
  K=tile_pass; case "$E" in *QTB_JIT=1*) K=qtjit;; esac
  env $E python tools/prof_pass.py --workload c3 --n 30 --reps 1 2>&1 | tail -1 | cut -c1-60
  env $E timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -s $S -c 1 \
    -o gpurun_out/prof_$TAG -f python tools/prof_pass.py --workload c3 --n 30 --reps 1 > gpurun_out/ncu_$TAG.log 2>&1
  echo ncu $TAG rc=$?
done
