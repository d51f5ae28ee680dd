# ablations on the window-search plan (13 heavy passes), with SM clock / power sampled under load
run() {
  tag=$1; shift
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 20 > gpurun_out/smi_$tag.csv &
  SMI=$!
  env "$@" QTB_WINDOW_SEARCH=1 QTB_JIT=1 QTB_JIT_CACHE_DIR=off python tools/prof_pass.py --reps 12 2>&1 | tail -2 | head -1 | cut -c1-300 | sed "s/^/$tag /"
  kill $SMI
  python - <<PY
import statistics
rows=[l.strip().split(',') for l in open('gpurun_out/smi_$tag.csv') if ',' in l]
rows=[(float(a),float(b)) for a,b in rows]
hot=[r for r in rows if r[1]>600]
if hot: print('$tag clocks under load: median sm %.0f MHz, median power %.0f W, n=%d' % (statistics.median(r[0] for r in hot), statistics.median(r[1] for r in hot), len(hot)))
else: print('$tag no hot samples', len(rows), max(r[1] for r in rows) if rows else None)
PY
}
run base QTB_JIT_DEBUG=0
run nost QTB_JIT_DEBUG=4
run nold QTB_JIT_DEBUG=8
run nofp QTB_JIT_DEBUG=16
run compute QTB_JIT_DEBUG=12
