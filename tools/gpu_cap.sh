for cap in 186 180 0; do
QTB_PASS_FP64=$cap timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cap$cap.json 2> gpurun_out/bench_cap$cap.err
python -c "
import json;d=json.load(open('gpurun_out/bench_cap$cap.json'))
print('cap$cap', d['value'], d['ms_per_step'], d['config']['passes_per_step'], d['roofline']['frac'], d['roofline_fp64']['frac'], d['clocks'])"
done
QTB_PASS_FP64=186 QTB_JIT=1 python tools/prof_pass.py --reps 2 | tail -2
