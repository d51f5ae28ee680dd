for kp in 1 0; do
QTB_JIT_KPARAM=$kp timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_kp$kp.json 2> gpurun_out/bench_kp$kp.err
python -c "
import json;d=json.load(open('gpurun_out/bench_kp$kp.json'))
print('kp$kp', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline_fp64']['frac'], d['clocks'])"
QTB_JIT_KPARAM=$kp QTB_JIT=1 python tools/prof_pass.py --reps 2 | tail -2
done
