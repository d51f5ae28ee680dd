python - <<'PY'
import sys, json, time
sys.path.insert(0, '.')
from bench import measure_incremental
from paper_2210_01076_b200 import Config, Simulator, workloads as W, jit_stats
w = W.config5(nmods=300)
r = measure_incremental(lambda n: Simulator(n, Config()), w, 300)
print(json.dumps({"uniform": r["uniform"], "tail": r["tail"], "jit": jit_stats()}))
PY
