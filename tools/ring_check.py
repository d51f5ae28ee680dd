"""Compiled passes vs the interpreter on the same plan (bit-identical by
design): max |diff| and norms at several sizes. QTB_JIT_RING selects the
compiled kernel variant."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_01076_b200 import StateVector, workloads as W

for n in [int(x) for x in (sys.argv[1:] or ["22", "26", "28"])]:
    w = W.config3(n=n, layers=20)
    res = {}
    for compiled in (False, True):
        st = StateVector(n, compiled=compiled)
        st.apply(w.gates)
        st.apply(w.gates)  # the second run uses the cached compiled passes
        nrm = st.norm_squared()
        idx = np.random.default_rng(1).integers(0, 1 << n, size=1 << 16)
        idx.sort()
        amps = st.read() if n <= 26 else np.concatenate([st.read(int(i), 1) for i in idx[:64]])
        res[compiled] = (nrm, amps)
        st.close()
    d = np.abs(res[True][1] - res[False][1]).max()
    print(f"n={n} ring={os.environ.get('QTB_JIT_RING', '1')} norm interp {res[False][0]!r} compiled {res[True][0]!r} "
          f"max|compiled-interp|={d:.3e} bitwise={bool((res[True][1] == res[False][1]).all())}", flush=True)
