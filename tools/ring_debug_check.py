"""Prints a digest of compiled-pass results (C3 family at 21 qubits and C5
family at 20 qubits through the ring kernel, with >= 4 tiles per CTA so the
ring reaches its steady state) -- run under QTB_JIT_DEBUG=1 (bounds-checked
kernels: a violation raises), =2 (the two consumer groups skewed by random
sleeps) and =0; the digests must be identical (tests/test_gpu_debug.py).
compute-sanitizer is closed on this GPU pool; these builds stand in for
memcheck (bounds) and racecheck (interleaving perturbation)."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_01076_b200 import StateVector, workloads as W  # noqa: E402

h = hashlib.sha256()
for w in (W.config3(n=21, layers=6), W.config5(n=20, ngates=600, nmods=0)):
    for rep in range(2):
        st = StateVector(w.n, compiled=True)
        st.apply(w.gates)
        h.update(st.read().tobytes())
        st.close()
print(h.hexdigest())
