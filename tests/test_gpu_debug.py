"""Debug builds of the compiled ring kernel (csrc/qt_jit.cpp QTB_JIT_DEBUG):
compute-sanitizer is closed on this GPU pool, so memory safety and the
cross-group synchronisation are checked by instrumented kernels instead --
every shared / global index range-checked (bit 0), and the two consumer
groups perturbed by pseudo-random sleeps (bit 1). The state must come out
bit-identical to the production kernels and no check may fire."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def digest(debug):
    env = dict(os.environ, QTB_JIT_DEBUG=str(debug))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ring_debug_check.py")],
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr
    return out.stdout.strip().splitlines()[-1]


def test_bounds_checked_and_skewed_ring_kernels_are_bit_identical(gpu):
    base = digest(0)
    assert digest(1) == base  # bounds checks: no violation, same bits
    assert digest(2) == base  # skewed groups: same bits
    assert digest(3) == base
