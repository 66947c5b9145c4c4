import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# The library runs tiny grids (<= 2048 elements at p <= 8, <= 256 above) on the one-launch v1
# kernel; the parity tests use small grids, so they disable that switch to exercise the fast
# kernels (tests that want the small-grid path re-enable it).
os.environ.setdefault("SC_SMALL_V1", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libsc.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_golden(name):
    """Parse 'key = value' lines (value a python expression of fractions / floats)."""
    from fractions import Fraction  # noqa: F401  (available to eval)
    import math  # noqa: F401
    out = {}
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, v = line.split("=", 1)
            out[k.strip()] = eval(v.strip(), {"Fraction": Fraction, "math": math, "__builtins__": {}})
    return out
