import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


# the host max-flow's threaded component path on small graphs too (read once
# per process by the library; the result does not depend on it)
os.environ.setdefault("IRLS_MAXFLOW_PAR_MIN", "1000")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running full-size case")
