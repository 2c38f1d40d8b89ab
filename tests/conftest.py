import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libosmpm.so")
    config.addinivalue_line("markers", "slow: long-running oracle physics checks")


GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_golden(name):
    """Rows of a whitespace table, '#' comments skipped; first token kept as str if not numeric."""
    rows = []
    with open(os.path.join(GOLDEN, name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            toks = line.split()
            try:
                rows.append([float(t) for t in toks])
            except ValueError:
                rows.append([toks[0]] + [float(t) for t in toks[1:]])
    return rows
