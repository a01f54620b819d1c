import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


_KAT = None


def load_kat():
    global _KAT
    if _KAT is None:
        with open(os.path.join(GOLDEN, "kat_small.json")) as f:
            _KAT = json.load(f)
    return _KAT


def load_npz(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture
def cuda():
    if not gpu_available():
        pytest.skip("no CUDA device")
    import torch
    return torch.device("cuda:0")


class TokenTable:
    """Minimal token table for the tests (the criterion path duck-types the
    table: len(), rep_id and symbol(); the reference's TokenTable,
    lexicon.py:20-59, provides the same)."""

    def __init__(self, symbols):
        self.symbols = list(symbols)
        self.ids = {s: i for i, s in enumerate(self.symbols)}

    def __len__(self):
        return len(self.symbols)

    def symbol(self, i):
        return self.symbols[i]

    @property
    def rep_id(self):
        return self.ids.get("<2>")
