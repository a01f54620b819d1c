"""The reference's own criterion tests, unchanged, against the shim
(the drop-in boundary).  tools/ref_suite.py aliases
asrkit.criterion to paper_1812_07625_b200.criterion and runs
tests/test_criterion.py, acceptance gates 1 and 6 and the trainer's
sharded-worker tests from the reference package installed in baseline/_ref
(prepared in the build container by `python tools/ref_suite.py prepare`)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.mark.gpu
def test_reference_criterion_suite_passes_unchanged():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(os.path.join(REF, "asrkit")) or not os.path.isdir(
            os.path.join(REF, "reftests")):
        pytest.skip("baseline/_ref not prepared (tools/ref_suite.py prepare)")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ref_suite.py"), "run"],
                         capture_output=True, text=True, timeout=1200)
    tail = "\n".join(res.stdout.splitlines()[-25:])
    assert res.returncode == 0, tail
