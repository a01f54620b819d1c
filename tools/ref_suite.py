#!/usr/bin/env python
"""Run the reference's OWN criterion tests against this repo's shim.

SURVEY §8(b) defines the drop-in as: the reference tests for this path run
unchanged with ``asrkit.criterion`` aliased to ``paper_1812_07625_b200``'s
criterion module.  Two steps:

    python tools/ref_suite.py prepare   # here (needs /root/reference): installs
                                        # the reference package into
                                        # baseline/_ref and copies its tests
                                        # there (git-ignored; it travels to
                                        # the GPU box with gpurun)
    python tools/ref_suite.py run       # on the GPU box: pytest on the copies

The run aliases ``sys.modules["asrkit.criterion"]`` to the shim before any
reference module imports it (the reference trainer's ``from .criterion
import make_criterion`` then binds the shim), and sets
``W2L_REFERENCE_ERRORS=asrkit.errors`` so the shim raises the reference's own
exception classes.  Nothing else of the reference is replaced: its
autodiff, trainer, lexicon, data and test oracles run as shipped.

Selected tests (the criterion path): tests/test_criterion.py (all),
acceptance gates 1 and 6 (test_acceptance.py:108-176, 411-452) and the
sharded-worker equivalence tests (test_trainer.py:224-242).
"""

from __future__ import annotations

import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"
DST = os.path.join(ROOT, "baseline", "_ref")
TESTS = ["conftest.py", "oracles.py", "test_criterion.py", "test_acceptance.py",
         "test_trainer.py"]
SELECT = ["test_criterion.py",
          "test_acceptance.py::test_1_losses_and_gradients_match_oracles",
          "test_acceptance.py::test_6_worker_gradients_and_resume",
          "test_trainer.py::test_worker_gradients_match_single_worker"]


def prepare() -> None:
    # the reference package, installed unmodified (the one offline install:
    # pip --no-index from a /tmp copy, since the build writes into its tree)
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF, src, ignore=shutil.ignore_patterns("__pycache__"))
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index",
                        "--no-build-isolation", "--find-links", "/opt/wheelhouse", "--no-deps",
                        "--upgrade", "--target", DST, src], check=True)
    tdir = os.path.join(DST, "reftests")
    os.makedirs(tdir, exist_ok=True)
    for name in TESTS:
        shutil.copy(os.path.join(REF, "tests", name), os.path.join(tdir, name))
    print(f"reference package and tests copied to {DST}")


class _AliasPlugin:
    """Installs the aliases before the test modules are collected."""

    def pytest_configure(self, config):  # noqa: D401
        import asrkit
        from paper_1812_07625_b200 import criterion as shim
        sys.modules["asrkit.criterion"] = shim
        asrkit.criterion = shim


def run(extra=()) -> int:
    tdir = os.path.join(DST, "reftests")
    if not os.path.isdir(os.path.join(DST, "asrkit")) or not os.path.isdir(tdir):
        print("baseline/_ref is not prepared (run `python tools/ref_suite.py prepare` where "
              "/root/reference exists)")
        return 2
    os.environ["W2L_REFERENCE_ERRORS"] = "asrkit.errors"
    sys.path[:0] = [ROOT, DST, tdir]
    import pytest
    os.chdir(tdir)
    return pytest.main(["-q", "-p", "no:cacheprovider", *SELECT, *extra],
                       plugins=[_AliasPlugin()])


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "run"
    if cmd == "prepare":
        prepare()
    else:
        sys.exit(run(sys.argv[2:]))
