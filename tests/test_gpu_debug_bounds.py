"""The bounds-assert build (csrc/common.cuh PERM_CHECK, `make debug`) on the
GPU: the smoke permanents and the zero-copy path's branches run against
libpermanent_b200_debug.so in a subprocess; any violated index bound traps
the kernel and fails the run.  Skipped when the debug library was not
built (tools/debug_bounds_check.sh runs the whole GPU suite against it)."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
LIB = ROOT / "paper_2510_03421_b200" / "libpermanent_b200_debug.so"
STAMP = LIB.with_suffix(".stamp")


def _sources_hash() -> str:
    """sha256 of the engine sources in the order the Makefile's debug target
    hashes them (csrc/*.cu, *.cuh and the header, sorted by path)."""
    import hashlib

    csrc = ROOT / "paper_2510_03421_b200" / "csrc"
    files = sorted([f"{p.name}" for p in csrc.glob("*.cu")] + [f"{p.name}" for p in csrc.glob("*.cuh")] +
                   ["../../include/permanent_b200.h"])
    h = hashlib.sha256()
    for f in files:
        h.update((csrc / f).read_bytes())
    return h.hexdigest()


def _debug_lib_current() -> bool:
    return LIB.exists() and STAMP.exists() and STAMP.read_text().strip() == _sources_hash()


@pytest.mark.skipif(not _debug_lib_current(),
                    reason="debug library absent or stale (make -C paper_2510_03421_b200/csrc debug)")
def test_bounds_checked_library_runs_clean():
    env = dict(os.environ, PERMANENT_B200_LIB=str(LIB))
    code = ("import __graft_entry__ as g; g.smoke(); "
            "from paper_2510_03421_b200 import _lib; import os; "
            "assert _lib.load()._name == os.environ['PERMANENT_B200_LIB']")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-x",
                        "tests/test_gpu_zero_copy.py"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
