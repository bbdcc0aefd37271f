"""``import permanent`` -> the B200 engine (drop-in for the reference package
/root/reference/pkg/src/permanent/__init__.py:1-111).

Put ``dropin/`` on PYTHONPATH (option A) and code written
against the reference -- including the reference's own test suite, see
profiles/r2_reference_suite.txt -- runs unchanged on the sm_100a kernels:
every public name of ``permanent`` and of its submodules resolves to the
module of ``paper_2510_03421_b200`` that implements it:

    permanent.core        -> paper_2510_03421_b200.core        (src/core.py)
    permanent.algorithms  -> paper_2510_03421_b200.algorithms  (src/algorithms.py)
    permanent.dispatch    -> paper_2510_03421_b200.dispatch    (src/dispatch.py)
    permanent.reference   -> paper_2510_03421_b200.reference   (src/reference.py)
    permanent.tuner       -> paper_2510_03421_b200.tuning      (src/tuner.py)
    permanent.svm         -> paper_2510_03421_b200.svm         (src/svm.py)
    permanent.oracles     -> paper_2510_03421_b200.precision   (src/oracles.py)
    permanent.iterate     -> paper_2510_03421_b200.iterate     (src/iterate.py)
    permanent.cli         -> paper_2510_03421_b200.cli         (src/cli.py)
"""
import importlib
import sys
from pathlib import Path

_ROOT = str(Path(__file__).resolve().parents[2])
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import paper_2510_03421_b200 as _engine  # noqa: E402
from paper_2510_03421_b200 import *  # noqa: E402,F401,F403
from paper_2510_03421_b200 import __all__, __version__  # noqa: E402,F401

_SUBMODULES = {"core": "core", "algorithms": "algorithms", "dispatch": "dispatch", "reference": "reference",
               "tuner": "tuning", "svm": "svm", "oracles": "precision", "iterate": "iterate", "cli": "cli"}
for _name, _target in _SUBMODULES.items():
    _mod = importlib.import_module(f"paper_2510_03421_b200.{_target}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod


def __getattr__(name):  # the engine's lazy extensions (batch kernels, sharding)
    return getattr(_engine, name)
