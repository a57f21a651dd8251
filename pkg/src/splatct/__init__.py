"""``splatct`` -- the reference package's import name, served by the B200 build.

Drop-in shim: ``import splatct`` / ``from splatct import fvr, projector, loss,
optim, ...`` resolve to ``paper_2411_04844_b200`` (repo root), whose modules
keep the reference's function names and signatures
(reference: pkg/src/splatct/__init__.py:1-35).  Put ``pkg/src`` on
``PYTHONPATH`` (or ``pip install -e pkg``) to use it.
"""

import importlib
import os
import sys

_ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..", ".."))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

_impl = importlib.import_module("paper_2411_04844_b200")
for _name in ("core", "fvr", "projector", "loss", "optim", "densify", "metrics", "phantom", "io",
              "cli", "distributed"):
    _mod = importlib.import_module(f"paper_2411_04844_b200.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

from paper_2411_04844_b200 import *  # noqa: E402,F401,F403
from paper_2411_04844_b200 import __all__, __version__  # noqa: E402,F401
