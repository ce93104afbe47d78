"""Alias `overlapsim` (the reference package name) to paper_2004_14020_b200 so
the reference's own test files run unmodified against this implementation.
Test infrastructure only (tests/test_reference_suite.py)."""
import importlib
import sys

import paper_2004_14020_b200 as _impl
from paper_2004_14020_b200 import *  # noqa: F401,F403

for _sub in ("dag", "costmodel", "collective", "batching", "ordering", "transfer", "pipeline", "sim"):
    sys.modules[f"{__name__}.{_sub}"] = importlib.import_module(f"paper_2004_14020_b200.{_sub}")
    globals()[_sub] = sys.modules[f"{__name__}.{_sub}"]
__version__ = _impl.__version__
