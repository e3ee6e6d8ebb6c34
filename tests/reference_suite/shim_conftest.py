"""Import shim for running the REFERENCE's own test suite (pkg/tests of
arxiv/paper_0910_4711) against this drop-in: every `vqkit` module the tests
import resolves to the matching module of paper_0910_4711_b200 (SURVEY.md
8(c), "Run these files against vqb200 via a conftest import shim").

tools/reference_suite.py copies this file to baseline/_ref/conftest.py, next
to the copied tests (baseline/_ref is git-ignored; the reference's sources
never enter the repo).  Nothing here is product code."""

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))  # baseline/_ref/.. /..
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_0910_4711_b200 as _pkg  # noqa: E402
from paper_0910_4711_b200 import (  # noqa: E402
    cli as _cli,
    codec as _codec,
    core as _core,
    errors as _errors,
    kernels as _kernels,
    parallel as _parallel,
    storage as _storage,
    sweep as _sweep,
)

sys.modules["vqkit"] = _pkg
for _name, _mod in {"core": _core, "codec": _codec, "parallel": _parallel, "storage": _storage,
                    "cli": _cli, "errors": _errors, "bench": _sweep, "_kernels": _kernels}.items():
    sys.modules[f"vqkit.{_name}"] = _mod
    setattr(_pkg, _name, _mod)
