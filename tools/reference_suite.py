"""Stage the reference's own test suite for a run against the drop-in.

In the build container (where /root/reference exists): copies
/root/reference/pkg/tests to baseline/_ref/pkg_tests (git-ignored, travels to
the GPU box with gpurun) and installs tests/reference_suite/shim_conftest.py
as baseline/_ref/conftest.py.  Then, on the B200:

    python -m pytest baseline/_ref/pkg_tests -q -rfE -p no:cacheprovider

Usage: python tools/reference_suite.py
"""
import os
import shutil

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = "/root/reference/pkg/tests"
DST = os.path.join(ROOT, "baseline", "_ref", "pkg_tests")

if __name__ == "__main__":
    if not os.path.isdir(SRC):
        raise SystemExit(f"{SRC} not found (stage the suite in the build container)")
    shutil.rmtree(DST, ignore_errors=True)
    shutil.copytree(SRC, DST)
    shutil.copy(os.path.join(ROOT, "tests", "reference_suite", "shim_conftest.py"),
                os.path.join(ROOT, "baseline", "_ref", "conftest.py"))
    print("staged", DST)
