"""pytest plugin: run the reference package's OWN test suite with every
``springsim.Engine`` replaced by the B200 engine (reference_backend.enable).

Used by tools/reftests/run.sh on a GPU box; the reference package and a copy of
its tests live in the git-ignored baseline/_ref (installed from /root/reference
with pip --target, never committed).  SS_REFTEST_PRECISION picks f64 (bitwise
mode, default) or f32.
"""

import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
for p in (ROOT, os.path.join(ROOT, "baseline", "_ref")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    from paper_2207_09334_b200 import reference_backend
    precision = os.environ.get("SS_REFTEST_PRECISION", "f64")
    cls = reference_backend.enable(precision)
    import springsim.engine
    assert springsim.engine.Engine is cls
    config._ss_engine = cls


def pytest_report_header(config):
    import springsim
    return [f"springsim from {os.path.dirname(springsim.__file__)}; Engine -> "
            f"paper_2207_09334_b200 GPU engine ({os.environ.get('SS_REFTEST_PRECISION', 'f64')})"]
