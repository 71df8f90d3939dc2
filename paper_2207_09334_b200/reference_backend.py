"""Route an installed reference ``springsim`` package through this engine --
the maintainer-side binding of INTEGRATION.md §2, shipped and tested.

``enable(precision)`` subclasses :class:`paper_2207_09334_b200.Engine` with the
reference constructor signature and rebinds ``Engine`` in every springsim
module that uses it: ``springsim.engine`` (``simulate``, ``total_force`` look it
up at call time, engine.py:471, 528) and the modules that imported the name
(bench.py:16, analysis.py:22, service.py:27).  ``disable()`` restores them.
precision="f64" is bitwise the reference's serial mode; "f32" is the 1e-4
production mode.
"""

from __future__ import annotations

import importlib

from .engine import DivergenceError as _GpuDivergenceError
from .engine import Engine as _GpuEngine

_MODULES = ("springsim", "springsim.engine", "springsim.bench", "springsim.analysis", "springsim.service")
_saved: dict = {}


def enable(precision: str = "f64"):
    """Make ``springsim.Engine`` (and every module's imported copy) this engine."""
    ref_engine = importlib.import_module("springsim.engine")

    class DivergenceError(ref_engine.DivergenceError, _GpuDivergenceError):
        """Caught as either package's DivergenceError (the reference's
        analysis and tests catch springsim.engine.DivergenceError)."""

        def __init__(self, mass_id: int, step: int):
            RuntimeError.__init__(self, _GpuDivergenceError.MESSAGE.format(step=step, mass_id=mass_id))
            self.mass_id, self.step = mass_id, step

    class Engine(_GpuEngine):
        _divergence_error = DivergenceError

        def __init__(self, scene, integrator=ref_engine.VERLET, mode=ref_engine.SERIAL, threads=None):
            super().__init__(scene, integrator=integrator, mode=mode, threads=threads, precision=precision)

    for name in _MODULES:
        try:
            mod = importlib.import_module(name)
        except ImportError:            # e.g. the service's optional dependencies
            continue
        if hasattr(mod, "Engine"):
            _saved.setdefault(name, mod.Engine)
            mod.Engine = Engine
    return Engine


def disable() -> None:
    """Restore the reference's own Engine everywhere ``enable`` replaced it."""
    for name, original in list(_saved.items()):
        importlib.import_module(name).Engine = original
        del _saved[name]
