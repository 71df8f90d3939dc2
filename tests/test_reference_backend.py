"""The maintainer-side binding against the real reference
package, when it is importable (this container; not the GPU box)."""
import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture
def springsim():
    if not os.path.isdir(REF):
        pytest.skip("reference package not present")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    try:
        import springsim as s
    except ImportError as exc:  # pragma: no cover
        pytest.skip(f"reference not importable: {exc}")
    yield s
    sys.path.remove(REF)


def test_enable_routes_every_engine_user(springsim):
    """After enable(), simulate / bench_scene / run_beam_experiment construct
    this package's engine (on a GPU-less host that engine fails loudly: no CPU
    fallback), and disable() restores the reference's."""
    import springsim.bench as rbench
    import springsim.engine as reng
    from paper_2207_09334_b200 import _lib, reference_backend
    original = reng.Engine
    Engine = reference_backend.enable(precision="f32")
    try:
        assert reng.Engine is Engine and rbench.Engine is Engine and springsim.Engine is Engine
        assert issubclass(Engine, __import__("paper_2207_09334_b200").Engine)
        scene = rbench.block_scene(2)
        if _lib.device_count() == 0:
            with pytest.raises(_lib.CudaError):
                rbench.bench_scene(scene, steps=100)
            with pytest.raises(_lib.CudaError):
                reng.simulate(scene, 0.01)
    finally:
        reference_backend.disable()
    assert reng.Engine is original and rbench.Engine is original


def test_divergence_is_the_reference_exception(springsim):
    """The routed engine raises a DivergenceError that the reference's own
    callers catch (springsim.engine.DivergenceError, analysis.py re-raises it
    as a time-step RuntimeError) and that this package's callers catch too,
    with the reference's message and attributes."""
    import springsim.engine as reng
    from paper_2207_09334_b200 import reference_backend
    from paper_2207_09334_b200.engine import DivergenceError as Ours
    Engine = reference_backend.enable()
    try:
        err = Engine._divergence_error(7, 41)
        assert isinstance(err, reng.DivergenceError) and isinstance(err, Ours)
        assert (err.mass_id, err.step) == (7, 41)
        assert str(err) == str(reng.DivergenceError(7, 41))
    finally:
        reference_backend.disable()
