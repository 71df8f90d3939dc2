"""Physical observables within 1% of the CPU reference.

The protocols are the reference's own (analysis.py:507-561 for the
cantilever ring-down; SURVEY §8d for the multi-material cube); the golden
values were produced by the unmodified reference on the CPU
(tests/golden/make_observables.py -> tests/golden/observables.json).  The
spectral estimators are restated below from analysis.py:83-128.
"""
import json
import os

import numpy as np
import pytest

from paper_2207_09334_b200 import Engine, lattice as L, simulate

GOLD = os.path.join(os.path.dirname(__file__), "golden", "observables.json")


def _golden(name):
    if not os.path.exists(GOLD):
        pytest.skip("observables.json not generated")
    g = json.load(open(GOLD))
    if name not in g:
        pytest.skip(f"{name} not in observables.json")
    return g[name]


def fft_dominant_frequency(values, spacing):
    """analysis.py:100-128: Hann window, largest rfft peak, parabolic
    refinement in log magnitude."""
    values = np.asarray(values, dtype=np.float64)
    n = values.size
    centered = values - values.mean()
    magnitude = np.abs(np.fft.rfft(centered * np.hanning(n)))
    magnitude[0] = 0.0
    peak = int(np.argmax(magnitude))
    shift = 0.0
    if 1 <= peak < magnitude.size - 1:
        tiny = magnitude[peak] * 1e-12
        lo, mid, hi = np.log(magnitude[peak - 1:peak + 2] + tiny)
        curvature = lo - 2.0 * mid + hi
        if curvature != 0.0:
            shift = float(np.clip(0.5 * (lo - hi) / curvature, -0.5, 0.5))
    return (peak + shift) / (n * spacing)


def zero_cross_frequency(values, reference, duration):
    """analysis.py:83-97."""
    signs = np.sign(np.asarray(values) - reference)
    signs = signs[signs != 0.0]
    crossings = 0 if signs.size < 2 else int(np.count_nonzero(np.diff(signs)))
    return crossings / (2.0 * duration)


def beam_ring_down(g, precision):
    """run_beam_experiment (analysis.py:507-561) with the golden calibration."""
    scene = L.beam_lattice(length=g["length"])
    eng = Engine(scene, integrator="verlet", precision=precision)
    per = g["tip_load"] / len(g["tip_ids"])
    for i in g["tip_ids"]:
        eng.set_external_force(i, (0.0, -per, 0.0))
    eng.set_damping(g["damping"])
    eng.step(g["relax_steps"])
    deflection = float(eng.x[g["probe"], 1] - g["reference_y"])
    for i in g["tip_ids"]:
        eng.set_external_force(i, (0.0, 0.0, 0.0))
    eng.set_damping(0.0)
    run = simulate(scene, g["trace_duration"], traces=(g["probe"],), sample_every=g["sample_every"],
                   engine=eng)
    tr = run.position_series(g["probe"], axis=1)
    return deflection, tr


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("beam", ["beam_20x4x4", "beam_40x4x4"])
def test_cantilever_tip_deflection_and_frequency(beam, precision):
    g = _golden(beam)
    deflection, tr = beam_ring_down(g, precision)
    assert abs(deflection - g["relaxed_deflection"]) <= 0.01 * abs(g["relaxed_deflection"])
    assert len(tr.values) == g["samples"]
    fft = fft_dominant_frequency(tr.values, tr.spacing)
    assert abs(fft - g["fft_hz"]) <= 0.01 * g["fft_hz"]
    zc = zero_cross_frequency(tr.values, g["reference_y"], tr.duration)
    assert abs(zc - g["zero_cross_hz"]) <= 0.01 * g["zero_cross_hz"]
    if precision == "f64":                       # same arithmetic as the reference: far inside 1%
        assert abs(fft - g["fft_hz"]) <= 1e-6 * g["fft_hz"]


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("cube", ["cube_mm_12", "cube_mm_42"])
def test_multi_material_cube_natural_frequency(cube, precision):
    """Config 2: FFT of the far-corner x trace of the released, x-stretched
    two-material cube, GPU vs CPU reference, within 1%."""
    g = _golden(cube)
    scene = L.multi_material_cube(g["cells"], stiff_factor=g["stiff_factor"], stretch=g["stretch"])
    run = simulate(scene, g["seconds"], traces=(g["probe"],), sample_every=g["sample_every"],
                   precision=precision)
    tr = run.position_series(g["probe"], axis=0)
    assert len(tr.values) == g["samples"]
    fft = fft_dominant_frequency(tr.values, tr.spacing)
    assert abs(fft - g["fft_hz"]) <= 0.01 * g["fft_hz"]
