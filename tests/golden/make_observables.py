"""Generate tests/golden/observables.json with the REFERENCE package (CPU).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_observables.py

Physical-observable oracles of SURVEY Appendix C, computed by the unmodified
reference (springsim) on this container's CPU:

* cantilever ring-downs (reference analysis.py:507-561, run_beam_experiment)
  for the 20x4x4 and 40x4x4 beams: the calibrated tip load, the probe and
  tip masses, the step counts, the damped-relaxed tip deflection and the
  FFT / zero-cross frequency of the released ring-down;
* config 3, an ensemble of actuated crawlers (demos/crawler.py) with
  1e-9 m position jitter: net travel per instance after 8 s (the walker is
  chaotic, SURVEY §7 d', so fp32 is judged on the ensemble mean);
* config 2, the multi-material natural-frequency cube (SURVEY §8d recipe:
  block_scene(n), k x10 where both endpoints have x < side/2, released from
  a 0.1% x-stretch about the centroid at rest): FFT dominant frequency of the
  far-corner x trace over 2 s (sample_every 10).

The GPU tests (tests/test_observables.py) rerun the same protocols through
paper_2207_09334_b200 and require agreement within 1%.
"""
import json
import math
import os
import sys
import time

import numpy as np

from springsim import analysis as A
from springsim import bench as B
from springsim.engine import Engine, simulate

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "observables.json")


def beam_case(length):
    beam = A.BeamSpec(length=length)
    cfg = A.BeamRunConfig()
    t0 = time.time()
    scene = A.beam_lattice(beam)
    tip_ids, probe = A._tip_layer(scene, beam)
    reference = float(scene.masses[probe].x[1])
    modal = A.assemble_modal_system(scene)
    f_est = A._bending_mode_estimate(modal)
    tip_load = A._calibrated_tip_load(scene, modal, tip_ids, probe, cfg.tip_deflection)
    per_mass = 1.0 / len(tip_ids)
    eng = Engine(scene, integrator=cfg.integrator, mode=cfg.mode)
    for i in tip_ids:
        eng.set_external_force(i, (0.0, -tip_load * per_mass, 0.0))
    eng.set_damping(cfg.damping)
    settle = 6.0 * eng.dt / cfg.damping
    relax = max(0.5, 4.0 / f_est, settle)
    relax_steps = max(1, math.ceil(relax / eng.dt - 1e-9))
    eng.step(relax_steps)
    deflection = float(eng.x[probe, 1] - reference)
    for i in tip_ids:
        eng.set_external_force(i, (0.0, 0.0, 0.0))
    eng.set_damping(0.0)
    duration = cfg.trace_cycles / f_est
    run = simulate(scene, duration, traces=(probe,), sample_every=cfg.sample_every, engine=eng)
    tr = run.position_series(probe, axis=1)
    return {
        "length": length, "tip_ids": list(tip_ids), "probe": probe, "reference_y": reference,
        "tip_load": tip_load, "modal_hz": f_est, "damping": cfg.damping,
        "relax_steps": relax_steps, "trace_duration": duration, "sample_every": cfg.sample_every,
        "relaxed_deflection": deflection,
        "fft_hz": A.fft_dominant_frequency(tr), "zero_cross_hz": A.zero_cross_frequency(tr, reference),
        "samples": int(len(tr.values)), "cpu_seconds": round(time.time() - t0, 1),
    }


def cube_case(cells, seconds=2.0, stiff=10.0, stretch=1e-3, threads=8):
    t0 = time.time()
    scene = B.block_scene(cells)
    side = cells * 0.1
    for s in scene.springs:
        if scene.masses[s.i].x[0] < side / 2 and scene.masses[s.j].x[0] < side / 2:
            s.k = s.k * stiff
    xs = np.array([m.x for m in scene.masses])
    cx = xs[:, 0].mean()
    for m in scene.masses:
        x = list(m.x)
        x[0] = cx + (x[0] - cx) * (1.0 + stretch)
        m.x = tuple(x)
    corner = scene.mass_count - 1                    # (n, n, n) corner: last lexicographic id
    eng = Engine(scene, integrator="verlet", mode="parallel-det", threads=threads)
    run = simulate(scene, seconds, traces=(corner,), sample_every=10, engine=eng)
    tr = run.position_series(corner, axis=0)
    return {"cells": cells, "springs": scene.spring_count, "stiff_factor": stiff, "stretch": stretch,
            "seconds": seconds, "sample_every": 10, "probe": corner,
            "fft_hz": A.fft_dominant_frequency(tr), "samples": int(len(tr.values)),
            "cpu_seconds": round(time.time() - t0, 1)}


def crawler_ensemble(copies=16, jitter=1e-9, seed=5, seconds=8.0):
    """Config 3: the actuated crawler (demos/crawler.py:27-71, damping 2e-4),
    `copies` instances whose initial positions carry N(0, jitter) noise
    (instance 0 exact; numpy default_rng(seed).normal(0, jitter, (copies, N, 3))),
    each run by the reference for `seconds`; net x-centre travel per instance."""
    sys.path.insert(0, "/root/reference/pkg/demos")
    from crawler import build_crawler
    t0 = time.time()
    base = build_crawler()
    n = base.mass_count
    noise = np.random.default_rng(seed).normal(0.0, jitter, (copies, n, 3))
    noise[0] = 0.0
    travel = []
    for c in range(copies):
        scene = build_crawler()
        for i, m in enumerate(scene.masses):
            m.x = tuple(np.asarray(m.x, dtype=np.float64) + noise[c, i])
        eng = Engine(scene)
        eng.set_damping(2e-4)
        start = float(np.mean(eng.x[:, 0]))
        eng.step(int(round(seconds / scene.dt)))
        travel.append(float(np.mean(eng.x[:, 0])) - start)
    return {"copies": copies, "jitter": jitter, "seed": seed, "seconds": seconds, "damping": 2e-4,
            "travel": travel, "mean_travel": float(np.mean(travel)), "std_travel": float(np.std(travel)),
            "cpu_seconds": round(time.time() - t0, 1)}


if __name__ == "__main__":
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    which = sys.argv[1:] or ["beam20", "beam40", "cube12", "cube42"]
    for w in which:
        if w == "beam20":
            out["beam_20x4x4"] = beam_case(2.0)
        elif w == "beam40":
            out["beam_40x4x4"] = beam_case(4.0)
        elif w == "cube12":
            out["cube_mm_12"] = cube_case(12)
        elif w == "cube42":
            out["cube_mm_42"] = cube_case(42)
        elif w == "crawler":
            out["crawler_ensemble"] = crawler_ensemble()
        json.dump(out, open(OUT, "w"), indent=1)
        print(w, json.dumps(out.get({"beam20": "beam_20x4x4", "beam40": "beam_40x4x4",
                                     "cube12": "cube_mm_12", "cube42": "cube_mm_42",
                                     "crawler": "crawler_ensemble"}[w])), flush=True)
