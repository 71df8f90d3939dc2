"""Shared helpers: golden-fixture loading, GPU marker, oracle import path."""

from __future__ import annotations

import glob
import os
import sys
from types import SimpleNamespace

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_cases(prefix: str = "") -> list[str]:
    names = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        name = os.path.basename(p)[:-4]
        if name.startswith(prefix) and "checkpoints" in np.load(p).files:
            names.append(name)
    return names


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def golden_arrays(d) -> SimpleNamespace:
    """Inputs of a golden case as a SceneArrays-like namespace."""
    labels = [str(s) for s in d["in_group_labels"]]
    modes = [str(s) for s in d["in_group_mode"]]
    num = d["in_group_num"]
    gp = [(labels[g], modes[g], float(num[g, 0]), float(num[g, 1]), float(num[g, 2]))
          for g in range(len(labels))]
    planes = [(d["in_planes"][p, :3].copy(), float(d["in_planes"][p, 3]),
               float(d["in_planes"][p, 4]), float(d["in_planes"][p, 5]))
              for p in range(d["in_planes"].shape[0])]
    return SimpleNamespace(
        x=d["in_x"], v=d["in_v"], m=d["in_m"], f_ext=d["in_f_ext"], fixed=d["in_fixed"],
        si=d["in_si"], sj=d["in_sj"], k=d["in_k"], l0=d["in_l0"], group=d["in_group"],
        group_params=gp, planes=planes, gravity=d["in_gravity"], dt=float(d["in_dt"]),
        damping=float(d["in_damping"]))


def golden_scene(d):
    """Golden inputs as an ArrayScene of the product package."""
    from paper_2207_09334_b200.model import ActuationGroup, ArrayScene, ContactPlane
    a = golden_arrays(d)
    groups = {label: ActuationGroup(label, mode=mode, amplitude=amp, frequency=f, phase=ph)
              for (label, mode, amp, f, ph) in a.group_params}
    planes = [ContactPlane(normal=tuple(float(c) for c in p[0]), offset=p[1], penalty=p[2],
                           friction=p[3]) for p in a.planes]
    return ArrayScene(x=a.x, m=a.m, si=a.si, sj=a.sj, k=a.k, l0=a.l0, v=a.v, f_ext=a.f_ext,
                      fixed=a.fixed, gravity=tuple(a.gravity), dt=a.dt, damping=a.damping,
                      groups=groups, group=a.group, planes=planes)


@pytest.fixture
def has_gpu():
    from paper_2207_09334_b200 import _lib
    return _lib.device_count() > 0
