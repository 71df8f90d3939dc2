"""Batches of independent scene instances (SURVEY §8e "batches of independent
robot instances shard trivially", §8f row 3).

``replicate`` stacks ``copies`` instances of one scene into a single
block-diagonal :class:`ArrayScene`: instance ``c`` owns masses
``[c*N, (c+1)*N)`` and springs ``[c*S, (c+1)*S)`` in the same relative order,
so every mass keeps the reference's per-mass summation order and an
instance of the batch steps exactly like the scene alone (bitwise in fp64).
Instances share gravity, dt, damping, actuation groups and contact planes;
they overlap in space but never interact (there is no spring between them
and contact is per mass).  An optional seeded position jitter turns the
batch into an ensemble for chaotic scenes (the walker, SURVEY §7 d').

One engine steps the whole batch, so a population of tiny robots fills a
B200 instead of paying one launch per robot per step; across GPUs the
batch shards by instance with no exchange (``shard``).
"""

from __future__ import annotations

import numpy as np

from .model import ActuationGroup, ArrayScene, ContactPlane, scene_arrays


def jitter_noise(n_masses: int, copies: int, jitter: float, seed: int = 0) -> np.ndarray:
    """(copies, N, 3) N(0, jitter) position offsets, instance 0 exact."""
    noise = np.random.default_rng(seed).normal(0.0, jitter, (copies, n_masses, 3))
    noise[0] = 0.0
    return noise


def replicate(scene, copies: int, jitter: float = 0.0, seed: int = 0) -> ArrayScene:
    """Block-diagonal batch of ``copies`` instances of ``scene`` (a Scene,
    ArrayScene or reference Scene)."""
    if copies < 1:
        raise ValueError("copies must be >= 1")
    a = scene_arrays(scene)
    n, s = a.x.shape[0], a.si.shape[0]
    x = np.tile(a.x, (copies, 1))
    if jitter > 0.0:
        x = x + jitter_noise(n, copies, jitter, seed).reshape(-1, 3)
    off = (np.arange(copies, dtype=np.int64) * n)[:, None]
    si = (a.si[None, :] + off).reshape(-1)
    sj = (a.sj[None, :] + off).reshape(-1)
    group = None if a.group is None else np.tile(a.group, copies)
    groups = {}
    for label, mode, amp, freq, phase in a.group_params:
        groups[label] = ActuationGroup(label, mode=mode, amplitude=amp, frequency=freq, phase=phase)
    out = ArrayScene(x=x, m=np.tile(a.m, copies), si=si, sj=sj, k=np.tile(a.k, copies),
                     l0=np.tile(a.l0, copies), v=np.tile(a.v, (copies, 1)),
                     f_ext=np.tile(a.f_ext, (copies, 1)), fixed=np.tile(a.fixed, copies),
                     gravity=tuple(a.gravity), dt=a.dt, damping=a.damping, groups=groups,
                     group=group, planes=[ContactPlane(normal=tuple(float(c) for c in nrm), offset=off_,
                                                       penalty=pen, friction=fr)
                                          for nrm, off_, pen, fr in a.planes])
    out.instances = copies
    out.instance_masses = n
    out.instance_springs = s
    return out


def per_instance(values: np.ndarray, copies: int) -> np.ndarray:
    """View an (copies*N, ...) array as (copies, N, ...)."""
    values = np.asarray(values)
    return values.reshape((copies, values.shape[0] // copies) + values.shape[1:])


def shard(copies: int, ranks: int, rank: int) -> tuple[int, int]:
    """Instances [lo, hi) of a rank: batches split across GPUs by instance,
    no data-path exchange ("scaling": weak)."""
    base, extra = divmod(copies, ranks)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


__all__ = ["replicate", "per_instance", "jitter_noise", "shard"]
