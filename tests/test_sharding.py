"""x-slab sharding: host partition logic (CPU, gloo world_size 2) and the
sharded GPU path on one device (virtual shards) vs the single-device engine."""

import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2207_09334_b200 import Engine
from paper_2207_09334_b200 import lattice as L
from paper_2207_09334_b200.sharded import ShardGroup, cube_slab, excited_velocities, slab_planes


def test_slab_planes_partition():
    for nx in (4, 10, 92, 314):
        for n in (1, 2, 3, 8):
            spans = [slab_planes(nx, n, r) for r in range(n)]
            assert spans[0][0] == 0 and spans[-1][1] == nx
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_slabs_cover_the_cube_once():
    cells, n = 6, 3
    nx = cells + 1
    full = L.block_scene(cells)
    plane = nx * nx
    owned_springs = 0
    for r in range(n):
        s = cube_slab(cells, *slab_planes(nx, n, r))
        g_si = s.scene.si + s.first_global
        g_sj = s.scene.sj + s.first_global
        lo = s.i_lo * plane
        hi = s.i_hi * plane
        own = (g_si >= lo) & (g_si < hi)            # lower endpoint owned: counted once
        owned_springs += int(own.sum())
        # every spring touching an owned mass is present, in global id order
        touch = ((full.si >= lo) & (full.si < hi)) | ((full.sj >= lo) & (full.sj < hi))
        assert np.array_equal(g_si, full.si[touch]) and np.array_equal(g_sj, full.sj[touch])
        assert s.scene.k.tobytes() == full.k[touch].tobytes()
        assert s.scene.x[s.owned].tobytes() == full.x[lo:hi].tobytes()
        assert s.scene.fixed[s.recv_lo].all() and s.scene.fixed[s.recv_hi].all()
        assert not s.scene.fixed[s.owned].any()
    assert owned_springs == full.spring_count


def _gloo_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cells = 7
        nx = cells + 1
        s = cube_slab(cells, *slab_planes(nx, world, rank))
        send_hi = (s.send_hi + s.first_global).tolist()
        recv_lo = (s.recv_lo + s.first_global).tolist()
        send_lo = (s.send_lo + s.first_global).tolist()
        recv_hi = (s.recv_hi + s.first_global).tolist()
        got = [None] * world
        dist.all_gather_object(got, {"send_hi": send_hi, "recv_lo": recv_lo, "send_lo": send_lo,
                                     "recv_hi": recv_hi, "owned": s.n_owned})
        ok = True
        for r in range(world - 1):                  # rank r's upper plane feeds r+1's lower halo
            ok &= got[r]["send_hi"] == got[r + 1]["recv_lo"]
            ok &= got[r + 1]["send_lo"] == got[r]["recv_hi"]
        ok &= sum(g["owned"] for g in got) == nx ** 3
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_halo_lists_agree_across_ranks_gloo():
    """world_size-2 gloo run of the N>1 host path: neighbouring ranks agree on
    the exchanged planes, and the owned masses partition the cube."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("shards", [2, 3])
def test_virtual_shards_match_single_device(precision, shards):
    """The sharded path (slab scenes + halo exchange every substep) against one
    engine on the whole cube.  fp64: bitwise (owned masses keep their global
    spring-id summation order).  fp32: force evaluation uses tile-local
    coordinates whose anchors depend on the tiling, so agreement is to fp32
    rounding: <= 1e-4 of the displacement."""
    cells = 11
    full = L.excite(L.block_scene(cells), seed=11)
    v = excited_velocities(full.mass_count)
    assert v.tobytes() == full.v.tobytes()
    one = Engine(full, precision=precision)
    grp = ShardGroup(cells, shards, precision=precision, v_global=v)
    one.step(37)
    grp.step(37)
    if precision == "f64":
        assert grp.positions().tobytes() == one.x.tobytes()
        assert grp.velocities().tobytes() == one.v.tobytes()
    else:
        disp = np.abs(one.x - full.x).max()
        assert np.abs(grp.positions() - one.x).max() <= 1e-4 * disp


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["copy", "p2p"])
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("shards", [2, 3])
def test_virtual_shards_rk4(precision, shards, transport):
    """Sharded RK4 (four exchanges per step): every stage's trial
    positions reach the neighbours' halos before the next stage -- plane
    copies between stages, or pushed by the stage kernels themselves into
    the neighbours' stage buffers (p2p).  fp64 bitwise against one engine;
    fp32 to rounding."""
    cells = 9
    full = L.excite(L.block_scene(cells), seed=11)
    v = excited_velocities(full.mass_count)
    one = Engine(full, integrator="rk4", precision=precision)
    grp = ShardGroup(cells, shards, precision=precision, v_global=v, integrator="rk4", transport=transport)
    for n in (1, 12):
        one.step(n)
        grp.step(n)
        if precision == "f64":
            assert grp.positions().tobytes() == one.x.tobytes()
            assert grp.velocities().tobytes() == one.v.tobytes()
        else:
            disp = np.abs(one.x - full.x).max()
            assert np.abs(grp.positions() - one.x).max() <= 1e-4 * disp


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["copy", "p2p"])
@pytest.mark.parametrize("integrator", ["verlet", "rk4"])
@pytest.mark.parametrize("where", ["boundary", "interior"])
def test_sharded_divergence_matches_one_engine(transport, integrator, where):
    """A mass launched at 1e300 m/s (its springs overflow): one engine raises DivergenceError
    (engine.py:375-381) at some step for its lowest non-finite mass.  The
    shards share one divergence step, so all of them stop after that same
    step, the error names the same global mass and step, and the assembled
    state is the single engine's diverged state."""
    from paper_2207_09334_b200 import DivergenceError
    cells = 9
    full = L.excite(L.block_scene(cells), seed=11)
    nx = cells + 1
    plane = nx * nx
    i = 5 if where == "boundary" else 7                     # x-plane 5 borders the 2-shard split
    victim = i * plane + plane // 2
    full.v[victim] = (1e300, 0.0, 0.0)
    v = full.v.copy()
    one = Engine(full, integrator=integrator, precision="f64")
    with pytest.raises(DivergenceError) as e1:
        one.step(40)
    grp = ShardGroup(cells, 2, precision="f64", v_global=v, integrator=integrator, transport=transport)
    with pytest.raises(DivergenceError) as e2:
        grp.step(40)
    assert (e2.value.mass_id, e2.value.step) == (e1.value.mass_id, e1.value.step)
    assert all(e.n == one.n for e in grp.engines)
    np.testing.assert_array_equal(grp.positions(), one.x)
    np.testing.assert_array_equal(grp.velocities(), one.v)


@pytest.mark.gpu
@pytest.mark.parametrize("integrator", ["verlet", "rk4"])
def test_nccl_transport_self_loop(integrator):
    """Exercise the NCCL path on one GPU: a single rank whose lower and upper
    'neighbours' are itself.  After a step, each halo plane must hold the
    positions of the plane it is wired to (transport + pack/unpack check;
    RK4 exchanges after each of its four stages)."""
    import ctypes as C

    import torch  # noqa: F401  (loads libnccl.so.2 into the process)

    from paper_2207_09334_b200 import _lib
    from paper_2207_09334_b200.sharded import attach_halo
    cells = 5
    nx = cells + 1
    s = cube_slab(cells, 1, nx - 1, v_global=excited_velocities(nx ** 3))
    # fp64: absolute positions travel (in fp32 only the displacement r does,
    # which is consistent only between the two copies of the SAME mass)
    eng = Engine(s.scene, precision="f64", integrator=integrator)
    attach_halo(eng, s)
    uid = C.create_string_buffer(128)
    _lib.check(_lib.lib().ss_nccl_unique_id(uid))
    _lib.check(_lib.lib().ss_halo_nccl(eng.handle, uid.raw, 1, 0, 0, 0))
    n0 = eng.launch_count
    eng.step(3)
    x = eng.x
    # per step: the stage kernels plus a pack and an unpack per exchange
    assert eng.launch_count - n0 == 3 * (4 * 3 if integrator == "rk4" else 3)
    assert x[s.recv_lo].tobytes() == x[s.send_lo].tobytes()
    assert x[s.recv_hi].tobytes() == x[s.send_hi].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("precision,layout", [("f64", "auto"), ("f32", "auto"), ("f64", "csr")])
@pytest.mark.parametrize("shards", [2, 3])
def test_peer_memory_shards_match_single_device(precision, layout, shards):
    """The fused peer-memory exchange of the multi-GPU path (step kernels
    store boundary planes into the neighbours' buffers, release/acquire step
    flags, ghost masses written only by their neighbour; kernels.cuh xchg_*)
    between the shards of one process: fp64 bitwise equal to one engine on
    the whole cube (tiled and CSR layouts), fp32 within fp32 rounding of the
    displacement."""
    cells = 11
    full = L.excite(L.block_scene(cells), seed=11)
    v = excited_velocities(full.mass_count)
    one = Engine(full, precision=precision)
    grp = ShardGroup(cells, shards, precision=precision, v_global=v, transport="p2p", layout=layout)
    one.step(41)
    grp.step(41)
    if precision == "f64":
        assert grp.positions().tobytes() == one.x.tobytes()
        assert grp.velocities().tobytes() == one.v.tobytes()
    else:
        disp = np.abs(one.x - full.x).max()
        assert np.abs(grp.positions() - one.x).max() <= 1e-4 * disp


def _ipc_worker(rank, world, port, cells, steps, precision, q, integrator="verlet"):
    """One shard per process, all on cuda:0: the cross-process (CUDA IPC)
    mailbox mapping and the device-side flag protocol, as under torchrun."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2207_09334_b200.sharded import attach_halo, attach_peers
        nx = cells + 1
        s = cube_slab(cells, *slab_planes(nx, world, rank),
                      v_global=excited_velocities(nx ** 3))
        eng = Engine(s.scene, integrator=integrator, precision=precision, device=0)
        attach_halo(eng, s)
        attach_peers(eng, rank, world)
        for _ in range(steps // 7):
            eng.step(7)
        eng.step(steps % 7)
        q.put((rank, s.i_lo, eng.x[s.owned].copy(), eng.v[s.owned].copy(), None))
        eng.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, -1, None, None, repr(exc)))


@pytest.mark.gpu
@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,integrator", [(2, "verlet"), (3, "verlet"), (3, "rk4")])
def test_peer_memory_shards_across_processes(world, integrator):
    """Two or three processes, one shard each, sharing one GPU (with three,
    the middle shard exchanges with two neighbours): mailboxes mapped with
    cudaIpcOpenMemHandle, planes pushed and landed every substep (RK4: every
    stage, into the neighbours' IPC-mapped stage buffers) with no host round
    trip; the assembled fp64 state is bitwise the single engine's."""
    cells, steps = 9, 30
    full = L.excite(L.block_scene(cells), seed=11)
    one = Engine(full, precision="f64", integrator=integrator)
    one.step(steps)
    ref_x, ref_v = one.x.copy(), one.v.copy()
    one.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000) + 7 + world + (20 if integrator == "rk4" else 0)
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, cells, steps, "f64", q, integrator))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=500) for _ in procs], key=lambda t: t[1])
    for p in procs:
        p.join(timeout=60)
    errs = [r[4] for r in res if r[4]]
    assert not errs, errs
    x = np.concatenate([r[2] for r in res])
    v = np.concatenate([r[3] for r in res])
    assert x.tobytes() == ref_x.tobytes()
    assert v.tobytes() == ref_v.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_peer_memory_shards_euler(precision):
    """The fused exchange under forward Euler (positions from the old
    velocities): 3 shards, fp64 bitwise, fp32 to rounding."""
    cells = 11
    full = L.excite(L.block_scene(cells), seed=11)
    v = excited_velocities(full.mass_count)
    one = Engine(full, integrator="euler", precision=precision)
    grp = ShardGroup(cells, 3, precision=precision, v_global=v, transport="p2p", integrator="euler")
    one.step(29)
    grp.step(29)
    if precision == "f64":
        assert grp.positions().tobytes() == one.x.tobytes()
        assert grp.velocities().tobytes() == one.v.tobytes()
    else:
        disp = np.abs(one.x - full.x).max()
        assert np.abs(grp.positions() - one.x).max() <= 1e-4 * disp


# ------------------------------------------------ any x-major voxel lattice

def _loaded_beam():
    """The 40x4x4 cantilever of configs[0]: fixed root layer, gravity, a tip
    load (f_ext) and damping (reference analysis.py:435-476)."""
    b = L.beam_lattice(length=4.0, gravity=(0.0, -9.81, 0.0))
    f = np.zeros((b.mass_count, 3))
    f[b.x[:, 0] > 3.95, 1] = -0.02
    b.f_ext = f
    b.damping = 1e-4
    return b


@pytest.mark.parametrize("shards", [2, 3, 5])
def test_scene_slabs_of_a_beam_cover_it_once(shards):
    from paper_2207_09334_b200.sharded import scene_slab, slab_ranges
    b = _loaded_beam()
    ranges = slab_ranges(b, shards)
    assert ranges[0][0] == 0 and ranges[-1][1] == b.mass_count
    owned_springs = 0
    for r in range(shards):
        s = scene_slab(b, ranges, r)
        g = s.global_ids
        lo, hi = ranges[r]
        touch = ((b.si >= lo) & (b.si < hi)) | ((b.sj >= lo) & (b.sj < hi))
        assert np.array_equal(g[s.scene.si], b.si[touch]) and np.array_equal(g[s.scene.sj], b.sj[touch])
        assert s.scene.k.tobytes() == b.k[touch].tobytes() and s.scene.l0.tobytes() == b.l0[touch].tobytes()
        assert s.scene.f_ext[s.owned].tobytes() == b.f_ext[lo:hi].tobytes()
        assert np.array_equal(s.scene.fixed[s.owned], b.fixed[lo:hi])
        assert s.scene.fixed[s.recv_lo].all() and s.scene.fixed[s.recv_hi].all()
        owned_springs += int(((g[s.scene.si] >= lo) & (g[s.scene.si] < hi)).sum())
        if r + 1 < shards:
            t = scene_slab(b, ranges, r + 1)
            assert np.array_equal(g[s.send_hi], t.global_ids[t.recv_lo])
            assert np.array_equal(t.global_ids[t.send_lo], g[s.recv_hi])
    assert owned_springs == b.spring_count


def test_scene_slabs_reject_non_x_major_and_long_springs():
    from paper_2207_09334_b200.sharded import scene_slab, slab_ranges
    c = L.block_scene(4)
    rev = L.block_scene(4)
    rev.x = rev.x[::-1].copy()
    with pytest.raises(ValueError, match="not ordered by x"):
        slab_ranges(rev, 2)
    ranges = slab_ranges(c, 3)
    c.si = np.append(c.si, 0)
    c.sj = np.append(c.sj, c.mass_count - 1)           # a spring across the whole cube
    c.k = np.append(c.k, 1.0)
    c.l0 = np.append(c.l0, 1.0)
    with pytest.raises(ValueError, match="non-adjacent"):
        scene_slab(c, ranges, 0)


def _gloo_beam_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2207_09334_b200.sharded import scene_slab, slab_ranges
        b = _loaded_beam()
        s = scene_slab(b, slab_ranges(b, world), rank)
        g = s.global_ids
        got = [None] * world
        dist.all_gather_object(got, {"send_hi": g[s.send_hi].tolist(), "recv_lo": g[s.recv_lo].tolist(),
                                     "send_lo": g[s.send_lo].tolist(), "recv_hi": g[s.recv_hi].tolist(),
                                     "owned": s.n_owned})
        ok = all(got[r]["send_hi"] == got[r + 1]["recv_lo"] and got[r + 1]["send_lo"] == got[r]["recv_hi"]
                 for r in range(world - 1))
        ok &= sum(x["owned"] for x in got) == b.mass_count
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_beam_halo_lists_agree_across_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000) + 3
    procs = [ctx.Process(target=_gloo_beam_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def _assemble(grp):
    return (np.concatenate([e.x[s.owned] for e, s in zip(grp.engines, grp.slabs)]),
            np.concatenate([e.v[s.owned] for e, s in zip(grp.engines, grp.slabs)]))


@pytest.mark.gpu
@pytest.mark.parametrize("transport,integrator", [("copy", "verlet"), ("p2p", "verlet"), ("copy", "euler"),
                                                  ("p2p", "euler"), ("copy", "rk4"), ("p2p", "rk4")])
@pytest.mark.parametrize("shards", [2, 3])
def test_sharded_beam_bitwise(transport, shards, integrator):
    """configs[0]'s loaded cantilever split into x-slabs (fixed root,
    gravity, tip load, damping): fp64 bitwise equal to one engine."""
    from paper_2207_09334_b200.sharded import ShardGroup
    b = _loaded_beam()
    one = Engine(b, integrator=integrator, precision="f64")
    grp = ShardGroup.from_scene(b, shards, precision="f64", transport=transport, integrator=integrator)
    for n in (13, 50):
        one.step(n)
        grp.step(n)
        x, v = _assemble(grp)
        assert x.tobytes() == one.x.tobytes() and v.tobytes() == one.v.tobytes()


@pytest.mark.gpu
def test_sharded_multi_material_cube_bitwise():
    """configs[1]'s multi-material stretched cube (n=14) in 3 slabs, p2p."""
    from paper_2207_09334_b200.sharded import ShardGroup
    c = L.multi_material_cube(14)
    one = Engine(c, precision="f64")
    grp = ShardGroup.from_scene(c, 3, precision="f64", transport="p2p")
    one.step(60)
    grp.step(60)
    x, v = _assemble(grp)
    assert x.tobytes() == one.x.tobytes() and v.tobytes() == one.v.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["p2p", "copy"])
def test_sharded_general_graph_bitwise(transport):
    """A cube whose every spring has its own stiffness (so every tile
    overflows the 64-entry dictionary and steps on the inline general-graph
    format) in 3 slabs: bitwise the single engine."""
    from paper_2207_09334_b200.sharded import ShardGroup
    c = L.excite(L.block_scene(12), seed=7)
    c.k = c.k * (1.0 + 1e-7 * np.arange(c.k.size))
    one = Engine(c, precision="f64")
    assert one.info()["tile_kernel"] == 5
    grp = ShardGroup.from_scene(c, 3, precision="f64", transport=transport)
    for n in (7, 40):
        one.step(n)
        grp.step(n)
        x, v = _assemble(grp)
        assert x.tobytes() == one.x.tobytes() and v.tobytes() == one.v.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["p2p", "copy"])
@pytest.mark.parametrize("integrator", ["verlet", "rk4"])
def test_sharded_general_graph_fp32(transport, integrator):
    """The fp32 general-graph format (rest vectors formed from the staged
    X0, tile_lean_kernel INLINE; sharded Verlet on its boundary-tiles-first
    variant) in 3 slabs, within fp32 rounding of one engine."""
    from paper_2207_09334_b200.sharded import ShardGroup
    c = L.excite(L.block_scene(12), seed=7)
    c.k = c.k * (1.0 + 1e-7 * np.arange(c.k.size))
    one = Engine(c, precision="f32", integrator=integrator)
    assert one.info()["tile_kernel"] == 6
    grp = ShardGroup.from_scene(c, 3, precision="f32", transport=transport, integrator=integrator)
    assert all(e.info()["tile_kernel"] == 6 for e in grp.engines)
    one.step(40)
    grp.step(40)
    x, _ = _assemble(grp)
    disp = np.abs(one.x - c.x).max()
    assert np.abs(x - one.x).max() <= 1e-4 * disp


@pytest.mark.gpu
@pytest.mark.parametrize("transport,integrator", [("copy", "verlet"), ("p2p", "verlet"), ("p2p", "rk4"),
                                                  ("copy", "euler")])
def test_thin_slabs(transport, integrator):
    """6 x-planes in 5 slabs: one-plane slabs whose every mass is both a
    boundary mass and a neighbour's ghost; fp64 bitwise equal to one engine."""
    cells = 5
    full = L.excite(L.block_scene(cells), seed=11)
    v = excited_velocities(full.mass_count)
    one = Engine(full, integrator=integrator, precision="f64")
    grp = ShardGroup(cells, 5, precision="f64", v_global=v, integrator=integrator, transport=transport)
    for n in (3, 40):
        one.step(n)
        grp.step(n)
        assert grp.positions().tobytes() == one.x.tobytes()
        assert grp.velocities().tobytes() == one.v.tobytes()


def _crawler_line(copies: int):
    """``copies`` crawlers (demos/crawler.py: floor contact with friction,
    two sinusoid actuation groups, damping) side by side along x, so the
    batch is x-major and splits into x-slabs between walkers."""
    from paper_2207_09334_b200 import crawler_scene, replicate
    b = replicate(crawler_scene(), copies)
    n = b.instance_masses
    span = np.ptp(b.x[:n, 0]) + 0.25
    b.x[:, 0] += np.repeat(np.arange(copies) * span, n)
    return b


@pytest.mark.gpu
@pytest.mark.parametrize("transport,integrator", [("copy", "verlet"), ("p2p", "verlet"), ("p2p", "euler"),
                                                  ("copy", "rk4"), ("p2p", "rk4")])
def test_sharded_walkers_with_groups_and_contact(transport, integrator):
    """A line of 6 walkers (actuation groups, floor contact and friction,
    damping) in 3 x-slabs: fp64 bitwise equal to one engine."""
    from paper_2207_09334_b200.sharded import ShardGroup
    line = _crawler_line(6)
    one = Engine(line, integrator=integrator, precision="f64")
    grp = ShardGroup.from_scene(line, 3, precision="f64", transport=transport, integrator=integrator)
    for n in (17, 300):
        one.step(n)
        grp.step(n)
        x, v = _assemble(grp)
        assert x.tobytes() == one.x.tobytes() and v.tobytes() == one.v.tobytes()


def _ipc_beam_worker(rank, world, port, steps, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2207_09334_b200.sharded import attach_halo, attach_peers, scene_slab, slab_ranges
        b = _loaded_beam()
        s = scene_slab(b, slab_ranges(b, world), rank)
        eng = Engine(s.scene, integrator="verlet", precision="f64", device=0)
        attach_halo(eng, s)
        attach_peers(eng, rank, world)
        eng.step(steps)
        q.put((rank, s.i_lo, eng.x[s.owned].copy(), eng.v[s.owned].copy(), None))
        eng.close()
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, -1, None, None, repr(exc)))


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_sharded_beam_across_processes():
    """The loaded beam in two processes (one slab each, CUDA-IPC mapped
    peer buffers, device-side flags): bitwise the single engine."""
    steps, world = 40, 2
    one = Engine(_loaded_beam(), precision="f64")
    one.step(steps)
    ref_x, ref_v = one.x.copy(), one.v.copy()
    one.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000) + 11
    procs = [ctx.Process(target=_ipc_beam_worker, args=(r, world, port, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=500) for _ in procs], key=lambda t: t[1])
    for p in procs:
        p.join(timeout=60)
    errs = [r[4] for r in res if r[4]]
    assert not errs, errs
    assert np.concatenate([r[2] for r in res]).tobytes() == ref_x.tobytes()
    assert np.concatenate([r[3] for r in res]).tobytes() == ref_v.tobytes()
