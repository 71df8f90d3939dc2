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
def test_nccl_transport_self_loop():
    """Exercise the NCCL path on one GPU: a single rank whose lower and upper
    'neighbours' are itself.  After a step, each halo plane must hold the
    positions of the plane it is wired to (transport + pack/unpack check)."""
    import ctypes as C

    import torch  # noqa: F401  (loads libnccl.so.2 into the process)

    from paper_2207_09334_b200 import _lib
    from paper_2207_09334_b200.sharded import attach_halo
    cells = 5
    nx = cells + 1
    s = cube_slab(cells, 1, nx - 1, v_global=excited_velocities(nx ** 3))
    # fp64: absolute positions travel (in fp32 only the displacement r does,
    # which is consistent only between the two copies of the SAME mass)
    eng = Engine(s.scene, precision="f64")
    attach_halo(eng, s)
    uid = C.create_string_buffer(128)
    _lib.check(_lib.lib().ss_nccl_unique_id(uid))
    _lib.check(_lib.lib().ss_halo_nccl(eng.handle, uid.raw, 1, 0, 0, 0))
    eng.step(3)
    x = eng.x
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


def _ipc_worker(rank, world, port, cells, steps, precision, q):
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
        eng = Engine(s.scene, integrator="verlet", precision=precision, device=0)
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
def test_peer_memory_shards_across_processes():
    """Two processes, one shard each, sharing one GPU: mailboxes mapped with
    cudaIpcOpenMemHandle, planes pushed and landed every substep with no host
    round trip; the assembled fp64 state is bitwise the single engine's."""
    cells, steps, world = 9, 30, 2
    full = L.excite(L.block_scene(cells), seed=11)
    one = Engine(full, precision="f64")
    one.step(steps)
    ref_x, ref_v = one.x.copy(), one.v.copy()
    one.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000) + 7
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, cells, steps, "f64", q)) for r in range(world)]
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
