"""Host-side partition logic (CPU): every rank's local element set and ordering,
and — across two real processes (gloo) — agreement of both ends on the order of
the partition faces they exchange (SURVEY §8(e) protocol: sorted by the lower
rank's global face slot 4k+f)."""
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import dg_inputs as di
from paper_1211_0582_b200.dg import Solver


def _local(rank, P, VX, E, part=None, partition=0):
    s = Solver(2, device=-1, rank=rank, nranks=P, partition=partition)
    s.mesh_upload(VX, E, part)
    ids = s.local_elements()
    EToE, EToF, _, _ = s.get_maps()
    s.close()
    return ids, EToE, EToF


@pytest.mark.parametrize("P", [2, 3, 4])
def test_local_sets_cover_mesh_boundary_first(P):
    VX, E = di.kuhn_box(4)
    E, _ = di.shuffle_elements(E, 9)
    K = E.shape[0]
    part = np.random.default_rng(P).integers(0, P, K).astype(np.int32)
    owner = np.empty(K, np.int64)
    allids = []
    for r in range(P):
        ids, EToE, _ = _local(r, P, VX, E, part)
        assert np.all(part[ids] == r)
        owner[ids] = r
        allids.append(ids)
        # partition-boundary elements (a face on another rank) first, then the interior ones,
        # each group ascending (a stage writes the boundary tiles first: DESIGN.md §10)
        bnd = np.array([np.any(part[EToE[k]] != r) for k in ids])
        nb = int(bnd.sum())
        assert bnd[:nb].all() and not bnd[nb:].any()
        assert np.all(np.diff(ids[:nb]) > 0) and np.all(np.diff(ids[nb:]) > 0)
    assert sorted(np.concatenate(allids).tolist()) == list(range(K))


def test_default_partition_is_z_slabs_on_weak_scaling_mesh():
    P, n = 4, 3
    VX, E = di.kuhn_box(n, nz=n * P)
    K = E.shape[0]
    for r in range(P):
        ids, _, _ = _local(r, P, VX, E)
        assert sorted(ids.tolist()) == list(range(r * K // P, (r + 1) * K // P))
        zc = VX[E[ids]].mean(axis=1)[:, 2]
        assert zc.min() > r - 1e-12 and zc.max() < r + 1 - 1e-12   # z-slab [r, r+1)


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_rcb_partition_balanced_compact_and_shared(P):
    # recursive coordinate bisection (DG_PARTITION_RCB): every element owned once, part sizes
    # within one element of K/P, and far fewer partition faces than a random owner map
    VX, E = di.kuhn_box(4)
    E, _ = di.shuffle_elements(E, 3)
    K = E.shape[0]
    owner = -np.ones(K, np.int64)
    for r in range(P):
        ids, EToE, _ = _local(r, P, VX, E, partition=1)
        assert np.all(owner[ids] == -1)
        owner[ids] = r
        assert abs(len(ids) - K / P) <= 1
    assert np.all(owner >= 0)
    cross = int(sum(owner[k] != owner[EToE[k, f]] for k in range(K) for f in range(4)))
    rnd = np.random.default_rng(0).integers(0, P, K)
    cross_rnd = int(sum(rnd[k] != rnd[EToE[k, f]] for k in range(K) for f in range(4)))
    assert cross < 0.35 * cross_rnd
    # P = 2 on a cube: the split is the median plane of the first (x) axis
    if P == 2:
        xc = VX[E].mean(axis=1)[:, 0]
        assert xc[owner == 0].max() <= xc[owner == 1].min() + 1e-12


def _cross_faces(rank, peer, ids, EToE, EToF, part):
    """This rank's send order to `peer`: its faces toward peer sorted by the lower rank's slot."""
    out = []
    for k in ids:
        for f in range(4):
            k2, f2 = int(EToE[k, f]), int(EToF[k, f])
            if part[k2] == peer and k2 != k:
                key = 4 * k + f if rank < peer else 4 * k2 + f2
                out.append((key, 4 * k + f, 4 * k2 + f2))
    out.sort()
    return out


def _worker(rank, world, port, q, how="random"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        VX, E = di.kuhn_box(3)
        E, _ = di.shuffle_elements(E, 4)
        K = E.shape[0]
        if how == "rcb":  # the library's recursive coordinate bisection, computed by each process
            part = np.zeros(K, np.int32)
            for r in range(world):
                part[_local(r, world, VX, E, partition=1)[0]] = r
            ids, EToE, EToF = _local(rank, world, VX, E, partition=1)
        else:
            part = np.random.default_rng(11).integers(0, world, K).astype(np.int32)
            ids, EToE, EToF = _local(rank, world, VX, E, part)
        peer = 1 - rank
        mine = _cross_faces(rank, peer, ids, EToE, EToF, part)
        # exchange my (my_slot, their_slot) sequence; the peer's sequence must be the mirror
        import torch
        n_mine = torch.tensor([len(mine)], dtype=torch.int64)
        n_peer = torch.zeros(1, dtype=torch.int64)
        if rank == 0:
            dist.send(n_mine, 1); dist.recv(n_peer, 1)
        else:
            dist.recv(n_peer, 0); dist.send(n_mine, 0)
        assert int(n_peer) == len(mine)
        a = torch.tensor([[m, t] for _, m, t in mine], dtype=torch.int64)
        b = torch.zeros_like(a)
        if rank == 0:
            dist.send(a, 1); dist.recv(b, 1)
        else:
            dist.recv(b, 0); dist.send(a, 0)
        # record i that I send (my face m -> their face t) is what the peer receives for its face t from my m
        assert torch.equal(b[:, 0], a[:, 1]) and torch.equal(b[:, 1], a[:, 0])
        q.put((rank, len(mine), None))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, -1, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("how", ["random", "rcb"])
def test_two_process_gloo_ghost_face_order_agrees(how):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + (7 if how == "rcb" else 0)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, how)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, n, err in res:
        assert err is None, err
        assert n > 0
