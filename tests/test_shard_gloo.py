"""World-size-2 (and 3) gloo run of the sharded path's host logic on CPU: every rank builds its shard plan
with libvol's `vol_plan_shard` (the same planner `vol_create` uses for the NCCL transport), then performs
the per-iteration halo exchange schedule — one message per peer, blocks in the plan's send order, received
into the ghost rows in the plan's receive order — over a torch.distributed gloo process group, and checks
that every ghost row holds exactly the owner's data."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1604_03734_b200 import plan_shard
        from synth import random_instance
        s = random_instance(600, seed=21, extent=6)
        c = s.coords.numpy()
        # contiguous ranges along x (the route axis), ties by y then z
        key = (c[:, 0].astype(np.int64) * 4096 + c[:, 1]) * 4096 + c[:, 2]
        order = np.argsort(key, kind="stable")
        part = np.empty(len(c), np.int32)
        for r in range(world):
            part[order[r * len(c) // world:(r + 1) * len(c) // world]] = r
        plan = plan_shard(c, part, world, rank)
        local = np.nonzero(part == rank)[0]
        assert plan["n_local"] == len(local)
        # the message payload per block: the owner's (ū, p_x, p_y, p_z) rows; here f and W stand in
        f = s.f.numpy()
        W = s.W.numpy()
        send_g = plan["send"]
        ghost_g = plan["ghost"]
        recv = np.zeros((len(ghost_g), 2, 512), np.float32)
        off_s = np.concatenate([[0], np.cumsum(plan["peer_send"])])
        off_r = np.concatenate([[0], np.cumsum(plan["peer_recv"])])
        reqs = []
        sendbufs = []
        for peer in range(world):
            if peer == rank:
                continue
            blk = send_g[off_s[peer]:off_s[peer + 1]]
            assert np.all(part[blk] == rank)
            buf = torch.from_numpy(np.stack([f[blk], W[blk]], 1).copy())
            sendbufs.append(buf)
            if len(blk):
                reqs.append(dist.isend(buf, dst=peer))
            n = int(plan["peer_recv"][peer])
            if n:
                rb = torch.empty(n, 2, 512)
                reqs.append((dist.irecv(rb, src=peer), rb, off_r[peer]))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                recv[r[2]:r[2] + len(r[1])] = r[1].numpy()
            else:
                r.wait()
        # every ghost row holds the owner's data, and the ghost set is what the stencil reads
        assert np.array_equal(recv[:, 0], f[ghost_g]) and np.array_equal(recv[:, 1], W[ghost_g])
        assert np.all(part[ghost_g] != rank)
        counts = torch.tensor([plan["n_local"], plan["n_ghost"]])
        allc = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, counts)
        assert sum(int(a[0]) for a in allc) == len(c)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", int(plan["n_ghost"])))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, f"error: {e!r}", 0))


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_halo_exchange(world):
    from paper_1604_03734_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(60)
    assert all(r[1] == "ok" for r in res), res
    assert all(r[2] > 0 for r in res)


def _oracle_worker(rank, world, port, q):
    """Sharded Chambolle–Pock on the CPU oracle: each rank iterates its own blocks plus the plan's ghost
    rows one iteration at a time and refreshes the ghosts' (ū, p) from their owners over gloo between
    iterations — the data the GPU path exchanges.  Its own blocks must equal the single-volume oracle
    bit for bit (SURVEY §8(e) correctness gate, exercised here without CUDA)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_1604_03734_b200 import plan_shard
        from synth import random_instance
        s = random_instance(500, seed=23, extent=6, w_density=0.75, w_max=3, lam=0.6, eps=0.02, iters=12)
        c = s.coords.numpy()
        f, W = s.f.numpy(), s.W.numpy()
        key = (c[:, 0].astype(np.int64) * 4096 + c[:, 1]) * 4096 + c[:, 2]
        order = np.argsort(key, kind="stable")
        part = np.empty(len(c), np.int32)
        for r in range(world):
            part[order[r * len(c) // world:(r + 1) * len(c) // world]] = r
        plan = plan_shard(c, part, world, rank)
        local = np.nonzero(part == rank)[0]
        ghost = plan["ghost"]
        rows = np.concatenate([local, ghost])
        row_of = {int(g): i for i, g in enumerate(rows)}
        off_s = np.concatenate([[0], np.cumsum(plan["peer_send"])])
        off_r = np.concatenate([[0], np.cumsum(plan["peer_recv"])])
        kw = dict(theta=s.theta, data_term=s.data_term, init=s.init, precision="f32")
        state = None
        for it in range(s.iters):
            state = oracle.regularise(c[rows], f[rows], W[rows], s.lam, s.eps, s.tau, s.sigma, 1, state=state, **kw)
            u, ub, p = state
            reqs, keep = [], []
            for peer in range(world):
                if peer == rank:
                    continue
                blk = [row_of[int(g)] for g in plan["send"][off_s[peer]:off_s[peer + 1]]]
                if blk:
                    buf = torch.from_numpy(np.stack([ub[blk], p[0][blk], p[1][blk], p[2][blk]], 1).copy())
                    keep.append(buf)
                    reqs.append(dist.isend(buf, dst=peer))
                n = int(plan["peer_recv"][peer])
                if n:
                    rb = torch.empty(n, 4, 512)
                    reqs.append((dist.irecv(rb, src=peer), rb, len(local) + off_r[peer]))
            for r in reqs:
                if isinstance(r, tuple):
                    r[0].wait()
                    a, b = r[2], r[2] + len(r[1])
                    ub[a:b] = r[1][:, 0].numpy()
                    for k in range(3):
                        p[k][a:b] = r[1][:, 1 + k].numpy()
                else:
                    r.wait()
            state = (u, ub, p)
        u_single, _, _ = oracle.regularise_scene(s, precision="f32")
        ok = np.array_equal(state[0][:len(local)].view(np.uint32), u_single[local].view(np.uint32))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok" if ok else "u differs from the single-volume oracle", len(ghost)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, f"error: {e!r}", 0))


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_oracle_equals_single_volume(world):
    from paper_1604_03734_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_oracle_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
    assert all(r[1] == "ok" for r in res), res
    assert all(r[2] > 0 for r in res)
