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


def _route_part(c, world):
    """The product partition (libvol vol_partition_route) with a straight route along x through the block
    set: arc length = x of the block centre, ties by (x, y, z) — every rank gets one contiguous x range."""
    from paper_1604_03734_b200 import partition_route
    lo, hi = float(c[:, 0].min()), float(c[:, 0].max()) + 1.0
    return partition_route(c, np.array([[lo, 0.0, 0.0], [hi, 0.0, 0.0]]), 1.0, world)


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
        part = _route_part(c, world)
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
        part = _route_part(c, world)
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


def _exchange(plan, rank, world, local_n, row_of, fields):
    """One halo exchange over gloo in the plan's order: every peer gets its send blocks' rows of each
    field, and the ghost rows [local_n + recv_off, ...) receive the owners' rows (in place)."""
    off_s = np.concatenate([[0], np.cumsum(plan["peer_send"])])
    off_r = np.concatenate([[0], np.cumsum(plan["peer_recv"])])
    k = len(fields)
    reqs, keep = [], []
    for peer in range(world):
        if peer == rank:
            continue
        blk = [row_of[int(g)] for g in plan["send"][off_s[peer]:off_s[peer + 1]]]
        if blk:
            buf = torch.from_numpy(np.stack([np.asarray(fl[blk], np.float32) for fl in fields], 1).copy())
            keep.append(buf)
            reqs.append(dist.isend(buf, dst=peer))
        n = int(plan["peer_recv"][peer])
        if n:
            rb = torch.empty(n, k, 512)
            reqs.append((dist.irecv(rb, src=peer), rb, local_n + off_r[peer]))
    for r in reqs:
        if isinstance(r, tuple):
            r[0].wait()
            a, b = r[2], r[2] + len(r[1])
            for j, fl in enumerate(fields):
                fl[a:b] = r[1][:, j].numpy()
        else:
            r.wait()


def _skew_worker(rank, world, port, q, exchange_p):
    """The product (skewed) schedule of the sharded GPU path, replayed with the CPU oracle's phases on
    each rank's blocks plus the plan's ghost rows (csrc/shard.cu nccl_skew):
        X(ū^0, p^0) · dual · { X(u^j, p^{j+1}) · primal · dual }_{j < iters−1} · X(u, p^iters) · primal
    ū is never exchanged inside the loop: each rank recomputes the primal step of the ghost voxels from
    the exchanged u^j and p^{j+1} (the +face primal recompute of k_skew), and its own blocks must come
    out bit-identical to the single-volume oracle.  exchange_p=False drops p^{j+1} from the loop's
    messages (only u^j is sent): the ghosts' p is then the rank's own dual step of the ghost voxels,
    which reads ū beyond the halo, and the result must differ (the check has teeth).  (Dropping u^j
    instead would not: here every rank runs the primal phase on the ghost rows too, and a ghost
    face voxel's u^{j+1} depends only on its own u^j and on p^{j+1} of the voxel and its −neighbours,
    all exchanged or local; the kernels recompute that primal step without storing it and take u^j from
    the message.)"""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_1604_03734_b200 import plan_shard
        from synth import random_instance
        s = random_instance(500, seed=29, extent=6, w_density=0.75, w_max=3, lam=0.6, eps=0.02, iters=14)
        c = s.coords.numpy()
        f, W = s.f.numpy(), s.W.numpy()
        part = _route_part(c, world)
        plan = plan_shard(c, part, world, rank)
        local = np.nonzero(part == rank)[0]
        ghost = plan["ghost"]
        # context rows: the remaining face neighbours of the ghost blocks, with their static W only.  The
        # oracle masks p_a(v) by the validity of edge v → v + ê_a (Eq. 4 as written), which needs Ω one
        # block beyond a ghost; the kernels read p as stored instead (p_a = +0 on invalid edges, the
        # iteration's invariant), so the GPU path needs no such rows.  Their u and p are never exchanged
        # and never reach a local block's result.
        known = set(local.tolist()) | set(ghost.tolist())
        key = {tuple(x): i for i, x in enumerate(c.tolist())}
        ctx = sorted({key[t] for g in ghost for a in range(3) for d in (-1, 1)
                      for t in [tuple(c[g] + d * np.eye(3, dtype=np.int32)[a])] if t in key} - known)
        rows = np.concatenate([local, ghost, np.asarray(ctx, np.int64)]).astype(np.int64)
        row_of = {int(g): i for i, g in enumerate(rows)}
        cr, fr, Wr = c[rows], f[rows], W[rows]
        nbr = oracle.neighbours(cr)
        kw = dict(theta=s.theta, data_term=s.data_term, precision="f32", nbr=nbr)
        # init (warm): u = ū = f, p = 0 — zero iterations of the oracle
        u, ub, p = oracle.regularise(cr, fr, Wr, s.lam, s.eps, s.tau, s.sigma, 0, theta=s.theta,
                                     data_term=s.data_term, init=s.init, precision="f32", nbr=nbr)
        st = (u, ub, p)
        ph = lambda which: oracle.phase(cr, fr, Wr, s.lam, s.eps, s.tau, s.sigma, which, st, **kw)
        X = lambda ufield, loop=True: _exchange(plan, rank, world, len(local), row_of,
                                                [ufield] + ([p[0], p[1], p[2]] if exchange_p or not loop else []))
        X(ub, loop=False)
        ph("dual")
        for j in range(s.iters - 1):
            X(u)                  # (u^j, p^{j+1})
            ph("primal")          # u^{j+1}, ū^{j+1} (own rows and the ghost rows' recompute)
            ph("dual")            # p^{j+2}
        X(u)                      # (u^{iters-1}, p^{iters})
        ph("primal")
        u_single, _, _ = oracle.regularise_scene(s, precision="f32")
        ok = np.array_equal(u[:len(local)].view(np.uint32), u_single[local].view(np.uint32))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, len(ghost)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, f"error: {e!r}", 0))


def _run(target, world, *extra):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + extra) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(60)
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_skewed_schedule_oracle_equals_single_volume(world):
    from paper_1604_03734_b200 import build
    build.build()
    res = _run(_skew_worker, world, True)
    assert all(r[1] is True for r in res), res
    assert all(r[2] > 0 for r in res)


def test_gloo_skewed_schedule_needs_the_p_halo():
    from paper_1604_03734_b200 import build
    build.build()
    res = _run(_skew_worker, 2, False)
    assert all(not isinstance(r[1], str) for r in res), res
    assert not all(r[1] for r in res)


def _gid_worker(rank, world, port, q):
    """The binding's per-group NCCL unique id (volume._group_nccl_id): one id per live group, shared by all
    its ranks, a different id for a new group — even one created after the first is destroyed (weak keys
    plus the group's name and ranks; an id() key could hand the new group the old id)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1604_03734_b200 import volume
        g1 = dist.new_group(list(range(world)))
        a = volume._group_nccl_id(g1, "cpu")
        a2 = volume._group_nccl_id(g1, "cpu")
        dist.destroy_process_group(g1)
        del g1
        g2 = dist.new_group(list(range(world)))
        b = volume._group_nccl_id(g2, "cpu")
        ids = [None] * world
        dist.all_gather_object(ids, (a, b))
        ok = a == a2 and a != b and all(x == (a, b) for x in ids)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, 0))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, f"error: {e!r}", 0))


def test_group_unique_id_per_live_group():
    from paper_1604_03734_b200 import build
    build.build()
    res = _run(_gid_worker, 2)
    assert all(r[1] is True for r in res), res


def _gen_worker(rank, world, port, q):
    """bench.py's per-shard generation under torch.distributed (here gloo on the CPU): each rank generates
    the candidates of its arc range, all-gathers the allocated coordinates, takes the exact route partition
    and regenerates the blocks that changed owner.  The union over ranks must equal the single-process
    scene, block for block, and the owner map must be vol_partition_route of the whole block set."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        from paper_1604_03734_b200 import partition_route
        from synth import scenes
        plan = scenes.city_plan(0, length=6.0, device="cpu")
        c_r, f_r, W_r = bench.shard_generate(plan, world, rank, chunk_blocks=512)
        allc = bench.gather_coords(c_r, world, torch.device("cpu"))
        sh = bench.shard_assemble(plan, world, rank, allc, c_r, f_r, W_r, chunk_blocks=512)
        mine = torch.from_numpy(sh["part"] == rank)
        ok = np.array_equal(sh["part"], partition_route(sh["coords"], plan.route, plan.block_edge, world))
        fs = [None] * world
        dist.all_gather_object(fs, (sh["f"].numpy(), sh["W"].numpy()))
        if rank == 0:
            whole = scenes.city(0, length=6.0, chunk_blocks=512)
            coords = sh["coords"]
            f = torch.empty(coords.shape[0], 512)
            W = torch.empty(coords.shape[0], 512)
            for r, (fr, Wr) in enumerate(fs):
                m = torch.from_numpy(sh["part"] == r)
                f[m], W[m] = torch.from_numpy(fr), torch.from_numpy(Wr)
            key = lambda c: (c[:, 0].long() * 65536 + c[:, 1].long()) * 65536 + c[:, 2].long()
            i1, i2 = torch.argsort(key(coords)), torch.argsort(key(whole.coords))
            ok = ok and torch.equal(coords[i1], whole.coords[i2]) and torch.equal(f[i1], whole.f[i2]) \
                and torch.equal(W[i1], whole.W[i2])
        ok = ok and bool(mine.any())
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, int(sh["moved"])))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, f"error: {e!r}", 0))


def test_bench_per_shard_generation_gloo():
    from paper_1604_03734_b200 import build
    build.build()
    res = _run(_gen_worker, 2)
    assert all(r[1] is True for r in res), res
