"""Python surface of the C ABI (SURVEY §8(b) "Python surface"): `Volume(coords, f, W, group=None)`,
`.regularise(...)`, `.u()`, `.energy(...)`.  PyTorch provides device memory (the workspace), the
CUDA stream and the process group; the method itself runs in libvol.so's kernels.

Inputs may be torch tensors (CUDA or CPU, pinned or not) or numpy arrays; the library detects
host/device pointers.  Names follow the paper: λ (lam), ε (eps, Huber), τ (tau), σ (sigma),
θ (theta), f (fused TSDF), W (fusion weight), u / ū (primal / relaxed primal), p (dual).
"""
from __future__ import annotations

import ctypes
import weakref

import numpy as np
import torch

from . import _native as N


def _ptr(x):
    """(pointer, keep-alive object) of a contiguous torch tensor or numpy array."""
    if isinstance(x, torch.Tensor):
        if not x.is_contiguous():
            x = x.contiguous()
        return ctypes.c_void_p(x.data_ptr()), x
    a = np.ascontiguousarray(x)
    return ctypes.c_void_p(a.ctypes.data), a


def _as(x, dtype_t, dtype_np):
    if isinstance(x, torch.Tensor):
        return x.to(dtype_t).contiguous() if x.dtype != dtype_t else x.contiguous()
    return np.ascontiguousarray(x, dtype=dtype_np)


def _require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1604_03734_b200 needs a CUDA device (B200); there is no CPU fallback")


def block_hash(x: int, y: int, z: int, T: int) -> int:
    return int(N.lib().vol_block_hash(x, y, z, T))


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    N.check(N.lib().vol_nccl_unique_id(buf))
    return buf.raw


def plan_shard(coords, part, world: int, rank: int) -> dict:
    """Host-only shard plan of `rank`; no GPU needed."""
    c = np.ascontiguousarray(coords, dtype=np.int32).reshape(-1, 3)
    pt = np.ascontiguousarray(part, dtype=np.int32)
    n = c.shape[0]
    L = N.lib()
    nl, ng, ns = (ctypes.c_int64() for _ in range(3))
    N.check(L.vol_plan_shard(c.ctypes.data, n, pt.ctypes.data, world, rank, ctypes.byref(nl), ctypes.byref(ng),
                             ctypes.byref(ns), None, None, None, None))
    ghost = np.zeros(max(ng.value, 1), np.int64)
    send = np.zeros(max(ns.value, 1), np.int64)
    psend = np.zeros(world, np.int64)
    precv = np.zeros(world, np.int64)
    N.check(L.vol_plan_shard(c.ctypes.data, n, pt.ctypes.data, world, rank, None, None, None, ghost.ctypes.data,
                             send.ctypes.data, psend.ctypes.data, precv.ctypes.data))
    return dict(n_local=nl.value, n_ghost=ng.value, ghost=ghost[:ng.value], send=send[:ns.value],
                peer_send=psend, peer_recv=precv)


def partition_route(coords, route, block_edge: float, world: int, return_arc: bool = False):
    """Route-axis partition (``vol_partition_route``; host only): owner rank per block —
    blocks ordered by the arc length of the nearest route point (ties by x, y, z), cut into `world`
    contiguous ranges of equal block count.  `route` is the polyline [m, 3] in metres, `block_edge`
    the block edge in metres (8 × voxel).  Returns int32 part [n] (and float64 arc [n])."""
    c = np.ascontiguousarray(coords.cpu().numpy() if isinstance(coords, torch.Tensor) else coords,
                             dtype=np.int32).reshape(-1, 3)
    r = np.ascontiguousarray(route, dtype=np.float64).reshape(-1, 3)
    part = np.zeros(c.shape[0], np.int32)
    arc = np.zeros(c.shape[0], np.float64)
    N.check(N.lib().vol_partition_route(c.ctypes.data, c.shape[0], r.ctypes.data, r.shape[0], float(block_edge),
                                        int(world), part.ctypes.data, arc.ctypes.data))
    return (part, arc) if return_arc else part


def release_comms():
    """Destroy libvol's cached NCCL communicators (teardown, after every sharded volume is closed)."""
    N.check(N.lib().vol_release_comms())


# one NCCL unique id per live process group: weak keys, so a destroyed group's entry disappears with it
# (an id() key could be reused by a later group and hand it a stale id); the group's name and ranks are
# checked too
_GROUP_IDS = weakref.WeakKeyDictionary()


def _group_nccl_id(group, device) -> bytes:
    """One NCCL unique id per torch.distributed group (created by the group's rank 0, broadcast once);
    libvol caches the communicator built from it, so later volumes of the group reuse it."""
    import torch.distributed as dist_mod
    sig = (getattr(group, "group_name", None), tuple(dist_mod.get_process_group_ranks(group)))
    ent = _GROUP_IDS.get(group)
    if ent is None or ent[0] != sig:
        idbuf = torch.zeros(128, dtype=torch.uint8)
        if dist_mod.get_rank(group) == 0:
            idbuf = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8).clone()
        src = dist_mod.get_global_rank(group, 0)
        if dist_mod.get_backend(group) == "nccl":
            idd = idbuf.to(device)
            dist_mod.broadcast(idd, src=src, group=group)
            idbuf = idd.cpu()
        else:
            dist_mod.broadcast(idbuf, src=src, group=group)
        _GROUP_IDS[group] = (sig, bytes(idbuf.numpy().tobytes()))
    return _GROUP_IDS[group][1]


class Volume:
    """A hashed voxel-block volume resident on one GPU (or one shard of a sharded volume).

    coords: int32 [n_global, 3] block coordinates; f, W: float32 [n_local, 512] (blocks this rank
    owns, in global order).  For sharding pass `part` (owner rank per block) and either a
    torch.distributed `group` (NCCL transport; the unique id is broadcast through the group) or
    `loopback=(rank, world)` for the one-process test transport.
    """

    def __init__(self, coords, f, W, *, part=None, group=None, loopback=None, device=None, stream=None):
        _require_cuda()
        self._lib = N.lib()
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        coords = _as(coords, torch.int32, np.int32)
        f = _as(f, torch.float32, np.float32)
        # W as uint8 (exact observation counts) takes vol_create_w8: a quarter of the bytes to copy
        w8 = (W.dtype == torch.uint8) if isinstance(W, torch.Tensor) else (np.asarray(W).dtype == np.uint8)
        W = _as(W, torch.uint8, np.uint8) if w8 else _as(W, torch.float32, np.float32)
        n = int(coords.shape[0])
        self.n_global = n
        dist = None
        self._keep = []
        if part is not None:
            part_np = np.ascontiguousarray(part.cpu().numpy() if isinstance(part, torch.Tensor) else part, dtype=np.int32)
            if group is not None:
                import torch.distributed as dist_mod
                rank, world = dist_mod.get_rank(group), dist_mod.get_world_size(group)
                nid = ctypes.create_string_buffer(_group_nccl_id(group, self.device), 128)
                self._keep.append(nid)
                dist = N.vol_dist(rank, world, part_np.ctypes.data, ctypes.cast(nid, ctypes.c_void_p))
            elif loopback is not None:
                rank, world = loopback
                dist = N.vol_dist(rank, world, part_np.ctypes.data, None)
            else:
                raise ValueError("part given without group or loopback")
            self._keep.append(part_np)
            self.rank, self.world = rank, world
        else:
            self.rank, self.world = 0, 1
        with torch.cuda.device(self.device):
            self.stream = torch.cuda.current_stream(self.device) if stream is None else stream
            cp, ck = _ptr(coords)
            fp, fk = _ptr(f)
            wp, wk = _ptr(W)
            dptr = ctypes.byref(dist) if dist is not None else None
            if dist is not None and isinstance(coords, torch.Tensor) and coords.is_cuda:
                # vol_workspace_bytes reads device coordinates on the legacy default stream (it takes no
                # stream): they must be complete
                self.stream.synchronize()
            nbytes = self._lib.vol_workspace_bytes(cp, n, dptr)
            if nbytes == 0:
                raise N.VolError(N.VOL_EINVAL, "vol_workspace_bytes failed (bad coordinates or partition)")
            self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
            h = ctypes.c_void_p()
            create = self._lib.vol_create_w8 if w8 else self._lib.vol_create
            N.check(create(cp, n, fp, wp, dptr, ctypes.c_void_p(self.workspace.data_ptr()), nbytes,
                           ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h)))
            del ck, fk, wk
        self._h = h
        nl, ng, no = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        N.check(self._lib.vol_info(self._h, ctypes.byref(nl), ctypes.byref(ng), ctypes.byref(no)))
        self.n_local, self.n_ghost, self.n_omega = nl.value, ng.value, no.value

    # -- solver ---------------------------------------------------------------------------------
    @staticmethod
    def _opts(theta=1.0, data_term=0, init=0, resume=False, kernel=0, freeze=True, exchange=True):
        o = N.vol_opts()
        N.lib().vol_default_opts(ctypes.byref(o))
        o.theta, o.data_term, o.init, o.resume, o.kernel = float(theta), int(data_term), int(init), int(bool(resume)), int(kernel)
        o.freeze = int(bool(freeze))
        o.exchange = int(bool(exchange))
        return o

    def regularise(self, lam: float, eps: float, tau: float, sigma: float, iters: int, *, theta: float = 1.0,
                   data_term: int = 0, init: int = 0, resume: bool = False, kernel: int = 0, freeze: bool = True,
                   exchange: bool = True):
        """`iters` Chambolle–Pock iterations (asynchronous on the volume's stream).  `exchange=False`
        (sharded volumes) replaces the halo exchange by a no-op: wrong results, timing only."""
        o = self._opts(theta, data_term, init, resume, kernel, freeze, exchange)
        N.check(self._lib.vol_regularise(self._h, lam, eps, tau, sigma, int(iters), ctypes.byref(o)))
        return self

    def regularise_scene(self, scene, iters=None, **kw):
        it = scene.iters if iters is None else iters
        kw.setdefault("theta", scene.theta)
        kw.setdefault("data_term", scene.data_term)
        kw.setdefault("init", scene.init)
        return self.regularise(scene.lam, scene.eps, scene.tau, scene.sigma, it, **kw)

    def shard_timing(self):
        """(interior_ms, exchange_ms, boundary_ms) of the last iteration of the last sharded call: launch A,
        the halo chain (pack → NCCL → unpack, communication stream) and launch B, from CUDA events."""
        a, c, b = ctypes.c_float(), ctypes.c_float(), ctypes.c_float()
        N.check(self._lib.vol_shard_timing(self._h, ctypes.byref(a), ctypes.byref(c), ctypes.byref(b)))
        return a.value, c.value, b.value

    @property
    def last_launches(self) -> int:
        return int(self._lib.vol_last_launches(self._h))

    def sync(self):
        N.check(self._lib.vol_sync(self._h))

    # -- read-back ------------------------------------------------------------------------------
    def read_u(self, out):
        """Copy u [n_local, 512] into `out` (host or device tensor / numpy array)."""
        p, k = _ptr(out)
        N.check(self._lib.vol_read_u(self._h, p))
        return out

    def u(self, device=None) -> torch.Tensor:
        out = torch.empty(self.n_local, 512, dtype=torch.float32, device=self.device if device is None else device)
        self.read_u(out)
        if out.device.type == "cuda":
            self.sync()
        return out

    def energy(self, lam: float, eps: float, data_term: int = 0):
        """(primal, dual) energies of the current state (fp64, deterministic)."""
        P, D = ctypes.c_double(), ctypes.c_double()
        N.check(self._lib.vol_energy(self._h, lam, eps, data_term, ctypes.byref(P), ctypes.byref(D)))
        return P.value, D.value

    def state(self, device="cpu"):
        """(u, ū, p[3]) in the caller's block order, as tensors on `device` (CPU by default)."""
        u = torch.empty(self.n_local, 512, device=device)
        ub = torch.empty(self.n_local, 512, device=device)
        p = torch.empty(3, self.n_local, 512, device=device)
        N.check(self._lib.vol_read_state(self._h, ctypes.c_void_p(u.data_ptr()), ctypes.c_void_p(ub.data_ptr()),
                                         ctypes.c_void_p(p.data_ptr())))
        if u.device.type == "cuda":
            self.sync()
        return u, ub, p

    def load_state(self, u, ub, p):
        keep = [_ptr(_as(x, torch.float32, np.float32)) for x in (u, ub, p)]
        N.check(self._lib.vol_load_state(self._h, *(k[0] for k in keep)))

    def tables(self):
        """(T, bucket_start[T+1] uint32, bucket_entry[n] int32, nbr[n, 6] int32) as numpy arrays."""
        T = ctypes.c_uint32()
        N.check(self._lib.vol_read_tables(self._h, ctypes.byref(T), None, None, None))
        bs = np.zeros(T.value + 1, np.uint32)
        be = np.zeros(self.n_global, np.int32)
        nbr = np.zeros((self.n_global, 6), np.int32)
        N.check(self._lib.vol_read_tables(self._h, None, bs.ctypes.data, be.ctypes.data, nbr.ctypes.data))
        return T.value, bs, be, nbr

    # -- surface -----------------------------------------------------------
    def extract(self, voxel: float, w_min: float = 0.0, field: str = "u", device=None, out=None) -> torch.Tensor:
        """Ω-restricted zero level set of u (or f) as a triangle soup [m, 3, 3] float32 (vol_extract).
        With `out` (a float32 [cap, 3, 3] tensor) the triangles go into it in one call if they fit."""
        fid = {"u": 0, "f": 1}[field]
        if out is not None:
            m = ctypes.c_int64()
            st = self._lib.vol_extract(self._h, fid, float(voxel), float(w_min), ctypes.c_void_p(out.data_ptr()),
                                       int(out.shape[0]), ctypes.byref(m))
            if st == N.VOL_OK:
                return out[:m.value]
            if st != N.VOL_ENOMEM:
                N.check(st)
        n = ctypes.c_int64()
        N.check(self._lib.vol_extract(self._h, fid, float(voxel), float(w_min), None, 0, ctypes.byref(n)))
        out = torch.empty(max(n.value, 1), 3, 3, dtype=torch.float32, device=self.device if device is None else device)
        m = ctypes.c_int64()
        N.check(self._lib.vol_extract(self._h, fid, float(voxel), float(w_min), ctypes.c_void_p(out.data_ptr()),
                                      n.value, ctypes.byref(m)))
        return out[:m.value]

    # -- direct-store halo transport (vol.h "Direct-store halo transport") --------------------------
    def peer_info(self) -> np.ndarray:
        n = ctypes.c_int64()
        N.check(self._lib.vol_peer_info(self._h, None, 0, ctypes.byref(n)))
        info = np.zeros(n.value, np.int64)
        N.check(self._lib.vol_peer_info(self._h, info.ctypes.data, n.value, ctypes.byref(n)))
        return info

    def connect_peer(self, peer: int, workspace_ptr: int, info: np.ndarray):
        info = np.ascontiguousarray(info, np.int64)
        N.check(self._lib.vol_connect_peer(self._h, int(peer), ctypes.c_void_p(int(workspace_ptr)), info.ctypes.data,
                                           info.shape[0]))

    def ipc_handle(self):
        buf = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        N.check(self._lib.vol_ipc_handle(self._h, buf, ctypes.byref(off)))
        return buf.raw, off.value

    def connect_peer_ipc(self, peer: int, handle: bytes, offset: int, info: np.ndarray):
        info = np.ascontiguousarray(info, np.int64)
        hb = ctypes.create_string_buffer(bytes(handle), 64)
        N.check(self._lib.vol_connect_peer_ipc(self._h, int(peer), hb, int(offset), info.ctypes.data, info.shape[0]))

    @property
    def transport(self) -> str:
        return {0: "none", 1: "nccl", 2: "loopback", 3: "peer"}[int(self._lib.vol_transport(self._h))]

    def connect_peers(self, group):
        """Direct-store transport over a torch.distributed group (collective): every rank publishes its
        workspace's CUDA IPC handle and peer descriptor, and opens its peers' (NVLink peer access)."""
        import torch.distributed as dist_mod
        handle, off = self.ipc_handle()
        mine = (self.rank, handle, off, self.peer_info().tolist())
        allv = [None] * dist_mod.get_world_size(group)
        dist_mod.all_gather_object(allv, mine, group=group)
        for q, h, o, info in allv:
            if q != self.rank:
                self.connect_peer_ipc(q, h, o, np.asarray(info, np.int64))

    def close(self):
        if getattr(self, "_h", None):
            self._lib.vol_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


# -- TSDF fusion (paper §III-A, Eq. 1) -----------------------------------------

_fuse_cap_hint = [65536]


def fuse(depth, poses, intr, voxel: float, mu: float, max_range: float, w_max: float, *, max_blocks=None,
         stream=None, return_first=True, stats=None, prev=None):
    """Fuse K posed depth maps into hashed voxel blocks on the GPU (``vol_fuse``).

    depth [K, H, W] float32 metres, poses [K, 12] float32 row-major T_gc (camera-to-global), intr
    (fx, fy, cx, cy).  Returns CUDA tensors (coords int32 [n, 3] sorted by (x, y, z), first frame
    int32 [n], f float32 [n, 512], W float32 [n, 512]) — ready for :class:`Volume`.  Pass a dict as
    `stats` to receive the call's counters (pixels_valid, blocks, block_frames, voxel_updates; this
    synchronises the stream).  `prev` = (coords, f, W) of an earlier fusion continues it with the new depth
    maps (vol_fuse_incremental, reading F-11): the result equals fusing all frames in one call.
    """
    _require_cuda()
    L = N.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    depth = depth if isinstance(depth, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(depth, np.float32))
    poses = poses if isinstance(poses, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(poses, np.float32))
    depth = depth.to(torch.float32).contiguous()
    if depth.dim() == 2:
        depth = depth[None]
    poses = poses.to(torch.float32).reshape(-1, 12).contiguous()
    K, H, Wd = (int(v) for v in depth.shape)
    if poses.shape[0] != K:
        raise ValueError(f"{poses.shape[0]} poses for {K} depth maps")
    it = [float(v) for v in (intr.tolist() if hasattr(intr, "tolist") else intr)]
    cam = N.vol_camera(it[0], it[1], it[2], it[3], Wd, H)
    prm = N.vol_fusion_params(float(voxel), float(mu), float(max_range), float(w_max))
    s = torch.cuda.current_stream(dev) if stream is None else stream
    if prev is not None:
        pxyz = _as(prev[0], torch.int32, np.int32)
        pf = _as(prev[1], torch.float32, np.float32)
        pW = _as(prev[2], torch.float32, np.float32)
        n_prev = int(pxyz.shape[0])
        (pxp, pxk), (pfp, pfk), (pwp, pwk) = _ptr(pxyz), _ptr(pf), _ptr(pW)
    else:
        n_prev, pxp, pfp, pwp = 0, None, None, None
    # capacity: twice the block count of the previous call (a high-water hint like an allocator's, so a
    # stream of similar fusions sizes its buffers right the first time), at least 2·n_prev and 65536;
    # on overflow the call is retried with 4x the capacity
    cap = int(max_blocks) if max_blocks else max(65536, 2 * n_prev, _fuse_cap_hint[0])
    while True:
        xyz = torch.empty(cap, 3, dtype=torch.int32, device=dev)
        first = torch.empty(cap, dtype=torch.int32, device=dev)
        f = torch.empty(cap, 512, dtype=torch.float32, device=dev)
        W = torch.empty(cap, 512, dtype=torch.float32, device=dev)
        nbytes = L.vol_fuse_workspace_bytes(cap, K, ctypes.byref(cam))
        ws = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
        n = ctypes.c_int64()
        sts = N.vol_fusion_stats()
        st = L.vol_fuse_incremental(pxp, pfp, pwp, n_prev, ctypes.c_void_p(depth.data_ptr()), K, ctypes.byref(cam),
                        ctypes.c_void_p(poses.data_ptr()),
                        ctypes.byref(prm), cap, ctypes.c_void_p(ws.data_ptr()), nbytes, ctypes.c_void_p(s.cuda_stream),
                        ctypes.c_void_p(xyz.data_ptr()), ctypes.c_void_p(first.data_ptr()),
                        ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(W.data_ptr()), ctypes.byref(n),
                        ctypes.byref(sts) if stats is not None else None)
        if st == N.VOL_ENOMEM and not max_blocks and n.value > cap:
            cap = 4 * cap      # the count reached is only a lower bound once the capacity is exceeded
            continue
        N.check(st)
        break
    m = n.value
    if not max_blocks:
        _fuse_cap_hint[0] = max(65536, 2 * m)
    if stats is not None:
        stats.update({k: getattr(sts, k) for k, _ in N.vol_fusion_stats._fields_})
    out = (xyz[:m], first[:m], f[:m], W[:m])
    return out if return_first else (out[0], out[2], out[3])


# -- loopback groups (one process, one GPU; tests of the sharded path) --------------------------------

def _handles(vols):
    arr = (ctypes.c_void_p * len(vols))(*[v._h.value for v in vols])
    return arr


def connect_group(vols, transport: str = "copy"):
    """Connect loopback shards (one process).  transport "copy": pack → device copies → unpack per exchange;
    "peer": the direct-store transport, each volume writing its boundary blocks into the others'
    workspaces (the in-process form of the NVLink peer path)."""
    N.check(N.lib().vol_group_connect(_handles(vols), len(vols)))
    if transport == "peer":
        infos = [v.peer_info() for v in vols]
        for r, v in enumerate(vols):
            for q, w in enumerate(vols):
                if q != r:
                    v.connect_peer(q, w.workspace.data_ptr(), infos[q])
    elif transport != "copy":
        raise ValueError(transport)


def regularise_group(vols, lam, eps, tau, sigma, iters, **kw):
    o = Volume._opts(**kw)
    N.check(N.lib().vol_regularise_group(_handles(vols), len(vols), lam, eps, tau, sigma, int(iters), ctypes.byref(o)))


def group_energy(vols, lam, eps, data_term=0):
    P, D = ctypes.c_double(), ctypes.c_double()
    N.check(N.lib().vol_group_energy(_handles(vols), len(vols), lam, eps, data_term, ctypes.byref(P), ctypes.byref(D)))
    return P.value, D.value
