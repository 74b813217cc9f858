"""Python surface of the depth-map estimation ABI (include/vol.h: vol_stereo, vol_stereo_census,
vol_stereo_tensor, vol_disparity_to_depth; paper §IV).  Argument marshalling only — every step runs in
libvol.so's kernels; no CPU fallback."""
from __future__ import annotations

import ctypes

import torch

from . import _native as N


def _cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1604_03734_b200.stereo needs a CUDA device (B200); there is no CPU fallback")


def params(width, height, **kw) -> N.vol_stereo_params:
    """vol_stereo_params with the library defaults (Table I weights), overridden by keyword."""
    p = N.vol_stereo_params()
    N.lib().vol_stereo_default_params(ctypes.byref(p))
    p.width, p.height = int(width), int(height)
    names = {name for name, _ in N.vol_stereo_params._fields_}
    for k, v in kw.items():
        k = "lam" if k == "lambda_" else k
        if k not in names:
            raise TypeError(f"unknown stereo parameter {k!r} (known: {sorted(names - {'width', 'height'})})")
        setattr(p, k, v)
    return p


_WS = {}


def _f32(x, dev):
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(x)
    return t.to(device=dev, dtype=torch.float32).contiguous()


def stereo(left, right, *, stream=None, return_all=False, **kw):
    """Disparity maps [F, H, W] of rectified pairs left, right [F, H, W] (or [H, W]) on the GPU."""
    _cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    L = _f32(left, dev)
    R = _f32(right, dev)
    squeeze = L.dim() == 2
    if squeeze:
        L, R = L[None], R[None]
    F, H, W = (int(v) for v in L.shape)
    p = params(W, H, **kw)
    d = torch.empty(F, H, W, device=dev)
    w = torch.empty(2, F, H, W, device=dev) if return_all else None
    a = torch.empty(F, H, W, device=dev) if return_all else None
    s = torch.cuda.current_stream(dev) if stream is None else stream
    nbytes = int(N.lib().vol_stereo_workspace_bytes(F, ctypes.byref(p)))
    # one workspace per (device, size), reused across calls: the library caches the captured solve
    # (a CUDA graph) per workspace and parameter set
    key = (dev.index, nbytes)
    ws = _WS.get(key)
    if ws is None:
        if len(_WS) >= 4:
            _WS.pop(next(iter(_WS)))
        ws = _WS[key] = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    ptr = lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None
    N.check(N.lib().vol_stereo(ptr(L), ptr(R), F, ctypes.byref(p), ptr(ws), nbytes, ctypes.c_void_p(s.cuda_stream),
                               ptr(d), ptr(w), ptr(a)))
    if squeeze:
        d = d[0]
        if return_all:
            w, a = w[:, 0], a[0]
    return (d, w, a) if return_all else d


def census(img, window=5):
    _cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    I = _f32(img, dev)
    I3 = I[None] if I.dim() == 2 else I
    F, H, W = (int(v) for v in I3.shape)
    out = torch.empty(F, H, W, dtype=torch.int32, device=dev)
    N.check(N.lib().vol_stereo_census(ctypes.c_void_p(I3.data_ptr()), F, H, W, window,
                                      ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream),
                                      ctypes.c_void_p(out.data_ptr())))
    return out[0] if I.dim() == 2 else out


def tensor(img, beta=1.0, gamma=4.0):
    """(T11, T12, T22) stacked as [3, F, H, W] (or [3, H, W])."""
    _cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    I = _f32(img, dev)
    I3 = I[None] if I.dim() == 2 else I
    F, H, W = (int(v) for v in I3.shape)
    out = torch.empty(3, F, H, W, device=dev)
    N.check(N.lib().vol_stereo_tensor(ctypes.c_void_p(I3.data_ptr()), F, H, W, float(beta), float(gamma),
                                      ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream),
                                      ctypes.c_void_p(out.data_ptr())))
    return out[:, 0] if I.dim() == 2 else out


def disparity_to_depth(disp, fx_baseline, d_min=0.0):
    _cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    D = _f32(disp, dev)
    out = torch.empty_like(D)
    N.check(N.lib().vol_disparity_to_depth(ctypes.c_void_p(D.data_ptr()), D.numel(), float(fx_baseline),
                                           float(d_min), ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream),
                                           ctypes.c_void_p(out.data_ptr())))
    return out
