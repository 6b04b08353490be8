"""Thin ctypes binding of ``libglint.so`` (include/glint.h). Argument
marshalling only: every step of the glint path runs in the CUDA kernel.

There is no CPU fallback: if the library is missing or no sm_100 device is
present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GLINT_LIB") or os.path.join(_HERE, "libglint.so")

GLINT_OK, GLINT_EINVAL, GLINT_EALIGN, GLINT_EDEVICE, GLINT_ELIMIT, GLINT_ECUDA, GLINT_ENOMEM, GLINT_EALIAS = \
    0, -1, -2, -3, -4, -5, -6, -7
FLAG_INVALID, FLAG_DEGENERATE, FLAG_RATIO_CLAMPED, FLAG_P_CLAMPED, FLAG_UV_RANGE = 1, 2, 4, 8, 16
MAX_LIGHTS = 16
ZQ = 4096
NANG = 256

EXPORTS = ["glint_version", "glint_strerror", "glint_last_cuda_error", "glint_build_tables", "glint_create",
           "glint_destroy", "glint_eval", "glint_eval_batch", "glint_eval_host", "glint_eval_host_batch",
           "glint_get_tables", "glint_launch_count", "glint_count_active"]


class GlintError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        msg = f"{what} failed: {code} ({strerror(code)})"
        if code == GLINT_ECUDA:
            msg += f", cudaError {lib().glint_last_cuda_error()}"
        super().__init__(msg)


class glint_light(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pos_or_dir", C.c_float * 3), ("intensity", C.c_float * 3),
                ("reserved", C.c_int32)]


class glint_scene(C.Structure):
    _fields_ = [("seed", C.c_uint32), ("ndf_kind", C.c_int32), ("max_ratio_level", C.c_int32),
                ("beta", C.c_float), ("f0", C.c_float * 3), ("view_kind", C.c_int32), ("view", C.c_float * 3),
                ("n_lights", C.c_int32), ("eval_mode", C.c_int32), ("reserved", C.c_int32 * 3),
                ("lights", glint_light * MAX_LIGHTS)]


class glint_gbuffer(C.Structure):
    _fields_ = [("duv", C.c_void_p), ("uvm", C.c_void_p), ("nrm", C.c_void_p), ("pos", C.c_void_p),
                ("mat", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32), ("pitch", C.c_int64),
                ("x0", C.c_int32), ("y0", C.c_int32)]


# glint_debug_rec (184 words) as a numpy structured dtype
DEBUG_REC_DTYPE = np.dtype([
    ("P", "<f4"), ("r", "<f4"), ("psi", "<f4"),
    ("ls", "<i4", 4), ("lr", "<i4", 4), ("jo", "<i4", 4),
    ("w", "<f4", 4), ("n", "<f4", 4),
    ("lx", "<i4", 12), ("ly", "<i4", 12),
    ("p", "<f4"), ("cx0", "<i4"), ("cy0", "<i4"),
    ("T", "<u4", 4), ("sigma", "<f4", 4), ("m1", "<f4", 4), ("cap", "<f4", 4),
    ("hash", "<u4", 48), ("count", "<f4", 48),
    ("C", "<f4"), ("Dp", "<f4"), ("flags", "<u4"), ("light_active", "<u4"), 
    ("sfx", "<f4", 4), ("sfy", "<f4", 4), ("afx", "<f4"), ("afy", "<f4"), ("pge1", "<f4", 4), ("reserved", "<u4", 4),
])
DEBUG_REC_BYTES = 184 * 4
assert DEBUG_REC_DTYPE.itemsize == DEBUG_REC_BYTES

_lib = None


def lib():
    """Load libglint.so (built in-tree by __graft_entry__.build()). Raises if
    it is missing: there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        L.glint_version.restype = C.c_int
        L.glint_strerror.argtypes = [C.c_int]
        L.glint_strerror.restype = C.c_char_p
        L.glint_last_cuda_error.restype = C.c_int
        L.glint_build_tables.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.glint_build_tables.restype = C.c_int
        L.glint_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
        L.glint_create.restype = C.c_int
        L.glint_destroy.argtypes = [C.c_void_p]
        L.glint_destroy.restype = C.c_int
        L.glint_eval.argtypes = [C.c_void_p, C.POINTER(glint_gbuffer), C.POINTER(glint_scene), C.c_void_p,
                                 C.c_int64, C.c_void_p, C.c_void_p]
        L.glint_eval.restype = C.c_int
        L.glint_eval_batch.argtypes = [C.c_void_p, C.c_int, C.POINTER(glint_gbuffer), C.POINTER(glint_scene),
                                       C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_void_p]
        L.glint_eval_batch.restype = C.c_int
        L.glint_eval_host.argtypes = [C.c_void_p, C.POINTER(glint_gbuffer), C.POINTER(glint_scene), C.c_void_p,
                                      C.c_int64, C.c_void_p]
        L.glint_eval_host.restype = C.c_int
        L.glint_eval_host_batch.argtypes = [C.c_void_p, C.c_int, C.POINTER(glint_gbuffer), C.POINTER(glint_scene),
                                            C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.c_void_p]
        L.glint_eval_host_batch.restype = C.c_int
        L.glint_get_tables.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.glint_get_tables.restype = C.c_int
        L.glint_launch_count.argtypes = [C.c_void_p]
        L.glint_launch_count.restype = C.c_int64
        L.glint_count_active.argtypes = [C.c_void_p, C.POINTER(glint_gbuffer), C.POINTER(glint_scene), C.c_void_p,
                                         C.c_void_p]
        L.glint_count_active.restype = C.c_int
        _lib = L
    return _lib


def strerror(code: int) -> str:
    return lib().glint_strerror(code).decode()


def version() -> int:
    return lib().glint_version()


def build_tables():
    """Host-side tables exactly as glint_create uploads them (no GPU needed)."""
    z = np.zeros(ZQ, np.float32)
    c = np.zeros(NANG, np.float32)
    s = np.zeros(NANG, np.float32)
    rc = lib().glint_build_tables(z.ctypes.data, c.ctypes.data, s.ctypes.data)
    if rc:
        raise GlintError(rc, "glint_build_tables")
    return z, c, s


def scene_struct(scene) -> glint_scene:
    s = glint_scene()
    s.seed = int(scene.seed) & 0xFFFFFFFF
    s.ndf_kind = {"ggx": 0, "beckmann": 1}[scene.ndf]
    s.max_ratio_level = int(scene.max_ratio_level)
    s.beta = float(scene.beta)
    s.f0[:] = [float(x) for x in scene.f0]
    s.view_kind = {"point": 0, "directional": 1}[scene.view_kind]
    s.view[:] = [float(x) for x in scene.view]
    if len(scene.lights) > MAX_LIGHTS:
        raise ValueError(f"at most {MAX_LIGHTS} lights")
    s.n_lights = len(scene.lights)
    s.eval_mode = 3 if getattr(scene, "method", "ours") == "zk" else {48: 0, 64: 1, 160: 2}[int(getattr(scene, "draws", 48))]
    for i, lt in enumerate(scene.lights):
        s.lights[i].kind = {"point": 0, "directional": 1}[lt.kind]
        s.lights[i].pos_or_dir[:] = [float(x) for x in lt.pos_or_dir]
        s.lights[i].intensity[:] = [float(x) for x in lt.intensity]
    return s


def _gbuffer_struct(gb, origin=(0, 0)) -> glint_gbuffer:
    planes = gb.planes()
    H, W = int(planes[0].shape[0]), int(planes[0].shape[1])
    for p in planes:
        if tuple(p.shape) != (H, W, 4) or p.dtype.__str__() not in ("torch.float32",):
            raise ValueError("G-buffer planes must be float32 tensors of shape (H, W, 4)")
        if p.stride(2) != 1 or p.stride(1) != 4:
            raise ValueError("G-buffer planes must be (row-)contiguous float4 arrays")
    pitch = planes[0].stride(0) // 4
    if any(p.stride(0) // 4 != pitch for p in planes):
        raise ValueError("all planes must share one row pitch")
    g = glint_gbuffer()
    g.duv, g.uvm, g.nrm, g.pos, g.mat = [p.data_ptr() for p in planes]
    g.width, g.height, g.pitch = W, H, pitch
    g.x0, g.y0 = int(origin[0]), int(origin[1])
    return g


def _check_out(out, g, device_type: str, what: str):
    """The output must hold the tile at its origin: float32, (rows, cols, 4)
    with rows >= y0 + H and cols >= x0 + W, float4 rows (stride(2) == 1,
    stride(1) == 4, stride(0) a multiple of 4), on the right device -- else
    the kernel or the D2H copy would write past it."""
    import torch
    if not isinstance(out, torch.Tensor) or out.dtype != torch.float32 or out.dim() != 3 or out.shape[2] != 4:
        raise ValueError(f"{what}: out must be a float32 tensor of shape (rows, cols, 4)")
    if out.device.type != device_type:
        raise ValueError(f"{what}: out must be a {device_type} tensor")
    if out.stride(2) != 1 or out.stride(1) != 4 or out.stride(0) % 4 != 0 or out.stride(0) < 4 * out.shape[1]:
        raise ValueError(f"{what}: out must be a row-pitched float4 array (stride(2) == 1, stride(1) == 4)")
    if out.shape[0] < g.y0 + g.height or out.shape[1] < g.x0 + g.width:
        raise ValueError(f"{what}: out of shape {tuple(out.shape)} cannot hold a {g.height}x{g.width} tile at "
                         f"origin (x0, y0) = ({g.x0}, {g.y0})")


class Context:
    """A glint context on one CUDA device (tables resident in HBM)."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        h = C.c_void_p()
        rc = lib().glint_create(C.byref(h), self.device)
        if rc:
            raise GlintError(rc, "glint_create")
        self._h = h

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().glint_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def tables(self):
        z = np.zeros(ZQ, np.float32)
        c = np.zeros(NANG, np.float32)
        s = np.zeros(NANG, np.float32)
        rc = lib().glint_get_tables(self._h, z.ctypes.data, c.ctypes.data, s.ctypes.data)
        if rc:
            raise GlintError(rc, "glint_get_tables")
        return z, c, s

    def launch_count(self) -> int:
        return int(lib().glint_launch_count(self._h))


def glint_eval(ctx: Context, gb, scene, out=None, debug: bool = False, stream=None, origin=(0, 0)):
    """Shade a device-resident G-buffer (synth.GBuffer of CUDA tensors).
    Returns the (H, W, 4) float32 radiance tensor (RGB + flag bits) and, if
    ``debug``, the (H*W, n_lights) debug records as a numpy structured array
    (copied to host, synchronising). ``origin`` = (x0, y0): the tile's place
    in ``out`` (a larger frame; glint.h tile origin)."""
    import torch
    planes = gb.planes()
    dev = planes[0].device
    if dev.type != "cuda":
        raise ValueError("glint_eval needs CUDA tensors (use glint_eval_host for host buffers)")
    g = _gbuffer_struct(gb, origin)
    sc = scene_struct(scene)
    if out is None:
        out = torch.empty((g.y0 + g.height, g.x0 + g.width, 4), dtype=torch.float32, device=dev)
    _check_out(out, g, "cuda", "glint_eval")
    dbg = None
    if debug:
        dbg = torch.zeros(max(1, g.width * g.height * sc.n_lights * DEBUG_REC_BYTES // 4),
                          dtype=torch.int32, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    rc = lib().glint_eval(ctx.handle, C.byref(g), C.byref(sc), out.data_ptr(), out.stride(0) // 4,
                          dbg.data_ptr() if dbg is not None else None, C.c_void_p(s.cuda_stream))
    if rc:
        raise GlintError(rc, "glint_eval")
    if debug:
        n = g.width * g.height * sc.n_lights
        rec = dbg.cpu().numpy().view(np.uint8)[: n * DEBUG_REC_BYTES].view(DEBUG_REC_DTYPE)
        return out, rec.reshape(g.width * g.height, sc.n_lights)
    return out


def glint_eval_batch(ctx: Context, gbs, scenes, outs=None, stream=None, origins=None):
    """Shade independent device-resident frames with one call (the launches
    are chained with programmatic dependent launch; include/glint.h). Frame f's
    result equals glint_eval(ctx, gbs[f], scenes[f]) bit for bit. Returns the
    list of (H, W, 4) radiance tensors."""
    import torch
    n = len(gbs)
    if len(scenes) != n or (outs is not None and len(outs) != n):
        raise ValueError("gbs, scenes and outs must have the same length")
    if n == 0:
        return []
    dev = gbs[0].planes()[0].device
    if any(g.planes()[0].device != dev for g in gbs) or dev.type != "cuda":
        raise ValueError("glint_eval_batch needs CUDA tensors on one device")
    origins = origins or [(0, 0)] * n
    G = (glint_gbuffer * n)(*[_gbuffer_struct(g, o) for g, o in zip(gbs, origins)])
    S = (glint_scene * n)(*[scene_struct(sc) for sc in scenes])
    if outs is None:
        outs = [torch.empty((G[f].y0 + G[f].height, G[f].x0 + G[f].width, 4), dtype=torch.float32, device=dev)
                for f in range(n)]
    for f, o in enumerate(outs):
        _check_out(o, G[f], "cuda", "glint_eval_batch")
    P = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    Q = (C.c_int64 * n)(*[o.stride(0) // 4 for o in outs])
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    rc = lib().glint_eval_batch(ctx.handle, n, G, S, P, Q, C.c_void_p(s.cuda_stream))
    if rc:
        raise GlintError(rc, "glint_eval_batch")
    return outs


def glint_eval_host(ctx: Context, gb, scene, out=None, stream=None, origin=(0, 0)):
    """End-to-end: host (ideally pinned) G-buffer in, host radiance out; the
    library pipelines H2D / kernel / D2H over row chunks. Synchronous."""
    import torch
    g = _gbuffer_struct(gb, origin)
    if gb.planes()[0].device.type != "cpu":
        raise ValueError("glint_eval_host needs host tensors")
    sc = scene_struct(scene)
    if out is None:
        out = torch.empty((g.y0 + g.height, g.x0 + g.width, 4), dtype=torch.float32).pin_memory()
    _check_out(out, g, "cpu", "glint_eval_host")
    s = stream if stream is not None else torch.cuda.current_stream(ctx.device)
    rc = lib().glint_eval_host(ctx.handle, C.byref(g), C.byref(sc), out.data_ptr(), out.stride(0) // 4,
                               C.c_void_p(s.cuda_stream))
    if rc:
        raise GlintError(rc, "glint_eval_host")
    return out


def glint_eval_host_batch(ctx: Context, gbs, scenes, outs=None, stream=None, origins=None):
    """End-to-end over several frames: host (ideally pinned) G-buffers in,
    host radiance out, one continuous copy/compute pipeline across the frames.
    Frame f equals glint_eval_host(ctx, gbs[f], scenes[f]) bit for bit.
    Synchronous; returns the list of (H, W, 4) host tensors."""
    import torch
    n = len(gbs)
    if len(scenes) != n or (outs is not None and len(outs) != n):
        raise ValueError("gbs, scenes and outs must have the same length")
    if n == 0:
        return []
    if any(g.planes()[0].device.type != "cpu" for g in gbs):
        raise ValueError("glint_eval_host_batch needs host tensors")
    origins = origins or [(0, 0)] * n
    G = (glint_gbuffer * n)(*[_gbuffer_struct(g, o) for g, o in zip(gbs, origins)])
    S = (glint_scene * n)(*[scene_struct(sc) for sc in scenes])
    if outs is None:
        outs = [torch.empty((G[f].y0 + G[f].height, G[f].x0 + G[f].width, 4), dtype=torch.float32).pin_memory()
                for f in range(n)]
    for f, o in enumerate(outs):
        _check_out(o, G[f], "cpu", "glint_eval_host_batch")
    P = (C.c_void_p * n)(*[o.data_ptr() for o in outs])
    Q = (C.c_int64 * n)(*[o.stride(0) // 4 for o in outs])
    s = stream if stream is not None else torch.cuda.current_stream(ctx.device)
    rc = lib().glint_eval_host_batch(ctx.handle, n, G, S, P, Q, C.c_void_p(s.cuda_stream))
    if rc:
        raise GlintError(rc, "glint_eval_host_batch")
    return outs


def glint_count_active(ctx: Context, gb, scene, stream=None) -> int:
    """The number of (pixel, light) evaluations glint_eval does on ``gb``
    (valid pixels with a non-degenerate footprint x lights active there),
    counted on the device with the kernel's own decisions. Synchronising."""
    import torch
    dev = gb.planes()[0].device
    if dev.type != "cuda":
        raise ValueError("glint_count_active needs CUDA tensors")
    g = _gbuffer_struct(gb)
    sc = scene_struct(scene)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    rc = lib().glint_count_active(ctx.handle, C.byref(g), C.byref(sc), cnt.data_ptr(), C.c_void_p(s.cuda_stream))
    if rc:
        raise GlintError(rc, "glint_count_active")
    return int(cnt.item())
