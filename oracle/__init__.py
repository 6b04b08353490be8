"""CPU oracle for the glint hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The
product path (``paper_2306_05051_b200``) never imports it and shares no code
with it.

The arithmetic lives in ``glint_oracle.c`` (plain scalar C, fp32 contract for
every value that decides an integer, fp64 for radiance); this module only
builds it with gcc, marshals arguments with ctypes and fans pixel ranges out
over host threads (ctypes releases the GIL during the call).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "glint_oracle.c")
_LIB = os.path.join(_HERE, "libglint_oracle.so")
CFLAGS = ["-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
          "-fno-tree-vectorize", "-fPIC", "-shared"]

MAX_LIGHTS = 16
ZQ = 4096
FLAG_INVALID, FLAG_DEGENERATE, FLAG_RATIO_CLAMPED, FLAG_P_CLAMPED, FLAG_UV_RANGE = 1, 2, 4, 8, 16


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no contraction, no fast-math)."""
    hdr = os.path.join(_HERE, "glint_oracle.h")
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= max(os.path.getmtime(_SRC), os.path.getmtime(hdr))):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


class _Light(C.Structure):
    _fields_ = [("kind", C.c_int32), ("pos_or_dir", C.c_float * 3),
                ("intensity", C.c_float * 3), ("pad_", C.c_int32)]


class _Scene(C.Structure):
    _fields_ = [("seed", C.c_uint32), ("ndf_kind", C.c_int32), ("max_ratio_level", C.c_int32),
                ("beta", C.c_float), ("f0", C.c_float * 3), ("view_kind", C.c_int32),
                ("view", C.c_float * 3), ("n_lights", C.c_int32), ("sampler", C.c_int32),
                ("eval_mode", C.c_int32), ("pad_", C.c_int32 * 2), ("lights", _Light * MAX_LIGHTS)]


REC_DTYPE = np.dtype([
    ("P", "<f4"), ("r", "<f4"), ("psi", "<f4"),
    ("ls", "<i4", 4), ("lr", "<i4", 4), ("jo", "<i4", 4),
    ("w", "<f4", 4), ("n", "<f4", 4),
    ("lx", "<i4", 12), ("ly", "<i4", 12),
    ("p", "<f4"), ("cx0", "<i4"), ("cy0", "<i4"),
    ("T", "<u4", 4), ("sigma", "<f4", 4), ("m1", "<f4", 4), ("cap", "<f4", 4),
    ("hash", "<u4", 48), ("count", "<f4", 48),
    ("C", "<f4"), ("Dp", "<f4"), ("flags", "<u4"), ("light_active", "<u4"), 
    ("sfx", "<f4", 4), ("sfy", "<f4", 4), ("afx", "<f4"), ("afy", "<f4"), ("pge1", "<f4", 4), ("pad_", "<u4", 4),
])
assert REC_DTYPE.itemsize == 184 * 4

_lib = None
_lock = threading.Lock()


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            fp = C.POINTER(C.c_float)
            L.orc_init.restype = C.c_int
            for nm in ("orc_ztable", "orc_costable", "orc_sintable"):
                getattr(L, nm).restype = fp
            L.orc_eval.argtypes = [C.c_void_p] * 5 + [C.c_int64, C.POINTER(_Scene),
                                                      C.c_void_p, C.c_void_p, C.c_void_p]
            L.orc_eval.restype = C.c_int
            L.orc_exp2.argtypes = [C.c_float]; L.orc_exp2.restype = C.c_float
            L.orc_rsqrt.argtypes = [C.c_float]; L.orc_rsqrt.restype = C.c_float
            L.orc_rcp.argtypes = [C.c_float]; L.orc_rcp.restype = C.c_float
            L.orc_log2_1mp.argtypes = [C.c_float]; L.orc_log2_1mp.restype = C.c_float
            L.orc_atan2_turns.argtypes = [C.c_float, C.c_float]; L.orc_atan2_turns.restype = C.c_float
            L.orc_lowbias32.argtypes = [C.c_uint32]; L.orc_lowbias32.restype = C.c_uint32
            L.orc_draw_hash.argtypes = [C.c_uint32]; L.orc_draw_hash.restype = C.c_uint32
            L.orc_footprint.argtypes = [fp, fp, fp, fp]; L.orc_footprint.restype = C.c_int
            i4p = C.POINTER(C.c_int32)
            L.orc_lattice.argtypes = [C.c_float, C.c_float, C.c_float, C.c_int32, i4p, i4p, i4p, fp,
                                      C.POINTER(C.c_uint32)]
            i4p10 = C.POINTER(C.c_int32)
            L.orc_lattice10.argtypes = [C.c_float, C.c_float, C.c_float, C.c_int32, i4p10, i4p10, i4p10, fp,
                                        C.POINTER(C.c_uint32)]
            L.orc_grid_uv.argtypes = [C.c_float, C.c_float, C.c_int32, C.c_int32, C.c_int32, fp, fp]
            L.orc_grid_uv.restype = None
            i8p = C.POINTER(C.c_int64)
            L.orc_simplex.argtypes = [C.c_float, C.c_float, i8p, i8p, fp]
            L.orc_simplex.restype = None
            L.orc_gate_params.argtypes = [C.c_float, C.c_float, C.POINTER(C.c_uint32), fp, fp, fp]
            L.orc_gate_params.restype = None
            L.orc_gated_count.argtypes = [C.c_uint32, C.c_uint32, C.c_float, C.c_float, C.c_float]
            L.orc_gated_count.restype = C.c_float
            L.orc_ratio.argtypes = [C.c_int32] + [C.c_float] * 5
            L.orc_ratio.restype = C.c_float
            d3 = C.c_double * 3
            L.orc_smith_g2.argtypes = [C.c_int32, C.c_double, C.c_double, d3, d3]
            L.orc_smith_g2.restype = C.c_double
            L.orc_schlick.argtypes = [C.c_double, C.c_double]
            L.orc_schlick.restype = C.c_double
            L.orc_shell.argtypes = [C.POINTER(_Scene), C.c_int32, C.c_float * 3, C.c_float * 3, C.c_float, C.c_float,
                                    C.c_double, d3]
            L.orc_shell.restype = C.c_int
            f16 = C.c_float * 16
            L.orc_zk_probes.argtypes = [C.c_float * 4, C.c_float, C.c_float, f16, f16, fp, C.POINTER(C.c_uint32)]
            L.orc_zk_probes.restype = C.c_int
            L.orc_zk_lod.argtypes = [C.c_float, C.POINTER(C.c_int32), fp]
            L.orc_zk_lod.restype = None
            L.orc_zk_count.argtypes = [C.c_uint32, C.c_float, C.c_float]
            L.orc_zk_count.restype = C.c_float
            L.orc_contract_checksum.argtypes = [C.c_int32, C.c_uint64, C.c_uint64]
            L.orc_contract_checksum.restype = C.c_uint64
            L.orc_init()
            _lib = L
    return _lib


# --------------------------------------------------------------------------- tables
def ztable() -> np.ndarray:
    return np.ctypeslib.as_array(lib().orc_ztable(), shape=(ZQ,)).copy()


def costable() -> np.ndarray:
    return np.ctypeslib.as_array(lib().orc_costable(), shape=(256,)).copy()


def sintable() -> np.ndarray:
    return np.ctypeslib.as_array(lib().orc_sintable(), shape=(256,)).copy()


# --------------------------------------------------------------------------- scene
def eval_mode_of(scene) -> int:
    """0/1/2 = the method with 48 draws or its 64/160-draw ablations; 3 = the
    Zirr & Kaplanyan-style baseline (scene.method == "zk")."""
    if getattr(scene, "method", "ours") == "zk":
        return 3
    return {48: 0, 64: 1, 160: 2}[int(getattr(scene, "draws", 48))]


def scene_struct(scene, sampler: str = "gated") -> _Scene:
    """Marshal a scene description (any object with the SceneParams fields)."""
    s = _Scene()
    s.seed = int(scene.seed) & 0xFFFFFFFF
    s.ndf_kind = {"ggx": 0, "beckmann": 1}[scene.ndf]
    s.max_ratio_level = int(scene.max_ratio_level)
    s.beta = float(scene.beta)
    s.f0[:] = [float(x) for x in scene.f0]
    s.view_kind = 0 if scene.view_kind == "point" else 1
    s.view[:] = [float(x) for x in scene.view]
    if len(scene.lights) > MAX_LIGHTS:
        raise ValueError("too many lights")
    s.n_lights = len(scene.lights)
    s.sampler = {"gated": 0, "exact": 1}[sampler]
    s.eval_mode = eval_mode_of(scene)
    for i, lt in enumerate(scene.lights):
        s.lights[i].kind = 0 if lt.kind == "point" else 1
        s.lights[i].pos_or_dir[:] = [float(x) for x in lt.pos_or_dir]
        s.lights[i].intensity[:] = [float(x) for x in lt.intensity]
    return s


def _planes(gb):
    """(duv, uvm, nrm, pos, mat) as C-contiguous float32 (n, 4) arrays."""
    out = []
    for name in ("duv", "uvm", "nrm", "pos", "mat"):
        a = getattr(gb, name) if not isinstance(gb, dict) else gb[name]
        if hasattr(a, "detach"):
            a = a.detach().cpu().numpy()
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1, 4))
        out.append(a)
    n = out[0].shape[0]
    assert all(p.shape[0] == n for p in out)
    return out


def eval(gb, scene, debug: bool = False, threads: int | None = None, sampler: str = "gated",
         chunk: int = 4096):
    """Evaluate every pixel of ``gb`` (object/dict with duv, uvm, nrm, pos, mat
    float32 planes of shape (..., 4)). Returns (rgb float64 (n,3), flags uint32
    (n,), records (n, n_lights) REC_DTYPE or None)."""
    L = lib()
    planes = _planes(gb)
    n = planes[0].shape[0]
    sc = scene_struct(scene, sampler)
    nl = sc.n_lights
    rgb = np.zeros((n, 3), np.float64)
    flags = np.zeros((n,), np.uint32)
    rec = np.zeros((n, nl), REC_DTYPE) if debug else None
    threads = threads or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 1)

    def run(lo, hi):
        ptrs = [p[lo:hi].ctypes.data for p in planes]
        rc = L.orc_eval(*ptrs, hi - lo, C.byref(sc), rgb[lo:hi].ctypes.data,
                        flags[lo:hi].ctypes.data,
                        rec[lo:hi].ctypes.data if debug else None)
        if rc != 0:
            raise RuntimeError(f"orc_eval failed: {rc}")

    ranges = [(lo, min(n, lo + chunk)) for lo in range(0, n, chunk)]
    if threads <= 1 or len(ranges) <= 1:
        for lo, hi in ranges:
            run(lo, hi)
    else:
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(lambda r: run(*r), ranges))
    return rgb, flags, rec


# --------------------------------------------------------------------------- primitives
def exp2(y: float) -> float:
    return lib().orc_exp2(y)


def rsqrt(x: float) -> float:
    return lib().orc_rsqrt(x)


def rcp(x: float) -> float:
    return lib().orc_rcp(x)


def log2_1mp(p: float) -> float:
    return lib().orc_log2_1mp(p)


def atan2_turns(y: float, x: float) -> float:
    return lib().orc_atan2_turns(y, x)


def lowbias32(x: int) -> int:
    return lib().orc_lowbias32(x & 0xFFFFFFFF)


def draw_hash(x: int) -> int:
    return lib().orc_draw_hash(x & 0xFFFFFFFF)


def footprint(duv):
    P, r, psi = C.c_float(), C.c_float(), C.c_float()
    arr = (C.c_float * 4)(*[float(x) for x in duv])
    ok = lib().orc_footprint(arr, C.byref(P), C.byref(r), C.byref(psi))
    return P.value, r.value, psi.value, bool(ok)


def lattice(P: float, r: float, psi: float, K: int = 8):
    ls, lr, jo = (C.c_int32 * 4)(), (C.c_int32 * 4)(), (C.c_int32 * 4)()
    w = (C.c_float * 4)()
    fl = C.c_uint32(0)
    lib().orc_lattice(P, r, psi, K, ls, lr, jo, w, C.byref(fl))
    return list(ls), list(lr), list(jo), list(w), fl.value


def lattice10(P: float, r: float, psi: float, K: int = 8):
    ls, lr, jo = (C.c_int32 * 10)(), (C.c_int32 * 10)(), (C.c_int32 * 10)()
    w = (C.c_float * 10)()
    fl = C.c_uint32(0)
    lib().orc_lattice10(P, r, psi, K, ls, lr, jo, w, C.byref(fl))
    return list(ls), list(lr), list(jo), list(w), fl.value


def grid_uv(u, v, ls, lr, jo):
    x, y = C.c_float(), C.c_float()
    lib().orc_grid_uv(u, v, ls, lr, jo, C.byref(x), C.byref(y))
    return x.value, y.value


def simplex(x, y):
    lx, ly, be = (C.c_int64 * 3)(), (C.c_int64 * 3)(), (C.c_float * 3)()
    lib().orc_simplex(x, y, lx, ly, be)
    return list(lx), list(ly), list(be)


def gate_params(n: float, p: float):
    T, s, m1, cap = C.c_uint32(), C.c_float(), C.c_float(), C.c_float()
    lib().orc_gate_params(n, p, C.byref(T), C.byref(s), C.byref(m1), C.byref(cap))
    return T.value, s.value, m1.value, cap.value


def gated_count(h: int, T: int, sigma: float, m1: float, cap: float) -> int:
    return int(lib().orc_gated_count(h & 0xFFFFFFFF, T, sigma, m1, cap))


def ratio(ndf: str, ax, ay, hx, hy, hz) -> float:
    return lib().orc_ratio({"ggx": 0, "beckmann": 1}[ndf], ax, ay, hx, hy, hz)


def smith_g2(ndf: str, ax, ay, wi_local, wo_local) -> float:
    d3 = C.c_double * 3
    return lib().orc_smith_g2({"ggx": 0, "beckmann": 1}[ndf], ax, ay, d3(*wi_local), d3(*wo_local))


def schlick(f0: float, cos_t: float) -> float:
    return lib().orc_schlick(f0, cos_t)


def shell(scene, light: int, nrm, pos, ax: float, ay: float, Dp: float):
    """The S9 radiance shell of one light (fp64): (rgb contribution, added?)
    for a pixel with normal ``nrm``, position ``pos`` and D_P = ``Dp``."""
    f3 = C.c_float * 3
    rgb = (C.c_double * 3)()
    sc = scene_struct(scene)
    added = lib().orc_shell(C.byref(sc), light, f3(*[float(x) for x in nrm[:3]]), f3(*[float(x) for x in pos[:3]]),
                            ax, ay, Dp, rgb)
    return np.array(list(rgb)), bool(added)


# --------------------------------------------------------------------------- ZK baseline pieces
def zk_probes(duv, u: float, v: float):
    """(n, uk[n], vk[n], probe area, flags) of the ZK baseline's footprint probes."""
    uk, vk = (C.c_float * 16)(), (C.c_float * 16)()
    A, fl = C.c_float(), C.c_uint32(0)
    n = lib().orc_zk_probes((C.c_float * 4)(*[float(x) for x in duv]), u, v, uk, vk, C.byref(A), C.byref(fl))
    return n, list(uk)[:n], list(vk)[:n], A.value, fl.value


def zk_lod(A: float):
    k, t = C.c_int32(), C.c_float()
    lib().orc_zk_lod(A, C.byref(k), C.byref(t))
    return k.value, t.value


def zk_count(w: int, nt: float, p: float) -> int:
    return int(lib().orc_zk_count(w & 0xFFFFFFFF, nt, p))


def contract_checksum(fn: int, lo: int, hi: int, threads: int | None = None) -> int:
    """orc_contract_checksum over [lo, hi), split over host threads (the sum is
    order-independent, mod 2^64)."""
    threads = threads or (len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else 1)
    step = max(1, (hi - lo + 4 * threads - 1) // (4 * threads))
    parts = [(a, min(hi, a + step)) for a in range(lo, hi, step)]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        sums = list(ex.map(lambda r: lib().orc_contract_checksum(fn, r[0], r[1]), parts))
    return sum(sums) % (1 << 64)
