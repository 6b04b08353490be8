"""Seeded synthetic G-buffers shaped like the paper's workloads.

This module is the ONLY code shared by the product path, the oracle tests and
the bench: it produces inputs (uv, screen-space uv derivatives, normals,
positions, materials, lights) and holds none of the method's arithmetic
(footprints, grids, hashing, counting and radiance are computed independently
by the CUDA kernel and by ``oracle/``).

The paper measures on Unity scenes (Plane 90/25 deg, Heightmap, Sponza,
Sphere, Monkey) whose assets are not available; these analytic
scenes stand in for them (BASELINE.json configs C1..C5):

* C1  64x64 flat quad, constant derivatives, directional view/light.
* C2  1920x1080 infinite ground plane, pinhole camera (60 deg FOV) at
      elevations 5..85 (+90) deg, one point light, per-tile log2 density.
* C3  3840x2160, 32 analytic spheres on a plane, anisotropic roughness,
      log-uniform density, one point light.
* C4  C3 with 16 point lights and 8 jittered frames.
* C5  64-frame zoom path (0.5 -> 500 units) over the plane + spheres, 4 lights.

All geometry is computed in float64 with analytic ray differentials and
stored as float32 structure-of-arrays planes (H, W, 4):

    duv = (du/dx, dv/dx, du/dy, dv/dy)
    uvm = (u, v, object/tile id bits, meta bits)   meta bit0 = valid pixel
    nrm = (nx, ny, nz, 0)
    pos = (x, y, z, 0)  world position
    mat = (alpha_x, alpha_y, N flakes per unit uv^2, R)

uv is kept tile-local in [0, 1) with the tile id folded into the object id so
fp32 keeps its fractional bits at fine LODs (SURVEY §7 "fp32 UV precision").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence, Tuple

import torch

F64 = torch.float64


# ----------------------------------------------------------------------------- scene
@dataclass
class Light:
    kind: str = "point"                     # "point" | "directional"
    pos_or_dir: Tuple[float, float, float] = (0.0, 0.0, 1.0)
    intensity: Tuple[float, float, float] = (1.0, 1.0, 1.0)


@dataclass
class SceneParams:
    seed: int = 1
    ndf: str = "ggx"                        # "ggx" | "beckmann"
    max_ratio_level: int = 8                # K
    beta: float = 0.05                      # angular cell size (micro-roughness)
    f0: Tuple[float, float, float] = (0.9, 0.9, 0.9)
    view_kind: str = "point"                # "point" camera position | "directional"
    view: Tuple[float, float, float] = (0.0, 0.0, 1.0)
    lights: List[Light] = field(default_factory=list)
    draws: int = 48                         # 48 (the paper's method); 64 / 160 = its ablations
    method: str = "ours"                    # "ours" | "zk" (Zirr & Kaplanyan-style baseline)


@dataclass
class GBuffer:
    duv: torch.Tensor
    uvm: torch.Tensor
    nrm: torch.Tensor
    pos: torch.Tensor
    mat: torch.Tensor

    @property
    def height(self) -> int:
        return int(self.duv.shape[0])

    @property
    def width(self) -> int:
        return int(self.duv.shape[1])

    def planes(self):
        return (self.duv, self.uvm, self.nrm, self.pos, self.mat)

    def to(self, device, non_blocking=False) -> "GBuffer":
        return GBuffer(*[p.to(device, non_blocking=non_blocking).contiguous() for p in self.planes()])

    def pin(self) -> "GBuffer":
        return GBuffer(*[p.contiguous().pin_memory() for p in self.planes()])

    def crop(self, y0, y1, x0, x1) -> "GBuffer":
        return GBuffer(*[p[y0:y1, x0:x1].contiguous() for p in self.planes()])

    def flat(self) -> "GBuffer":
        return GBuffer(*[p.reshape(1, -1, 4) for p in self.planes()])

    def take(self, idx: torch.Tensor) -> "GBuffer":
        """Pixels at flat indices ``idx`` as a (1, len, 4) buffer."""
        return GBuffer(*[p.reshape(-1, 4)[idx.to(p.device)].reshape(1, -1, 4).contiguous()
                         for p in self.planes()])

    def valid_count(self) -> int:
        meta = self.uvm[..., 3].contiguous().view(torch.int32)
        return int((meta & 1).sum().item())

    @property
    def nbytes(self) -> int:
        return sum(p.numel() * p.element_size() for p in self.planes())


@dataclass
class Frame:
    name: str
    gbuf: GBuffer
    scene: SceneParams


# ----------------------------------------------------------------------------- helpers
def _bits_to_f32(x: torch.Tensor) -> torch.Tensor:
    """int64 values in [0, 2^32) -> float32 tensor carrying those 32 bits."""
    x = x & 0xFFFFFFFF
    x = torch.where(x >= 2 ** 31, x - 2 ** 32, x)
    return x.to(torch.int32).view(torch.float32)


def _mix64(x: torch.Tensor) -> torch.Tensor:
    """splitmix64-style integer mixer on int64 tensors (input-generator only)."""
    m = 0xFFFFFFFFFFFFFFFF
    x = x & m
    # torch int64 arithmetic wraps; emulate unsigned with masking of shifts
    x = (x ^ ((x >> 30) & 0x3FFFFFFFF)) * -4658895280553007687  # 0xbf58476d1ce4e5b9
    x = (x ^ ((x >> 27) & 0x1FFFFFFFFF)) * -7723592293110705685  # 0x94d049bb133111eb
    x = x ^ ((x >> 31) & 0x1FFFFFFFF)
    return x


def _uniform01(key: torch.Tensor) -> torch.Tensor:
    """Deterministic float64 in [0,1) from an int64 key tensor."""
    return ((_mix64(key) >> 11) & ((1 << 53) - 1)).to(F64) / float(1 << 53)


def _normalize(v: torch.Tensor) -> torch.Tensor:
    return v / torch.linalg.vector_norm(v, dim=-1, keepdim=True)


def _camera(width, height, fov_deg, cam, look, window, jitter=(0.0, 0.0), device="cpu"):
    """Pinhole camera rays for the pixel window. Returns origin (3,), d (h,w,3)
    unnormalised direction, dd/dx, dd/dy (3,) (d is affine in pixel coords)."""
    cam = torch.tensor(cam, dtype=F64, device=device)
    look = torch.tensor(look, dtype=F64, device=device)
    f = _normalize(look - cam)
    zup = torch.tensor([0.0, 0.0, 1.0], dtype=F64, device=device)
    right = torch.linalg.cross(f, zup)
    if float(torch.linalg.vector_norm(right)) < 1e-9:      # looking straight down
        right = torch.tensor([1.0, 0.0, 0.0], dtype=F64, device=device)
    right = _normalize(right)
    up = torch.linalg.cross(right, f)
    th = math.tan(math.radians(fov_deg) * 0.5)
    aspect = width / height
    y0, y1, x0, x1 = window
    px = torch.arange(x0, x1, dtype=F64, device=device) + 0.5 + jitter[0]
    py = torch.arange(y0, y1, dtype=F64, device=device) + 0.5 + jitter[1]
    sx = (2.0 * px / width - 1.0) * th * aspect
    sy = (1.0 - 2.0 * py / height) * th
    d = f + sx[None, :, None] * right + sy[:, None, None] * up
    ddx = right * (2.0 * th * aspect / width)
    ddy = -up * (2.0 * th / height)
    return cam, d, ddx, ddy


def _pack(u, v, obj, valid, duv4, nrm3, pos3, mat4):
    """Assemble float32 SoA planes; invalid pixels are zeroed (meta bit0 = 0)."""
    h, w = u.shape
    dev = u.device
    validf = valid.to(F64)
    tile_u = torch.floor(u)
    tile_v = torch.floor(v)
    lu = torch.where(valid, u - tile_u, torch.zeros_like(u))
    lv = torch.where(valid, v - tile_v, torch.zeros_like(v))
    # fold the uv tile into the object id (uv stays local in [0,1))
    key = (obj.to(torch.int64) * 1000003 + tile_u.clamp(-2**30, 2**30).to(torch.int64) * 7919
           + tile_v.clamp(-2**30, 2**30).to(torch.int64) * 104729)
    objbits = _mix64(key) & 0xFFFFFFFF
    objbits = torch.where(valid, objbits, torch.zeros_like(objbits))
    uvm = torch.empty(h, w, 4, dtype=torch.float32, device=dev)
    uvm[..., 0] = lu.to(torch.float32)
    uvm[..., 1] = lv.to(torch.float32)
    uvm[..., 2] = _bits_to_f32(objbits)
    uvm[..., 3] = _bits_to_f32(valid.to(torch.int64))
    duv = (duv4 * validf[..., None]).to(torch.float32)
    nrm = torch.zeros(h, w, 4, dtype=torch.float32, device=dev)
    nrm[..., :3] = torch.where(valid[..., None], nrm3, torch.tensor([0.0, 0.0, 1.0], dtype=F64, device=dev)).to(torch.float32)
    pos = torch.zeros(h, w, 4, dtype=torch.float32, device=dev)
    pos[..., :3] = (pos3 * validf[..., None]).to(torch.float32)
    mat = (mat4 * validf[..., None] + (1.0 - validf[..., None]) * torch.tensor([0.5, 0.5, 1.0, 0.5], dtype=F64, device=dev)).to(torch.float32)
    return GBuffer(duv.contiguous(), uvm.contiguous(), nrm.contiguous(), pos.contiguous(), mat.contiguous())


# ----------------------------------------------------------------------------- C1
def c1(ndf: str = "ggx", variant: str = "mirror", seed: int = 1, device="cpu") -> Frame:
    """64x64 flat quad, uv = pixel/64 (variant "centers": (pixel+1/2)/64),
    duv/dx = (1/64, 0), duv/dy = (0, 1/64), n = +z, distant view at 30 deg,
    directional light at 30 deg off-normal: "mirror" azimuth (h = n) or "az90".
    alpha 0.3, N = 1e5 per unit uv^2, R = 0.034, hash seed 1 (BASELINE.json C1)."""
    n = 64
    off = 0.5 if variant == "centers" else 0.0
    ys, xs = torch.meshgrid(torch.arange(n, dtype=F64), torch.arange(n, dtype=F64), indexing="ij")
    u = (xs + off) / n
    v = (ys + off) / n
    duv4 = torch.tensor([1.0 / n, 0.0, 0.0, 1.0 / n], dtype=F64).expand(n, n, 4)
    nrm3 = torch.tensor([0.0, 0.0, 1.0], dtype=F64).expand(n, n, 3)
    pos3 = torch.stack([u, v, torch.zeros_like(u)], -1)
    mat4 = torch.tensor([0.3, 0.3, 1e5, 0.034], dtype=F64).expand(n, n, 4)
    valid = torch.ones(n, n, dtype=torch.bool)
    gb = _pack_c1(u, v, duv4, nrm3, pos3, mat4)
    s30, c30 = math.sin(math.radians(30)), math.cos(math.radians(30))
    if variant == "az90":
        ldir = (0.0, s30, c30)
    else:
        ldir = (-s30, 0.0, c30)
    scene = SceneParams(seed=seed, ndf=ndf, view_kind="directional", view=(s30, 0.0, c30),
                        lights=[Light("directional", ldir, (1.0, 1.0, 1.0))])
    del valid
    return Frame(f"C1-{ndf}-{variant}", gb.to(device), scene)


def _pack_c1(u, v, duv4, nrm3, pos3, mat4):
    """C1 keeps uv literal (no tile folding; obj = 0)."""
    h, w = u.shape
    uvm = torch.zeros(h, w, 4, dtype=torch.float32)
    uvm[..., 0] = u.to(torch.float32)
    uvm[..., 1] = v.to(torch.float32)
    uvm[..., 2] = _bits_to_f32(torch.zeros(h, w, dtype=torch.int64))
    uvm[..., 3] = _bits_to_f32(torch.ones(h, w, dtype=torch.int64))
    nrm = torch.zeros(h, w, 4, dtype=torch.float32)
    nrm[..., :3] = nrm3.to(torch.float32)
    pos = torch.zeros(h, w, 4, dtype=torch.float32)
    pos[..., :3] = pos3.to(torch.float32)
    return GBuffer(duv4.to(torch.float32).contiguous(), uvm, nrm, pos, mat4.to(torch.float32).contiguous())


# ----------------------------------------------------------------------------- C2
C2_ELEVATIONS = (5, 15, 25, 35, 45, 55, 65, 75, 85, 90)


def c2(elevation_deg: float, width: int = 1920, height: int = 1080, ndf: str = "ggx",
       window: Optional[Tuple[int, int, int, int]] = None, seed: int = 1, scene_seed: int = 12,
       alpha: float = 0.2, R: float = 0.034, device="cpu") -> Frame:
    """Infinite ground plane z = 0 seen by a pinhole camera (vertical FOV 60 deg)
    at distance 10 from the origin and the given elevation; uv = world xy split
    into 1x1 material tiles; per-tile density N = 2^U(8,20); one point light at
    the camera's mirror position about the normal, I = d^2 (BASELINE.json C2)."""
    window = window or (0, height, 0, width)
    e = math.radians(elevation_deg)
    D = 10.0
    cam = (0.0, -D * math.cos(e), D * math.sin(e))
    o, d, ddx, ddy = _camera(width, height, 60.0, cam, (0.0, 0.0, 0.0), window, device=device)
    dz = d[..., 2]
    valid = dz < -1e-9
    t = torch.where(valid, -o[2] / dz, torch.zeros_like(dz))
    P = o + t[..., None] * d
    # ray differentials: dt/dx = cz/dz^2 ddz/dx ; dP/dx = t ddx + dt/dx d
    dtdx = torch.where(valid, o[2] / (dz * dz) * ddx[2], torch.zeros_like(dz))
    dtdy = torch.where(valid, o[2] / (dz * dz) * ddy[2], torch.zeros_like(dz))
    dPdx = t[..., None] * ddx + dtdx[..., None] * d
    dPdy = t[..., None] * ddy + dtdy[..., None] * d
    u, v = P[..., 0], P[..., 1]
    duv4 = torch.stack([dPdx[..., 0], dPdx[..., 1], dPdy[..., 0], dPdy[..., 1]], -1)
    tu, tv = torch.floor(u), torch.floor(v)
    tkey = (tu.clamp(-2**30, 2**30).to(torch.int64) * 73856093
            + tv.clamp(-2**30, 2**30).to(torch.int64) * 19349663 + scene_seed * 83492791)
    N = torch.exp2(8.0 + 12.0 * _uniform01(tkey))
    a = torch.full_like(u, alpha)
    mat4 = torch.stack([a, a, N, torch.full_like(u, R)], -1)
    nrm3 = torch.zeros_like(P)
    nrm3[..., 2] = 1.0
    gb = _pack(u, v, torch.zeros_like(u, dtype=torch.int64), valid, duv4, nrm3, P, mat4)
    lpos = (0.0, D * math.cos(e), D * math.sin(e))
    scene = SceneParams(seed=seed, ndf=ndf, view_kind="point", view=cam,
                        lights=[Light("point", lpos, (D * D,) * 3)])
    return Frame(f"C2-e{elevation_deg:g}-{ndf}", gb, scene)


def c2_frames(width=1920, height=1080, ndf="ggx", elevations: Sequence[float] = C2_ELEVATIONS,
              device="cpu"):
    return [c2(e, width, height, ndf=ndf, device=device) for e in elevations]


# ----------------------------------------------------------------------------- C3/C4/C5
def _spheres(scene_seed: int, n: int = 32, device="cpu"):
    """32 spheres, radius U(0.5,3), resting on z = 0, centres uniform in
    [-20,20]^2 without overlap (rejection, deterministic)."""
    ctr, rad = [], []
    k = 0
    while len(ctr) < n:
        key = torch.tensor([scene_seed * 1000003 + k * 4 + j for j in range(3)], dtype=torch.int64)
        r3 = _uniform01(key).tolist()
        k += 1
        r = 0.5 + 2.5 * r3[0]
        x, y = -20.0 + 40.0 * r3[1], -20.0 + 40.0 * r3[2]
        if all((x - cx) ** 2 + (y - cy) ** 2 > (r + cr) ** 2 for (cx, cy, _), cr in zip(ctr, rad)):
            ctr.append((x, y, r))
            rad.append(r)
    return (torch.tensor(ctr, dtype=F64, device=device), torch.tensor(rad, dtype=F64, device=device))


def _object_materials(scene_seed: int, n_obj: int, device="cpu"):
    """Per object: alpha_x, alpha_y ~ U(0.05, 0.6), N log-uniform [1e3, 1e7]."""
    key = torch.arange(n_obj, dtype=torch.int64, device=device) * 3 + scene_seed * 7777
    ax = 0.05 + 0.55 * _uniform01(key)
    ay = 0.05 + 0.55 * _uniform01(key + 1)
    N = 10.0 ** (3.0 + 4.0 * _uniform01(key + 2))
    return ax, ay, N


def spheres_scene_gbuffer(width, height, cam, look, scene_seed, window=None, jitter=(0.0, 0.0),
                          R=0.034, fov=60.0, device="cpu") -> GBuffer:
    """Analytic G-buffer of 32 spheres on the plane z = 0 (plane = object 32)."""
    window = window or (0, height, 0, width)
    ctr, rad = _spheres(scene_seed, device=device)
    ax_o, ay_o, N_o = _object_materials(scene_seed, ctr.shape[0] + 1, device=device)
    o, d, ddx, ddy = _camera(width, height, fov, cam, look, window, jitter, device=device)
    h, w = d.shape[:2]
    best_t = torch.full((h, w), float("inf"), dtype=F64, device=device)
    best_i = torch.full((h, w), -1, dtype=torch.int64, device=device)
    dd = (d * d).sum(-1)
    for i in range(ctr.shape[0]):
        oc = o - ctr[i]
        b = (d * oc).sum(-1)
        c = float((oc * oc).sum() - rad[i] ** 2)
        disc = b * b - dd * c
        ok = disc > 0
        t = (-b - torch.sqrt(torch.clamp(disc, min=0.0))) / dd
        ok = ok & (t > 1e-6) & (t < best_t)
        best_t = torch.where(ok, t, best_t)
        best_i = torch.where(ok, torch.full_like(best_i, i), best_i)
    # ground plane z = 0
    dz = d[..., 2]
    tp = torch.where(dz < -1e-9, -o[2] / dz, torch.full_like(dz, float("inf")))
    okp = tp < best_t
    best_t = torch.where(okp, tp, best_t)
    best_i = torch.where(okp, torch.full_like(best_i, ctr.shape[0]), best_i)
    valid = torch.isfinite(best_t)
    t = torch.where(valid, best_t, torch.zeros_like(best_t))
    P = o + t[..., None] * d
    is_plane = best_i == ctr.shape[0]
    ci = ctr[best_i.clamp(0, ctr.shape[0] - 1)]
    ri = rad[best_i.clamp(0, ctr.shape[0] - 1)]
    nS = (P - ci) / ri[..., None]
    nP = torch.zeros_like(P)
    nP[..., 2] = 1.0
    nrm = torch.where(is_plane[..., None], nP, nS)
    nrm = _normalize(nrm)
    dn = (d * nrm).sum(-1)
    dn = torch.where(dn.abs() < 1e-12, torch.full_like(dn, -1e-12), dn)
    # ray differentials on the tangent plane: dt = -t (n.dd) / (n.d)
    dtdx = -t * (nrm * ddx).sum(-1) / dn
    dtdy = -t * (nrm * ddy).sum(-1) / dn
    dPdx = t[..., None] * ddx + dtdx[..., None] * d
    dPdy = t[..., None] * ddy + dtdy[..., None] * d
    # uv: plane -> world xy; sphere -> (azimuth/2pi * ceil(2 pi r), polar/pi * ceil(pi r))
    lx, ly, lz = (P - ci).unbind(-1)
    rxy2 = torch.clamp(lx * lx + ly * ly, min=1e-30)
    az = torch.atan2(ly, lx)
    Su = torch.ceil(2 * math.pi * ri)
    Sv = torch.ceil(math.pi * ri)
    cz = torch.clamp(lz / ri, -1.0, 1.0)
    pol = torch.acos(cz)
    us = (az / (2 * math.pi) + 0.5) * Su
    vs = pol / math.pi * Sv
    daz_dP = torch.stack([-ly / rxy2, lx / rxy2, torch.zeros_like(lx)], -1)
    sinp = torch.sqrt(torch.clamp(1.0 - cz * cz, min=1e-30))
    dpol_dP = torch.stack([torch.zeros_like(lx), torch.zeros_like(lx), -1.0 / (ri * sinp)], -1)
    dus = Su / (2 * math.pi)
    dvs = Sv / math.pi
    dudx_s = dus * (daz_dP * dPdx).sum(-1)
    dudy_s = dus * (daz_dP * dPdy).sum(-1)
    dvdx_s = dvs * (dpol_dP * dPdx).sum(-1)
    dvdy_s = dvs * (dpol_dP * dPdy).sum(-1)
    u = torch.where(is_plane, P[..., 0], us)
    v = torch.where(is_plane, P[..., 1], vs)
    duv4 = torch.stack([torch.where(is_plane, dPdx[..., 0], dudx_s), torch.where(is_plane, dPdx[..., 1], dvdx_s),
                        torch.where(is_plane, dPdy[..., 0], dudy_s), torch.where(is_plane, dPdy[..., 1], dvdy_s)], -1)
    # poles of the sphere parameterisation are flagged invalid
    valid = valid & (is_plane | (sinp > 1e-3))
    oid = best_i.clamp(min=0)
    mat4 = torch.stack([ax_o[oid], ay_o[oid], N_o[oid], torch.full_like(t, R)], -1)
    return _pack(u, v, oid, valid, duv4, nrm, P, mat4)


C3_CAM = (0.0, -35.0, 12.0)
C3_LOOK = (0.0, 0.0, 1.0)


def c3(width=3840, height=2160, window=None, ndf="ggx", seed=1, scene_seed=13, device="cpu") -> Frame:
    gb = spheres_scene_gbuffer(width, height, C3_CAM, C3_LOOK, scene_seed, window, device=device)
    L = (10.0, -10.0, 20.0)
    scene = SceneParams(seed=seed, ndf=ndf, view_kind="point", view=C3_CAM,
                        lights=[Light("point", L, (600.0,) * 3)])
    return Frame("C3", gb, scene)


def hemisphere_lights(n, radius, intensity, key_seed, height_min=0.0):
    ls = []
    for i in range(n):
        r2 = _uniform01(torch.tensor([key_seed * 131 + i * 2, key_seed * 131 + i * 2 + 1])).tolist()
        z = height_min / radius + (1.0 - height_min / radius) * r2[0]
        phi = 2 * math.pi * r2[1]
        s = math.sqrt(max(0.0, 1.0 - z * z))
        ls.append(Light("point", (radius * s * math.cos(phi), radius * s * math.sin(phi), radius * z),
                        (intensity,) * 3))
    return ls


def c4(frame: int, width=3840, height=2160, window=None, ndf="ggx", seed=1, scene_seed=14,
       device="cpu") -> Frame:
    """C3 geometry, 16 point lights on the upper hemisphere (radius 25,
    I = 25^2/16 each), sub-pixel camera jitter per frame (8 frames)."""
    j = _uniform01(torch.tensor([scene_seed * 31 + frame * 2, scene_seed * 31 + frame * 2 + 1])).tolist()
    gb = spheres_scene_gbuffer(width, height, C3_CAM, C3_LOOK, 13, window, (j[0] - 0.5, j[1] - 0.5),
                               device=device)
    scene = SceneParams(seed=seed, ndf=ndf, view_kind="point", view=C3_CAM,
                        lights=hemisphere_lights(16, 25.0, 25.0 ** 2 / 16, scene_seed, height_min=2.0))
    return Frame(f"C4-f{frame}", gb, scene)


def c5(frame: int, width=3840, height=2160, window=None, ndf="ggx", seed=1, scene_seed=15,
       device="cpu") -> Frame:
    """Zoom path: look-at origin, elevation 30 deg, distance 0.5 * 1000^(f/63)
    (0.5 -> 500 units over 64 frames), 4 point lights (radius 30, height 20)."""
    dist = 0.5 * 1000.0 ** (frame / 63.0)
    e = math.radians(30.0)
    cam = (0.0, -dist * math.cos(e), dist * math.sin(e))
    gb = spheres_scene_gbuffer(width, height, cam, (0.0, 0.0, 0.0), 13, window, device=device)
    lights = []
    for i in range(4):
        ph = 2 * math.pi * (i + 0.25) / 4
        lights.append(Light("point", (30 * math.cos(ph), 30 * math.sin(ph), 20.0), (1300.0,) * 3))
    scene = SceneParams(seed=seed, ndf=ndf, view_kind="point", view=cam, lights=lights)
    return Frame(f"C5-f{frame}", gb, scene)


# ----------------------------------------------------------------------------- random stress
def random_gbuffer(h: int, w: int, seed: int, device="cpu") -> GBuffer:
    """Adversarial random G-buffer: derivatives spanning 2^-30..2^4 with random
    orientation and anisotropy up to ~2^12 (beyond the 2^8 clamp), random
    normals in the upper hemisphere, some invalid and some degenerate pixels."""
    g = torch.Generator().manual_seed(seed)
    n = h * w
    U = lambda *s: torch.rand(*s, generator=g, dtype=F64)
    lgP = -30.0 + 34.0 * U(n)
    lgr = 12.0 * U(n) ** 2
    th = 2 * math.pi * U(n)
    smax = torch.exp2(0.5 * (lgP + lgr))
    smin = torch.exp2(0.5 * (lgP - lgr))
    # J = Rot(th) diag(smax, smin) Rot(th2)^T
    th2 = 2 * math.pi * U(n)
    c, s = torch.cos(th), torch.sin(th)
    c2_, s2_ = torch.cos(th2), torch.sin(th2)
    J00 = c * smax * c2_ + s * smin * s2_
    J01 = c * smax * s2_ - s * smin * c2_
    J10 = s * smax * c2_ - c * smin * s2_
    J11 = s * smax * s2_ + c * smin * c2_
    duv4 = torch.stack([J00, J10, J01, J11], -1)
    # some exactly isotropic, axis aligned and degenerate pixels
    kind = (U(n) * 10).floor()
    iso = torch.exp2(0.5 * lgP)
    duv4 = torch.where((kind == 0)[:, None], torch.stack([iso, 0 * iso, 0 * iso, iso], -1), duv4)
    duv4 = torch.where((kind == 1)[:, None], torch.zeros_like(duv4), duv4)
    u = U(n)
    v = U(n)
    ct = U(n) ** 0.5
    ph = 2 * math.pi * U(n)
    st = torch.sqrt(1 - ct * ct)
    nrm3 = torch.stack([st * torch.cos(ph), st * torch.sin(ph), ct], -1)
    flip = (kind == 2)
    nrm3 = torch.where(flip[:, None], -nrm3, nrm3)
    pos3 = torch.stack([U(n) * 4 - 2, U(n) * 4 - 2, U(n) * 0.5], -1)
    a_x = 0.02 + 1.1 * U(n)
    a_y = torch.where(U(n) < 0.5, a_x, 0.02 + 1.1 * U(n))
    N = 10.0 ** (1.0 + 8.0 * U(n))
    Rr = 0.005 + 0.6 * U(n)
    mat4 = torch.stack([a_x, a_y, N, Rr], -1)
    valid = U(n) > 0.05
    obj = (U(n) * 1e6).to(torch.int64)
    gb = _pack(u.reshape(h, w), v.reshape(h, w), obj.reshape(h, w), valid.reshape(h, w),
               duv4.reshape(h, w, 4), nrm3.reshape(h, w, 3), pos3.reshape(h, w, 3), mat4.reshape(h, w, 4))
    return gb.to(device)


def random_scene(seed: int, n_lights: int = 3, ndf: str = "ggx") -> SceneParams:
    g = torch.Generator().manual_seed(seed + 17)
    U = lambda: float(torch.rand(1, generator=g, dtype=F64))
    lights = []
    for i in range(n_lights):
        if i % 2 == 0:
            lights.append(Light("point", (4 * U() - 2, 4 * U() - 2, 0.5 + 4 * U()), (U() * 5, U() * 5, U() * 5)))
        else:
            z = U()
            lights.append(Light("directional", (U() - 0.5, U() - 0.5, z), (U(), U(), U())))
    return SceneParams(seed=seed, ndf=ndf, max_ratio_level=8, beta=0.02 + 0.1 * U(),
                       f0=(U(), U(), U()), view_kind="point", view=(0.3, -2.0, 3.0), lights=lights)
