"""Seeded synthetic inputs for the BASELINE.json configs.

This module is the ONLY code shared by the CUDA path and the oracle: it draws
random numbers and places cameras, and holds none of the rasterizer's
arithmetic (no projection, compositing, loss or gradient).  Everything is
drawn with numpy's PCG64 ``default_rng(seed)`` in fp64 in the order written
below, then cast to fp32.  Seeds: config i uses seed i.

Stand-in note: the paper measures on Replica / TUM-RGBD /
ScanNet / ScanNet++ (P:232-236), which are not in this container.  These
volume-filling synthetic scenes mirror the frame sizes and Gaussian counts of
those runs (1200x680 / 500k ~ Replica sub-map; 640x480 / 100k ~ TUM,
P:230) and are heavier per pixel than the paper's surface-hugging maps.

Layouts match include/gs.h: four float32 [N,4] arrays (mean_opa, quat,
logscale, rgb), views as float32 [V,12] = (R row-major 9, t 3), world->camera.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Camera:
    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    z_near: float = 0.2   # R5
    z_far: float = 100.0  # R5

    def as_tuple(self):
        return (self.width, self.height, self.fx, self.fy, self.cx, self.cy,
                self.z_near, self.z_far)

    @property
    def tiles(self):
        return ((self.width + 15) // 16) * ((self.height + 15) // 16)


@dataclass
class Scene:
    name: str
    cam: Camera
    mean_opa: np.ndarray  # [N,4] f32 (x, y, z, opacity logit)
    quat: np.ndarray      # [N,4] f32 (w, x, y, z)
    logscale: np.ndarray  # [N,4] f32 (ln sx, ln sy, ln sz, 0)
    rgb: np.ndarray       # [N,4] f32 (r, g, b, 0)
    views: np.ndarray     # [V,12] f32 world->camera (R row-major, t)
    seed: int
    extra: dict = field(default_factory=dict)

    @property
    def n(self):
        return self.mean_opa.shape[0]

    def params(self):
        return self.mean_opa, self.quat, self.logscale, self.rgb

    def params64(self):
        """fp64 copies (exact promotion of the fp32 values) for the oracle."""
        m = self.mean_opa.astype(np.float64)
        return dict(mean=m[:, :3].copy(), quat=self.quat.astype(np.float64),
                    logscale=self.logscale[:, :3].astype(np.float64),
                    logit=m[:, 3].copy(), rgb=self.rgb[:, :3].astype(np.float64))


def _unit_quats(rng, n):
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q


def _pack(mean, logit, quat, logscale, rgb):
    n = mean.shape[0]
    mo = np.zeros((n, 4), np.float32)
    mo[:, :3] = mean
    mo[:, 3] = logit
    ls = np.zeros((n, 4), np.float32)
    ls[:, :3] = logscale
    c = np.zeros((n, 4), np.float32)
    c[:, :3] = rgb
    return mo, quat.astype(np.float32), ls, c


def look_at(position, target, up=(0.0, -1.0, 0.0)):
    """World->camera (R, t) for a camera at `position` looking at `target`.

    Camera axes: z forward, x right, y down (image rows), so world "up" is -y
    (SURVEY §8(d)).  Rows of R are the camera axes in world coordinates.
    """
    position = np.asarray(position, np.float64)
    f = np.asarray(target, np.float64) - position
    f /= np.linalg.norm(f)
    x = np.cross(f, np.asarray(up, np.float64))
    x /= np.linalg.norm(x)
    y = np.cross(f, x)
    R = np.stack([x, y, f])
    t = -R @ position
    return R, t


def _view_row(R, t):
    return np.concatenate([np.asarray(R, np.float64).reshape(9),
                           np.asarray(t, np.float64)]).astype(np.float32)


def identity_view():
    return _view_row(np.eye(3), np.zeros(3))


def _frustum_means(rng, n, cam, z0, z1):
    """Uniform in the frustum volume: p(z) ~ z^2 on [z0, z1], pixel uniform."""
    u = rng.random(n)
    z = np.cbrt(z0 ** 3 + u * (z1 ** 3 - z0 ** 3))
    px = rng.uniform(-0.5, cam.width - 0.5, n)
    py = rng.uniform(-0.5, cam.height - 0.5, n)
    x = (px - cam.cx) * z / cam.fx
    y = (py - cam.cy) * z / cam.fy
    return np.stack([x, y, z], axis=1)


def _perturbed_copy(rng, s: Scene):
    """Targets of [3]/[4]: a perturbed copy."""
    n = s.n
    mo = s.mean_opa.astype(np.float64).copy()
    mo[:, :3] += rng.normal(0.0, 0.01, (n, 3))
    mo[:, 3] += rng.normal(0.0, 0.3, n)
    ls = s.logscale.astype(np.float64).copy()
    ls[:, :3] += rng.normal(0.0, 0.1, (n, 3))
    c = s.rgb.astype(np.float64).copy()
    c[:, :3] += rng.normal(0.0, 0.05, (n, 3))
    return (mo.astype(np.float32), s.quat.copy(), ls.astype(np.float32),
            c.astype(np.float32))


def config0(seed=0) -> Scene:
    """BJ.configs[0]: tiny scene, 256 Gaussians, 64x48, fx=fy=60, cx=32, cy=24."""
    rng = np.random.default_rng(seed)
    cam = Camera(64, 48, 60.0, 60.0, 32.0, 24.0)
    n = 256
    mean = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n),
                     rng.uniform(1, 4, n)], axis=1)
    logscale = rng.normal(-2.5, 0.3, (n, 3))
    quat = _unit_quats(rng, n)
    logit = rng.normal(0.0, 1.0, n)
    rgb = rng.uniform(0, 1, (n, 3))
    mo, q, ls, c = _pack(mean, logit, quat, logscale, rgb)
    tgt_color = rng.uniform(0, 1, (3, cam.height, cam.width)).astype(np.float32)
    tgt_depth = rng.uniform(1, 4, (cam.height, cam.width)).astype(np.float32)
    return Scene("tiny", cam, mo, q, ls, c, identity_view()[None], seed,
                 dict(tgt_color=tgt_color[None], tgt_depth=tgt_depth[None]))


def _frustum_scene(name, seed, n, cam, ls_mu, ls_sd, lo_sd):
    rng = np.random.default_rng(seed)
    mean = _frustum_means(rng, n, cam, 0.5, 5.0)
    logscale = rng.normal(ls_mu, ls_sd, (n, 3))
    quat = _unit_quats(rng, n)
    logit = rng.normal(0.0, lo_sd, n)
    rgb = rng.uniform(0, 1, (n, 3))
    mo, q, ls, c = _pack(mean, logit, quat, logscale, rgb)
    return rng, Scene(name, cam, mo, q, ls, c, identity_view()[None], seed)


def config1(seed=1) -> Scene:
    """BJ.configs[1]: single-view render, 100k Gaussians, 640x480, fx=fy=525."""
    cam = Camera(640, 480, 525.0, 525.0, 319.5, 239.5)
    rng, s = _frustum_scene("single_view", seed, 100_000, cam, -4.0, 0.5, 1.5)
    s.extra["tgt_color"] = rng.uniform(0, 1, (1, 3, cam.height, cam.width)).astype(np.float32)
    s.extra["tgt_depth"] = rng.uniform(0.5, 5.0, (1, cam.height, cam.width)).astype(np.float32)
    return s


def _small_rotation(rng, deg):
    axis = rng.standard_normal(3)
    axis /= np.linalg.norm(axis)
    th = np.deg2rad(deg)
    K = np.array([[0, -axis[2], axis[1]], [axis[2], 0, -axis[0]], [-axis[1], axis[0], 0]])
    return np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K


def config2(seed=2, n=200_000) -> Scene:
    """BJ.configs[2]: tracking, 200k Gaussians, 1200x680, fx=fy=600.

    GT pose = identity; start = exp(delta) GT with 2 deg about a random axis and
    5 cm along a random direction (left perturbation).  Targets are rendered
    from the GT pose by whichever side consumes the scene."""
    cam = Camera(1200, 680, 600.0, 600.0, 599.5, 339.5)
    rng, s = _frustum_scene("tracking", seed, n, cam, -4.0, 0.5, 1.5)
    dR = _small_rotation(rng, 2.0)
    d = rng.standard_normal(3)
    d *= 0.05 / np.linalg.norm(d)
    s.extra["gt_view"] = identity_view()
    s.extra["start_view"] = _view_row(dR, d)  # exp(delta)*I = (dR, d)
    s.extra["iters"] = 100
    return s


def arc_views(center, radius, arc_len, n_views):
    """Cameras evenly spaced on an arc of the given length (xz-plane, centred
    on the reference camera at the origin), each looking at `center`."""
    center = np.asarray(center, np.float64)
    span = arc_len / radius
    views = []
    for k in range(n_views):
        th = (k / (n_views - 1) - 0.5) * span if n_views > 1 else 0.0
        pos = center + radius * np.array([np.sin(th), 0.0, -np.cos(th)])
        views.append(_view_row(*look_at(pos, center)))
    return np.stack(views)


def config3(seed=3, n=500_000, n_views=8) -> Scene:
    """BJ.configs[3]: sub-map mapping, 500k Gaussians, 1200x680, 8 views on a
    1 m arc of radius 2.75 m about c = (0, 0, 2.75)."""
    cam = Camera(1200, 680, 600.0, 600.0, 599.5, 339.5)
    rng, s = _frustum_scene("submap", seed, n, cam, -4.0, 0.5, 1.5)
    s.views = arc_views((0.0, 0.0, 2.75), 2.75, 1.0, n_views)
    s.extra["target_params"] = _perturbed_copy(rng, s)
    return s


def config4(seed=4, n=2_000_000, n_views=64) -> Scene:
    """BJ.configs[4]: large mapping, 2M Gaussians in a 2.5 m ball, 1920x1080,
    fx=fy=960, 64 views on a horizontal circle of radius 3 m."""
    rng = np.random.default_rng(seed)
    cam = Camera(1920, 1080, 960.0, 960.0, 959.5, 539.5)
    d = rng.standard_normal((n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = 2.5 * np.cbrt(rng.random(n))
    mean = d * r[:, None]
    logscale = rng.normal(-4.5, 0.6, (n, 3))
    quat = _unit_quats(rng, n)
    logit = rng.normal(0.0, 2.0, n)
    rgb = rng.uniform(0, 1, (n, 3))
    mo, q, ls, c = _pack(mean, logit, quat, logscale, rgb)
    views = []
    for k in range(n_views):
        ph = 2 * np.pi * k / n_views
        pos = 3.0 * np.array([np.sin(ph), 0.0, -np.cos(ph)])
        views.append(_view_row(*look_at(pos, (0.0, 0.0, 0.0))))
    s = Scene("large", cam, mo, q, ls, c, np.stack(views), seed)
    s.extra["target_params"] = _perturbed_copy(rng, s)
    return s


def random_scene(seed, n, width, height, f=None, z=(1.0, 4.0), ls=(-2.5, 0.3),
                 lo=(0.0, 1.0), spread=1.0):
    """Small randomised scenes for property / FD / edge-case tests."""
    rng = np.random.default_rng(seed)
    f = f if f is not None else 0.9 * width
    cam = Camera(width, height, f, f, (width - 1) / 2, (height - 1) / 2)
    zz = rng.uniform(z[0], z[1], n)
    x = rng.uniform(-spread, spread, n) * zz * (width / 2) / f
    y = rng.uniform(-spread, spread, n) * zz * (height / 2) / f
    mean = np.stack([x, y, zz], axis=1)
    logscale = rng.normal(ls[0], ls[1], (n, 3))
    quat = _unit_quats(rng, n)
    logit = rng.normal(lo[0], lo[1], n)
    rgb = rng.uniform(0, 1, (n, 3))
    mo, q, l, c = _pack(mean, logit, quat, logscale, rgb)
    return Scene(f"random{seed}", cam, mo, q, l, c, identity_view()[None], seed)


def upstream_maps(seed, cam: Camera):
    """Random upstream gradients G_C [3,H,W], G_D, G_A ~ N(0,1)."""
    rng = np.random.default_rng(seed + 1000)
    gc = rng.standard_normal((3, cam.height, cam.width)).astype(np.float32)
    gd = rng.standard_normal((cam.height, cam.width)).astype(np.float32)
    ga = rng.standard_normal((cam.height, cam.width)).astype(np.float32)
    return gc, gd, ga


# depth unit of the synthetic sensor frames: 0.2 mm (TUM-RGBD's factor 5000;
# DESIGN.md R42)
DEPTH_SCALE = 1.0 / 5000.0


def quantize_rgbd(color, depth, scale=DEPTH_SCALE):
    """A synthetic RGB-D frame in the sensors' format (R42):
    rgb8 = round(clip(C, 0, 1) * 255) as [H, W, 3] uint8 and
    depth16 = round(D / scale) clipped to [0, 65535] as [H, W] uint16, from
    fp32 planar colour [3, H, W] and depth [H, W] (e.g. a target render)."""
    c = np.clip(np.asarray(color, np.float64), 0.0, 1.0)
    rgb8 = np.rint(c * 255.0).astype(np.uint8).transpose(1, 2, 0).copy()
    d16 = np.clip(np.rint(np.asarray(depth, np.float64) / float(np.float32(scale))), 0, 65535).astype(np.uint16)
    return rgb8, d16


CONFIGS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}
