"""Seeded synthetic light-field generator shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no warp W_k, blur B, decimation
D, weights, prox or solver step).  It renders a light field from an analytic
layered scene, the way a camera array would see it, and adds the paper's mixed
noise (reading A21).  Both sides of every parity test read
the same fp32 arrays produced here.

Scene recipe:
  * "hci": a slanted background plane plus ``n_objects`` depth-ordered rectangles
    and disks (10-35 % of the side), each with a constant disparity in
    [-omega_max, omega_max] (the HCI range, ~[-1.5, 1.5] px per angular step);
    textures are checkerboards (period 4-16 px), sinusoidal gratings (period
    3-12 px, random angle), sums of random sinusoids ("smooth noise") or flat,
    contrast 0.2-0.5, clipped to [0.05, 0.95].
  * "natural": a 1/f^2-spectrum texture (FFT-synthesised at 2x HR, sampled
    nearest) plus a few sharp-edged patches, on a smooth disparity plane in
    [-omega_max, omega_max].
A scene point at reference-view HR position z with disparity d appears in view k
at z - dtheta_k * d (dtheta_k = theta_k - theta_0 in angular steps; rho pairs with
the column axis, tau with the row axis).  Each LR pixel (i, j)
averages ``ss x ss`` point samples of the rendered view over the HR area
[zeta*i - zeta/2, zeta*i + zeta/2) x [...] (a box sensor footprint), so the
observations are NOT produced by the solver's own operator (occlusions are
rendered, the PSF is a box) - that only matters for PSNR realism, not parity.
``omega`` is the disparity of the front-most surface at each reference HR pixel.

Noise (reading A21): Gaussian sigma on the [0, 1] scale first, then nu % of the
pixels (chosen without replacement) set to 0 or 1 with probability 1/2, then
clamp to [0, 1].  Per-view noise streams: SeedSequence(noise_seed).spawn(s_k)
with the Philox bit generator.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, asdict

import numpy as np

__all__ = ["CONFIGS", "LightField", "SolverDefaults", "make_lightfield", "grid_offsets",
           "random_instance", "get_config"]


@dataclass(frozen=True)
class SolverDefaults:
    """Solver constants for the bench/parity configs (reading A20; frozen before timing).
    Chosen by a PSNR sweep of the GPU solver over lambda2 x lambda_reg x theta x sigma_e on
    C2/C3/C4 at N = 10 (tools/sweep.py, DESIGN.md §3 A20)."""
    lambda1: float = 1.0
    lambda2: float = 0.1
    lambda_reg: float = 0.5
    sigma_s: float = 3.0
    sigma_e: float = 0.2
    sigma_o1: float = 0.5
    sigma_o2: float = 0.2
    theta: float = 4.0
    radius: int = 2          # 5x5 NLTV window
    cg_max_iters: int = 5    # K = 5
    cg_tol: float = 0.0      # tau = 0: exactly K steps (reading A18)


@dataclass
class MisrDefaults:
    """Solver constants for the MISR use of the method:
    l1 data term only (lambda2 = 0), BTV regulariser -- offset weights alpha^(|dx|+|dy|)
    with no edge or occlusion weighting (sigma_e, sigma_o -> inf) -- on frames
    with global sub-pixel shifts (constant disparity)."""
    lambda1: float = 1.0
    lambda2: float = 0.0
    lambda_reg: float = 0.1       # M1 oracle sweep (lambda_reg x theta x alpha): 19.4 dB bicubic -> 24.6 dB at N = 20
    sigma_s: float = 3.0          # unused: offset_weights override w_d
    sigma_e: float = math.inf
    sigma_o1: float = math.inf
    sigma_o2: float = math.inf
    theta: float = 4.0
    radius: int = 2
    cg_max_iters: int = 5
    cg_tol: float = 0.0
    btv_alpha: float = 0.7

    @property
    def offset_weights(self):
        return btv_weights(self.radius, self.btv_alpha)


def btv_weights(radius: int, alpha: float) -> list:
    """BTV offset weights alpha^(|dx|+|dy|) in the offset order of reading A9 (row-major dy, dx
    over the (2r+1)^2 window, centre skipped) -- the lfsr_params.offset_weights layout."""
    return [float(alpha) ** (abs(dx) + abs(dy)) for dy in range(-radius, radius + 1)
            for dx in range(-radius, radius + 1) if (dy, dx) != (0, 0)]


@dataclass(frozen=True)
class Config:
    name: str
    grid: int           # angular grid side (grid x grid views)
    lr_h: int
    lr_w: int
    scale: int
    sigma: float        # Gaussian std on [0, 1]
    nu: float           # impulse percentage
    omega_max: float
    kind: str
    n_iters: int
    note: str = ""

    @property
    def n_views(self):
        return self.grid * self.grid

    @property
    def ref_view(self):
        return 0 if self.kind == "misr" else self.n_views // 2

    @property
    def H(self):
        return self.lr_h * self.scale

    @property
    def W(self):
        return self.lr_w * self.scale


# BASELINE.json configs -> SURVEY §8d.1 table.
CONFIGS = {
    "C1": Config("C1", 3, 32, 32, 2, 0.02, 5.0, 1.5, "hci", 20, "3x3 views, 32x32 LR -> x2 (64x64 HR)"),
    "C2": Config("C2", 5, 256, 256, 2, 0.02, 5.0, 1.5, "hci", 10, "5x5 views, 256x256 LR -> x2 (512x512 HR)"),
    "C3": Config("C3", 9, 256, 256, 2, 0.05, 20.0, 1.5, "hci", 10, "9x9 views, 256x256 LR -> x2 (512x512 HR), sigma=0.05 + 20% impulse"),
    "C4": Config("C4", 9, 171, 171, 3, 0.05, 20.0, 1.5, "hci", 10, "9x9 views, 171x171 LR -> x3 (513x513 HR)"),
    "C5": Config("C5", 9, 512, 512, 4, 0.02, 5.0, 1.0, "natural", 10, "9x9 views, 512x512 LR -> x4 (2048x2048 HR)"),
    # MISR: grid x grid frames with global shifts of 1/zeta LR px (= 1 HR px),
    # constant disparity 1, natural-image texture (DIV8K-shaped; tab:mfsr)
    "M1": Config("M1", 2, 32, 32, 2, 0.02, 5.0, 1.0, "misr", 20, "MISR 4 frames x2, 32x32 LR -> 64x64 HR"),
    "M2": Config("M2", 2, 1024, 1024, 2, 0.02, 5.0, 1.0, "misr", 10, "MISR 4 frames x2 (1/2-px shifts), 1024^2 LR -> 2048^2 HR"),
    "M3": Config("M3", 3, 512, 512, 3, 0.02, 5.0, 1.0, "misr", 10, "MISR 9 frames x3 (1/3-px shifts), 512^2 LR -> 1536^2 HR"),
}


def misr_offsets(grid: int) -> np.ndarray:
    """[grid*grid][2] = (drho, dtau) = (b, a) HR px for a, b in [0, grid): the MISR frame
    shifts (1/zeta LR px steps at zeta = grid), frame 0 unshifted (the reference)."""
    out = np.zeros((grid * grid, 2), dtype=np.float32)
    for a in range(grid):
        for b in range(grid):
            out[a * grid + b] = (b, a)
    return out


def get_config(name: str) -> Config:
    return CONFIGS[name]


def defaults_for(cfg) -> "SolverDefaults | MisrDefaults":
    """The frozen solver constants of a config: MisrDefaults for the MISR configs."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return MisrDefaults() if cfg.kind == "misr" else SolverDefaults()


def grid_offsets(grid: int) -> np.ndarray:
    """[grid*grid][2] = (drho, dtau) = theta_k - theta_0 for a square angular grid,
    views row-major (row = tau, column = rho), theta_0 at the centre (reading A13)."""
    c = (grid - 1) / 2.0
    out = np.zeros((grid * grid, 2), dtype=np.float32)
    for a in range(grid):
        for b in range(grid):
            out[a * grid + b] = (b - c, a - c)
    return out


@dataclass
class LightField:
    y: np.ndarray             # [n_views][lr_h][lr_w] fp32 noisy LR views
    view_offsets: np.ndarray  # [n_views][2] fp32 (drho, dtau)
    omega: np.ndarray         # [H][W] fp32 disparity of the reference view (HR px / step)
    x_gt: np.ndarray          # [H][W] fp32 ground-truth reference view
    scale: int
    ref_view: int
    meta: dict = field(default_factory=dict)

    @property
    def n_views(self):
        return self.y.shape[0]


# ----------------------------------------------------------------------------- textures
def _texture(rng, kind):
    """Returns a callable (Y, X) -> intensity in reference HR coordinates."""
    base = rng.uniform(0.2, 0.8)
    contrast = rng.uniform(0.2, 0.5)
    if kind == "checker":
        period = rng.uniform(4, 16)
        phase = rng.uniform(0, period, size=2)
        return lambda Y, X: base + contrast * (
            ((np.floor((Y + phase[0]) / period) + np.floor((X + phase[1]) / period)) % 2) - 0.5)
    if kind == "grating":
        period = rng.uniform(3, 12)
        ang = rng.uniform(0, math.pi)
        c, s = math.cos(ang), math.sin(ang)
        ph = rng.uniform(0, 2 * math.pi)
        return lambda Y, X: base + 0.5 * contrast * np.sin(2 * math.pi * (c * X + s * Y) / period + ph)
    if kind == "noise":
        n = 6
        periods = rng.uniform(6, 40, size=n)
        angs = rng.uniform(0, math.pi, size=n)
        phs = rng.uniform(0, 2 * math.pi, size=n)
        amps = rng.uniform(0.5, 1.0, size=n)
        amps = amps / amps.sum()

        def f(Y, X):
            v = np.zeros(np.broadcast(Y, X).shape)
            for i in range(n):
                v += amps[i] * np.sin(2 * math.pi * (math.cos(angs[i]) * X + math.sin(angs[i]) * Y) / periods[i] + phs[i])
            return base + 0.5 * contrast * v
        return f
    return lambda Y, X: np.full(np.broadcast(Y, X).shape, base)


class _Layer:
    def __init__(self, shape, params, disp, tex):
        self.shape = shape      # "rect" | "disk" | "plane"
        self.params = params
        self.disp = disp        # constant or (a, b, c): d = a + b*Y + c*X
        self.tex = tex

    def disparity(self, Y, X):
        if isinstance(self.disp, tuple):
            a, b, c = self.disp
            return a + b * Y + c * X
        return np.full(np.broadcast(Y, X).shape, float(self.disp))

    def ref_position(self, Yv, Xv, drho, dtau):
        """Reference-view position z seen at view position z' (z' = z - dtheta d(z))."""
        if isinstance(self.disp, tuple):
            Y, X = Yv, Xv
            for _ in range(3):  # fixed point; the plane is gentle
                d = self.disparity(Y, X)
                Y, X = Yv + dtau * d, Xv + drho * d
            return Y, X
        d = float(self.disp)
        return Yv + dtau * d, Xv + drho * d

    def inside(self, Y, X):
        if self.shape == "plane":
            return np.ones(np.broadcast(Y, X).shape, dtype=bool)
        if self.shape == "rect":
            y0, x0, y1, x1 = self.params
            return (Y >= y0) & (Y < y1) & (X >= x0) & (X < x1)
        cy, cx, r = self.params
        return (Y - cy) ** 2 + (X - cx) ** 2 < r * r


def _natural_texture(rng, H, W):
    over = 2
    n = max(H, W) * over
    fy = np.fft.fftfreq(n)[:, None]
    fx = np.fft.rfftfreq(n)[None, :]
    f2 = fy * fy + fx * fx
    f2[0, 0] = 1.0
    amp = 1.0 / f2  # 1/f^2 power spectrum -> amplitude 1/f ... use 1/f^2 amplitude for smoothness
    amp = np.sqrt(amp)
    amp[0, 0] = 0.0
    spec = amp * (rng.standard_normal(amp.shape) + 1j * rng.standard_normal(amp.shape))
    img = np.fft.irfft2(spec, s=(n, n))
    img = (img - img.mean()) / (img.std() + 1e-12)
    img = 0.5 + 0.12 * img
    img = np.clip(img, 0.05, 0.95).astype(np.float32)

    def f(Y, X):
        iy = np.clip(np.floor(Y * over).astype(np.int64) % n, 0, n - 1)
        ix = np.clip(np.floor(X * over).astype(np.int64) % n, 0, n - 1)
        return img[iy, ix]
    return f


def _build_scene(kind, H, W, omega_max, rng, n_objects):
    layers = []
    if kind == "misr":   # one textured plane at constant disparity omega_max: frames are global shifts
        layers.append(_Layer("plane", None, float(omega_max), _natural_texture(rng, H, W)))
        return layers
    if kind == "natural":
        # smooth disparity plane over the whole frame within [-omega_max, omega_max]
        d0 = rng.uniform(-0.3, 0.3) * omega_max
        gy = rng.uniform(-1, 1) * (omega_max - abs(d0)) / max(H, 1)
        gx = rng.uniform(-1, 1) * (omega_max - abs(d0)) / max(W, 1)
        a = d0 - gy * H / 2 - gx * W / 2
        tex = _natural_texture(rng, H, W)
        layers.append(_Layer("plane", None, (a, gy, gx), tex))
        for _ in range(3):  # a few sharp edges, riding the same plane
            h_ = rng.uniform(0.1, 0.3) * H
            w_ = rng.uniform(0.1, 0.3) * W
            y0 = rng.uniform(0, H - h_)
            x0 = rng.uniform(0, W - w_)
            off = rng.uniform(-0.25, 0.25)
            layers.append(_Layer("rect", (y0, x0, y0 + h_, x0 + w_), (a, gy, gx),
                                 (lambda t, o: (lambda Y, X: t(Y, X) + o))(tex, off)))
        return layers
    # "hci": background plane + depth-ordered objects
    span = omega_max * rng.uniform(0.3, 0.6)
    gy = rng.uniform(-1, 1) * span / H
    gx = rng.uniform(-1, 1) * span / W
    a = rng.uniform(-omega_max, omega_max) * 0.3 - gy * H / 2 - gx * W / 2
    tex_kinds = ["checker", "grating", "noise", "flat"]
    layers.append(_Layer("plane", None, (a, gy, gx), _texture(rng, rng.choice(["noise", "grating"]))))
    objs = []
    for _ in range(n_objects):
        side = rng.uniform(0.10, 0.35) * min(H, W)
        d = rng.uniform(-omega_max, omega_max)
        tex = _texture(rng, rng.choice(tex_kinds))
        if rng.uniform() < 0.5:
            y0 = rng.uniform(-0.1 * H, H - 0.6 * side)
            x0 = rng.uniform(-0.1 * W, W - 0.6 * side)
            h_ = side * rng.uniform(0.6, 1.4)
            objs.append(_Layer("rect", (y0, x0, y0 + h_, x0 + side), d, tex))
        else:
            objs.append(_Layer("disk", (rng.uniform(0, H), rng.uniform(0, W), side / 2), d, tex))
    objs.sort(key=lambda L: L.disp)  # larger disparity = nearer = drawn later (on top)
    return layers + objs


def _render(layers, Ys, Xs, drho, dtau):
    """Front-most layer colour at view-k positions (Ys, Xs); also its disparity."""
    img = np.zeros(Ys.shape)
    disp = np.zeros(Ys.shape)
    for L in layers:  # back to front
        Yr, Xr = L.ref_position(Ys, Xs, drho, dtau)
        msk = L.inside(Yr, Xr)
        if not msk.any():
            continue
        img[msk] = L.tex(Yr[msk], Xr[msk])       # evaluate textures only where the layer is seen
        disp[msk] = L.disparity(Yr[msk], Xr[msk])
    return img, disp


def make_lightfield(cfg: Config | str, seed: int | None = None, ss: int = 2,
                    views: np.ndarray | None = None, noise: bool = True) -> LightField:
    """Render a synthetic LF for config ``cfg`` (a Config or a CONFIGS key).

    scene_seed = 1000 + config#, noise_seed = 2000 + config# unless ``seed`` overrides
    both.  ``views`` optionally replaces the full angular grid by a
    subset of (drho, dtau) offsets (the reference view must be among them)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    cnum = int(cfg.name[1:]) if cfg.name[1:].isdigit() else 0
    scene_seed = 1000 + cnum if seed is None else seed
    noise_seed = 2000 + cnum if seed is None else seed + 1
    rng = np.random.Generator(np.random.Philox(scene_seed))
    H, W, z = cfg.H, cfg.W, cfg.scale
    layers = _build_scene(cfg.kind, H, W, cfg.omega_max, rng, n_objects=8)
    if views is not None:
        vo = np.asarray(views, dtype=np.float32)
    else:
        vo = misr_offsets(cfg.grid) if cfg.kind == "misr" else grid_offsets(cfg.grid)
    ref = int(np.argmin(np.abs(vo).sum(axis=1)))

    # reference view at HR (area average over each HR pixel) and its disparity map
    Yc, Xc = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    gt = np.zeros((H, W))
    for sy in range(ss):
        for sx in range(ss):
            im, _ = _render(layers, Yc + (sy + 0.5) / ss - 0.5, Xc + (sx + 0.5) / ss - 0.5, 0.0, 0.0)
            gt += im
    gt /= ss * ss
    _, omega = _render(layers, Yc, Xc, 0.0, 0.0)
    omega = np.clip(omega, -cfg.omega_max, cfg.omega_max)

    # LR views: box footprint of zeta x zeta HR pixels around (zeta*i, zeta*j)
    h, w = cfg.lr_h, cfg.lr_w
    Yl, Xl = np.meshgrid(np.arange(h, dtype=np.float64) * z, np.arange(w, dtype=np.float64) * z, indexing="ij")
    y = np.zeros((len(vo), h, w), dtype=np.float32)
    nss = max(ss, 2)
    for k in range(len(vo)):
        drho, dtau = float(vo[k, 0]), float(vo[k, 1])
        acc = np.zeros((h, w))
        for sy in range(nss):
            for sx in range(nss):
                oy = ((sy + 0.5) / nss - 0.5) * z
                ox = ((sx + 0.5) / nss - 0.5) * z
                im, _ = _render(layers, Yl + oy, Xl + ox, drho, dtau)
                acc += im
        y[k] = (acc / (nss * nss)).astype(np.float32)
    y = np.clip(y, 0.0, 1.0)
    if noise:
        y = add_mixed_noise(y, cfg.sigma, cfg.nu, noise_seed)
    return LightField(y=y.astype(np.float32), view_offsets=vo.astype(np.float32),
                      omega=omega.astype(np.float32), x_gt=gt.astype(np.float32),
                      scale=z, ref_view=ref,
                      meta={"config": cfg.name, "scene_seed": scene_seed, "noise_seed": noise_seed,
                            "kind": cfg.kind, "sigma": cfg.sigma, "nu": cfg.nu, "ss": ss})


def add_mixed_noise(y: np.ndarray, sigma: float, nu: float, noise_seed: int) -> np.ndarray:
    """Gaussian (sigma on [0,1]) then nu % salt-and-pepper without replacement, clamp (A21)."""
    out = np.array(y, dtype=np.float64, copy=True)
    children = np.random.SeedSequence(noise_seed).spawn(out.shape[0])
    for k in range(out.shape[0]):
        g = np.random.Generator(np.random.Philox(children[k]))
        v = out[k]
        if sigma > 0:
            v = v + g.normal(0.0, sigma, size=v.shape)
        n = v.size
        cnt = int(math.floor(nu * n / 100.0))
        if cnt > 0:
            idx = g.choice(n, size=cnt, replace=False)
            flat = v.reshape(-1)
            flat[idx] = (g.uniform(size=cnt) < 0.5).astype(np.float64)
            v = flat.reshape(v.shape)
        out[k] = np.clip(v, 0.0, 1.0)
    return out.astype(np.float32)


def random_instance(seed: int, n_views: int, lr_h: int, lr_w: int, scale: int,
                    omega_max: float = 1.5, grid: int | None = None):
    """Small random instance for operator tests: (y, view_offsets, omega, x) fp32.
    Offsets are generic fractional values (so warps are not integer translations)."""
    g = np.random.Generator(np.random.Philox(seed))
    H, W = lr_h * scale, lr_w * scale
    if grid is not None:
        vo = grid_offsets(grid)[:n_views]
    else:
        vo = g.uniform(-2.0, 2.0, size=(n_views, 2)).astype(np.float32)
    # smooth-ish disparity with a discontinuity
    Y, X = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
    om = omega_max * (0.6 * np.sin(2 * np.pi * Y / max(H, 2) * g.uniform(0.5, 1.5))
                      * np.cos(2 * np.pi * X / max(W, 2) * g.uniform(0.5, 1.5)))
    om = om + np.where(X > W * g.uniform(0.3, 0.7), 0.4 * omega_max, 0.0)
    om = np.clip(om, -omega_max, omega_max).astype(np.float32)
    x = g.uniform(0.0, 1.0, size=(H, W)).astype(np.float32)
    y = g.uniform(0.0, 1.0, size=(n_views, lr_h, lr_w)).astype(np.float32)
    return y, vo.astype(np.float32), om, x


def config_dict(cfg: Config) -> dict:
    return asdict(cfg)


def per_view_disparity(omega: np.ndarray, n_views: int, amp: float = 0.2, seed: int = 0) -> np.ndarray:
    """[n_views][H][W] fp32 per-view disparity maps omega_k on theta_0's grid (LFSR_DISP_PER_VIEW,
    reading A34): the shared map plus a smooth per-view perturbation of amplitude `amp` (a
    low-frequency sinusoid with a random phase and direction per view), e.g. the per-view
    estimates a disparity estimator would return.  Input generator only; no method arithmetic."""
    g = np.random.Generator(np.random.Philox(seed))
    H, W = omega.shape
    Y, X = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    out = np.empty((n_views, H, W), np.float32)
    for k in range(n_views):
        fy, fx = g.uniform(0.5, 2.0, size=2) / np.array([max(H, 2), max(W, 2)])
        ph = g.uniform(0.0, 2.0 * np.pi)
        out[k] = (omega + amp * np.sin(2.0 * np.pi * (fy * Y + fx * X) + ph)).astype(np.float32)
    return out


def motion_psf(length: int, angle_deg: float = 45.0) -> np.ndarray:
    """Normalised linear motion-blur kernel (the 45-degree motion blur of P:L962), fp32
    [(2r+1)][(2r+1)] with r = (length-1)//2: a centred segment whose projection on the
    dominant axis spans `length` pixels, rasterised by dense sampling.  Input generator only."""
    r = (length - 1) // 2
    a = np.deg2rad(angle_deg)
    c, s = np.cos(a), -np.sin(a)          # row axis points down
    half = (length - 1) / 2.0 / max(abs(c), abs(s))
    k = np.zeros((2 * r + 1, 2 * r + 1))
    for t in np.linspace(-half, half, 64 * length):
        k[int(round(r + t * s)), int(round(r + t * c))] += 1.0
    return (k / k.sum()).astype(np.float32)
