"""CPU fp64 oracle for the ADMM LF-SR hot path (arXiv 2206.05047) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2206_05047_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle.c`` (plain C, fp64, one loop nest per operator,
each citing the PAPER.md passage it follows).  This module is only ctypes
marshalling: numpy arrays in, numpy arrays out.  Inputs are promoted to fp64.

Parity status: every function is pinned by ``tests/test_oracle_pins.py`` (see the
header of ``oracle.c`` for the pin of each function); none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc -O2 -fopenmp, strict IEEE: no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               "-Wall", "-Wno-unknown-pragmas", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [("n_views", ctypes.c_int32), ("lr_h", ctypes.c_int32), ("lr_w", ctypes.c_int32),
                ("scale", ctypes.c_int32), ("ref_view", ctypes.c_int32), ("radius", ctypes.c_int32),
                ("lambda1", ctypes.c_double), ("lambda2", ctypes.c_double),
                ("lambda_reg", ctypes.c_double), ("sigma_s", ctypes.c_double),
                ("sigma_e", ctypes.c_double), ("sigma_o1", ctypes.c_double),
                ("sigma_o2", ctypes.c_double), ("theta", ctypes.c_double),
                ("cg_max_iters", ctypes.c_int32), ("cg_tol", ctypes.c_double),
                ("reweight_every_iter", ctypes.c_int32),
                ("offset_weights", ctypes.POINTER(ctypes.c_double)), ("disp_per_view", ctypes.c_int32),
                ("psf", ctypes.POINTER(ctypes.c_double)), ("psf_radius", ctypes.c_int32),
                ("paper_adjoint", ctypes.c_int32)]


class _Stats(ctypes.Structure):
    _fields_ = [("iter", ctypes.c_int32), ("cg_iters", ctypes.c_int32),
                ("breakdown", ctypes.c_int32), ("nonfinite", ctypes.c_int32),
                ("J", ctypes.c_double), ("data_l1", ctypes.c_double), ("data_l2", ctypes.c_double),
                ("reg_l1", ctypes.c_double), ("primal_res", ctypes.c_double),
                ("cg_pi0", ctypes.c_double), ("cg_pi_last", ctypes.c_double)]


class _GdStats(ctypes.Structure):
    _fields_ = [("iter", ctypes.c_int32), ("ls_evals", ctypes.c_int32),
                ("ls_failed", ctypes.c_int32), ("nonfinite", ctypes.c_int32),
                ("J", ctypes.c_double), ("data_l1", ctypes.c_double), ("data_l2", ctypes.c_double),
                ("reg_l1", ctypes.c_double), ("step", ctypes.c_double), ("grad_sq", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        D = ctypes.POINTER(ctypes.c_double)
        P = ctypes.POINTER(_Params)
        I = ctypes.c_int
        sig = {
            "or_blur_taps": (I, [I, D]),
            "or_apply_D": (None, [I, I, I, D, D]),
            "or_apply_DT": (None, [I, I, I, D, D]),
            "or_apply_B": (None, [I, I, I, D, D, D]),
            "or_apply_W": (None, [I, I, D, D, ctypes.c_double, ctypes.c_double, D]),
            "or_apply_WT": (None, [I, I, D, D, ctypes.c_double, ctypes.c_double, D]),
            "or_apply_A": (None, [P, D, D, D, D]),
            "or_apply_AT": (None, [P, D, D, D, D]),
            "or_offsets": (I, [I, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
            "or_apply_S": (None, [I, I, I, ctypes.c_double, D, D, D]),
            "or_apply_ST": (None, [I, I, I, ctypes.c_double, D, D, D]),
            "or_apply_Sw": (None, [I, I, I, D, D, D, D]),
            "or_apply_STw": (None, [I, I, I, D, D, D, D]),
            "or_weights_m": (None, [I, I, ctypes.c_double, ctypes.c_double, D, D, D]),
            "or_setup_wo": (None, [P, D, D, D, D, D, D]),
            "or_bicubic": (None, [I, I, I, D, D]),
            "or_normal": (None, [P, D, D, D, D, D]),
            "or_admm": (I, [P, D, D, D, D, I, D, D, D, D, ctypes.POINTER(_Stats)]),
            "or_cost": (ctypes.c_double, [P, D, D, D, D, D, D]),
            "or_gradient": (ctypes.c_double, [P, D, D, D, D, D, D, D]),
            "or_apply_Bk": (None, [I, I, I, D, D, D]),
            "or_apply_WTb": (None, [I, I, D, D, ctypes.c_double, ctypes.c_double, D]),
            "or_apply_BkT": (None, [I, I, I, D, D, D]),
            "or_rgb_to_ycbcr": (None, [ctypes.c_size_t, D, D, D, D]),
            "or_ycbcr_to_rgb": (None, [ctypes.c_size_t, D, D, D, D]),
            "or_gd": (I, [P, D, D, D, D, I, ctypes.c_double, I, I, ctypes.c_double, D, D,
                          ctypes.POINTER(_GdStats)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype = res
            f.argtypes = args
    return _lib


def _d(a):
    """fp64 C-contiguous view (or copy) of a; None passes through."""
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


@dataclass
class Params:
    """Solver parameters (SURVEY §8b lfsr_params; defaults = reading A20 starting point)."""
    n_views: int
    lr_h: int
    lr_w: int
    scale: int = 2
    ref_view: int = 0
    radius: int = 2
    lambda1: float = 1.0
    lambda2: float = 10.0
    lambda_reg: float = 0.1
    sigma_s: float = 3.0
    sigma_e: float = 0.01
    sigma_o1: float = 0.5
    sigma_o2: float = 0.2
    theta: float = 1.0
    cg_max_iters: int = 5
    cg_tol: float = 0.0
    reweight_every_iter: int = 1
    offset_weights: Optional[Sequence[float]] = None   # s_d weights overriding exp(-|d|^2/sigma_s)
    disp_per_view: int = 0      # 1: omega is [n_views][H][W] (view k warped with omega_k, A34)
    psf: Optional[np.ndarray] = None   # user convolution kernel [(2r+1)][(2r+1)] replacing the Gaussian (A36)
    paper_adjoint: int = 0      # 1: A^T uses the paper's backward warp W_k^* with omega_0 (A37)

    @property
    def H(self):
        return self.lr_h * self.scale

    @property
    def W(self):
        return self.lr_w * self.scale

    @property
    def s_d(self):
        return (2 * self.radius + 1) ** 2 - 1

    def c(self):
        ow = None
        if self.offset_weights is not None:
            self._ow = np.ascontiguousarray(self.offset_weights, dtype=np.float64)   # kept alive with self
            assert self._ow.shape == (self.s_d,), "offset_weights must have s_d entries"
            ow = _ptr(self._ow)
        kp, kr = None, 0
        if self.psf is not None:
            self._psf = np.ascontiguousarray(self.psf, dtype=np.float64)
            assert self._psf.ndim == 2 and self._psf.shape[0] == self._psf.shape[1] and self._psf.shape[0] % 2 == 1
            kp, kr = _ptr(self._psf), (self._psf.shape[0] - 1) // 2
        return _Params(self.n_views, self.lr_h, self.lr_w, self.scale, self.ref_view, self.radius,
                       self.lambda1, self.lambda2, self.lambda_reg, self.sigma_s, self.sigma_e,
                       self.sigma_o1, self.sigma_o2, self.theta, self.cg_max_iters, self.cg_tol,
                       self.reweight_every_iter, ow, int(self.disp_per_view), kp, kr, int(self.paper_adjoint))


def blur_taps(scale: int) -> np.ndarray:
    buf = np.zeros(64)
    R = lib().or_blur_taps(scale, _ptr(buf))
    return buf[: 2 * R + 1].copy()


def offsets(radius: int):
    dys = (ctypes.c_int * 1024)()
    dxs = (ctypes.c_int * 1024)()
    n = lib().or_offsets(radius, dys, dxs)
    return [(dys[i], dxs[i]) for i in range(n)]


def apply_D(x, scale):
    x = _d(x)
    H, W = x.shape
    out = np.zeros((H // scale, W // scale))
    lib().or_apply_D(H, W, scale, _ptr(x), _ptr(out))
    return out


def apply_DT(y, scale):
    y = _d(y)
    h, w = y.shape
    out = np.zeros((h * scale, w * scale))
    lib().or_apply_DT(h * scale, w * scale, scale, _ptr(y), _ptr(out))
    return out


def apply_B(x, scale):
    x = _d(x)
    H, W = x.shape
    taps = blur_taps(scale)
    R = (len(taps) - 1) // 2
    out = np.zeros_like(x)
    lib().or_apply_B(H, W, R, _ptr(taps), _ptr(x), _ptr(out))
    return out


def apply_Bk(x, k, transpose: bool = False):
    """B with a user convolution kernel k (reading A36), or its transpose."""
    x, k = _d(x), _d(k)
    H, W = x.shape
    out = np.zeros_like(x)
    f = lib().or_apply_BkT if transpose else lib().or_apply_Bk
    f(H, W, (k.shape[0] - 1) // 2, _ptr(k), _ptr(x), _ptr(out))
    return out


def apply_W(x, omega, drho, dtau):
    x, omega = _d(x), _d(omega)
    out = np.zeros_like(x)
    lib().or_apply_W(x.shape[0], x.shape[1], _ptr(x), _ptr(omega), float(drho), float(dtau), _ptr(out))
    return out


def apply_WTb(u, omega0, drho, dtau):
    """The paper's backward warp W_k^* (reading A37): u(z - dtheta_k omega_0(z))."""
    u, omega0 = _d(u), _d(omega0)
    out = np.zeros_like(u)
    lib().or_apply_WTb(u.shape[0], u.shape[1], _ptr(u), _ptr(omega0), float(drho), float(dtau), _ptr(out))
    return out


def apply_WT(t, omega, drho, dtau):
    t, omega = _d(t), _d(omega)
    out = np.zeros_like(t)
    lib().or_apply_WT(t.shape[0], t.shape[1], _ptr(t), _ptr(omega), float(drho), float(dtau), _ptr(out))
    return out


def apply_A(P: Params, view_offsets, omega, x):
    vo, om, x = _d(view_offsets), _d(omega), _d(x)
    out = np.zeros((P.n_views, P.lr_h, P.lr_w))
    pc = P.c()
    lib().or_apply_A(ctypes.byref(pc), _ptr(vo), _ptr(om), _ptr(x), _ptr(out))
    return out


def apply_AT(P: Params, view_offsets, omega, r):
    vo, om, r = _d(view_offsets), _d(omega), _d(r)
    out = np.zeros((P.H, P.W))
    pc = P.c()
    lib().or_apply_AT(ctypes.byref(pc), _ptr(vo), _ptr(om), _ptr(r), _ptr(out))
    return out


def apply_S(x, m, radius, sigma_s, weights=None):
    """S; weights: optional s_d offset weights replacing exp(-|d|^2/sigma_s)."""
    x, m = _d(x), _d(m)
    H, W = x.shape
    sd = (2 * radius + 1) ** 2 - 1
    out = np.zeros((sd, H, W))
    if weights is None:
        lib().or_apply_S(H, W, radius, float(sigma_s), _ptr(m), _ptr(x), _ptr(out))
    else:
        wv = _d(weights)
        lib().or_apply_Sw(H, W, radius, _ptr(wv), _ptr(m), _ptr(x), _ptr(out))
    return out


def apply_ST(h, m, radius, sigma_s, weights=None):
    """S^T; weights as in apply_S."""
    h, m = _d(h), _d(m)
    _, H, W = h.shape
    out = np.zeros((H, W))
    if weights is None:
        lib().or_apply_ST(H, W, radius, float(sigma_s), _ptr(m), _ptr(h), _ptr(out))
    else:
        wv = _d(weights)
        lib().or_apply_STw(H, W, radius, _ptr(wv), _ptr(m), _ptr(h), _ptr(out))
    return out


def weights_m(x, wo, lambda_reg, sigma_e):
    x, wo = _d(x), _d(wo)
    H, W = x.shape
    out = np.zeros((H, W))
    lib().or_weights_m(H, W, float(lambda_reg), float(sigma_e), _ptr(wo), _ptr(x), _ptr(out))
    return out


def setup_wo(P: Params, y, view_offsets, omega):
    """Returns (w_o, b, p) on the HR grid."""
    y, vo, om = _d(y), _d(view_offsets), _d(omega)
    wo = np.zeros((P.H, P.W))
    b = np.zeros((P.H, P.W))
    p = np.zeros((P.H, P.W))
    pc = P.c()
    lib().or_setup_wo(ctypes.byref(pc), _ptr(y), _ptr(vo), _ptr(om), _ptr(wo), _ptr(b), _ptr(p))
    return wo, b, p


def bicubic(yref, scale):
    yref = _d(yref)
    h, w = yref.shape
    out = np.zeros((h * scale, w * scale))
    lib().or_bicubic(h, w, scale, _ptr(yref), _ptr(out))
    return out


def normal(P: Params, view_offsets, omega, m, p):
    vo, om, m, p = _d(view_offsets), _d(omega), _d(m), _d(p)
    out = np.zeros((P.H, P.W))
    pc = P.c()
    lib().or_normal(ctypes.byref(pc), _ptr(vo), _ptr(om), _ptr(m), _ptr(p), _ptr(out))
    return out


def cost(P: Params, y, view_offsets, omega, m, x):
    y, vo, om, m, x = _d(y), _d(view_offsets), _d(omega), _d(m), _d(x)
    t = np.zeros(3)
    pc = P.c()
    J = lib().or_cost(ctypes.byref(pc), _ptr(y), _ptr(vo), _ptr(om), _ptr(m), _ptr(x), _ptr(t))
    return J, t


@dataclass
class AdmmResult:
    x_iters: np.ndarray          # [N+1][H][W], x^0 .. x^N
    wA: np.ndarray               # [n_views][h][w]
    wS: np.ndarray               # [s_d][H][W]
    stats: list = field(default_factory=list)
    status: int = 0


STAT_KEYS = ("iter", "cg_iters", "breakdown", "nonfinite", "J", "data_l1", "data_l2", "reg_l1",
             "primal_res", "cg_pi0", "cg_pi_last")


def admm(P: Params, y, view_offsets, omega, n_iters: int, x0=None) -> AdmmResult:
    """Algorithm 1 + Algorithm 2 in fp64; see oracle.c or_admm."""
    y, vo, om, x0 = _d(y), _d(view_offsets), _d(omega), _d(x0)
    xs = np.zeros((n_iters + 1, P.H, P.W))
    xo = np.zeros((P.H, P.W))
    wA = np.zeros((P.n_views, P.lr_h, P.lr_w))
    wS = np.zeros((P.s_d, P.H, P.W))
    st = (_Stats * max(n_iters, 1))()
    pc = P.c()
    rc = lib().or_admm(ctypes.byref(pc), _ptr(y), _ptr(vo), _ptr(om), _ptr(x0), int(n_iters),
                       _ptr(xs), _ptr(xo), _ptr(wA), _ptr(wS), st)
    if rc == 1:
        raise ValueError("oracle: invalid parameters")
    stats = [{k: getattr(st[i], k) for k in STAT_KEYS} for i in range(n_iters)]
    return AdmmResult(xs, wA, wS, stats, rc)


def gradient(P: Params, y, view_offsets, omega, m, x):
    """J(x) and its subgradient sum_k A_k^T (l1 sgn(e_k) + 2 l2 e_k) + S_w^T sgn(S_w x) for the
    weight map m (reading A30).  Returns (J, terms3, g)."""
    y, vo, om, m, x = _d(y), _d(view_offsets), _d(omega), _d(m), _d(x)
    g = np.zeros((P.H, P.W))
    t = np.zeros(3)
    pc = P.c()
    J = lib().or_gradient(ctypes.byref(pc), _ptr(y), _ptr(vo), _ptr(om), _ptr(m), _ptr(x), _ptr(g), _ptr(t))
    return J, t, g


GD_STAT_KEYS = ("iter", "ls_evals", "ls_failed", "nonfinite", "J", "data_l1", "data_l2", "reg_l1",
                "step", "grad_sq")


@dataclass
class GdResult:
    x_iters: np.ndarray          # [N+1][H][W], x^0 .. x^N
    stats: list = field(default_factory=list)
    status: int = 0


def gd(P: Params, y, view_offsets, omega, n_iters: int, step: float, line_search: bool = False,
       max_halvings: int = 30, armijo_c: float = 1e-4, x0=None) -> GdResult:
    """gd / gd-ls baselines of the solver comparison (readings A30-A33); see
    oracle.c or_gd.  CU of iteration n: 2 + stats[n]["ls_evals"] (A33)."""
    y, vo, om, x0 = _d(y), _d(view_offsets), _d(omega), _d(x0)
    xs = np.zeros((n_iters + 1, P.H, P.W))
    st = (_GdStats * max(n_iters, 1))()
    pc = P.c()
    rc = lib().or_gd(ctypes.byref(pc), _ptr(y), _ptr(vo), _ptr(om), _ptr(x0), int(n_iters), float(step),
                     int(bool(line_search)), int(max_halvings), float(armijo_c), _ptr(xs), None, st)
    if rc == 1:
        raise ValueError("oracle: invalid parameters")
    stats = [{k: getattr(st[i], k) for k in GD_STAT_KEYS} for i in range(n_iters)]
    return GdResult(xs, stats, rc)


def rgb_to_ycbcr(rgb):
    """Planar [3][...] RGB -> (Y, Cb, Cr), full-range BT.601 (reading A35)."""
    rgb = _d(rgb)
    shp = rgb.shape[1:]
    n = int(np.prod(shp))
    y, cb, cr = np.zeros(shp), np.zeros(shp), np.zeros(shp)
    lib().or_rgb_to_ycbcr(n, _ptr(rgb), _ptr(y), _ptr(cb), _ptr(cr))
    return y, cb, cr


def ycbcr_to_rgb(y, cb, cr):
    y, cb, cr = _d(y), _d(cb), _d(cr)
    out = np.zeros((3,) + y.shape)
    lib().or_ycbcr_to_rgb(int(y.size), _ptr(y), _ptr(cb), _ptr(cr), _ptr(out))
    return out


def color_sr(P: Params, lr_rgb, view_offsets, omega, n_iters: int):
    """The paper's colour strategy: ADMM on the Y channel of the views, bicubic
    up-sampling of the reference view's Cb and Cr, back to RGB.
    lr_rgb: [n_views][3][h][w].  Returns planar [3][H][W]."""
    lr_rgb = _d(lr_rgb)
    ys = np.stack([rgb_to_ycbcr(v)[0] for v in lr_rgb])
    _, cb, cr = rgb_to_ycbcr(lr_rgb[P.ref_view])
    xY = admm(P, ys, view_offsets, omega, n_iters).x_iters[-1]
    return ycbcr_to_rgb(xY, bicubic(cb, P.scale), bicubic(cr, P.scale))


def psnr(x, gt, crop: int = 8) -> float:
    """PSNR = 10 log10(1/MSE) on x clamped to [0,1], border crop (reading A25)."""
    x = np.clip(np.asarray(x, dtype=np.float64), 0.0, 1.0)
    gt = np.asarray(gt, dtype=np.float64)
    if crop > 0:
        x = x[crop:-crop, crop:-crop]
        gt = gt[crop:-crop, crop:-crop]
    mse = float(np.mean((x - gt) ** 2))
    return math.inf if mse == 0 else 10.0 * math.log10(1.0 / mse)
