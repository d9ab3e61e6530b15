"""Thin ctypes binding of liblfsr.so (include/lfsr.h) — argument marshalling only.

Every step of the ADMM hot path runs in the library's sm_100a kernels; this
module converts numpy arrays / torch tensors to pointers and status codes to
exceptions.  There is no CPU fallback: if liblfsr.so is missing or no B200 is
visible, constructing a :class:`Solver` raises.

Names follow the paper (arXiv 2206.05047): ``lambda1``/``lambda2``,
``theta`` (vartheta), ``cg_max_iters`` K and ``cg_tol`` tau,
``scale`` zeta, ``view_offsets`` theta_k - theta_0.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, fields

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LFSR_LIB") or os.path.join(_HERE, "liblfsr.so")

LFSR_OK, LFSR_ERR_INVALID_ARG, LFSR_ERR_STATE, LFSR_ERR_OOM, LFSR_ERR_CUDA, LFSR_ERR_NCCL, \
    LFSR_ERR_DIVERGED, LFSR_ERR_UNSUPPORTED = range(8)
STATUS_NAMES = ["OK", "INVALID_ARG", "STATE", "OOM", "CUDA", "NCCL", "DIVERGED", "UNSUPPORTED"]
MEM_HOST, MEM_DEVICE = 0, 1
OP_A, OP_AT, OP_S, OP_ST, OP_NORMAL, OP_WEIGHTS, OP_GRAD, OP_BICUBIC = range(8)
OPS = {"A": OP_A, "AT": OP_AT, "S": OP_S, "ST": OP_ST, "NORMAL": OP_NORMAL, "WEIGHTS": OP_WEIGHTS, "GRAD": OP_GRAD,
       "BICUBIC": OP_BICUBIC}

# every symbol include/lfsr.h declares (checked by tests/test_abi.py)
EXPORTS = ("lfsr_create", "lfsr_set_observations", "lfsr_admm_run", "lfsr_admm_enqueue", "lfsr_admm_stats",
           "lfsr_get_hr", "lfsr_get_state", "lfsr_op_apply", "lfsr_launches_per_iter", "lfsr_tile_config", "lfsr_profile",
           "lfsr_profile_read", "lfsr_strip_plan", "lfsr_destroy", "lfsr_last_error", "lfsr_abi_version",
           "lfsr_gd_run", "lfsr_gd_launches_per_iter", "lfsr_rgb_to_ycbcr", "lfsr_ycbcr_to_rgb", "lfsr_solve_batch",
           "lfsr_get_stream", "lfsr_fast_path", "lfsr_normal_path", "lfsr_profile_read_split")


class LFSRError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__("LFSR_ERR_%s: %s" % (name, msg))


class _CParams(ctypes.Structure):
    _fields_ = [("n_views", ctypes.c_int32), ("lr_height", ctypes.c_int32), ("lr_width", ctypes.c_int32),
                ("scale", ctypes.c_int32), ("ref_view", ctypes.c_int32), ("nltv_radius", ctypes.c_int32),
                ("lambda1", ctypes.c_float), ("lambda2", ctypes.c_float), ("lambda_reg", ctypes.c_float),
                ("sigma_s", ctypes.c_float), ("sigma_e", ctypes.c_float), ("sigma_o1", ctypes.c_float),
                ("sigma_o2", ctypes.c_float), ("theta", ctypes.c_float), ("cg_max_iters", ctypes.c_int32),
                ("cg_tol", ctypes.c_float), ("reweight_every_iter", ctypes.c_int32), ("device", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("n_ranks", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p),
                ("stream", ctypes.c_void_p), ("offset_weights", ctypes.POINTER(ctypes.c_float)),
                ("psf", ctypes.POINTER(ctypes.c_float)), ("psf_radius", ctypes.c_int32),
                ("paper_adjoint", ctypes.c_int32)]


class _CStats(ctypes.Structure):
    _fields_ = [("iter", ctypes.c_int32), ("cg_iters", ctypes.c_int32), ("breakdown", ctypes.c_int32),
                ("nonfinite", ctypes.c_int32), ("J", ctypes.c_double), ("data_l1", ctypes.c_double),
                ("data_l2", ctypes.c_double), ("reg_l1", ctypes.c_double), ("primal_res", ctypes.c_double),
                ("cg_pi0", ctypes.c_double), ("cg_pi_last", ctypes.c_double)]


STAT_KEYS = [f[0] for f in _CStats._fields_]


class _CGdParams(ctypes.Structure):
    _fields_ = [("step", ctypes.c_float), ("line_search", ctypes.c_int32), ("max_trials", ctypes.c_int32),
                ("armijo_c", ctypes.c_float)]


class _CGdStats(ctypes.Structure):
    _fields_ = [("iter", ctypes.c_int32), ("ls_evals", ctypes.c_int32), ("ls_failed", ctypes.c_int32),
                ("nonfinite", ctypes.c_int32), ("cu", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("J", ctypes.c_double), ("data_l1", ctypes.c_double), ("data_l2", ctypes.c_double),
                ("reg_l1", ctypes.c_double), ("step", ctypes.c_double), ("grad_sq", ctypes.c_double)]


GD_STAT_KEYS = [f[0] for f in _CGdStats._fields_ if f[0] != "pad"]


class _CStrip(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("rank", "tile_row0", "tile_row1", "lr_row0", "lr_row1", "hr_row0",
                                               "hr_row1", "halo_top", "halo_bottom")]


STRIP_KEYS = [f[0] for f in _CStrip._fields_]

_lib = None


def load_library(path: str = LIB_PATH):
    """Load liblfsr.so; raises if it has not been built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError("liblfsr.so not found at %s — build it with `python -c 'import __graft_entry__ as g; "
                           "g.build()'` (nvcc, sm_100a); there is no CPU fallback" % path)
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    st = ctypes.c_int
    lib.lfsr_create.argtypes = [P(_CParams), P(vp)]
    lib.lfsr_create.restype = st
    lib.lfsr_set_observations.argtypes = [vp, vp, vp, vp, ctypes.c_int, vp, ctypes.c_int]
    lib.lfsr_set_observations.restype = st
    lib.lfsr_admm_run.argtypes = [vp, ctypes.c_int32, P(_CStats)]
    lib.lfsr_admm_run.restype = st
    lib.lfsr_admm_enqueue.argtypes = [vp, ctypes.c_int32]
    lib.lfsr_admm_enqueue.restype = st
    lib.lfsr_admm_stats.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, P(_CStats)]
    lib.lfsr_admm_stats.restype = st
    lib.lfsr_profile.argtypes = [vp, ctypes.c_int32]
    lib.lfsr_profile.restype = st
    lib.lfsr_profile_read.argtypes = [vp, P(ctypes.c_double), P(ctypes.c_int64)]
    lib.lfsr_profile_read.restype = st
    lib.lfsr_profile_read_split.argtypes = [vp, P(ctypes.c_double), P(ctypes.c_int64)]
    lib.lfsr_profile_read_split.restype = st
    lib.lfsr_get_hr.argtypes = [vp, vp, ctypes.c_int]
    lib.lfsr_get_hr.restype = st
    lib.lfsr_get_state.argtypes = [vp, vp, vp, vp, vp, ctypes.c_int]
    lib.lfsr_get_state.restype = st
    lib.lfsr_op_apply.argtypes = [vp, ctypes.c_int, vp, vp, ctypes.c_int]
    lib.lfsr_op_apply.restype = st
    lib.lfsr_launches_per_iter.argtypes = [vp]
    lib.lfsr_launches_per_iter.restype = ctypes.c_int32
    i32p = ctypes.POINTER(ctypes.c_int32)
    lib.lfsr_tile_config.argtypes = [vp, i32p, i32p, i32p, i32p]
    lib.lfsr_tile_config.restype = st
    lib.lfsr_fast_path.argtypes = [vp, i32p, i32p]
    lib.lfsr_fast_path.restype = st
    lib.lfsr_normal_path.argtypes = [vp, i32p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_double)]
    lib.lfsr_normal_path.restype = st
    lib.lfsr_destroy.argtypes = [vp]
    lib.lfsr_destroy.restype = None
    lib.lfsr_last_error.argtypes = [vp]
    lib.lfsr_last_error.restype = ctypes.c_char_p
    lib.lfsr_strip_plan.argtypes = [P(_CParams), ctypes.c_int32, P(_CStrip)]
    lib.lfsr_strip_plan.restype = st
    lib.lfsr_gd_run.argtypes = [vp, P(_CGdParams), ctypes.c_int32, P(_CGdStats)]
    lib.lfsr_gd_run.restype = st
    lib.lfsr_gd_launches_per_iter.argtypes = [vp]
    lib.lfsr_gd_launches_per_iter.restype = ctypes.c_int32
    lib.lfsr_solve_batch.argtypes = [vp, ctypes.c_int32, P(vp), P(vp), P(vp), ctypes.c_int32, P(vp)]
    lib.lfsr_solve_batch.restype = st
    lib.lfsr_rgb_to_ycbcr.argtypes = [vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.lfsr_rgb_to_ycbcr.restype = st
    lib.lfsr_ycbcr_to_rgb.argtypes = [vp, vp, vp, vp, ctypes.c_size_t, vp]
    lib.lfsr_ycbcr_to_rgb.restype = st
    lib.lfsr_get_stream.argtypes = [vp, P(vp)]
    lib.lfsr_get_stream.restype = st
    lib.lfsr_abi_version.argtypes = []
    lib.lfsr_abi_version.restype = ctypes.c_int32
    _lib = lib
    return lib


@dataclass
class Params:
    """lfsr_params (include/lfsr.h).  Defaults: reading A20, K=5, 5x5 window."""
    n_views: int
    lr_height: int
    lr_width: int
    scale: int = 2
    ref_view: int = 0
    nltv_radius: int = 2
    lambda1: float = 1.0
    lambda2: float = 0.1
    lambda_reg: float = 0.5
    sigma_s: float = 3.0
    sigma_e: float = 0.2
    sigma_o1: float = 0.5
    sigma_o2: float = 0.2
    theta: float = 4.0
    cg_max_iters: int = 5
    cg_tol: float = 0.0
    reweight_every_iter: int = 1
    device: int = 0
    n_ranks: int = 1          # HR row strips
    rank: int = 0             # this process's strip (NCCL mode) or -1: all strips in this ctx
    nccl_unique_id: bytes | None = None
    offset_weights: object = None   # s_d floats (e.g. BTV alpha^(|dx|+|dy|)) replacing exp(-|d|^2/sigma_s)
    psf: object = None              # user blur kernel [(2r+1)][(2r+1)] replacing the Gaussian (A36)
    paper_adjoint: int = 0          # 1: the paper's backward-warp adjoint W_k^* with omega_0 (A37)

    @property
    def H(self):
        return self.lr_height * self.scale

    @property
    def W(self):
        return self.lr_width * self.scale

    @property
    def s_d(self):
        return (2 * self.nltv_radius + 1) ** 2 - 1

    def to_c(self, stream=None) -> _CParams:
        c = _CParams()
        for f in fields(self):
            if f.name not in ("nccl_unique_id", "offset_weights", "psf"):
                setattr(c, f.name, getattr(self, f.name))
        self._ow = None
        if self.offset_weights is not None:
            ow = [float(v) for v in self.offset_weights]
            if len(ow) != self.s_d:
                raise LFSRError(1, "offset_weights must have s_d = %d entries" % self.s_d)
            self._ow = (ctypes.c_float * len(ow))(*ow)   # copied by lfsr_create
            c.offset_weights = ctypes.cast(self._ow, ctypes.POINTER(ctypes.c_float))
        self._psf = None
        if self.psf is not None:
            k = np.ascontiguousarray(self.psf, dtype=np.float32)
            if k.ndim != 2 or k.shape[0] != k.shape[1] or k.shape[0] % 2 != 1:
                raise LFSRError(1, "psf must be a square kernel of odd size")
            self._psf = k   # copied by lfsr_create
            c.psf = k.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
            c.psf_radius = (k.shape[0] - 1) // 2
        self._uid = None
        if self.nccl_unique_id is not None:
            self._uid = ctypes.create_string_buffer(bytes(self.nccl_unique_id), 128)
            c.nccl_unique_id = ctypes.cast(self._uid, ctypes.c_void_p)
        c.stream = stream
        return c


def _is_torch(a):
    return type(a).__module__.startswith("torch")


class Solver:
    """One lfsr_ctx.  Inputs may be numpy arrays (host) or torch tensors (host or cuda)."""

    def __init__(self, params: Params, stream: int | None = None):
        self.lib = load_library()
        self.params = params
        cp = params.to_c(stream)
        h = ctypes.c_void_p()
        s = self.lib.lfsr_create(ctypes.byref(cp), ctypes.byref(h))
        if s != LFSR_OK:
            raise LFSRError(s, self.lib.lfsr_last_error(None).decode())
        self._h = h
        self._keep = []
        self._user_stream = stream is not None
        self._ext = None   # torch view of the ctx-owned stream (device-tensor calls, see _dev_call)

    # -- helpers ------------------------------------------------------------
    def _check(self, s):
        if s != LFSR_OK:
            raise LFSRError(s, self.lib.lfsr_last_error(self._h).decode())

    @staticmethod
    def _ptr_in(a):
        """(pointer, mem, keepalive) of a float32 contiguous input."""
        if a is None:
            return None, None, None
        if _is_torch(a):
            import torch
            t = a.detach()
            if t.dtype != torch.float32:
                t = t.float()
            t = t.contiguous()
            return t.data_ptr(), (MEM_DEVICE if t.is_cuda else MEM_HOST), t
        arr = np.ascontiguousarray(a, dtype=np.float32)
        return arr.ctypes.data, MEM_HOST, arr

    def _dev_call(self, fn, tensors):
        """Run fn() (a C call reading / writing the device tensors `tensors`) ordered against torch's
        current stream.  With a caller-supplied stream the caller orders its own work (that stream
        is the ctx stream).  With the ctx-owned stream: the ctx stream waits for torch's current
        stream before the call and torch's current stream waits for the ctx stream after it.  The
        library keeps no caller pointer past the work that call enqueues, so that wait also covers
        the tensors' memory (marshalling temporaries included): torch's caching allocator reuses a
        freed block only in the order of the stream it was allocated on, which is now behind the
        ctx's work.  (No record_stream: the ctx stream dies with the ctx, and the allocator would
        later record an event on it.)"""
        if self._user_stream or not tensors:
            return fn()
        import torch
        dev = tensors[0].device
        if self._ext is None:
            sp = ctypes.c_void_p()
            self._check(self.lib.lfsr_get_stream(self._h, ctypes.byref(sp)))
            self._ext = torch.cuda.ExternalStream(sp.value, device=dev)
        cur = torch.cuda.current_stream(dev)
        self._ext.wait_stream(cur)
        try:
            return fn()
        finally:
            cur.wait_stream(self._ext)

    def close(self):
        if getattr(self, "_h", None):
            self.lib.lfsr_destroy(self._h)
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

    # -- API ----------------------------------------------------------------
    def set_observations(self, lr_views, view_offsets, disparity, x0=None):
        ptrs = [self._ptr_in(a) for a in (lr_views, view_offsets, disparity, x0)]
        mems = {p[1] for p in ptrs if p[1] is not None}
        if len(mems) != 1:
            raise ValueError("all inputs of one call must be either host or device memory")
        mem = mems.pop()
        # [H][W]: one shared map (LFSR_DISP_SHARED); [n_views][H][W]: omega_k per view (LFSR_DISP_PER_VIEW, A34)
        disp_mode = 1 if len(tuple(disparity.shape)) == 3 else 0
        call = lambda: self.lib.lfsr_set_observations(self._h, ptrs[0][0], ptrs[1][0], ptrs[2][0], disp_mode,
                                                      ptrs[3][0], mem)
        dev = [p[2] for p in ptrs if p[2] is not None] if mem == MEM_DEVICE else []
        self._check(self._dev_call(call, dev))

    def admm_run(self, n_iters: int, want_stats: bool = True):
        st = (_CStats * max(int(n_iters), 1))() if want_stats else None
        s = self.lib.lfsr_admm_run(self._h, int(n_iters), st)
        stats = [{k: getattr(st[i], k) for k in STAT_KEYS} for i in range(n_iters)] if want_stats else None
        if s == LFSR_ERR_DIVERGED:
            err = LFSRError(s, self.lib.lfsr_last_error(self._h).decode())
            err.stats = stats
            raise err
        self._check(s)
        return stats

    def admm_enqueue(self, n_iters: int):
        """Stream-ordered launch of n_iters iterations; no host sync (see lfsr_admm_stats)."""
        self._check(self.lib.lfsr_admm_enqueue(self._h, int(n_iters)))

    def admm_stats(self, first_iter: int, n_iters: int):
        st = (_CStats * max(int(n_iters), 1))()
        s = self.lib.lfsr_admm_stats(self._h, int(first_iter), int(n_iters), st)
        stats = [{k: getattr(st[i], k) for k in STAT_KEYS} for i in range(n_iters)]
        if s == LFSR_ERR_DIVERGED:
            err = LFSRError(s, self.lib.lfsr_last_error(self._h).decode())
            err.stats = stats
            raise err
        self._check(s)
        return stats

    def gd_run(self, n_iters: int, step: float, line_search: bool = False, max_trials: int = 30,
               armijo_c: float = 1e-4, want_stats: bool = True):
        """gd / gd-ls iterations (lfsr_gd_run, readings A30-A33)."""
        gp = _CGdParams(float(step), 1 if line_search else 0, int(max_trials), float(armijo_c))
        st = (_CGdStats * max(int(n_iters), 1))() if want_stats else None
        s = self.lib.lfsr_gd_run(self._h, ctypes.byref(gp), int(n_iters), st)
        stats = [{k: getattr(st[i], k) for k in GD_STAT_KEYS} for i in range(n_iters)] if want_stats else None
        if s == LFSR_ERR_DIVERGED:
            err = LFSRError(s, self.lib.lfsr_last_error(self._h).decode())
            err.stats = stats
            raise err
        self._check(s)
        return stats

    def solve_batch(self, fields, n_iters: int, outs=None):
        """lfsr_solve_batch: fields = [(lr_views, view_offsets, disparity), ...] host arrays (page-locked
        torch tensors for overlapped copies, or numpy); returns the HR estimates (into `outs` if given)."""
        n = len(fields)
        keep = []
        arrs = [[], [], []]
        for f in fields:
            for j, a in enumerate(f):
                ptr, mem, k = self._ptr_in(a)
                if mem != MEM_HOST:
                    raise ValueError("lfsr_solve_batch takes host arrays")
                keep.append(k)
                arrs[j].append(ptr)
        p = self.params
        if outs is None:
            outs = [np.empty((p.H, p.W), np.float32) for _ in range(n)]
        optr = [o.data_ptr() if _is_torch(o) else o.ctypes.data for o in outs]
        A = lambda v: (ctypes.c_void_p * n)(*v)
        self._check(self.lib.lfsr_solve_batch(self._h, n, A(arrs[0]), A(arrs[1]), A(arrs[2]), int(n_iters),
                                              A(optr)))
        return outs

    def gd_launches_per_iter(self) -> int:
        return int(self.lib.lfsr_gd_launches_per_iter(self._h))

    def profile(self, enable: bool = True):
        self._check(self.lib.lfsr_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        """(ms[3], launches[3]) accumulated for (wz tile, normal tile, cg update) kernels."""
        ms = (ctypes.c_double * 3)()
        n = (ctypes.c_int64 * 3)()
        self._check(self.lib.lfsr_profile_read(self._h, ms, n))
        return list(ms), list(n)


    def profile_read_split(self):
        """lfsr_profile_read_split: (stencil-kernel ms, irregular-row ms, passes) of the assembled operator."""
        ms = (ctypes.c_double * 2)()
        n = ctypes.c_int64()
        self._check(self.lib.lfsr_profile_read_split(self._h, ms, ctypes.byref(n)))
        return list(ms), int(n.value)
    def get_hr(self, out=None):
        """Returns x [H][W]: into `out` (torch tensor, host or device) or a new numpy array."""
        H, W = self.params.H, self.params.W
        if out is None:
            out = np.empty((H, W), dtype=np.float32)
            self._check(self.lib.lfsr_get_hr(self._h, out.ctypes.data, MEM_HOST))
            return out
        mem = MEM_DEVICE if (_is_torch(out) and out.is_cuda) else MEM_HOST
        ptr = out.data_ptr() if _is_torch(out) else out.ctypes.data
        self._check(self._dev_call(lambda: self.lib.lfsr_get_hr(self._h, ptr, mem), [out] if mem == MEM_DEVICE else []))
        return out

    def get_state(self):
        p = self.params
        wA = np.empty((p.n_views, p.lr_height, p.lr_width), np.float32)
        wS = np.empty((p.s_d, p.H, p.W), np.float32)
        x = np.empty((p.H, p.W), np.float32)
        m = np.empty((p.H, p.W), np.float32)
        self._check(self.lib.lfsr_get_state(self._h, wA.ctypes.data, wS.ctypes.data, x.ctypes.data,
                                            m.ctypes.data, MEM_HOST))
        return {"wA": wA, "wS": wS, "x": x, "m": m}

    def op(self, name: str, inp):
        p = self.params
        op = OPS[name]
        out_shape = {OP_A: (p.n_views, p.lr_height, p.lr_width), OP_AT: (p.H, p.W),
                     OP_S: (p.s_d, p.H, p.W), OP_ST: (p.H, p.W), OP_NORMAL: (p.H, p.W),
                     OP_WEIGHTS: (p.H, p.W), OP_GRAD: (p.H, p.W), OP_BICUBIC: (p.H, p.W)}[op]
        ptr, mem, keep = self._ptr_in(inp)
        if mem == MEM_DEVICE:
            import torch
            out = torch.empty(out_shape, dtype=torch.float32, device=keep.device)
            self._check(self._dev_call(lambda: self.lib.lfsr_op_apply(self._h, op, ptr, out.data_ptr(), MEM_DEVICE),
                                       [keep, out]))
            return out
        out = np.empty(out_shape, np.float32)
        self._check(self.lib.lfsr_op_apply(self._h, op, ptr, out.ctypes.data, MEM_HOST))
        return out

    @property
    def launches_per_iter(self) -> int:
        return int(self.lib.lfsr_launches_per_iter(self._h))

    @property
    def fast_path(self) -> dict:
        """lfsr_fast_path: whether the MISR stencil path runs, with its rectangles."""
        act = ctypes.c_int32()
        rect = (ctypes.c_int32 * 8)()
        self._check(self.lib.lfsr_fast_path(self._h, ctypes.byref(act), rect))
        return {"misr": bool(act.value), "zs": tuple(rect[:4]), "owned": tuple(rect[4:])}

    @property
    def normal_path(self) -> dict:
        """lfsr_normal_path: which implementation applies the CG operator (0 tile kernel, 1 MISR,
        2 assembled), the irregular / total row counts and the assembly time."""
        path, nirr, ntot, ms = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        self._check(self.lib.lfsr_normal_path(self._h, ctypes.byref(path), ctypes.byref(nirr), ctypes.byref(ntot),
                                              ctypes.byref(ms)))
        return {"path": int(path.value), "name": ("tile", "misr", "assembled")[path.value],
                "irregular_rows": int(nirr.value), "total_rows": int(ntot.value), "setup_ms": float(ms.value)}

    @property
    def tile_config(self) -> dict:
        """lfsr_tile_config: the fused kernel's tiling (tile rows, view groups, warps per CTA)."""
        b, g, w, wn = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        self._check(self.lib.lfsr_tile_config(self._h, ctypes.byref(b), ctypes.byref(g), ctypes.byref(w),
                                              ctypes.byref(wn)))
        return {"tile_rows": b.value, "view_groups": g.value, "warps_per_cta": w.value, "cg_warps_per_cta": wn.value}


def strip_plan(params: Params, max_shift_rows: int):
    """Row-strip plan of the multi-GPU decomposition (lfsr_strip_plan; no device needed)."""
    lib = load_library()
    out = (_CStrip * params.n_ranks)()
    cp = params.to_c()
    s = lib.lfsr_strip_plan(ctypes.byref(cp), int(max_shift_rows), out)
    if s != LFSR_OK:
        raise LFSRError(s, lib.lfsr_last_error(None).decode())
    return [{k: getattr(out[i], k) for k in STRIP_KEYS} for i in range(params.n_ranks)]


def params_for(lf_meta_or_cfg, defaults=None, **over) -> Params:
    """Params for an lfsr_synth config (shape fields) + SolverDefaults (numbers)."""
    cfg = lf_meta_or_cfg
    d = {} if defaults is None else {k: getattr(defaults, k) for k in
                                      ("lambda1", "lambda2", "lambda_reg", "sigma_s", "sigma_e", "sigma_o1",
                                       "sigma_o2", "theta", "cg_max_iters", "cg_tol")}
    if defaults is not None:
        d["nltv_radius"] = defaults.radius
        if getattr(defaults, "offset_weights", None) is not None:
            d["offset_weights"] = list(defaults.offset_weights)
    d.update(n_views=cfg.n_views, lr_height=cfg.lr_h, lr_width=cfg.lr_w, scale=cfg.scale, ref_view=cfg.ref_view)
    d.update(over)
    return Params(**d)


def psnr(x, gt, crop: int = 8) -> float:
    """PSNR = 10 log10(1/MSE) of clip(x, 0, 1) vs gt on an interior crop (reading A25)."""
    x = np.clip(np.asarray(x, dtype=np.float64), 0.0, 1.0)
    gt = np.asarray(gt, dtype=np.float64)
    if crop > 0:
        x, gt = x[crop:-crop, crop:-crop], gt[crop:-crop, crop:-crop]
    mse = float(np.mean((x - gt) ** 2))
    return math.inf if mse == 0 else 10.0 * math.log10(1.0 / mse)


def _color_check(s, what):
    if s != LFSR_OK:
        raise LFSRError(s, what)


def rgb_to_ycbcr(rgb, stream: int | None = None):
    """Planar [3][...] fp32 CUDA tensor -> (Y, Cb, Cr) CUDA tensors (lfsr_rgb_to_ycbcr, BT.601, A35)."""
    import torch
    assert rgb.is_cuda and rgb.dtype == torch.float32 and rgb.is_contiguous() and rgb.shape[0] == 3
    y, cb, cr = (torch.empty(rgb.shape[1:], dtype=torch.float32, device=rgb.device) for _ in range(3))
    st = stream if stream is not None else torch.cuda.current_stream(rgb.device).cuda_stream
    _color_check(load_library().lfsr_rgb_to_ycbcr(rgb.data_ptr(), y.data_ptr(), cb.data_ptr(), cr.data_ptr(),
                                                   y.numel(), st), "lfsr_rgb_to_ycbcr")
    return y, cb, cr


def ycbcr_to_rgb(y, cb, cr, stream: int | None = None):
    import torch
    for t in (y, cb, cr):
        assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.shape == y.shape
    rgb = torch.empty((3,) + tuple(y.shape), dtype=torch.float32, device=y.device)
    st = stream if stream is not None else torch.cuda.current_stream(y.device).cuda_stream
    _color_check(load_library().lfsr_ycbcr_to_rgb(y.data_ptr(), cb.data_ptr(), cr.data_ptr(), rgb.data_ptr(),
                                                   y.numel(), st), "lfsr_ycbcr_to_rgb")
    return rgb


def color_super_resolve(params: Params, lr_rgb, view_offsets, disparity, n_iters: int, x0=None):
    """The paper's colour strategy: ADMM on the Y channel of every view, the
    bicubic up-sampling (LFSR_OP_BICUBIC) of the reference view's Cb and Cr, back to
    RGB -- every step in liblfsr kernels.  lr_rgb: [n_views][3][h][w] fp32 CUDA tensor;
    view_offsets / disparity as for Solver.set_observations (CUDA tensors).  Returns
    ([3][H][W] CUDA tensor, ADMM stats)."""
    import torch
    caller = torch.cuda.current_stream(lr_rgb.device)
    ts = torch.cuda.Stream(device=lr_rgb.device)   # one real stream for every call below (the legacy
    ts.wait_stream(caller)                          # default stream's NULL handle would give the ctx its own)
    with torch.cuda.stream(ts):
        out = _color_sr_on(params, lr_rgb, view_offsets, disparity, n_iters, x0, ts.cuda_stream)
    caller.wait_stream(ts)
    return out


def _color_sr_on(params, lr_rgb, view_offsets, disparity, n_iters, x0, stream):
    import torch
    nv = lr_rgb.shape[0]
    assert lr_rgb.is_cuda and lr_rgb.dtype == torch.float32 and lr_rgb.is_contiguous() and lr_rgb.shape[1] == 3
    hw = tuple(lr_rgb.shape[2:])
    ys = torch.empty((nv,) + hw, dtype=torch.float32, device=lr_rgb.device)
    cbs = torch.empty((2, nv) + hw, dtype=torch.float32, device=lr_rgb.device)   # Cb, Cr of every view
    n = ys[0].numel()
    lib = load_library()
    for k in range(nv):   # Y straight into the view stack (no copies)
        _color_check(lib.lfsr_rgb_to_ycbcr(lr_rgb[k].data_ptr(), ys[k].data_ptr(), cbs[0, k].data_ptr(),
                                           cbs[1, k].data_ptr(), n, stream), "lfsr_rgb_to_ycbcr")
    chroma = (cbs[0, params.ref_view], cbs[1, params.ref_view])
    with Solver(params, stream=stream) as s:
        s.set_observations(ys, view_offsets, disparity, x0)
        stats = s.admm_run(n_iters)
        xY = torch.empty((params.H, params.W), dtype=torch.float32, device=lr_rgb.device)
        s.get_hr(xY)
        cb_hr, cr_hr = s.op("BICUBIC", chroma[0]), s.op("BICUBIC", chroma[1])
    return ycbcr_to_rgb(xY, cb_hr, cr_hr, stream), stats
