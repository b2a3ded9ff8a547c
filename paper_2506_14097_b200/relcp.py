"""Thin Python binding of librelcp.so (include/relcp.h).

Argument marshalling only: every step of the ReLCP hot path runs in the CUDA
kernels behind the C ABI.  torch is used for device memory and the stream.
There is no CPU fallback: `Context` raises if the library or a CUDA device is
missing.  Names follow the ABI (relcp_generate_contacts -> generate_contacts).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import build as _build

INERTIAL = 0
OVERDAMPED = 1
MAX_REC = 64

OK = 0
E_ARG, E_CUDA, E_CAPACITY, E_DEGENERATE, E_NAN, E_STATE = -1, -2, -3, -4, -5, -6
W_MAX_ITER, W_RECURSION_CAP, W_SNSD_NONCONV = 1, 2, 3

EXPORTS = ["relcp_default_params", "relcp_create", "relcp_destroy", "relcp_last_error", "relcp_set_params",
           "relcp_generate_contacts", "relcp_prepare_operator", "relcp_delassus_apply", "relcp_wrench",
           "relcp_solve_lcp", "relcp_check_and_augment", "relcp_step", "relcp_get_pairs", "relcp_snsd_pairs",
           "relcp_get_stats", "relcp_reset_stats", "relcp_set_timing", "relcp_load_constraints",
           "relcp_dd_plan_host", "relcp_dd_nccl_unique_id", "relcp_dd_create", "relcp_dd_destroy",
           "relcp_dd_last_error", "relcp_dd_load", "relcp_dd_info_get", "relcp_dd_delassus_apply", "relcp_dd_get_u",
           "relcp_dd_solve_lcp", "relcp_dd_step"]

P = ctypes.c_void_p
i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double


class Params(ctypes.Structure):
    _fields_ = [("dynamics", i32), ("max_recursions", i32), ("dt", f64), ("eps_ncp", f64), ("cutoff", f64),
                ("lcp_tol", f64), ("lcp_max_iter", i64), ("check_every", i32), ("power_iters", i32),
                ("box", f64 * 3), ("xi", f64), ("n_dirs", i32), ("solver", i32), ("reorder", i32),
                ("layout", i32), ("cluster", i32), ("snsd_cert", i32),
                ("k6_pipe", i32), ("k6_bpw", i32)]


SOLVER_BB, SOLVER_APGD, SOLVER_APGD_FUSED = 0, 1, 2
REORDER_OFF, REORDER_AUTO, REORDER_ON = 0, 1, 2
LAYOUT_CSR, LAYOUT_JDS, LAYOUT_AUTO = 0, 1, 2


class Bodies(ctypes.Structure):
    _fields_ = [("n", i64), ("pos", P), ("quat", P), ("axes", P), ("vel", P), ("inv_mass", P),
                ("inv_inertia", P), ("kinematic", P), ("shape", P)]


class Constraints(ctypes.Structure):
    _fields_ = [("capacity", i64), ("count", i64), ("ia", P), ("ib", P), ("gen", P), ("n", P), ("ta", P),
                ("tb", P), ("phi", P), ("q", P), ("lam", P), ("g", P)]


class SolveReport(ctypes.Structure):
    _fields_ = [("iterations", i64), ("residual", f64), ("converged", i32), ("pad", i32), ("objective", f64),
                ("L", f64)]


class Stats(ctypes.Structure):
    _fields_ = [("launches", i64), ("lcp_iterations", i64), ("iter_timed", i64), ("scatter_ms", f64),
                ("gather_ms", f64), ("split_timed", i64), ("iter_ms", f64), ("n_guard", i64),
                ("jds_solves", i64), ("op_layout", i32), ("pad", i32), ("cluster_solves", i64),
                ("snsd_multistart", i64)]


class StepReport(ctypes.Structure):
    _fields_ = [("recursions", i32), ("status", i32), ("n_pairs", i64), ("margin", f64), ("max_overlap", f64),
                ("n_c", i64 * MAX_REC), ("lcp_iters", i64 * MAX_REC), ("residual", f64 * MAX_REC),
                ("f_n", f64 * MAX_REC), ("ms_generate", f64), ("ms_solve", f64), ("ms_check", f64),
                ("snsd_nonconv", i64), ("n_guard", i64)]

    def as_dict(self):
        r = self.recursions
        return dict(recursions=r, status=self.status, n_pairs=self.n_pairs, margin=self.margin,
                    max_overlap=self.max_overlap, n_c=list(self.n_c[:r + 1]),
                    iterations=list(self.lcp_iters[:r + 1]), residuals=list(self.residual[:r + 1]),
                    f=list(self.f_n[:r + 1]), ms_generate=self.ms_generate, ms_solve=self.ms_solve,
                    ms_check=self.ms_check, snsd_nonconv=self.snsd_nonconv, n_guard=self.n_guard)


class DDInfo(ctypes.Structure):
    _fields_ = [("n_own", i64), ("n_ghost", i64), ("row_lo", i64), ("row_hi", i64), ("n_recv", i64),
                ("n_boundary", i64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load librelcp.so (building it if absent); raises if it cannot."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("RELCP_LIB", _build.LIB)  # tuning variants (tools/sweep)
    if not os.path.exists(path):
        if not build_if_missing:
            raise RuntimeError(f"librelcp.so missing at {path}; run paper_2506_14097_b200.build")
        _build.build()
    L = ctypes.CDLL(path)
    L.relcp_default_params.argtypes = [ctypes.POINTER(Params)]
    L.relcp_default_params.restype = None
    L.relcp_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(Params), P]
    L.relcp_destroy.argtypes = [P]
    L.relcp_last_error.argtypes = [P]
    L.relcp_last_error.restype = ctypes.c_char_p
    L.relcp_set_params.argtypes = [P, ctypes.POINTER(Params)]
    L.relcp_generate_contacts.argtypes = [P, ctypes.POINTER(Bodies), ctypes.POINTER(Constraints),
                                          ctypes.POINTER(i64)]
    L.relcp_prepare_operator.argtypes = [P, ctypes.POINTER(Bodies), ctypes.POINTER(Constraints)]
    L.relcp_delassus_apply.argtypes = [P, ctypes.POINTER(Bodies), ctypes.POINTER(Constraints), P, P, f64]
    L.relcp_wrench.argtypes = [P, ctypes.POINTER(Bodies), ctypes.POINTER(Constraints), P, P, P]
    L.relcp_solve_lcp.argtypes = [P, ctypes.POINTER(Bodies), ctypes.POINTER(Constraints),
                                  ctypes.POINTER(SolveReport)]
    L.relcp_check_and_augment.argtypes = [P, ctypes.POINTER(Bodies), ctypes.POINTER(Constraints), i32,
                                          ctypes.POINTER(i64), ctypes.POINTER(f64)]
    L.relcp_step.argtypes = [P, ctypes.POINTER(Bodies), P, ctypes.POINTER(Constraints), ctypes.POINTER(StepReport)]
    L.relcp_get_pairs.argtypes = [P, P, P, i64, ctypes.POINTER(i64)]
    L.relcp_snsd_pairs.argtypes = [P, ctypes.POINTER(Bodies), i64, P, P, P, P, P, P, P]
    L.relcp_get_stats.argtypes = [P, ctypes.POINTER(Stats)]
    L.relcp_reset_stats.argtypes = [P]
    L.relcp_set_timing.argtypes = [P, i32]
    L.relcp_load_constraints.argtypes = [P, ctypes.POINTER(Bodies), ctypes.POINTER(Constraints), i64, P, P, P, P,
                                         P, P]
    L.relcp_dd_plan_host.argtypes = [i32, P, i64, P, P, i32, ctypes.POINTER(DDInfo), P, P, P, P]
    L.relcp_dd_nccl_unique_id.argtypes = [P]
    L.relcp_dd_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(Params), P, i32, P, i32, P]
    L.relcp_dd_destroy.argtypes = [P]
    L.relcp_dd_last_error.argtypes = [P]
    L.relcp_dd_last_error.restype = ctypes.c_char_p
    L.relcp_dd_load.argtypes = [P, ctypes.POINTER(Bodies), ctypes.POINTER(Constraints)]
    L.relcp_dd_info_get.argtypes = [P, i32, ctypes.POINTER(DDInfo)]
    L.relcp_dd_delassus_apply.argtypes = [P, P, P, f64]
    L.relcp_dd_get_u.argtypes = [P, P]
    L.relcp_dd_solve_lcp.argtypes = [P, ctypes.POINTER(Constraints), ctypes.POINTER(SolveReport)]
    L.relcp_dd_step.argtypes = [P, ctypes.POINTER(Bodies), P, ctypes.POINTER(Constraints), ctypes.POINTER(StepReport)]
    for name in EXPORTS:
        if name not in ("relcp_default_params", "relcp_last_error", "relcp_dd_last_error"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


class RelcpError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"relcp error {code}: {msg}")
        self.code = code


def default_params(**kw) -> Params:
    p = Params()
    load().relcp_default_params(ctypes.byref(p))
    for k, v in kw.items():
        if k == "box":
            for i in range(3):
                p.box[i] = float(v[i])
        else:
            setattr(p, k, v)
    return p


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _dptr(t, dtype, numel: int, name: str, optional: bool = False):
    """Device pointer of a tensor handed to the library: CUDA, `dtype`,
    contiguous, at least `numel` elements.  Anything else raises ValueError
    here (a host, strided or short buffer would fault inside a kernel)."""
    if t is None:
        if optional:
            return None
        raise ValueError(f"{name}: required")
    ok = (torch.is_tensor(t) and t.is_cuda and t.dtype == dtype and t.is_contiguous()
          and t.numel() >= numel)
    if not ok:
        desc = (f"{t.dtype} on {t.device}, contiguous={t.is_contiguous()}, numel={t.numel()}"
                if torch.is_tensor(t) else type(t).__name__)
        raise ValueError(f"{name}: need a contiguous CUDA {dtype} tensor with >= {numel} elements, got {desc}")
    return ctypes.c_void_p(t.data_ptr())


class BodyState:
    """Device-resident SoA body arrays (fp64; kinematic int32)."""

    def __init__(self, pos, quat, axes, vel=None, inv_mass=None, inv_inertia=None, kinematic=None,
                 device="cuda", shape=None):
        def t(a, dt=torch.float64):
            if a is None:
                return None
            return torch.as_tensor(np.ascontiguousarray(a) if isinstance(a, np.ndarray) else a, dtype=dt,
                                   device=device).contiguous()
        self.pos, self.quat, self.axes = t(pos), t(quat), t(axes)
        self.vel, self.inv_mass, self.inv_inertia = t(vel), t(inv_mass), t(inv_inertia)
        self.kinematic = t(kinematic, torch.int32)
        self.shape = t(shape, torch.int32)
        self.n = self.pos.shape[0]

    @classmethod
    def from_scene(cls, sc, device="cuda"):
        return cls(sc["pos"], sc["quat"], sc["axes"], sc.get("vel"), sc.get("inv_mass"), sc.get("inv_inertia"),
                   sc.get("kinematic"), device=device, shape=sc.get("shape"))

    def view(self) -> Bodies:
        n, f, i = self.n, torch.float64, torch.int32
        return Bodies(n, _dptr(self.pos, f, 3 * n, "pos"), _dptr(self.quat, f, 4 * n, "quat"),
                      _dptr(self.axes, f, 3 * n, "axes"), _dptr(self.vel, f, 6 * n, "vel", True),
                      _dptr(self.inv_mass, f, n, "inv_mass", True), _dptr(self.inv_inertia, f, 3 * n, "inv_inertia", True),
                      _dptr(self.kinematic, i, n, "kinematic", True), _dptr(self.shape, i, n, "shape", True))


class ConstraintStore:
    """Caller-owned SoA constraint store (include/relcp.h relcp_constraints)."""

    def __init__(self, capacity: int, device="cuda"):
        cap = max(int(capacity), 1)
        self.capacity = cap
        self.count = 0
        z32 = lambda: torch.zeros(cap, dtype=torch.int32, device=device)
        z64 = lambda *s: torch.zeros(*s, dtype=torch.float64, device=device)
        self.ia, self.ib, self.gen = z32(), z32(), z32()
        self.n, self.ta, self.tb = z64(3, cap), z64(3, cap), z64(3, cap)
        self.phi, self.q, self.lam, self.g = z64(cap), z64(cap), z64(cap), z64(cap)
        self._view = None

    @classmethod
    def from_rows(cls, ia, ib, nrm, ta, tb, q=None, lam=None, capacity=None, device="cuda"):
        m = len(ia)
        cs = cls(capacity or m, device)
        cs.count = m
        if m:
            cs.ia[:m] = torch.as_tensor(np.asarray(ia), dtype=torch.int32)
            cs.ib[:m] = torch.as_tensor(np.asarray(ib), dtype=torch.int32)
            cs.n[:, :m] = torch.as_tensor(np.asarray(nrm, dtype=np.float64).T)
            cs.ta[:, :m] = torch.as_tensor(np.asarray(ta, dtype=np.float64).T)
            cs.tb[:, :m] = torch.as_tensor(np.asarray(tb, dtype=np.float64).T)
            if q is not None:
                cs.q[:m] = torch.as_tensor(np.asarray(q, dtype=np.float64))
            if lam is not None:
                cs.lam[:m] = torch.as_tensor(np.asarray(lam, dtype=np.float64))
        return cs

    def view(self) -> Constraints:
        c, f, i = self.capacity, torch.float64, torch.int32
        v = Constraints(c, self.count, _dptr(self.ia, i, c, "ia"), _dptr(self.ib, i, c, "ib"),
                        _dptr(self.gen, i, c, "gen"), _dptr(self.n, f, 3 * c, "n"), _dptr(self.ta, f, 3 * c, "ta"),
                        _dptr(self.tb, f, 3 * c, "tb"), _dptr(self.phi, f, c, "phi"), _dptr(self.q, f, c, "q"),
                        _dptr(self.lam, f, c, "lambda"), _dptr(self.g, f, c, "g"))
        self._view = v
        return v

    def sync_from(self, v: Constraints):
        self.count = int(v.count)

    def to_numpy(self):
        m = self.count
        c = lambda t: t[..., :m].cpu().numpy()
        return dict(ia=c(self.ia), ib=c(self.ib), gen=c(self.gen), n=c(self.n).T.copy(), ta=c(self.ta).T.copy(),
                    tb=c(self.tb).T.copy(), phi=c(self.phi), q=c(self.q), lam=c(self.lam), g=c(self.g))


class Context:
    """relcp_ctx bound to a torch CUDA stream."""

    def __init__(self, params: Params | None = None, stream: torch.cuda.Stream | None = None, **kw):
        if not torch.cuda.is_available():
            raise RuntimeError("relcp: no CUDA device (there is no CPU fallback)")
        self.L = load()
        self.params = params if params is not None else default_params(**kw)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        h = P()
        rc = self.L.relcp_create(ctypes.byref(h), ctypes.byref(self.params), P(self.stream.cuda_stream))
        if rc != OK:
            raise RelcpError(rc, "relcp_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.relcp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, allow_warn=True):
        if rc < 0 or (rc > 0 and not allow_warn):
            raise RelcpError(rc, self.L.relcp_last_error(self.h).decode(errors="replace"))
        return rc

    def set_params(self, **kw):
        for k, v in kw.items():
            if k == "box":
                for i in range(3):
                    self.params.box[i] = float(v[i])
            else:
                setattr(self.params, k, v)
        self._check(self.L.relcp_set_params(self.h, ctypes.byref(self.params)))

    # ---- ABI calls
    def generate_contacts(self, bodies: BodyState, cs: ConstraintStore):
        bv, cv = bodies.view(), cs.view()
        n = i64()
        rc = self.L.relcp_generate_contacts(self.h, ctypes.byref(bv), ctypes.byref(cv), ctypes.byref(n))
        cs.sync_from(cv)
        self._check(rc)
        return int(n.value), rc

    def load_constraints(self, bodies: BodyState, cs: ConstraintStore, ia, ib, n, ra, rb, phi):
        """Given network rows; n, ra, rb as (m, 3) (host or device), ia, ib, phi (m,)."""
        dev = "cuda"
        t32 = lambda a: torch.as_tensor(np.asarray(a) if not torch.is_tensor(a) else a, dtype=torch.int32,
                                        device=dev).contiguous()
        tpl = lambda a: torch.as_tensor(np.asarray(a) if not torch.is_tensor(a) else a, dtype=torch.float64,
                                        device=dev).T.contiguous()
        ia_t, ib_t = t32(ia), t32(ib)
        n_t, ra_t, rb_t = tpl(n), tpl(ra), tpl(rb)
        phi_t = torch.as_tensor(np.asarray(phi) if not torch.is_tensor(phi) else phi, dtype=torch.float64,
                                device=dev).contiguous()
        bv, cv = bodies.view(), cs.view()
        m, f = ia_t.numel(), torch.float64
        rc = self.L.relcp_load_constraints(self.h, ctypes.byref(bv), ctypes.byref(cv), m,
                                           _dptr(ia_t, torch.int32, m, "ia"), _dptr(ib_t, torch.int32, m, "ib"),
                                           _dptr(n_t, f, 3 * m, "n"), _dptr(ra_t, f, 3 * m, "ra"),
                                           _dptr(rb_t, f, 3 * m, "rb"), _dptr(phi_t, f, m, "phi"))
        cs.sync_from(cv)
        self._check(rc)

    def prepare_operator(self, bodies: BodyState, cs: ConstraintStore):
        bv, cv = bodies.view(), cs.view()
        self._check(self.L.relcp_prepare_operator(self.h, ctypes.byref(bv), ctypes.byref(cv)))
        self._op = (bv, cv)

    def delassus_apply(self, bodies: BodyState, cs: ConstraintStore, x: torch.Tensor, y: torch.Tensor,
                       scale: float = 1.0):
        bv, cv = bodies.view(), cs.view()
        m = cs.count
        self._check(self.L.relcp_delassus_apply(self.h, ctypes.byref(bv), ctypes.byref(cv),
                                                _dptr(x, torch.float64, m, "x"), _dptr(y, torch.float64, m, "y"),
                                                float(scale)))

    def wrench(self, bodies: BodyState, cs: ConstraintStore, x: torch.Tensor, F=None, U=None):
        bv, cv = bodies.view(), cs.view()
        f, m, n = torch.float64, cs.count, bodies.n
        self._check(self.L.relcp_wrench(self.h, ctypes.byref(bv), ctypes.byref(cv), _dptr(x, f, m, "x"),
                                        _dptr(F, f, 6 * n, "F", True), _dptr(U, f, 6 * n, "U", True)))

    def solve_lcp(self, bodies: BodyState, cs: ConstraintStore):
        bv, cv = bodies.view(), cs.view()
        rep = SolveReport()
        rc = self.L.relcp_solve_lcp(self.h, ctypes.byref(bv), ctypes.byref(cv), ctypes.byref(rep))
        self._check(rc)
        return dict(iterations=rep.iterations, residual=rep.residual, converged=bool(rep.converged),
                    objective=rep.objective, L=rep.L, status=rc)

    def check_and_augment(self, bodies: BodyState, cs: ConstraintStore, recursion: int):
        bv, cv = bodies.view(), cs.view()
        n = i64()
        mp = f64()
        rc = self.L.relcp_check_and_augment(self.h, ctypes.byref(bv), ctypes.byref(cv), int(recursion),
                                            ctypes.byref(n), ctypes.byref(mp))
        cs.sync_from(cv)
        self._check(rc)
        return int(n.value), float(mp.value)

    def step(self, bodies: BodyState, cs: ConstraintStore, f_ext: torch.Tensor | None = None):
        bv, cv = bodies.view(), cs.view()
        rep = StepReport()
        fe = _dptr(f_ext, torch.float64, 6 * bodies.n, "f_ext", True)
        rc = self.L.relcp_step(self.h, ctypes.byref(bv), fe, ctypes.byref(cv), ctypes.byref(rep))
        cs.sync_from(cv)
        self._check(rc)
        d = rep.as_dict()
        d["rc"] = rc
        return d

    def stats(self):
        st = Stats()
        self._check(self.L.relcp_get_stats(self.h, ctypes.byref(st)))
        return dict(launches=st.launches, lcp_iterations=st.lcp_iterations, iter_timed=st.iter_timed,
                    scatter_ms=st.scatter_ms, gather_ms=st.gather_ms, split_timed=st.split_timed,
                    iter_ms=st.iter_ms, n_guard=st.n_guard, jds_solves=st.jds_solves, op_layout=st.op_layout,
                    cluster_solves=st.cluster_solves, snsd_multistart=st.snsd_multistart)

    def reset_stats(self):
        self._check(self.L.relcp_reset_stats(self.h))

    def set_timing(self, on: bool):
        self._check(self.L.relcp_set_timing(self.h, 1 if on else 0))

    def get_pairs(self):
        n = i64()
        self._check(self.L.relcp_get_pairs(self.h, None, None, 0, ctypes.byref(n)))
        m = int(n.value)
        pi = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
        pj = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
        self._check(self.L.relcp_get_pairs(self.h, _ptr(pi), _ptr(pj), m, ctypes.byref(n)))
        return pi[:m], pj[:m]

    def snsd_pairs(self, bodies: BodyState, pi, pj):
        def idx(a):
            if torch.is_tensor(a):
                return a.to(device="cuda", dtype=torch.int32).contiguous()
            return torch.as_tensor(np.asarray(a), dtype=torch.int32, device="cuda")
        pi, pj = idx(pi), idx(pj)
        m = pi.numel()
        phi = torch.empty(max(m, 1), dtype=torch.float64, device="cuda")
        nrm = torch.empty(3, max(m, 1), dtype=torch.float64, device="cuda")
        ra = torch.empty_like(nrm)
        rb = torch.empty_like(nrm)
        st = torch.empty(max(m, 1), dtype=torch.int32, device="cuda")
        bv = bodies.view()
        if pj.numel() != m:
            raise ValueError("snsd_pairs: pi and pj differ in length")
        self._check(self.L.relcp_snsd_pairs(self.h, ctypes.byref(bv), m, _dptr(pi, torch.int32, m, "pi"),
                                            _dptr(pj, torch.int32, m, "pj"), _ptr(phi), _ptr(nrm), _ptr(ra), _ptr(rb),
                                            _ptr(st)))
        torch.cuda.synchronize()
        return phi[:m], nrm[:, :m], ra[:, :m], rb[:, :m], st[:m]


# ---------------------------------------------------------------- domain decomposition
def dd_plan_host(part_off, ia, ib, part: int):
    """Host-only partition plan of `part` (relcp_dd_plan_host; no device):
    info dict + ghost (global ids), gseg, rseg, recv_list (numpy)."""
    L = load()
    off = np.ascontiguousarray(part_off, dtype=np.int64)
    ia = np.ascontiguousarray(ia, dtype=np.int32)
    ib = np.ascontiguousarray(ib, dtype=np.int32)
    K = len(off) - 1
    info = DDInfo()
    p = lambda a: a.ctypes.data_as(P) if a is not None and a.size else None
    rc = L.relcp_dd_plan_host(K, p(off), len(ia), p(ia), p(ib), int(part), ctypes.byref(info), None, None, None, None)
    if rc != OK:
        raise RelcpError(rc, "relcp_dd_plan_host")
    ghost = np.empty(info.n_ghost, dtype=np.int64)
    gseg = np.empty(K + 1, dtype=np.int64)
    rseg = np.empty(K + 1, dtype=np.int64)
    recv = np.empty(info.n_recv, dtype=np.int32)
    rc = L.relcp_dd_plan_host(K, p(off), len(ia), p(ia), p(ib), int(part), ctypes.byref(info), p(ghost), p(gseg),
                              p(rseg), p(recv))
    if rc != OK:
        raise RelcpError(rc, "relcp_dd_plan_host")
    return dict(info=info.as_dict(), ghost=ghost, gseg=gseg, rseg=rseg, recv_list=recv)


def dd_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = load().relcp_dd_nccl_unique_id(ctypes.cast(buf, P))
    if rc != OK:
        raise RelcpError(rc, "relcp_dd_nccl_unique_id")
    return buf.raw


class DomainDecomposition:
    """relcp_dd: the Delassus operator / BB solve split over K body ranges.
    rank < 0: all K parts here (VIRTUAL, one device); rank >= 0: this process
    holds part `rank` of K (NCCL; nccl_uid from dd_nccl_unique_id on rank 0)."""

    def __init__(self, part_off, rank: int = -1, nccl_uid: bytes | None = None, params: Params | None = None,
                 stream: torch.cuda.Stream | None = None, **kw):
        if not torch.cuda.is_available():
            raise RuntimeError("relcp: no CUDA device (there is no CPU fallback)")
        self.L = load()
        self.params = params if params is not None else default_params(**kw)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.off = np.ascontiguousarray(part_off, dtype=np.int64)
        uid = ctypes.create_string_buffer(nccl_uid, 128) if nccl_uid is not None else None
        h = P()
        rc = self.L.relcp_dd_create(ctypes.byref(h), ctypes.byref(self.params), P(self.stream.cuda_stream),
                                    len(self.off) - 1, self.off.ctypes.data_as(P), int(rank),
                                    ctypes.cast(uid, P) if uid is not None else None)
        if rc != OK:
            raise RelcpError(rc, "relcp_dd_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.relcp_dd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc < 0:
            raise RelcpError(rc, self.L.relcp_dd_last_error(self.h).decode(errors="replace"))
        return rc

    def load(self, bodies: BodyState, cs: ConstraintStore):
        self._views = (bodies.view(), cs.view())
        self._check(self.L.relcp_dd_load(self.h, ctypes.byref(self._views[0]), ctypes.byref(self._views[1])))

    def info(self, part: int):
        inf = DDInfo()
        self._check(self.L.relcp_dd_info_get(self.h, int(part), ctypes.byref(inf)))
        return inf.as_dict()

    def delassus_apply(self, x: torch.Tensor, y: torch.Tensor, scale: float = 1.0):
        m = int(self._views[1].count)
        self._check(self.L.relcp_dd_delassus_apply(self.h, _dptr(x, torch.float64, m, "x"),
                                                   _dptr(y, torch.float64, m, "y"), float(scale)))

    def get_u(self, U: torch.Tensor):
        n = int(self._views[0].n)
        self._check(self.L.relcp_dd_get_u(self.h, _dptr(U, torch.float64, 6 * n, "U")))

    def step(self, bodies: BodyState, cs: ConstraintStore, f_ext: torch.Tensor | None = None):
        """relcp_dd_step: Algorithm 1 with domain-decomposed LCP solves."""
        bv, cv = bodies.view(), cs.view()
        rep = StepReport()
        fe = _dptr(f_ext, torch.float64, 6 * bodies.n, "f_ext", True)
        rc = self.L.relcp_dd_step(self.h, ctypes.byref(bv), fe, ctypes.byref(cv), ctypes.byref(rep))
        cs.sync_from(cv)
        self._check(rc)
        d = rep.as_dict()
        d["rc"] = rc
        return d

    def solve_lcp(self, cs: ConstraintStore):
        cv = cs.view()
        rep = SolveReport()
        rc = self._check(self.L.relcp_dd_solve_lcp(self.h, ctypes.byref(cv), ctypes.byref(rep)))
        return dict(iterations=rep.iterations, residual=rep.residual, converged=bool(rep.converged),
                    objective=rep.objective, L=rep.L, status=rc)
