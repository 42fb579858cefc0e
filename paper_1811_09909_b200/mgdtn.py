"""Thin ctypes binding of libmgdtn.so (include/mgdtn.h), same names as the C ABI.

Argument marshalling only: every step of the method runs in the library's
CUDA kernels.  PyTorch provides device memory (the caller-owned workspace),
the stream and pinned host buffers.  There is no CPU fallback: if the shared
library or a CUDA device is missing, construction raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmgdtn.so")

MG_OK = 0
MG_HDG, MG_SIPG_H, MG_IIPG_H, MG_NIPG_H = 0, 1, 2, 3
MG_BUILD_NONSYMMETRIC = 1
MG_SMOOTH_BLOCK_JACOBI, MG_SMOOTH_CHEBYSHEV, MG_SMOOTH_LUSGS = 0, 1, 2
STATUS = {0: "converged", 1: "maxit", 2: "diverged", 3: "breakdown"}
ERRORS = {-1: "MG_ERR_ARG", -2: "MG_ERR_SHAPE", -3: "MG_ERR_SINGULAR_LOCAL", -4: "MG_ERR_NOT_SPD",
          -5: "MG_ERR_CUDA", -6: "MG_ERR_NCCL", -7: "MG_ERR_STATE", -8: "MG_ERR_WORKSPACE",
          -9: "MG_ERR_UNSUPPORTED"}


class mg_quad_mesh(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("x0", C.c_double), ("y0", C.c_double),
                ("h", C.c_double)]


class mg_partition(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("px", C.c_int32), ("py", C.c_int32),
                ("nccl_id", C.c_void_p), ("gather_ne", C.c_int32), ("loopback", C.c_void_p)]


class mg_smoother_cfg(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nu_pre", C.c_int32), ("nu_post", C.c_int32),
                ("omega", C.c_double), ("cheb_ratio", C.c_double), ("lmax_iters", C.c_int32),
                ("lmax_safety", C.c_double), ("nu_doubling", C.c_int32)]


# exported symbols and their argtypes (must match include/mgdtn.h)
_P = C.c_void_p
_SIGS = {
    "mg_build_hierarchy": [C.POINTER(mg_quad_mesh), C.c_int32, C.c_int32, C.POINTER(mg_partition), _P,
                           C.POINTER(C.c_void_p)],
    "mg_build_hierarchy_ex": [C.POINTER(mg_quad_mesh), C.c_int32, C.c_int32, C.POINTER(mg_partition),
                              C.c_int32, _P, C.POINTER(C.c_void_p)],
    "mg_workspace_bytes": [_P, C.POINTER(C.c_size_t)],
    "mg_bind_workspace": [_P, _P, C.c_size_t],
    "mg_setup_dtn": [_P, _P, _P, _P, C.POINTER(mg_smoother_cfg)],
    "mg_assemble_rhs": [_P, _P, C.c_double, _P, _P, _P],
    "mg_apply": [_P, C.c_int32, _P, _P],
    "mg_vcycle": [_P, _P, _P],
    "mg_smooth": [_P, C.c_int32, _P, _P, C.c_int32],
    "mg_local_correct": [_P, C.c_int32, _P, _P],
    "mg_restrict": [_P, C.c_int32, _P, _P],
    "mg_prolong": [_P, C.c_int32, _P, _P],
    "mg_pcg_solve": [_P, _P, _P, C.c_double, C.c_int32, C.POINTER(C.c_int32),
                     C.POINTER(C.c_double), C.POINTER(C.c_int32), _P],
    "mg_solve_host": [_P, _P, _P, _P, _P, C.c_double, _P, C.POINTER(mg_smoother_cfg), C.c_double,
                      C.c_int32, _P, C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_int32)],
    "mg_mg_solve": [_P, _P, _P, C.c_double, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                    C.POINTER(C.c_int32), _P],
    "mg_gmres_solve": [_P, _P, _P, C.c_double, C.c_int32, _P, C.POINTER(C.c_int32),
                       C.POINTER(C.c_double), C.POINTER(C.c_int32), _P],
    "mg_staging_bytes": [_P, C.c_int32, C.c_int32, C.POINTER(C.c_size_t)],
    "mg_bind_staging": [_P, _P, C.c_size_t],
    "mg_recover_volume": [_P, _P, _P, C.c_double, _P, _P, C.POINTER(C.c_double)],
    "mg_num_levels": [_P, C.POINTER(C.c_int32)],
    "mg_level_info": [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                      C.POINTER(C.c_int32), C.POINTER(C.c_int64)],
    "mg_copy_element_dtn": [_P, C.c_int32, _P],
    "mg_gather_element_dtn": [_P, C.c_int32, _P, C.c_int64, _P],
    "mg_debug_set_element_dtn": [_P, C.c_int32, _P],
    "mg_level_lambda_max": [_P, C.c_int32, C.POINTER(C.c_double)],
    "mg_last_launch_count": [_P, C.POINTER(C.c_int64)],
    "mg_total_launch_count": [_P, C.POINTER(C.c_int64)],
    "mg_set_use_graphs": [_P, C.c_int32],
    "mg_set_option": [_P, C.c_int32, C.c_int64],
    "mg_check_invariants": [_P, _P],
    "mg_partition_plan": [C.POINTER(mg_quad_mesh), C.c_int32, C.c_int32, C.POINTER(mg_partition),
                          C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32), _P],
    "mg_partition_side_edges": [C.POINTER(mg_quad_mesh), C.c_int32, C.c_int32,
                                C.POINTER(mg_partition), C.c_int32, C.c_int32, _P,
                                C.POINTER(C.c_int32)],
    "mg_get_nccl_unique_id": [_P],
    "mg_loopback_create": [C.c_int32],
    "mg_loopback_destroy": [_P],
    "mg_loopback_abort": [_P],
    "mg_agglomerate_seeds": [C.c_int64, C.c_int64, _P, _P, _P, C.c_int32, _P, C.c_int32, _P, _P, _P,
                             _P, _P, C.POINTER(C.c_int64)],
    "mg_macro_edge_params": [C.c_int64, _P, C.c_int64, _P, C.c_int64, _P, _P, _P, _P],
    "mg_macro_edge_transfer": [C.c_int64, _P, C.c_int32, _P, _P],
    "mg_last_error": [_P],
    "mg_last_error_index": [_P],
    "mg_destroy": [_P],
}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libmgdtn.so (raises if absent -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `python -m paper_1811_09909_b200.build` "
                          "(or __graft_entry__.build()) first")
    lib = C.CDLL(path)
    for name, args in _SIGS.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = C.c_int
    lib.mg_last_error.restype = C.c_char_p
    lib.mg_last_error_index.restype = C.c_int64
    lib.mg_destroy.restype = None
    lib.mg_loopback_create.restype = C.c_void_p
    lib.mg_loopback_destroy.restype = None
    lib.mg_loopback_abort.restype = None
    _lib = lib
    return lib


class MGError(RuntimeError):
    pass


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


@dataclass
class SmootherConfig:
    kind: int = MG_SMOOTH_BLOCK_JACOBI
    nu_pre: int = 2
    nu_post: int = 2
    omega: float = 1.0
    cheb_ratio: float = 30.0
    lmax_iters: int = 20
    lmax_safety: float = 1.05
    nu_doubling: bool = False

    def c(self):
        return mg_smoother_cfg(self.kind, self.nu_pre, self.nu_post, self.omega, self.cheb_ratio,
                               self.lmax_iters, self.lmax_safety, int(self.nu_doubling))


class _Ordered:
    """Order the library stream after the caller's current stream and back."""

    def __init__(self, stream, device):
        self.s = stream
        self.cur = torch.cuda.current_stream(device)

    def __enter__(self):
        if self.cur != self.s:
            self.s.wait_stream(self.cur)
        return self

    def __exit__(self, *exc):
        if self.cur != self.s:
            self.cur.wait_stream(self.s)
        return False


@dataclass
class Partition:
    """Element-block partition of the global mesh over px x py ranks (mg_partition).

    nccl_id: the 128-byte id from nccl_unique_id() on rank 0 (NCCL, one process per
    GPU); loopback: a LoopbackHub instead (virtual ranks in one process, tests)."""
    rank: int
    nranks: int
    px: int
    py: int
    nccl_id: bytes | None = None
    gather_ne: int = 0
    loopback: "LoopbackHub | None" = None

    def c(self):
        self._id = None if self.nccl_id is None else C.create_string_buffer(bytes(self.nccl_id), 128)
        return mg_partition(self.rank, self.nranks, self.px, self.py,
                            None if self._id is None else C.cast(self._id, C.c_void_p),
                            self.gather_ne, None if self.loopback is None else self.loopback.handle)

    def block(self, nx: int, ny: int):
        """(ox, oy, bx, by): this rank's element block of an nx x ny level."""
        bx, by = nx // self.px, ny // self.py
        return (self.rank % self.px) * bx, (self.rank // self.px) * by, bx, by


class LoopbackHub:
    """Communicator hub for `n` virtual ranks in this process on one GPU (tests)."""

    def __init__(self, n: int):
        self.lib = load_library()
        self.handle = C.c_void_p(self.lib.mg_loopback_create(n))
        self.n = n

    def abort(self):
        """A rank failed: release the others from their collectives (they raise MGError)."""
        if self.handle:
            self.lib.mg_loopback_abort(self.handle)

    def close(self):
        if self.handle:
            self.lib.mg_loopback_destroy(self.handle)
            self.handle = None


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(128)
    rc = lib.mg_get_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc != MG_OK:
        raise MGError(f"mg_get_nccl_unique_id: {ERRORS.get(rc, rc)}")
    return buf.raw


def agglomerate_seeds(edge_elem, cx, cy, seeds, nlev: int, stream=None):
    """Seed-point agglomeration (mg_agglomerate_seeds): device
    tensors in (edge_elem int32 [nedge, 2], cx / cy float64 [ne], seeds int32),
    device tensors out: labels int32 [nlev-1, ne], skeleton uint8 [nlev-1, nedge],
    macro-edge ids int32 [nlev-1, nedge]; and the macro-edge count per level (list)."""
    import torch
    lib = load_library()
    ne, nedge = int(cx.numel()), int(edge_elem.shape[0])
    for t, dt in ((edge_elem, torch.int32), (cx, torch.float64), (cy, torch.float64),
                  (seeds, torch.int32)):
        if not t.is_cuda or t.dtype != dt or not t.is_contiguous():
            raise MGError(f"agglomerate_seeds: expected a contiguous CUDA {dt} tensor")
    dev = cx.device
    labels = torch.empty((max(nlev - 1, 1), ne), dtype=torch.int32, device=dev)
    skel = torch.empty((max(nlev - 1, 1), nedge), dtype=torch.uint8, device=dev)
    medge = torch.empty((max(nlev - 1, 1), nedge), dtype=torch.int32, device=dev)
    nme = (C.c_int64 * max(nlev - 1, 1))()
    st = torch.cuda.current_stream(dev) if stream is None else stream
    bad = C.c_int64(-1)
    rc = lib.mg_agglomerate_seeds(ne, nedge, _ptr(edge_elem), _ptr(cx), _ptr(cy), int(seeds.numel()),
                                  _ptr(seeds), int(nlev), _ptr(labels), _ptr(skel), _ptr(medge),
                                  C.cast(nme, C.c_void_p), C.c_void_p(st.cuda_stream), C.byref(bad))
    if rc != 0:
        raise MGError(f"mg_agglomerate_seeds: {ERRORS.get(rc, rc)} (element {bad.value})")
    return labels, skel, medge, list(nme)[:nlev - 1]


def macro_edge_params(medge, nmedge: int, edge_vert, vx, vy, stream=None):
    """Arc-length parameter of one level's macro-edges (mg_macro_edge_params, reading
    A5): device tensors in (medge int32 [nedge], edge_vert int32 [nedge, 2], vx / vy
    float64 [nvert]); device float64 [nedge, 2] out (-1 where not parameterised)."""
    import torch
    lib = load_library()
    for t, dt in ((medge, torch.int32), (edge_vert, torch.int32), (vx, torch.float64),
                  (vy, torch.float64)):
        if not t.is_cuda or t.dtype != dt or not t.is_contiguous():
            raise MGError(f"macro_edge_params: expected a contiguous CUDA {dt} tensor")
    nedge = int(medge.numel())
    s = torch.empty((nedge, 2), dtype=torch.float64, device=medge.device)
    st = torch.cuda.current_stream(medge.device) if stream is None else stream
    rc = lib.mg_macro_edge_params(nedge, _ptr(medge), int(nmedge), _ptr(edge_vert), int(vx.numel()),
                                  _ptr(vx), _ptr(vy), _ptr(s), C.c_void_p(st.cuda_stream))
    if rc != 0:
        raise MGError(f"mg_macro_edge_params: {ERRORS.get(rc, rc)}")
    return s


def macro_edge_transfer(s, p: int, stream=None):
    """P^p transfer blocks J_e of the parameterised macro-edges (mg_macro_edge_transfer,
    reading A6): device float64 [nedge, 2] in, device float64 [nedge, p+1, p+1] out."""
    import torch
    lib = load_library()
    if not s.is_cuda or s.dtype != torch.float64 or not s.is_contiguous():
        raise MGError("macro_edge_transfer: expected a contiguous CUDA float64 tensor")
    nedge = int(s.shape[0])
    J = torch.empty((nedge, p + 1, p + 1), dtype=torch.float64, device=s.device)
    st = torch.cuda.current_stream(s.device) if stream is None else stream
    rc = lib.mg_macro_edge_transfer(nedge, _ptr(s), int(p), _ptr(J), C.c_void_p(st.cuda_stream))
    if rc != 0:
        raise MGError(f"mg_macro_edge_transfer: {ERRORS.get(rc, rc)}")
    return J


def partition_plan(nx: int, ny: int, p: int, part: Partition, n_h_levels: int = 0):
    """Host-only decomposition (no device work): dict(nlevels, gather_level, levels=[...]),
    levels[k-1] = dict(nx, ny, ox, oy, gnx, gny, dmask, imask) of paper level k."""
    lib = load_library()
    mesh = mg_quad_mesh(nx, ny, 0.0, 0.0, 1.0 / nx)
    info = np.zeros(8 * 64, dtype=np.int32)
    nl, gl = C.c_int32(), C.c_int32()
    pc = part.c()
    rc = lib.mg_partition_plan(C.byref(mesh), p, n_h_levels, C.byref(pc), 64, C.byref(nl),
                               C.byref(gl), C.c_void_p(info.ctypes.data))
    if rc != MG_OK:
        raise MGError(f"mg_partition_plan: {ERRORS.get(rc, rc)}")
    keys = ("nx", "ny", "ox", "oy", "gnx", "gny", "dmask", "imask")
    levels = [dict(zip(keys, info[8 * k:8 * k + 8].tolist())) for k in range(nl.value)]
    return dict(nlevels=nl.value, gather_level=gl.value, levels=levels)


def partition_side_edges(nx: int, ny: int, p: int, part: Partition, level: int, side: int,
                         n_h_levels: int = 0) -> np.ndarray:
    """Global edge ids of an interface side of a level's block, in halo-message order."""
    lib = load_library()
    mesh = mg_quad_mesh(nx, ny, 0.0, 0.0, 1.0 / nx)
    pc = part.c()
    cnt = C.c_int32()
    rc = lib.mg_partition_side_edges(C.byref(mesh), p, n_h_levels, C.byref(pc), level, side, None,
                                     C.byref(cnt))
    if rc != MG_OK:
        raise MGError(f"mg_partition_side_edges: {ERRORS.get(rc, rc)}")
    out = np.zeros(cnt.value, dtype=np.int64)
    if cnt.value:
        lib.mg_partition_side_edges(C.byref(mesh), p, n_h_levels, C.byref(pc), level, side,
                                    C.c_void_p(out.ctypes.data), C.byref(cnt))
    return out


class MGSolver:
    """One context of the C ABI on a CUDA device (own stream unless given).

    partition: None (one GPU) or a Partition -- then nx, ny are the GLOBAL mesh and
    every array argument is this rank's element block / its local edge numbering.
    nonsymmetric: build with MG_BUILD_NONSYMMETRIC (IIPG-H / NIPG-H elements; full
    element maps, LU blocks; solve with mg_solve / gmres_solve, block-Jacobi only)."""

    def __init__(self, nx: int, ny: int | None = None, p: int = 1, h: float | None = None,
                 n_h_levels: int = 0, device="cuda", stream: torch.cuda.Stream | None = None,
                 partition: Partition | None = None, nonsymmetric: bool = False):
        if not torch.cuda.is_available():
            raise MGError("MGSolver needs a CUDA device (no CPU fallback)")
        self.lib = load_library()
        ny = nx if ny is None else ny
        self.partition = partition
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        # the library works on its own (capturable) stream; every call orders it
        # after the caller's current stream and the caller after it (_Ordered)
        self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        self.nx, self.ny, self.p = nx, ny, p
        mesh = mg_quad_mesh(nx, ny, 0.0, 0.0, h if h is not None else 1.0 / nx)
        ctx = C.c_void_p()
        self._pc = None if partition is None else partition.c()
        self.nonsymmetric = bool(nonsymmetric)
        rc = self.lib.mg_build_hierarchy_ex(C.byref(mesh), p, n_h_levels,
                                            None if self._pc is None else C.byref(self._pc),
                                            MG_BUILD_NONSYMMETRIC if nonsymmetric else 0,
                                            C.c_void_p(self.stream.cuda_stream), C.byref(ctx))
        if rc != MG_OK:
            raise MGError(f"mg_build_hierarchy failed: {ERRORS.get(rc, rc)}")
        self.ctx = ctx
        nb = C.c_size_t()
        self._chk(self.lib.mg_workspace_bytes(self.ctx, C.byref(nb)), "mg_workspace_bytes")
        self.workspace = torch.empty(nb.value, dtype=torch.uint8, device=self.device)
        with self._ordered():
            rc = self.lib.mg_bind_workspace(self.ctx, _ptr(self.workspace), nb.value)
        self._chk(rc, "mg_bind_workspace")
        self.staging = None
        nl = C.c_int32()
        self._chk(self.lib.mg_num_levels(self.ctx, C.byref(nl)), "mg_num_levels")
        self.nlevels = nl.value

    # ------------------------------------------------------------------ helpers
    def _ordered(self):
        return _Ordered(self.stream, self.device)

    def _call(self, name, *args):
        """Call an ABI function ordered against the caller's stream; raise on error."""
        with self._ordered():
            rc = getattr(self.lib, name)(self.ctx, *args)
        self._chk(rc, name)

    def _chk(self, rc, what):
        if rc != MG_OK:
            msg = self.lib.mg_last_error(self.ctx).decode() if getattr(self, "ctx", None) else ""
            idx = self.lib.mg_last_error_index(self.ctx) if getattr(self, "ctx", None) else -1
            raise MGError(f"{what}: {ERRORS.get(rc, rc)}: {msg} (index {idx})")

    def level_info(self, level: int):
        nx, ny, p, nd = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        self._chk(self.lib.mg_level_info(self.ctx, level, C.byref(nx), C.byref(ny), C.byref(p),
                                         C.byref(nd)), "mg_level_info")
        return dict(nx=nx.value, ny=ny.value, p=p.value, ndof=nd.value)

    def ndof(self, level: int | None = None) -> int:
        return self.level_info(self.nlevels if level is None else level)["ndof"]

    def _vec(self, level=None):
        return torch.zeros(self.ndof(level), dtype=torch.float64, device=self.device)

    @staticmethod
    def _dev(x, dtype):
        return x.to(dtype=dtype).contiguous() if torch.is_tensor(x) else torch.as_tensor(
            np.ascontiguousarray(x), dtype=dtype)

    def _d(self, x, dtype=torch.float64):
        if x is None:
            return None
        t = self._dev(x, dtype)
        return t.to(self.device) if t.device != self.device else t

    # ------------------------------------------------------------------ ABI calls
    def setup(self, K, method, tau, smoother: SmootherConfig | None = None):
        sm = smoother or SmootherConfig()
        self._K = self._d(K)
        self._m = self._d(method, torch.int8)
        self._tau = self._d(tau)
        cfg = sm.c()
        self._call("mg_setup_dtn", _ptr(self._K), _ptr(self._m), _ptr(self._tau),
                                        C.byref(cfg))

    def assemble_rhs(self, f_qp=None, f_const=0.0, gD_qp=None):
        g = self._vec()
        lam_bc = self._vec()
        f = self._d(f_qp)
        gd = self._d(gD_qp)
        self._call("mg_assemble_rhs", _ptr(f), float(f_const), _ptr(gd), _ptr(g),
                                           _ptr(lam_bc))
        return g, lam_bc

    def apply(self, level: int, x, y=None):
        x = self._d(x)
        y = self._vec(level) if y is None else y
        self._call("mg_apply", level, _ptr(x), _ptr(y))
        return y

    def vcycle(self, r, z=None):
        r = self._d(r)
        z = self._vec() if z is None else z
        self._call("mg_vcycle", _ptr(r), _ptr(z))
        return z

    def smooth(self, level: int, r, e, nsteps: int):
        r = self._d(r)
        e = self._d(e).clone()
        self._call("mg_smooth", level, _ptr(r), _ptr(e), nsteps)
        return e

    def local_correct(self, level: int, res, e):
        res = self._d(res)
        e = self._d(e).clone()
        self._call("mg_local_correct", level, _ptr(res), _ptr(e))
        return e

    def restrict(self, level: int, res):
        res = self._d(res)
        rc = self._vec(level - 1)
        self._call("mg_restrict", level, _ptr(res), _ptr(rc))
        return rc

    def prolong(self, level: int, ec, e):
        ec = self._d(ec)
        e = self._d(e).clone()
        self._call("mg_prolong", level, _ptr(ec), _ptr(e))
        return e

    def pcg_solve(self, g, rtol=1e-10, maxit=2000, lam=None, history=False):
        g = self._d(g)
        lam = self._vec() if lam is None else lam
        it, rel, st = C.c_int32(), C.c_double(), C.c_int32()
        hist = np.zeros(maxit + 1) if history else None
        hp = hist.ctypes.data_as(C.c_void_p) if history else None
        self._call("mg_pcg_solve", _ptr(g), _ptr(lam), rtol, maxit, C.byref(it),
                                        C.byref(rel), C.byref(st), hp)
        info = dict(iters=it.value, relres=rel.value, status=STATUS[st.value])
        if history:
            info["hist"] = hist[: it.value + 1]
        return lam, info

    def mg_solve(self, g, tol=1e-9, maxit=200, history=False):
        """MG as a solver (mg_mg_solve)."""
        g = self._d(g)
        lam = self._vec()
        it, rel, st = C.c_int32(), C.c_double(), C.c_int32()
        hist = np.zeros(maxit + 1) if history else None
        self._call("mg_mg_solve", _ptr(g), _ptr(lam), tol, maxit, C.byref(it), C.byref(rel),
                   C.byref(st), hist.ctypes.data_as(C.c_void_p) if history else None)
        info = dict(iters=it.value, relres=rel.value, status=STATUS[st.value])
        if history:
            info["hist"] = hist[: it.value + 1]
        return lam, info

    def gmres_solve(self, g, tol=1e-9, maxit=200, history=False):
        """Left-preconditioned full GMRES (mg_gmres_solve)."""
        g = self._d(g)
        lam = self._vec()
        basis = torch.empty((maxit + 1) * self.ndof(), dtype=torch.float64, device=self.device)
        it, rel, st = C.c_int32(), C.c_double(), C.c_int32()
        hist = np.zeros(maxit + 1) if history else None
        self._call("mg_gmres_solve", _ptr(g), _ptr(lam), tol, maxit, _ptr(basis), C.byref(it),
                   C.byref(rel), C.byref(st), hist.ctypes.data_as(C.c_void_p) if history else None)
        info = dict(iters=it.value, relres=rel.value, status=STATUS[st.value])
        if history:
            info["hist"] = hist[: it.value + 1]
        return lam, info

    def bind_staging(self, with_f: bool, with_gD: bool):
        nb = C.c_size_t()
        self._chk(self.lib.mg_staging_bytes(self.ctx, int(with_f), int(with_gD), C.byref(nb)),
                  "mg_staging_bytes")
        if self.staging is None or self.staging.numel() < nb.value:
            self.staging = torch.empty(nb.value, dtype=torch.uint8, device=self.device)
            self._chk(self.lib.mg_bind_staging(self.ctx, _ptr(self.staging), nb.value),
                      "mg_bind_staging")

    def solve_host(self, K, method, tau, f_qp=None, f_const=0.0, gD_qp=None,
                   smoother: SmootherConfig | None = None, rtol=1e-10, maxit=2000, out=None):
        """The user call with HOST buffers (numpy or pinned CPU tensors)."""
        def host(a, dt):
            if a is None:
                return None
            if torch.is_tensor(a):
                assert a.device.type == "cpu" and a.is_contiguous()
                return a
            return np.ascontiguousarray(a, dtype=dt)

        def hp(a):
            if a is None:
                return None
            return C.c_void_p(a.data_ptr()) if torch.is_tensor(a) else a.ctypes.data_as(C.c_void_p)
        K, method, tau = host(K, np.float64), host(method, np.int8), host(tau, np.float64)
        f_qp, gD_qp = host(f_qp, np.float64), host(gD_qp, np.float64)
        self.bind_staging(f_qp is not None, gD_qp is not None)
        out = np.empty(self.ndof()) if out is None else out
        cfg = (smoother or SmootherConfig()).c()
        it, rel, st = C.c_int32(), C.c_double(), C.c_int32()
        self._call("mg_solve_host", hp(K), hp(method), hp(tau), hp(f_qp), float(f_const),
                                         hp(gD_qp), C.byref(cfg), rtol, maxit, hp(out), C.byref(it),
                                         C.byref(rel), C.byref(st))
        return out, dict(iters=it.value, relres=rel.value, status=STATUS[st.value])

    def recover_volume(self, lam_full, f_qp=None, f_const=0.0, q_exact_qp=None):
        """q_T per element (GLL nodal [ne][(p+1)^2]) from the full trace; with q_exact
        samples also the L2 error (mg_recover_volume)."""
        lam_full = self._d(lam_full)
        f = self._d(f_qp)
        qe = self._d(q_exact_qp)
        info = self.level_info(self.nlevels)
        q = torch.empty((info["nx"] * info["ny"], (self.p + 1) ** 2), dtype=torch.float64,
                        device=self.device)
        err = C.c_double(float("nan"))
        self._call("mg_recover_volume", _ptr(lam_full), _ptr(f), float(f_const), _ptr(q),
                   _ptr(qe), C.byref(err) if qe is not None else None)
        return q, (err.value if qe is not None else None)

    def element_dtn(self, level: int):
        info = self.level_info(level)
        m = 4 * (info["p"] + 1)
        out = torch.empty((info["nx"] * info["ny"], m, m), dtype=torch.float64, device=self.device)
        self._call("mg_copy_element_dtn", level, _ptr(out))
        return out

    def gather_element_dtn(self, level: int, elems):
        """Dense DtN maps [n][m][m] of the given element ids (full-size sampling)."""
        info = self.level_info(level)
        m = 4 * (info["p"] + 1)
        idx = self._d(elems, torch.int64)
        out = torch.empty((idx.numel(), m, m), dtype=torch.float64, device=self.device)
        self._call("mg_gather_element_dtn", level, _ptr(idx), idx.numel(), _ptr(out))
        return out

    def set_element_dtn(self, level: int, S):
        S = self._d(S)
        self._call("mg_debug_set_element_dtn", level, _ptr(S))

    def lambda_max(self, level: int) -> float:
        v = C.c_double()
        self._call("mg_level_lambda_max", level, C.byref(v))
        return v.value

    def last_launch_count(self) -> int:
        v = C.c_int64()
        self._chk(self.lib.mg_last_launch_count(self.ctx, C.byref(v)), "mg_last_launch_count")
        return v.value

    def total_launch_count(self) -> int:
        v = C.c_int64()
        self._chk(self.lib.mg_total_launch_count(self.ctx, C.byref(v)), "mg_total_launch_count")
        return v.value

    def use_graphs(self, on: bool):
        self._chk(self.lib.mg_set_use_graphs(self.ctx, int(on)), "mg_set_use_graphs")

    OPT_SWEEP, OPT_APPLY_GRID_CAP, OPT_COMM_TIMEOUT_MS, OPT_GATHER_NE, OPT_KEEP_FINE_MAPS = 1, 2, 3, 4, 5

    def check_invariants(self):
        """mg_check_invariants: dict(const_mode, nonfinite, atomic_apply_diff); raises MGError
        if an invariant fails."""
        rep = (C.c_double * 4)()
        self._call("mg_check_invariants", rep)
        return dict(const_mode=rep[0], nonfinite=rep[1], atomic_apply_diff=rep[2])

    def set_option(self, key: int, value: int):
        """mg_set_option: execution options (kernel choice / grid size) for tests."""
        self._chk(self.lib.mg_set_option(self.ctx, int(key), int(value)), "mg_set_option")

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.mg_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def smoother_from_config(cfg) -> SmootherConfig:
    """SmootherConfig of a workloads.Config (V(nu, nu), BJ or Chebyshev)."""
    return SmootherConfig(kind=cfg.smoother, nu_pre=cfg.nu, nu_post=cfg.nu)
