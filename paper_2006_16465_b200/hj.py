"""Thin ctypes binding of libhj.so (include/hj.h) — argument marshalling only.

Every step of the solve runs in the CUDA kernels of libhj.so; there is no Python or CPU
fallback: if the library is missing or no sm_100 device is usable, calls raise.
Names follow the C-ABI: ``jacobi_solve``, ``jacobi_solve_device``, ``jacobi_solve_dist``,
``hj_resource_figures``, ``hj_nccl_unique_id``, ``hj_last_error`` and the ``Plan`` wrappers of
``hj_plan_*`` (``Plan``; ``DistPlan`` for NCCL row slabs; ``PeerPlan`` for row slabs over the
peer-memory transport).  ``mode``: "hier" (the paper's hierarchical cycle), "classic" (global-
memory Jacobi), "mg" (multigrid V-cycles with the hierarchical cycle as smoother).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhj.so")

HJ_OK, HJ_NOT_CONVERGED, HJ_ERR_INVALID_ARG, HJ_ERR_INVALID_CONFIG = 0, 1, 2, 3
HJ_ERR_NUMERIC, HJ_ERR_CUDA, HJ_ERR_NCCL, HJ_ERR_OOM, HJ_ERR_PEER = 4, 5, 6, 7, 8
STATUS_NAMES = {0: "HJ_OK", 1: "HJ_NOT_CONVERGED", 2: "HJ_ERR_INVALID_ARG", 3: "HJ_ERR_INVALID_CONFIG",
                4: "HJ_ERR_NUMERIC", 5: "HJ_ERR_CUDA", 6: "HJ_ERR_NCCL", 7: "HJ_ERR_OOM", 8: "HJ_ERR_PEER"}
MODES = {"hier": 0, "hierarchical": 0, "classic": 1, "mg": 2, "multigrid": 2}
DTYPES = {"f64": 0, "float64": 0, "f32": 1, "float32": 1}
TOL_MODES = {"rel": 0, "relative": 0, "abs": 1, "absolute": 1}
KERNELS = {"auto": 0, "smem": 1}
KERNEL_KINDS = {0: "reg2d", 1: "smem2d", 2: "classic2d", 3: "reg1d", 4: "smem1d", 5: "classic1d", 6: "regt"}

_P = ctypes.c_void_p


class hj_problem(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("nx", ctypes.c_int64), ("ny", ctypes.c_int64),
                ("h", ctypes.c_double), ("f", _P), ("bc", _P), ("x0", _P), ("stencil", _P)]


def _nstencil(dim, nx, ny):
    """Length of hj_problem.stencil: 2D {a, c, e, f, d}; 1D planes [a | d | c] (DESIGN.md c23)."""
    return 3 * nx * ny if dim == 1 else 5


class hj_params(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("dtype", ctypes.c_int), ("tile_x", ctypes.c_int32),
                ("tile_y", ctypes.c_int32), ("k", ctypes.c_int32), ("overlap", ctypes.c_int32),
                ("tol", ctypes.c_double), ("tol_mode", ctypes.c_int), ("ref_residual", ctypes.c_double),
                ("max_cycles", ctypes.c_int64), ("kernel", ctypes.c_int), ("overlap_y", ctypes.c_int32),
                ("mg_nu1", ctypes.c_int32), ("mg_nu2", ctypes.c_int32), ("mg_omega", ctypes.c_double),
                ("mg_coarse_cycles", ctypes.c_int32), ("mg_levels", ctypes.c_int32)]


class hj_result(ctypes.Structure):
    _fields_ = [("x", _P), ("history", _P), ("cycles", ctypes.c_int64), ("converged", ctypes.c_int32),
                ("initial_residual", ctypes.c_double), ("final_residual", ctypes.c_double),
                ("seconds_solve", ctypes.c_double), ("seconds_total", ctypes.c_double)]


class hj_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("nccl_id", ctypes.c_char_p),
                ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64)]


class HJError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libhj.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() "
                              "(python -m paper_2006_16465_b200.build)")
        if "HJ_NCCL_LIB" not in os.environ:
            # share torch's NCCL (if its wheel is installed) instead of the system copy
            try:
                import nvidia.nccl
                p = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
                if os.path.exists(p):
                    os.environ["HJ_NCCL_LIB"] = p
            except ImportError:
                pass
        L = ctypes.CDLL(LIB_PATH)
        pp, pr, res = ctypes.POINTER(hj_problem), ctypes.POINTER(hj_params), ctypes.POINTER(hj_result)
        for name, args in [("jacobi_solve", [pp, pr, res]),
                           ("jacobi_solve_device", [pp, pr, res, _P]),
                           ("hj_plan_create", [pp, pr, _P, ctypes.POINTER(_P)]),
                           ("hj_plan_reset", [_P]),
                           ("hj_plan_run", [_P, ctypes.c_int64, ctypes.POINTER(ctypes.c_float)]),
                           ("hj_plan_solve", [_P, res]),
                           ("hj_plan_destroy", [_P]),
                           ("hj_nccl_unique_id", [ctypes.c_char_p]),
                           ("jacobi_solve_dist", [pp, pr, res, ctypes.POINTER(hj_dist)]),
                           ("hj_plan_create_dist", [pp, pr, ctypes.POINTER(hj_dist), _P, ctypes.POINTER(_P)]),
                           ("hj_plan_create_peer", [pp, pr, ctypes.POINTER(hj_dist), _P, ctypes.POINTER(_P)]),
                           ("hj_plan_peer_export", [_P, _P]),
                           ("hj_plan_peer_attach", [_P, _P]),
                           ("hj_resource_figures", [pp, pr, ctypes.POINTER(ctypes.c_int64),
                                                    ctypes.POINTER(ctypes.c_int64),
                                                    ctypes.POINTER(ctypes.c_int64)])]:
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        L.hj_last_error.restype = ctypes.c_char_p
        L.hj_last_error.argtypes = []
        L.hj_history_capacity.restype = ctypes.c_int64
        L.hj_history_capacity.argtypes = [ctypes.POINTER(hj_params)]
        L.hj_plan_kernel_kind.restype = ctypes.c_int32
        L.hj_plan_kernel_kind.argtypes = [_P]
        L.hj_plan_launches_per_cycle.restype = ctypes.c_int32
        L.hj_plan_launches_per_cycle.argtypes = [_P]
        _lib = L
    return _lib


def history_capacity(prm) -> int:
    """hj_history_capacity: entries of the residual history a solve with these params keeps."""
    return int(lib().hj_history_capacity(ctypes.byref(prm)))


def hj_last_error() -> str:
    return lib().hj_last_error().decode()


def _check(st, ok=(HJ_OK, HJ_NOT_CONVERGED)):
    if st not in ok:
        raise HJError(st, hj_last_error())
    return st


def make_params(mode="hier", dtype="f64", tile=(32, 32), k=None, overlap=0, tol=1e-4, tol_mode="rel",
                ref_residual=0.0, max_cycles=10**6, kernel="auto", nu1=0, nu2=0, omega=0.0,
                coarse_cycles=0, levels=0):
    """hj_params.  mode "mg": multigrid V-cycles (nu1/nu2 smoothing cycles, damping omega,
    coarse_cycles on the coarsest grid, at most `levels` grids; zeros = the library defaults)."""
    tx, ty = tile if isinstance(tile, (tuple, list)) else (tile, 1)
    if k is None:
        k = 1 if MODES[mode] == 1 else (4 if MODES[mode] == 2 else 16)
    ox, oy = overlap if isinstance(overlap, (tuple, list)) else (overlap, -1)
    return hj_params(MODES[mode], DTYPES[dtype], tx, ty, k, ox,
                     float(tol), TOL_MODES[tol_mode], float(ref_residual), int(max_cycles), KERNELS[kernel], oy,
                     int(nu1), int(nu2), float(omega), int(coarse_cycles), int(levels))


def _host(a, n, name):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if a.size != n:
        raise ValueError(f"{name}: expected {n} values, got {a.size}")
    return a


def _hp(a):
    return None if a is None else a.ctypes.data


def jacobi_solve(dim, nx, ny, h, f, bc=None, x0=None, *, history=True, stencil=None, **params):
    """Host-buffer solve (H2D/D2H inside).  Returns dict(x, history, cycles, converged, status, ...).
    ``stencil``: general coefficients (numpy; hj_problem.stencil), f is then b and h is unused."""
    n = nx * ny
    f = _host(f, n, "f")
    bc = _host(bc, 2 * ny if dim == 1 else 2 * nx + 2 * ny, "bc")   # dim 1: per problem
    x0 = _host(x0, n, "x0")
    stencil = _host(stencil, _nstencil(dim, nx, ny), "stencil")
    prm = make_params(**params)
    x = np.empty(n)
    hist = np.empty(history_capacity(prm)) if history else None
    pb = hj_problem(dim, nx, ny, float(h), _hp(f), _hp(bc), _hp(x0), _hp(stencil))
    res = hj_result(x.ctypes.data, _hp(hist), 0, 0, 0.0, 0.0, 0.0, 0.0)
    st = _check(lib().jacobi_solve(ctypes.byref(pb), ctypes.byref(prm), ctypes.byref(res)),
                ok=(HJ_OK, HJ_NOT_CONVERGED, HJ_ERR_NUMERIC))
    return _result(res, st, x.reshape((ny, nx)) if (dim == 2 or ny > 1) else x,
                   None if hist is None else hist[: res.cycles + 1])


def _result(res, st, x, hist):
    return dict(x=x, history=hist, cycles=res.cycles, converged=bool(res.converged), status=st,
                initial_residual=res.initial_residual, final_residual=res.final_residual,
                seconds_solve=res.seconds_solve, seconds_total=res.seconds_total)


def _dptr(t):
    return None if t is None else t.data_ptr()


def jacobi_solve_device(dim, nx, ny, h, f, bc=None, x0=None, *, history=True, stream=None,
                        stencil=None, **params):
    """Device solve on torch CUDA tensors (float64, stencil included).  Returns torch tensors."""
    import torch
    prm = make_params(**params)
    dev = f.device
    x = torch.empty(nx * ny, dtype=torch.float64, device=dev)
    hist = torch.empty(history_capacity(prm), dtype=torch.float64, device=dev) if history else None
    pb = hj_problem(dim, nx, ny, float(h), _dptr(f), _dptr(bc), _dptr(x0), _dptr(stencil))
    res = hj_result(_dptr(x), _dptr(hist), 0, 0, 0.0, 0.0, 0.0, 0.0)
    s = stream if stream is not None else torch.cuda.current_stream(dev).cuda_stream
    st = _check(lib().jacobi_solve_device(ctypes.byref(pb), ctypes.byref(prm), ctypes.byref(res), s),
                ok=(HJ_OK, HJ_NOT_CONVERGED, HJ_ERR_NUMERIC))
    return _result(res, st, x.view(ny, nx) if (dim == 2 or ny > 1) else x,
                   None if hist is None else hist[: res.cycles + 1])


def hj_resource_figures(dim, nx, ny, **params):
    prm = make_params(**params)
    pb = hj_problem(dim, nx, ny, 1.0 / (nx + 1), None, None, None, None)
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().hj_resource_figures(ctypes.byref(pb), ctypes.byref(prm), ctypes.byref(a),
                                     ctypes.byref(b), ctypes.byref(c)), ok=(HJ_OK,))
    return a.value, b.value, c.value


def hj_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().hj_nccl_unique_id(buf), ok=(HJ_OK,))
    return buf.raw


def jacobi_solve_dist(nx, ny, h, f_local, bc, x0_local, *, rank, nranks, nccl_id: bytes,
                      row_begin, row_end, history=True, stencil=None, **params):
    """Row-slab solve on this rank's GPU (host buffers of the local rows)."""
    nloc = nx * (row_end - row_begin)
    f = _host(f_local, nloc, "f")
    bc = _host(bc, 2 * nx + 2 * ny, "bc")
    x0 = _host(x0_local, nloc, "x0")
    stencil = _host(stencil, 5, "stencil")
    prm = make_params(**params)
    x = np.empty(nloc)
    hist = np.empty(history_capacity(prm)) if history else None
    pb = hj_problem(2, nx, ny, float(h), _hp(f), _hp(bc), _hp(x0), _hp(stencil))
    res = hj_result(x.ctypes.data, _hp(hist), 0, 0, 0.0, 0.0, 0.0, 0.0)
    idbuf = ctypes.create_string_buffer(nccl_id, 128)
    d = hj_dist(rank, nranks, ctypes.cast(idbuf, ctypes.c_char_p), row_begin, row_end)
    st = _check(lib().jacobi_solve_dist(ctypes.byref(pb), ctypes.byref(prm), ctypes.byref(res),
                                        ctypes.byref(d)), ok=(HJ_OK, HJ_NOT_CONVERGED, HJ_ERR_NUMERIC))
    return _result(res, st, x.reshape((row_end - row_begin, nx)),
                   None if hist is None else hist[: res.cycles + 1])


class Plan:
    """hj_plan_*: device-resident state for repeated cycles (bench, resume)."""

    def __init__(self, dim, nx, ny, h, f, bc=None, x0=None, *, stream=None, stencil=None, **params):
        import torch
        self.prm = make_params(**params)
        self.dim, self.nx, self.ny = dim, nx, ny
        if stencil is not None and not isinstance(stencil, torch.Tensor):
            stencil = torch.as_tensor(np.ascontiguousarray(stencil, dtype=np.float64), device=f.device)
        self._keep = (f, bc, x0, stencil)
        self.stream = stream if stream is not None else torch.cuda.current_stream(f.device).cuda_stream
        torch.cuda.synchronize(f.device)   # inputs may have been written on another stream
        pb = hj_problem(dim, nx, ny, float(h), _dptr(f), _dptr(bc), _dptr(x0), _dptr(stencil))
        self._p = _P()
        self._create(pb)
        self.launches_per_cycle_static = lib().hj_plan_launches_per_cycle(self._p)

    def _create(self, pb):
        _check(lib().hj_plan_create(ctypes.byref(pb), ctypes.byref(self.prm), self.stream,
                                    ctypes.byref(self._p)), ok=(HJ_OK,))

    def reset(self):
        _check(lib().hj_plan_reset(self._p), ok=(HJ_OK,))

    def run(self, ncycles, timed=False):
        """Launch ncycles cycles; with timed=True return the summed cycle-kernel ms (events)."""
        ms = ctypes.c_float(0.0)
        _check(lib().hj_plan_run(self._p, int(ncycles), ctypes.byref(ms) if timed else None), ok=(HJ_OK,))
        return ms.value if timed else None

    def solve(self, history=True):
        import torch
        dev = self._keep[0].device
        x = torch.empty(self.nx * self.ny, dtype=torch.float64, device=dev)
        cap = history_capacity(self.prm)
        hist = torch.empty(cap, dtype=torch.float64, device=dev) if history else None
        res = hj_result(_dptr(x), _dptr(hist), 0, 0, 0.0, 0.0, 0.0, 0.0)
        st = _check(lib().hj_plan_solve(self._p, ctypes.byref(res)),
                    ok=(HJ_OK, HJ_NOT_CONVERGED, HJ_ERR_NUMERIC))
        # the history is truncated at the capacity (include/hj.h)
        return _result(res, st, x.view(self.ny, self.nx) if self.dim == 2 or self.ny > 1 else x,
                       None if hist is None else hist[: min(res.cycles + 1, cap)])

    def kernel_kind(self) -> str:
        return KERNEL_KINDS.get(lib().hj_plan_kernel_kind(self._p), "?")

    def launches_per_cycle(self):
        return lib().hj_plan_launches_per_cycle(self._p)

    def close(self):
        if self._p:
            lib().hj_plan_destroy(self._p)
            self._p = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DistPlan(Plan):
    """hj_plan_create_dist: this rank's row slab [row_begin, row_end) of a 2D grid (device
    tensors f, x0 of the local rows; bc the full ring).  Collective over all ranks."""

    def __init__(self, nx, ny, h, f, bc, x0, *, rank, nranks, nccl_id: bytes, row_begin, row_end,
                 stream=None, stencil=None, **params):
        self._dist_args = (rank, nranks, nccl_id, row_begin, row_end)
        self.ny_global = ny
        # the problem handed to the C-ABI carries the GLOBAL ny; solve() views the local rows
        super().__init__(2, nx, row_end - row_begin, h, f, bc, x0, stream=stream, stencil=stencil,
                         **params)

    def _create(self, pb):
        rank, nranks, nccl_id, rb, re = self._dist_args
        pb.ny = self.ny_global
        self._idbuf = ctypes.create_string_buffer(nccl_id, 128)
        d = hj_dist(rank, nranks, ctypes.cast(self._idbuf, ctypes.c_char_p), rb, re)
        _check(lib().hj_plan_create_dist(ctypes.byref(pb), ctypes.byref(self.prm), ctypes.byref(d),
                                         self.stream, ctypes.byref(self._p)), ok=(HJ_OK,))


PEER_HANDLE_BYTES = 512   # HJ_PEER_HANDLE_BYTES


class PeerPlan(Plan):
    """hj_plan_create_peer: this rank's row slab with the peer-memory transport (CUDA IPC; the
    halo rows, residual row sums and per-cycle signals are stored by the library's kernels into
    the other ranks' buffers — no NCCL).  After construction call ``connect()`` on every rank
    (``allgather(bytes) -> list[bytes]`` in rank order; default: torch.distributed)."""

    def __init__(self, nx, ny, h, f, bc, x0, *, rank, nranks, row_begin, row_end, stream=None,
                 stencil=None, **params):
        self._dist_args = (rank, nranks, row_begin, row_end)
        self.ny_global = ny
        super().__init__(2, nx, row_end - row_begin, h, f, bc, x0, stream=stream, stencil=stencil,
                         **params)

    def _create(self, pb):
        rank, nranks, rb, re = self._dist_args
        pb.ny = self.ny_global
        d = hj_dist(rank, nranks, None, rb, re)
        _check(lib().hj_plan_create_peer(ctypes.byref(pb), ctypes.byref(self.prm), ctypes.byref(d),
                                         self.stream, ctypes.byref(self._p)), ok=(HJ_OK,))

    def export(self) -> bytes:
        buf = ctypes.create_string_buffer(PEER_HANDLE_BYTES)
        _check(lib().hj_plan_peer_export(self._p, buf), ok=(HJ_OK,))
        return buf.raw

    def attach(self, blobs):
        """blobs: every rank's export() in rank order.  Collective (runs the initial exchange)."""
        allb = b"".join(bytes(b) for b in blobs)
        if len(allb) != PEER_HANDLE_BYTES * self._dist_args[1]:
            raise ValueError("attach needs one blob per rank")
        buf = ctypes.create_string_buffer(allb, len(allb))
        _check(lib().hj_plan_peer_attach(self._p, buf), ok=(HJ_OK,))
        self.launches_per_cycle_static = lib().hj_plan_launches_per_cycle(self._p)

    def connect(self, allgather=None):
        if allgather is None:
            import torch.distributed as dist
            def allgather(b):
                out = [None] * dist.get_world_size()
                dist.all_gather_object(out, b)
                return out
        self.attach(allgather(self.export()))
