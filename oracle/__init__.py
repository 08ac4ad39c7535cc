"""CPU oracle for the hierarchical Jacobi solver — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2006_16465_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle/hjo.cpp`` (plain single-threaded C++, built with
``-O2 -ffp-contract=off``); this module only builds it on demand and marshals
numpy arrays through ctypes.  Every function cites the PAPER.md passage it
follows in ``hjo.cpp``.

Parity status: pinned by tests/test_oracle_pins.py against
closed forms (cos(pi h) decay, discrete exact solutions, direct solves,
brute-force dense cycle matrices, the paper's printed resource figures) —
and, for the exact iterates of the hierarchical schedule with k>1 on many tiles
(no closed form), through limits (k=1, one tile), brute force at tiny sizes, an
independent vectorised NumPy re-implementation matched bit for bit
(tests/test_oracle_vectorized.py), structure (halo locality, order independence)
and cross-implementation cycle counts.  The multigrid V-cycle is pinned in
tests/test_oracle_mg.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hjo.cpp")
_LIB = os.path.join(_HERE, "libhjo.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle/hjo.cpp into oracle/libhjo.so (g++)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
            P = ctypes.c_void_p
            lib.hjo_solve.restype = i32
            lib.hjo_solve.argtypes = [i32, i64, i64, d, P, P, P, P, i32, i32, i64, i64, i64, i64, i32,
                                      d, i32, d, i64, i32, P, P, ctypes.POINTER(i64),
                                      ctypes.POINTER(i32)]
            lib.hjo_block_plan.restype = i64
            lib.hjo_block_plan.argtypes = [i64, i64, i64, i64, P, P, P, P]
            lib.hjo_residual.restype = d
            lib.hjo_residual.argtypes = [i32, i64, i64, d, P, P, P]
            lib.hjo_residual_general.restype = d
            lib.hjo_residual_general.argtypes = [i32, i64, i64, P, P, P, P]
            lib.hjo_solve_mg.restype = i32
            lib.hjo_solve_mg.argtypes = [i32, i64, i64, d, P, P, P, i32, i64, i64, i32, i32, i32, d, i32,
                                         i32, d, i32, d, i64, P, P, ctypes.POINTER(i64),
                                         ctypes.POINTER(i32), ctypes.POINTER(i32)]
            lib.hjo_mg_transfer.restype = i64
            lib.hjo_mg_transfer.argtypes = [i32, i32, i64, i64, P, P, P, P]
            lib.hjo_resource_figures.restype = i32
            lib.hjo_resource_figures.argtypes = [i32, i64, i64, i64, i64, i64, i64, i64,
                                                 ctypes.POINTER(i64), ctypes.POINTER(i64),
                                                 ctypes.POINTER(i64)]
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a, n, name):
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if a.size != n:
        raise ValueError(f"{name}: expected {n} values, got {a.size}")
    return a


def solve(dim, nx, ny, h, f, bc=None, x0=None, *, mode="hier", dtype="f64", tile=(32, 32), k=16,
          overlap=0, tol=1e-4, tol_mode="rel", ref_residual=0.0, max_cycles=10**7, tile_order=0,
          history=True, stencil=None):
    """Run the oracle solver.  Returns dict(x, history, cycles, converged, status).

    ``x`` has shape (ny, nx) in 2D and (nx,) in 1D; ``history[c]`` = ||f - A x_c||_2.
    ``stencil`` (general coefficients, reading c23): 2D {a, c, e, f, d} (Eq. 10), 1D the planes
    [a | d | c] of nx*ny values each (Eq. 4); ``f`` is then b and ``h`` is unused.
    ``max_cycles`` cycles are run if ``tol`` is never met (``tol=0`` runs exactly
    ``max_cycles`` cycles unless the residual is exactly zero).
    """
    lib = _load()
    n = nx * ny
    f = _f64(f, n, "f")
    nbc = 2 * ny if dim == 1 else 2 * nx + 2 * ny   # dim 1: ny independent problems
    bc = _f64(bc, nbc, "bc")
    x0 = _f64(x0, n, "x0")
    if stencil is not None:
        stencil = _f64(stencil, 3 * n if dim == 1 else 5, "stencil")
    x = np.zeros(n, dtype=np.float64)
    hist = np.full(max_cycles + 1, np.nan) if history else None
    cyc = ctypes.c_int64(0)
    conv = ctypes.c_int(0)
    tx, ty = (tile if isinstance(tile, (tuple, list)) else (tile, 1))
    ox, oy = (overlap if isinstance(overlap, (tuple, list)) else (overlap, overlap if dim == 2 else 0))
    st = lib.hjo_solve(dim, nx, ny, float(h), _ptr(f), _ptr(bc), _ptr(x0), _ptr(stencil),
                       {"hier": 0, "classic": 1}[mode], {"f64": 0, "f32": 1}[dtype], tx, ty, ox, oy, k,
                       float(tol), {"rel": 0, "abs": 1}[tol_mode], float(ref_residual),
                       int(max_cycles), int(tile_order), _ptr(x), _ptr(hist),
                       ctypes.byref(cyc), ctypes.byref(conv))
    if st == 2:
        raise ValueError("oracle: invalid argument")
    c = cyc.value
    return dict(x=x.reshape((ny, nx)) if (dim == 2 or ny > 1) else x,
                history=None if hist is None else hist[: c + 1].copy(),
                cycles=c, converged=bool(conv.value), status=st)


def solve_mg(dim, nx, ny, h, f, bc=None, x0=None, *, dtype="f64", tile=(32, 32), k=4, nu1=1, nu2=1,
             omega=None, coarse_cycles=1, levels=0, tol=1e-6, tol_mode="rel", ref_residual=0.0,
             max_cycles=1000, history=True):
    """Multigrid V-cycles with the hierarchical cycle as smoother (DESIGN.md
    reading c24).  ``omega`` defaults to 4/5 (2D) and 2/3 (1D), the textbook smoothing weights
    of damped Jacobi.  Returns dict(x, history, cycles, converged, status, levels); one cycle =
    one V-cycle."""
    lib = _load()
    n = nx * ny
    f = _f64(f, n, "f")
    bc = _f64(bc, 2 * ny if dim == 1 else 2 * nx + 2 * ny, "bc")
    x0 = _f64(x0, n, "x0")
    if omega is None:
        omega = 0.8 if dim == 2 else 2.0 / 3.0
    x = np.zeros(n, dtype=np.float64)
    hist = np.full(max_cycles + 1, np.nan) if history else None
    cyc, conv, lev = ctypes.c_int64(0), ctypes.c_int(0), ctypes.c_int(0)
    tx, ty = (tile if isinstance(tile, (tuple, list)) else (tile, 1))
    st = lib.hjo_solve_mg(dim, nx, ny, float(h), _ptr(f), _ptr(bc), _ptr(x0), {"f64": 0, "f32": 1}[dtype],
                          tx, ty, k, nu1, nu2, float(omega), coarse_cycles, levels, float(tol),
                          {"rel": 0, "abs": 1}[tol_mode], float(ref_residual), int(max_cycles), _ptr(x),
                          _ptr(hist), ctypes.byref(cyc), ctypes.byref(conv), ctypes.byref(lev))
    if st == 2:
        raise ValueError("oracle: invalid argument")
    c = cyc.value
    return dict(x=x.reshape((ny, nx)) if (dim == 2 or ny > 1) else x,
                history=None if hist is None else hist[: c + 1].copy(),
                cycles=c, converged=bool(conv.value), status=st, levels=lev.value)


def mg_transfer(dim, op, nx, ny, x, a, bc=None):
    """The multigrid transfer steps alone (double): op "restrict" -> coarse h2f = 4 R s of the fine
    iterate x with rhs a (= h^2 f; s = a - stencil(x)); op "correct" -> x + P a for the coarse
    interior a.  1D: ny independent problems."""
    lib = _load()
    x = _f64(x, nx * ny, "x")
    bc = _f64(bc, 2 * ny if dim == 1 else 2 * nx + 2 * ny, "bc")
    nxc, nyc = (nx - 1) // 2, ((ny - 1) // 2 if dim == 2 else ny)
    if op == "restrict":
        a = _f64(a, nx * ny, "a")
        out = np.zeros(nxc * nyc)
    else:
        a = _f64(a, nxc * nyc, "a")
        out = np.zeros(nx * ny)
    w = lib.hjo_mg_transfer(dim, 0 if op == "restrict" else 1, nx, ny, _ptr(x), _ptr(bc), _ptr(a), _ptr(out))
    if w < 0:
        raise ValueError("oracle: invalid transfer")
    return out


def residual(dim, nx, ny, h, f, bc, x):
    """||f - A x||_2 (unscaled, A = stencil / h^2) of an interior iterate x."""
    lib = _load()
    n = nx * ny
    f = _f64(f, n, "f")
    x = _f64(x, n, "x")
    bc = _f64(bc, 2 * ny if dim == 1 else 2 * nx + 2 * ny, "bc")
    return lib.hjo_residual(dim, nx, ny, float(h), _ptr(f), _ptr(bc), _ptr(x))


def residual_general(dim, nx, ny, f, bc, x, stencil):
    """General-coefficient residual by its definition: 2D ||b - Ax||_2, 1D ||D^-1 (b - Ax)||_2."""
    lib = _load()
    n = nx * ny
    f = _f64(f, n, "f")
    x = _f64(x, n, "x")
    bc = _f64(bc, 2 * ny if dim == 1 else 2 * nx + 2 * ny, "bc")
    stencil = _f64(stencil, 3 * n if dim == 1 else 5, "stencil")
    return lib.hjo_residual_general(dim, nx, ny, _ptr(f), _ptr(bc), _ptr(x), _ptr(stencil))


def resource_figures(dim, nx, ny, tx, ty=1, bytes_per_value=8, overlap=0):
    """(tiles, threads, shared bytes per block by the paper's formula)."""
    lib = _load()
    ox, oy = (overlap if isinstance(overlap, (tuple, list)) else (overlap, overlap if dim == 2 else 0))
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    st = lib.hjo_resource_figures(dim, nx, ny, tx, ty, ox, oy, bytes_per_value, ctypes.byref(a),
                                  ctypes.byref(b), ctypes.byref(c))
    if st != 0:
        raise ValueError("oracle: invalid configuration")
    return a.value, b.value, c.value


def block_plan(n, tile, overlap=0):
    """Blocks of one dimension: list of (start, width, own_lo, own_hi), 1-based inclusive."""
    lib = _load()
    cap = n + 1
    arrs = [np.zeros(cap, dtype=np.int64) for _ in range(4)]
    nb = lib.hjo_block_plan(n, tile, overlap, cap, *[a.ctypes.data_as(ctypes.c_void_p) for a in arrs])
    if nb < 0:
        raise ValueError("oracle: invalid block plan")
    return [tuple(int(a[b]) for a in arrs) for b in range(nb)]
