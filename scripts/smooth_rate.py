"""Analysis (not product code, not the oracle): the asymptotic per-cycle contraction of the hierarchical
cycle (32x32 tiles, k = 16 sub-iterations with the tile's halo frozen) on the
SMOOTHEST error mode of an n x n Dirichlet grid, by power iteration of the homogeneous cycle (f = 0,
g = 0) started from sin(pi x) sin(pi y): r(n) = -ln(||e_{c+1}|| / ||e_c||) once the ratio settles.
Classic Jacobi contracts that mode by cos(pi h) per sweep, so kappa = r / (-ln cos(pi h)) is the number
of classic sweeps one cycle is worth on it.  Used to bound the cycles the 16384^2 time-to-1e-6 solve still
needs after its measured trajectory (profiles/r02_ttt_1e-6_16384_partial.json).
    python scripts/smooth_rate.py 2048 4096 8192 [cycles]"""
import math
import sys

import numpy as np

T, K = 32, 16


def cycle(x, n):
    """One hierarchical cycle of the homogeneous problem on the interior x (n x n, zero ring)."""
    nt = n // T
    X = np.zeros((n + 2, n + 2))
    X[1:-1, 1:-1] = x
    t = np.empty((nt, nt, T + 2, T + 2))
    for a in range(T + 2):  # tile (ty, tx) row a = padded row ty*T + a
        t[:, :, a, :] = np.lib.stride_tricks.as_strided(
            X[a:], shape=(nt, nt, T + 2), strides=(T * X.strides[0], T * X.strides[1], X.strides[1]))
    for _ in range(K):  # Jacobi on every tile's interior, its ring (the halo) frozen
        t[:, :, 1:-1, 1:-1] = 0.25 * ((t[:, :, 1:-1, :-2] + t[:, :, 1:-1, 2:]) + (t[:, :, :-2, 1:-1] + t[:, :, 2:, 1:-1]))
    return t[:, :, 1:-1, 1:-1].transpose(0, 2, 1, 3).reshape(n, n)


def rate(n, cycles):
    h = 1.0 / (n + 1)
    s = np.sin(math.pi * h * np.arange(1, n + 1))
    x = np.outer(s, s)
    prev = np.linalg.norm(x)
    out = []
    for c in range(cycles):
        x = cycle(x, n)
        nr = np.linalg.norm(x)
        out.append(-math.log(nr / prev))
        x /= nr  # keep the scale
        prev = 1.0
    sweep = -math.log(math.cos(math.pi * h))
    return out, sweep


if __name__ == "__main__":
    args = [int(a) for a in sys.argv[1:]] or [2048, 4096]
    cyc = 12
    if len(args) > 1 and args[-1] < 256:
        cyc = args.pop()
    for n in args:
        r, sw = rate(n, cyc)
        print(f"n={n}: per-cycle rate {r[-1]:.6e} (last 3: {', '.join(f'{v:.6e}' for v in r[-3:])}); "
              f"classic sweep {sw:.6e}; kappa = {r[-1] / sw:.4f} sweeps per cycle", flush=True)
