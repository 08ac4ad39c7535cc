"""Brute-force dense constructions used to PIN the oracle (tiny grids only).

Nothing here calls or copies the oracle's loops.  The hierarchical cycle is
built as an explicit affine map on the ringed snapshot vector z:

    x_next = M z + g

from per-tile local Jacobi matrices: for tile t with
interior node set I_t, the local iteration is u <- J_t u + B_t z + d_t (J_t the
Jacobi matrix D^-1 (D - A) restricted to I_t, B_t the coupling to the frozen
halo nodes, d_t = D^-1 b on I_t), so after k sub-iterations starting from
u_0 = E_t z:
    u_k = J_t^k E_t z + sum_{j<k} J_t^j (B_t z + d_t).
Nodes are numbered on the ringed grid: (i, j) -> j*(nx+2) + i, ring included.
"""
from __future__ import annotations

import numpy as np


def ringed_index(nx, ny, dim):
    if dim == 1:
        return lambda i, j=0: i
    return lambda i, j: j * (nx + 2) + i


def neighbours(dim, i, j):
    if dim == 1:
        return [(i - 1, 0), (i + 1, 0)]
    return [(i - 1, j), (i + 1, j), (i, j - 1), (i, j + 1)]


def tiles(dim, nx, ny, tx, ty):
    """Interior index ranges of the o=0 tiles, ragged last tile (reading c10)."""
    out = []
    if dim == 1:
        for a in range((nx + tx - 1) // tx):
            out.append([(i, 0) for i in range(1 + a * tx, min((a + 1) * tx, nx) + 1)])
        return out
    for b in range((ny + ty - 1) // ty):
        for a in range((nx + tx - 1) // tx):
            out.append([(i, j) for j in range(1 + b * ty, min((b + 1) * ty, ny) + 1)
                        for i in range(1 + a * tx, min((a + 1) * tx, nx) + 1)])
    return out


def cycle_affine(dim, nx, ny, h, f, tx, ty, k):
    """Dense (M, g) with x_next_interior = M @ z_ringed + g  (o = 0)."""
    if dim == 1:
        ny = 1
    nz = (nx + 2) if dim == 1 else (nx + 2) * (ny + 2)
    idx = ringed_index(nx, ny, dim)
    diag_inv = 0.5 if dim == 1 else 0.25          # 1/a_ii for the h^2-scaled stencil
    b = (h * h) * np.asarray(f, dtype=np.float64).reshape(-1)
    interior = [(i, 0) for i in range(1, nx + 1)] if dim == 1 else \
        [(i, j) for j in range(1, ny + 1) for i in range(1, nx + 1)]
    out_pos = {p: q for q, p in enumerate(interior)}
    M = np.zeros((len(interior), nz))
    g = np.zeros(len(interior))
    for T in tiles(dim, nx, ny, tx, ty):
        loc = {p: q for q, p in enumerate(T)}
        w = len(T)
        J = np.zeros((w, w))
        B = np.zeros((w, nz))
        d = np.zeros(w)
        E = np.zeros((w, nz))
        for q, (i, j) in enumerate(T):
            E[q, idx(i, j)] = 1.0
            d[q] = diag_inv * b[out_pos[(i, j)]]
            for (ii, jj) in neighbours(dim, i, j):
                if (ii, jj) in loc:
                    J[q, loc[(ii, jj)]] += diag_inv
                else:
                    B[q, idx(ii, jj)] += diag_inv   # frozen halo (or Dirichlet ring) node
        Mt = np.linalg.matrix_power(J, k) @ E
        S = np.zeros((w, w))
        Jp = np.eye(w)
        for _ in range(k):
            S += Jp
            Jp = Jp @ J
        Mt += S @ B
        gt = S @ d
        for q, p in enumerate(T):
            M[out_pos[p]] = Mt[q]
            g[out_pos[p]] = gt[q]
    return M, g, interior, idx


def ringed_vector(dim, nx, ny, bc, x):
    """Assemble z (ringed snapshot) from interior x and ring data bc."""
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    if dim == 1:
        z = np.zeros(nx + 2)
        z[1:-1] = x
        if bc is not None:
            z[0], z[-1] = bc[0], bc[1]
        return z
    z = np.zeros((ny + 2, nx + 2))
    z[1:-1, 1:-1] = x.reshape(ny, nx)
    if bc is not None:
        z[0, 1:-1] = bc[:nx]
        z[-1, 1:-1] = bc[nx:2 * nx]
        z[1:-1, 0] = bc[2 * nx:2 * nx + ny]
        z[1:-1, -1] = bc[2 * nx + ny:]
    return z.reshape(-1)


def poisson_matrix(dim, nx, ny=1):
    """Sparse h^2-scaled Poisson matrix (2 on the diagonal in 1D, 4 in 2D)."""
    import scipy.sparse as sp
    T1 = sp.diags([-np.ones(nx - 1), 2 * np.ones(nx), -np.ones(nx - 1)], [-1, 0, 1])
    if dim == 1:
        return T1.tocsr()
    Ty = sp.diags([-np.ones(ny - 1), 2 * np.ones(ny), -np.ones(ny - 1)], [-1, 0, 1])
    return (sp.kron(sp.identity(ny), T1) + sp.kron(Ty, sp.identity(nx))).tocsr()


def direct_solve(dim, nx, ny, h, f, bc=None):
    """x* of the discrete Dirichlet problem by a sparse direct solve (scipy)."""
    import scipy.sparse.linalg as spla
    A = poisson_matrix(dim, nx, ny)
    rhs = (h * h) * np.asarray(f, dtype=np.float64).reshape(-1).copy()
    if bc is not None:
        if dim == 1:
            rhs[0] += bc[0]
            rhs[-1] += bc[1]
        else:
            r = rhs.reshape(ny, nx)
            r[0, :] += bc[:nx]
            r[-1, :] += bc[nx:2 * nx]
            r[:, 0] += bc[2 * nx:2 * nx + ny]
            r[:, -1] += bc[2 * nx + ny:]
            rhs = r.reshape(-1)
    return spla.spsolve(A.tocsc(), rhs)
