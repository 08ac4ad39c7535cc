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


def plan_1d(n, T, o):
    """Blocks along one dimension written out by hand from the paper's rule (independent of the
    oracle's block_plan): o = 0 -> consecutive tiles, ragged last (reading c10); o > 0 -> starts
    1 + b(T-o), last block shifted to end at n, half-split ownership with the left block taking
    the odd extra point.  Returns [(lo, hi, own_lo, own_hi)]."""
    if o == 0:
        return [(s, min(s + T - 1, n), s, min(s + T - 1, n)) for s in range(1, n + 1, T)]
    starts = []
    s = 1
    while True:
        if s + T - 1 >= n:
            starts.append(n - T + 1)
            break
        starts.append(s)
        s += T - o
    blocks = [[st, st + T - 1, None, None] for st in starts]
    blocks[0][2], blocks[-1][3] = 1, n
    for a, b in zip(blocks, blocks[1:]):
        overlap = list(range(b[0], a[1] + 1))
        left = (len(overlap) + 1) // 2
        a[3] = overlap[left - 1]
        b[2] = overlap[left - 1] + 1
    return [tuple(x) for x in blocks]


def tiles(dim, nx, ny, tx, ty, ox=0, oy=0):
    """(interior points, owned points) of every block."""
    out = []
    px = plan_1d(nx, tx, ox)
    if dim == 1:
        for lo, hi, a0, a1 in px:
            out.append(([(i, 0) for i in range(lo, hi + 1)], [(i, 0) for i in range(a0, a1 + 1)]))
        return out
    py = plan_1d(ny, ty, oy)
    for ylo, yhi, b0, b1 in py:
        for xlo, xhi, a0, a1 in px:
            out.append(([(i, j) for j in range(ylo, yhi + 1) for i in range(xlo, xhi + 1)],
                        [(i, j) for j in range(b0, b1 + 1) for i in range(a0, a1 + 1)]))
    return out


def cycle_affine(dim, nx, ny, h, f, tx, ty, k, ox=0, oy=0):
    """Dense (M, g) with x_next_interior = M @ z_ringed + g (rows from the owning block)."""
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
    for T, owned in tiles(dim, nx, ny, tx, ty, ox, oy):
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
        for p in owned:
            M[out_pos[p]] = Mt[loc[p]]
            g[out_pos[p]] = gt[loc[p]]
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


def cycle_affine_general(dim, nx, ny, stencil, b, tx, ty, k, ox=0, oy=0):
    """(M, g) of one hierarchical cycle for the general coefficients (Eq. 4 / Eq. 10) with EXACT
    quotients: the Jacobi matrix of the tile is -D^-1 (offdiag) restricted to the tile, d_t = b/d."""
    if dim == 1:
        ny = 1
    nz = (nx + 2) if dim == 1 else (nx + 2) * (ny + 2)
    idx = ringed_index(nx, ny, dim)
    b = np.asarray(b, dtype=np.float64).reshape(-1)
    st = np.asarray(stencil, dtype=np.float64)

    def coef(i, j):  # [(neighbour, coefficient)], diagonal
        if dim == 1:
            a, d, c = st[i - 1], st[nx + i - 1], st[2 * nx + i - 1]
            return [((i - 1, 0), a), ((i + 1, 0), c)], d
        a, c, e, f, d = st
        return [((i - 1, j), a), ((i + 1, j), c), ((i, j - 1), e), ((i, j + 1), f)], d

    interior = [(i, 0) for i in range(1, nx + 1)] if dim == 1 else \
        [(i, j) for j in range(1, ny + 1) for i in range(1, nx + 1)]
    out_pos = {p: q for q, p in enumerate(interior)}
    M = np.zeros((len(interior), nz))
    g = np.zeros(len(interior))
    for T, owned in tiles(dim, nx, ny, tx, ty, ox, oy):
        loc = {p: q for q, p in enumerate(T)}
        w = len(T)
        J, B, d_t, E = np.zeros((w, w)), np.zeros((w, nz)), np.zeros(w), np.zeros((w, nz))
        for q, (i, j) in enumerate(T):
            E[q, idx(i, j)] = 1.0
            nb, dd = coef(i, j)
            d_t[q] = b[out_pos[(i, j)]] / dd
            for (ii, jj), cc in nb:
                if (ii, jj) in loc:
                    J[q, loc[(ii, jj)]] += -cc / dd
                else:
                    B[q, idx(ii, jj)] += -cc / dd
        S = np.zeros((w, w))
        Jp = np.eye(w)
        for _ in range(k):
            S += Jp
            Jp = Jp @ J
        Mt = Jp @ E + S @ B
        gt = S @ d_t
        for p in owned:
            M[out_pos[p]] = Mt[loc[p]]
            g[out_pos[p]] = gt[loc[p]]
    return M, g


def general_matrix(dim, nx, ny, stencil):
    """Dense A of Eq. 4 (1D, one problem) / Eq. 10 (2D) on the interior unknowns."""
    st = np.asarray(stencil, dtype=np.float64)
    if dim == 1:
        a, d, c = st[:nx], st[nx:2 * nx], st[2 * nx:]
        return np.diag(d) + np.diag(a[1:], -1) + np.diag(c[:-1], 1)
    a, c, e, f, d = st
    n = nx * ny
    A = np.zeros((n, n))
    for j in range(ny):
        for i in range(nx):
            r = j * nx + i
            A[r, r] = d
            if i > 0: A[r, r - 1] = a
            if i < nx - 1: A[r, r + 1] = c
            if j > 0: A[r, r - nx] = e
            if j < ny - 1: A[r, r + nx] = f
    return A


def general_rhs(dim, nx, ny, stencil, b, bc):
    """b with the Dirichlet ring moved to the right-hand side."""
    st = np.asarray(stencil, dtype=np.float64)
    rhs = np.asarray(b, dtype=np.float64).reshape(-1).copy()
    if bc is None:
        return rhs
    if dim == 1:
        rhs[0] -= st[0] * bc[0]
        rhs[-1] -= st[3 * nx - 1] * bc[1]
        return rhs
    a, c, e, f, d = st
    r = rhs.reshape(ny, nx)
    r[0, :] -= e * bc[:nx]
    r[-1, :] -= f * bc[nx:2 * nx]
    r[:, 0] -= a * bc[2 * nx:2 * nx + ny]
    r[:, -1] -= c * bc[2 * nx + ny:]
    return r.reshape(-1)


# ------------------------------------------------------------------ multigrid (NEXT #4) -----
# Dense, matrix-level constructions of the textbook V-cycle (Briggs et al., the reference of
# PAPER.md:17) with the hierarchical damped-Jacobi smoother, written from the definitions of
# DESIGN.md reading c24 — none of the oracle's loops.  Everything is in the h^2-scaled form:
# level l solves K_l z = b_l (K = the 5-/3-point stencil with 4 / 2 on the diagonal, z ringed).

def smoother_affine(dim, nx, ny, tx, ty, k, omega):
    """(M, G) with x_next = M z + G b for one hierarchical cycle of DAMPED Jacobi (b = h^2 f on
    the interior, z the ringed snapshot): per tile u <- J_w u + w (B z + D^-1 b), J_w = (1-w) I + w J."""
    if dim == 1:
        ny = 1
    nz = (nx + 2) if dim == 1 else (nx + 2) * (ny + 2)
    idx = ringed_index(nx, ny, dim)
    dinv = 0.5 if dim == 1 else 0.25
    interior = [(i, 0) for i in range(1, nx + 1)] if dim == 1 else \
        [(i, j) for j in range(1, ny + 1) for i in range(1, nx + 1)]
    pos = {p: q for q, p in enumerate(interior)}
    n = len(interior)
    M = np.zeros((n, nz))
    G = np.zeros((n, n))
    for T, owned in tiles(dim, nx, ny, tx, ty):
        loc = {p: q for q, p in enumerate(T)}
        w = len(T)
        J, B, E, D = np.zeros((w, w)), np.zeros((w, nz)), np.zeros((w, nz)), np.zeros((w, n))
        for q, (i, j) in enumerate(T):
            E[q, idx(i, j)] = 1.0
            D[q, pos[(i, j)]] = dinv
            for (ii, jj) in neighbours(dim, i, j):
                if (ii, jj) in loc:
                    J[q, loc[(ii, jj)]] += dinv
                else:
                    B[q, idx(ii, jj)] += dinv
        Jw = (1.0 - omega) * np.eye(w) + omega * J
        S = np.zeros((w, w))
        Jp = np.eye(w)
        for _ in range(k):
            S += Jp
            Jp = Jp @ Jw
        Mt = Jp @ E + omega * (S @ B)
        Gt = omega * (S @ D)
        for p in owned:
            M[pos[p]] = Mt[loc[p]]
            G[pos[p]] = Gt[loc[p]]
    return M, G


def stencil_ringed(dim, nx, ny):
    """K (interior x ringed): (K z)_p = diag z_p - sum of the neighbours (ring included)."""
    if dim == 1:
        ny = 1
    idx = ringed_index(nx, ny, dim)
    interior = [(i, 0) for i in range(1, nx + 1)] if dim == 1 else \
        [(i, j) for j in range(1, ny + 1) for i in range(1, nx + 1)]
    nz = (nx + 2) if dim == 1 else (nx + 2) * (ny + 2)
    K = np.zeros((len(interior), nz))
    for q, (i, j) in enumerate(interior):
        K[q, idx(i, j)] = 2.0 if dim == 1 else 4.0
        for (ii, jj) in neighbours(dim, i, j):
            K[q, idx(ii, jj)] -= 1.0
    return K


def full_weighting(dim, nx, ny):
    """R (coarse x fine interior): 1D (1/4)[1 2 1], 2D (1/16)[1 2 1; 2 4 2; 1 2 1] centred on the
    fine point 2I (1-based ringed), the standard full-weighting operator."""
    nxc = (nx - 1) // 2
    if dim == 1:
        R = np.zeros((nxc, nx))
        for I in range(1, nxc + 1):
            for di, w in ((-1, 0.25), (0, 0.5), (1, 0.25)):
                R[I - 1, 2 * I + di - 1] = w
        return R
    nyc = (ny - 1) // 2
    R = np.zeros((nxc * nyc, nx * ny))
    w1 = {-1: 0.25, 0: 0.5, 1: 0.25}
    for J in range(1, nyc + 1):
        for I in range(1, nxc + 1):
            for dj in (-1, 0, 1):
                for di in (-1, 0, 1):
                    R[(J - 1) * nxc + I - 1, (2 * J + dj - 1) * nx + (2 * I + di - 1)] = w1[di] * w1[dj]
    return R


def linear_interpolation(dim, nx, ny):
    """P (fine x coarse interior): (bi)linear interpolation with zero coarse ring; P = 2^dim R^T."""
    return (2.0 ** dim) * full_weighting(dim, nx, ny).T


def mg_sizes(n):
    s = [n]
    while s[-1] >= 3 and s[-1] % 2 == 1:
        s.append((s[-1] - 1) // 2)
    return s


def vcycle_dense(dim, nx, ny, tile, k, nu1, nu2, omega, coarse_cycles):
    """Return V(x, b, ring) -> x_next: one V-cycle on the interior x of level 0 (b = h^2 f, ring =
    the ringed vector's ring values as a ringed array with zero interior), built from dense
    smoother maps, K, R and P of every level."""
    sx = mg_sizes(nx)
    sy = mg_sizes(ny) if dim == 2 else [1] * len(sx)
    L = min(len(sx), len(sy))
    lev = []
    for l in range(L):
        n1, n2 = sx[l], sy[l]
        t = (min(tile[0], n1), min(tile[1], n2) if dim == 2 else 1)
        Mw, Gw = smoother_affine(dim, n1, n2, t[0], t[1], k, omega)
        M1, G1 = smoother_affine(dim, n1, n2, t[0], t[1], k, 1.0)
        lev.append(dict(nx=n1, ny=n2, Mw=Mw, Gw=Gw, M1=M1, G1=G1, K=stencil_ringed(dim, n1, n2)))
    for l in range(L - 1):
        lev[l]["R"] = full_weighting(dim, lev[l]["nx"], lev[l]["ny"])
        lev[l]["P"] = linear_interpolation(dim, lev[l]["nx"], lev[l]["ny"])

    def ringed(l, x, ring):
        z = ring.copy()
        d = lev[l]
        if dim == 1:
            z[1:-1] = x
        else:
            z.reshape(d["ny"] + 2, d["nx"] + 2)[1:-1, 1:-1] = x.reshape(d["ny"], d["nx"])
        return z

    def V(l, x, b, ring):
        d = lev[l]
        if l == L - 1:
            for _ in range(coarse_cycles):
                x = d["M1"] @ ringed(l, x, ring) + d["G1"] @ b
            return x
        for _ in range(nu1):
            x = d["Mw"] @ ringed(l, x, ring) + d["Gw"] @ b
        s = b - d["K"] @ ringed(l, x, ring)
        c = lev[l + 1]
        nzc = (c["nx"] + 2) * ((c["ny"] + 2) if dim == 2 else 1)
        e = V(l + 1, np.zeros(c["nx"] * (c["ny"] if dim == 2 else 1)), 4.0 * (d["R"] @ s), np.zeros(nzc))
        x = x + d["P"] @ e
        for _ in range(nu2):
            x = d["Mw"] @ ringed(l, x, ring) + d["Gw"] @ b
        return x

    return V, L
