import numpy as np


def example_6x6(sp):
    """tests/oracles.hpp:53-62."""
    return sp.CsrMatrix.from_dense([[4, -2, 0, 0, 1, 0], [-2, 4, 1, 0, 0, 0], [0, 1, 4, 1, 2, 0],
                                    [0, 0, 1, 4, 0, 2], [1, 0, 2, 0, 4, 0], [0, 0, 0, 2, 0, 4]])


def from_npz(sp, d):
    return sp.CsrMatrix(len(d["rp"]) - 1, len(d["rp"]) - 1, d["rp"], d["ci"], d["v"])


def random_vector(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def random_spd(sp, n, seed, density=0.2):
    """Symmetric diagonally dominant (tests/oracles.hpp:126-147 analogue)."""
    rng = np.random.default_rng(seed)
    a = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < density:
                v = -rng.uniform(0.1, 2.0)
                a[i, j] = a[j, i] = v
    for i in range(n):
        a[i, i] = np.abs(a[i]).sum() + rng.uniform(0.5, 1.5)
    return sp.CsrMatrix.from_dense(a)


def random_sparse(sp, n, seed, density=0.2, mirror=True):
    """tests/oracles.hpp:101-122 analogue (nonzero diagonal n + U[0.1, 2])."""
    rng = np.random.default_rng(seed)
    a = np.zeros((n, n))
    for i in range(n):
        a[i, i] = n + rng.uniform(0.1, 2.0)
        for j in range(i + 1, n):
            if rng.random() < density:
                v = rng.uniform(0.1, 2.0) * (1 if rng.random() < 0.5 else -1)
                a[i, j] = v
                a[j, i] = v if mirror else rng.uniform(0.1, 2.0) * (1 if rng.random() < 0.5 else -1)
    return sp.CsrMatrix.from_dense(a)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def stencil27_varied(sp, nx, ny, nz, seed=0):
    """27-point operator on an nx*ny*nz grid whose 26 off-diagonal values differ by
    direction (and the diagonal dominates), neighbours outside the grid dropped."""
    rng = np.random.default_rng(seed)
    w = -rng.uniform(0.5, 1.5, (3, 3, 3))
    w[1, 1, 1] = 30.0
    n = nx * ny * nz
    iz, iy, ix = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    rows, cols, vals = [], [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                jx, jy, jz = ix + dx, iy + dy, iz + dz
                ok = (jx >= 0) & (jx < nx) & (jy >= 0) & (jy < ny) & (jz >= 0) & (jz < nz)
                rows.append(((iz * ny + iy) * nx + ix)[ok])
                cols.append(((jz * ny + jy) * nx + jx)[ok])
                vals.append(np.full(ok.sum(), w[dz + 1, dy + 1, dx + 1]))
    r, c, v = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, r + 1, 1)
    return sp.CsrMatrix(n, n, np.cumsum(rp), c.astype(np.int32), v)
