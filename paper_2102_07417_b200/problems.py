"""Synthetic workloads for the five BASELINE configs (host-side input producers).

These build the level-0 operator and right-hand side; they are not on the
solve path.  Node order is x fastest, then y, then z, exactly as the
reference generators (``amgkit/problems.py:27-33``), and every operator comes
out as canonical CSR (ascending unique columns per row, no stored zeros), the
same storage ``SparseMatrix.from_coo`` produces (``amgkit/sparse.py:149-156``).

* config 1 -- ``poisson7(64, 64, 64)``: restates ``gen_poisson7``
  (``amgkit/problems.py:48-52``): diagonal 6, face neighbours -1.
* config 2 / 5 -- ``hetero27``: 26-neighbour diffusion with a per-cell
  lognormal conductivity; this generator is not in the reference (its
  ``gen_heterogeneous`` is 2-D 5-point only, ``problems.py:202-237``), so the
  definition is pinned here:
  offset weight w = 1/|o|^2 (1, 1/2, 1/3); coupling
  c_ij = w * 2 k_i k_j / (k_i + k_j) (harmonic mean); k = exp(sigma * N(0,1))
  per cell from ``default_rng(seed)`` (or per ``block``^3 cell block);
  an eliminated Dirichlet neighbour adds w * k_i to the diagonal, following
  ``gen_heterogeneous``'s convention (``problems.py:223-231``).
* config 3 -- ``elasticity3d``: trilinear Q1 hexahedra on the unit cube
  (element size h = 1/n), 3 dofs per node, node-major xyz dof order, the
  x = 0 face clamped (its dofs eliminated) -- restating
  ``gen_elasticity3d`` / ``hex_element_stiffness``
  (``amgkit/problems.py:91-199``) with a per-element Young's modulus
  E_e = exp(sigma * N(0,1)) from ``default_rng(seed)`` (sigma = 1) and
  nu = 0.3; K_e = E_e * h * K_unit (3-D elasticity scales linearly in h).
  RHS: body load (0, 0, -1) per node times the nodal volume h^3, times
  (1 + 0.01 N(0,1)) per dof from ``default_rng(seed + 1)``.
* config 4 -- ``rtanis7``: ``gen_rotated_anisotropy(nx, ny, nz, theta=0,
  kx=1, ky=1, kz=eps)`` (``problems.py:62-88``); with theta = 0 the cross
  terms vanish exactly and are eliminated, leaving a 7-point stencil with
  diagonal 2 (kx + ky + kz).

RHS for every scalar config: ``default_rng(seed).uniform(-1, 1, n)``.
"""
from __future__ import annotations

import numpy as np

__all__ = ["Csr", "poisson7", "rtanis7", "hetero27", "elasticity3d", "hex_stiffness", "rhs_uniform", "rhs_body_load",
           "build_config", "build_rhs", "CONFIGS"]


class Csr:
    """Plain CSR triple with the reference dtypes (int64 / int32 / float64)."""

    __slots__ = ("nrows", "ncols", "row_offsets", "col_indices", "values")

    def __init__(self, nrows, ncols, row_offsets, col_indices, values):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(col_indices, dtype=np.int32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)

    @property
    def nnz(self):
        return int(self.col_indices.size)

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def as_tuple(self):
        """(nrows, ncols, row_offsets, col_indices, values): ``amgkit.SparseMatrix``'s positional arguments."""
        return (self.nrows, self.ncols, self.row_offsets, self.col_indices, self.values)

    def __repr__(self):
        return f"Csr({self.nrows}x{self.ncols}, nnz={self.nnz})"


def _offsets27():
    # lexicographic (dz, dy, dx): for a fixed row this is ascending column order
    return [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


def _assemble(nx, ny, nz, offsets, coupling, diag_fn, chunk_planes=16):
    """Assemble a stencil operator directly into sorted CSR, z-slab by z-slab.

    ``offsets`` is a list of (dx, dy, dz) in ascending column order, the
    centre (0, 0, 0) included; ``coupling(k0, k1, o, idx, nbr, inside)``
    returns the (positive) off-diagonal conductance for the slab and
    ``diag_fn(diag_acc, idx)`` finalises the diagonal.
    Couplings that are exactly zero are dropped (eliminated), as
    ``from_coo``'s ``eliminate_zeros`` does.
    """
    n = nx * ny * nz
    plane = nx * ny
    counts = np.zeros(n, dtype=np.int64)
    col_parts, val_parts = [], []
    for z0 in range(0, nz, chunk_planes):
        z1 = min(nz, z0 + chunk_planes)
        idx = np.arange(z0 * plane, z1 * plane, dtype=np.int64)
        ii = idx % nx
        jj = (idx // nx) % ny
        kk = idx // plane
        m = idx.size
        cols = np.empty((len(offsets), m), dtype=np.int64)
        vals = np.empty((len(offsets), m), dtype=np.float64)
        keep = np.zeros((len(offsets), m), dtype=bool)
        diag = np.zeros(m)
        centre = None
        for t, (dx, dy, dz) in enumerate(offsets):
            if dx == 0 and dy == 0 and dz == 0:
                centre = t
                continue
            ni, nj, nk = ii + dx, jj + dy, kk + dz
            inside = (0 <= ni) & (ni < nx) & (0 <= nj) & (nj < ny) & (0 <= nk) & (nk < nz)
            nbr = ni + nx * (nj + ny * nk)
            c = coupling((dx, dy, dz), idx, np.where(inside, nbr, idx), inside)
            diag += c
            cols[t] = nbr
            vals[t] = -c
            keep[t] = inside & (c != 0.0)
        cols[centre] = idx
        vals[centre] = diag_fn(diag, idx)
        keep[centre] = vals[centre] != 0.0
        counts[idx] = keep.sum(axis=0)
        kt = keep.T
        col_parts.append(cols.T[kt].astype(np.int32))
        val_parts.append(vals.T[kt])
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return Csr(n, n, off, np.concatenate(col_parts), np.concatenate(val_parts))


def poisson7(nx, ny, nz):
    """7-point Laplacian; restates ``gen_poisson7`` (``amgkit/problems.py:48-52``)."""
    offs = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    coupling = lambda o, idx, nbr, inside: np.where(inside, 1.0, 0.0)
    return _assemble(nx, ny, nz, offs, coupling, lambda d, idx: np.full(idx.size, 6.0))


def rtanis7(nx, ny, nz, kx=1.0, ky=1.0, kz=1e-3):
    """``gen_rotated_anisotropy`` at theta = 0 (``amgkit/problems.py:62-88``).

    The rotated tensor at theta = 0 is diag(kx, ky, kz) exactly and the four
    cross entries are zero (eliminated), so only the axis couplings remain;
    the diagonal is 2 (kx + ky + kz) regardless of boundary elimination.
    """
    kxx, kyy, kzz = float(kx), float(ky), float(kz)
    offs = [(0, 0, -1), (0, -1, 0), (-1, 0, 0), (0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1)]
    w = {(0, 0, -1): kzz, (0, 0, 1): kzz, (0, -1, 0): kyy, (0, 1, 0): kyy, (-1, 0, 0): kxx, (1, 0, 0): kxx}
    coupling = lambda o, idx, nbr, inside: np.where(inside, w[o], 0.0)
    centre = 2.0 * (kxx + kyy + kzz)
    return _assemble(nx, ny, nz, offs, coupling, lambda d, idx: np.full(idx.size, centre))


def conductivity(nx, ny, nz, sigma, seed, block=1):
    """Per-cell lognormal conductivity k = exp(sigma * N(0, 1)).

    ``block`` > 1 draws one normal per block^3 cell block (correlated blocks,
    config 5); blocks are numbered x fastest like the nodes.
    """
    rng = np.random.default_rng(seed)
    if block == 1:
        return np.exp(sigma * rng.standard_normal(nx * ny * nz))
    bx, by, bz = -(-nx // block), -(-ny // block), -(-nz // block)
    g = rng.standard_normal(bx * by * bz).reshape(bz, by, bx)
    g = np.repeat(np.repeat(np.repeat(g, block, axis=0), block, axis=1), block, axis=2)
    return np.exp(sigma * g[:nz, :ny, :nx].reshape(-1))


def hetero27(nx, ny, nz, sigma=2.0, seed=42, block=1):
    """27-point heterogeneous diffusion (configs 2 and 5); see module doc."""
    k = conductivity(nx, ny, nz, sigma, seed, block)

    def coupling(o, idx, nbr, inside):
        dx, dy, dz = o
        w = 1.0 / float(dx * dx + dy * dy + dz * dz)
        ki = k[idx]
        kj = k[nbr]
        return np.where(inside, w * (2.0 * ki * kj / (ki + kj)), w * ki)

    return _assemble(nx, ny, nz, _offsets27(), coupling, lambda d, idx: d)


def hex_stiffness(e, nu, hx=1.0, hy=1.0, hz=1.0):
    """Q1 hexahedron stiffness (8 nodes x 3 dofs, 2x2x2 Gauss); restates
    ``hex_element_stiffness`` (``amgkit/problems.py:91-139``): node order x
    fastest, dof order node-major xyz."""
    lam = e * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = e / (2.0 * (1.0 + nu))
    d = np.zeros((6, 6))
    d[:3, :3] = lam
    d[np.arange(3), np.arange(3)] += 2.0 * mu
    d[3:, 3:] = np.eye(3) * mu
    corners = np.array([[sx, sy, sz] for sz in (-1, 1) for sy in (-1, 1) for sx in (-1, 1)], dtype=float)
    g = np.array([-1.0, 1.0]) / np.sqrt(3.0)
    half = np.array([hx, hy, hz]) / 2.0
    detj = float(np.prod(half))
    ke = np.zeros((24, 24))
    for gx in g:
        for gy in g:
            for gz in g:
                xi = (gx, gy, gz)
                dn = np.empty((8, 3))
                for a in range(8):
                    sx, sy, sz = corners[a]
                    dn[a, 0] = sx * (1 + sy * xi[1]) * (1 + sz * xi[2]) / 8.0
                    dn[a, 1] = sy * (1 + sx * xi[0]) * (1 + sz * xi[2]) / 8.0
                    dn[a, 2] = sz * (1 + sx * xi[0]) * (1 + sy * xi[1]) / 8.0
                dn = dn / half
                bm = np.zeros((6, 24))
                for a in range(8):
                    bx, by, bz = dn[a]
                    c = 3 * a
                    bm[0, c], bm[1, c + 1], bm[2, c + 2] = bx, by, bz
                    bm[3, c], bm[3, c + 1] = by, bx
                    bm[4, c + 1], bm[4, c + 2] = bz, by
                    bm[5, c], bm[5, c + 2] = bz, bx
                ke += bm.T @ d @ bm * detj
    return ke


def elasticity3d(nx, ny, nz, sigma=1.0, nu=0.3, seed=42):
    """Config-3 operator and node coordinates (see module doc)."""
    import scipy.sparse as sp

    h = 1.0 / nx
    mx, my, mz = nx + 1, ny + 1, nz + 1
    node = lambda i, j, k: i + mx * (j + my * k)
    ke = hex_stiffness(1.0, nu, h, h, h)
    young = np.exp(sigma * np.random.default_rng(seed).standard_normal(nx * ny * nz))
    ei, ej, ek = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    # element e = ei + nx * (ej + ny * ek) (x fastest, like the nodes)
    ei, ej, ek = ei.transpose(2, 1, 0).ravel(), ej.transpose(2, 1, 0).ravel(), ek.transpose(2, 1, 0).ravel()
    corners = np.stack([node(ei + dx, ej + dy, ek + dz) for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)], axis=1)
    dofs = (3 * corners[:, :, None] + np.arange(3)).reshape(-1, 24)
    n_nodes = mx * my * mz
    keep_node = np.ones(n_nodes, dtype=bool)
    keep_node[np.arange(n_nodes) % mx == 0] = False  # clamp x = 0
    keep_dof = np.repeat(keep_node, 3)
    new_dof = np.full(3 * n_nodes, -1, dtype=np.int64)
    new_dof[keep_dof] = np.arange(int(keep_dof.sum()))
    nd = int(keep_dof.sum())
    rows_l, cols_l, vals_l = [], [], []
    chunk = 1 << 16
    for e0 in range(0, dofs.shape[0], chunk):
        dd = dofs[e0:e0 + chunk]
        r = np.repeat(dd, 24, axis=1).ravel()
        c = np.tile(dd, (1, 24)).ravel()
        v = (young[e0:e0 + chunk, None] * ke.ravel()[None, :]).ravel()
        ok = keep_dof[r] & keep_dof[c]
        rows_l.append(new_dof[r[ok]])
        cols_l.append(new_dof[c[ok]])
        vals_l.append(v[ok])
    m = sp.coo_matrix((np.concatenate(vals_l), (np.concatenate(rows_l), np.concatenate(cols_l))), shape=(nd, nd)).tocsr()
    m.sum_duplicates()
    m.sort_indices()
    m.eliminate_zeros()
    ii, jj, kk = np.meshgrid(np.arange(mx), np.arange(my), np.arange(mz), indexing="ij")
    coords = np.empty((n_nodes, 3))
    flat = node(ii, jj, kk).ravel()
    coords[flat, 0] = ii.ravel() * h
    coords[flat, 1] = jj.ravel() * h
    coords[flat, 2] = kk.ravel() * h
    return Csr(nd, nd, m.indptr, m.indices, m.data), coords[keep_node]


def rhs_body_load(n_dofs, h, seed=42):
    """Config-3 RHS: (0, 0, -1) h^3 per node times (1 + 0.01 N(0,1)) per dof."""
    f = np.zeros(n_dofs)
    f[2::3] = -(h ** 3)
    return f * (1.0 + 0.01 * np.random.default_rng(seed + 1).standard_normal(n_dofs))


def rhs_uniform(n, seed=42):
    """``default_rng(seed).uniform(-1, 1, n)`` (BASELINE RHS for configs 1, 2, 4, 5)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


# name -> (generator, args, kwargs, amg recipe); the recipe is what the
# hierarchy export feeds to the reference ``AmgConfig``.
CONFIGS = {
    "c1_poisson7_64": (poisson7, (64, 64, 64), {}, {"smoother": "fsai"}),
    "c2_hetero27_128": (hetero27, (128, 128, 128), {"sigma": 2.0, "seed": 42}, {"smoother": "fsai"}),
    "c3_elasticity_64": (elasticity3d, (64, 64, 64), {"sigma": 1.0, "nu": 0.3, "seed": 42},
                         {"smoother": "fsai", "interp": "bamg", "testspace": "rigid_body", "n_test_vectors": 6}),
    "c4_rtanis7_256": (rtanis7, (256, 256, 256), {"kx": 1.0, "ky": 1.0, "kz": 1e-3}, {"smoother": "fsai"}),
    "c5_hetero27_512": (hetero27, (512, 512, 256), {"sigma": 3.0, "seed": 42, "block": 4}, {"smoother": "fsai"}),
    # reduced-size stand-ins used by tests and smoke runs
    "t_poisson7_16": (poisson7, (16, 16, 16), {}, {"smoother": "fsai"}),
    "t_hetero27_24": (hetero27, (24, 24, 24), {"sigma": 2.0, "seed": 42}, {"smoother": "fsai"}),
    "t_rtanis7_32": (rtanis7, (32, 32, 32), {"kx": 1.0, "ky": 1.0, "kz": 1e-3}, {"smoother": "fsai"}),
    # config 4's x-y planes with a quarter of its z extent (tuning stand-in: same per-plane coarsening)
    "t_rtanis7_256x64": (rtanis7, (256, 256, 64), {"kx": 1.0, "ky": 1.0, "kz": 1e-3}, {"smoother": "fsai"}),
    "t_elasticity_12": (elasticity3d, (12, 12, 12), {"sigma": 1.0, "nu": 0.3, "seed": 42},
                        {"smoother": "fsai", "interp": "bamg", "testspace": "rigid_body", "n_test_vectors": 6}),
}


def build_config(name, with_coords=False):
    """Level-0 operator of a named config (and node coordinates for elasticity)."""
    fn, args, kwargs, _ = CONFIGS[name]
    out = fn(*args, **kwargs)
    if isinstance(out, tuple):
        return out if with_coords else out[0]
    return (out, None) if with_coords else out


def build_rhs(name, n):
    """Right-hand side of a named config (seed 42)."""
    fn, args, kwargs, _ = CONFIGS[name]
    if fn is elasticity3d:
        return rhs_body_load(n, 1.0 / args[0], kwargs.get("seed", 42))
    return rhs_uniform(n, 42)
