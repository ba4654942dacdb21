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
* config 4 -- ``rtanis7``: ``gen_rotated_anisotropy(nx, ny, nz, theta=0,
  kx=1, ky=1, kz=eps)`` (``problems.py:62-88``); with theta = 0 the cross
  terms vanish exactly and are eliminated, leaving a 7-point stencil with
  diagonal 2 (kx + ky + kz).

RHS for every scalar config: ``default_rng(seed).uniform(-1, 1, n)``.
"""
from __future__ import annotations

import numpy as np

__all__ = ["Csr", "poisson7", "rtanis7", "hetero27", "rhs_uniform", "build_config", "CONFIGS"]


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


def rhs_uniform(n, seed=42):
    """``default_rng(seed).uniform(-1, 1, n)`` (BASELINE RHS for configs 1, 2, 4, 5)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


# name -> (generator, args, kwargs, amg recipe); the recipe is what the
# hierarchy export feeds to the reference ``AmgConfig``.
CONFIGS = {
    "c1_poisson7_64": (poisson7, (64, 64, 64), {}, {"smoother": "fsai"}),
    "c2_hetero27_128": (hetero27, (128, 128, 128), {"sigma": 2.0, "seed": 42}, {"smoother": "fsai"}),
    "c4_rtanis7_256": (rtanis7, (256, 256, 256), {"kx": 1.0, "ky": 1.0, "kz": 1e-3}, {"smoother": "fsai"}),
    "c5_hetero27_512": (hetero27, (512, 512, 256), {"sigma": 3.0, "seed": 42, "block": 4}, {"smoother": "fsai"}),
    # reduced-size stand-ins used by tests and smoke runs
    "t_poisson7_16": (poisson7, (16, 16, 16), {}, {"smoother": "fsai"}),
    "t_hetero27_24": (hetero27, (24, 24, 24), {"sigma": 2.0, "seed": 42}, {"smoother": "fsai"}),
    "t_rtanis7_32": (rtanis7, (32, 32, 32), {"kx": 1.0, "ky": 1.0, "kz": 1e-3}, {"smoother": "fsai"}),
}


def build_config(name):
    """Level-0 operator of a named config."""
    fn, args, kwargs, _ = CONFIGS[name]
    return fn(*args, **kwargs)
