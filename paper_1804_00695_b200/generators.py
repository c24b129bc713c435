"""Synthetic inputs for the five BASELINE.json configurations.

These are input builders (test and benchmark infrastructure), not the hot
path.  Row-sorted CSR is produced directly (no COO lexsort), so a 256^3
brick stencil (449M entries) builds in seconds.

* Stencils use the reference's conventions (generators.py:26-45, 98-142):
  flat index with the first axis fastest, centre weight = number of
  neighbours (7-pt 6/-1, 27-pt 26/-1, 13-pt big star 12/-1, elasticity
  3x3 blocks I + 0.5).  ``laplace2d`` (5-pt, 4/-1) is config 1's operator,
  which the reference lacks; tests pin it against the reference's own
  entry builder applied to 2D offsets.
* ``aggregation`` is the plain 2x2(x2) aggregation prolongator of config 2
  (one 1.0 per fine row); R = P^T.
* ``rmat_graph`` is a Graph500-parameter R-MAT (a,b,c,d = .57,.19,.19,.05,
  edge factor 16) seeded with SplitMix64 (rng.py), symmetrised,
  de-duplicated and loop-free like the reference's ``to_undirected_pattern``
  (triangles.py:56-68).  Vertex labels are scrambled with a SplitMix64
  random-key permutation, as Graph500 does.
"""

import numpy as np

from . import rng as _rng
from .csr import CsrMatrix, transpose
from .errors import GridError

LAPLACE2D = "laplace2d"
LAPLACE3D = "laplace3d"
BIGSTAR2D = "bigstar2d"
BRICK3D = "brick3d"
ELASTICITY3D = "elasticity3d"
STENCIL_KINDS = (LAPLACE2D, LAPLACE3D, BIGSTAR2D, BRICK3D, ELASTICITY3D)


def _offsets(kind):
    if kind == LAPLACE2D:
        return [((0, 0), 4.0)] + [(s, -1.0) for s in ((-1, 0), (1, 0), (0, -1), (0, 1))]
    if kind == LAPLACE3D:
        nb = [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]
        return [((0, 0, 0), 6.0)] + [(s, -1.0) for s in nb]
    if kind == BIGSTAR2D:
        nb = [(-1, 0), (1, 0), (0, -1), (0, 1), (-2, 0), (2, 0), (0, -2), (0, 2),
              (-1, -1), (-1, 1), (1, -1), (1, 1)]
        return [((0, 0), 12.0)] + [(s, -1.0) for s in nb]
    if kind in (BRICK3D, ELASTICITY3D):
        nb = [(x, y, z) for x in (-1, 0, 1) for y in (-1, 0, 1) for z in (-1, 0, 1)
              if (x, y, z) != (0, 0, 0)]
        return [((0, 0, 0), 26.0)] + [(s, -1.0) for s in nb]
    raise GridError("unknown stencil kind %r" % (kind,))


def _scalar_rows(kind, dims, lo, hi):
    """(row_len, cols, vals) of scalar stencil rows [lo, hi), row-sorted."""
    offs = _offsets(kind)
    strides = [1]
    for d in dims[:-1]:
        strides.append(strides[-1] * d)
    # ascending linear shift == ascending column within every row
    offs.sort(key=lambda o: sum(s * st for s, st in zip(o[0], strides)))
    idx = np.arange(lo, hi, dtype=np.int64)
    coord = [(idx // st) % d for st, d in zip(strides, dims)]
    k = len(offs)
    keep = np.ones((hi - lo, k), dtype=bool)
    cand = np.empty((hi - lo, k), dtype=np.int64)
    vals = np.empty(k, dtype=np.float64)
    for j, (shift, w) in enumerate(offs):
        ok = keep[:, j]
        for ax, s in enumerate(shift):
            if s:
                ok &= (coord[ax] + s >= 0) & (coord[ax] + s < dims[ax])
        cand[:, j] = idx + sum(s * st for s, st in zip(shift, strides))
        vals[j] = w
    return keep.sum(axis=1), cand[keep], np.ascontiguousarray(np.broadcast_to(vals, keep.shape)[keep])


def _check_dims(kind, dims):
    dims = tuple(int(d) for d in dims)
    want = 2 if kind in (LAPLACE2D, BIGSTAR2D) else 3
    if len(dims) != want:
        raise GridError("%s needs %d grid dims" % (kind, want))
    if any(d <= 0 for d in dims):
        raise GridError("grid dims must be positive")
    return dims


def stencil_rows(kind: str, dims, lo: int, hi: int) -> CsrMatrix:
    """Rows [lo, hi) of a scalar stencil operator (a row shard, full column
    space) -- what one rank of the row partition builds."""
    dims = _check_dims(kind, dims)
    n = int(np.prod(dims))
    row_len, cols, v = _scalar_rows(kind, dims, lo, hi)
    ptr = np.zeros(hi - lo + 1, dtype=np.int64)
    np.cumsum(row_len, out=ptr[1:])
    return CsrMatrix._adopt(hi - lo, n, ptr, cols, v)


def stencil(kind: str, dims) -> CsrMatrix:
    """Grid operator with row-sorted columns (first axis fastest)."""
    dims = _check_dims(kind, dims)
    n = int(np.prod(dims))
    row_len, cols, v = _scalar_rows(kind, dims, 0, n)
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(row_len, out=ptr[1:])
    if kind != ELASTICITY3D:
        return CsrMatrix._adopt(n, n, ptr, cols, np.ascontiguousarray(v))
    # 3 dofs per point: each scalar entry becomes a dense 3x3 block
    block = np.eye(3) + 0.5 * np.ones((3, 3))
    rl3 = np.repeat(row_len * 3, 3)
    ptr3 = np.zeros(3 * n + 1, dtype=np.int64)
    np.cumsum(rl3, out=ptr3[1:])
    # vectorised expansion: dof row 3i+r lists 3c+d for each neighbour c, dof d
    rows_of = np.repeat(np.arange(n), row_len)
    c3 = (3 * cols[:, None] + np.arange(3)[None, :])       # (nnz, 3)
    w3 = v[:, None, None] * block[None, :, :]               # (nnz, r, d)
    out_c = np.empty(9 * cols.shape[0], dtype=np.int64)
    out_v = np.empty(9 * cols.shape[0], dtype=np.float64)
    for r in range(3):
        # dof-row 3*i + r occupies [ptr3[3i+r], ptr3[3i+r+1])
        start = ptr3[3 * rows_of + r] + 3 * (np.arange(cols.shape[0]) - ptr[rows_of])
        pos = start[:, None] + np.arange(3)[None, :]
        out_c[pos.ravel()] = c3.ravel()
        out_v[pos.ravel()] = w3[:, r, :].ravel()
    return CsrMatrix._adopt(3 * n, 3 * n, ptr3, out_c, out_v)


def aggregation(dims, factor: int = 2):
    """(P, R): P maps each fine point to its factor^d aggregate (value 1.0),
    coarse dims ceil(d / factor); R = P^T."""
    dims = tuple(int(d) for d in dims)
    coarse = tuple(-(-d // factor) for d in dims)
    n = int(np.prod(dims))
    idx = np.arange(n, dtype=np.int64)
    agg = np.zeros(n, dtype=np.int64)
    fs, cs = 1, 1
    for d, c in zip(dims, coarse):
        agg += ((idx // fs) % d // factor) * cs
        fs *= d
        cs *= c
    nc = int(np.prod(coarse))
    p = CsrMatrix._adopt(n, nc, np.arange(n + 1, dtype=np.int64), agg, np.ones(n))
    return p, transpose(p)


def rmat_edges(scale: int, edge_factor: int = 16, seed: int = 22,
               a: float = 0.57, b: float = 0.19, c: float = 0.19,
               batch: int = 1 << 22):
    """Directed R-MAT edge list (u, v) of 2^scale vertices.

    Edge e, level l consumes SplitMix64 output e*scale + l + 1 of
    PortableRng(seed); the vertex permutation uses PortableRng(seed ^ GAMMA).
    """
    n = 1 << scale
    m = n * edge_factor
    u = np.empty(m, dtype=np.int64)
    v = np.empty(m, dtype=np.int64)
    ab, abc = a + b, a + b + c
    for e0 in range(0, m, batch):
        e1 = min(m, e0 + batch)
        cnt = e1 - e0
        r = _rng.unit_interval(_rng.stream(seed, e0 * scale, cnt * scale)).reshape(cnt, scale)
        bit_u = (r >= ab).astype(np.int64)                       # quadrants c, d
        bit_v = ((r >= a) & (r < ab)) | (r >= abc)               # quadrants b, d
        w = (np.int64(1) << np.arange(scale - 1, -1, -1, dtype=np.int64))
        u[e0:e1] = bit_u @ w
        v[e0:e1] = bit_v.astype(np.int64) @ w
    keys = _rng.stream(seed ^ _rng.GAMMA, 0, n)
    perm = np.empty(n, dtype=np.int64)
    perm[np.argsort(keys, kind="stable")] = np.arange(n, dtype=np.int64)
    return perm[u], perm[v]


def undirected_pattern(u, v, n: int) -> CsrMatrix:
    """Symmetrised, de-duplicated, loop-free pattern of an edge list."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    keep = u != v
    u, v = u[keep], v[keep]
    key = np.concatenate([u * n + v, v * n + u])
    key = np.unique(key)
    rows, cols = key // n, key % n
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
    return CsrMatrix._adopt(n, n, ptr, cols, None)


def rmat_graph(scale: int, edge_factor: int = 16, seed: int = 22) -> CsrMatrix:
    u, v = rmat_edges(scale, edge_factor, seed)
    return undirected_pattern(u, v, 1 << scale)


def rmat_graph_device(scale: int, edge_factor: int = 16, seed: int = 22,
                      a: float = 0.57, b: float = 0.19, c: float = 0.19):
    """``rmat_graph`` built in HBM (csrc/tsg_graph.cu):
    same SplitMix64 draws, relabelling and de-duplication, so the DeviceCsr
    equals the host builder's matrix entry for entry."""
    from . import _lib
    return _lib.d_rmat_graph(scale, edge_factor, seed, a, b, c)


def stencil_device(kind: str, dims, lo: int = None, hi: int = None):
    """``stencil`` (or ``stencil_rows`` for a row range) built in HBM
    (csrc/tsg_build.cu): the same rows, columns and values as the host
    builder, as a DeviceCsr."""
    from . import _lib
    dims = _check_dims(kind, dims)
    if kind not in STENCIL_KINDS:
        raise GridError("unknown stencil kind %r" % (kind,))
    if lo is None:
        return _lib.d_stencil(kind, dims)
    return _lib.d_stencil(kind, dims, int(lo), int(hi))


def aggregation_device(dims, factor: int = 2):
    """``aggregation`` built in HBM: (P, R) as DeviceCsr, R = P^T assembled
    directly (each aggregate lists its fine points in ascending order)."""
    from . import _lib
    dims = tuple(int(d) for d in dims)
    if any(d <= 0 for d in dims):
        raise GridError("grid dims must be positive")
    return _lib.d_aggregation(dims, factor)


def with_unit_values(g: CsrMatrix) -> CsrMatrix:
    return CsrMatrix._adopt(g.num_rows, g.num_cols, g.row_ptr, g.col_idx, np.ones(g.nnz))


def random_rhs(num_rows: int, num_cols: int, delta: int, seed: int) -> CsrMatrix:
    """Exactly delta distinct columns per row in SplitMix64 draw order
    (unsorted), values in (0, 1]; the reference's random RHS recipe
    (generators.py:248-272).  Sequential; test sizes only."""
    if delta > num_cols or delta < 0 or num_rows < 0:
        raise GridError("bad random RHS shape")
    g = _rng.PortableRng(seed)
    cols = np.empty(num_rows * delta, dtype=np.int64)
    vals = np.empty(num_rows * delta, dtype=np.float64)
    p = 0
    for _ in range(num_rows):
        for col in g.sample_without_replacement(num_cols, delta):
            cols[p] = col
            vals[p] = g.uniform_open_closed()
            p += 1
    return CsrMatrix._adopt(num_rows, num_cols, np.arange(num_rows + 1, dtype=np.int64) * delta,
                            cols, vals)


# ---------------------------------------------------------------- reference problems
# The reference's problem builders for its benchmark CLI (generators.py:51-246):
# a stencil spec, exact nnz / byte sizes, target-byte grid search and the
# geometric (bi/tri)linear interpolation pair.  Input builders, not hot path.

from dataclasses import dataclass as _dataclass


@_dataclass(frozen=True)
class StencilSpec:
    """Stencil family + per-axis grid point counts (generators.py:51-83)."""

    kind: str
    grid_dims: tuple

    def __post_init__(self):
        if self.kind not in STENCIL_KINDS:
            raise GridError("unknown stencil kind %r" % (self.kind,))
        dims = tuple(int(d) for d in self.grid_dims)
        object.__setattr__(self, "grid_dims", dims)
        if any(d <= 0 for d in dims):
            raise GridError("grid dims must be positive")
        want = 2 if self.kind in (BIGSTAR2D, LAPLACE2D) else 3
        if len(dims) != want:
            raise GridError("%s needs %d grid dims, got %d" % (self.kind, want, len(dims)))

    @property
    def rank(self) -> int:
        return len(self.grid_dims)

    @property
    def dofs_per_point(self) -> int:
        return 3 if self.kind == ELASTICITY3D else 1

    @property
    def num_points(self) -> int:
        return int(np.prod(self.grid_dims))

    @property
    def matrix_rows(self) -> int:
        return self.num_points * self.dofs_per_point


def generate_stencil(spec: StencilSpec) -> CsrMatrix:
    """The reference's entry point (generators.py:115-142): dims >= 5."""
    if any(d < 5 for d in spec.grid_dims):
        raise GridError("stencil grids need every dim >= 5")
    return stencil(spec.kind, spec.grid_dims)


def stencil_nnz(kind: str, grid_dims) -> int:
    """Exact nnz without building: each offset keeps the points whose shifted
    neighbour stays in the grid (generators.py:145-160)."""
    spec = StencilSpec(kind, tuple(grid_dims))
    total = 0
    for shift, _ in _offsets(kind):
        k = 1
        for ax, s in enumerate(shift):
            k *= max(spec.grid_dims[ax] - abs(s), 0)
        total += k
    return total * spec.dofs_per_point ** 2


def stencil_byte_size(kind: str, grid_dims) -> int:
    spec = StencilSpec(kind, tuple(grid_dims))
    return 8 * (spec.matrix_rows + 1) + 16 * stencil_nnz(kind, grid_dims)


def grid_for_target_bytes(kind: str, target_bytes: int, max_dim: int = 513):
    """Smallest odd cubic (square in 2D) grid reaching target_bytes
    (generators.py:168-179)."""
    rank = 2 if kind in (BIGSTAR2D, LAPLACE2D) else 3
    for n in range(5, max_dim + 1, 2):
        dims = (n,) * rank
        if stencil_byte_size(kind, dims) >= target_bytes:
            return dims
    raise GridError("no grid up to %d^%d reaches %d bytes" % (max_dim, rank, target_bytes))


def generate_interpolation(spec: StencilSpec):
    """(P, R = P^T) coarsening by two on every axis (generators.py:182-245):
    coarse points on even coordinates, odd points average their two coarse
    neighbours, per-axis weights multiplied (all powers of two, so exact).
    Vectorised: one pass per choice pattern of the 2^rank neighbour combos."""
    dims = spec.grid_dims
    for d in dims:
        if d < 3 or d % 2 == 0:
            raise GridError("interpolation needs odd grid dims >= 3, got %r" % (dims,))
    coarse = [(d + 1) // 2 for d in dims]
    n = spec.num_points
    idx = np.arange(n, dtype=np.int64)
    coords, div = [], 1
    for d in dims:
        coords.append((idx // div) % d)
        div *= d
    cstride = np.cumprod([1] + coarse[:-1]).astype(np.int64)
    rows, cols, vals = [], [], []
    for combo in range(1 << len(dims)):
        ok = np.ones(n, dtype=bool)
        col = np.zeros(n, dtype=np.int64)
        w = np.ones(n, dtype=np.float64)
        for ax in range(len(dims)):
            x = coords[ax]
            odd = (x & 1) == 1
            up = (combo >> ax) & 1
            if up:
                ok &= odd
            col += cstride[ax] * (x // 2 + up)
            w *= np.where(odd, 0.5, 1.0)
        rows.append(idx[ok])
        cols.append(col[ok])
        vals.append(w[ok])
    rows, cols, vals = np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)
    dofs = spec.dofs_per_point
    if dofs > 1:
        d = np.arange(dofs)
        rows = (dofs * rows[:, None] + d[None, :]).ravel()
        cols = (dofs * cols[:, None] + d[None, :]).ravel()
        vals = np.repeat(vals, dofs)
    p = CsrMatrix.from_coo(rows, cols, vals, n * dofs, int(np.prod(coarse)) * dofs)
    return p, transpose(p)


generate_random_rhs = random_rhs
