"""Synthetic Helmholtz systems for the BASELINE configurations (host-side setup).

Not on the hot path: these build the CSR inputs (``ia``/``ja`` int64,
``aa`` complex128, exactly the reference ``CsrMatrix`` layout,
``sparse.py:60-103``) that the solver consumes.  They are vectorised numpy
replacements for the reference's per-row Python loop
(``helmholtz.py:115-168``, ``assemble``), which needs ~4.5 s per million rows.

* :func:`helmholtz_fd` -- the reference's (2*dim+1)-point central-difference
  stencil with a unit interior source and zero Dirichlet data, i.e. what
  ``assemble(load_problem_config(...))`` produces (``helmholtz.py:115-168``,
  ``:211-249``).  With ``damping == 0`` the arrays are bitwise identical to the
  reference (checked by ``tests/test_oracle.py`` against ``tests/golden/problems.npz``,
  made from it by ``tests/golden/make_golden.py``).
  ``damping = eps`` shifts the diagonal by ``-i * eps * k^2`` (complex
  damping ``k^2 (1 + i eps)``; BASELINE configs C1/C5).
* :func:`helmholtz_27pt` -- 27-point stencil, diagonal ``26/(3h^2) - k^2(1+i eps)``,
  off-diagonals ``-1/(3h^2)`` (BASELINE config C4).
* :func:`cylinder_p1fe` -- P1 tetrahedral FE Helmholtz on a cylinder (BASELINE
  config C3; irregular FE rows, up to 15 nonzeros).
* :func:`config_problem` -- the named BASELINE configurations.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = ["helmholtz_fd", "helmholtz_27pt", "cylinder_p1fe", "config_problem", "CONFIGS"]


def _csr_from_mask(mask: np.ndarray, cols: np.ndarray, vals: np.ndarray):
    """Row-major compaction of an (n, w) stencil table into CSR arrays."""
    counts = mask.sum(axis=1, dtype=np.int64)
    ia = np.zeros(mask.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=ia[1:])
    ja = cols[mask]
    aa = np.broadcast_to(vals, mask.shape)[mask]
    return ia, np.ascontiguousarray(ja, dtype=np.int64), np.ascontiguousarray(aa, dtype=np.complex128)


def helmholtz_fd(dim: int, cells: int, length: float = 1.0, frequency: float = 0.0,
                 velocity: float = 1.0, damping: float = 0.0, source: complex = 1 + 0j):
    """(2*dim+1)-point FD Helmholtz system on ``(cells-1)**dim`` interior nodes.

    Returns ``(n, ia, ja, aa, b)``.  Scalars follow ``helmholtz.py:218-244``
    term by term (``inv_h2 = 1/(h*h)``, diagonal ``2*dim*inv_h2 - k2``,
    neighbours ``-inv_h2``); columns of each row come out ascending, as
    ``coo_to_csr`` sorts them (``sparse.py:203-214``).
    """
    if dim not in (1, 2, 3) or cells < 3:
        raise ValueError("dim must be 1..3 and cells >= 3")
    m = cells - 1
    h = length / cells
    inv_h2 = 1.0 / (h * h)
    k = 2.0 * math.pi * frequency / velocity
    k2 = k**2
    n = m**dim
    diag = complex(2 * dim * inv_h2 - k2)
    if damping:
        diag = complex(diag.real, -k2 * damping)
    off = complex(-inv_h2)
    strides = [m**a for a in range(dim)]
    flat = np.arange(n, dtype=np.int64)
    coords = [(flat // s) % m for s in strides]
    # ascending column order: -s_{d-1} .. -s_0, 0, +s_0 .. +s_{d-1}
    offsets, valid, values = [], [], []
    for a in reversed(range(dim)):
        offsets.append(-strides[a]); valid.append(coords[a] > 0); values.append(off)
    offsets.append(0); valid.append(np.ones(n, dtype=bool)); values.append(diag)
    for a in range(dim):
        offsets.append(strides[a]); valid.append(coords[a] < m - 1); values.append(off)
    mask = np.stack(valid, axis=1)
    cols = flat[:, None] + np.asarray(offsets, dtype=np.int64)[None, :]
    ia, ja, aa = _csr_from_mask(mask, cols, np.asarray(values, dtype=np.complex128)[None, :])
    # rhs: zero Dirichlet contributions (inv_h2 * 0j) then + source, helmholtz.py:256-257
    b = np.zeros(n, dtype=np.complex128)
    b += complex(source)
    return n, ia, ja, aa, b


def helmholtz_27pt(m: int, k2: float = 100.0, damping: float = 0.05, length: float = 1.0,
                   source: complex = 1 + 0j):
    """27-point Helmholtz stencil on an ``m**3`` interior grid (config C4)."""
    h = length / (m + 1)
    inv_3h2 = 1.0 / (3.0 * h * h)
    diag = complex(26.0 * inv_3h2 - k2, -k2 * damping)
    off = complex(-inv_3h2)
    n = m**3
    flat = np.arange(n, dtype=np.int64)
    ix, iy, iz = flat % m, (flat // m) % m, flat // (m * m)
    offsets, valid, values = [], [], []
    lo = [c > 0 for c in (ix, iy, iz)]
    hi = [c < m - 1 for c in (ix, iy, iz)]
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = None
                for d, l, u in ((dx, lo[0], hi[0]), (dy, lo[1], hi[1]), (dz, lo[2], hi[2])):
                    if d:
                        c = l if d < 0 else u
                        ok = c if ok is None else (ok & c)
                if ok is None:
                    ok = np.ones(n, dtype=bool)
                offsets.append(dx + dy * m + dz * m * m)
                valid.append(ok)
                values.append(diag if (dx, dy, dz) == (0, 0, 0) else off)
    mask = np.stack(valid, axis=1)
    del valid, lo, hi, ix, iy, iz
    cols = flat[:, None] + np.asarray(offsets, dtype=np.int64)[None, :]
    ia, ja, aa = _csr_from_mask(mask, cols, np.asarray(values, dtype=np.complex128)[None, :])
    b = np.full(n, complex(source), dtype=np.complex128)
    return n, ia, ja, aa, b


def cylinder_p1fe(m: int, length: float = 2.0, wavelengths: float = 2.0, damping: float = 0.1,
                  source: complex = 1 + 0j):
    """P1 finite-element Helmholtz system on a cylinder (BASELINE config C3,
    "cylinder-like synthetic P1-FE"; the paper's Cylinder3D matrices are not
    available).  Grid spacing h = 2/m over [-1, 1]^2 x [0, length], Kuhn
    split of every cube into 6 congruent tetrahedra, tetrahedra kept when all
    four vertices lie in the unit-radius cylinder; ``A = K - k^2 (1 + i eps) M``
    with P1 stiffness K and consistent mass M, natural (Neumann) boundary, and
    ``k = 2*pi*wavelengths``; unit point source at the node nearest the axis
    midpoint.  Interior rows have 15 nonzeros (the Kuhn 15-point stencil),
    boundary rows fewer -- the irregular row lengths of an FE matrix.
    Returns ``(n, ia, ja, aa, b)``; columns ascend in each row.
    """
    import scipy.sparse as sp
    h = 2.0 / m
    mz = int(round(length / h))
    nx, ny, nz = m + 1, m + 1, mz + 1
    gx = -1.0 + h * np.arange(nx)
    inside2d = (gx[:, None] ** 2 + gx[None, :] ** 2) <= 1.0 + 1e-12  # [ix, iy]
    # Kuhn tetrahedra of the unit cube: vertex sequences 0 -> e_a -> e_a+e_b -> (1,1,1)
    import itertools
    cube = {}
    tets = []
    for perm in itertools.permutations(range(3)):
        v = [np.zeros(3, dtype=np.int64)]
        for a in perm:
            w = v[-1].copy()
            w[a] = 1
            v.append(w)
        tets.append(np.stack(v))
    # element matrices (all six tetrahedra are congruent up to reflection)
    ke, me = [], []
    for tv in tets:
        X = tv.astype(np.float64) * h
        T = np.vstack([np.ones(4), X.T])  # 4x4
        Ginv = np.linalg.inv(T)          # rows: barycentric coefficient vectors
        grads = Ginv[:, 1:]              # (4, 3)
        vol = abs(np.linalg.det(T)) / 6.0
        ke.append(vol * grads @ grads.T)
        me.append(vol / 20.0 * (np.ones((4, 4)) + np.eye(4)))
    k2 = (2.0 * math.pi * wavelengths) ** 2
    shift = complex(k2, k2 * damping)
    # cube origins (ix, iy, iz) with all corners inside the cylinder
    cx, cy = np.nonzero(inside2d[:-1, :-1] & inside2d[1:, :-1] & inside2d[:-1, 1:] & inside2d[1:, 1:])
    if cx.size == 0:
        raise ValueError("grid too coarse for the cylinder")
    cz = np.arange(nz - 1, dtype=np.int64)
    ox = np.repeat(cx, cz.size)
    oy = np.repeat(cy, cz.size)
    oz = np.tile(cz, cx.size)
    gid = lambda x, y, z: (z * ny + y) * nx + x  # noqa: E731  (lexicographic grid id, x fastest)
    rows, cols, vals = [], [], []
    for t, tv in enumerate(tets):
        nodes = [gid(ox + tv[a, 0], oy + tv[a, 1], oz + tv[a, 2]) for a in range(4)]
        loc = ke[t] - shift * me[t]
        for a in range(4):
            for c in range(4):
                rows.append(nodes[a])
                cols.append(nodes[c])
                vals.append(np.full(ox.size, loc[a, c], dtype=np.complex128))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    vals = np.concatenate(vals)
    used = np.unique(rows)
    remap = np.full(nx * ny * nz, -1, dtype=np.int64)
    remap[used] = np.arange(used.size, dtype=np.int64)
    n = int(used.size)
    A = sp.coo_matrix((vals, (remap[rows], remap[cols])), shape=(n, n)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    ia = A.indptr.astype(np.int64)
    ja = A.indices.astype(np.int64)
    aa = np.ascontiguousarray(A.data, dtype=np.complex128)
    # point source nearest the axis midpoint
    mid = gid(int(np.argmin(np.abs(gx))), int(np.argmin(np.abs(gx))), nz // 2)
    b = np.zeros(n, dtype=np.complex128)
    b[remap[mid] if remap[mid] >= 0 else n // 2] = complex(source)
    return n, ia, ja, aa, b


# Named BASELINE.json configurations.  C1 is exactly the reference
# CPU path: load_problem_config-style dim=3, cells=33, frequency=1.5 (k = 3*pi).
CONFIGS = {
    "C1": dict(kind="fd", dim=3, cells=33, frequency=1.5, damping=0.0, tol=1e-8),
    "C3": dict(kind="p1fe", m=108, length=2.0, wavelengths=2.0, damping=0.1, tol=1e-8),
    "C4": dict(kind="27pt", m=200, k2=100.0, damping=0.05, tol=1e-8),
    "C5": dict(kind="fd", dim=3, cells=257, frequency=257 / 12.0, damping=0.3, tol=1e-8),
}


def config_problem(name: str, scale: int | None = None):
    """Build a named configuration; ``scale`` overrides the grid size (tests)."""
    c = CONFIGS[name]
    if c["kind"] == "fd":
        cells = scale + 1 if scale else c["cells"]
        freq = c["frequency"] if not scale or name != "C5" else cells / 12.0
        return helmholtz_fd(c["dim"], cells, frequency=freq, damping=c["damping"])
    m = scale or c["m"]
    if c["kind"] == "p1fe":
        return cylinder_p1fe(m, c["length"], c["wavelengths"], c["damping"])
    return helmholtz_27pt(m, k2=c["k2"], damping=c["damping"])
