"""Synthetic Helmholtz systems for the BASELINE configurations (host-side setup).

Not on the hot path: these build the CSR inputs (``ia``/``ja`` int64,
``aa`` complex128, exactly the reference ``CsrMatrix`` layout,
``sparse.py:60-103``) that the solver consumes.  They are vectorised numpy
replacements for the reference's per-row Python loop
(``helmholtz.py:206-259``), which needs ~4.5 s per million rows.

* :func:`helmholtz_fd` -- the reference's (2*dim+1)-point central-difference
  stencil with a unit interior source and zero Dirichlet data, i.e. what
  ``assemble(load_problem_config(...))`` produces (``helmholtz.py:302-339``).
  With ``damping == 0`` the arrays are bitwise identical to the reference
  (checked by ``tests/test_problems.py`` against fixtures made from it).
  ``damping = eps`` shifts the diagonal by ``-i * eps * k^2`` (complex
  damping ``k^2 (1 + i eps)``; BASELINE configs C1/C5).
* :func:`helmholtz_27pt` -- 27-point stencil, diagonal ``26/(3h^2) - k^2(1+i eps)``,
  off-diagonals ``-1/(3h^2)`` (BASELINE config C4).
* :func:`config_problem` -- the named BASELINE configurations.
"""
from __future__ import annotations

import math

import numpy as np

__all__ = ["helmholtz_fd", "helmholtz_27pt", "config_problem", "CONFIGS"]


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


# Named BASELINE.json configurations.  C1 is exactly the reference
# CPU path: load_problem_config-style dim=3, cells=33, frequency=1.5 (k = 3*pi).
CONFIGS = {
    "C1": dict(kind="fd", dim=3, cells=33, frequency=1.5, damping=0.0, tol=1e-8),
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
    return helmholtz_27pt(m, k2=c["k2"], damping=c["damping"])
