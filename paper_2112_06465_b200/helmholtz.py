"""Helmholtz test systems for the bench CLI's ``--problem`` (host setup;
drop-in for the constant-field part of zlinalg helmholtz.py).

``assemble`` builds the same (2*dim+1)-point system as the reference
(helmholtz.py:115-168) -- bitwise: same scalars, same CSR order, same
right-hand side accumulation -- but vectorised (problems.helmholtz_fd)
instead of a per-row Python loop, which needs ~4.5 s per million rows.
Constant ``source`` / ``dirichlet_value`` fields are supported; callable
fields and ``velocity_field`` (the reference's manufactured-solution
machinery, out of scope per SURVEY.md section 2) raise ParameterError.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import problems
from .errors import ParameterError, ParseError
from .sparse import CsrMatrix
from .vecops import ZVector

__all__ = ["HelmholtzProblem", "assemble", "load_problem_config"]


@dataclass(frozen=True)
class HelmholtzProblem:
    """Box-domain acoustic problem (helmholtz.py:31-106): ``cells_per_axis``
    intervals per axis, spacing ``domain_length / cells_per_axis``."""

    dim: int
    cells_per_axis: int
    domain_length: float = 1.0
    frequency: float = 0.0
    velocity: float = 1.0
    dirichlet_value: object = 0j
    source: object = 0j
    velocity_field: object = None

    def __post_init__(self):
        checks = (  # (condition, message) -- the reference's ParameterError texts (helmholtz.py:52-65)
            (self.dim in (1, 2, 3), f"dim must be 1, 2, or 3, got {self.dim!r}"),
            (self.cells_per_axis >= 3, f"cells_per_axis must be at least 3, got {self.cells_per_axis!r}"),
            (self.domain_length > 0 and math.isfinite(self.domain_length),
             f"domain_length must be positive, got {self.domain_length!r}"),
            (self.velocity > 0 and math.isfinite(self.velocity), f"velocity must be positive, got {self.velocity!r}"),
            (self.frequency >= 0 and math.isfinite(self.frequency),
             f"frequency must be nonnegative, got {self.frequency!r}"),
        )
        for ok, message in checks:
            if not ok:
                raise ParameterError(message)

    @property
    def wavenumber(self) -> float:
        return 2.0 * math.pi * self.frequency / self.velocity

    @property
    def spacing(self) -> float:
        return self.domain_length / self.cells_per_axis

    @property
    def interior_per_axis(self) -> int:
        return self.cells_per_axis - 1

    @property
    def n_unknowns(self) -> int:
        return self.interior_per_axis**self.dim


def assemble(p: HelmholtzProblem):
    """(CsrMatrix, ZVector) of problem ``p`` (helmholtz.py:115-168) for
    constant fields.  Right-hand side per row: 0 + inv_h2 * g once per
    boundary-adjacent side (axis order), then + source -- the reference's
    accumulation, so the bits match."""
    if callable(p.source) or callable(p.dirichlet_value) or p.velocity_field is not None:
        raise ParameterError("callable fields / velocity_field are not supported by the device drop-in")
    n, ia, ja, aa, _ = problems.helmholtz_fd(p.dim, p.cells_per_axis, p.domain_length, p.frequency, p.velocity,
                                             0.0, 0j)
    m = p.interior_per_axis
    h = p.spacing
    inv_h2 = 1.0 / (h * h)
    contrib = inv_h2 * complex(p.dirichlet_value)
    flat = np.arange(n, dtype=np.int64)
    sides = np.zeros(n, dtype=np.int64)
    for a in range(p.dim):
        c = (flat // m**a) % m
        sides += (c == 0).astype(np.int64) + (c == m - 1).astype(np.int64)
    rhs = np.zeros(n, dtype=np.complex128)
    for k in range(int(sides.max()) if n else 0):
        rhs[sides > k] += contrib
    rhs += complex(p.source)
    return CsrMatrix(n, n, aa, ja, ia, validate=False), ZVector(rhs)


_KEY_TYPES = {"dim": int, "cells": int, "length": float, "frequency": float, "velocity": float}


def _config_values(path):
    """key -> typed value of a key=value file ('#' comments), ParseError with line numbers."""
    values = {}
    with open(path, "r", encoding="ascii") as fh:
        for lineno, raw in enumerate(fh, start=1):
            text = raw.split("#", 1)[0].strip()
            if not text:
                continue
            key, eq, val = text.partition("=")
            if not eq:
                raise ParseError(f"expected key=value, got {text!r}", line=lineno)
            key, val = key.strip().lower(), val.strip()
            convert = _KEY_TYPES.get(key)
            if convert is None:
                raise ParseError(f"unknown key {key!r}", line=lineno)
            try:
                values[key] = convert(val)
            except ValueError:
                raise ParseError(f"bad value for {key}: {val!r}", line=lineno) from None
    return values


def load_problem_config(path) -> HelmholtzProblem:
    """Problem file (helmholtz.py:211-249): dim and cells required; length,
    frequency, velocity default to 1, 0, 1; unit interior source."""
    v = _config_values(path)
    missing = [k for k in ("dim", "cells") if k not in v]
    if missing:
        raise ParseError(f"missing required key {missing[0]!r}")
    try:
        return HelmholtzProblem(dim=v["dim"], cells_per_axis=v["cells"], domain_length=v.get("length", 1.0),
                                frequency=v.get("frequency", 0.0), velocity=v.get("velocity", 1.0), source=1 + 0j)
    except ParameterError as exc:
        raise ParseError(str(exc)) from exc
