"""Host-side data types of the shifted-solve path.

Mirrors the reference's `Grid`, `Model` and `Problem`
(/root/reference/pkg/src/rbainv/mesh.py:36-162) field for field, so a
reference `rbainv.Problem` and a problem built here are interchangeable on
both sides of the drop-in boundary.  Two fields are added for the 3-D
edge-element problems the reference cannot build:

* ``Problem.sources``  (S, N) -- one row per transmitter loop; ``f`` is row 0.
* ``Problem.dof_coords`` (N, 3) -- edge midpoints, used by the host
  nested-dissection ordering (geometric separators).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

__all__ = ["Grid", "Model", "Problem"]


@dataclass(frozen=True)
class Grid:
    """Cell/face structure (reference mesh.py:36-56).

    For 3-D edge elements ``nodes`` are mesh vertices, ``cells`` the tet
    vertex quadruples, and ``dof_of_node`` holds the dof of each mesh *edge*
    (-1 on the PEC boundary)."""

    dimension: int
    nodes: np.ndarray
    cells: np.ndarray
    cell_measure: np.ndarray
    face_cells: np.ndarray
    face_measure: np.ndarray
    dof_of_node: np.ndarray
    dof_count: int
    cell_tags: np.ndarray = None

    @property
    def cell_count(self) -> int:
        return self.cells.shape[0]

    def cell_centroids(self) -> np.ndarray:
        return self.nodes[self.cells].mean(axis=1)


@dataclass
class Model:
    """Log-conductivity per cell plus the reference model (mesh.py:62-88)."""

    m: np.ndarray
    m_ref: np.ndarray

    def __post_init__(self):
        self.m = np.asarray(self.m, dtype=float).copy()
        self.m_ref = np.asarray(self.m_ref, dtype=float).copy()
        if self.m.shape != self.m_ref.shape or self.m.ndim != 1:
            raise ValueError("m and m_ref must be 1-D arrays of equal length")
        if not (np.all(np.isfinite(self.m)) and np.all(np.isfinite(self.m_ref))):
            raise ValueError("model entries must be finite")

    @property
    def cell_count(self) -> int:
        return self.m.size

    def sigma(self) -> np.ndarray:
        return np.exp(self.m)

    def version_tag(self) -> str:
        # same cache key as the reference (mesh.py:84-85)
        return hashlib.sha1(self.m.tobytes()).hexdigest()[:16]

    def perturbed(self, delta: np.ndarray, scale: float = 1.0) -> "Model":
        return Model(self.m + scale * delta, self.m_ref)


@dataclass
class Problem:
    """Assembled static operators of one mesh (mesh.py:127-162)."""

    grid: Grid
    K: sp.csr_matrix
    cell_dofs: np.ndarray
    mass_local: np.ndarray
    stiff_local: np.ndarray
    f: np.ndarray
    Q: sp.csr_matrix
    receivers: np.ndarray
    spec: object
    _scatter: tuple = None
    sources: np.ndarray = None
    dof_coords: np.ndarray = None
    m_true: np.ndarray = None
    sigma_background: float = 0.01
    extra: dict = field(default_factory=dict)

    @property
    def dof_count(self) -> int:
        return self.grid.dof_count

    @property
    def receiver_count(self) -> int:
        return self.Q.shape[0]

    @property
    def source_count(self) -> int:
        return 1 if self.sources is None else self.sources.shape[0]

    def source_matrix(self) -> np.ndarray:
        """(S, N) right-hand sides; the reference's single ``f`` is S=1."""
        if self.sources is None:
            return np.asarray(self.f, dtype=float)[None, :]
        return self.sources

    def reference_model(self) -> Model:
        sb = getattr(self.spec, "sigma_background", self.sigma_background)
        m_ref = np.full(self.grid.cell_count, np.log(sb))
        return Model(m_ref.copy(), m_ref)

    def true_model(self) -> Model:
        ref = self.reference_model()
        if self.m_true is None:
            return ref
        return Model(self.m_true, ref.m_ref)

    def ensure_scatter(self) -> tuple:
        """The reference's cached COO pattern for ``assemble_M``
        (mesh.py:319-323,342-343); built lazily because only the CPU
        reference consumes it."""
        if self._scatter is None:
            k = self.cell_dofs.shape[1]
            rows = np.repeat(self.cell_dofs, k, axis=1).ravel()
            cols = np.tile(self.cell_dofs, (1, k)).ravel()
            keep = (rows >= 0) & (cols >= 0)
            cell_of = np.repeat(np.arange(self.grid.cell_count), k * k)[keep]
            self._scatter = (rows[keep], cols[keep], keep, cell_of)
        return self._scatter
