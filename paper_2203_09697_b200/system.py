"""Atomic systems (positions + atomic numbers) and the synthetic generator.

AtomicSystem keeps the reference's validation rules (egn/system.py:23-58);
random_cloud is the reference's rejection sampler (egn/system.py:129-166),
used to produce identical synthetic inputs on the GPU box, where the
reference package is not installed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MIN_SEPARATION = 1e-12
CLOUD_SPECIES = (1, 6, 7, 8, 14, 29)


@dataclass(frozen=True)
class AtomicSystem:
    """positions, atomic numbers (egn/system.py:23-58) and, as an extension for periodic
    slabs, an optional cell (3x3, rows = lattice vectors) with per-axis
    periodic flags.  cell None (the reference's only case) = non-periodic."""

    positions: np.ndarray
    atomic_numbers: np.ndarray
    identifier: str | None = None
    cell: np.ndarray | None = None
    pbc: tuple = (False, False, False)

    def __post_init__(self):
        pos = np.asarray(self.positions, dtype=np.float64)
        z = np.asarray(self.atomic_numbers, dtype=np.int64)
        object.__setattr__(self, "positions", pos)
        object.__setattr__(self, "atomic_numbers", z)
        pbc = tuple(bool(x) for x in np.broadcast_to(np.asarray(self.pbc, dtype=bool), (3,)))
        object.__setattr__(self, "pbc", pbc)
        if self.cell is not None:
            cell = np.asarray(self.cell, dtype=np.float64)
            if cell.shape != (3, 3) or not np.all(np.isfinite(cell)):
                raise ValueError("cell must be a finite 3x3 matrix (rows = lattice vectors)")
            if any(pbc) and abs(np.linalg.det(cell)) <= 1e-12:
                raise ValueError("periodic cell must have nonzero volume")
            object.__setattr__(self, "cell", cell)
        elif any(pbc):
            raise ValueError("periodic axes need a cell")
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise ValueError(f"positions must have shape (n, 3), got {pos.shape}")
        if z.shape != (pos.shape[0],):
            raise ValueError("positions and atomic_numbers disagree on atom count")
        if pos.shape[0] < 1:
            raise ValueError("system must contain at least one atom")
        if np.any(z < 1):
            raise ValueError("atomic numbers must be >= 1")
        if not np.all(np.isfinite(pos)):
            raise ValueError("positions must be finite")

    @property
    def n(self) -> int:
        return self.positions.shape[0]

    @property
    def periodic(self) -> bool:
        return any(self.pbc)

    def with_positions(self, positions) -> "AtomicSystem":
        return AtomicSystem(positions, self.atomic_numbers, self.identifier, self.cell, self.pbc)


def random_cloud(n: int, density: float, rng: np.random.Generator, max_tries_per_atom: int = 500) -> AtomicSystem:
    if n < 1:
        raise ValueError("n must be >= 1")
    if density <= 0:
        raise ValueError("density must be positive")
    min_dist = 0.8 * density ** (-1.0 / 3.0)
    side = (n / density) ** (1.0 / 3.0)
    placed = np.empty((n, 3))
    for i in range(n):
        for _ in range(max_tries_per_atom):
            cand = rng.uniform(0.0, side, size=3)
            if i == 0 or np.sqrt(((placed[:i] - cand) ** 2).sum(axis=1)).min() >= min_dist:
                placed[i] = cand
                break
        else:
            raise RuntimeError(f"could not place atom {i + 1}/{n} at density {density} "
                               f"after {max_tries_per_atom} tries")
    z = rng.choice(CLOUD_SPECIES, size=n).astype(np.int64)
    return AtomicSystem(placed, z)
