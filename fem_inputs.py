"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no basis, quadrature, geometry
or operator); it only defines the workload presets of BASELINE.json and the
counter-based random generator both sides draw from (SURVEY.md §8c reading
R14).  The CUDA path implements the same generator independently (splitmix64
in `paper_1611_03029_b200/csrc/kernels_mg.cu`, `u01_splitmix`) for the random start vector of the eigenvalue estimate
(SURVEY.md §8c O6); the oracle uses `uniform_pm1` below.

Generator (R14): x_i = 2 * ((z_i >> 11) * 2^-53) - 1, z_i = splitmix64 output
number i (0-based) of the stream seeded with `seed`, i = GLOBAL index, so the
vector does not depend on the partition.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Tuple

import numpy as np

GOLDEN_GAMMA = np.uint64(0x9E3779B97F4A7C15)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)

CG, SIPG = 0, 1
DIRICHLET, NEUMANN = 0, 1


def splitmix64(seed: int, start: int, count: int) -> np.ndarray:
    """Outputs start..start+count-1 of the splitmix64 stream seeded with `seed`."""
    with np.errstate(over="ignore"):
        i = np.arange(start, start + count, dtype=np.uint64) + np.uint64(1)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GOLDEN_GAMMA
        z = (z ^ (z >> np.uint64(30))) * MIX1
        z = (z ^ (z >> np.uint64(27))) * MIX2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform_pm1(seed: int, count: int, start: int = 0) -> np.ndarray:
    """x_i ~ U[-1, 1) from splitmix64 (reading R14), float64."""
    z = splitmix64(seed, start, count)
    return 2.0 * ((z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53) - 1.0


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration."""
    name: str
    method: int              # CG or SIPG
    degree: int
    cells: Tuple[int, int, int]
    deform_eps: float
    seed: int                # random x seed (R14)
    rhs: str                 # "manufactured" (O8) or "random_apply" (R15)
    lo: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    hi: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    bc: Tuple[int, ...] = field(default=(DIRICHLET,) * 6)
    penalty_factor: float = 2.0
    description: str = ""

    def n_dofs(self) -> int:
        k, (nx, ny, nz) = self.degree, self.cells
        if self.method == CG:
            return (k * nx + 1) * (k * ny + 1) * (k * nz + 1)
        return nx * ny * nz * (k + 1) ** 3


# BASELINE.json configs[0..4] = C1..C5.
C1 = Workload("C1", CG, 2, (8, 8, 8), 0.0, 0, "random_apply",
              description="CG Q2 Cartesian 8^3, apply + diagonal, x~U[-1,1) seed 0")
C2 = Workload("C2", CG, 4, (32, 32, 32), 0.05, 0, "manufactured",
              description="CG Q4 deformed 32^3 (eps=0.05), GMG-CG to 1e-10")
C3 = Workload("C3", SIPG, 4, (32, 32, 32), 0.0, 0, "manufactured",
              description="SIPG Q4 Cartesian 32^3, sigma=2(k+1)^2/h, GMG-CG to 1e-10")
C4 = Workload("C4", CG, 4, (128, 128, 128), 0.0, 7, "random_apply",
              description="CG Q4 Cartesian 128^3, x~U[-1,1) seed 7, b=A x7 (R15)")
C5 = Workload("C5", SIPG, 6, (64, 64, 64), 0.05, 0, "manufactured",
              description="SIPG Q6 deformed 64^3 (eps=0.05), GMG-CG to 1e-10")
CONFIGS = {w.name: w for w in (C1, C2, C3, C4, C5)}


def scaled(w: Workload, cells: Tuple[int, int, int], name: str | None = None) -> Workload:
    """Same workload recipe on a smaller mesh (parity cases the oracle finishes in seconds)."""
    return Workload(name or f"{w.name}@{cells[0]}x{cells[1]}x{cells[2]}", w.method, w.degree,
                    cells, w.deform_eps, w.seed, w.rhs, w.lo, w.hi, w.bc,
                    w.penalty_factor, w.description)
