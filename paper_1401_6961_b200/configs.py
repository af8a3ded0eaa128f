"""Synthetic BASELINE systems -- host-side input prep.

The paper's (H2O)_n B3LYP/6-31G** droplets are not available; BASELINE.json
names seeded synthetic stand-ins, generated here deterministically:

  c1  32 s centers on a 4x4x2 lattice, 1.4 A, +-0.1 A jitter (1 shell each)
  c2  256-center chain, 1.5 A, +-0.05 A jitter; even = heavy (s3, s1, p2),
      odd = light (s3)
  c3  256 three-center units in a cube at 0.0334 units/A^3
  c4  the c3 recipe with 512 units (tau sweep)
  c5  the c3 recipe with 4096 units (28,672 functions)

Density (all configs): P_ii = 1, P_ij = s_ij exp(-|R_i - R_j| / 1.5 A) with
s_ij = +-U[0.5, 1] from a counter-based SplitMix64 stream (seed + 100), drawn
per function pair in post-Hilbert order.  Geometry seed = config index.
Units are Bohr internally (BOHR_PER_ANGSTROM, basis.py:15 of the reference).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .basis import BOHR_PER_ANGSTROM, Atom, BasisSystem, GaussianShell, assign_offsets
from .inputs import SplitMix64, hilbert_order

LIGHT_S3 = [(3.42525, 0.15433), (0.62391, 0.53533), (0.16886, 0.44463)]
HEAVY_S3 = [(5.0, 0.15433), (1.2, 0.53533), (0.35, 0.44463)]
HEAVY_S1 = [(0.25, 1.0)]
HEAVY_P2 = [(1.5, 0.5), (0.4, 0.5)]

OH_BOHR = 1.81
HOH_ANGLE = math.radians(104.5)
MIN_HEAVY_SEPARATION = 4.0
UNITS_PER_A3 = 0.0334
DECAY_A = 1.5

GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def splitmix64_block(seed: int, start: int, count: int) -> np.ndarray:
    """Outputs start..start+count-1 of SplitMix64(seed), vectorised.

    Output k equals mix(seed + (k+1) * golden mod 2^64), exactly what the
    sequential generator (basis.py:120-125) yields on its k-th call.
    """
    k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & M64) + k * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


@dataclass
class Config:
    name: str
    system: BasisSystem
    P: np.ndarray
    tau_2e: float = 1e-8
    tau_ovlp: float = 1e-11
    leaf_size: int = 10

    @property
    def n_functions(self):
        return self.system.n_functions

    @property
    def n_shells(self):
        return self.system.n_shells


def decay_density(system: BasisSystem, seed: int) -> np.ndarray:
    """P_ij = s_ij exp(-r_ij / 1.5 A), P_ii = 1, exactly symmetric."""
    n = system.n_functions
    ctr = np.empty((n, 3))
    for sh in system.shells:
        ctr[sh.function_offset:sh.function_offset + sh.n_functions] = sh.center
    decay = 1.0 / (DECAY_A * BOHR_PER_ANGSTROM)
    P = np.empty((n, n))
    rows = max(1, (1 << 22) // max(n, 1))
    for r0 in range(0, n, rows):
        r1 = min(n, r0 + rows)
        d = ctr[r0:r1, None, :] - ctr[None, :, :]
        dist = np.sqrt(np.einsum("ijk,ijk->ij", d, d))
        z = splitmix64_block(seed, r0 * n, (r1 - r0) * n).reshape(r1 - r0, n)
        mag = 0.5 + 0.5 * ((z & np.uint64((1 << 53) - 1)).astype(np.float64) / 2.0 ** 53)
        sign = np.where((z >> np.uint64(63)) != 0, -1.0, 1.0)
        P[r0:r1] = sign * mag * np.exp(-decay * dist)
    iu = np.triu_indices(n, 1)
    P[(iu[1], iu[0])] = P[iu]          # mirror the upper triangle
    np.fill_diagonal(P, 1.0)
    return P


def decay_density_device(system: BasisSystem, seed: int, device="cuda"):
    """decay_density on the GPU (torch): same recipe and SplitMix64 stream.

    Values agree with the numpy version up to the last-ulp rounding of
    exp/sqrt; used by bench.py so that the 6.6 GB c5 density is generated in
    well under a second instead of ~1 minute on the host.
    """
    import torch
    n = system.n_functions
    ctr_h = np.empty((n, 3))
    for sh in system.shells:
        ctr_h[sh.function_offset:sh.function_offset + sh.n_functions] = sh.center
    ctr = torch.from_numpy(ctr_h).to(device)
    decay = 1.0 / (DECAY_A * BOHR_PER_ANGSTROM)
    P = torch.empty((n, n), dtype=torch.float64, device=device)

    def as_i64(x):
        x &= M64
        return x - (1 << 64) if x >= (1 << 63) else x

    def srl(z, s):  # logical right shift of int64 bit patterns
        return (z >> s) & ((1 << (64 - s)) - 1)

    rows = max(1, (1 << 25) // max(n, 1))
    g = as_i64(GOLDEN)
    m1, m2 = as_i64(0xBF58476D1CE4E5B9), as_i64(0x94D049BB133111EB)
    for r0 in range(0, n, rows):
        r1 = min(n, r0 + rows)
        d = ctr[r0:r1, None, :] - ctr[None, :, :]
        dist = torch.sqrt((d * d).sum(-1))
        k = torch.arange(r0 * n + 1, r1 * n + 1, dtype=torch.int64, device=device)
        z = as_i64(seed) + k * g
        z = (z ^ srl(z, 30)) * m1
        z = (z ^ srl(z, 27)) * m2
        z = z ^ srl(z, 31)
        mag = 0.5 + 0.5 * ((z & ((1 << 53) - 1)).to(torch.float64) / 2.0 ** 53)
        sign = torch.where(z < 0, -1.0, 1.0).to(torch.float64)
        P[r0:r1] = (sign * mag).view(r1 - r0, n) * torch.exp(-decay * dist)
        # mirror the upper triangle: earlier rows' upper parts, then this block
        if r0:
            P[r0:r1, :r0] = P[:r0, r0:r1].T
        blk = P[r0:r1, r0:r1]
        P[r0:r1, r0:r1] = torch.triu(blk) + torch.triu(blk, 1).T
    P.fill_diagonal_(1.0)
    return P


def _finish(name, shells, atoms, seed, host_density=True, **kw) -> Config:
    system = BasisSystem(shells=assign_offsets(shells), atoms=atoms)
    system, _ = hilbert_order(system)
    P = decay_density(system, seed + 100) if host_density else None
    cfg = Config(name=name, system=system, P=P, **kw)
    cfg.density_seed = seed + 100
    return cfg


def _heavy(center):
    return [GaussianShell(center=center.copy(), primitives=HEAVY_S3),
            GaussianShell(center=center.copy(), primitives=HEAVY_S1),
            GaussianShell(center=center.copy(), primitives=HEAVY_P2, l=1)]


def _light(center):
    return [GaussianShell(center=center.copy(), primitives=LIGHT_S3)]


def config1(seed: int = 1) -> Config:
    rng = SplitMix64(seed)
    shells, atoms = [], []
    for ix in range(4):
        for iy in range(4):
            for iz in range(2):
                pos = np.array([ix, iy, iz], dtype=float) * 1.4
                pos += np.array([(2.0 * rng.uniform() - 1.0) * 0.1 for _ in range(3)])
                pos *= BOHR_PER_ANGSTROM
                atoms.append(Atom("H", pos))
                shells += _light(pos)
    return _finish("c1", shells, atoms, seed)


def config2(seed: int = 2, n_centers: int = 256) -> Config:
    rng = SplitMix64(seed)
    shells, atoms = [], []
    for c in range(n_centers):
        pos = np.array([c * 1.5, 0.0, 0.0])
        pos += np.array([(2.0 * rng.uniform() - 1.0) * 0.05 for _ in range(3)])
        pos *= BOHR_PER_ANGSTROM
        if c % 2 == 0:
            atoms.append(Atom("O", pos))
            shells += _heavy(pos)
        else:
            atoms.append(Atom("H", pos))
            shells += _light(pos)
    return _finish("c2", shells, atoms, seed)


def cube_cluster(n_units: int, seed: int, name: str, host_density: bool = True) -> Config:
    """Units packed in a cube at 0.0334 units/A^3, heavy-heavy >= 4 Bohr."""
    rng = SplitMix64(seed)
    side = (n_units / UNITS_PER_A3) ** (1.0 / 3.0) * BOHR_PER_ANGSTROM
    centers = np.empty((n_units, 3))
    placed = 0
    while placed < n_units:
        for _ in range(100000):
            cand = np.array([rng.uniform() * side for _ in range(3)])
            if placed == 0:
                break
            d = centers[:placed] - cand
            if np.min(np.einsum("ij,ij->i", d, d)) >= MIN_HEAVY_SEPARATION ** 2:
                break
        else:
            raise RuntimeError("cube packing failed")
        centers[placed] = cand
        placed += 1
    shells, atoms = [], []
    for ctr in centers:
        e1 = rng.unit_vector()
        raw = rng.unit_vector()
        e2 = raw - np.dot(raw, e1) * e1
        while np.linalg.norm(e2) < 1e-8:
            raw = rng.unit_vector()
            e2 = raw - np.dot(raw, e1) * e1
        e2 /= np.linalg.norm(e2)
        h1 = ctr + OH_BOHR * e1
        h2 = ctr + OH_BOHR * (math.cos(HOH_ANGLE) * e1 + math.sin(HOH_ANGLE) * e2)
        atoms += [Atom("O", ctr), Atom("H", h1), Atom("H", h2)]
        shells += _heavy(ctr) + _light(h1) + _light(h2)
    return _finish(name, shells, atoms, seed, host_density)


def config3(seed: int = 3, n_units: int = 256, host_density: bool = True) -> Config:
    return cube_cluster(n_units, seed, "c3", host_density)


def config4(seed: int = 4, n_units: int = 512, tau_2e: float = 1e-8,
            host_density: bool = True) -> Config:
    cfg = cube_cluster(n_units, seed, "c4", host_density)
    cfg.tau_2e = tau_2e
    cfg.tau_ovlp = 1e-3 * tau_2e
    return cfg


def config5(seed: int = 5, n_units: int = 4096, host_density: bool = True) -> Config:
    return cube_cluster(n_units, seed, "c5", host_density)


def make(name: str, **kw) -> Config:
    return {"c1": config1, "c2": config2, "c3": config3, "c4": config4,
            "c5": config5}[name](**kw)
