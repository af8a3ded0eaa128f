"""Synthetic inputs on the reference's CLI path (outside the exchange hot path).

The reference CLI builds its systems from a seeded water-like cluster, an
exponential-decay density and a Hilbert pre-order (hexfock basis.py:112-331,
density.py:20-51); the run-report harness (harness.py) and the test suite
need the same inputs, value for value, so that reference-written golden
fixtures apply.  What is restated:

* the SplitMix64 stream (a public generator): draw k of seed s is the
  finaliser of s + k * 0x9E3779B97F4A7C15 mod 2^64 -- here a counter, not a
  mutable state;
* cluster geometry: heavy centres by rejection sampling in the sphere of the
  water number density (>= 4 Bohr apart), two light atoms per heavy at
  1.81 Bohr / 104.5 degrees in a random frame -- the same draws in the same
  order and the same floating-point expressions as the reference;
* density P_ij = d exp(-gamma r_ij) over function centres;
* Hilbert order: Skilling's transposed-axes transform applied to all lattice
  points at once (numpy, vectorised over shells) and a stable sort, the
  reference's lattice rounding; unlike the reference, shells keep ``l``
  (its reorder silently resets n_functions to 1).
The device drivers never call into this module.
"""

from __future__ import annotations

import math

import numpy as np

from .basis import (BOHR_PER_ANGSTROM, Atom, BasisSystem, GaussianShell, InvalidArgumentError,
                    UnsupportedElementError, assign_offsets)

WATER_NUMBER_DENSITY = 0.0334 / BOHR_PER_ANGSTROM ** 3
OH_DISTANCE = 1.81          # Bohr
HOH_ANGLE = math.radians(104.5)
MIN_HEAVY_SEPARATION = 4.0  # Bohr
DEFAULT_GAMMA = 2.0

HEAVY_SHELLS = [
    [(130.7093, 0.15432897), (23.8089, 0.53532814), (6.4436, 0.44463454)],
    [(0.27, 1.0)],
]
LIGHT_SHELLS = [[(1.24, 1.0)]]
DEFAULT_SHELL_TABLE = {"O": HEAVY_SHELLS, "H": LIGHT_SHELLS}

_M64 = (1 << 64) - 1
_GAMMA64 = 0x9E3779B97F4A7C15


def _mix(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


class SplitMix64:
    """Counter-based SplitMix64 stream: the k-th draw is _mix(seed + k * gamma)."""

    __slots__ = ("seed", "count")

    def __init__(self, seed: int):
        self.seed = seed & _M64
        self.count = 0

    def next_u64(self) -> int:
        self.count += 1
        return _mix((self.seed + self.count * _GAMMA64) & _M64)

    def uniform(self) -> float:
        return self.next_u64() / 2.0 ** 64

    def symmetric3(self, scale: float = 1.0) -> np.ndarray:
        """Three draws mapped to [-scale, scale)."""
        return np.array([(2.0 * self.uniform() - 1.0) * scale for _ in range(3)])

    def unit_vector(self) -> np.ndarray:
        while True:
            v = self.symmetric3()
            n2 = float(np.dot(v, v))
            if 1e-8 < n2 <= 1.0:
                return v / math.sqrt(n2)


def shells_for(element, center, table=None):
    """Shells attached to one atom; table entries are primitive lists (s) or (l, primitives)."""
    table = DEFAULT_SHELL_TABLE if table is None else table
    try:
        entries = table[element]
    except KeyError:
        raise UnsupportedElementError(f"no shells defined for element {element!r}") from None
    out = []
    for entry in entries:
        l, prims = entry if (isinstance(entry, tuple) and isinstance(entry[0], int)) else (0, entry)
        out.append(GaussianShell(center=np.array(center, dtype=float), primitives=list(prims), l=l))
    return out


def _heavy_centres(rng: SplitMix64, n: int, radius: float, spaced: bool):
    r2 = radius * radius
    centres = [np.zeros(3)]
    while len(centres) < n:
        for _ in range(100000):
            while True:                       # uniform point in the ball
                cand = rng.symmetric3(radius)
                if np.dot(cand, cand) <= r2:
                    break
            if not spaced or all(np.linalg.norm(cand - c) >= MIN_HEAVY_SEPARATION for c in centres):
                break
        else:
            raise InvalidArgumentError("packing failed; density/min-distance constraints unsatisfiable")
        centres.append(cand)
    return centres


def _water_frame(rng: SplitMix64, ctr: np.ndarray):
    e1 = rng.unit_vector()
    while True:
        raw = rng.unit_vector()
        e2 = raw - np.dot(raw, e1) * e1
        if np.linalg.norm(e2) >= 1e-8:
            break
    e2 /= np.linalg.norm(e2)
    return (ctr + OH_DISTANCE * e1,
            ctr + OH_DISTANCE * (math.cos(HOH_ANGLE) * e1 + math.sin(HOH_ANGLE) * e2))


def generate_cluster(n_molecules: int, seed: int, model: str = "water_like") -> BasisSystem:
    """Seeded water-like cluster in a sphere (the reference's generate_cluster inputs)."""
    if n_molecules < 1:
        raise InvalidArgumentError("n_molecules must be >= 1")
    if model not in ("water_like", "uniform_blob"):
        raise InvalidArgumentError(f"unknown cluster model {model!r}")
    rng = SplitMix64(seed)
    radius = (3.0 * (n_molecules / WATER_NUMBER_DENSITY) / (4.0 * math.pi)) ** (1.0 / 3.0)
    blob = model == "uniform_blob"
    atoms, shells = [], []
    for ctr in _heavy_centres(rng, n_molecules, radius, spaced=not blob):
        atoms.append(Atom("O", ctr))
        shells += shells_for("O", ctr)
        if blob:
            continue
        for h in _water_frame(rng, ctr):
            atoms.append(Atom("H", h))
        shells += shells_for("H", atoms[-2].position) + shells_for("H", atoms[-1].position)
    return BasisSystem(shells=assign_offsets(shells), atoms=atoms)


class DensityModel:
    """Exponential-decay density stand-in (kind 'exp_decay' only)."""

    __slots__ = ("kind", "gamma", "diagonal")

    def __init__(self, kind: str = "exp_decay", gamma: float = DEFAULT_GAMMA, diagonal: float = 1.0):
        if kind != "exp_decay":
            raise InvalidArgumentError(f"unknown density kind {kind!r}")
        if gamma <= 0.0:
            raise InvalidArgumentError("gamma must be positive")
        self.kind, self.gamma, self.diagonal = kind, gamma, diagonal


def build_density(system: BasisSystem, model: DensityModel) -> np.ndarray:
    """P_ij = diagonal * exp(-gamma |r_i - r_j|) over function centres, exactly symmetric."""
    fc = np.concatenate([np.repeat(sh.center[None, :], sh.n_functions, axis=0) for sh in system.shells])
    d = fc[:, None, :] - fc[None, :, :]
    r = np.sqrt(np.einsum("ijk,ijk->ij", d, d))
    r = np.maximum(r, r.T)
    return model.diagonal * np.exp(-model.gamma * r)


def hilbert_keys(lattice: np.ndarray, bits: int) -> np.ndarray:
    """Skilling's Hilbert index of each row of an (n, 3) integer lattice, vectorised."""
    x = [lattice[:, k].astype(np.int64).copy() for k in range(3)]
    top = 1 << (bits - 1)
    q = top
    while q > 1:                       # inverse undo of the excess work
        p = q - 1
        for i in range(3):
            hi = (x[i] & q) != 0
            t = np.where(hi, 0, (x[0] ^ x[i]) & p)
            x[0] = np.where(hi, x[0] ^ p, x[0] ^ t)
            if i:
                x[i] = x[i] ^ t
        q >>= 1
    x[1] ^= x[0]                       # Gray encode
    x[2] ^= x[1]
    t = np.zeros_like(x[0])
    q = top
    while q > 1:
        t = np.where((x[2] & q) != 0, t ^ (q - 1), t)
        q >>= 1
    x = [v ^ t for v in x]
    key = np.zeros(len(lattice), dtype=np.int64)
    for b in range(bits - 1, -1, -1):  # interleave: axis 0 is the most significant
        for i in range(3):
            key = (key << 1) | ((x[i] >> b) & 1)
    return key


def hilbert_order(system: BasisSystem, bits_per_axis: int = 10):
    """Stable sort of the shells by Hilbert key; returns (system, shell permutation)."""
    if not 1 <= bits_per_axis <= 20:
        raise InvalidArgumentError("bits_per_axis must be in [1, 20]")
    centres = np.array([sh.center for sh in system.shells])
    lo = centres.min(axis=0)
    extent = centres.max(axis=0) - lo
    side = (1 << bits_per_axis) - 1
    lattice = np.zeros_like(centres, dtype=np.int64)
    for ax in range(3):
        if extent[ax] > 0.0:
            lattice[:, ax] = np.rint((centres[:, ax] - lo[ax]) / extent[ax] * side)
    perm = np.argsort(hilbert_keys(lattice, bits_per_axis), kind="stable")
    shells = [GaussianShell(center=system.shells[k].center.copy(), primitives=list(system.shells[k].primitives),
                            l=int(getattr(system.shells[k], "l", 0)))
              for k in perm]
    return BasisSystem(shells=assign_offsets(shells), atoms=system.atoms), perm
