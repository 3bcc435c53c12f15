"""Deterministic synthetic instances with the structure of the QAPLIB families
named in BASELINE.json (no QAPLIB files ship with the reference except toy2,
pkg/README.md:115-119).  Generators are seeded SplitMix64 streams evaluated with
NumPy, so the CPU oracle and the GPU path see identical bytes on any machine.

  tai_a   symmetric uniform 0..99 flow and distance (Taillard "a")
  tai_b   clustered Euclidean distances, heavy-tailed asymmetric flows with many
          zeros (Taillard "b"; deltas exceed int32 -> exercises the int64 state)
  tai_c   grey-pattern: 0/1 flow block, inverse-square repulsion on a torus (tai256c)
  nug     Manhattan grid distances, sparse small symmetric flows (Nugent)
  sko     Manhattan grid distances, flows 0..10 with ~30 % zeros (Skorin-Kapov)
  rand    the reference's own `random_instance` (instance.py:194-209): asymmetric
          uniform 0..99 with zero diagonals
"""

from __future__ import annotations

import numpy as np

from .instance import Instance, random_instance
from .rng import SplitMix64, derive_seed, raw_stream


def _uniform(seed: int, count: int, span: int) -> np.ndarray:
    return (raw_stream(seed, count) % np.uint64(span)).astype(np.int64)


def _unit_floats(seed: int, count: int) -> np.ndarray:
    return (raw_stream(seed, count) >> np.uint64(11)).astype(np.float64) / float(1 << 53)


def _symmetric_from_upper(vals: np.ndarray, n: int) -> np.ndarray:
    m = np.zeros((n, n), dtype=np.int64)
    iu = np.triu_indices(n, k=1)
    m[iu] = vals
    return m + m.T


def _grid(n: int) -> tuple[int, int]:
    rows = int(np.floor(np.sqrt(n)))
    while n % rows:
        rows -= 1
    return rows, n // rows


def _manhattan(n: int) -> np.ndarray:
    rows, cols = _grid(n)
    r, c = np.divmod(np.arange(n), cols)
    return (np.abs(r[:, None] - r[None, :]) + np.abs(c[:, None] - c[None, :])).astype(np.int64)


def tai_a(n: int, seed: int = 1234) -> Instance:
    m = n * (n - 1) // 2
    flow = _symmetric_from_upper(_uniform(derive_seed(seed, 1), m, 100), n)
    dist = _symmetric_from_upper(_uniform(derive_seed(seed, 2), m, 100), n)
    return Instance(f"tai{n}a-shaped", n, flow, dist)


def tai_b(n: int, seed: int = 1234) -> Instance:
    clusters = max(2, n // 12)
    cu = _unit_floats(derive_seed(seed, 3), 2 * clusters).reshape(clusters, 2) * 1000.0
    which = _uniform(derive_seed(seed, 4), n, clusters)
    jitter = (_unit_floats(derive_seed(seed, 5), 2 * n).reshape(n, 2) - 0.5) * 120.0
    pts = cu[which] + jitter
    dist = np.rint(np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1))).astype(np.int64)
    np.fill_diagonal(dist, 0)
    u = _unit_floats(derive_seed(seed, 6), n * n).reshape(n, n)
    gate = _unit_floats(derive_seed(seed, 7), n * n).reshape(n, n)
    flow = np.where(gate < 0.45, 0, np.floor(10.0 ** (5.0 * u))).astype(np.int64)
    np.fill_diagonal(flow, 0)
    return Instance(f"tai{n}b-shaped", n, flow, dist)


def tai_c(n: int = 256, density: int | None = None) -> Instance:
    side = int(round(np.sqrt(n)))
    if side * side != n:
        raise ValueError("tai_c needs a square n")
    m = density if density is not None else max(2, (92 * n) // 256)
    flow = np.zeros((n, n), dtype=np.int64)
    flow[:m, :m] = 1
    np.fill_diagonal(flow, 0)
    r, c = np.divmod(np.arange(n), side)
    dr = np.abs(r[:, None] - r[None, :]); dr = np.minimum(dr, side - dr)
    dc = np.abs(c[:, None] - c[None, :]); dc = np.minimum(dc, side - dc)
    sq = dr * dr + dc * dc
    dist = np.zeros((n, n), dtype=np.int64)
    nz = sq > 0
    dist[nz] = 100000 // sq[nz]
    return Instance(f"tai{n}c-shaped", n, flow, dist)


def nug(n: int = 12, seed: int = 1234) -> Instance:
    m = n * (n - 1) // 2
    vals = _uniform(derive_seed(seed, 8), m, 11)
    keep = _uniform(derive_seed(seed, 9), m, 100) < 55
    flow = _symmetric_from_upper(np.where(keep, vals, 0), n)
    return Instance(f"nug{n}-shaped", n, flow, _manhattan(n))


def sko(n: int = 100, seed: int = 1234) -> Instance:
    m = n * (n - 1) // 2
    vals = _uniform(derive_seed(seed, 10), m, 11)
    keep = _uniform(derive_seed(seed, 11), m, 100) < 70
    flow = _symmetric_from_upper(np.where(keep, vals, 0), n)
    return Instance(f"sko{n}-shaped", n, flow, _manhattan(n))


def rand(n: int, seed: int = 1234) -> Instance:
    return random_instance(n, SplitMix64(derive_seed(seed, 0)), name=f"rand{n}")


def by_name(name: str, seed: int = 1234) -> Instance:
    """'tai100a', 'tai150b', 'tai256c', 'nug12', 'sko100', 'rand30' -> shaped instance."""
    import re

    m = re.fullmatch(r"(tai|nug|sko|rand)(\d+)([abc]?)", name)
    if not m:
        raise ValueError(f"unknown shape {name!r}")
    fam, n, suffix = m.group(1), int(m.group(2)), m.group(3)
    if fam == "tai":
        return {"a": tai_a, "b": tai_b}[suffix](n, seed) if suffix in ("a", "b") else tai_c(n)
    if fam == "nug":
        return nug(n, seed)
    if fam == "sko":
        return sko(n, seed)
    return rand(n, seed)
