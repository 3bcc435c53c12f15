"""SplitMix64 streams for start permutations and tenure draws.

The search kernels are deterministic; all randomness is in the inputs derived
here (reference: /root/reference/pkg/src/qapsolve/rng.py).  The same recurrence
runs on the device for batched multi-start (csrc/search_kernel.cuh: mix64,
randbelow_seq), so host-drawn and device-drawn starts are bit-identical.

    state_{k+1} = state_k + GAMMA  (mod 2^64)          rng.py:35-37
    out_k       = mix64(state_k)                       rng.py:15-20
    start seed  = mix64(master + GAMMA*(index+1))      rng.py:62-70
"""

from __future__ import annotations

import numpy as np

MASK64 = 0xFFFFFFFFFFFFFFFF
GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB


def mix64(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * _M1) & MASK64
    z = ((z ^ (z >> 27)) * _M2) & MASK64
    return z ^ (z >> 31)


def derive_seed(master_seed: int, start_index: int) -> int:
    """Generator state owned by start `start_index` under `master_seed`."""
    if start_index < 0:
        raise ValueError(f"start_index must be non-negative, got {start_index}")
    return mix64(master_seed + GAMMA * (start_index + 1))


class SplitMix64:
    """Additive-counter generator; `state` is the last counter value used."""

    __slots__ = ("_state",)

    def __init__(self, seed: int):
        self._state = seed & MASK64

    @property
    def state(self) -> int:
        return self._state

    def next64(self) -> int:
        self._state = (self._state + GAMMA) & MASK64
        return mix64(self._state)

    def randbelow(self, bound: int) -> int:
        """Uniform draw from range(bound); rejects the biased tail of the 64-bit range."""
        if bound <= 0:
            raise ValueError(f"bound must be positive, got {bound}")
        tail = (1 << 64) % bound
        while True:
            r = self.next64()
            if r < (1 << 64) - tail:
                return r % bound

    def randint(self, low: int, high: int) -> int:
        if high < low:
            raise ValueError(f"empty interval [{low}, {high}]")
        return low + self.randbelow(high - low + 1)

    def shuffle(self, seq) -> None:
        """Fisher-Yates from the top index down (rng.py:55-59)."""
        i = len(seq) - 1
        while i > 0:
            j = self.randbelow(i + 1)
            seq[i], seq[j] = seq[j], seq[i]
            i -= 1


def raw_stream(seed: int, count: int) -> np.ndarray:
    """First `count` outputs of SplitMix64(seed) as uint64, vectorised."""
    with np.errstate(over="ignore"):
        k = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed & MASK64) + np.uint64(GAMMA) * k
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
        return z ^ (z >> np.uint64(31))
