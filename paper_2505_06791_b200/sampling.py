"""Halton sampling (mirrors ``maniplan/sampling.py``).

Samples are generated on the device in FP64 with unfused IEEE operations, so
they are bit-identical to the reference stream (``cp_halton`` in
csrc/device/cprrtc_device.cuh; the planner kernel draws from the same
function).  ``first_primes``, ``radical_inverse`` and ``trial_seed_offset``
are tiny host helpers kept for API parity.
"""

from __future__ import annotations

import numpy as np

__all__ = ["first_primes", "radical_inverse", "HaltonState", "trial_seed_offset",
           "TRIAL_SEED_STRIDE"]

TRIAL_SEED_STRIDE = 10_000


def first_primes(n: int) -> list:
    out, c = [], 2
    while len(out) < n:
        if all(c % p for p in out):
            out.append(c)
        c += 1
    return out


def radical_inverse(index: int, base: int) -> float:
    f, scale, i = 0.0, 1.0 / base, index
    while i > 0:
        f += (i % base) * scale
        scale /= base
        i //= base
    return f


def trial_seed_offset(base: int, trial_index: int) -> int:
    return base + trial_index * TRIAL_SEED_STRIDE


class HaltonState:
    """Halton stream; index starts at 1, shifted by ``seed_offset``."""

    def __init__(self, dim: int, seed_offset: int = 0):
        if dim < 1:
            raise ValueError("dim must be >= 1")
        if seed_offset < 0:
            raise ValueError("seed_offset must be >= 0")
        self.bases = first_primes(dim)
        self.index = 1
        self.seed_offset = seed_offset

    @property
    def dim(self) -> int:
        return len(self.bases)

    def next_unit(self) -> np.ndarray:
        u = self.next_samples(np.tile([0.0, 1.0], (self.dim, 1)), 1)[0]
        return u

    def next_sample(self, limits) -> np.ndarray:
        return self.next_samples(limits, 1)[0]

    def next_samples(self, limits, count: int) -> np.ndarray:
        """``count`` consecutive samples mapped into [lo, hi] (device, FP64)."""
        from . import kernels
        from .planner import _stub_robot
        limits = np.asarray(limits, dtype=float)
        if limits.shape != (self.dim, 2):
            raise ValueError(f"limits must have shape ({self.dim}, 2)")
        out = kernels.halton_batch(_stub_robot(self.dim), count, self.index, self.seed_offset,
                                   limits=limits)
        self.index += count
        return out
