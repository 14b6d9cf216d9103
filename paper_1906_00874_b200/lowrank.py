"""Host-side low-rank types shared with the reference API.

``LowRank`` (value ``a @ b.T``), ``TruncationControl`` and
``SingularBlockError`` keep the reference's names and contracts
(``lowrank.py:18-80``).  There is deliberately no CPU arithmetic here: every
truncation, triangular solve and product of the factorization runs in the
sm_100a kernels behind ``include/hlu_b200.h``.  The single-block helpers
``add_truncated`` / ``compress_dense`` / ``recompress`` are provided as
one-op device launches (see ``device_ops``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class SingularBlockError(ArithmeticError):
    """An unpivoted LU met a pivot ``|p| <= 1e-12 * max|A|`` (``lowrank.py:18``)."""

    def __init__(self, message, block_path=""):
        super().__init__(message)
        self.block_path = block_path


@dataclass(frozen=True)
class TruncationControl:
    """Keep singular values ``sigma_i > eps * sigma_1``; cap the rank at ``kmax``."""

    eps: float = 1e-8
    kmax: int | None = None

    def __post_init__(self):
        if self.eps < 0:
            raise ValueError("eps must be >= 0")
        if self.kmax is not None and self.kmax < 0:
            raise ValueError("kmax must be >= 0 if set")


class LowRank:
    """Factor pair ``a (m, k)``, ``b (n, k)`` representing ``a @ b.T``."""

    __slots__ = ("a", "b")

    def __init__(self, a, b):
        a = np.ascontiguousarray(a, dtype=float)
        b = np.ascontiguousarray(b, dtype=float)
        if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[1]:
            raise ValueError("factors must be 2-d with matching column counts")
        self.a = a
        self.b = b

    @classmethod
    def zeros(cls, m, n):
        return cls(np.zeros((m, 0)), np.zeros((n, 0)))

    k = property(lambda self: self.a.shape[1])
    shape = property(lambda self: (self.a.shape[0], self.b.shape[0]))

    def value(self):
        return self.a @ self.b.T

    def neg(self):
        return LowRank(-self.a, self.b)

    def copy(self):
        return LowRank(self.a.copy(), self.b.copy())

    def __repr__(self):
        return f"LowRank({self.shape[0]}x{self.shape[1]}, k={self.k})"
