"""SPOW_p feature map metadata (reference expansions.py).  The CUDA kernels
generate phi on chip; this module only describes it (dimension, NDMI table)
so callers and tests can reason about state layouts."""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .errors import InvalidSpec


class ExpansionKind(str, Enum):
    TPOW = "tpow"
    SPOW = "spow"
    TSPOW = "tspow"


@dataclass(frozen=True)
class ExpansionSpec:
    """(kind, p, d) as in reference expansions.py:50-89.  Only SPOW runs on the
    CUDA path (the north star names SPOW_p); TPOW/TSPOW raise InvalidSpec."""

    kind: ExpansionKind
    p: int
    d: int
    d_tile: int | None = None

    def __post_init__(self):
        object.__setattr__(self, "kind", ExpansionKind(self.kind))
        if self.p < 1:
            raise InvalidSpec(f"power degree must be >= 1, got {self.p}")
        if self.d < 1:
            raise InvalidSpec(f"input dimension must be >= 1, got {self.d}")

    @classmethod
    def spow(cls, p: int, d: int) -> "ExpansionSpec":
        return cls(ExpansionKind.SPOW, p, d)

    def require_spow(self) -> "ExpansionSpec":
        if self.kind is not ExpansionKind.SPOW:
            raise InvalidSpec(f"{self.kind.value} expansions are not on the CUDA path; use spow")
        return self


def expansion_dim(spec: ExpansionSpec) -> int:
    """D = C(d+p-1, p) for SPOW (expansions.py:87-99)."""
    spec.require_spow()
    return math.comb(spec.d + spec.p - 1, spec.p)


def monomial_table(spec: ExpansionSpec):
    """(idx [D, p] int32, weights [D] float64) in the reference row order
    (expansions.py:171-198), produced by the C library."""
    spec.require_spow()
    D = expansion_dim(spec)
    idx = np.zeros((D, spec.p), dtype=np.int32)
    w = np.zeros(D, dtype=np.float64)
    _lib.check(_lib.load().pa_feature_table(spec.p, spec.d, idx.ctypes.data_as(ctypes.c_void_p),
                                            w.ctypes.data_as(ctypes.c_void_p)), "feature table")
    return idx, w
