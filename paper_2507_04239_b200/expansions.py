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


_KIND_CODE = {ExpansionKind.SPOW: 0, ExpansionKind.TPOW: 1, ExpansionKind.TSPOW: 2}


@dataclass(frozen=True)
class ExpansionSpec:
    """(kind, p, d[, d_tile]) as in reference expansions.py:50-89.

    All three kinds satisfy <phi(x), phi(y)> = (x . y)^p (reference
    expansions.py:3-5), so attention outputs and gradients do not depend on the
    kind and power_full serves every kind; only the state representation of
    update_state / query_state does, and those operators run the kind's own
    monomial table on the device."""

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
        if self.kind is ExpansionKind.TSPOW:
            if self.d_tile is None:
                raise InvalidSpec("tspow requires d_tile")
            if not 1 <= self.d_tile <= self.d or self.d % self.d_tile:
                raise InvalidSpec(f"d_tile={self.d_tile} must divide d={self.d} and lie in [1, d]")
        elif self.d_tile is not None:
            raise InvalidSpec(f"{self.kind.value} does not take d_tile")

    @classmethod
    def spow(cls, p: int, d: int) -> "ExpansionSpec":
        return cls(ExpansionKind.SPOW, p, d)

    @classmethod
    def tpow(cls, p: int, d: int) -> "ExpansionSpec":
        return cls(ExpansionKind.TPOW, p, d)

    @classmethod
    def tspow(cls, p: int, d: int, d_tile: int) -> "ExpansionSpec":
        return cls(ExpansionKind.TSPOW, p, d, d_tile)

    @property
    def code(self) -> int:
        return _KIND_CODE[self.kind]


def expansion_dim(spec: ExpansionSpec) -> int:
    """D: C(d+p-1, p) (spow), d^p (tpow), C(d/d_tile+p-1, p) d_tile^p (tspow);
    reference expansions.py:87-99."""
    if spec.kind is ExpansionKind.SPOW:
        return math.comb(spec.d + spec.p - 1, spec.p)
    if spec.kind is ExpansionKind.TPOW:
        return spec.d ** spec.p
    return math.comb(spec.d // spec.d_tile + spec.p - 1, spec.p) * spec.d_tile ** spec.p


_TABLES: dict = {}


def monomial_table(spec: ExpansionSpec):
    """(idx [D, p] int32, weights [D] float64) in the reference row order
    (expansions.py:171-198), produced by the C library (cached per spec)."""
    if spec in _TABLES:
        return _TABLES[spec]
    if spec.p > 4:
        raise InvalidSpec(f"the CUDA kernels take p <= 4, got {spec.p}")
    D = expansion_dim(spec)
    idx = np.zeros((D, spec.p), dtype=np.int32)
    w = np.zeros(D, dtype=np.float64)
    _lib.check(_lib.load().pa_expansion_table(spec.code, spec.p, spec.d, spec.d_tile or 0,
                                              idx.ctypes.data_as(ctypes.c_void_p),
                                              w.ctypes.data_as(ctypes.c_void_p)), "monomial table")
    idx.setflags(write=False)
    w.setflags(write=False)
    _TABLES[spec] = (idx, w)
    return idx, w
