"""Slot-indexed coding tables (read side) and the quantizer binding.

``CodingTables`` mirrors the attributes of the reference class
(/root/reference/pkg/src/csrdtans/entropy.py:333-401) over numpy arrays.
The table *construction* (quantize + build_tables, entropy.py:223-436) runs in
the C++ encoder; ``quantize`` below exposes that same C++ quantizer with the
reference signature for parity tests.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ParameterError


class _Escape:
    """Singleton marker for the escape entry (entropy.py:46-58)."""

    _instance = None

    def __new__(cls):
        if cls._instance is None:
            cls._instance = super().__new__(cls)
        return cls._instance

    def __repr__(self):
        return "ESCAPE"


ESCAPE = _Escape()


@dataclass(eq=False)
class CodingTables:
    """Slot arrays of one symbol domain: symbol bits, escape flag, digit, base."""

    sym: np.ndarray      # uint64 [k]; 0 where escape
    escape: np.ndarray   # bool   [k]
    digits: np.ndarray   # uint8  [k]
    bases: np.ndarray    # int32  [k]
    _memo: dict = field(default_factory=dict, repr=False)

    @property
    def k(self) -> int:
        return len(self.sym)

    @property
    def symbols(self) -> tuple:
        if "symbols" not in self._memo:
            self._memo["symbols"] = tuple(
                ESCAPE if e else int(s) for s, e in zip(self.sym.tolist(), self.escape.tolist()))
        return self._memo["symbols"]

    @property
    def escape_base(self) -> int:
        return int(self.bases[self.escape].max()) if self.escape.any() else 0

    def has_symbol(self, symbol) -> bool:
        if symbol is ESCAPE:
            return bool(self.escape.any())
        return bool(np.any((self.sym == np.uint64(symbol)) & ~self.escape))

    def base_of(self, symbol) -> int:
        if symbol is ESCAPE:
            return self.escape_base
        hit = np.nonzero((self.sym == np.uint64(symbol)) & ~self.escape)[0]
        if len(hit) == 0:
            raise KeyError(symbol)
        return int(self.bases[hit[0]])

    def retained_symbols(self) -> tuple:
        return tuple(sorted(set(self.sym[~self.escape].tolist())))

    def pad_symbol(self):
        """entropy.py:392-401 — the retained symbol with the strictly largest
        base, lowest slot on ties; None for escape-only tables."""
        if not (~self.escape).any():
            return None
        b = np.where(self.escape, -1, self.bases)
        return int(self.sym[int(np.argmax(b))])

    def __eq__(self, other) -> bool:
        if not isinstance(other, CodingTables):
            return NotImplemented
        return (np.array_equal(self.sym, other.sym) and np.array_equal(self.escape, other.escape)
                and np.array_equal(self.digits, other.digits)
                and np.array_equal(self.bases, other.bases))


def quantize_counts(symbols, counts, k: int, m: int, raw_width_bits: int, never_retain=()):
    """The C++ quantizer (entropy.py:223-321) on integer symbols.

    ``symbols`` must be distinct non-negative integers < 2^64 in the order
    the reference's ``SymbolDistribution`` holds them (the container passes
    them ascending).  Returns ``(multiplicities, escape_multiplicity,
    escape_slots)``.
    """
    sy = np.ascontiguousarray(np.asarray(symbols, dtype=np.uint64))
    ct = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
    if len(sy) != len(ct):
        raise ParameterError("symbols and counts must have equal length")
    nv = np.ascontiguousarray(np.asarray(sorted(never_retain), dtype=np.uint64))
    mult = np.zeros(max(len(sy), 1), dtype=np.int32)
    em = ctypes.c_int32()
    es = ctypes.c_int32()
    L = _native.lib()
    _native.check(L.dtans_quantize(
        len(sy), sy.ctypes.data if len(sy) else None, ct.ctypes.data if len(ct) else None,
        k, m, raw_width_bits, len(nv), nv.ctypes.data if len(nv) else None,
        mult.ctypes.data, ctypes.addressof(em), ctypes.addressof(es)))
    return mult[: len(sy)], em.value, es.value
