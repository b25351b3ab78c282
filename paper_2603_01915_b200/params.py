"""dtANS stream geometry (mirror of ``DtansParams``).

Reference: /root/reference/pkg/src/csrdtans/codec.py:27-108.  The container
and the sm_100a kernel are specialised to the production geometry
(W=2^32, K=4096, M=256, l=8, o=3, f=2), exactly the set the reference
container accepts (/root/reference/pkg/src/csrdtans/container.py:95-109).
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ParameterError


def _is_pow2(x: int) -> bool:
    return x >= 1 and (x & (x - 1)) == 0


@dataclass(frozen=True)
class DtansParams:
    w: int
    k: int
    m: int
    l: int
    o: int
    f: int

    @classmethod
    def production(cls) -> "DtansParams":
        return cls(w=2**32, k=4096, m=256, l=8, o=3, f=2)

    @classmethod
    def toy(cls) -> "DtansParams":
        return cls(w=4, k=8, m=4, l=2, o=3, f=2)

    @property
    def w_log2(self) -> int:
        return self.w.bit_length() - 1

    @property
    def k_log2(self) -> int:
        return self.k.bit_length() - 1

    @property
    def m_log2(self) -> int:
        return self.m.bit_length() - 1

    def check_groups(self) -> list:
        """codec.py:59-72 — l positions split into f groups, earlier larger."""
        sizes = [self.l // self.f] * self.f
        for i in range(self.l % self.f):
            sizes[i] += 1
        groups, pos = [], 0
        for size in sizes:
            groups.append(list(range(pos, pos + size)))
            pos += size
        return groups

    def validate(self) -> None:
        problems = validate_params(self)
        if problems:
            raise ParameterError("; ".join(problems))


def validate_params(p: DtansParams) -> list:
    """codec.py:80-108 — every parameter constraint, as violation strings."""
    problems = []
    for name in ("w", "k", "m"):
        v = getattr(p, name)
        if not _is_pow2(v) or v < 2:
            problems.append(f"{name} = {v} is not a power of two >= 2")
    if p.l < 1 or p.o < 1 or p.f < 0:
        problems.append(f"need l >= 1, o >= 1, f >= 0 (got l={p.l}, o={p.o}, f={p.f})")
        return problems
    if problems:
        return problems
    if p.m > p.k:
        problems.append(f"multiplicity cap m = {p.m} exceeds table size k = {p.k}")
    if p.k**p.l < p.w**p.o:
        problems.append(f"k^l = {p.k**p.l} < w^o = {p.w**p.o}: words are not representable as slots")
    elif p.k**p.l >= p.w ** (p.o + 1):
        problems.append(f"o = {p.o} wastes words: k^l = {p.k**p.l} >= w^(o+1) = {p.w**(p.o+1)}")
    if p.m**p.l > p.w**p.f:
        problems.append(f"m^l = {p.m**p.l} > w^f = {p.w**p.f}: checks cannot drain the state")
    if p.f > p.o:
        problems.append(f"f = {p.f} exceeds words per segment o = {p.o}")
    return problems


PRODUCTION = DtansParams.production()


def require_container_params(p: DtansParams, precision: int) -> None:
    """container.py:95-109 plus this build's specialisation: the kernel and
    the C++ encoder implement exactly the production geometry."""
    p.validate()
    if p.k**p.l != p.w**p.o:
        raise ParameterError("container params must satisfy k^l == w^o")
    if p.w != 2**32:
        raise ParameterError("container streams are 4-byte words; w must be 2^32")
    if p.m > 256:
        raise ParameterError("slot records store base - 1 in one byte; m <= 256")
    if p.l % 2 != 0:
        raise ParameterError("l must be even: segments interleave deltas and values")
    group = -(-p.l // p.f)
    if group * p.m_log2 > p.w_log2:
        raise ParameterError("check groups too long for 64-bit state arithmetic")
    if precision not in (4, 8):
        raise ParameterError("precision must be 4 or 8 bytes")
    if (p.k, p.l, p.o, p.f) != (4096, 8, 3, 2):
        raise ParameterError(
            "this build implements the production segment geometry "
            "(k=4096, l=8, o=3, f=2); got "
            f"k={p.k}, l={p.l}, o={p.o}, f={p.f}")
