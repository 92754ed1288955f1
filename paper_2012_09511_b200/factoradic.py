"""Factoradic <-> decimal conversion at the host boundary (Python integers are the BigCount).

Mirrors include/pbb/factoradic.hpp and src/factoradic.cpp of the reference:
  to_decimal      src/factoradic.cpp:18-28
  from_decimal    src/factoradic.cpp:38-45
  compare         src/factoradic.cpp:51-57
  midpoint        src/factoradic.cpp:59-93 (digit form; the device steal kernel uses the same)
Digits are most-significant first; digit l has radix n-l and weight (n-1-l)!.
"""
from __future__ import annotations

from math import factorial
from typing import List, Optional, Sequence

__all__ = ["validate", "to_decimal", "from_decimal", "compare", "midpoint", "factorial"]


def validate(digits: Sequence[int]) -> None:
    n = len(digits)
    for l, d in enumerate(digits):
        if d < 0 or d > n - 1 - l:
            raise ValueError(f"factoradic digit {d} out of radix at level {l}")


def to_decimal(digits: Sequence[int]) -> int:
    validate(digits)
    n = len(digits)
    acc = 0
    for l, d in enumerate(digits):
        acc = acc * (n - l) + d
    return acc


def from_decimal(x: int, n: int) -> List[int]:
    if x < 0:
        raise ValueError("negative position")
    out = [0] * n
    rest = x
    for l in range(n - 1, -1, -1):
        rest, out[l] = divmod(rest, n - l)
    if rest:
        raise ValueError("from_decimal: value >= n!")
    return out


def compare(a: Sequence[int], b: Sequence[int]) -> int:
    if len(a) != len(b):
        raise ValueError("factoradic length mismatch")
    for x, y in zip(a, b):
        if x != y:
            return -1 if x < y else 1
    return 0


def midpoint(a: Sequence[int], b: Optional[Sequence[int]]) -> List[int]:
    """floor((a+b)/2) on digit vectors; b=None stands for n!. Requires a < b."""
    validate(a)
    n = len(a)
    if b is not None:
        validate(b)
        if len(b) != n:
            raise ValueError("factoradic length mismatch")
        if compare(a, b) >= 0:
            raise ValueError("midpoint requires a < b")
        s = [0] * n
        carry = 0
        for l in range(n - 1, -1, -1):
            carry, s[l] = divmod(a[l] + b[l] + carry, n - l)
    else:
        s = list(a)
        carry = 1
    out = [0] * n
    rem = carry
    for l in range(n):
        rem, out[l] = (rem * (n - l) + s[l]) % 2, (rem * (n - l) + s[l]) // 2
    return out
