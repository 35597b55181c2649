"""Algorithmic flop and byte model of one precoder.

The per-solve counts restate the reference's closed forms (flops.py:35-69:
direct 4K^3 + K - 1, CG T(8K^2 + 46K - 6) per right-hand side, Jac-PCG CG +
4K^2 + 2K); the precoder adds the Hermitian Gram 4MK(K+1), W = beta H X
8MK^2 and the coupling B = beta (A - xi I) X 8K^3.  Real flops; one complex
MAC = 8 flops.  Bytes = read H once + write W once.
"""

from __future__ import annotations


def solve_flops(method: str, K: int, T: int) -> int:
    if method == "direct":
        return 4 * K ** 3 + K - 1
    cg = T * (8 * K ** 2 + 46 * K - 6)
    if method == "cg":
        return K * cg
    if method == "jacpcg":
        return K * (cg + 4 * K ** 2 + 2 * K)
    raise ValueError(f"unknown method {method!r}")


def precoder_flops(M: int, K: int, T: int, method: str = "jacpcg") -> int:
    return 4 * M * K * (K + 1) + solve_flops(method, K, T) + 8 * M * K * K + 8 * K ** 3


def precoder_bytes(M: int, K: int, complex_bytes: int) -> int:
    return 2 * M * K * complex_bytes
