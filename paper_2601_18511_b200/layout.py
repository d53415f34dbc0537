"""App. A index maps of the coefficient-encoded block layout (host side).

Same functions and error behaviour as the reference's ``hesim.bitrev``
(pkg/src/hesim/bitrev.py:14-70), written as integer bit manipulation plus
vectorised tables, and the derived maps the MLWE PCMM needs:

* ``sigma(t, k)`` = f(bitReverse(t, log k), log k): the hidden column carried by
  MLWE component t of a coefficient-encoded block.  With the nibble swap
  x = 16(t mod 16) + t div 16 between component order and the paper's MLWE index,
  sigma(t) = g(x) (PAPER.md:660-667 read with width 8, as bitrev.py:36-37 does).
* ``coeff_index(token, col, d, k)`` / ``coeff_table``: where a matrix entry lives in
  the RLWE coefficient vector.
"""

from __future__ import annotations

import numpy as np


def _check(x: int, bits: int, what: str) -> None:
    if not 0 <= x < (1 << bits):
        raise ValueError(f"{x} is not a {what}")


def bit_reverse(x: int, k: int) -> int:
    """Reverse x as a k-bit string (bitrev.py:14-21)."""
    _check(x, k, f"{k}-bit value")
    return int(format(x, f"0{k}b")[::-1], 2) if k else 0


def rotate_bits_down(x: int, k: int) -> int:
    """f(x, k): cyclic right shift by one in k bits (bitrev.py:24-29)."""
    _check(x, k, f"{k}-bit value")
    return (x >> 1) | ((x & 1) << (k - 1))


def byte_mix(x: int) -> int:
    """g: bits a7..a0 -> a3 a4 a5 a6 a7 a0 a1 a2 (bitrev.py:32-45)."""
    _check(x, 8, "byte")
    hi = x >> 3          # a7..a3
    lo = x & 7           # a2..a0
    # output bits 7..3 = a3 a4 a5 a6 a7 (reverse of hi), bits 2..0 = a0 a1 a2 (reverse of lo)
    return (int(format(hi, "05b")[::-1], 2) << 3) | int(format(lo, "03b")[::-1], 2)


def half_reverse(x: int) -> int:
    """h: fix bit 11, reverse the low 11 bits (bitrev.py:48-54)."""
    _check(x, 12, "12-bit value")
    return (x & 2048) | bit_reverse(x & 2047, 11)


def shuffle_matrix(mat, perm=byte_mix) -> np.ndarray:
    """Conjugate a square matrix by a permutation: M'[i][j] = M[p(i)][p(j)] (bitrev.py:57-70)."""
    mat = np.asarray(mat)
    if mat.ndim != 2 or mat.shape[0] != mat.shape[1]:
        raise ValueError("matrix must be square")
    n = mat.shape[0]
    try:
        idx = np.array([perm(i) for i in range(n)], dtype=np.intp)
    except ValueError as exc:  # e.g. byte_mix on a non-byte index
        raise ValueError("permutation domain larger than the matrix") from exc
    if idx.max() >= n or idx.min() < 0:
        raise ValueError("permutation domain larger than the matrix")
    return mat[np.ix_(idx, idx)].copy()


def bit_reverse_table(k: int) -> np.ndarray:
    n = 1 << k
    v = np.arange(n, dtype=np.int64)
    r = np.zeros(n, dtype=np.int64)
    for b in range(k):
        r |= ((v >> b) & 1) << (k - 1 - b)
    return r


def nibble_swap(x: int) -> int:
    """MLWE index x = 16i + j <-> component t = i + 16j."""
    _check(x, 8, "byte")
    return ((x & 15) << 4) | (x >> 4)


def sigma_table(k: int) -> np.ndarray:
    """sigma(t) = f(bitReverse(t, log k), log k) for t < k."""
    lk = k.bit_length() - 1
    if k != 1 << lk or k < 2:
        raise ValueError("k must be a power of two >= 2")
    b = bit_reverse_table(lk)
    return (b >> 1) | ((b & 1) << (lk - 1))


def sigma(t: int, k: int) -> int:
    return int(sigma_table(k)[t])


def coeff_table(d: int, k: int):
    """(token, col-in-block) for each coefficient c = t + k m of one RLWE block;
    token = -1 marks the zero imaginary half (m >= d/2)."""
    half = d // 2
    lh = half.bit_length() - 1
    br = bit_reverse_table(lh)
    sig = sigma_table(k)
    c = np.arange(d * k)
    t, m = c % k, c // k
    token = np.where(m < half, br[np.minimum(m, half - 1)], -1)
    return token, sig[t]


def block_permutation(n: int, k: int) -> np.ndarray:
    """Index map of the k x k block conjugation used by the PCMM plan:
    GEMM row/col x = k r + t reads source index k r + sigma(t)."""
    if n % k:
        raise ValueError(f"dimension {n} is not a multiple of k = {k}")
    sig = sigma_table(k)
    x = np.arange(n)
    return (x // k) * k + sig[x % k]
