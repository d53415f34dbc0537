"""CKKS slot encoding (canonical embedding) for the slot-domain PCMM.

hesim's PCMM (matmul.py:152-176) works on *slots*: a d x d matrix packed row-major into d^2 slots,
tiled across the slot vector (packing.py:1-17), rotated by np.roll (slotsim.py:294-301).  On a
real CKKS ciphertext of degree N the slot vector has n = N/2 complex entries z_j, slot j being the
evaluation of the message polynomial at zeta^(5^j) (zeta = exp(i pi / N)), so the automorphism
X -> X^(5^r) rotates the slots left by r -- hesim's rotate(ct, r).  Real-valued hesim slots map to
the real parts.

    encode(z)  m = round(scale * sigma^-1(z)):  m_i = (1/N) sum_{e odd} Z[e] zeta^(-e i), with
               Z[5^j] = z_j, Z[-5^j] = conj(z_j)  (one length-2N FFT)
    decode(m)  z_j = m(zeta^(5^j)) / scale        (one length-2N FFT)

Host-side float64 (plaintext preparation at plan time and test-side decoding), like hesim's own
encode; the ciphertext arithmetic runs on the device (he_slot_pcmm_*).
"""

from __future__ import annotations

import numpy as np


def slot_exponents(N: int) -> np.ndarray:
    """e_j = 5^j mod 2N for the n = N/2 slots."""
    n = N // 2
    e = np.empty(n, dtype=np.int64)
    v = 1
    for j in range(n):
        e[j] = v
        v = v * 5 % (2 * N)
    return e


def rotation_galois(N: int, r: int) -> int:
    """Galois element of a left slot rotation by r: 5^r mod 2N."""
    return pow(5, r % (N // 2), 2 * N)


def encode(values, N: int, scale: float) -> np.ndarray:
    """Slot values (real or complex, length dividing N/2: tiled like hesim's encode) -> int64 coefficients."""
    n = N // 2
    z = np.asarray(values)
    if z.ndim != 1 or n % z.size:
        raise ValueError(f"length {z.size} does not divide the {n} slots")
    z = np.tile(z.astype(np.complex128), n // z.size)
    e = slot_exponents(N)
    Z = np.zeros(2 * N, dtype=np.complex128)
    Z[e] = z
    Z[(2 * N - e) % (2 * N)] = np.conj(z)
    m = np.fft.fft(Z)[:N].real / N
    return np.rint(m * scale).astype(np.int64)


def decode(coeffs, N: int, scale: float, n_vals: int | None = None, real: bool = True) -> np.ndarray:
    """Centred integer coefficients (length N) -> slot values (first n_vals; real parts by default)."""
    m = np.asarray(coeffs, dtype=np.float64)
    if m.size != N:
        raise ValueError(f"need {N} coefficients, got {m.size}")
    pad = np.zeros(2 * N, dtype=np.complex128)
    pad[:N] = m
    F = np.fft.ifft(pad) * (2 * N)      # F[e] = sum_i m_i zeta^(e i)
    z = F[slot_exponents(N)] / scale
    z = z[:n_vals] if n_vals is not None else z
    return z.real.copy() if real else z
