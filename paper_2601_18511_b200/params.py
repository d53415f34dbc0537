"""Scheme parameters for the MLWE PCMM / Rhombus PCMv path.

Mirrors the role of ``hesim.SimParams`` (slotsim.py:86-129): a frozen, JSON-
serialisable parameter record with the same reject-unknown-keys policy as the
reference CLI's ``--config`` loader (cli.py:37-46).

Ring: R_N = Z[X]/(X^N + 1), N = d * k; MLWE degree d, rank k (PAPER.md:54-55:
"MLWE ciphertext formats of degree 256 and rank 256", N = 2^16).  Level l keeps
limbs q_0..q_l; the PCMM input sits at level 1 (two limbs) and the
op consumes exactly one level by rescaling away q_1.

Prime choice (the paper does not pin it; SURVEY.md §7 "Choosing Delta_w"):
  q_0  the base prime, < 2^30: a centred residue takes 4 signed 8-bit digits, and the NTT can run
       Harvey-lazy butterflies (values in [0, 4q) fit a u32);
  q_1  the PCMM *scale prime*, Delta_w = q_1 exactly, so the output scale equals the
       input scale Delta after the rescale.  The default q_1 ~ 2^20 gives ~15-16
       bits of weight precision for Llama-scale weights (|W| < 2^-6), above the
       paper's 12-bit target, and needs 3 ciphertext digits.
Both are NTT-friendly: q = 1 mod 2N.

Chain: moduli[2:] are the primes of the levels above the PCMM's
level 1 -- "lower the total level to 4; SlotToCoeffs to level 1": the factorized SlotToCoeffs consumes
q_4, q_3, q_2 (three slot linear maps, one level each) and hands the PCMM its (q_0, q_1) input.  The
kernels of the PCMM / PCMv / ring packing use q_0, q_1 and P only; he_chain.cu runs the levels above.
"""

from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass, field


def is_prime(n: int) -> bool:
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def ntt_primes(two_n: int, below: int, count: int) -> list[int]:
    """The `count` largest primes p < below with p = 1 (mod two_n)."""
    out = []
    c = (below - 1) // two_n
    while c > 0 and len(out) < count:
        p = c * two_n + 1
        if p < below and is_prime(p):
            out.append(p)
        c -= 1
    if len(out) < count:
        raise ValueError(f"not enough NTT primes below {below} for 2N={two_n}")
    return out


def signed_digits(bound: int) -> int:
    """Number of balanced base-256 digits (each in [-128, 127]) needed for |v| <= bound."""
    n = 1
    while 127 * ((256 ** n - 1) // 255) < bound:
        n += 1
    return n


_KNOWN = ("name", "mlwe_degree", "mlwe_rank", "moduli", "log_delta", "rhombus_degree", "special_prime", "seed")


@dataclass(frozen=True)
class HeParams:
    """CKKS/MLWE parameters.  ``moduli[0]`` is the base prime, ``moduli[1]`` the
    PCMM scale prime consumed by the rescale."""

    mlwe_degree: int = 256
    mlwe_rank: int = 256
    moduli: tuple[int, ...] = (1073479681, 1179649)
    log_delta: int = 26
    rhombus_degree: int = 4096
    special_prime: int = 1071513601   # P of the hybrid key switches (Rhombus decompose / packing)
    seed: int | None = None
    name: str = "llama"

    def __post_init__(self):
        d, k = self.mlwe_degree, self.mlwe_rank
        for v, what in ((d, "mlwe_degree"), (k, "mlwe_rank")):
            if v < 2 or v & (v - 1):
                raise ValueError(f"{what} must be a power of two >= 2, got {v}")
        object.__setattr__(self, "moduli", tuple(int(q) for q in self.moduli))
        if not 2 <= len(self.moduli) <= 7:
            raise ValueError("moduli: (q0, q1) for the PCMM's level 1, plus up to 5 chain primes above it")
        for q in self.moduli:
            if not is_prime(q):
                raise ValueError(f"modulus {q} is not prime")
            if (q - 1) % (2 * self.N):
                raise ValueError(f"modulus {q} is not 1 mod 2N = {2 * self.N}")
            if q >= 1 << 30:
                raise ValueError(f"modulus {q} must be below 2^30 (lazy NTT butterflies)")
        if len(set(self.moduli)) != len(self.moduli):
            raise ValueError("moduli must be distinct")
        P = int(self.special_prime)
        object.__setattr__(self, "special_prime", P)
        if not is_prime(P) or (P - 1) % (2 * self.N) or P >= 1 << 30 or P in self.moduli:
            raise ValueError("special_prime must be an NTT-friendly prime below 2^30, distinct from the moduli")
        if not 1 <= self.log_delta <= 40:
            raise ValueError("log_delta must be in [1, 40]")
        if self.rhombus_degree & (self.rhombus_degree - 1) or self.N % self.rhombus_degree:
            raise ValueError("rhombus_degree must be a power of two dividing N")

    # -- derived ----------------------------------------------------------
    @property
    def N(self) -> int:
        return self.mlwe_degree * self.mlwe_rank

    @property
    def tokens(self) -> int:
        """Real rows per RLWE ciphertext: the Ecd_coeff real half."""
        return self.mlwe_degree // 2

    @property
    def width(self) -> int:
        """Words per MLWE ciphertext: b (d) + a (d * k).  65 792 at d = k = 256."""
        return self.mlwe_degree * (1 + self.mlwe_rank)

    @property
    def top_level(self) -> int:
        return len(self.moduli) - 1

    @property
    def delta(self) -> float:
        return float(2 ** self.log_delta)

    @property
    def ks_moduli(self) -> tuple[int, int, int]:
        """(q0, q1, P): the moduli of the hybrid key-switching keys."""
        return (self.moduli[0], self.moduli[1], self.special_prime)

    @property
    def rho(self) -> int:
        """Degree-N ciphertext splits into rho = N / rhombus_degree RLWE pieces."""
        return self.N // self.rhombus_degree

    @property
    def delta_w(self) -> int:
        """Weight scale: the scale prime itself, so Delta * Delta_w / q1 == Delta."""
        return self.moduli[1]

    def ct_digits(self, limb: int) -> int:
        """Balanced 8-bit digits of a centred residue mod moduli[limb]."""
        return signed_digits(self.moduli[limb] // 2)

    def to_dict(self) -> dict:
        out = asdict(self)
        out["moduli"] = list(self.moduli)
        return out

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True)

    @classmethod
    def from_dict(cls, data: dict) -> "HeParams":
        unknown = set(data) - set(_KNOWN)
        if unknown:
            raise ValueError(f"unknown parameter keys: {sorted(unknown)}")
        kw = dict(data)
        if "moduli" in kw:
            kw["moduli"] = tuple(kw["moduli"])
        return cls(**kw)

    @classmethod
    def from_json(cls, path) -> "HeParams":
        with open(path) as fh:
            return cls.from_dict(json.load(fh))

    # -- presets ----------------------------------------------------------
    @classmethod
    def llama(cls, **kw) -> "HeParams":
        """N = 2^16, MLWE (256, 256); q0 < 2^30, q1 ~ 2^20 (the bench / metric preset)."""
        return cls(**kw)

    @classmethod
    def wide(cls, **kw) -> "HeParams":
        """N = 2^16 with two ~30-bit primes (4 + 4 ciphertext digits, 4 weight digits)."""
        pr = ntt_primes(2 * 65536, 1 << 30, 3)
        kw.setdefault("moduli", tuple(pr[:2]))
        kw.setdefault("special_prime", pr[2])
        kw.setdefault("name", "wide")
        return cls(**kw)

    @classmethod
    def llama_chain(cls, levels: int = 3, **kw) -> "HeParams":
        """The llama preset plus `levels` ~30-bit primes above q1 (default 3: input at level 4, the factorized
        SlotToCoeffs consumes three levels and outputs the PCMM's level-1 input)."""
        base = cls.llama()
        extra = [p for p in ntt_primes(2 * base.N, 1 << 30, levels + 4) if p not in (*base.moduli, base.special_prime)]
        kw.setdefault("moduli", tuple(base.moduli) + tuple(extra[:levels]))
        kw.setdefault("name", "llama_chain")
        return cls(**kw)

    @classmethod
    def toy_chain(cls, levels: int = 3, **kw) -> "HeParams":
        """The toy ring (N = 512) with `levels` chain primes above q1."""
        base = cls.toy()
        extra = [p for p in ntt_primes(2 * base.N, 1 << 30, levels + 4) if p not in (*base.moduli, base.special_prime)]
        kw.setdefault("moduli", tuple(base.moduli) + tuple(extra[:levels]))
        for k in ("mlwe_degree", "mlwe_rank", "special_prime", "rhombus_degree"):
            kw.setdefault(k, getattr(base, k))
        kw.setdefault("name", "toy_chain")
        return cls(**kw)

    @classmethod
    def toy(cls, **kw) -> "HeParams":
        """N = 512, MLWE degree 32 (16 tokens), rank 16: BASELINE config 1's toy ring
        (SURVEY.md §8c), 16-column ciphertext batch like hesim's d=16 PCMM."""
        kw.setdefault("mlwe_degree", 32)
        kw.setdefault("mlwe_rank", 16)
        big = ntt_primes(1024, 1 << 30, 2)
        kw.setdefault("moduli", (big[0], ntt_primes(1024, 1 << 21, 1)[0]))
        kw.setdefault("special_prime", big[1])
        kw.setdefault("rhombus_degree", 128)
        kw.setdefault("name", "toy")
        return cls(**kw)
