"""Context, ledger and ciphertext containers -- the host mirror of hesim's L0 types.

``HeContext`` plays ``hesim.SlotContext``'s role (slotsim.py:163-205): it owns the
parameters, the cost ledger and (lazily) the device-side context of the C ABI
(NTT tables, constants).  Contexts are not thread-safe; parallel callers
``fork()`` a child with a private ledger and ``merge()`` it back in task order,
exactly as in the reference (slotsim.py:192-205).

Ciphertexts live in device memory as torch int32 tensors holding u32 residues
(torch is the allocator/stream plumbing; every computation goes through the C ABI).
"""

from __future__ import annotations

import ctypes
import json
import os
import secrets
from dataclasses import dataclass, field

import numpy as np

from . import native
from .errors import NeedsBootstrapError
from .params import HeParams

LEDGER_COUNTERS = ("ct_rotations", "cc_mults", "pc_mults", "pt_rotations", "pt_mults", "rescales", "bootstraps")


@dataclass
class CostLedger:
    """Operation counters with hesim.CostLedger's field names and methods
    (slotsim.py:31-83): the performance contract of a kernel."""

    ct_rotations: int = 0
    cc_mults: int = 0
    pc_mults: int = 0
    pt_rotations: int = 0
    pt_mults: int = 0
    rescales: int = 0
    bootstraps: int = 0
    min_level_reached: int | None = None

    def observe_level(self, level: int) -> None:
        if self.min_level_reached is None or level < self.min_level_reached:
            self.min_level_reached = level

    def snapshot(self) -> dict:
        return {n: getattr(self, n) for n in LEDGER_COUNTERS}

    def diff(self, earlier: dict) -> dict:
        return {n: getattr(self, n) - earlier[n] for n in LEDGER_COUNTERS}

    def merge(self, other: "CostLedger") -> None:
        for n in LEDGER_COUNTERS:
            setattr(self, n, getattr(self, n) + getattr(other, n))
        if other.min_level_reached is not None:
            self.observe_level(other.min_level_reached)

    def add_c(self, c: native.HeLedgerC) -> None:
        for n in LEDGER_COUNTERS:
            setattr(self, n, getattr(self, n) + int(getattr(c, n)))

    def to_dict(self) -> dict:
        out = self.snapshot()
        out["min_level_reached"] = self.min_level_reached
        return out

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), sort_keys=True)

    @classmethod
    def from_dict(cls, data: dict) -> "CostLedger":
        return cls(**{k: data[k] for k in (*LEDGER_COUNTERS, "min_level_reached") if k in data})


def _torch():
    import torch  # local import: the CPU-only test suite never needs a device

    return torch


def current_stream_handle(device=None) -> int:
    torch = _torch()
    return torch.cuda.current_stream(device).cuda_stream


class _DeviceCtx:
    """Owns the he_context* of one CUDA device."""

    def __init__(self, params: HeParams, device_index: int, rng_key: bytes | None = None):
        torch = _torch()
        self.device_index = device_index
        p = native.HeParamsC()
        p.mlwe_degree = params.mlwe_degree
        p.mlwe_rank = params.mlwe_rank
        p.moduli[0], p.moduli[1] = params.moduli[:2]
        p.log_delta = params.log_delta
        p.rhombus_degree = params.rhombus_degree
        p.special_prime = params.special_prime
        h = ctypes.c_void_p()
        with torch.cuda.device(device_index):
            native.call("he_context_create", ctypes.byref(p), ctypes.byref(h))
        self.handle = h
        if rng_key is not None:
            native.call("he_context_set_rng_key", h, rng_key)

    def __del__(self):
        try:
            if self.handle:
                native.lib().he_context_destroy(self.handle)
        except Exception:
            pass


@dataclass
class SecretKey:
    """Ternary secret s (int32 [N]) and its NTT per limb (u32 [2, N]), on the device."""

    s: object
    s_ntt: object
    seed: int


@dataclass
class CtBlocks:
    """A batch of level-`level` RLWE ciphertexts encrypting a (d/2) x n_cols activation
    block in the App. A coefficient layout.  data: int32 view of u32
    residues, shape [n_cols / k, limbs, 2 (a, b), N].  Plays hesim.PackedMatrix's role
    (packing.py:32-53): a container with a layout tag checked at kernel boundaries."""

    data: object
    level: int
    n_cols: int
    layout: str = "app_a_coeff"

    @property
    def is_ct(self) -> bool:
        return True

    @property
    def n_ct(self) -> int:
        return int(self.data.shape[0])


@dataclass
class MlweBlocks:
    """Level-0 output of the MLWE PCMM: b' composed back into n_out/k RLWE
    polynomials (out_b [n_out/k, N]) and a' as n_out MLWE rows (out_a [n_out, k*d])."""

    out_b: object
    out_a: object
    level: int
    n_rows: int
    layout: str = "mlwe_rows"

    @property
    def is_ct(self) -> bool:
        return True


class HeContext:
    """Parameters + ledger + device context (hesim.SlotContext's role).

    rng="secure" (default): secrets, masks, errors and key-switching keys are sampled from ChaCha20
    under a fresh 256-bit os.urandom key held by the device context; `seed` arguments are nonces and
    default to fresh random ones (never pass the same seed to two encryptions).  rng="seeded": the
    deterministic splitmix64 path the CPU oracle reproduces word for word -- tests and benchmarks
    only, NOT secure (everything derives from 64-bit seeds)."""

    def __init__(self, params: HeParams | None = None, device=None, rng: str = "secure"):
        if rng not in ("secure", "seeded"):
            raise ValueError(f"rng must be 'secure' or 'seeded', got {rng!r}")
        self.params = params or HeParams.llama()
        self.ledger = CostLedger(min_level_reached=self.params.top_level)
        self._device = device
        self._dev: _DeviceCtx | None = None
        self.rng = rng

    def nonce(self, seed=None) -> int:
        """The seed a sampling call uses: the caller's, or (secure contexts) a fresh random nonce."""
        if seed is not None:
            return int(seed)
        if self.rng == "seeded":
            raise ValueError("a seeded (test) context needs explicit seeds")
        return secrets.randbits(63)

    # -- device --------------------------------------------------------------
    @property
    def device(self):
        torch = _torch()
        if self._device is None:
            if not torch.cuda.is_available():
                raise RuntimeError("the MLWE PCMM path runs on CUDA only (no CPU fallback)")
            self._device = torch.device("cuda", torch.cuda.current_device())
        return torch.device(self._device)

    @property
    def handle(self):
        if self._dev is None:
            dev = self.device
            self._dev = _DeviceCtx(self.params, dev.index if dev.index is not None else 0,
                                   os.urandom(32) if self.rng == "secure" else None)
        return self._dev.handle

    def stream(self) -> int:
        return current_stream_handle(self.device)

    # -- ledger fork / merge (slotsim.py:192-205) -----------------------------
    def fork(self) -> "HeContext":
        child = HeContext.__new__(HeContext)
        child.params = self.params
        child.ledger = CostLedger(min_level_reached=self.params.top_level)
        child._device = self._device
        child._dev = self._dev
        child.rng = self.rng
        return child

    def merge(self, child: "HeContext") -> None:
        self.ledger.merge(child.ledger)

    # -- keys / encryption (test and bench plumbing, all on the device) -------
    def keygen(self, seed: int | None = None) -> SecretKey:
        torch = _torch()
        seed = self.nonce(seed)
        N = self.params.N
        s = torch.empty(N, dtype=torch.int32, device=self.device)
        s_ntt = torch.empty((2, N), dtype=torch.int32, device=self.device)
        native.call("he_keygen", self.handle, seed, s.data_ptr(), s_ntt.data_ptr(), self.stream())
        return SecretKey(s, s_ntt, seed)

    def encrypt_acts(self, sk: SecretKey, acts, seed: int | None = None, r0: int = 0, out=None) -> CtBlocks:
        """Coefficient-encode and encrypt a (d/2) x n_in activation matrix at level 1
        (hesim.pack_sheared / encrypt_matrix role, packing.py:81-91)."""
        torch = _torch()
        seed = self.nonce(seed)
        acts_t = torch.as_tensor(acts, dtype=torch.float64, device=self.device).contiguous()
        tokens, n_in = acts_t.shape
        if tokens != self.params.tokens:
            raise ValueError(f"activation block must have {self.params.tokens} rows, got {tokens}")
        if n_in % self.params.mlwe_rank:
            raise ValueError(f"n_in ({n_in}) must be a multiple of k = {self.params.mlwe_rank}")
        n_ct = n_in // self.params.mlwe_rank
        if out is None:
            out = torch.empty((n_ct, 2, 2, self.params.N), dtype=torch.int32, device=self.device)
        native.call("he_encrypt_acts", self.handle, sk.s_ntt.data_ptr(), acts_t.data_ptr(), n_in, seed, r0,
                    out.data_ptr(), self.stream())
        return CtBlocks(out, level=1, n_cols=n_in)

    def decrypt_phase(self, sk: SecretKey, X: CtBlocks, limb: int = 0):
        torch = _torch()
        ph = torch.empty((X.n_ct, self.params.N), dtype=torch.int64, device=self.device)
        native.call("he_decrypt_rlwe", self.handle, sk.s_ntt.data_ptr(), X.data.data_ptr(), X.n_ct,
                    int(X.data.shape[1]), limb, ph.data_ptr(), self.stream())
        return ph

    def decrypt_acts(self, sk: SecretKey, X: CtBlocks) -> np.ndarray:
        """Decrypt + decode an RLWE block batch back to (d/2) x n_cols floats."""
        ph = self.decrypt_phase(sk, X).cpu().numpy()
        return decode_blocks(self.params, ph, X.n_cols)

    def decrypt_pcmm(self, sk: SecretKey, Y: MlweBlocks, rows=None) -> np.ndarray:
        """Decrypt MLWE output rows on the device and decode to a (d/2) x n_out matrix
        (rows not requested are NaN)."""
        torch = _torch()
        p = self.params
        d, k = p.mlwe_degree, p.mlwe_rank
        n_out = Y.n_rows
        row0, n_rows = (0, n_out) if rows is None else rows
        ph = torch.empty((n_rows, d), dtype=torch.int64, device=self.device)
        native.call("he_decrypt_mlwe", self.handle, sk.s.data_ptr(), Y.out_b.data_ptr(), Y.out_a.data_ptr(),
                    n_out, row0, n_rows, ph.data_ptr(), self.stream())
        return decode_mlwe_rows(p, ph.cpu().numpy(), row0, n_out)


def decode_blocks(params: HeParams, phase: np.ndarray, n_cols: int) -> np.ndarray:
    """Inverse of the App. A coefficient encoding for a batch of RLWE phases [n_ct, N]."""
    from .layout import coeff_table

    d, k = params.mlwe_degree, params.mlwe_rank
    token, col = coeff_table(d, k)
    out = np.zeros((params.tokens, n_cols))
    live = token >= 0
    for r in range(n_cols // k):
        out[token[live], k * r + col[live]] = phase[r, live] / params.delta
    return out


def decode_mlwe_rows(params: HeParams, phase: np.ndarray, row0: int, n_out: int) -> np.ndarray:
    """MLWE output row y (block y // k, component y % k) carries output column
    k (y // k) + sigma(y % k); position m < d/2 is token bitReverse(m)."""
    from .layout import bit_reverse_table, sigma_table

    d, k = params.mlwe_degree, params.mlwe_rank
    half = d // 2
    br = bit_reverse_table(half.bit_length() - 1)
    sig = sigma_table(k)
    out = np.full((half, n_out), np.nan)
    y = row0 + np.arange(phase.shape[0])
    cols = (y // k) * k + np.asarray(sig)[y % k]
    out[np.asarray(br)[:, None], cols[None, :]] = (phase[:, :half] / params.delta).T
    return out


def require_level(level: int) -> None:
    if level < 1:
        raise NeedsBootstrapError("pcmm needs one level")
