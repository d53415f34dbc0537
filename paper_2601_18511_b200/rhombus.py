"""Rhombus PCMv at RLWE degree n = rhombus_degree -- the generation-stage
plaintext-matrix x ciphertext-vector product.

The reference has no PCMv; the entry points follow the calling convention of
its PCMM (pkg/src/hesim/matmul.py:77-162): a weight-side plan built once, a kernel call
``(ctx, plan, keys, x) -> y`` that validates before any compute, raises the reference's
exceptions, consumes one level and records its work in ``ctx.ledger``.

Pipeline (all on the device, include/he_b200.h he_rhombus_*; restated in
oracle/he_oracle_rhombus.c):
  decompose   hybrid key switch s -> s'(X^rho) at degree N, then the free X^rho split into
              rho = N/n RLWE-n pieces
  Rhombus MVM coefficient-encoded pt x ct products in the NTT domain, summed over pieces, then
              PackLWEs output packing with Galois key switches at degree n
  compose     rescale by q1 and the free interleave back to degree N
Vector layout: element e at degree-N coefficient (e / n) + rho h(e mod n), h fixing the top
bit and reversing the others (hesim bitrev.half_reverse).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import native
from .context import HeContext, SecretKey, _torch, require_level


@dataclass
class RhombusKeys:
    s_small: object      # int32 [n]      sparse-ring secret s'
    s_up: object         # int32 [N]      s'(X^rho)
    s_up_ntt: object     # u32 [2, N]     NTT of s'(X^rho) per limb (decryption)
    ksk_dec: object      # u32 [2,2,3,N]  key switch s -> s'(X^rho), NTT domain
    gal: object          # u32 [log n,2,2,3,n] Galois keys, NTT domain


@dataclass
class CtVector:
    """One degree-N RLWE ciphertext holding an n_vals vector in the Rhombus layout.
    data: int32 view of u32, [limbs, 2 (a, b), N] (limbs = level + 1)."""

    data: object
    level: int
    n_vals: int
    key: str = "s"          # "s" (input key) or "s_up" (after the PCMv)
    layout: str = "rhombus_h"

    @property
    def is_ct(self) -> bool:
        return True


@dataclass
class RhombusPlan:
    n_out: int
    n_in: int
    wpt: object
    _handle: object = field(default=None, repr=False)
    _workspace: object = field(default=None, repr=False)
    layout: str = "rhombus_h"

    def workspace(self, device):
        torch = _torch()
        n = ctypes.c_uint64()
        native.call("he_rhombus_workspace_bytes", self._handle, ctypes.byref(n))
        if self._workspace is None or self._workspace.numel() * 4 < n.value:
            self._workspace = torch.empty((n.value + 3) // 4, dtype=torch.int32, device=device)
        return self._workspace

    def __del__(self):
        try:
            if self._handle:
                native.lib().he_rhombus_plan_destroy(self._handle)
        except Exception:
            pass


def rhombus_keygen(ctx: HeContext, sk: SecretKey, seed: int) -> RhombusKeys:
    torch = _torch()
    p = ctx.params
    N, n = p.N, p.rhombus_degree
    lg = n.bit_length() - 1
    dev = ctx.device
    keys = RhombusKeys(
        s_small=torch.empty(n, dtype=torch.int32, device=dev),
        s_up=torch.empty(N, dtype=torch.int32, device=dev),
        s_up_ntt=torch.empty((2, N), dtype=torch.int32, device=dev),
        ksk_dec=torch.empty((2, 2, 3, N), dtype=torch.int32, device=dev),
        gal=torch.empty((lg, 2, 2, 3, n), dtype=torch.int32, device=dev))
    native.call("he_rhombus_keygen", ctx.handle, seed, sk.s.data_ptr(), keys.s_small.data_ptr(), keys.s_up.data_ptr(),
                keys.s_up_ntt.data_ptr(), keys.ksk_dec.data_ptr(), keys.gal.data_ptr(), ctx.stream())
    return keys


def encrypt_vector(ctx: HeContext, sk: SecretKey, v, seed: int, r0: int = 0) -> CtVector:
    torch = _torch()
    vt = torch.as_tensor(v, dtype=torch.float64, device=ctx.device).contiguous().reshape(-1)
    out = torch.empty((1, 2, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    native.call("he_encrypt_vector", ctx.handle, sk.s_ntt.data_ptr(), vt.data_ptr(), int(vt.numel()), seed, r0,
                out.data_ptr(), ctx.stream())
    return CtVector(out[0], level=1, n_vals=int(vt.numel()))


def make_rhombus_plan(ctx: HeContext, weights) -> RhombusPlan:
    """W~ = round(q1 W) as NTT-domain plaintexts, rows/columns in the h layout."""
    torch = _torch()
    w = torch.as_tensor(weights, dtype=torch.float64, device=ctx.device)
    if w.ndim != 2:
        raise ValueError("weights must be a matrix")
    if not bool(torch.isfinite(w).all()):
        raise ValueError("weights must be finite")
    w = w.contiguous()
    n_out, n_in = (int(s) for s in w.shape)
    nb = ctypes.c_uint64()
    native.call("he_rhombus_weight_bytes", ctx.handle, n_out, n_in, ctypes.byref(nb))
    wpt = torch.empty(nb.value // 4, dtype=torch.int32, device=ctx.device)
    native.call("he_rhombus_encode_weights", ctx.handle, w.data_ptr(), n_out, n_in, wpt.data_ptr(), ctx.stream())
    h = ctypes.c_void_p()
    native.call("he_rhombus_plan_create", ctx.handle, wpt.data_ptr(), n_out, n_in, ctypes.byref(h))
    return RhombusPlan(n_out, n_in, wpt, _handle=h)


def pcmv_rhombus(ctx: HeContext, plan: RhombusPlan, keys: RhombusKeys, x: CtVector) -> CtVector:
    torch = _torch()
    if not isinstance(x, CtVector):
        raise TypeError("pcmv consumes a ciphertext operand")
    if x.n_vals != plan.n_in:
        raise ValueError(f"dim mismatch: plan {plan.n_in}, operand {x.n_vals}")
    if x.layout != plan.layout:
        raise ValueError(f"layout mismatch: plan expects {plan.layout}, got {x.layout}")
    if x.key != "s":
        raise ValueError("pcmv input must be under the degree-N secret s")
    require_level(x.level)
    if x.level != 1:
        raise ValueError(f"the Rhombus PCMv runs at level 1, operand is at level {x.level}")
    out = torch.empty((1, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    ws = plan.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_rhombus_run", plan._handle, x.data.data_ptr(), x.level, keys.ksk_dec.data_ptr(),
                keys.gal.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    ctx.ledger.observe_level(x.level - 1)
    return CtVector(out, level=0, n_vals=plan.n_out, key="s_up")


def decrypt_vector(ctx: HeContext, secret_ntt, y: CtVector) -> np.ndarray:
    """Decrypt (limb 0) and decode a Rhombus-layout vector."""
    torch = _torch()
    p = ctx.params
    limbs = int(y.data.shape[0])
    ph = torch.empty((1, p.N), dtype=torch.int64, device=ctx.device)
    native.call("he_decrypt_rlwe", ctx.handle, secret_ntt.data_ptr(), y.data.data_ptr(), 1, limbs, 0, ph.data_ptr(),
                ctx.stream())
    return decode_vector(p, ph[0].cpu().numpy(), y.n_vals)


def vector_positions(params, n_vals: int) -> np.ndarray:
    """degree-N coefficient of each vector element (the Rhombus h layout)."""
    n, rho = params.rhombus_degree, params.rho
    e = np.arange(n_vals)
    k = e % n
    lo = n.bit_length() - 2
    br = np.zeros_like(k)
    low = k & (n // 2 - 1)
    for b in range(lo):
        br |= ((low >> b) & 1) << (lo - 1 - b)
    hk = (k & (n // 2)) | br
    return (e // n) + rho * hk


def decode_vector(params, phase: np.ndarray, n_vals: int) -> np.ndarray:
    return phase[vector_positions(params, n_vals)] / params.delta


def clear_pcmv(weights, v) -> np.ndarray:
    return np.asarray(weights, float) @ np.asarray(v, float)


def pcmv_rhombus_shard(ctx: HeContext, plan: RhombusPlan, keys: RhombusKeys, x: CtVector, piece0: int = 0,
                       opiece0: int = 0):
    """One shard of a sharded PCMv (sharding.pcmv_rhombus_sharded): `plan` covers W[n opiece0 ..,
    n piece0 ..]; returns its LEVEL-1 composed partial output, int32 view of u32 [2 limbs, 2, N]."""
    torch = _torch()
    if not isinstance(x, CtVector):
        raise TypeError("pcmv consumes a ciphertext operand")
    if x.key != "s":
        raise ValueError("pcmv input must be under the degree-N secret s")
    require_level(x.level)
    if x.level != 1:
        raise ValueError(f"the Rhombus PCMv runs at level 1, operand is at level {x.level}")
    out = torch.empty((2, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    ws = plan.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_rhombus_run_shard", plan._handle, x.data.data_ptr(), x.level, keys.ksk_dec.data_ptr(),
                keys.gal.data_ptr(), int(piece0), int(opiece0), out.data_ptr(), ws.data_ptr(), ws.numel() * 4,
                ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    return out


def combine_rhombus_parts(ctx: HeContext, parts, n_vals: int) -> CtVector:
    """Sum level-1 shard outputs [count, 2, 2, N] mod q_i and rescale once -> level-0 CtVector."""
    torch = _torch()
    parts = parts.contiguous()
    out = torch.empty((1, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    led = native.HeLedgerC()
    native.call("he_rhombus_combine", ctx.handle, parts.data_ptr(), int(parts.shape[0]), out.data_ptr(), ctx.stream(),
                ctypes.byref(led))
    ctx.ledger.add_c(led)
    ctx.ledger.observe_level(0)
    return CtVector(out, level=0, n_vals=n_vals, key="s_up")
