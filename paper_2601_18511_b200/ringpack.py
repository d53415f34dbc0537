"""MLWE -> RLWE ring packing of the PCMM output (the hand-off toward
Half-Bootstrap).

The MLWE PCMM leaves each output row as an MLWE ciphertext of degree d and rank k; this step
packs every block of k rows back into ONE level-0 RLWE ciphertext under the degree-N secret,
in the activation coefficient layout of ``HeContext.encrypt_acts`` (so the result is a
``CtBlocks`` the next projection can consume, and its all-gather shrinks ~128x).

Pipeline (all on the device, include/he_b200.h he_pcmm_run_level1 / he_ring_pack_*;
restated in oracle/he_oracle_rhombus.c): the PCMM at level 1 without the rescale (both limbs'
words), then one of two packings, then the rescale by q1 -> level 0:
  "keyswitch" (or_mlwe_to_rlwe): MLWE -> RLWE key switching -- block Y's packed phase is
      b'_Y + sum_j alpha_j(X) s_j(X^k), alpha_j[t + k m] = a'_{kY+t}[j][m]; one hybrid key switch
      (dnum 2, special prime P) per component j from s_j(X^k) to s, summed before one ModDown.
      k keys (~805 MB at Llama parameters), 6 NTTs per (block, j), no automorphisms.
  "keyswitch1" (default, or_mlwe_to_rlwe1): the same with ONE digit (alpha_j mod q0 q1 itself) and two special primes
      P1 = P, P2 (he_ring_pack_special2): 4 NTTs per (block, j) instead of 6, 8 key planes instead of 12.
  "trace" (or_ring_pack): PackLWEs over the subring Z[X^k] on leaves C_y with A_y[k m - j] =
      a'_y[j][m], B_y[k m] = b'_y[m] scaled by k^-1: log2 k levels of E + X^{k/2^l} O +
      sigma_g(E - X^{k/2^l} O), g = 1 + 2^l d, each automorphism followed by a Galois key switch.
      log2 k keys, ~16 NTTs per row.
hesim has no counterpart (its PCMM output stays in slots); the calling convention follows
its PCMM (matmul.py:152-162) like the rest of this package.
"""

from __future__ import annotations

import ctypes

import numpy as np
from dataclasses import dataclass, field

from . import native
from .context import CtBlocks, HeContext, SecretKey, _torch
from .pcmm import MlwePcmmPlan, _check_operand, _note_read


METHODS = {"keyswitch": 0, "trace": 1, "keyswitch1": 2}


def _method(method: str) -> int:
    if method not in METHODS:
        raise ValueError(f"unknown ring packing method {method!r} (expected one of {sorted(METHODS)})")
    return METHODS[method]


@dataclass
class RingPackKeys:
    gal: object          # keyswitch: u32 [k, 2, 2, 3, N] keys s_j(X^k) -> s; trace: u32 [log2 k, 2, 2, 3, N]
                         # Galois keys sigma_{1 + 2^l d}(s) -> s; keyswitch1: u32 [k, 2, 4, N] one-digit keys
                         # modulo q0 q1 P1 P2; NTT domain
    method: str = "keyswitch1"


@dataclass
class RingPackPlan:
    n_out: int
    method: str = "keyswitch1"
    _handle: object = field(default=None, repr=False)
    _workspace: object = field(default=None, repr=False)
    _raw: tuple = field(default=None, repr=False)
    _ctx_keepalive: object = field(default=None, repr=False)

    def workspace(self, device):
        torch = _torch()
        n = ctypes.c_uint64()
        native.call("he_ring_pack_workspace_bytes", self._handle, ctypes.byref(n))
        if self._workspace is None or self._workspace.numel() * 4 < n.value:
            self._workspace = torch.empty((n.value + 3) // 4, dtype=torch.int32, device=device)
        return self._workspace

    def raw(self, ctx: HeContext):
        """level-1 PCMM words: raw_b [2, n_out/k, N], raw_a [2, n_out, N] (reused across calls)"""
        torch = _torch()
        p = ctx.params
        if self._raw is None:
            self._raw = (torch.empty((2, self.n_out // p.mlwe_rank, p.N), dtype=torch.int32, device=ctx.device),
                         torch.empty((2, self.n_out, p.N), dtype=torch.int32, device=ctx.device))
        return self._raw

    def __del__(self):
        try:
            if self._handle:
                native.lib().he_ring_pack_plan_destroy(self._handle)
        except Exception:
            pass


def ring_pack_keygen(ctx: HeContext, sk: SecretKey, seed: int | None = None, method: str = "keyswitch1") -> RingPackKeys:
    torch = _torch()
    seed = ctx.nonce(seed)
    m = _method(method)
    nb = ctypes.c_uint64()
    native.call("he_ring_pack_key_bytes", ctx.handle, m, ctypes.byref(nb))
    N = ctx.params.N
    shape = (nb.value // (4 * 8 * N), 2, 4, N) if m == 2 else (nb.value // (4 * 12 * N), 2, 2, 3, N)
    gal = torch.empty(shape, dtype=torch.int32, device=ctx.device)
    native.call("he_ring_pack_keygen", ctx.handle, m, seed, sk.s.data_ptr(), gal.data_ptr(), ctx.stream())
    return RingPackKeys(gal, method)


def make_ring_pack_plan(ctx: HeContext, n_out: int, method: str = "keyswitch1") -> RingPackPlan:
    h = ctypes.c_void_p()
    native.call("he_ring_pack_plan_create", ctx.handle, int(n_out), _method(method), ctypes.byref(h))
    return RingPackPlan(int(n_out), method, _handle=h, _ctx_keepalive=ctx._dev)


def pcmm_level1(ctx: HeContext, plan: MlwePcmmPlan, X: CtBlocks, raw_b=None, raw_a=None):
    """The PCMM's un-rescaled level-1 words of both limbs (he_pcmm_run_level1)."""
    torch = _torch()
    _check_operand(ctx, plan, X)
    p = ctx.params
    if raw_b is None:
        raw_b = torch.empty((2, plan.n_out // p.mlwe_rank, p.N), dtype=torch.int32, device=ctx.device)
    if raw_a is None:
        raw_a = torch.empty((2, plan.n_out, p.N), dtype=torch.int32, device=ctx.device)
    ws = plan.workspace(ctx.device)
    native.call("he_pcmm_run_level1", plan._handle, X.data.data_ptr(), X.level, raw_b.data_ptr(), raw_a.data_ptr(),
                ws.data_ptr(), ws.numel(), ctx.stream())
    _note_read(X)
    return raw_b, raw_a


def ring_pack(ctx: HeContext, rp: RingPackPlan, keys: RingPackKeys, raw_b, raw_a, out=None) -> CtBlocks:
    torch = _torch()
    p = ctx.params
    if keys.method != rp.method:
        raise ValueError(f"key/plan mismatch: keys for {keys.method!r}, plan for {rp.method!r}")
    if rp._ctx_keepalive is not None and rp._ctx_keepalive is not ctx._dev:
        raise ValueError("ring-pack plan was built under another HeContext")
    if out is None:
        out = torch.empty((rp.n_out // p.mlwe_rank, 1, 2, p.N), dtype=torch.int32, device=ctx.device)
    ws = rp.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_ring_pack_run", rp._handle, raw_b.data_ptr(), raw_a.data_ptr(), keys.gal.data_ptr(),
                out.data_ptr(), ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    return CtBlocks(out, level=0, n_cols=rp.n_out)


def pcmm_packed(ctx: HeContext, plan: MlwePcmmPlan, rp: RingPackPlan, keys: RingPackKeys, X: CtBlocks,
                out=None) -> CtBlocks:
    """Level-1 RLWE block batch encrypting A ((d/2) x n_in) -> level-0 RLWE block batch encrypting
    A @ W^T ((d/2) x n_out) in the input's own layout: the MLWE PCMM then ring packing."""
    if rp.n_out != plan.n_out:
        raise ValueError(f"dim mismatch: ring-pack plan {rp.n_out}, pcmm plan {plan.n_out}")
    raw_b, raw_a = rp.raw(ctx)
    pcmm_level1(ctx, plan, X, raw_b, raw_a)
    k = ctx.params.mlwe_rank
    led = native.HeLedgerC()
    led.pc_mults = (plan.n_out // k) * (plan.n_in // k)
    ctx.ledger.add_c(led)
    Y = ring_pack(ctx, rp, keys, raw_b, raw_a, out)
    ctx.ledger.observe_level(X.level - 1)
    return Y


def mod_raise(ctx: HeContext, Y: CtBlocks, primes) -> object:
    """ModRaise of level-0 RLWE blocks (e.g. the packed PCMM output) into the primes of a bootstrapping
    chain: int32 view of u32 [n_ct, len(primes), 2, N] (he_mod_raise).  The hand-off to Half-Bootstrap
    (PAPER.md:64); the bootstrapping itself is not part of this repository."""
    torch = _torch()
    if Y.level != 0:
        raise ValueError(f"ModRaise takes level-0 ciphertexts, got level {Y.level}")
    pr = torch.as_tensor(np.asarray(primes, dtype=np.int64).astype(np.uint32).view(np.int32), device=ctx.device)
    n_ct = int(Y.data.shape[0])
    out = torch.empty((n_ct, len(primes), 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    native.call("he_mod_raise", ctx.handle, Y.data.data_ptr(), n_ct, pr.data_ptr(), len(primes), out.data_ptr(),
                ctx.stream())
    return out
