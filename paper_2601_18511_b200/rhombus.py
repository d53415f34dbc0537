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
Split point (Rhombus's input/output packing): the input vector uses a window
w = n >> split -- element e at degree-N coefficient (e / w) + rho h_w(e mod w), h_w fixing the top bit
and reversing the others (hesim bitrev.half_reverse, at w = n) -- so each product
of one plaintext with one input piece yields n / w inner products and the output packing needs w - 1
Galois key switches per output piece instead of n - 1.  Default: the largest split the input allows
(w = the smallest power of two >= n_in / rho): 255 key switches per 4096 outputs at n_in = 4096.
Output layout (any split): element r at (r / n) + rho h(r mod n).
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


def rhombus_window(params, n_in: int, split=None) -> int:
    """Input window w = n >> split.  Default: the largest split point whose rho pieces still hold the
    n_in values (w = the smallest power of two >= n_in / rho, at most n)."""
    n, rho = params.rhombus_degree, params.rho
    if split is None:
        w = 1
        while w * rho < n_in:
            w *= 2
        return min(w, n)
    split = int(split)
    if split < 0 or (n >> split) < 1:
        raise ValueError(f"split point {split} outside [0, log2 {n}]")
    w = n >> split
    if w * rho < n_in:
        raise ValueError(f"dim mismatch: split {split} (window {w} x {rho} pieces) cannot hold {n_in} values")
    return w


@dataclass
class CtVector:
    """One degree-N RLWE ciphertext holding an n_vals vector in the Rhombus layout.
    data: int32 view of u32, [limbs, 2 (a, b), N] (limbs = level + 1).  window: the input layout's
    window (0 = the output layout, window n)."""

    data: object
    level: int
    n_vals: int
    key: str = "s"          # "s" (input key) or "s_up" (after the PCMv)
    layout: str = "rhombus_h"
    window: int = 0

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
    window: int = 0
    groups: int = 1
    group: int = 0
    _ctx_keepalive: object = field(default=None, repr=False)

    @property
    def split(self) -> int:
        return int(self.info()[1])

    def info(self) -> list[int]:
        """{window, split, groups, group, input pieces, output pieces, leaves}"""
        buf = (ctypes.c_uint32 * 7)()
        native.call("he_rhombus_plan_info", self._handle, buf)
        return list(buf)

    def key_switches(self) -> int:
        """Galois key switches of one run (one GPU): (w - 1) per output piece."""
        i = self.info()
        return (i[0] // i[2] - 1) * i[5]

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


def rhombus_keygen(ctx: HeContext, sk: SecretKey, seed: int | None = None) -> RhombusKeys:
    torch = _torch()
    seed = ctx.nonce(seed)
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


def encrypt_vector(ctx: HeContext, sk: SecretKey, v, seed: int | None = None, r0: int = 0, window=None,
                   split=None) -> CtVector:
    """Encrypt an n_in-vector in the PCMv input layout of window w (default rhombus_window(n_in))."""
    torch = _torch()
    seed = ctx.nonce(seed)
    vt = torch.as_tensor(v, dtype=torch.float64, device=ctx.device).contiguous().reshape(-1)
    n_vals = int(vt.numel())
    w = int(window) if window is not None else rhombus_window(ctx.params, n_vals, split)
    out = torch.empty((1, 2, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    native.call("he_encrypt_vector_w", ctx.handle, sk.s_ntt.data_ptr(), vt.data_ptr(), n_vals, w, seed, r0,
                out.data_ptr(), ctx.stream())
    return CtVector(out[0], level=1, n_vals=n_vals, window=w)


def make_rhombus_plan(ctx: HeContext, weights, *, split=None, window=None, groups: int = 1,
                      group: int = 0) -> RhombusPlan:
    """W~ = round(q1 W) as NTT-domain plaintexts of the windowed layout (window = n >> split; default the
    largest split the input allows).  groups > 1: the leaf-interleaved row shard `group` of a
    multi-GPU run (sharding.pcmv_rhombus_sharded); column shards pass the full vector's window."""
    torch = _torch()
    w = torch.as_tensor(weights, dtype=torch.float64, device=ctx.device)
    if w.ndim != 2:
        raise ValueError("weights must be a matrix")
    if not bool(torch.isfinite(w).all()):
        raise ValueError("weights must be finite")
    w = w.contiguous()
    n_out, n_in = (int(s) for s in w.shape)
    win = int(window) if window is not None else rhombus_window(ctx.params, n_in, split)
    nb = ctypes.c_uint64()
    native.call("he_rhombus_weight_bytes_w", ctx.handle, n_out, n_in, win, int(groups), ctypes.byref(nb))
    wpt = torch.empty(nb.value // 4, dtype=torch.int32, device=ctx.device)
    native.call("he_rhombus_encode_weights_w", ctx.handle, w.data_ptr(), n_out, n_in, win, int(groups), int(group),
                wpt.data_ptr(), ctx.stream())
    h = ctypes.c_void_p()
    native.call("he_rhombus_plan_create_w", ctx.handle, wpt.data_ptr(), n_out, n_in, win, int(groups), int(group),
                ctypes.byref(h))
    return RhombusPlan(n_out, n_in, wpt, _handle=h, window=win, groups=int(groups), group=int(group),
                       _ctx_keepalive=ctx._dev)


def _check_input(ctx: HeContext, plan: RhombusPlan, x, full_width: bool = True):
    if not isinstance(x, CtVector):
        raise TypeError("pcmv consumes a ciphertext operand")
    if plan._ctx_keepalive is not None and plan._ctx_keepalive is not ctx._dev:
        raise ValueError("plan was built under another HeContext")
    if full_width and x.n_vals != plan.n_in:
        raise ValueError(f"dim mismatch: plan {plan.n_in}, operand {x.n_vals}")
    if x.layout != plan.layout or (x.window or ctx.params.rhombus_degree) != plan.window:
        raise ValueError(f"layout mismatch: plan expects {plan.layout} window {plan.window}, "
                         f"got {x.layout} window {x.window or ctx.params.rhombus_degree}")
    if x.key != "s":
        raise ValueError("pcmv input must be under the degree-N secret s")
    require_level(x.level)
    if x.level != 1:
        raise ValueError(f"the Rhombus PCMv runs at level 1, operand is at level {x.level}")


def pcmv_rhombus(ctx: HeContext, plan: RhombusPlan, keys: RhombusKeys, x: CtVector) -> CtVector:
    torch = _torch()
    _check_input(ctx, plan, x)
    if plan.groups != 1:
        raise ValueError("a leaf-interleaved shard plan runs through sharding.pcmv_rhombus_sharded")
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


def vector_positions(params, n_vals: int, window=None) -> np.ndarray:
    """degree-N coefficient of each vector element: (e / w) + rho h_w(e mod w); window None = n (the
    output layout)."""
    n, rho = params.rhombus_degree, params.rho
    w = n if not window else int(window)
    e = np.arange(n_vals)
    k = e % w
    if w < 2:
        return (e // w).astype(np.int64)
    lo = w.bit_length() - 2
    br = np.zeros_like(k)
    low = k & (w // 2 - 1)
    for b in range(lo):
        br |= ((low >> b) & 1) << (lo - 1 - b)
    hk = (k & (w // 2)) | br
    return (e // w) + rho * hk


def decode_vector(params, phase: np.ndarray, n_vals: int) -> np.ndarray:
    return phase[vector_positions(params, n_vals)] / params.delta


def clear_pcmv(weights, v) -> np.ndarray:
    return np.asarray(weights, float) @ np.asarray(v, float)


def pcmv_rhombus_shard(ctx: HeContext, plan: RhombusPlan, keys: RhombusKeys, x: CtVector, piece0: int = 0,
                       opiece0: int = 0):
    """One column shard of a sharded PCMv (sharding.pcmv_rhombus_sharded): `plan` covers the columns
    [w piece0, ..) of W (window w = the input's); returns its LEVEL-1 composed partial output, int32
    view of u32 [2 limbs, 2, N]."""
    torch = _torch()
    _check_input(ctx, plan, x, full_width=False)
    out = torch.empty((2, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    ws = plan.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_rhombus_run_shard", plan._handle, x.data.data_ptr(), x.level, keys.ksk_dec.data_ptr(),
                keys.gal.data_ptr(), int(piece0), int(opiece0), out.data_ptr(), ws.data_ptr(), ws.numel() * 4,
                ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    return out


def pcmv_rhombus_subtree(ctx: HeContext, plan: RhombusPlan, keys: RhombusKeys, x: CtVector):
    """One leaf-interleaved row shard (plan.groups > 1): products of its leaves and the packing levels
    below the top log2(groups); returns its subtree roots, int32 view of u32 [2 limbs, p_out, 2, n]."""
    torch = _torch()
    _check_input(ctx, plan, x)
    p_out = -(-plan.n_out // ctx.params.rhombus_degree)
    roots = torch.empty((2, p_out, 2, ctx.params.rhombus_degree), dtype=torch.int32, device=ctx.device)
    ws = plan.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_rhombus_run_subtree", plan._handle, x.data.data_ptr(), x.level, keys.ksk_dec.data_ptr(),
                keys.gal.data_ptr(), roots.data_ptr(), ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    return roots


def finish_rhombus_subtrees(ctx: HeContext, plan: RhombusPlan, keys: RhombusKeys, roots) -> CtVector:
    """Top log2(groups) packing levels over the gathered roots [groups, 2, p_out, 2, n] (rank order),
    rescale and compose -> the level-0 CtVector (the one-GPU run's words)."""
    torch = _torch()
    roots = roots.contiguous()
    if int(roots.shape[0]) != plan.groups:
        raise ValueError(f"expected {plan.groups} subtree roots, got {int(roots.shape[0])}")
    out = torch.empty((1, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    ws = plan.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_rhombus_finish", plan._handle, roots.data_ptr(), keys.gal.data_ptr(), out.data_ptr(),
                ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    ctx.ledger.observe_level(0)
    return CtVector(out, level=0, n_vals=plan.n_out, key="s_up")


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
