"""Slot-domain τ-PCMM on the GPU: hesim's own PCMM (pcmm_bsgs, matmul.py:165-176) on real CKKS
ciphertexts (the kernel behind PC-attention).

Same operator API and semantics as the reference:
  make_slot_pcmm_plan(ctx, W, shear_power=0, split=None)   ~ make_pcmm_plan (matmul.py:77-100)
  pcmm_slot_bsgs(ctx, plan, keys, B)                       ~ pcmm_bsgs      (matmul.py:165-176)
  encrypt_packed(ctx, sk, M, shear_power, seed)            ~ pack_sheared   (packing.py:81-91)
A d x d matrix lives row-major in d^2 slots, tiled across the N/2 CKKS slots; the plan's weight
blocks are col_shear(shift_rows(W), l) rolled per (k, jb) exactly as _block_clear (matmul.py:103-105),
CKKS-encoded at scale Delta_w = q1 (slots.py); the op spends (b - 1) + (g - 1) rotations, d
plaintext products and one rescale, like the reference's ledger.  The error contract is the
reference's (_check_operand, matmul.py:139-149), raised before any launch.

Device pipeline (he_slot_pcmm_run, he_rhombus.cu): hoisted baby rotations (one digit decomposition
of the input, X -> X^(5^(i d)) as NTT-index permutations of the digits, one hybrid key switch each),
per giant group a fused NTT-domain multiply-accumulate, the giant rotation at level 1, one rescale.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import native, slots
from .context import HeContext, SecretKey, _torch, require_level
from .errors import NeedsBootstrapError


# ---- cleartext permutations (restated from hesim packing.py:95-130)
def shift_rows(m: np.ndarray) -> np.ndarray:
    d = m.shape[0]
    i, j = np.indices((d, d))
    return m[i, (i + j) % d]


def shift_cols(m: np.ndarray) -> np.ndarray:
    d = m.shape[0]
    i, j = np.indices((d, d))
    return m[(i + j) % d, j]


def col_shear(m: np.ndarray, power: int) -> np.ndarray:
    """M[(i + l j) % d, j]  (shift_cols iterated l times)."""
    d = m.shape[0]
    i, j = np.indices((d, d))
    return np.asarray(m)[(i + power * j) % d, j]


def clear_slot_pcmm(A, B, shear_power: int) -> np.ndarray:
    """What the kernel decodes to: col_shear(A @ B, l) (hesim clear_pcmm, matmul.py:179-181)."""
    return col_shear(np.asarray(A, float) @ np.asarray(B, float), shear_power)


@dataclass(frozen=True)
class BsgsSplit:
    baby: int
    giant: int

    def __post_init__(self):
        if self.baby < 1 or self.giant < 1:
            raise ValueError("split factors must be positive")


def default_split(d: int) -> BsgsSplit:
    """b = g = sqrt(d) when square, else the smallest divisor >= sqrt(d) (matmul.py:49-55)."""
    r = math.isqrt(d)
    if r * r == d:
        return BsgsSplit(r, d // r)
    b = next(b for b in range(r + 1, d + 1) if d % b == 0)
    return BsgsSplit(b, d // b)


@dataclass
class PackedCt:
    """A d x d matrix in the slots of one RLWE ciphertext (hesim PackedMatrix with a ciphertext
    payload).  data: int32 view of u32 [limbs, 2 (a, b), N]."""

    data: object
    level: int
    dim: int
    shear_power: int = 0
    scale: float = 0.0   # encoding scale when known (checked against the plan's input_scale)

    @property
    def is_ct(self) -> bool:
        return True


@dataclass
class SlotPcmmKeys:
    baby: object       # [b - 1, 4, 2, 3, N] gadget rotation keys for steps i d
    giant: object      # [g - 1, 4, 2, 3, N] gadget rotation keys for steps j b d
    steps: tuple = ()


@dataclass
class SlotPcmmPlan:
    dim: int
    shear_power: int
    split: BsgsSplit
    base_clear: np.ndarray
    pts: object = None                  # u32 [d, 2, N] NTT domain (block k = i + j b)
    _handle: object = field(default=None, repr=False)
    _workspace: object = field(default=None, repr=False)

    def workspace(self, device):
        torch = _torch()
        n = ctypes.c_uint64()
        native.call("he_slot_pcmm_workspace_bytes", self._handle, ctypes.byref(n))
        if self._workspace is None or self._workspace.numel() * 4 < n.value:
            self._workspace = torch.empty((n.value + 3) // 4, dtype=torch.int32, device=device)
        return self._workspace

    def __del__(self):
        try:
            if self._handle:
                native.lib().he_slot_pcmm_plan_destroy(self._handle)
        except Exception:
            pass


def block_clear(plan: SlotPcmmPlan, k: int, jb: int) -> np.ndarray:
    """matmul.py:103-105: roll(roll(base, -k, axis=1), -r, axis=0), r = -l k - jb."""
    r = -plan.shear_power * k - jb
    return np.roll(np.roll(plan.base_clear, -k, axis=1), -r, axis=0)


def plan_blocks(plan: SlotPcmmPlan) -> list:
    """The d weight blocks in kernel order k = i + j b (block (i, j) = _block_clear(i + j b, j b))."""
    b, g = plan.split.baby, plan.split.giant
    return [block_clear(plan, i + j * b, j * b) for j in range(g) for i in range(b)]


def encode_blocks(params, plan: SlotPcmmPlan, pt_shift: int = 0) -> np.ndarray:
    """int64 [d, N]: each block flattened row-major, tiled, CKKS-encoded at scale q1 2^pt_shift."""
    sc = float(params.delta_w) * 2.0 ** pt_shift
    return np.stack([slots.encode(blk.reshape(-1), params.N, sc) for blk in plan_blocks(plan)])


def make_slot_pcmm_plan(ctx: HeContext, weights, shear_power: int = 0, split: BsgsSplit | None = None,
                        pt_shift: int = 0, lazy: bool = False) -> SlotPcmmPlan:
    """hesim make_pcmm_plan (matmul.py:77-100) on the device.  Defaults reproduce hesim's scales (weights at
    q1, operand at Delta).  Precision options: lazy -- lazy-ModDown BSGS (baby rotations
    kept mod PQ, weight blocks also mod P, one ModDown per group; needs split.baby % 8 == 0); pt_shift t --
    weight blocks at q1 2^t with the operand encrypted at plan.input_scale = Delta / 2^t (the product still
    lands at Delta), trading the weights' rounding error for operand noise."""
    torch = _torch()
    w = np.asarray(weights, dtype=float)
    d = w.shape[0]
    if w.ndim != 2 or w.shape != (d, d):
        raise ValueError("weights must be square")
    if shear_power < 0:
        raise ValueError("shear_power must be non-negative")
    if split is None:
        split = default_split(d)
    if split.baby * split.giant != d:
        raise ValueError(f"split {split.baby}x{split.giant} does not cover dim {d}")
    if d * d > ctx.params.N // 2 or (ctx.params.N // 2) % (d * d):
        raise ValueError(f"{d}x{d} does not tile the {ctx.params.N // 2} slots")
    if not np.isfinite(w).all():
        raise ValueError("weights must be finite")
    plan = SlotPcmmPlan(d, shear_power, split, col_shear(shift_rows(w), shear_power))
    pt = torch.from_numpy(encode_blocks(ctx.params, plan, pt_shift)).to(ctx.device)
    nm = 3 if lazy else 2
    plan.pts = torch.empty((d, nm, ctx.params.N), dtype=torch.int32, device=ctx.device)
    native.call("he_slot_pcmm_encode_pts_ext", ctx.handle, pt.data_ptr(), d, nm, plan.pts.data_ptr(), ctx.stream())
    h = ctypes.c_void_p()
    if lazy:
        native.call("he_slot_bsgs_plan_create_ext", ctx.handle, plan.pts.data_ptr(), split.baby, split.giant, d, 1,
                    ctypes.byref(h))
    else:
        native.call("he_slot_pcmm_plan_create", ctx.handle, plan.pts.data_ptr(), d, split.baby, split.giant,
                    ctypes.byref(h))
    plan._handle = h
    plan.lazy, plan.pt_shift = lazy, pt_shift
    plan.input_scale = ctx.params.delta / 2.0 ** pt_shift
    return plan


def slot_pcmm_keygen(ctx: HeContext, sk: SecretKey, plan: SlotPcmmPlan, seed: int | None = None) -> SlotPcmmKeys:
    """Rotation keys the plan's BSGS schedule needs: baby steps i d, giant steps j b d."""
    torch = _torch()
    seed = ctx.nonce(seed)
    d, b, g = plan.dim, plan.split.baby, plan.split.giant
    N = ctx.params.N

    def gen(steps):
        keys = torch.empty((max(len(steps), 1), 4, 2, 3, N), dtype=torch.int32, device=ctx.device)
        if steps:
            arr = (ctypes.c_int32 * len(steps))(*steps)
            native.call("he_slot_rotation_keygen", ctx.handle, seed, sk.s.data_ptr(), arr, len(steps), keys.data_ptr(),
                        ctx.stream())
        return keys

    baby = [i * d for i in range(1, b)]
    giant = [j * b * d for j in range(1, g)]
    return SlotPcmmKeys(gen(baby), gen(giant), tuple(baby + giant))


def encrypt_packed(ctx: HeContext, sk: SecretKey, mat, shear_power: int, seed: int | None = None, r0: int = 0,
                   scale: float | None = None) -> PackedCt:
    """Encrypt col_shear(mat, l) row-major in the slots at scale Delta (or a plan's input_scale), level 1
    (hesim pack_sheared)."""
    torch = _torch()
    seed = ctx.nonce(seed)
    m = np.asarray(mat, dtype=float)
    d = m.shape[0]
    if m.shape != (d, d):
        raise ValueError("only square matrices are packed")
    if d * d > ctx.params.N // 2 or (ctx.params.N // 2) % (d * d):
        raise ValueError(f"{d}x{d} does not tile the {ctx.params.N // 2} slots")
    sc = ctx.params.delta if scale is None else float(scale)
    pt = torch.from_numpy(slots.encode(col_shear(m, shear_power).reshape(-1), ctx.params.N, sc)[None])
    pt = pt.to(ctx.device)
    out = torch.empty((2, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    native.call("he_encrypt_poly", ctx.handle, sk.s_ntt.data_ptr(), pt.data_ptr(), 1, seed, r0, out.data_ptr(),
                ctx.stream())
    return PackedCt(out, level=1, dim=d, shear_power=shear_power, scale=sc)


def _check_operand(plan: SlotPcmmPlan, B) -> None:
    """matmul.py:139-149, before any launch."""
    if not getattr(B, "is_ct", False) or not isinstance(B, PackedCt):
        raise TypeError("pcmm consumes a ciphertext operand")
    if B.dim != plan.dim:
        raise ValueError(f"dim mismatch: plan {plan.dim}, operand {B.dim}")
    if B.shear_power != plan.shear_power + 1:
        raise ValueError(f"shear chain broken: plan expects operand power {plan.shear_power + 1}, "
                         f"got {B.shear_power}")
    if B.level < 1:
        raise NeedsBootstrapError("pcmm needs one level")
    want = getattr(plan, "input_scale", None)
    if B.scale and want and B.scale != want:
        raise ValueError(f"scale mismatch: plan expects operand scale {want}, got {B.scale}")


def check_keys(ctx: HeContext, keys: SlotPcmmKeys, steps, giant_components: int = 4) -> None:
    """The rotation keys must be the ones the plan's schedule reads: same steps, gadget baby keys
    (4 components), giant keys with the plan's component count (2 for plain keys); raised before any
    launch (a mismatched layout would make the kernels read past the key buffers)."""
    if not isinstance(keys, SlotPcmmKeys):
        raise TypeError("expected SlotPcmmKeys")
    steps = tuple(int(s) for s in steps)
    if tuple(int(s) for s in keys.steps) != steps:
        raise ValueError(f"key/plan mismatch: keys for rotation steps {tuple(keys.steps)[:6]}..., plan needs "
                         f"{steps[:6]}...")
    N = ctx.params.N
    if tuple(int(v) for v in keys.baby.shape[1:]) != (4, 2, 3, N):
        raise ValueError(f"baby keys have shape {tuple(keys.baby.shape)}, expected [b-1, 4, 2, 3, {N}]")
    if tuple(int(v) for v in keys.giant.shape[1:]) != (giant_components, 2, 3, N):
        raise ValueError(f"giant keys have shape {tuple(keys.giant.shape)}, expected [g-1, {giant_components}, 2, 3, {N}]")


def pcmm_slot_bsgs(ctx: HeContext, plan: SlotPcmmPlan, keys: SlotPcmmKeys, B: PackedCt) -> PackedCt:
    """hesim pcmm_bsgs on the GPU: B (shear power l + 1, level 1) -> A B (shear power l, level 0)."""
    torch = _torch()
    _check_operand(plan, B)
    d, b, g = plan.dim, plan.split.baby, plan.split.giant
    check_keys(ctx, keys, [i * d for i in range(1, b)] + [j * b * d for j in range(1, g)])
    if tuple(int(v) for v in B.data.shape) != (2, 2, ctx.params.N):
        raise ValueError(f"ciphertext has shape {tuple(B.data.shape)}, expected (2, 2, {ctx.params.N})")
    require_level(B.level)
    if B.level != 1:
        raise ValueError(f"the slot-domain PCMM runs at level 1, operand is at level {B.level}")
    out = torch.empty((1, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    ws = plan.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_slot_pcmm_run", plan._handle, B.data.data_ptr(), B.level, keys.baby.data_ptr(),
                keys.giant.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    ctx.ledger.observe_level(B.level - 1)
    return PackedCt(out, level=B.level - 1, dim=plan.dim, shear_power=plan.shear_power, scale=ctx.params.delta)


def pcmm_slot_depth1(ctx: HeContext, plan: SlotPcmmPlan, keys: SlotPcmmKeys, B: PackedCt) -> PackedCt:
    """hesim pcmm_depth1 (matmul.py:152-162): the full k-sum with d - 1 input rotations and one fused
    multiply-accumulate -- the b = d, g = 1 corner of the BSGS schedule, so it runs on a plan made with
    split=BsgsSplit(d, 1) (its blocks are exactly depth1's (k, 0) blocks); the input rotations are
    hoisted and batched into one pass."""
    if plan.split.giant != 1:
        raise ValueError("pcmm_slot_depth1 needs a plan made with split=BsgsSplit(d, 1)")
    return pcmm_slot_bsgs(ctx, plan, keys, B)


def decrypt_packed(ctx: HeContext, sk: SecretKey, Y: PackedCt) -> np.ndarray:
    """Decrypt (limb 0) and decode the first d x d tile of the slots (hesim decode_packed)."""
    torch = _torch()
    limbs = int(Y.data.shape[0])
    ph = torch.empty((1, ctx.params.N), dtype=torch.int64, device=ctx.device)
    native.call("he_decrypt_rlwe", ctx.handle, sk.s_ntt.data_ptr(), Y.data.data_ptr(), 1, limbs, 0, ph.data_ptr(),
                ctx.stream())
    z = slots.decode(ph[0].cpu().numpy(), ctx.params.N, ctx.params.delta, Y.dim * Y.dim)
    return z.reshape(Y.dim, Y.dim)


# ---------------------------------------------------------------- general slot linear maps (pc_linear over rotations)
def make_slot_linear_plan(ctx: HeContext, masks, steps) -> SlotPcmmPlan:
    """out = rescale(sum_t masks[t] * rot(ct, steps[t])), steps[0] = 0: hesim's pc_linear over rotated
    copies (slotsim.py:330-370) as one device op (he_slot_lt_plan_create + he_slot_pcmm_run); masks are
    slot vectors (tiled) encoded at scale q1."""
    torch = _torch()
    steps = [int(v) for v in steps]
    if len(masks) != len(steps) or not steps or steps[0] != 0:
        raise ValueError("need one mask per step and steps[0] == 0")
    N = ctx.params.N
    pt = torch.from_numpy(np.stack([slots.encode(np.asarray(m, float).reshape(-1), N, float(ctx.params.delta_w))
                                    for m in masks])).to(ctx.device)
    n = len(steps)
    plan = SlotPcmmPlan(n, 0, BsgsSplit(n, 1), np.zeros((0, 0)))
    plan.pts = torch.empty((n, 2, N), dtype=torch.int32, device=ctx.device)
    native.call("he_slot_pcmm_encode_pts", ctx.handle, pt.data_ptr(), n, plan.pts.data_ptr(), ctx.stream())
    arr = (ctypes.c_int32 * n)(*steps)
    h = ctypes.c_void_p()
    native.call("he_slot_lt_plan_create", ctx.handle, plan.pts.data_ptr(), n, arr, ctypes.byref(h))
    plan._handle = h
    plan.steps = tuple(steps)
    return plan


def slot_linear_keygen(ctx: HeContext, sk: SecretKey, plan: SlotPcmmPlan, seed: int | None = None) -> SlotPcmmKeys:
    torch = _torch()
    seed = ctx.nonce(seed)
    N = ctx.params.N
    st = list(plan.steps[1:])
    keys = torch.empty((max(len(st), 1), 4, 2, 3, N), dtype=torch.int32, device=ctx.device)
    if st:
        arr = (ctypes.c_int32 * len(st))(*st)
        native.call("he_slot_rotation_keygen", ctx.handle, seed, sk.s.data_ptr(), arr, len(st), keys.data_ptr(),
                    ctx.stream())
    return SlotPcmmKeys(keys, keys[:1], tuple(st))


def slot_linear(ctx: HeContext, plan: SlotPcmmPlan, keys: SlotPcmmKeys, X: PackedCt) -> PackedCt:
    torch = _torch()
    if not isinstance(X, PackedCt):
        raise TypeError("slot_linear consumes a ciphertext operand")
    check_keys(ctx, keys, plan.steps[1:])
    if tuple(int(v) for v in X.data.shape) != (2, 2, ctx.params.N):
        raise ValueError(f"ciphertext has shape {tuple(X.data.shape)}, expected (2, 2, {ctx.params.N})")
    require_level(X.level)
    if X.level != 1:
        raise ValueError(f"slot linear maps run at level 1, operand is at level {X.level}")
    out = torch.empty((1, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    ws = plan.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_slot_pcmm_run", plan._handle, X.data.data_ptr(), X.level, keys.baby.data_ptr(), keys.giant.data_ptr(),
                out.data_ptr(), ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    ctx.ledger.observe_level(X.level - 1)
    return PackedCt(out, level=X.level - 1, dim=X.dim, shear_power=X.shear_power, scale=X.scale)


def rope_masks(d: int, positions) -> tuple:
    """pipeline.py:280-288: cos/sin masks for column-packed vectors (dimension i, token j)."""
    th = np.asarray(positions, float)[:, None] * (10.0 ** (-4.0 * np.arange(d // 2) / d))[None, :]
    c = np.vstack([th.T, th.T])
    cos, sin = np.cos(c), np.sin(c)
    sin[: d // 2] *= -1.0
    return cos, sin


def make_rope_plan(ctx: HeContext, d: int, positions, shear_power: int) -> SlotPcmmPlan:
    """hesim rope_packed (pipeline.py:291-307): cos * x + sin * rowrot(x, d/2) -- one rotation, one level."""
    cos, sin = rope_masks(d, positions)
    return make_slot_linear_plan(ctx, [col_shear(cos, shear_power), col_shear(sin, shear_power)], [0, (d // 2) * d])
