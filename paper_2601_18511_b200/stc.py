"""SlotToCoeffs: slot-encoded activations -> the App. A coefficient layout the MLWE
PCMM consumes, with the bit-reversal of PAPER.md:639-661 fused into the transform.

The paper's attention phase leaves a 128 x 256 activation block per ciphertext in the *slots*,
ct_s[i + 128 j] = A[i][f(j, 8)], and SlotToCoeffs moves slot bitReverse(c, 15) to
coefficient c (ct_d[i][j + 16k] = ct_s[bitReverse(i + 16j + 256k, 15)]).  Composed, that is
exactly the coefficient layout `HeContext.encrypt_acts` produces (c = t + k m <-> A[bitReverse(m)][sigma(t)],
DESIGN.md §2), so the PCMM runs on StC output unchanged.

Algebra.  With n = N/2 slots and slot j = evaluation at zeta^(e_j), e_j = 5^j mod 2N (slots.py), a message
whose slots are z maps to the polynomial m' = sum_s z_s X^(c(s)) (c(s) = bitReverse(s, log n) < N/2) when
the new slots are w = M z with M[j][s] = zeta^(e_j c(s)).  For complex z the imaginary parts land at
X^(N/2 + c(s)) (i = zeta^(e_j N/2) for every j), i.e. M is the whole map -- no conjugation key.  It runs as
one BSGS slot linear map (he_slot_bsgs_plan_create + he_slot_pcmm_run): diagonals u_k[j] = M[j][j + k],
baby steps i < b, giant steps j b, term (i, j) pre-rotated by -j b:  pt_(i,j)[s] = zeta^(e_(s - j b) c(s + i)),
encoded at scale q1 and rescaled by q1 (one level).  n plaintexts (N = 2^16: 32 768 x 2 limbs x 256 KiB
= 17 GiB of HBM, b = 256, g = 128 -> 382 rotation keys); the plaintexts are built on the device with
torch.fft at plan time (host numpy would take minutes at N = 2^16) -- plan preparation, not the op.

Level: the map consumes one level like every pc_linear.  With this context's two-prime chain (q0, q1) the
StC output is at level 0; feeding the PCMM (level 1) needs a third prime above q1 -- the paper's "lower
level -> StC" step sits on a deeper chain.  The coefficient layout is checked here by
decrypt_acts on the StC output.  No reference interface exists (hesim has no StC)."""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import native, slots
from .context import CtBlocks, HeContext, SecretKey, _torch, require_level
from .errors import NeedsBootstrapError
from .layout import bit_reverse_table, coeff_table
from .slotpcmm import BsgsSplit, SlotPcmmKeys, SlotPcmmPlan, check_keys


DEFAULT_PT_SHIFT = 1    # plaintexts at 2 q1, input slots at Delta / 2 (see make_slot_to_coeffs_plan)


@dataclass
class SlotBlocks:
    """Slot-encoded activation ciphertexts: data [n_ct, limbs, 2, N]; ct r carries columns k r .. k r + k - 1
    as ct_s[i + (d/2) j] = A[i][k r + f(j, log k)]."""

    data: object
    level: int
    n_cols: int
    scale: float = 0.0
    layout: str = "app_a_slots"

    @property
    def is_ct(self) -> bool:
        return True

    @property
    def n_ct(self) -> int:
        return int(self.data.shape[0])


def stc_split(n: int) -> BsgsSplit:
    """b >= g powers of two with b g = n (baby rotations are hoisted, giant ones are not)."""
    lb = (n.bit_length() - 1 + 1) // 2
    return BsgsSplit(1 << lb, n >> lb)


def slot_of_coeff(N: int) -> np.ndarray:
    """c -> slot bitReverse(c, log(N/2)) for the n = N/2 live coefficients."""
    return bit_reverse_table((N // 2).bit_length() - 1)


def slot_vectors(params, acts) -> np.ndarray:
    """(d/2) x n_in activations -> [n_in / k, N/2] slot vectors: slot bitReverse(c) holds the value the App. A
    layout puts at coefficient c (so StC lands it there)."""
    a = np.asarray(acts, dtype=float)
    d, k = params.mlwe_degree, params.mlwe_rank
    if a.shape[0] != d // 2 or a.shape[1] % k:
        raise ValueError(f"activation block must be {d // 2} x (multiple of {k}), got {a.shape}")
    n = params.N // 2
    token, col = coeff_table(d, k)
    token, col = token[:n], col[:n]
    rev = slot_of_coeff(params.N)
    out = np.zeros((a.shape[1] // k, n))
    for r in range(a.shape[1] // k):
        out[r, rev] = a[token, k * r + col]
    return out


def stc_plaintexts(params, split: BsgsSplit, k0: int, count: int, device="cpu", pt_shift: int = 0):
    """int64 [count, N] coefficients of terms k0 .. k0 + count - 1 (term k = i + j b), encoded at scale
    q1 2^pt_shift."""
    torch = _torch()
    N, n, b = params.N, params.N // 2, split.baby
    e = torch.as_tensor(slots.slot_exponents(N), device=device)
    cs = torch.as_tensor(np.argsort(slot_of_coeff(N)), device=device)    # c(s) = bitReverse(s) (involution)
    s = torch.arange(n, device=device)
    kk = torch.arange(k0, k0 + count, device=device)
    i, j = (kk % b)[:, None], (kk // b)[:, None]
    expo = (e[(s[None, :] - j * b) % n] * cs[(s[None, :] + i) % n]) % (2 * N)
    ang = expo.to(torch.float64) * (np.pi / N)
    z = torch.complex(torch.cos(ang), torch.sin(ang))
    Z = torch.zeros((count, 2 * N), dtype=torch.complex128, device=device)
    Z[:, e] = z
    Z[:, (2 * N - e) % (2 * N)] = z.conj()
    m = torch.fft.fft(Z, dim=1)[:, :N].real / N
    return torch.round(m * float(params.delta_w) * 2.0 ** pt_shift).to(torch.int64)


def make_slot_to_coeffs_plan(ctx: HeContext, split: BsgsSplit | None = None, batch: int = 256,
                             pt_shift: int = DEFAULT_PT_SHIFT, lazy: bool = True) -> SlotPcmmPlan:
    """The n = N/2 diagonals of M, BSGS-ordered and NTT'd into [n, 2, N] device residues, encoded at scale
    q1 2^pt_shift: the output keeps scale Delta when the input slots carry Delta / 2^pt_shift
    (plan.input_scale, what encrypt_slots uses).  lazy (default): the baby rotations stay in the PQ basis
    straight from the key MAC and each giant group sum is ModDown'd once after the products (plaintexts also
    mod P, HE_SLOT_LAZY_MODDOWN), so their ModDown rounding noise (~60 per coefficient with the dense key) is
    never amplified by the map.  Error (tools/stc_precision.py, N = 2^16): lazy 13.1 / 13.5 / 12.5 bits at
    pt_shift 0 / 1 / 2 (plaintext rounding vs input noise balance at 1); eager ModDown 10.7 bits at 0, 11.6
    at -1 (rotation noise, amplified sqrt(n), dominates)."""
    torch = _torch()
    N, n = ctx.params.N, ctx.params.N // 2
    split = split or stc_split(n)
    if split.baby * split.giant != n:
        raise ValueError(f"split {split.baby}x{split.giant} does not cover the {n} slots")
    plan = SlotPcmmPlan(n, 0, split, np.zeros((0, 0)))
    nm = 3 if lazy else 2
    plan.pts = torch.empty((n, nm, N), dtype=torch.int32, device=ctx.device)
    # small rings build the plaintexts on the host (deterministic, and the same integers the oracle tests
    # use: a device FFT can round a coefficient at .5 the other way); N = 2^16 needs the device's FFT
    dev = "cpu" if N <= 8192 else ctx.device
    for k0 in range(0, n, batch):
        cnt = min(batch, n - k0)
        pt = stc_plaintexts(ctx.params, split, k0, cnt, dev, pt_shift).to(ctx.device).contiguous()
        native.call("he_slot_pcmm_encode_pts_ext", ctx.handle, pt.data_ptr(), cnt, nm, plan.pts[k0].data_ptr(),
                    ctx.stream())
    h = ctypes.c_void_p()
    # lazy plans also switch the giant rotations with plain dnum-2 keys (HE_SLOT_PLAIN_GIANT): after the
    # products their noise lands at scale Delta q1, so the gadget split buys nothing there
    native.call("he_slot_bsgs_plan_create_ext", ctx.handle, plan.pts.data_ptr(), split.baby, split.giant, 1,
                3 if lazy else 0, ctypes.byref(h))
    plan.lazy = lazy
    plan.plain_giant = lazy
    plan._handle = h
    b, g = split.baby, split.giant
    plan.steps = tuple(range(1, b)) + tuple(j * b for j in range(1, g))
    plan.pt_shift = pt_shift
    plan.input_scale = ctx.params.delta / 2.0 ** pt_shift
    return plan


def slot_to_coeffs_keygen(ctx: HeContext, sk: SecretKey, plan: SlotPcmmPlan, seed: int | None = None) -> SlotPcmmKeys:
    """Gadget rotation keys for baby steps 1 .. b-1 and giant steps j b."""
    torch = _torch()
    seed = ctx.nonce(seed)
    N, b, g = ctx.params.N, plan.split.baby, plan.split.giant

    def gen(steps, plain=False):
        keys = torch.empty((max(len(steps), 1), 2 if plain else 4, 2, 3, N), dtype=torch.int32, device=ctx.device)
        if steps:
            arr = (ctypes.c_int32 * len(steps))(*steps)
            native.call("he_slot_rotation_keygen_plain" if plain else "he_slot_rotation_keygen", ctx.handle, seed,
                        sk.s.data_ptr(), arr, len(steps), keys.data_ptr(), ctx.stream())
        return keys

    baby, giant = list(range(1, b)), [j * b for j in range(1, g)]
    return SlotPcmmKeys(gen(baby), gen(giant, getattr(plan, "plain_giant", False)), tuple(baby + giant))


def encrypt_slots(ctx: HeContext, sk: SecretKey, acts, seed: int | None = None, r0: int = 0,
                  scale: float | None = None) -> SlotBlocks:
    """Slot-encode and encrypt a (d/2) x n_in activation block at level 1, one ct per k columns -- the state
    the attention phase leaves behind.  scale: the plan's input_scale (Delta 2^-pt_shift,
    Delta / 2 by default) so that StC lands at Delta; None = the default plan's."""
    torch = _torch()
    seed = ctx.nonce(seed)
    z = slot_vectors(ctx.params, acts)
    sc = ctx.params.delta / 2.0 ** DEFAULT_PT_SHIFT if scale is None else float(scale)
    pt = torch.from_numpy(np.stack([slots.encode(v, ctx.params.N, sc) for v in z])).to(ctx.device)
    out = torch.empty((z.shape[0], 2, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    native.call("he_encrypt_poly", ctx.handle, sk.s_ntt.data_ptr(), pt.data_ptr(), z.shape[0], seed, r0,
                out.data_ptr(), ctx.stream())
    return SlotBlocks(out, level=1, n_cols=int(np.asarray(acts).shape[1]), scale=sc)


def slot_to_coeffs(ctx: HeContext, plan: SlotPcmmPlan, keys: SlotPcmmKeys, X: SlotBlocks) -> CtBlocks:
    """SlotBlocks (level l) -> CtBlocks in the App. A coefficient layout (level l - 1); one BSGS map per ct."""
    torch = _torch()
    if not getattr(X, "is_ct", False) or not isinstance(X, SlotBlocks):
        raise TypeError("slot_to_coeffs consumes slot-encoded ciphertexts (SlotBlocks)")
    if X.level < 1:
        raise NeedsBootstrapError("slot_to_coeffs needs one level")
    require_level(X.level)
    if X.level != 1:
        raise ValueError(f"slot_to_coeffs runs at level 1 on this two-prime chain, operand is at level {X.level}")
    if X.scale and X.scale != plan.input_scale:
        raise ValueError(f"scale mismatch: plan expects input scale {plan.input_scale}, operand has {X.scale}")
    N = ctx.params.N
    b, g = plan.split.baby, plan.split.giant
    check_keys(ctx, keys, list(range(1, b)) + [j * b for j in range(1, g)],
               2 if getattr(plan, "plain_giant", False) else 4)
    if tuple(int(v) for v in X.data.shape) != (X.n_ct, 2, 2, N):
        raise ValueError(f"slot ciphertexts have shape {tuple(X.data.shape)}, expected ({X.n_ct}, 2, 2, {N})")
    out = torch.empty((X.n_ct, 1, 2, N), dtype=torch.int32, device=ctx.device)
    ws = plan.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_slot_pcmm_run_batch", plan._handle, X.data.data_ptr(), X.n_ct, X.level, keys.baby.data_ptr(),
                keys.giant.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    ctx.ledger.observe_level(X.level - 1)
    return CtBlocks(out, level=X.level - 1, n_cols=X.n_cols)
