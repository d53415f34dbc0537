"""The modulus chain above the PCMM's level 1: level lowering and the Cooley-Tukey-factorized SlotToCoeffs
 -- "Lower the total level to 4; Perform SlotToCoeffs to level 1", with
SlotToCoeffs as a homomorphic DFT in "variants of the Cooley-Tukey decomposition".

Factorization.  With n = N/2 slots (slot j <-> zeta^(5^j)) the map StC applies in the slots is
M[j][s] = zeta^(5^j bitReverse(s)) (stc.py).  Evaluating the polynomial sum_s z_s X^(bitReverse(s)) at the
points zeta^(5^j) is a radix-2 decimation-in-time recursion whose sub-problems are contiguous halves of z,
so M = L_log n ... L_1 with NO permutation (the bit reversal of PAPER.md:661 is absorbed, as in stc.py):
L_k (block length len = 2^k) maps (u, v) = (z[i + j], z[i + j + len/2]) to (u + w_j v, u - w_j v),
w_j = exp(i pi (5^j mod 4 len) / (2 len)) -- three slot diagonals (offsets 0, +-len/2).  Grouping r
consecutive layers gives 2^(r+1) - 1 diagonals at stride 2^k0 (fewer when they wrap around the n slots);
at N = 2^16 the 15 layers form three maps of 63, 63 and 32 diagonals, i.e. BSGS maps with 15 + 4, 15 + 4 and
15 + 1 rotations (54 in all, vs 382 for the dense one-level map of stc.py) and 160 plaintexts instead of
32 768.  Each map consumes one level (he_chain.cu: hybrid key switching with one digit per prime), so the
three run at levels 4, 3, 2 and hand the PCMM its level-1 input.

Scales: map k encodes its diagonals (|entries| <= 1) at q_k / 2^shift_k and rescales by q_k, so the scale drops
by 2^shift_k per map and the output lands at exactly Delta (the App. A coefficient layout `encrypt_acts`
produces) when the input slots carry Delta 2^(sum shift).  The default shifts (6, 6, 6) keep every map's
input at >= Delta 2^6: the baby rotations' key-switching noise (~600 per coefficient with one-prime digits
and P ~ 2^30), amplified by the remaining butterfly layers, then sits below the plaintexts' rounding
(~2^24-scale diagonals).  Measured at N = 2^16 (max error over 32 768 coefficients): shifts (0, 0, 3) 2^-6.2,
(3, 3, 3) 2^-12.2, (6, 6, 6) 2^-16.5, (10, 10, 10) 2^-13.0, (12, 12, 12) 2^-10.9.  No hesim interface exists (it has no StC);
the integer algorithm is restated in oracle/he_oracle_chain.c and checked word for word.
"""

from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass, field

import numpy as np

from . import native, slots
from .context import CtBlocks, HeContext, SecretKey, _torch
from .errors import NeedsBootstrapError
from .stc import SlotBlocks, slot_vectors


# ---------------------------------------------------------------- the chain device object
class _Chain:
    def __init__(self, ctx: HeContext):
        p = ctx.params
        primes = (ctypes.c_uint32 * len(p.moduli))(*p.moduli)
        h = ctypes.c_void_p()
        native.call("he_chain_create", ctx.handle, primes, len(p.moduli), ctypes.byref(h))
        self.handle = h
        self._dev = ctx._dev   # keeps the context (its RNG key, its q0 / q1 tables) alive

    def __del__(self):
        try:
            if self.handle:
                native.lib().he_chain_destroy(self.handle)
        except Exception:
            pass


def chain_of(ctx: HeContext) -> _Chain:
    if len(ctx.params.moduli) < 3:
        raise ValueError("this context has no chain above level 1 (use HeParams.llama_chain / toy_chain)")
    ch = getattr(ctx, "_chain", None)
    if ch is None or ch._dev is not ctx._dev:
        ch = _Chain(ctx)
        ctx._chain = ch
    return ch


def encrypt_slots_at(ctx: HeContext, sk: SecretKey, acts, level: int | None = None, seed: int | None = None,
                     scale: float | None = None, r0: int = 0) -> SlotBlocks:
    """Slot-encode and encrypt a (d/2) x n_in activation block at `level` (default: the top of the chain)."""
    torch = _torch()
    p = ctx.params
    level = p.top_level if level is None else int(level)
    if not 1 <= level <= p.top_level:
        raise ValueError(f"level {level} outside [1, {p.top_level}]")
    seed = ctx.nonce(seed)
    z = slot_vectors(p, acts)
    sc = p.delta if scale is None else float(scale)
    pt = torch.from_numpy(np.stack([slots.encode(v, p.N, sc) for v in z])).to(ctx.device)
    out = torch.empty((z.shape[0], level + 1, 2, p.N), dtype=torch.int32, device=ctx.device)
    native.call("he_chain_encrypt", chain_of(ctx).handle, sk.s.data_ptr(), pt.data_ptr(), z.shape[0], level, seed, r0,
                out.data_ptr(), ctx.stream())
    return SlotBlocks(out, level=level, n_cols=int(np.asarray(acts).shape[1]), scale=sc)


def encrypt_coeffs_at(ctx: HeContext, sk: SecretKey, pt, level: int | None = None, seed: int | None = None,
                      r0: int = 0) -> CtBlocks:
    """Encrypt int64 coefficient plaintexts [n_ct, N] (e.g. or_encode_acts of an activation block) at `level`."""
    torch = _torch()
    p = ctx.params
    level = p.top_level if level is None else int(level)
    if not 0 <= level <= p.top_level:
        raise ValueError(f"level {level} outside [0, {p.top_level}]")
    pt = torch.as_tensor(np.asarray(pt, dtype=np.int64)).reshape(-1, p.N).to(ctx.device)
    out = torch.empty((pt.shape[0], level + 1, 2, p.N), dtype=torch.int32, device=ctx.device)
    native.call("he_chain_encrypt", chain_of(ctx).handle, sk.s.data_ptr(), pt.data_ptr(), pt.shape[0], level,
                ctx.nonce(seed), r0, out.data_ptr(), ctx.stream())
    return CtBlocks(out, level=level, n_cols=0)


def decrypt_exact(ctx: HeContext, sk: SecretKey, data) -> np.ndarray:
    """The integer phase b + a s of chain ciphertexts [n_ct, level + 1, 2, N] by CRT over all their limbs
    (object array of Python ints, centred mod Q_level): e.g. m + q0 I(X) after ModRaise."""
    torch = _torch()
    p = ctx.params
    n_ct, nl = int(data.shape[0]), int(data.shape[1])
    ch = chain_of(ctx)
    res = []
    for j in range(nl):
        ph = torch.empty((n_ct, p.N), dtype=torch.int64, device=ctx.device)
        native.call("he_chain_decrypt", ch.handle, sk.s.data_ptr(), data.data_ptr(), n_ct, nl - 1, j, ph.data_ptr(),
                    ctx.stream())
        res.append(ph.cpu().numpy().astype(object))
    Q = 1
    for q in p.moduli[:nl]:
        Q *= q
    acc = np.zeros_like(res[0])
    for j, q in enumerate(p.moduli[:nl]):
        Qj = Q // q
        acc = acc + res[j] % q * Qj * pow(Qj, -1, q)
    acc = acc % Q
    return np.where(acc > Q // 2, acc - Q, acc)


def lower_level(X, level: int):
    """Drop the limbs above `level` (a ciphertext mod Q_L is one mod every divisor Q_l: no noise, no kernel)."""
    if not getattr(X, "is_ct", False):
        raise TypeError("lower_level takes a ciphertext container")
    if not 0 <= level <= X.level:
        raise ValueError(f"cannot lower level {X.level} to {level}")
    data = X.data[:, : level + 1].contiguous() if level < X.level else X.data
    return dataclasses.replace(X, data=data, level=level)


# ---------------------------------------------------------------- the Cooley-Tukey factorization (host, plan time)
def special_fft_layers(N: int) -> list[dict]:
    """L_1 .. L_log n as {slot offset: diagonal} (out = sum_o diag_o * roll(in, -o))."""
    n = N // 2
    e = slots.slot_exponents(N)
    x = np.arange(n)
    out = []
    ln = 2
    while ln <= n:
        h = ln // 2
        jj = x % ln
        first = jj < h
        w = np.exp(1j * np.pi * (e[jj % h] % (4 * ln)) / (2 * ln))
        D: dict = {}
        _merge(D, 0, np.where(first, 1.0, -w), n)
        _merge(D, h, np.where(first, w, 0.0), n)
        _merge(D, -h, np.where(first, 0.0, 1.0), n)
        out.append(D)
        ln *= 2
    return out


def special_ifft_layers(N: int) -> list[dict]:
    """The inverses of special_fft_layers' L_1 .. L_log n (same index): (x, y) at (p, p + len/2) ->
    ((x + y) / 2, (x - y) / (2 w_p)) -- three diagonals again, entries of modulus 1/2."""
    n = N // 2
    e = slots.slot_exponents(N)
    x = np.arange(n)
    out = []
    ln = 2
    while ln <= n:
        h = ln // 2
        jj = x % ln
        first = jj < h
        w = np.exp(1j * np.pi * (e[jj % h] % (4 * ln)) / (2 * ln))
        D: dict = {}
        _merge(D, 0, np.where(first, 0.5, -0.5 / w), n)
        _merge(D, h, np.where(first, 0.5, 0.0), n)
        _merge(D, -h, np.where(first, 0.0, 0.5 / w), n)
        out.append(D)
        ln *= 2
    return out


def _merge(D: dict, o: int, v, n: int) -> None:
    o %= n
    D[o] = D.get(o, 0) + np.asarray(v, dtype=np.complex128)


def compose(A: dict, B: dict, n: int) -> dict:
    """A @ B in diagonal form."""
    C: dict = {}
    for a, da in A.items():
        for b, db in B.items():
            _merge(C, a + b, da * np.roll(db, -a), n)
    return C


def apply_diagonals(D: dict, v):
    return sum(d * np.roll(v, -o) for o, d in D.items())


def layer_groups(log_n: int, levels: int) -> list[int]:
    """Layers per map, as even as possible, larger groups first."""
    return [log_n // levels + (1 if i < log_n % levels else 0) for i in range(levels)]


def stc_factors(N: int, levels: int = 3) -> list[dict]:
    """The maps G_1 .. G_levels (application order) with M = G_levels ... G_1; each entry:
    {"diags": {offset: diag}, "stride": 2^k0, "T": centre offset / stride, "count": terms}."""
    n = N // 2
    L = special_fft_layers(N)
    out, k = [], 0
    for sz in layer_groups(n.bit_length() - 1, levels):
        G = L[k]
        for lay in L[k + 1:k + sz]:
            G = compose(lay, G, n)
        stride = 1 << k
        span = n // stride
        T = (1 << sz) - 1
        if 2 * T + 1 > span:   # the offsets wrap around the slots: terms 0 .. span - 1
            T, count = 0, span
        else:
            count = 2 * T + 1
        out.append({"diags": G, "stride": stride, "T": T, "count": count})
        k += sz
    return out


def cts_factors(N: int, levels: int = 3) -> list[dict]:
    """CoeffToSlots = M^-1 = L_1^-1 ... L_log n^-1 as `levels` maps in application order: the layer groups of
    stc_factors taken last group first, each G_g^-1 = L_k^-1 ... L_(k + sz - 1)^-1 (same offsets, stride, T)."""
    n = N // 2
    Li = special_ifft_layers(N)
    groups, k = [], 0
    for sz in layer_groups(n.bit_length() - 1, levels):
        groups.append((k, sz))
        k += sz
    out = []
    for k, sz in reversed(groups):
        G = Li[k + sz - 1]
        for lay in reversed(Li[k:k + sz - 1]):
            G = compose(lay, G, n)
        stride = 1 << k
        span = n // stride
        T = (1 << sz) - 1
        if 2 * T + 1 > span:
            T, count = 0, span
        else:
            count = 2 * T + 1
        out.append({"diags": G, "stride": stride, "T": T, "count": count})
    return out


def bsgs_shape(count: int) -> tuple[int, int]:
    """b ~ 2 sqrt(count): a giant rotation needs its own digit decomposition (~4x the NTTs of a hoisted baby
    rotation at level 4), so fewer, larger giant groups win (63 terms: 16 x 4, 15 + 4 key switches)."""
    b = 1
    while b * b < 4 * count:
        b *= 2
    b = min(b, 1 << (count - 1).bit_length())
    return b, -(-count // b)


# ---------------------------------------------------------------- plans, keys, run
_SHARED_WS: dict = {}


@dataclass
class ChainMap:
    level: int
    b: int
    g: int
    stride: int
    T: int
    pts: object                          # u32 [b g][level + 1][N] NTT domain
    pts_int: object = None               # int64 [b g][N] (test access: the integers the oracle takes)
    n_slots: int = 0
    _handle: object = field(default=None, repr=False)
    _workspace: object = field(default=None, repr=False)

    @property
    def baby_steps(self) -> list[int]:
        return [i * self.stride for i in range(1, self.b)]

    @property
    def giant_steps(self) -> list[int]:
        return [(j * self.b - self.T) * self.stride for j in range(self.g)]

    @property
    def rotations(self) -> int:
        """key switches per ciphertext: b - 1 baby + the giant groups with a nonzero step"""
        return (self.b - 1) + sum(1 for s in self.giant_steps if s % self.n_slots)

    def workspace(self, device):
        """Scratch shared by every map on the device (grown to the largest need; calls on one stream)."""
        torch = _torch()
        nb = ctypes.c_uint64()
        native.call("he_chain_map_workspace_bytes", self._handle, ctypes.byref(nb))
        key = torch.device(device)
        ws = _SHARED_WS.get(key)
        if ws is None or ws.numel() * 4 < nb.value:
            _SHARED_WS.pop(key, None)
            ws = torch.empty((nb.value + 3) // 4, dtype=torch.int32, device=key)
            _SHARED_WS[key] = ws
        self._workspace = ws
        return ws

    def __del__(self):
        try:
            if self._handle:
                native.lib().he_chain_map_destroy(self._handle)
        except Exception:
            pass


@dataclass
class FactorizedStcPlan:
    maps: list
    input_level: int
    output_level: int
    input_scale: float
    shifts: tuple
    _chain: object = field(default=None, repr=False)
    pre_log2: int = 0                    # CoeffToSlots: the input is multiplied by 2^pre_log2 first

    @property
    def rotations(self) -> int:
        return sum(m.rotations for m in self.maps)

    @property
    def plaintexts(self) -> int:
        return sum(m.b * m.g for m in self.maps)


@dataclass
class ChainMapKeys:
    baby: object
    giant: object
    baby_steps: tuple
    giant_steps: tuple
    level: int


def make_factorized_stc_plan(ctx: HeContext, levels: int = 3, shifts=None,
                             input_level: int | None = None) -> FactorizedStcPlan:
    """The `levels` maps of the factorized SlotToCoeffs as chain BSGS plans (default: three, input at level 4 ->
    output at level 1, the PCMM's input level); map k's plaintexts at q_k / 2^shifts[k] (default 6 each),
    input slots at plan.input_scale = Delta 2^sum(shifts)."""
    return _factorized_plan(ctx, stc_factors, levels, (6,) * levels if shifts is None else shifts, input_level)


def make_factorized_cts_plan(ctx: HeContext, levels: int = 3, shifts=None, input_level: int | None = None,
                             pre_log2: int = 0) -> FactorizedStcPlan:
    """CoeffToSlots, the linear first half of the Half-Bootstrap after ModRaise: the inverse of the
    factorized SlotToCoeffs, M^-1 as `levels` chain maps (default: input at the top level).  A ciphertext whose
    phase has coefficients p_c comes out with slot s = (p_(bitReverse(s)) + i p_(N/2 + bitReverse(s))) times
    2^(pre_log2 - sum(shifts)) (SlotBlocks.scale): the input is multiplied by the integer 2^pre_log2 (no level) and
    map k's plaintexts are encoded at q_k 2^-shifts[k].

    Precision (measured at N = 2^16 on a ModRaised ciphertext, tools/cts_precision.py): the plaintext rounding of
    every map, ~2^-23.7 of an entry at scale q_k ~ 2^30 acting on slot values up to sqrt(N/2) |p| wide, dominates
    the key-switching noise until the shifts reach ~-10 each; past that the key-switching noise (absolute, ~2^20 in
    the slots) is what is left and the integer pre-multiplication lifts the signal over it.  The output -- |p| ~
    q0 |I| ~ 2^38 after ModRaise, times the total scale-up T -- has to stay inside the output modulus (output
    coefficients measured at 2^(30.3 + T)).  Default: T = log2 Q_out - 33.5; below 40 all of it as shifts (output
    level 1, q0 q1 ~ 2^50: T = 16, shifts (-6, -5, -5), 2^-16.4 q0), else pre_log2 8 and shifts of -12 (output
    level 2 on llama_chain(4): 2^-22.9 q0)."""
    p = ctx.params
    input_level = p.top_level if input_level is None else int(input_level)
    if shifts is None:
        out_level = input_level - levels
        qlog = sum(np.log2(float(q)) for q in p.moduli[:max(out_level, 0) + 1])
        T = max(int(np.floor(qlog - 33.5)), 0)
        if T >= 40 and pre_log2 == 0:
            pre_log2, T = 8, T - 8
        T = min(T, 12 * levels)
        shifts = tuple(-(T // levels + (1 if i < T % levels else 0)) for i in range(levels))
    plan = _factorized_plan(ctx, cts_factors, levels, shifts, input_level)
    if not 0 <= int(pre_log2) <= 31:
        raise ValueError("pre_log2 must be in [0, 31]")
    plan.pre_log2 = int(pre_log2)
    return plan


def _factorized_plan(ctx, factors, levels, shifts, input_level) -> FactorizedStcPlan:
    torch = _torch()
    p = ctx.params
    shifts = tuple(int(v) for v in shifts)
    if len(shifts) != levels or min(shifts) < -20 or max(shifts) > 20:
        raise ValueError(f"need {levels} shifts in [-20, 20], got {shifts}")
    input_level = levels + 1 if input_level is None else int(input_level)
    if input_level > p.top_level or input_level - levels < 0:
        raise ValueError(f"{levels} maps from level {input_level} do not fit the chain (top level {p.top_level})")
    ch = chain_of(ctx)
    N, n = p.N, p.N // 2
    maps = []
    for k, f in enumerate(factors(N, levels)):
        level = input_level - k
        scale = float(p.moduli[level]) / 2.0 ** shifts[k]
        b, g = bsgs_shape(f["count"])
        s, T = f["stride"], f["T"]
        pts = np.zeros((b * g, N), dtype=np.int64)
        for j in range(g):
            for i in range(b):
                t = i + j * b
                if t >= f["count"]:
                    continue
                d = f["diags"].get(((t - T) * s) % n)
                if d is None:
                    continue
                pts[t] = slots.encode(np.roll(d, (j * b - T) * s), N, scale)
        pt_dev = torch.from_numpy(pts).to(ctx.device)
        res = torch.empty((b * g, level + 1, N), dtype=torch.int32, device=ctx.device)
        native.call("he_chain_encode_pts", ch.handle, pt_dev.data_ptr(), b * g, level, res.data_ptr(), ctx.stream())
        h = ctypes.c_void_p()
        native.call("he_chain_map_create", ch.handle, res.data_ptr(), level, b, g, s, T, ctypes.byref(h))
        maps.append(ChainMap(level, b, g, s, T, res, pts, n, _handle=h))
    return FactorizedStcPlan(maps, input_level, input_level - levels, p.delta * 2.0 ** sum(shifts), shifts, _chain=ch)


def chain_map_keygen(ctx: HeContext, sk: SecretKey, m: ChainMap, seed: int | None = None) -> ChainMapKeys:
    torch = _torch()
    ch = chain_of(ctx)
    seed = ctx.nonce(seed)
    words = ctypes.c_uint64()
    native.call("he_chain_key_words", ch.handle, m.level, ctypes.byref(words))

    def gen(steps):
        keys = torch.empty((max(len(steps), 1), int(words.value)), dtype=torch.int32, device=ctx.device)
        if steps:
            arr = (ctypes.c_int32 * len(steps))(*steps)
            native.call("he_chain_rotation_keygen", ch.handle, seed, sk.s.data_ptr(), m.level, arr, len(steps),
                        keys.data_ptr(), ctx.stream())
        return keys

    return ChainMapKeys(gen(m.baby_steps), gen(m.giant_steps), tuple(m.baby_steps), tuple(m.giant_steps), m.level)


def factorized_stc_keygen(ctx: HeContext, sk: SecretKey, plan: FactorizedStcPlan, seed: int | None = None) -> list:
    return [chain_map_keygen(ctx, sk, m, None if seed is None else seed + 7919 * k) for k, m in enumerate(plan.maps)]


def chain_map(ctx: HeContext, m: ChainMap, keys: ChainMapKeys, data, level: int):
    """One map on ciphertexts data [n_ct, level + 1, 2, N] -> [n_ct, level, 2, N]."""
    torch = _torch()
    if level < 1:
        raise NeedsBootstrapError("a slot linear map needs one level")
    if level != m.level:
        raise ValueError(f"map built for level {m.level}, operand at level {level}")
    if tuple(keys.baby_steps) != tuple(m.baby_steps) or tuple(keys.giant_steps) != tuple(m.giant_steps) \
            or keys.level != m.level:
        raise ValueError("key/plan mismatch: rotation keys made for another map")
    n_ct = int(data.shape[0])
    if tuple(int(v) for v in data.shape[1:]) != (level + 1, 2, ctx.params.N):
        raise ValueError(f"ciphertexts have shape {tuple(data.shape)}, expected [n, {level + 1}, 2, {ctx.params.N}]")
    out = torch.empty((n_ct, level, 2, ctx.params.N), dtype=torch.int32, device=ctx.device)
    ws = m.workspace(ctx.device)
    led = native.HeLedgerC()
    native.call("he_chain_map_run", m._handle, data.data_ptr(), n_ct, level, keys.baby.data_ptr(), keys.giant.data_ptr(),
                out.data_ptr(), ws.data_ptr(), ws.numel() * 4, ctx.stream(), ctypes.byref(led))
    ctx.ledger.add_c(led)
    ctx.ledger.observe_level(level - 1)
    return out


def coeffs_to_slots_factorized(ctx: HeContext, plan: FactorizedStcPlan, keys: list, X) -> SlotBlocks:
    """Coefficient-encoded ciphertexts at plan.input_level (CtBlocks, or the raw [n_ct, level + 1, 2, N] tensor
    mod_raise returns) -> SlotBlocks at plan.output_level holding the coefficient pairs in the slots."""
    data = getattr(X, "data", X)
    level = getattr(X, "level", None)
    if level is None:
        if not hasattr(data, "shape") or len(data.shape) != 4:
            raise TypeError("coeffs_to_slots takes CtBlocks or a [n_ct, level + 1, 2, N] ciphertext tensor")
        level = int(data.shape[1]) - 1
    if isinstance(X, SlotBlocks):
        raise TypeError("coeffs_to_slots consumes coefficient-encoded ciphertexts, not SlotBlocks")
    if level < len(plan.maps):
        raise NeedsBootstrapError(f"the factorized CoeffToSlots needs {len(plan.maps)} levels, operand has {level}")
    if level != plan.input_level:
        raise ValueError(f"plan expects level {plan.input_level}, operand is at level {level}: lower it first")
    if len(keys) != len(plan.maps):
        raise ValueError("one key set per map")
    if plan.pre_log2:
        data = mul_pow2(ctx, data, plan.pre_log2)
    for m, k in zip(plan.maps, keys):
        data = chain_map(ctx, m, k, data, level)
        level -= 1
    return SlotBlocks(data, level=level, n_cols=getattr(X, "n_cols", 0),
                      scale=2.0 ** (plan.pre_log2 - sum(plan.shifts)), layout="coeff_pairs")


def mul_pow2(ctx: HeContext, data, e: int):
    """Chain ciphertexts [n_ct, l + 1, 2, N] times the integer 2^e, limb by limb (no level consumed)."""
    torch = _torch()
    nl = int(data.shape[1])
    q = torch.tensor(ctx.params.moduli[:nl], dtype=torch.int64, device=data.device).view(1, nl, 1, 1)
    return (((data.to(torch.int64) & 0xFFFFFFFF) << e) % q).to(torch.int32)


def slot_to_coeffs_factorized(ctx: HeContext, plan: FactorizedStcPlan, keys: list, X: SlotBlocks) -> CtBlocks:
    """SlotBlocks at plan.input_level -> CtBlocks in the App. A coefficient layout at plan.output_level (one level
    per map; a higher input is lowered first with `lower_level`)."""
    if not isinstance(X, SlotBlocks):
        raise TypeError("slot_to_coeffs consumes slot-encoded ciphertexts (SlotBlocks)")
    if X.level < len(plan.maps):
        raise NeedsBootstrapError(f"the factorized SlotToCoeffs needs {len(plan.maps)} levels, operand has {X.level}")
    if X.level != plan.input_level:
        raise ValueError(f"plan expects level {plan.input_level}, operand is at level {X.level}: lower it first")
    if X.scale and X.scale != plan.input_scale:
        raise ValueError(f"scale mismatch: plan expects input scale {plan.input_scale}, operand has {X.scale}")
    if len(keys) != len(plan.maps):
        raise ValueError("one key set per map")
    data, level = X.data, X.level
    for m, k in zip(plan.maps, keys):
        data = chain_map(ctx, m, k, data, level)
        level -= 1
    return CtBlocks(data, level=level, n_cols=X.n_cols)
