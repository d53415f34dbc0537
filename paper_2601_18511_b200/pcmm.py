"""MLWE-format PCMM (BCHPS24 Alg. 2 as used at PAPER.md:54-55,134) -- the drop-in entry points.

Mirrors the reference's operator API for a plaintext x ciphertext product
(pkg/src/hesim/matmul.py:77-181): a weight-side *plan* built once, and a kernel
call ``(ctx, plan, operand) -> result`` that validates before any compute, raises
the reference's exceptions, never mutates its inputs, consumes exactly one level
and records the work in ``ctx.ledger`` like one fused ``pc_linear`` per output
block (slotsim.py:330-370):

    make_pcmm_plan(ctx, weights, shear_power, split, on_the_fly)   (matmul.py:77-100)
        -> make_mlwe_pcmm_plan(ctx, weights, d_w=None)
    pcmm_depth1 / pcmm_bsgs(ctx, plan, B)                         (matmul.py:152-176)
        -> pcmm_mlwe(ctx, plan, X)
    clear_pcmm(A, B, shear_power)                                 (matmul.py:179-181)
        -> clear_pcmm(W, acts)

Work split (all on the device, through the C ABI in include/he_b200.h):
  plan:  W -> W~ = round(q1 W), k x k blocks conjugated by sigma, balanced int8 digit planes;
         spectral plans (the default) also hold G^ = NTT_L(weight segments) as int8 digit planes (K7 S1)
  run:   spectral -- K3 digits of the b' columns, K7 S2 window NTTs, K1 on the b' columns, K7 S3
         per-frequency tcgen05 modular GEMMs, K7 S4 inverse NTT + rescale + a' store;
         direct   -- K3 RLWE -> MLWE digit decomposition, then K1 tcgen05 modular GEMM over every
         column with the digit recombination, reduction mod q_i, rescale and b' compose fused in
         its epilogue.  Both produce the same words.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import native
from .context import CtBlocks, HeContext, MlweBlocks, _torch, require_level
from .params import signed_digits


@dataclass
class MlwePcmmPlan:
    """Weight side of the MLWE PCMM.  Immutable after creation and
    safe to share between forked contexts; the digit planes stay on the device."""

    n_out: int
    n_in: int
    d_w: int
    max_abs: int
    digits: object          # torch int8 [d_w, n_out, n_in]
    layout: str = "app_a_coeff"
    algo: str = "direct"    # "spectral": a' columns by blockwise NTT correlation (K7), b' on K1
    spec_weights: object = None   # torch int8, the spectral weights G^ (algo == "spectral")
    _handle: object = field(default=None, repr=False)
    _workspace: object = field(default=None, repr=False)
    _stream_bufs: object = field(default=None, repr=False)
    _copy_stream: object = field(default=None, repr=False)
    _ctx_keepalive: object = field(default=None, repr=False)   # the creating context's device state

    @property
    def shape(self) -> tuple[int, int]:
        return self.n_out, self.n_in

    def workspace_bytes(self) -> int:
        n = ctypes.c_uint64()
        native.call("he_pcmm_workspace_bytes", self._handle, ctypes.byref(n))
        return int(n.value)

    def workspace(self, device):
        """Scratch for one call: a per-device buffer shared by every plan (grown to the largest need),
        so the projections of a layer do not each pin their own multi-GB workspace.  Calls that share
        it must be ordered on one stream (the C ABI itself takes any caller-provided workspace)."""
        torch = _torch()
        need = self.workspace_bytes()
        key = torch.device(device)
        ws = _SHARED_WS.get(key)
        if ws is None or ws.numel() < need:
            _SHARED_WS.pop(key, None)
            ws = torch.empty(need, dtype=torch.int8, device=key)
            _SHARED_WS[key] = ws
        self._workspace = ws
        return ws

    def spectral_info(self) -> dict:
        """Spectral plans: transform length L, outputs per block, blocks, padded blocks."""
        info = (ctypes.c_uint32 * 4)()
        native.call("he_pcmm_spectral_info", self._handle, info)
        return {"L": info[0], "block_outputs": info[1], "blocks": info[2], "blocks_padded": info[3]}

    STAGES = ("decompose", "spectral_data", "modgemm", "spectral_gemm_q0", "spectral_gemm_q1", "spectral_inverse")

    def profile(self, enable: bool = True) -> None:
        """Record per-stage CUDA events on every launch of this plan (he_pcmm_profile)."""
        native.call("he_pcmm_profile", self._handle, 1 if enable else 0)

    def profile_read(self) -> dict:
        """{stage: (summed device ms, launches)} since profile() / the last read (synchronizes)."""
        n = len(self.STAGES)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_uint32 * n)()
        native.call("he_pcmm_profile_read", self._handle, ms, cnt, n)
        return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(self.STAGES) if cnt[i]}

    def __del__(self):
        try:
            if self._handle:
                native.lib().he_pcmm_plan_destroy(self._handle)
        except Exception:
            pass


ALGOS = ("spectral", "direct")
_SHARED_WS: dict = {}   # torch.device -> int8 workspace tensor (MlwePcmmPlan.workspace)


def make_mlwe_pcmm_plan(ctx: HeContext, weights, d_w: int | None = None, algo: str = "spectral") -> MlwePcmmPlan:
    """Encode the float weights W (n_out x n_in) for the MLWE PCMM.

    W~ = round_half_even(q1 * W) (Delta_w = q1 so the op keeps the input scale),
    each k x k block conjugated by sigma (PAPER.md:672 / bitrev.py:57-70 in component
    order), split into ``d_w`` balanced int8 digit planes; ``d_w`` defaults to the
    fewest digits that hold max|W~|.

    ``algo`` picks how the a' columns are computed -- the outputs are the same words:
      "spectral" (default): blockwise length-2k cyclic NTT correlations (K7: the a-part
                  GEMM's columns are twisted shifts of one polynomial),
                  per-frequency modular GEMMs on tcgen05; b' columns on K1;
      "direct":   K1 over all d (1 + k) GEMM columns (BCHPS24 Alg. 2 as a plain GEMM).
    """
    if algo not in ALGOS:
        raise ValueError(f"algo must be one of {ALGOS}, got {algo!r}")
    torch = _torch()
    p = ctx.params
    w = torch.as_tensor(weights, dtype=torch.float64, device=ctx.device)
    if w.ndim != 2:
        raise ValueError("weights must be a matrix")
    n_out, n_in = (int(s) for s in w.shape)
    k = p.mlwe_rank
    if n_out % k or n_in % k:
        raise ValueError(f"dim mismatch: weight dims ({n_out}, {n_in}) must be multiples of k = {k}")
    if not bool(torch.isfinite(w).all()):
        raise ValueError("weights must be finite")
    w = w.contiguous()
    mx = ctypes.c_uint64()
    native.call("he_pcmm_weight_maxabs", ctx.handle, w.data_ptr(), n_out, n_in, ctypes.byref(mx), ctx.stream())
    max_abs = int(mx.value)
    need = signed_digits(max_abs)
    if max_abs >= 1 << 31 or need > 4:
        raise ValueError(f"encoded weights too large (max |W~| = {max_abs} >= 2^31); rescale W")
    if d_w is None:
        d_w = need
    if not need <= d_w <= 4:
        raise ValueError(f"d_w = {d_w} cannot hold max |W~| = {max_abs} (needs >= {need})")
    digits = torch.empty((d_w, n_out, n_in), dtype=torch.int8, device=ctx.device)
    native.call("he_pcmm_encode_weights", ctx.handle, w.data_ptr(), n_out, n_in, d_w, digits.data_ptr(),
                ctx.stream())
    return _plan_from_digits(ctx, digits, n_out, n_in, d_w, max_abs, algo)


def _plan_from_digits(ctx: HeContext, digits, n_out: int, n_in: int, d_w: int, max_abs: int,
                      algo: str) -> MlwePcmmPlan:
    torch = _torch()
    h = ctypes.c_void_p()
    native.call("he_pcmm_plan_create", ctx.handle, digits.data_ptr(), n_out, n_in, d_w, ctypes.byref(h))
    plan = MlwePcmmPlan(n_out, n_in, d_w, max_abs, digits, algo=algo, _handle=h, _ctx_keepalive=ctx._dev)
    if algo == "spectral":
        nb = ctypes.c_uint64()
        native.call("he_pcmm_spectral_weight_bytes", h, ctypes.byref(nb))
        plan.spec_weights = torch.empty(int(nb.value), dtype=torch.int8, device=ctx.device)
        native.call("he_pcmm_spectral_prepare", h, plan.spec_weights.data_ptr(), ctx.stream())
    return plan


# ---------------------------------------------------------------- on-disk plan format
PLAN_FORMAT = "he-b200/mlwe-pcmm-plan/1"


def _param_key(params) -> dict:
    """The parameters a plan's digits depend on (ring, moduli, weight scale = q1)."""
    return {"N": int(params.N), "mlwe_degree": int(params.mlwe_degree), "mlwe_rank": int(params.mlwe_rank),
            "moduli": [int(q) for q in params.moduli], "delta_w": int(params.delta_w)}


def save_mlwe_pcmm_plan(ctx: HeContext, plan: MlwePcmmPlan, path) -> None:
    """Write the plan's pre-shuffled balanced int8 digit planes [d_w, n_out, n_in] (the expensive,
    weight-only part) plus a JSON header to one uncompressed .npz.  The spectral weights are not
    stored: he_pcmm_spectral_prepare rebuilds them from the digits on the device at load."""
    import json

    meta = {"format": PLAN_FORMAT, "params": _param_key(ctx.params), "n_out": plan.n_out, "n_in": plan.n_in,
            "d_w": plan.d_w, "max_abs": plan.max_abs, "layout": plan.layout, "algo": plan.algo}
    np.savez(path, meta=np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8),
             digits=plan.digits.cpu().numpy())


def load_mlwe_pcmm_plan(ctx: HeContext, path, algo: str | None = None) -> MlwePcmmPlan:
    """Rebuild a plan from save_mlwe_pcmm_plan's file on ctx's device (algo: the stored one unless
    given).  Raises ValueError if the file was made for other parameters or another format."""
    import json

    torch = _torch()
    with np.load(path) as z:
        meta = json.loads(bytes(z["meta"]).decode())
        if meta.get("format") != PLAN_FORMAT:
            raise ValueError(f"not an MLWE PCMM plan file ({meta.get('format')!r})")
        if meta["params"] != _param_key(ctx.params):
            raise ValueError(f"plan was encoded for {meta['params']}, context has {_param_key(ctx.params)}")
        digits = z["digits"]
    n_out, n_in, d_w = int(meta["n_out"]), int(meta["n_in"]), int(meta["d_w"])
    if digits.shape != (d_w, n_out, n_in) or digits.dtype != np.int8:
        raise ValueError(f"digit planes have shape {digits.shape} / {digits.dtype}")
    algo = algo or meta["algo"]
    if algo not in ALGOS:
        raise ValueError(f"algo must be one of {ALGOS}, got {algo!r}")
    dev = torch.from_numpy(np.ascontiguousarray(digits)).to(ctx.device)
    return _plan_from_digits(ctx, dev, n_out, n_in, d_w, int(meta["max_abs"]), algo)


def save_plan_bundle(ctx: HeContext, plans: dict, directory) -> None:
    """A model's projections (e.g. 32 layers x {q, k, v, o, up, gate, down}): one plan file per
    name plus index.json."""
    import json
    from pathlib import Path

    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    index = {"format": PLAN_FORMAT, "plans": {}}
    for name, plan in plans.items():
        fn = f"{name}.npz"
        save_mlwe_pcmm_plan(ctx, plan, d / fn)
        index["plans"][name] = {"file": fn, "shape": [plan.n_out, plan.n_in], "d_w": plan.d_w}
    (d / "index.json").write_text(json.dumps(index, indent=1))


def load_plan_bundle(ctx: HeContext, directory, algo: str | None = None, names=None) -> dict:
    import json
    from pathlib import Path

    d = Path(directory)
    index = json.loads((d / "index.json").read_text())
    if index.get("format") != PLAN_FORMAT:
        raise ValueError(f"not a plan bundle ({index.get('format')!r})")
    return {n: load_mlwe_pcmm_plan(ctx, d / e["file"], algo) for n, e in index["plans"].items()
            if names is None or n in names}


def _check_operand(ctx: HeContext, plan: MlwePcmmPlan, X) -> None:
    """Error contract of matmul.py:139-149, raised before any compute."""
    if not isinstance(X, CtBlocks):
        raise TypeError("pcmm consumes a ciphertext operand")
    if plan._ctx_keepalive is not None and plan._ctx_keepalive is not ctx._dev:
        raise ValueError("plan was built under another HeContext (its device tables); rebuild or load it here")
    if X.n_cols != plan.n_in:
        raise ValueError(f"dim mismatch: plan {plan.n_in}, operand {X.n_cols}")
    if X.layout != plan.layout:
        raise ValueError(f"layout mismatch: plan expects {plan.layout}, got {X.layout}")
    require_level(X.level)
    if X.level != 1:
        raise ValueError(f"the MLWE PCMM runs at level 1, operand is at level {X.level}; switch levels first")
    shape = tuple(int(s) for s in X.data.shape)
    if shape != (plan.n_in // ctx.params.mlwe_rank, 2, 2, ctx.params.N):
        raise ValueError(f"ciphertext batch has shape {shape}")


def _note_read(X, stream=None) -> None:
    """Mark that every access to X.data so far is queued on `stream` (the current one by default):
    pcmm_mlwe_to_host's input upload, on its own stream, waits for this event before overwriting
    X.data (and for the whole current stream when X carries none)."""
    torch = _torch()
    ev = torch.cuda.Event()
    ev.record(stream)
    X._read_done = ev


def pcmm_mlwe(ctx: HeContext, plan: MlwePcmmPlan, X: CtBlocks, out: MlweBlocks | None = None,
              gemm_events=None) -> MlweBlocks:
    """Level-1 RLWE block batch (encrypting A, (d/2) x n_in) -> level-0 MLWE blocks
    encrypting A @ W^T ((d/2) x n_out).  Exactly one level, one rescale per output block,
    zero ciphertext rotations.  ``gemm_events`` (two torch.cuda.Event) bracket the output
    stage (he_pcmm_gemm: K1, plus S3/S4 for spectral plans) on the current stream."""
    torch = _torch()
    _check_operand(ctx, plan, X)
    p = ctx.params
    if out is None:
        out_b = torch.empty((plan.n_out // p.mlwe_rank, p.N), dtype=torch.int32, device=ctx.device)
        out_a = torch.empty((plan.n_out, p.N), dtype=torch.int32, device=ctx.device)
        out = MlweBlocks(out_b, out_a, level=X.level - 1, n_rows=plan.n_out)
    ws = plan.workspace(ctx.device)
    led = native.HeLedgerC()
    st = ctx.stream()
    if gemm_events is None:
        native.call("he_pcmm_run", plan._handle, X.data.data_ptr(), X.level, out.out_b.data_ptr(),
                    out.out_a.data_ptr(), ws.data_ptr(), ws.numel(), st, ctypes.byref(led))
    else:  # the same two launches as he_pcmm_run, with events around K1
        native.call("he_pcmm_decompose", plan._handle, X.data.data_ptr(), ws.data_ptr(), ws.numel(), st)
        gemm_events[0].record()
        native.call("he_pcmm_gemm", plan._handle, ws.data_ptr(), out.out_b.data_ptr(), out.out_a.data_ptr(), st)
        gemm_events[1].record()
        k = ctx.params.mlwe_rank
        led.pc_mults = (plan.n_out // k) * (plan.n_in // k)
        led.rescales = plan.n_out // k
    _note_read(X)
    ctx.ledger.add_c(led)
    ctx.ledger.observe_level(X.level - 1)
    out.level = X.level - 1
    out.n_rows = plan.n_out
    return out


def pcmm_mlwe_into_peers(ctx: HeContext, plan: MlwePcmmPlan, X: CtBlocks, out_b_ptrs, out_a_ptrs,
                         dst_row0: int) -> None:
    """This rank's rows of the op with the output all-gather fused into the output stage: every
    word is stored into each pointer pair of ``out_b_ptrs`` / ``out_a_ptrs`` -- the FULL output
    buffers of all ranks (peer memory over NVLink, e.g. symmetric memory) -- at rows
    ``dst_row0 + y`` (he_pcmm_gemm_rows_peers).  Same ledger effect as pcmm_mlwe."""
    _check_operand(ctx, plan, X)
    n = len(out_a_ptrs)
    if n != len(out_b_ptrs) or not 1 <= n <= 8:
        raise ValueError("need 1..8 peer output pointer pairs")
    ws = plan.workspace(ctx.device)
    st = ctx.stream()
    native.call("he_pcmm_decompose", plan._handle, X.data.data_ptr(), ws.data_ptr(), ws.numel(), st)
    pb = (ctypes.c_void_p * n)(*[int(v) for v in out_b_ptrs])
    pa = (ctypes.c_void_p * n)(*[int(v) for v in out_a_ptrs])
    native.call("he_pcmm_gemm_rows_peers", plan._handle, ws.data_ptr(), 0, plan.n_out, pb, pa, n, dst_row0, st)
    _note_read(X)
    k = ctx.params.mlwe_rank
    ctx.ledger.pc_mults += (plan.n_out // k) * (plan.n_in // k)
    ctx.ledger.rescales += plan.n_out // k
    ctx.ledger.observe_level(X.level - 1)


def pcmm_mlwe_to_host(ctx: HeContext, plan: MlwePcmmPlan, X: CtBlocks, out_b_host, out_a_host,
                      x_host=None, chunk_rows: int = 512) -> MlweBlocks:
    """The same op as ``pcmm_mlwe`` with the level-0 output streamed into (pinned) host
    buffers ``out_b_host`` [n_out/k, N] and ``out_a_host`` [n_out, N]: the output stage runs
    over row chunks into two alternating device slices while a second stream copies the
    previous chunk to the host, so the 1 GB device->host transfer overlaps the compute.  ``x_host``
    (pinned, X.data's shape) is first copied into ``X.data`` on the current stream."""
    torch = _torch()
    _check_operand(ctx, plan, X)
    p = ctx.params
    k, N = p.mlwe_rank, p.N
    if chunk_rows % 256 or chunk_rows % k or chunk_rows <= 0:
        raise ValueError("chunk_rows must be a positive multiple of 256 and of k")
    if tuple(out_a_host.shape) != (plan.n_out, N) or tuple(out_b_host.shape) != (plan.n_out // k, N):
        raise ValueError("host output buffers have the wrong shape")
    dev = ctx.device
    st = torch.cuda.current_stream(dev)
    if x_host is not None and os.environ.get("HE_E2E_SERIAL_H2D"):   # measurement knob: the unoverlapped order
        X.data.copy_(x_host, non_blocking=True)
        x_host = None
    if x_host is not None:
        # the input goes up on its own stream: it only waits until the last queued access to X.data
        # (e.g. the previous call's decompose, recorded on X itself, whichever plan ran it) -- so
        # back-to-back calls overlap it with the previous call's device->host tail (the two directions
        # use separate copy engines); an X with no recorded access waits for the whole current stream
        if getattr(plan, "_h2d_stream", None) is None:
            plan._h2d_stream = torch.cuda.Stream(dev)
        hs = plan._h2d_stream
        last = getattr(X, "_read_done", None)
        if last is not None:
            hs.wait_event(last)
        else:
            hs.wait_stream(st)
        with torch.cuda.stream(hs):
            X.data.copy_(x_host, non_blocking=True)
        up = torch.cuda.Event()
        up.record(hs)
        st.wait_event(up)
    ws = plan.workspace(dev)
    if getattr(plan, "_stream_bufs", None) is None or plan._stream_bufs[0][1].shape[0] != chunk_rows:
        plan._stream_bufs = [(torch.empty((chunk_rows // k, N), dtype=torch.int32, device=dev),
                              torch.empty((chunk_rows, N), dtype=torch.int32, device=dev)) for _ in range(2)]
        plan._copy_stream = torch.cuda.Stream(dev)
    cs = plan._copy_stream
    native.call("he_pcmm_decompose", plan._handle, X.data.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream)
    _note_read(X, st)
    copied = [None, None]
    # a short first chunk starts the device->host stream sooner (the copies, not the compute, set the pace)
    first = min(256, chunk_rows) if plan.n_out > chunk_rows else chunk_rows
    starts = [0] + list(range(first, plan.n_out, chunk_rows))
    for c, row0 in enumerate(starts):
        rows = min(first if c == 0 else chunk_rows, plan.n_out - row0)
        slot = c % 2
        if copied[slot] is not None:
            st.wait_event(copied[slot])               # the slot's previous chunk has left the device
        bb, ba = plan._stream_bufs[slot]
        native.call("he_pcmm_gemm_rows", plan._handle, ws.data_ptr(), row0, rows, bb.data_ptr(), ba.data_ptr(),
                    st.cuda_stream)
        done = torch.cuda.Event()
        done.record(st)
        cs.wait_event(done)
        with torch.cuda.stream(cs):
            out_a_host[row0:row0 + rows].copy_(ba[:rows], non_blocking=True)
            out_b_host[row0 // k:(row0 + rows) // k].copy_(bb[:rows // k], non_blocking=True)
        copied[slot] = torch.cuda.Event()
        copied[slot].record(cs)
    for ev in copied:
        if ev is not None:
            st.wait_event(ev)
    ctx.ledger.pc_mults += (plan.n_out // k) * (plan.n_in // k)
    ctx.ledger.rescales += plan.n_out // k
    ctx.ledger.observe_level(X.level - 1)
    return MlweBlocks(out_b_host, out_a_host, level=X.level - 1, n_rows=plan.n_out)


def spectral_gemm_ops(params, n_out: int, n_in: int, limb: int, L: int, blocks: int) -> int:
    """Algorithmic int8 tensor-core ops of one K7 S3 launch (limb ``limb``): per frequency f < L a
    (n_out x R) x (R x blocks) product, R = n_in / k, every digit of G^ meeting every digit of A^."""
    D = params.ct_digits(limb)
    return 2 * L * n_out * (n_in // params.mlwe_rank) * blocks * D * D


def spectral_inverse_bytes(params, n_out: int, L: int, blocks: int) -> int:
    """Algorithmic HBM bytes of one K7 S4 launch: read C^ of both limbs (L x n_out x blocks u32
    each), write the a' words (n_out x N u32)."""
    return 2 * L * n_out * blocks * 4 + n_out * params.N * 4


def pcmm_ops(params, n_out: int, n_in: int, d_w: int) -> int:
    """Algorithmic int8 tensor-core ops of K1 per launch: 2 * n_out * n_in * width * d_w *
    (D_0 + D_1) (every weight digit meets every ciphertext digit of both limbs once)."""
    return 2 * n_out * n_in * params.width * d_w * (params.ct_digits(0) + params.ct_digits(1))


def word_ops(params, n_out: int, n_in: int, limbs: int = 2) -> int:
    """Word-level modular multiply-adds x 2: 2 * n_out * n_in * width * limbs."""
    return 2 * n_out * n_in * params.width * limbs


def clear_pcmm(weights, acts) -> np.ndarray:
    """Cleartext oracle of what ``pcmm_mlwe`` decrypts to: acts @ W^T, i.e.
    (W @ M)^T with M = acts^T (hesim.clear_pcmm(W, M, 0), matmul.py:179-181)."""
    return np.asarray(acts, float) @ np.asarray(weights, float).T
