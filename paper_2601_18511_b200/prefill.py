"""Encrypted projections in the reference's prefill: where the MLWE PCMM plugs in.

hesim's chunked prefill (pipeline.py:212-237) runs a public chunk in the clear and then the private
chunk through the same chunk engine (_forward_chunk, pipeline.py:177-192), whose seven projections
xn @ wq | wk | wv, attn @ wo, xn2 @ w_gate | w_up and h @ w_down are float GEMMs.  Here the private
chunk's projections run on ciphertexts: the chunk's rows are coefficient-encrypted at level 1 in
the App. A layout, multiplied by the plan of w^T with the GPU MLWE PCMM (pcmm_mlwe: one level, one
rescale) and decrypted by the key holder, who computes the non-linear parts (RMSNorm, RoPE,
attention, SiLU) in the clear.  This is the client/server split of a projection-only deployment;
the paper's full pipeline also keeps the non-linear parts encrypted (bootstrapping),
which is outside this repository.

The clear parts restate the reference's formulas (cited per function) so the result can be
compared with hesim's own chunked_prefill on the same config (tests/golden/prefill_golden.npz).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .context import HeContext, SecretKey
from .pcmm import make_mlwe_pcmm_plan, pcmm_mlwe


@dataclass(frozen=True)
class ToyConfig:
    """hesim ToyModelConfig (pipeline.py:47-61): shapes and seed of the toy decoder."""
    d_model: int = 32
    d_head: int = 16
    n_heads: int = 2
    d_ff: int = 64
    n_layers: int = 1
    seed: int = 0


def make_weights(cfg: ToyConfig) -> list:
    """pipeline.py:82-95: per layer (wq, wk, wv, wo, w_gate, w_up, w_down) at magnitude 1/sqrt(d_model),
    then w_out -- drawn in the reference's order from default_rng(seed)."""
    rng = np.random.default_rng(cfg.seed)
    s = 1.0 / np.sqrt(cfg.d_model)
    d, f = cfg.d_model, cfg.d_ff
    shapes = [(d, d), (d, d), (d, d), (d, d), (d, f), (d, f), (f, d)]
    layers = [[rng.standard_normal(sh) * s for sh in shapes] for _ in range(cfg.n_layers)]
    return layers, rng.standard_normal((d, d)) * s


def rms_norm(x, eps: float = 1e-8):            # pipeline.py:103-105
    x = np.asarray(x, dtype=float)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)


def apply_rope(x, positions):                  # pipeline.py:108-131 (half-split pairs, theta = pos 10^(-4j/d))
    x = np.asarray(x, dtype=float)
    d = x.shape[-1]
    th = np.asarray(positions, float)[:, None] * (10.0 ** (-4.0 * np.arange(d // 2) / d))[None, :]
    th = th.reshape(th.shape[0], *([1] * (x.ndim - 2)), d // 2)
    c, s = np.cos(th), np.sin(th)
    lo, hi = x[..., : d // 2], x[..., d // 2:]
    return np.concatenate([lo * c - hi * s, hi * c + lo * s], axis=-1)


def _softmax(s):                               # softmax.py:53-57
    z = np.exp(s - np.max(s, axis=-1, keepdims=True))
    return z / np.sum(z, axis=-1, keepdims=True)


def _silu(x):                                  # polyapprox.py:79-80
    return x / (1.0 + np.exp(-x))


def _attend(q, k_all, v_all, start, cfg):       # pipeline.py:160-174, causal over cache + chunk keys
    m, t = q.shape[0], k_all.shape[0]
    qh = q.reshape(m, cfg.n_heads, cfg.d_head)
    kh = k_all.reshape(t, cfg.n_heads, cfg.d_head)
    vh = v_all.reshape(t, cfg.n_heads, cfg.d_head)
    mask = np.arange(t)[None, :] > (start + np.arange(m))[:, None]
    out = []
    for h in range(cfg.n_heads):
        s = np.where(mask, -np.inf, qh[:, h] @ kh[:, h].T / np.sqrt(cfg.d_head))
        out.append(_softmax(s) @ vh[:, h])
    return np.stack(out, axis=1).reshape(m, cfg.d_model)


@dataclass
class Cache:
    k: list = field(default_factory=list)
    v: list = field(default_factory=list)


@dataclass
class EncryptedProjections:
    """The server side: one MLWE PCMM plan per projection (w^T, n_out x n_in) per layer."""
    plans: list
    seed: int = 1000
    calls: int = 0

    def apply(self, ctx: HeContext, sk: SecretKey, layer: int, name: str, x: np.ndarray) -> np.ndarray:
        """x @ w for the chunk rows x (<= tokens rows): encrypt (client) -> PCMM (server) -> decrypt."""
        plan = self.plans[layer][name]
        m = x.shape[0]
        block = np.zeros((ctx.params.tokens, plan.n_in))
        block[:m] = x
        self.calls += 1
        X = ctx.encrypt_acts(sk, block, seed=self.seed + self.calls)
        return ctx.decrypt_pcmm(sk, pcmm_mlwe(ctx, plan, X))[:m]


NAMES = ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")


def make_projection_plans(ctx: HeContext, layers, algo: str = "spectral") -> EncryptedProjections:
    return EncryptedProjections([{n: make_mlwe_pcmm_plan(ctx, np.ascontiguousarray(w.T), algo=algo)
                                  for n, w in zip(NAMES, lw)} for lw in layers])


def forward_chunk(x, cache: Cache, cfg: ToyConfig, layers, proj=None, ctx=None, sk=None):
    """pipeline.py:177-192; with ``proj`` the seven projections run as encrypted MLWE PCMMs."""
    start = cache.k[0].shape[0]
    pos = start + np.arange(x.shape[0])

    def mm(li, name, a):
        if proj is None:
            return a @ layers[li][NAMES.index(name)]
        return proj.apply(ctx, sk, li, name, a)

    for li in range(cfg.n_layers):
        xn = rms_norm(x)
        q = apply_rope(mm(li, "wq", xn).reshape(-1, cfg.n_heads, cfg.d_head), pos).reshape(x.shape[0], -1)
        k = apply_rope(mm(li, "wk", xn).reshape(-1, cfg.n_heads, cfg.d_head), pos).reshape(x.shape[0], -1)
        v = mm(li, "wv", xn)
        cache.k[li] = np.vstack([cache.k[li], k])
        cache.v[li] = np.vstack([cache.v[li], v])
        x = x + mm(li, "wo", _attend(q, cache.k[li], cache.v[li], start, cfg))
        xn2 = rms_norm(x)
        x = x + mm(li, "w_down", _silu(mm(li, "w_gate", xn2)) * mm(li, "w_up", xn2))
    return x


def chunked_prefill(tokens, ptok: int, cfg: ToyConfig, ctx: HeContext | None = None, sk: SecretKey | None = None,
                    proj: EncryptedProjections | None = None):
    """pipeline.py:212-237: public rows [0, ptok) in the clear, then the private rows -- with ``proj``,
    through encrypted projections.  Returns (logits of the last token, cache)."""
    tokens = np.atleast_2d(np.asarray(tokens, dtype=float))
    if not 0 <= ptok < tokens.shape[0]:
        raise ValueError("need 0 <= ptok < ntok")
    if proj is not None and tokens.shape[0] - ptok > ctx.params.tokens:
        raise ValueError(f"the private chunk has {tokens.shape[0] - ptok} rows; one activation block holds "
                         f"{ctx.params.tokens}")
    layers, w_out = make_weights(cfg)
    cache = Cache([np.zeros((0, cfg.d_model)) for _ in range(cfg.n_layers)],
                  [np.zeros((0, cfg.d_model)) for _ in range(cfg.n_layers)])
    if ptok:
        forward_chunk(tokens[:ptok], cache, cfg, layers)
    x = forward_chunk(tokens[ptok:], cache, cfg, layers, proj, ctx, sk)
    return rms_norm(x[-1]) @ w_out, cache


# ---------------------------------------------------------------- generation: the Rhombus PCMv plug-in point
@dataclass
class EncryptedVectorProjections:
    """Generation-stage projections of one token: each x @ w is an encrypted
    vector -> Rhombus PCMv (plan of w^T) -> decryption under the output key s'(X^rho)."""
    plans: list
    keys: object
    seed: int = 2000
    calls: int = 0

    def apply(self, ctx: HeContext, sk: SecretKey, layer: int, name: str, x: np.ndarray) -> np.ndarray:
        from .rhombus import decrypt_vector, encrypt_vector, pcmv_rhombus

        rows = []
        for row in np.atleast_2d(x):
            self.calls += 1
            ct = encrypt_vector(ctx, sk, row, seed=self.seed + self.calls)
            rows.append(decrypt_vector(ctx, self.keys.s_up_ntt, pcmv_rhombus(ctx, self.plans[layer][name], self.keys, ct)))
        return np.stack(rows)


def make_vector_projection_plans(ctx: HeContext, sk: SecretKey, layers, seed: int = 77) -> EncryptedVectorProjections:
    from .rhombus import make_rhombus_plan, rhombus_keygen

    keys = rhombus_keygen(ctx, sk, seed)
    return EncryptedVectorProjections([{n: make_rhombus_plan(ctx, np.ascontiguousarray(w.T))
                                        for n, w in zip(NAMES, lw)} for lw in layers], keys)


def decode_step(cache: Cache, token, cfg: ToyConfig, ctx: HeContext | None = None, sk: SecretKey | None = None,
                proj=None):
    """pipeline.py:240-247: one autoregressive row against the cache; with ``proj`` (e.g. the Rhombus
    PCMv projections) the seven projections run on ciphertexts.  Returns (logits, cache)."""
    layers, w_out = make_weights(cfg)
    x = forward_chunk(np.atleast_2d(np.asarray(token, dtype=float)), cache, cfg, layers, proj, ctx, sk)
    return rms_norm(x[-1]) @ w_out, cache
