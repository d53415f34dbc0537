"""The slot-domain PCMM in the reference's PC-attention flow (hesim pipeline.py:324-398).

hesim's pc_attention_encrypted multiplies the private, twice-sheared query block by the public key cache
(scores: make_pcmm_plan(K_pub^T / sqrt(d), shear 1) + pcmm_bsgs), runs an encrypted polynomial softmax
over the columns, and multiplies by the public value cache (make_pcmm_plan(V_pub, shear 0) +
pcmm_bsgs).  Both products here are the GPU slot-domain PCMM on real CKKS ciphertexts (slotpcmm.py);
RoPE and the softmax run on the key holder's side between them (the encrypted softmax needs ct x ct
multiplication and bootstrapping, outside this repository -- DESIGN.md §7), so this is the hybrid
client/server form of the same shear chain 2 -> 1 -> 0.
"""

from __future__ import annotations

import numpy as np

from .prefill import apply_rope
from .slotpcmm import decrypt_packed, encrypt_packed, make_slot_pcmm_plan, pcmm_slot_bsgs, slot_pcmm_keygen


def rope_columns(mat, positions):
    """pipeline.py:310-312: rotary-encode each column."""
    return apply_rope(np.asarray(mat, dtype=float).T, positions).T


def _softmax_columns(s):
    z = np.exp(s - np.max(s, axis=0, keepdims=True))
    return z / np.sum(z, axis=0, keepdims=True)


def clear_pc_attention(q, k_pub, v_pub, positions):
    """pipeline.py:315-321: private queries (columns) against the public cache."""
    qr = rope_columns(q, positions)
    s = np.asarray(k_pub, float).T @ qr / np.sqrt(q.shape[0])
    return np.asarray(v_pub, float) @ _softmax_columns(s)


def pc_attention_hybrid(ctx, sk, q, k_pub, v_pub, positions=None, seed: int | None = None) -> tuple[np.ndarray, dict]:
    """Private q (d x d, tokens as columns) against the public K/V cache blocks: two GPU slot-domain
    PCMMs on ciphertexts, RoPE and the column softmax on the key holder's side.  Returns (out, report).
    seed None: fresh nonces for every key and encryption (secure contexts); a seed: seed + 1 .. seed + 4."""
    q = np.asarray(q, float)
    d = q.shape[0]
    k_pub, v_pub = np.asarray(k_pub, float), np.asarray(v_pub, float)
    if q.shape != (d, d) or k_pub.shape != (d, d) or v_pub.shape != (d, d):
        raise ValueError("q and the public cache blocks must be d x d")
    if positions is None:
        positions = k_pub.shape[1] + np.arange(d)
    nonce = (lambda i: None) if seed is None else (lambda i: seed + i)
    before = ctx.ledger.snapshot()
    # scores: shear chain 2 -> 1 (client encrypts the rotary-encoded queries twice-sheared)
    s_plan = make_slot_pcmm_plan(ctx, k_pub.T / np.sqrt(d), shear_power=1)
    s_keys = slot_pcmm_keygen(ctx, sk, s_plan, nonce(1))
    q_ct = encrypt_packed(ctx, sk, rope_columns(q, positions), 2, seed=nonce(2))
    s_ct = pcmm_slot_bsgs(ctx, s_plan, s_keys, q_ct)
    # key holder: decrypt, undo the remaining shear, softmax over columns, re-encrypt once-sheared
    scores = decrypt_packed(ctx, sk, s_ct)
    i, j = np.indices((d, d))
    unsheared = np.empty_like(scores)
    unsheared[(i + j) % d, j] = scores        # s_ct holds col_shear(S, 1)[i, j] = S[(i + j) % d, j]
    probs = _softmax_columns(unsheared)
    p_ct = encrypt_packed(ctx, sk, probs, 1, seed=nonce(3))
    # values: shear chain 1 -> 0
    v_plan = make_slot_pcmm_plan(ctx, v_pub, shear_power=0)
    v_keys = slot_pcmm_keygen(ctx, sk, v_plan, nonce(4))
    out = decrypt_packed(ctx, sk, pcmm_slot_bsgs(ctx, v_plan, v_keys, p_ct))
    return out, {"ledger": ctx.ledger.diff(before), "scores": unsheared}
