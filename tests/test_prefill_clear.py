"""The clear restatement of hesim's chunked prefill (prefill.py) reproduces the reference's own
outputs (golden file from hesim) -- the baseline the encrypted-projection run is compared with."""
from pathlib import Path

import numpy as np
import pytest

from paper_2601_18511_b200.prefill import ToyConfig, chunked_prefill

G = np.load(Path(__file__).parent / "golden" / "prefill_golden.npz")


@pytest.mark.parametrize("name", ["toy", "toy2"])
def test_clear_restatement_matches_hesim(name):
    d_model, d_head, n_heads, d_ff, n_layers, seed, ptok = (int(v) for v in G[name + "_cfg"])
    cfg = ToyConfig(d_model, d_head, n_heads, d_ff, n_layers, seed)
    logits, cache = chunked_prefill(G[name + "_tokens"], ptok, cfg)
    np.testing.assert_allclose(logits, G[name + "_logits"], rtol=1e-12, atol=1e-12)
    for li in range(n_layers):
        np.testing.assert_allclose(cache.k[li], G[f"{name}_k{li}"], atol=1e-12)
        np.testing.assert_allclose(cache.v[li], G[f"{name}_v{li}"], atol=1e-12)


@pytest.mark.parametrize("name", ["toy", "toy2"])
def test_clear_decode_step_matches_hesim(name):
    from paper_2601_18511_b200.prefill import decode_step

    d_model, d_head, n_heads, d_ff, n_layers, seed, ptok = (int(v) for v in G[name + "_cfg"])
    cfg = ToyConfig(d_model, d_head, n_heads, d_ff, n_layers, seed)
    _, cache = chunked_prefill(G[name + "_tokens"], ptok, cfg)
    logits, _ = decode_step(cache, G[name + "_next"], cfg)
    np.testing.assert_allclose(logits, G[name + "_decode_logits"], rtol=1e-12, atol=1e-12)
