"""Golden chunked-prefill outputs from the reference (hesim pipeline.chunked_prefill, float64) for the
encrypted-projection prefill test (tests/test_gpu_prefill.py) and its clear restatement
(tests/test_prefill_clear.py).  Run in the build container: python tests/golden/make_prefill_golden.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hesim.pipeline import PrefillSplit, ToyModelConfig, chunked_prefill, decode_step, demo_tokens  # noqa: E402

out = {}
for name, cfg, ntok, ptok in (("toy", ToyModelConfig(d_model=32, d_head=16, n_heads=2, d_ff=64, n_layers=1, seed=0),
                               24, 12),
                              ("toy2", ToyModelConfig(d_model=32, d_head=32, n_heads=1, d_ff=48, n_layers=2, seed=3),
                               20, 6)):
    tok = demo_tokens(ntok, cfg.d_model, seed=7)
    logits, cache = chunked_prefill(tok, PrefillSplit(ntok, ptok, ntok - ptok), cfg)
    out[name + "_tokens"] = tok
    out[name + "_cfg"] = np.array([cfg.d_model, cfg.d_head, cfg.n_heads, cfg.d_ff, cfg.n_layers, cfg.seed, ptok])
    out[name + "_logits"] = logits
    for li in range(cfg.n_layers):
        out[f"{name}_k{li}"] = cache.k[li]
        out[f"{name}_v{li}"] = cache.v[li]
    nxt = demo_tokens(1, cfg.d_model, seed=11)[0]
    out[name + "_next"] = nxt
    out[name + "_decode_logits"] = decode_step(cache, nxt, cfg)[0]
np.savez(Path(__file__).with_name("prefill_golden.npz"), **out)
print("wrote", sorted(out))
