"""One Llama-2-7B decoder layer (d_model 4096, 32 heads, d_ff 11008) on 128 private tokens with the seven
projections as encrypted MLWE PCMMs on the GPU (prefill.py's projection-only split), random weights:
per-stage wall/device times and the deviation from the float layer.  GPU tool."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, native, pcmm_mlwe
from paper_2601_18511_b200.context import decode_mlwe_rows
from paper_2601_18511_b200.prefill import Cache, ToyConfig, forward_chunk

cfg = ToyConfig(d_model=4096, d_head=128, n_heads=32, d_ff=11008, n_layers=1, seed=0)
rng = np.random.default_rng(0)
s = 1.0 / np.sqrt(cfg.d_model)
d, f = cfg.d_model, cfg.d_ff
layers = [[rng.standard_normal(sh) * s for sh in [(d, d), (d, d), (d, d), (d, d), (d, f), (d, f), (f, d)]]]
# the down projection sees |h| up to ~10: keep its products inside the level-0 range (|value| < 8 at Delta 2^26)
layers[0][6] *= 0.25
x = rng.standard_normal((128, d))

P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
sk = ctx.keygen(1)
names = ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down")
t0 = time.perf_counter()
plans = {n: make_mlwe_pcmm_plan(ctx, np.ascontiguousarray(w.T)) for n, w in zip(names, layers[0])}
torch.cuda.synchronize()
print(f"plans: {time.perf_counter() - t0:.1f} s", flush=True)
times = {"encrypt": 0.0, "pcmm": 0.0, "decrypt (device)": 0.0, "decode (host)": 0.0}


class Proj:
    calls = 0

    def apply(self, ctx, sk, layer, name, a):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        X = ctx.encrypt_acts(sk, a, seed=100 + self.calls)
        ev[1].record()
        Y = pcmm_mlwe(ctx, plans[name], X)
        ev[2].record()
        ph = torch.empty((Y.n_rows, P.mlwe_degree), dtype=torch.int64, device="cuda")
        native.call("he_decrypt_mlwe", ctx.handle, sk.s.data_ptr(), Y.out_b.data_ptr(), Y.out_a.data_ptr(), Y.n_rows,
                    0, Y.n_rows, ph.data_ptr(), ctx.stream())
        ev[3].record()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = decode_mlwe_rows(P, ph.cpu().numpy(), 0, Y.n_rows)
        times["decode (host)"] += 1e3 * (time.perf_counter() - t0)
        times["encrypt"] += ev[0].elapsed_time(ev[1])
        times["pcmm"] += ev[1].elapsed_time(ev[2])
        times["decrypt (device)"] += ev[2].elapsed_time(ev[3])
        self.calls += 1
        return out


def run(proj):
    cache = Cache([np.zeros((0, d))], [np.zeros((0, d))])
    return forward_chunk(x, cache, cfg, layers, proj, ctx, sk)


t0 = time.perf_counter()
ref = run(None)
t_clear = time.perf_counter() - t0
run(Proj())                                   # warm-up
for k in times:
    times[k] = 0.0
t0 = time.perf_counter()
got = run(Proj())
t_enc = time.perf_counter() - t0
err = np.abs(got - ref).max()
print(f"layer: wall {t_enc * 1e3:.1f} ms (float layer on the host {t_clear * 1e3:.1f} ms); device ms: "
      + ", ".join(f"{k} {v:.2f}" for k, v in times.items())
      + f"; max |out - float| = {err:.2e} (|out| max {np.abs(ref).max():.1f})", flush=True)
