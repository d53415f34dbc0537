"""he_decrypt_mlwe device time for 4096 rows and the host decode time.  GPU tool."""
import math
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, native, pcmm_mlwe
from paper_2601_18511_b200.context import decode_mlwe_rows

P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
sk = ctx.keygen(1)
g = torch.Generator(device="cuda").manual_seed(1)
W = (torch.rand((4096, 4096), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) / 64
A = torch.rand((P.tokens, 4096), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
X = ctx.encrypt_acts(sk, A, seed=2)
Y = pcmm_mlwe(ctx, make_mlwe_pcmm_plan(ctx, W), X)
ph = torch.empty((4096, P.mlwe_degree), dtype=torch.int64, device="cuda")
for _ in range(2):
    native.call("he_decrypt_mlwe", ctx.handle, sk.s.data_ptr(), Y.out_b.data_ptr(), Y.out_a.data_ptr(), 4096, 0, 4096,
                ph.data_ptr(), ctx.stream())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
native.call("he_decrypt_mlwe", ctx.handle, sk.s.data_ptr(), Y.out_b.data_ptr(), Y.out_a.data_ptr(), 4096, 0, 4096,
            ph.data_ptr(), ctx.stream())
e1.record()
torch.cuda.synchronize()
t0 = time.perf_counter()
h = ph.cpu().numpy()
t1 = time.perf_counter()
decode_mlwe_rows(P, h, 0, 4096)
t2 = time.perf_counter()
print(f"{'direct' if os.environ.get('HE_DECRYPT_MLWE_DIRECT') else 'ntt'}: device {e0.elapsed_time(e1):.2f} ms, "
      f"D2H {1e3 * (t1 - t0):.2f} ms, host decode {1e3 * (t2 - t1):.2f} ms", flush=True)
