"""e2e of pcmm_mlwe_to_host at 4096x11008 vs chunk_rows, plus the plain pinned D2H floor.  GPU tool."""
import math, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, pcmm_mlwe, pcmm_mlwe_to_host

P = HeParams.llama()
ctx = HeContext(P, rng="seeded")
g = torch.Generator(device="cuda").manual_seed(1)
n_out, n_in = 4096, 11008
W = (torch.rand((n_out, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1) / math.sqrt(n_in)
A = torch.rand((P.tokens, n_in), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
X = ctx.encrypt_acts(ctx.keygen(1), A, seed=2)
plan = make_mlwe_pcmm_plan(ctx, W)
Y = pcmm_mlwe(ctx, plan, X)
h_in = torch.empty(X.data.shape, dtype=torch.int32, pin_memory=True)
h_in.copy_(X.data)
h_b = torch.empty(Y.out_b.shape, dtype=torch.int32, pin_memory=True)
h_a = torch.empty(Y.out_a.shape, dtype=torch.int32, pin_memory=True)
torch.cuda.synchronize()
# plain D2H floor
for _ in range(2):
    h_a.copy_(Y.out_a, non_blocking=True); h_b.copy_(Y.out_b, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    h_a.copy_(Y.out_a, non_blocking=True); h_b.copy_(Y.out_b, non_blocking=True)
torch.cuda.synchronize()
print(f"plain D2H of the output: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms ({(Y.out_a.numel() + Y.out_b.numel()) * 4 / 1e9:.3f} GB)")
for cr in (256, 512, 1024, 2048):
    for _ in range(2):
        pcmm_mlwe_to_host(ctx, plan, X, h_b, h_a, x_host=h_in, chunk_rows=cr)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        pcmm_mlwe_to_host(ctx, plan, X, h_b, h_a, x_host=h_in, chunk_rows=cr)
    torch.cuda.synchronize()
    print(f"chunk_rows={cr}: e2e {(time.perf_counter() - t) / 5 * 1e3:.2f} ms")
