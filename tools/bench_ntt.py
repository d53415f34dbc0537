"""K2 roofline: negacyclic NTT / INTT throughput vs HBM (algorithmic bytes = one read + one write
of every u32 word per transform).  python tools/bench_ntt.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2601_18511_b200 import HeContext, HeParams, native

HBM = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6544.3) \
    if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6544.3


def run(ctx, n, limb, batch, iters=20):
    q = ctx.params.moduli[limb]
    x = torch.randint(0, q, (batch, n), dtype=torch.int64, device="cuda").to(torch.int32)
    st = ctx.stream()
    out = {}
    for name in ("he_ntt_forward", "he_ntt_inverse"):
        for _ in range(100):   # ~20 ms of warm-up: clocks ramp before the timed region
            native.call(name, ctx.handle, x.data_ptr(), n, limb, batch, n, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            native.call(name, ctx.handle, x.data_ptr(), n, limb, batch, n, st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        gbs = 2 * 4 * n * batch / (ms * 1e-3) / 1e9
        out[name] = (ms, gbs, gbs / HBM)
    return out


def main():
    ctx = HeContext(HeParams.llama(), rng="seeded")
    res = {}
    # 268 MB per batch: larger than the 126 MB L2, so the transform streams from HBM
    sizes = ((65536, 1024), (4096, 16384)) if "--small" not in sys.argv else ((65536, 256), (4096, 4096))
    for n, batch in sizes:
        for limb in (0, 1):
            r = run(ctx, n, limb, batch)
            for k, (ms, gbs, frac) in r.items():
                key = f"{k.split('_')[-1]} n={n} limb={limb} batch={batch}"
                res[key] = {"ms": round(ms, 4), "GB/s": round(gbs, 1), "frac_hbm": round(frac, 3)}
                print(f"{key}: {ms:.4f} ms  {gbs:.0f} GB/s  {frac * 100:.1f}% of {HBM} GB/s", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
