"""Staged bring-up check of the CUDA path against the oracle (run on a GPU box).

python tools/gpu_check.py [--big]
"""

import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np
import torch

import oracle as O
from paper_2601_18511_b200 import HeContext, HeParams, make_mlwe_pcmm_plan, pcmm_mlwe


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def stage(name):
    print(f"--- {name}", flush=True)


def run(P, n_out, n_in, seed=1, rows=None, cols=None, full=False):
    ctx = HeContext(P, rng="seeded")
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    stage(f"keygen {P.name}")
    sk = ctx.keygen(7)
    s_o = O.keygen(P, 7)
    assert np.array_equal(sk.s.cpu().numpy(), s_o), "secret mismatch"
    stage("encrypt")
    X = ctx.encrypt_acts(sk, A, seed=11)
    torch.cuda.synchronize()
    ct_g = u32(X.data)
    pt = O.encode_acts(P, A)
    ct_o = O.encrypt(P, 11, s_o, pt)
    if not np.array_equal(ct_g, ct_o):
        bad = np.argwhere(ct_g != ct_o)
        print("encrypt mismatch at", bad[:5], "count", len(bad))
        # which part differs
        print("a equal:", np.array_equal(ct_g[:, :, 0], ct_o[:, :, 0]), "b equal:", np.array_equal(ct_g[:, :, 1], ct_o[:, :, 1]))
        raise SystemExit(1)
    print("encrypt bit-exact", ct_g.shape)
    dec = ctx.decrypt_acts(sk, X)
    print("decrypt err", np.abs(dec - A).max())
    stage("plan")
    plan = make_mlwe_pcmm_plan(ctx, W)
    torch.cuda.synchronize()
    Wt = O.encode_weights(P, W)
    print("d_w", plan.d_w, "max_abs", plan.max_abs, "oracle max", np.abs(Wt).max())
    dg = plan.digits.cpu().numpy().astype(np.int64)
    rec = sum(dg[i] * (256 ** i) for i in range(plan.d_w))
    assert np.array_equal(rec, Wt), "weight digits mismatch"
    print("weight digits exact")
    stage("pcmm")
    Y = pcmm_mlwe(ctx, plan, X)
    torch.cuda.synchronize()
    print("ledger", ctx.ledger.to_dict())
    out_a = u32(Y.out_a)
    out_b = u32(Y.out_b)
    d, k = P.mlwe_degree, P.mlwe_rank
    if rows is None:
        rows = list(range(n_out))
    if cols is None:
        cols = list(range(P.width))
    ref = O.pcmm(P, Wt, ct_o, rows=rows, cols=cols)
    got = np.zeros_like(ref)
    for i, y in enumerate(rows):
        for j, n in enumerate(cols):
            if n < d:
                got[i, j] = out_b[y // k, (y % k) + k * n]
            else:
                got[i, j] = out_a[y, n - d]
    ok = np.array_equal(got, ref)
    print("pcmm bit-exact:", ok, "mismatches:", int((got != ref).sum()), "of", ref.size)
    if not ok:
        bad = np.argwhere(got != ref)[:10]
        for i, j in bad:
            print("  row", rows[i], "col", cols[j], "got", got[i, j], "ref", ref[i, j])
    stage("decrypt-and-compare")
    nr = min(n_out, 64)
    out = ctx.decrypt_pcmm(sk, Y, rows=(0, nr))
    refm = A @ W.T
    err = np.nanmax(np.abs(out[:, :] - refm)[~np.isnan(out)])
    print(f"decrypted rows 0..{nr}: max err {err:.3e} = {-np.log2(err):.1f} bits")
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--bench", action="store_true")
    ap.add_argument("--time", action="store_true")
    a = ap.parse_args()
    print(torch.cuda.get_device_name(0))
    ok = run(HeParams.toy(), 48, 32)
    ok &= run(HeParams.toy(), 256, 384)
    if a.big:
        P = HeParams.llama()
        rows = [0, 1, 127, 128, 255, 1000, 4095]
        rng = np.random.default_rng(5)
        cols = sorted(set([0, 1, 255, 256, 257, 511, 512, P.width - 1] + list(rng.integers(0, P.width, 40))))
        ok &= run(P, 4096, 4096, rows=rows, cols=cols)
    print("ALL OK" if ok else "FAILURES")


if __name__ == "__main__" and "--time" not in sys.argv and "--rhombus" not in sys.argv:
    main()


def time_shape(n_out, n_in, iters=5):
    import ctypes
    from paper_2601_18511_b200 import native
    P = HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    rng = np.random.default_rng(3)
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
    sk = ctx.keygen(1)
    X = ctx.encrypt_acts(sk, A, seed=2)
    plan = make_mlwe_pcmm_plan(ctx, W)
    Y = pcmm_mlwe(ctx, plan, X)
    torch.cuda.synchronize()
    ws = plan.workspace(ctx.device)
    st = ctx.stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    tdec, tgemm = [], []
    for _ in range(iters):
        ev[0].record()
        native.call("he_pcmm_decompose", plan._handle, X.data.data_ptr(), ws.data_ptr(), ws.numel(), st)
        ev[1].record()
        native.call("he_pcmm_gemm", plan._handle, ws.data_ptr(), Y.out_b.data_ptr(), Y.out_a.data_ptr(), st)
        ev[2].record()
        torch.cuda.synchronize()
        tdec.append(ev[0].elapsed_time(ev[1]))
        tgemm.append(ev[1].elapsed_time(ev[2]))
    d0, d1 = P.ct_digits(0), P.ct_digits(1)
    ops = 2 * n_out * n_in * P.width * plan.d_w * (d0 + d1)
    g = min(tgemm)
    print(f"shape {n_out}x{n_in}: d_w={plan.d_w} decompose {min(tdec):.3f} ms, gemm {g:.3f} ms "
          f"-> {ops / g / 1e9:.1f} TOPS int8 ({ops/g/1e9/4500*100:.1f}% of 4.5 POPS); all {tgemm}")
    ws_bytes = ws.numel()
    print(f"  decompose writes {ws_bytes/1e9:.2f} GB -> {ws_bytes/min(tdec)/1e6:.0f} GB/s")


if __name__ == "__main__" and "--time" in sys.argv:
    time_shape(4096, 11008)


def time_rhombus(shapes=((4096, 11008), (14336, 4096)), iters=3):
    from paper_2601_18511_b200.rhombus import (clear_pcmv, decrypt_vector, encrypt_vector, make_rhombus_plan,
                                               pcmv_rhombus, rhombus_keygen)
    P = HeParams.llama()
    ctx = HeContext(P, rng="seeded")
    sk = ctx.keygen(7)
    t0 = time.time()
    keys = rhombus_keygen(ctx, sk, 99)
    torch.cuda.synchronize()
    print(f"rhombus keygen {time.time() - t0:.2f} s")
    for n_out, n_in in shapes:
        rng = np.random.default_rng(1)
        v = rng.uniform(-1, 1, n_in)
        W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
        x = encrypt_vector(ctx, sk, v, seed=5)
        plan = make_rhombus_plan(ctx, W)
        y = pcmv_rhombus(ctx, plan, keys, x)
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            y = pcmv_rhombus(ctx, plan, keys, x)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res = decrypt_vector(ctx, keys.s_up_ntt, y)
        err = np.abs(res - clear_pcmv(W, v)).max()
        print(f"rhombus PCMv {n_out}x{n_in}: {min(ts):.3f} ms (all {['%.2f' % t for t in ts]}), err {err:.2e} = {-np.log2(err):.1f} bits")


if __name__ == "__main__" and "--rhombus" in sys.argv:
    time_rhombus()
