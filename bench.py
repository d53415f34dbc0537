#!/usr/bin/env python
"""bench.py -- encrypted MLWE PCMM ms/op at 4096x11008x128 (CKKS N = 2^16) on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--shape 4096x11008]

One "step" = one MLWE PCMM op on the named Llama shape: the level-1
RLWE ciphertexts encrypting a 128 x n_in activation block go in, the level-0 MLWE
blocks encrypting (W @ M)^T come out.  At N > 1 GPUs (torchrun, one rank per GPU, NCCL)
the weight row-blocks are sharded over ranks: rank 0's input
ciphertexts are broadcast, every rank runs K3 + K1 on its rows, and the output blocks
are all-gathered -- all inside the timed region (strong scaling of one op).

``value`` is device time per op (CUDA events, max over ranks) with the inputs resident
in HBM; ``e2e`` is the same op through the public API with host buffers (pinned H2D of
the input ciphertexts, D2H of the full output) inside the timed region.  ``--impl
reference`` times the CPU restatement (oracle/, the port of the path) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np

METRIC = "encrypted PCMM ms/op @4096x11008x128 (N=2^16); modmul-GEMM TOPS vs INT8 peak"
INT8_PEAK_TOPS = 4500.0   # NVIDIA dense INT8 spec for B200 (no measured int8 figure in MEASURED_PEAKS.json)
WORKLOADS = {
    "4096x11008": "Llama-2-7B FFN down-proj PCMM 4096x11008x128, CKKS N=2^16, MLWE (256, 256) (BASELINE config 3, metric shape)",
    "11008x4096": "Llama-2-7B FFN up/gate-proj PCMM 11008x4096x128 (BASELINE config 3)",
    "4096x4096": "Llama-2-7B QKV-proj PCMM 4096x4096x128 (BASELINE config 2)",
    "14336x4096": "Llama-3-8B FFN up-proj PCMM 14336x4096x128 (BASELINE config 4)",
    "4096x14336": "Llama-3-8B FFN down-proj PCMM 4096x14336x128 (BASELINE config 4)",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--shape", default="4096x11008")
    ap.add_argument("--params", choices=["llama", "wide"], default="llama")
    ap.add_argument("--algo", choices=["spectral", "direct"], default="spectral",
                    help="a'-column algorithm (same output words): K7 spectral (default) or K1 direct GEMM")
    ap.add_argument("--no-direct", action="store_true", help="skip the side measurement of the direct K1 path")
    ap.add_argument("--no-fused", dest="fused", action="store_false",
                    help="N > 1: gather the output with NCCL all-gather instead of fusing it into the kernels' "
                         "peer-memory stores (the default, verified against the NCCL gather before timing)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="testing only: gloo with --one-device runs the N > 1 code path with every rank on cuda:0")
    ap.add_argument("--one-device", action="store_true", help="testing only: all ranks share cuda:0")
    ap.add_argument("--cpu-rows", type=int, default=256,
                    help="oracle sample rows for cpu_baseline: 256 = one output block, ~10 s on 16 host threads (0: skip)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the Rhombus PCMv / NTT side measurements")
    a = ap.parse_args()
    if a.warmup < 0 or a.steps < 1:
        ap.error("need --steps >= 1")
    return a


def shape_of(s: str):
    n_out, n_in = (int(v) for v in s.lower().split("x"))
    return n_out, n_in


def params_of(name):
    from paper_2601_18511_b200 import HeParams

    return HeParams.wide() if name == "wide" else HeParams.llama()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock and throttle reasons."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.002):
        self.samples, self.reasons, self.max_mhz, self._raw = [], set(), None, []
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as exc:  # pragma: no cover - depends on the box
            log("clock sampling unavailable:", exc)
        self.period = period
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                t = time.perf_counter()
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self._raw.append((t, mhz, mask))
            except Exception:
                pass
            self._stop.wait(self.period)

    def window(self, t0: float, t1: float):
        """Keep the samples taken inside the host-time window [t0, t1] (the timed region)."""
        inside = [r for r in self._raw if t0 <= r[0] <= t1]
        if not inside and self._raw:   # a region shorter than one sampling period: nearest sample
            inside = [min(self._raw, key=lambda r: abs(r[0] - (t0 + t1) / 2))]
        self.samples = [r[1] for r in inside]
        self.reasons = {name for _, _, mask in inside for bit, name in self.REASONS.items() if mask & bit and bit != 0x1}

    def __enter__(self):
        if self.ok:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.ok:
            self._t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- our arm
def run_ours(a, rank: int, world: int, local: int):
    import torch
    import torch.distributed as dist

    from paper_2601_18511_b200 import HeContext, make_mlwe_pcmm_plan, pcmm_mlwe
    from paper_2601_18511_b200.context import MlweBlocks
    from paper_2601_18511_b200.pcmm import pcmm_ops, spectral_gemm_ops, spectral_inverse_bytes
    from paper_2601_18511_b200.sharding import (all_gather_into, all_reduce_max, broadcast_input,
                                                pcmm_mlwe_sharded_fused, row_shards, shard_slots, symmetric_outputs)

    if a.one_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if a.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(a.dist_backend)
    P = params_of(a.params)
    k, N = P.mlwe_rank, P.N
    n_out, n_in = shape_of(a.shape)
    b0, b1 = row_shards(n_out, k, world)[rank]         # balanced output row-blocks of this rank
    per = shard_slots(n_out, k, world)                 # padded slots per rank for the all-gather
    rows = (b1 - b0) * k
    ctx = HeContext(P, device=dev, rng="seeded")

    # synthetic data, identical on every rank (seeded device generator)
    g = torch.Generator(device=dev).manual_seed(20260117)
    W = (torch.rand((n_out, n_in), generator=g, device=dev, dtype=torch.float64) * 2 - 1) / math.sqrt(n_in)
    A = torch.rand((P.tokens, n_in), generator=g, device=dev, dtype=torch.float64) * 2 - 1
    sk = ctx.keygen(7)
    X = ctx.encrypt_acts(sk, A, seed=11)
    if rows == 0:
        raise SystemExit("more ranks than output row blocks")
    plan = make_mlwe_pcmm_plan(ctx, W[b0 * k:b1 * k], algo=a.algo)
    out_b = torch.empty((per, N), dtype=torch.int32, device=dev)
    out_a = torch.empty((per * k, N), dtype=torch.int32, device=dev)
    Y = MlweBlocks(out_b[: b1 - b0], out_a[:rows], level=0, n_rows=rows)
    sym = symmetric_outputs(ctx, n_out) if world > 1 and a.fused else None
    if world > 1:
        all_b = torch.empty((per * world, N), dtype=torch.int32, device=dev)
        all_a = torch.empty((per * world * k, N), dtype=torch.int32, device=dev)
    del W
    torch.cuda.synchronize()
    fused_check = None
    if sym is not None:
        # one op each way before timing: the fused peer stores must equal the NCCL gather word for word
        fb, fa = pcmm_mlwe_sharded_fused(ctx, plan, X, n_out, b0 * k, sym)
        broadcast_input(X.data)
        pcmm_mlwe(ctx, plan, X, out=Y)
        all_gather_into(all_b, out_b)
        all_gather_into(all_a, out_a)
        spans = row_shards(n_out, k, world)
        ok = all(torch.equal(fb[c0:c1], all_b[r * per: r * per + (c1 - c0)]) and
                 torch.equal(fa[c0 * k:c1 * k], all_a[r * per * k:(r * per + (c1 - c0)) * k])
                 for r, (c0, c1) in enumerate(spans))
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
        flag = -all_reduce_max(-flag)
        fused_check = "equal to the NCCL all-gather" if int(flag) else "MISMATCH vs NCCL all-gather: fell back to NCCL"
        if not int(flag):
            sym = None

    stream = torch.cuda.current_stream(dev)

    def step():
        if sym is not None:   # output all-gather fused into the kernels' stores (peer memory over NVLink)
            pcmm_mlwe_sharded_fused(ctx, plan, X, n_out, b0 * k, sym)
            return
        if world > 1:
            broadcast_input(X.data)
        pcmm_mlwe(ctx, plan, X, out=Y)
        if world > 1:
            all_gather_into(all_b, out_b)
            all_gather_into(all_a, out_a)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    plan.profile(True)            # per-stage CUDA events on the launching stream (he_pcmm_profile)
    with ClockSampler(local) as clk:
        time.sleep(0.05)          # sampler at its steady rate before the timed region opens
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        t0.record(stream)
        for i in range(a.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
        h1 = time.perf_counter()
    clk.window(h0, h1)
    ms = t0.elapsed_time(t1) / a.steps
    stages = plan.profile_read()
    plan.profile(False)
    stage_ms = {name: v[0] / a.steps for name, v in stages.items()}
    # stage event pairs per step; the spectral data stage holds two kernel launches (one per limb)
    launches_per_step = sum(v[1] for v in stages.values()) // a.steps + (1 if a.algo == "spectral" else 0)
    if world > 1:
        names = sorted(stage_ms)
        tt = torch.tensor([ms] + [stage_ms[n] for n in names], dtype=torch.float64, device=dev)
        tt = all_reduce_max(tt)
        ms = float(tt[0])
        stage_ms = {n: float(v) for n, v in zip(names, tt[1:].tolist())}

    # ---------------- e2e through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        e2e = run_e2e(a, ctx, plan, X, Y, rank, world, dev, out_b, out_a,
                      all_b if world > 1 else None, all_a if world > 1 else None)

    # ---------------- roofline of the dominant kernel
    cublas = measure_cublas_int8(dev) if rank == 0 else None
    if a.algo == "direct":
        roof = k1_roofline(P, rows, n_in, plan.d_w, stage_ms["modgemm"], a.shape, cublas)
    else:
        # K7 S4 (spectral inverse + rescale + a' store) dominates: HBM roofline on its algorithmic bytes
        inv_ms = stage_ms["spectral_inverse"]
        si = plan.spectral_info()
        nbytes = spectral_inverse_bytes(P, rows, si["L"], si["blocks"])
        gbs = nbytes / (inv_ms * 1e-3) / 1e9
        hbm = measured_hbm()
        roof = {"bound": "hbm", "achieved": round(gbs, 1), "peak": hbm, "unit": "GB/s", "frac": round(gbs / hbm, 4),
                "traffic": load_traffic(a.shape, "spectral_inverse"),
                "kernel": f"he::spec_inverse{si['L']}_kernel (K7 S4: {si['L']}-pt INTT x 2 limbs, rescale, a' store)",
                "kernel_ms": round(inv_ms, 3), "algorithmic_bytes_per_launch": nbytes,
                "peak_note": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"}
        gops = sum(spectral_gemm_ops(P, rows, n_in, L, si["L"], si["blocks"]) for L in (0, 1))
        g_ms = stage_ms["spectral_gemm_q0"] + stage_ms["spectral_gemm_q1"]
        roof["spectral_gemm"] = {
            "kernel": "he::spec_gemm_kernel<4>/<3> (K7 S3, tcgen05 kind::i8, per-frequency modular GEMM)",
            "ms": round(g_ms, 3), "int8_ops": gops, "TOPS": round(gops / (g_ms * 1e-3) / 1e12, 1),
            "frac_int8_peak": round(gops / (g_ms * 1e-3) / 1e12 / INT8_PEAK_TOPS, 4),
            "traffic": load_traffic(a.shape, "spectral_gemm")}
        tr = roof["spectral_gemm"]["traffic"]
        if isinstance(tr, dict) and g_ms > 0:   # S3 is bound by its DRAM traffic (G^ reads + C^ writes), not the MMAs
            s3_gbs = (tr["q0"] + tr["q1"]) / (g_ms * 1e-3) / 1e9
            roof["spectral_gemm"]["dram_GBs"] = round(s3_gbs, 1)
            roof["spectral_gemm"]["frac_hbm"] = round(s3_gbs / hbm, 4)

    extras = {}
    if world > 1 and not a.no_extras:
        # the op that scales: row-sharded PCMM + ring packing, only the packed level-0 RLWE blocks are gathered
        # (2 N words per output block, ~128x less than the MLWE rows)
        pk = packed_sharded_side(ctx, plan, sk, X, n_out, rows, dev, a.steps)
        if rank == 0:
            extras["packed_sharded"] = pk
    if rank == 0 and world == 1 and a.algo == "spectral" and not a.no_direct:
        extras["direct_k1"] = direct_side(a, ctx, W_rows=(b0 * k, b1 * k), X=X, Y=Y, P=P, rows=rows, n_in=n_in,
                                          dev=dev, cublas=cublas, ref=Y)
    if rank == 0 and world == 1 and not a.no_extras:
        extras.update(side_measurements(P, dev))
        extras["llama_shapes"] = llama_shapes_side(P, dev)

    cpu = None
    if rank == 0 and world == 1 and a.cpu_rows > 0:
        cpu = cpu_baseline(P, A, plan, X, n_out, n_in, a.cpu_rows, W_seed_dev=dev, g_seed=20260117, Y=Y, ctx=ctx,
                           sk=sk)

    if rank == 0:
        d0, d1 = P.ct_digits(0), P.ct_digits(1)
        line = {
            "metric": METRIC, "value": round(ms, 3), "unit": "ms/op", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "mma_dtype": "s8xs8->s32",
            "data": "synthetic: W ~ U[-1,1)/sqrt(n_in), acts ~ U[-1,1) (seeded), fresh RLWE encryptions on device",
            "config": {"workload": WORKLOADS.get(a.shape, a.shape), "n_out": n_out, "n_in": n_in,
                       "tokens": P.tokens, "N": N, "mlwe": [P.mlwe_degree, P.mlwe_rank],
                       "moduli": list(P.moduli), "log_delta": P.log_delta,
                       "digits": {"weight": plan.d_w, "ct_q0": d0, "ct_q1": d1},
                       "algo": a.algo + (" (K7: a' by blockwise NTT correlation + per-frequency tcgen05 GEMMs; "
                              "b' on K1)" if a.algo == "spectral" else " (K1 over all columns)"),
                       "parallelism": f"row-shard x{world}" + (
                           "" if world == 1 else " + NCCL bcast + output all-gather fused into the kernels' peer "
                           "stores (symmetric memory / CUDA IPC over NVLink; " + str(fused_check) + ")"
                           if sym is not None else " + NCCL bcast/all-gather" + (
                               f" ({fused_check})" if fused_check else "")),
                       "l2": "inputs larger than L2: each op writes and reads a "
                             f"{plan.workspace_bytes() / 1e9:.2f} GB workspace"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * a.steps,
            "clocks": clk.summary(),
            "kernels_ms": {n: round(v, 3) for n, v in stage_ms.items()},
        }
        if cpu and cpu.get("parity"):
            # every output word vs the CPU spectral restatement, plus the first row block vs the direct oracle
            line["parity"] = dict(cpu["parity"], direct_block=cpu["direct"].get("parity"))
        if cpu and cpu.get("gpu_precision"):
            line["precision_bits"] = cpu["gpu_precision"]["precision_bits"]
        line.update(extras)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def packed_sharded_side(ctx, plan, sk, X, n_out, rows, dev, steps):
    """pcmm_packed_sharded timed like the headline (CUDA events on the launching stream, max over ranks)."""
    import torch
    import torch.distributed as dist

    from paper_2601_18511_b200 import make_ring_pack_plan, ring_pack_keygen
    from paper_2601_18511_b200.sharding import all_reduce_max, pcmm_packed_sharded

    try:
        rp = make_ring_pack_plan(ctx, rows)
        keys = ring_pack_keygen(ctx, sk, seed=47)
        for _ in range(2):
            pcmm_packed_sharded(ctx, plan, rp, keys, X, n_out)
        torch.cuda.synchronize()
        dist.barrier()
        stream = torch.cuda.current_stream(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            out = pcmm_packed_sharded(ctx, plan, rp, keys, X, n_out)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = float(all_reduce_max(torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev))[0])
        p = ctx.params
        return {"ms_per_op": round(ms, 3), "steps": steps, "output_blocks": int(out.data.shape[0]),
                "gather_bytes_per_op": (n_out // p.mlwe_rank) * 2 * p.N * 4,
                "mlwe_gather_bytes_per_op": n_out * p.width * 4,
                "what": "row-sharded PCMM at level 1 + MLWE->RLWE ring packing per rank, NCCL all-gather of the "
                        "packed level-0 RLWE blocks (sharding.pcmm_packed_sharded)"}
    except Exception as exc:   # a side measurement never breaks the headline line
        return {"error": repr(exc)}


def k1_roofline(P, rows, n_in, d_w, gemm_ms, shape, cublas):
    from paper_2601_18511_b200.pcmm import pcmm_ops

    ops = pcmm_ops(P, rows, n_in, d_w)
    achieved = ops / (gemm_ms * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": round(achieved, 1), "peak": INT8_PEAK_TOPS, "unit": "TOPS",
            "frac": round(achieved / INT8_PEAK_TOPS, 4), "traffic": load_traffic(shape, "modgemm"),
            "kernel": "he::modgemm2_kernel (K1, tcgen05 kind::i8)", "kernel_ms": round(gemm_ms, 3),
            "int8_ops_per_launch": ops,
            "peak_note": "NVIDIA dense INT8 spec (4.5 POPS); MEASURED_PEAKS.json has no int8 entry",
            "cublas_int8_tops_measured": cublas,
            "frac_of_cublas_int8_measured": round(achieved / cublas, 4) if cublas else None,
            "frac_of_2x_measured_bf16": round(achieved / (2 * measured_bf16()), 4) if measured_bf16() else None}


def direct_side(a, ctx, W_rows, X, Y, P, rows, n_in, dev, cublas, ref):
    """The direct K1 path (all d (1 + k) GEMM columns on tcgen05) on the same inputs: ms/op, its
    K1 roofline, and a word-for-word comparison with the spectral output (side measurement)."""
    import torch

    from paper_2601_18511_b200 import make_mlwe_pcmm_plan, pcmm_mlwe

    try:
        g = torch.Generator(device=dev).manual_seed(20260117)
        n_out = shape_of(a.shape)[0]
        W = (torch.rand((n_out, n_in), generator=g, device=dev, dtype=torch.float64) * 2 - 1) / math.sqrt(n_in)
        plan = make_mlwe_pcmm_plan(ctx, W[W_rows[0]:W_rows[1]], algo="direct")
        del W
        out = pcmm_mlwe(ctx, plan, X)
        same = bool(torch.equal(out.out_a, ref.out_a) and torch.equal(out.out_b, ref.out_b))
        for _ in range(2):
            pcmm_mlwe(ctx, plan, X, out=out)
        plan.profile(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            pcmm_mlwe(ctx, plan, X, out=out)
        e1.record()
        torch.cuda.synchronize()
        st = plan.profile_read()
        plan.profile(False)
        res = {"ms_per_op": round(e0.elapsed_time(e1) / 5, 3), "words_equal_spectral": same,
               "roofline": k1_roofline(P, rows, n_in, plan.d_w, st["modgemm"][0] / 5, a.shape, cublas)}
        del plan, out
        torch.cuda.empty_cache()
        return res
    except Exception as exc:  # side measurement never breaks the headline line
        return {"error": repr(exc)}


def run_e2e(a, ctx, plan, X, Y, rank, world, dev, out_b, out_a, all_b, all_a):
    """Same op through the public API with host buffers: pinned H2D of the input ciphertexts
    and D2H of the whole output inside the timed region.  N = 1: pcmm_mlwe_to_host (the K1
    row chunks stream to host memory while the next chunk computes); N > 1: broadcast,
    sharded pcmm_mlwe, all-gather, then rank 0 copies the gathered output to the host."""
    import torch
    import torch.distributed as dist

    from paper_2601_18511_b200 import pcmm_mlwe, pcmm_mlwe_to_host
    from paper_2601_18511_b200.sharding import all_gather_into, all_reduce_max, broadcast_input

    steps = a.e2e_steps or max(1, min(a.steps, 5))
    h_in = torch.empty(X.data.shape, dtype=torch.int32, pin_memory=True)
    h_in.copy_(X.data)
    src_b, src_a = (all_b, all_a) if world > 1 else (out_b, out_a)
    h_b = torch.empty(src_b.shape, dtype=torch.int32, pin_memory=True)
    h_a = torch.empty(src_a.shape, dtype=torch.int32, pin_memory=True)
    stream = torch.cuda.current_stream(dev)

    def step():
        if world == 1:
            pcmm_mlwe_to_host(ctx, plan, X, h_b[: plan.n_out // ctx.params.mlwe_rank], h_a[: plan.n_out], x_host=h_in)
            return
        if rank == 0:
            X.data.copy_(h_in, non_blocking=True)
        broadcast_input(X.data)
        pcmm_mlwe(ctx, plan, X, out=Y)
        all_gather_into(all_b, out_b)
        all_gather_into(all_a, out_a)
        if rank == 0:
            h_b.copy_(src_b, non_blocking=True)
            h_a.copy_(src_a, non_blocking=True)

    for _ in range(3):   # warm-up: streams, pinned pages, the plan's chunk buffers
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device=dev)
        tt = all_reduce_max(tt)
        ms = float(tt[0])
    return {"value": round(ms, 3), "unit": "ms/op", "h2d_bytes_per_step": int(h_in.numel() * 4),
            "d2h_bytes_per_step": int((plan.n_out // ctx.params.mlwe_rank + plan.n_out) * ctx.params.N * 4)
            if world == 1 else int((h_b.numel() + h_a.numel()) * 4), "steps": steps,
            "path": "pcmm_mlwe_to_host (row chunks streamed to pinned host memory)" if world == 1
            else "broadcast + pcmm_mlwe + all_gather + D2H on rank 0"}


def side_measurements(P, dev):
    """The other §8 rows, measured in the same run (not the headline metric):
    Rhombus PCMv at BASELINE config 5 shapes (device ms/op, decrypted precision) and the K2 NTT
    throughput against HBM (algorithmic bytes = one read + one write per word)."""
    import torch

    from paper_2601_18511_b200 import (HeContext, clear_pcmv, decrypt_vector, encrypt_vector, make_rhombus_plan,
                                       native, pcmv_rhombus, rhombus_keygen)

    out = {}
    try:
        ctx = HeContext(P, device=dev, rng="seeded")
        sk = ctx.keygen(17)
        keys = rhombus_keygen(ctx, sk, 23)
        rh = {}
        for n_out, n_in in ((4096, 11008), (14336, 4096)):
            rng = np.random.default_rng(n_out + n_in)
            v = rng.uniform(-1, 1, n_in)
            W = rng.uniform(-1, 1, (n_out, n_in)) / math.sqrt(n_in)
            x = encrypt_vector(ctx, sk, v, seed=5)
            plan = make_rhombus_plan(ctx, W)
            for _ in range(2):
                y = pcmv_rhombus(ctx, plan, keys, x)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                y = pcmv_rhombus(ctx, plan, keys, x)
            e1.record()
            torch.cuda.synchronize()
            err = float(np.abs(decrypt_vector(ctx, keys.s_up_ntt, y) - clear_pcmv(W, v)).max())
            gms = graph_ms(lambda: pcmv_rhombus(ctx, plan, keys, x))
            info = plan.info()
            rh[f"{n_out}x{n_in}"] = {"ms_per_op": round(e0.elapsed_time(e1) / 5, 3), "ms_per_op_cuda_graph": gms,
                                     "precision_bits": round(-math.log2(err), 1),
                                     "split_point": info[1], "window": info[0],
                                     "key_switches": plan.key_switches() + 1,
                                     "key_switches_split0": (P.rhombus_degree - 1) * -(-n_out // P.rhombus_degree) + 1,
                                     "pt_ct_products": info[6] * info[4]}
            del plan
        out["rhombus_pcmv"] = {"workload": "BASELINE config 5: Rhombus PCMv at RLWE degree 4096 "
                                           "(decompose KS -> MVM + PackLWEs -> rescale/compose), 1 GPU", **rh}
        hbm = measured_hbm()
        ntt = {}
        for n, batch in ((65536, 1024), (4096, 16384)):   # 268 MB per batch: larger than L2, streamed from HBM
            q = P.moduli[0]
            xt = torch.randint(0, q, (batch, n), dtype=torch.int64, device=dev).to(torch.int32)
            st = ctx.stream()
            for name in ("he_ntt_forward", "he_ntt_inverse"):
                for _ in range(50):
                    native.call(name, ctx.handle, xt.data_ptr(), n, 0, batch, n, st)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    native.call(name, ctx.handle, xt.data_ptr(), n, 0, batch, n, st)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / 10
                gbs = 2 * 4 * n * batch / (ms * 1e-3) / 1e9
                ntt[f"{name.split('_')[-1]} n={n} x{batch}"] = {"GB/s": round(gbs), "frac_hbm": round(gbs / hbm, 3)}
        out["ntt"] = {"peak_GBs": hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs", **ntt}
    except Exception as exc:  # side measurements never break the headline line
        out["side_measurement_error"] = repr(exc)
    try:
        out["ring_pack"] = ring_pack_side(P, dev)
    except Exception as exc:
        out["ring_pack_error"] = repr(exc)
    try:
        out["slot_pcmm"] = slot_pcmm_side(P, dev)
    except Exception as exc:
        out["slot_pcmm_error"] = repr(exc)
    try:
        out["slot_to_coeffs"] = stc_side(P, dev)
    except Exception as exc:
        out["slot_to_coeffs_error"] = repr(exc)
    try:
        out["chained_op"] = chain_side(dev)
    except Exception as exc:
        out["chained_op_error"] = repr(exc)
    return out


def chain_side(dev, n_in: int = 11008, n_out: int = 4096, reps=3):
    """§8f2 / §8f4 with the paper's pipeline: slot-encoded activations at level 5 -> lower to
    level 4 -> Cooley-Tukey-factorized SlotToCoeffs (three maps, levels 4 -> 1) -> the metric-shape MLWE PCMM ->
    ring packing -> ModRaise into the whole chain -> CoeffToSlots (three maps, levels 5 -> 2; the linear half of
    the Half-Bootstrap): device ms per stage and the precision of each hand-off."""
    import torch

    from paper_2601_18511_b200 import (HeContext, HeParams, clear_pcmm, make_mlwe_pcmm_plan, make_ring_pack_plan,
                                       mod_raise, pcmm_packed, ring_pack_keygen, slots)
    from paper_2601_18511_b200.chain import (coeffs_to_slots_factorized, decrypt_exact, encrypt_slots_at,
                                             factorized_stc_keygen, lower_level, make_factorized_cts_plan,
                                             make_factorized_stc_plan, slot_to_coeffs_factorized)
    from paper_2601_18511_b200.stc import slot_of_coeff

    P = HeParams.llama_chain(levels=4)
    ctx = HeContext(P, device=dev, rng="seeded")
    sk = ctx.keygen(71)
    rng = np.random.default_rng(73)
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    W = rng.uniform(-1, 1, (n_out, n_in)) / math.sqrt(n_in)
    plan = make_factorized_stc_plan(ctx, input_level=4)
    keys = factorized_stc_keygen(ctx, sk, plan, seed=75)
    cts = make_factorized_cts_plan(ctx)
    ckeys = factorized_stc_keygen(ctx, sk, cts, seed=81)
    X5 = encrypt_slots_at(ctx, sk, A, level=5, seed=77, scale=plan.input_scale)
    pp, rp, rk = make_mlwe_pcmm_plan(ctx, W), make_ring_pack_plan(ctx, n_out), ring_pack_keygen(ctx, sk, 79)
    raise_to = list(P.moduli)

    def run():
        Xc = slot_to_coeffs_factorized(ctx, plan, keys, lower_level(X5, 4))
        Yp = pcmm_packed(ctx, pp, rp, rk, Xc)
        R = mod_raise(ctx, Yp, raise_to)
        return Xc, Yp, R, coeffs_to_slots_factorized(ctx, cts, ckeys, R)

    Xc, Yp, R, Z = run()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    t = [0.0] * 4
    for _ in range(reps):
        ev[0].record()
        Xc = slot_to_coeffs_factorized(ctx, plan, keys, lower_level(X5, 4))
        ev[1].record()
        Yp = pcmm_packed(ctx, pp, rp, rk, Xc)
        ev[2].record()
        R = mod_raise(ctx, Yp, raise_to)
        ev[3].record()
        Z = coeffs_to_slots_factorized(ctx, cts, ckeys, R)
        ev[4].record()
        torch.cuda.synchronize()
        for i in range(4):
            t[i] += ev[i].elapsed_time(ev[i + 1]) / reps
    e_stc = float(np.abs(ctx.decrypt_acts(sk, Xc) - A).max())
    e_out = float(np.abs(ctx.decrypt_acts(sk, Yp) - clear_pcmm(W, A)).max())
    # CoeffToSlots: the slots of two output blocks vs the exact raised phase m + q0 I (CRT over all limbs)
    ph = np.asarray(decrypt_exact(ctx, sk, R[:2]), dtype=np.float64)
    c = np.argsort(slot_of_coeff(P.N))
    want = ph[:, c] + 1j * ph[:, P.N // 2 + c]
    zo = np.asarray(decrypt_exact(ctx, sk, Z.data[:2]), dtype=np.float64)
    got = np.stack([slots.decode(v, P.N, Z.scale, real=False) for v in zo])
    e_cts = float(np.abs(got - want).max())
    n_ct = X5.n_ct
    return {"workload": f"level-5 slot input ({n_ct} cts) -> lower to 4 -> factorized SlotToCoeffs (3 maps, "
                        f"{plan.rotations} rotations / ct, {plan.plaintexts} plaintexts) -> PCMM {n_out}x{n_in}x128 -> "
                        f"ring packing -> ModRaise into the {len(raise_to)}-prime chain -> factorized CoeffToSlots "
                        f"(3 maps, {cts.rotations} rotations / ct), N = {P.N}, 1 GPU",
            "ms_total": round(sum(t), 3), "ms_slot_to_coeffs": round(t[0], 3),
            "ms_slot_to_coeffs_per_ct": round(t[0] / n_ct, 3), "ms_pcmm_packed": round(t[1], 3),
            "ms_mod_raise": round(t[2], 3), "ms_coeffs_to_slots": round(t[3], 3),
            "ms_coeffs_to_slots_per_ct": round(t[3] / int(R.shape[0]), 3),
            "precision_bits_slot_to_coeffs": round(-math.log2(e_stc), 1),
            "precision_bits_output": round(-math.log2(e_out / float(np.abs(clear_pcmm(W, A)).max())), 1),
            "coeffs_to_slots_err_log2_q0": round(math.log2(e_cts / P.moduli[0]), 1),
            "coeffs_to_slots_err_log2_delta": round(math.log2(e_cts / P.delta), 1),
            "coeffs_to_slots_shifts": list(cts.shifts), "coeffs_to_slots_pre_log2": cts.pre_log2,
            "half_bootstrap": "ModRaise + CoeffToSlots built; EvalMod not built (DESIGN.md §7e)",
            "levels": {"input": 5, "lowered": 4, "after_stc": Xc.level, "after_pcmm_pack": Yp.level,
                       "raised": int(R.shape[1]) - 1, "after_cts": Z.level}}


def graph_ms(fn, reps=5):
    """Device ms per replay of the op captured into a CUDA graph (paper_2601_18511_b200.OpGraph)."""
    import torch

    from paper_2601_18511_b200 import OpGraph

    try:
        g = OpGraph(fn)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return round(e0.elapsed_time(e1) / reps, 3)
    except Exception:
        return None


def llama_shapes_side(P, dev, reps=5):
    """The spectral MLWE PCMM at every Llama-2-7B / Llama-3-8B projection shape (BASELINE configs 2-4; x 128
    tokens, N = 2^16): device ms/op (CUDA events, inputs resident), synthetic seeded weights and activations."""
    import torch

    from paper_2601_18511_b200 import HeContext, make_mlwe_pcmm_plan, pcmm_mlwe

    out = {"workload": "spectral MLWE PCMM (K7) at the Llama projection shapes x 128 tokens, N = 2^16, 1 GPU"}
    try:
        ctx = HeContext(P, device=dev, rng="seeded")
        sk = ctx.keygen(3)
        g = torch.Generator(device=dev).manual_seed(7)
        for n_out, n_in in ((4096, 4096), (4096, 11008), (11008, 4096), (14336, 4096), (4096, 14336)):
            W = (torch.rand((n_out, n_in), generator=g, device=dev, dtype=torch.float64) * 2 - 1) / math.sqrt(n_in)
            A = torch.rand((P.tokens, n_in), generator=g, device=dev, dtype=torch.float64) * 2 - 1
            X = ctx.encrypt_acts(sk, A, seed=2)
            plan = make_mlwe_pcmm_plan(ctx, W)
            Y = pcmm_mlwe(ctx, plan, X)
            for _ in range(2):
                pcmm_mlwe(ctx, plan, X, out=Y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(reps):
                pcmm_mlwe(ctx, plan, X, out=Y)
            e1.record()
            torch.cuda.synchronize()
            out[f"{n_out}x{n_in}"] = {"ms_per_op": round(e0.elapsed_time(e1) / reps, 3)}
            del W, A, X, plan, Y
            torch.cuda.empty_cache()
    except Exception as exc:   # a side line must not take the headline down
        out["error"] = repr(exc)
    return out


def slot_pcmm_side(P, dev, reps=5):
    """§8f3: hesim's own pcmm_bsgs schedule on real CKKS ciphertexts (slotpcmm.py), d x d in the N/2 slots:
    device ms/op and decrypted precision against clear_pcmm."""
    import torch

    from paper_2601_18511_b200 import (HeContext, clear_slot_pcmm, decrypt_packed, encrypt_packed,
                                       make_slot_pcmm_plan, pcmm_slot_bsgs, slot_pcmm_keygen)

    ctx = HeContext(P, device=dev, rng="seeded")
    sk = ctx.keygen(51)
    res = {}
    for d in (128, 64):
        rng = np.random.default_rng(d)
        W = rng.uniform(-1, 1, (d, d)) / math.sqrt(d)
        B = rng.uniform(-1, 1, (d, d))
        plan = make_slot_pcmm_plan(ctx, W, shear_power=0)
        keys = slot_pcmm_keygen(ctx, sk, plan, seed=53)
        X = encrypt_packed(ctx, sk, B, 1, seed=55)
        Y = pcmm_slot_bsgs(ctx, plan, keys, X)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            Y = pcmm_slot_bsgs(ctx, plan, keys, X)
        e1.record()
        torch.cuda.synchronize()
        ref = clear_slot_pcmm(W, B, 0)
        err = float(np.abs(decrypt_packed(ctx, sk, Y) - ref).max())
        gms = graph_ms(lambda: pcmm_slot_bsgs(ctx, plan, keys, X))
        res[f"d{d}"] = {"ms_per_op": round(e0.elapsed_time(e1) / reps, 3), "ms_per_op_cuda_graph": gms,
                        "rotations": plan.split.baby + plan.split.giant - 2, "split": [plan.split.baby, plan.split.giant],
                        "precision_bits": round(-math.log2(err / float(np.abs(ref).max())), 1)}
    return {"workload": f"hesim pcmm_bsgs schedule on CKKS ciphertexts, N = {P.N}, d x d in {P.N // 2} slots "
                        "(hoisted baby rotations, gadget key switching), 1 GPU", **res}


def stc_side(P, dev, reps=3):
    """§8f2: SlotToCoeffs (stc.py), slot-encoded activations -> the App. A coefficient layout: device ms per
    ciphertext and the decrypted precision against the activations."""
    import torch

    from paper_2601_18511_b200 import HeContext
    from paper_2601_18511_b200.stc import (encrypt_slots, make_slot_to_coeffs_plan, slot_to_coeffs,
                                           slot_to_coeffs_keygen)

    ctx = HeContext(P, device=dev, rng="seeded")
    sk = ctx.keygen(61)
    plan = make_slot_to_coeffs_plan(ctx)
    keys = slot_to_coeffs_keygen(ctx, sk, plan, seed=63)
    A = np.random.default_rng(65).uniform(-1, 1, (P.mlwe_degree // 2, 6 * P.mlwe_rank))
    X = encrypt_slots(ctx, sk, A, seed=67)
    Y = slot_to_coeffs(ctx, plan, keys, X)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    for _ in range(reps):
        Y = slot_to_coeffs(ctx, plan, keys, X)
    e1.record(torch.cuda.current_stream())
    torch.cuda.synchronize()
    err = float(np.abs(ctx.decrypt_acts(sk, Y) - A).max())
    b, g = plan.split.baby, plan.split.giant
    res = {"workload": f"SlotToCoeffs, N = {P.N}: one {b}x{g} BSGS map over the {P.N // 2} diagonals per ct "
                       f"(App. A bit-reversal fused, {'lazy' if plan.lazy else 'eager'} ModDown, {X.n_ct} cts "
                       "under one plan), 1 GPU",
           "ms_per_ct": round(e0.elapsed_time(e1) / reps / X.n_ct, 3), "rotations_per_ct": b + g - 2,
           "plaintext_bytes": int(plan.pts.numel() * 4), "precision_bits": round(-math.log2(err), 1)}
    del plan, keys, X, Y
    torch.cuda.empty_cache()
    return res


def ring_pack_side(P, dev, shape="4096x11008", reps=3):
    """§8f1: the PCMM followed by MLWE -> RLWE ring packing (the packed op), at the metric shape:
    device ms of the packing alone and of the whole packed op, the packed op end to end (pinned host
    input -> packed level-0 RLWE output on the host) and the decrypted precision."""
    import torch

    from paper_2601_18511_b200 import (HeContext, make_mlwe_pcmm_plan, make_ring_pack_plan, pcmm_level1,
                                       pcmm_packed, ring_pack, ring_pack_keygen)

    n_out, n_in = shape_of(shape)
    ctx = HeContext(P, device=dev, rng="seeded")
    g = torch.Generator(device=dev).manual_seed(31)
    W = (torch.rand((n_out, n_in), generator=g, device=dev, dtype=torch.float64) * 2 - 1) / math.sqrt(n_in)
    A = torch.rand((P.tokens, n_in), generator=g, device=dev, dtype=torch.float64) * 2 - 1
    sk = ctx.keygen(41)
    X = ctx.encrypt_acts(sk, A, seed=43)
    keys = ring_pack_keygen(ctx, sk, seed=47)
    plan = make_mlwe_pcmm_plan(ctx, W)
    rp = make_ring_pack_plan(ctx, n_out)
    Y = pcmm_packed(ctx, plan, rp, keys, X)
    torch.cuda.synchronize()
    ref = (A @ W.T).cpu().numpy()
    err = float(np.abs(ctx.decrypt_acts(sk, Y) - ref).max())
    raw_b, raw_a = rp.raw(ctx)
    x_host = X.data.cpu().pin_memory()
    y_host = torch.empty(Y.data.shape, dtype=Y.data.dtype).pin_memory()

    def e2e():
        X.data.copy_(x_host, non_blocking=True)
        pcmm_packed(ctx, plan, rp, keys, X, Y.data)
        y_host.copy_(Y.data, non_blocking=True)

    res = {}
    for name, fn in (("ring_pack_ms", lambda: ring_pack(ctx, rp, keys, raw_b, raw_a, Y.data)),
                     ("packed_op_ms", lambda: pcmm_packed(ctx, plan, rp, keys, X, Y.data)),
                     ("packed_e2e_ms", e2e)):
        fn()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name] = round(float(np.median(ts)), 3)
    return {"workload": f"{shape} PCMM + MLWE->RLWE key-switch packing (k = {P.mlwe_rank} hybrid key switches "
                        f"per block, one digit, special modulus P1 P2; method {rp.method}) -> "
                        f"{n_out // P.mlwe_rank} level-0 RLWE ciphertexts, 1 GPU",
            **res, "precision_bits": round(-math.log2(err / float(np.abs(ref).max())), 1),
            "output_bytes": int(Y.data.numel() * 4), "h2d_bytes": int(x_host.numel() * 4)}


def measured_hbm():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0


def measure_cublas_int8(dev):
    import torch

    try:
        n = 8192
        x = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
        y = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t()
        for _ in range(2):
            torch._int_mm(x, y)
        best = 1e9
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(5):
            e0.record()
            torch._int_mm(x, y)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return round(2 * n ** 3 / (best * 1e-3) / 1e12, 1)
    except Exception as exc:  # pragma: no cover
        log("cublas int8 probe failed:", exc)
        return None


def measured_bf16():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["bf16_tflops"])
    except Exception:
        return None


def load_traffic(shape: str, kernel: str):
    """dram read + write bytes per launch of `kernel` from the committed ncu --set full summary."""
    p = ROOT / "profiles" / "ncu_summary.json"
    try:
        ent = json.loads(p.read_text()).get(kernel, {}).get(shape)
        if ent:
            return ent.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


# ----------------------------------------------------------------- CPU baseline / reference arm
def cpu_baseline(P, A, plan, X, n_out, n_in, n_rows, W_seed_dev=None, g_seed=None, Y=None, ctx=None, sk=None):
    """Time the oracle (C restatement, OpenMP over all host threads) on n_rows output rows x
    all 65 792 columns x full K, both limbs + rescale; extrapolate to the full op.  The sample's words
    are then compared with the GPU output block of the same rows (every word), and the GPU rows are
    decrypted against the float product (precision in bits)."""
    import torch

    import oracle as O

    g = torch.Generator(device=W_seed_dev).manual_seed(g_seed)
    W = ((torch.rand((n_out, n_in), generator=g, device=W_seed_dev, dtype=torch.float64) * 2 - 1)
         / math.sqrt(n_in))
    W_full = W.cpu().numpy()
    del W
    W0 = W_full[: P.mlwe_rank]                   # first row block
    Wt = O.encode_weights(P, W0)
    ct = X.data.cpu().numpy().view(np.uint32)
    n_rows = min(n_rows, P.mlwe_rank)
    # the same algorithm as the GPU path on the CPU (he_oracle_spectral.c), on the FULL workload: no
    # extrapolation, and every output word compared with the GPU's
    Wt_full = O.encode_weights(P, W_full)
    del W_full
    O.pcmm_spectral(P, Wt_full[:8], ct)           # warm-up (thread pool, tables)
    t0 = time.perf_counter()
    ref_full = O.pcmm_spectral(P, Wt_full, ct)
    sp_s = time.perf_counter() - t0
    del Wt_full
    same_alg = {"value": round(sp_s * 1e3, 1), "unit": "ms/op", "cores": O.num_threads(), "kind": "port",
                "algorithm": "spectral (the GPU's overlap-save correlations, L = 4k; oracle/he_oracle_spectral.c)",
                "sample": f"the full op: all {n_out} output rows x {P.width} cols x K={n_in}, both limbs + rescale",
                "extrapolated": False}
    if Y is not None:
        k, d = P.mlwe_rank, P.mlwe_degree
        ga = Y.out_a.cpu().numpy().view(np.uint32)
        gb = Y.out_b.cpu().numpy().view(np.uint32).reshape(-1, P.N)   # [n_out / k][N], b'_(Y k + t)[m] at t + k m
        eq_a = int((ga == ref_full[:, d:]).sum())
        bref = ref_full[:, :d].reshape(-1, k, d).transpose(0, 2, 1).reshape(-1, P.N)   # [block][m][t] -> t + k m
        eq_b = int((gb == bref).sum())
        total = n_out * P.width
        same_alg["parity"] = {"words_checked": total, "words_equal": eq_a + eq_b == total,
                              "words_differing": total - eq_a - eq_b, "rows": [0, n_out],
                              "against": "oracle/he_oracle_spectral.c or_pcmm_spectral (every word of the output)"}
    del ref_full
    res = O.time_pcmm_sample(P, Wt, ct, n_rows)
    per_op = res["seconds"] * n_out / n_rows * 1e3
    parity = precision = None
    if Y is not None:
        ref = res.pop("words")
        k, d = P.mlwe_rank, P.mlwe_degree
        ga = Y.out_a[:n_rows].cpu().numpy().view(np.uint32)
        gb = Y.out_b[: -(-n_rows // k)].cpu().numpy().view(np.uint32)
        eq_a = int((ga == ref[:, d:]).sum())
        eq_b = sum(int((gb[y // k, y % k + k * np.arange(d)] == ref[y, :d]).sum()) for y in range(n_rows))
        total = n_rows * P.width
        parity = {"words_checked": total, "words_equal": eq_a + eq_b == total, "words_differing": total - eq_a - eq_b,
                  "rows": [0, n_rows], "against": "oracle/he_oracle.c or_pcmm (direct BCHPS24 Alg. 2, exact)"}
        if ctx is not None and sk is not None:
            dec = ctx.decrypt_pcmm(sk, Y, rows=(0, n_rows))[:, :n_rows]
            clear = A.cpu().numpy() @ W0[:n_rows].T
            err = float(np.abs(dec - clear).max())
            precision = {"precision_bits": round(-math.log2(err), 2), "max_abs_err": err,
                         "max_abs_out": float(np.abs(clear).max()), "rows": [0, n_rows]}
    else:
        res.pop("words", None)
    # context: the unencrypted product on the same host, numpy float64 (BLAS threads)
    rng = np.random.default_rng(0)
    Wf, Af = rng.standard_normal((n_out, n_in)), rng.standard_normal((P.tokens, n_in))
    Af @ Wf.T
    t0 = time.perf_counter()
    for _ in range(3):
        Af @ Wf.T
    floor_ms = (time.perf_counter() - t0) / 3 * 1e3
    # value: the same algorithm on the CPU, full workload (the hardware ratio); `direct`: BCHPS24 Alg. 2 as the
    # paper states it (the reference arm's algorithm), extrapolated from one row block (algorithm x hardware)
    return {"value": same_alg["value"], "unit": "ms/op", "cores": same_alg["cores"], "kind": "port",
            "sample": same_alg["sample"], "extrapolated": False, "algorithm": same_alg["algorithm"],
            "parity": same_alg.get("parity"),
            "direct": {"value": round(per_op, 1), "unit": "ms/op", "cores": res["threads"], "kind": "port",
                       "sample": f"oracle/ C restatement: {n_rows} of {n_out} output rows x {P.width} cols x "
                                 f"K={n_in}, both limbs + rescale, {res['seconds']:.2f} s, extrapolated "
                                 f"x{n_out / n_rows:.0f}",
                       "extrapolated": True, "sample_rows": n_rows, "extrapolation_factor": round(n_out / n_rows, 3),
                       "sample_seconds": round(res["seconds"], 3), "algorithm": "direct (BCHPS24 Alg. 2 as a GEMM)",
                       "parity": parity},
            "gpu_precision": precision,
            "plaintext_floor_ms": round(floor_ms, 2),
            "plaintext_floor": f"numpy float64 acts @ W.T ({P.tokens} x {n_in} x {n_out}) on the host, unencrypted",
            "hesim_context": hesim_context()}


def hesim_context():
    """the reference's own slot-domain pcmm_bsgs (float simulator) at its largest
    feasible size, measured in the build container by tools/hesim_context_timing.py (the reference is
    not on the GPU box) and committed under profiles/r01/."""
    f = Path(__file__).resolve().parent / "profiles" / "r01" / "hesim_pcmm_bsgs_cpu.json"
    try:
        d = json.loads(f.read_text())
        r = d["results"]["128"]
        return {"d": 128, "pcmm_bsgs_ms": round(1e3 * r["pcmm_bsgs_s"], 2), "plan_ms": round(1e3 * r["plan_s"], 2),
                "source": "profiles/r01/hesim_pcmm_bsgs_cpu.json (build container, not this host)"}
    except Exception:
        return None


def run_reference(a, rank: int, world: int):
    """--impl reference: the CPU restatement of the path (the reference package has no
    implementation of it) on the host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle as O

    P = params_of(a.params)
    n_out, n_in = shape_of(a.shape)
    k = P.mlwe_rank
    rng = np.random.default_rng(20260117)
    W0 = rng.uniform(-1, 1, (k, n_in)) / math.sqrt(n_in)
    A = rng.uniform(-1, 1, (P.tokens, n_in))
    s = O.keygen(P, 7)
    ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
    Wt = O.encode_weights(P, W0)
    rows = max(1, min(a.cpu_rows, k) // 16)
    for _ in range(a.warmup):
        O.pcmm(P, Wt, ct, rows=list(range(1)), cols=list(range(64)))
    vals = []
    for _ in range(a.steps):
        res = O.time_pcmm_sample(P, Wt, ct, rows)
        vals.append(res["seconds"] * n_out / rows * 1e3)
    v = float(np.median(vals))
    # context: the GPU path's own algorithm on the same host cores, full workload (one run, no extrapolation)
    Wf = rng.uniform(-1, 1, (n_out, n_in)) / math.sqrt(n_in)
    Wtf = O.encode_weights(P, Wf)
    del Wf
    O.pcmm_spectral(P, Wtf[:8], ct)
    t0 = time.perf_counter()
    O.pcmm_spectral(P, Wtf, ct)
    sp_ms = (time.perf_counter() - t0) * 1e3
    del Wtf
    line = {
        "metric": METRIC, "value": round(v, 1), "unit": "ms/op", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(v, 1), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "impl": "reference",
        "data": "synthetic: W ~ U[-1,1)/sqrt(n_in), acts ~ U[-1,1) (seeded), fresh RLWE encryptions (CPU)",
        "config": {"workload": WORKLOADS.get(a.shape, a.shape), "n_out": n_out, "n_in": n_in, "N": P.N,
                   "mlwe": [P.mlwe_degree, P.mlwe_rank], "moduli": list(P.moduli)},
        "cpu_baseline": {"value": round(v, 1), "unit": "ms/op", "cores": O.num_threads(), "kind": "port",
                         "sample": f"per step {rows} of {n_out} output rows x {P.width} cols x K={n_in}, both "
                                   f"limbs + rescale, extrapolated x{n_out / rows:.0f} (oracle/he_oracle.c, OpenMP)",
                         "extrapolated": True, "sample_rows": rows, "extrapolation_factor": round(n_out / rows, 3),
                         "algorithm": "direct (BCHPS24 Alg. 2 as a GEMM)"},
        "extrapolated": True,
        "e2e": {"value": round(v, 1), "unit": "ms/op", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "same_algorithm_cpu": {"value": round(sp_ms, 1), "unit": "ms/op", "cores": O.num_threads(),
                               "algorithm": "spectral (oracle/he_oracle_spectral.c), the full op, not extrapolated"},
        "note": "hesim (the reference package) does not implement the MLWE PCMM (SPEC.md:8); the reference "
                "arm times the CPU restatement of the path (BCHPS24 Alg. 2); same_algorithm_cpu is the GPU "
                "path's algorithm on the same cores",
    }
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank, world)
    else:
        run_ours(a, rank, world, local)


if __name__ == "__main__":
    main()
