"""N > 1 host logic on CPU: world_size 2 (and 3) gloo processes run the row-sharded PCMM
data flow -- input broadcast, per-rank shard, padded all-gather, trim -- with each rank's
shard computed by the oracle, and must reassemble exactly the unsharded output."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2601_18511_b200.params import HeParams
from paper_2601_18511_b200.sharding import broadcast_input, gather_row_shards, row_shards, shard_slots


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n_out, n_in, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = HeParams.toy()
        k, N, d = P.mlwe_rank, P.N, P.mlwe_degree
        rng = np.random.default_rng(0)
        W = rng.uniform(-1, 1, (n_out, n_in)) / np.sqrt(n_in)
        A = rng.uniform(-1, 1, (P.tokens, n_in))
        s = O.keygen(P, 7)
        # only rank 0 holds the input; the broadcast delivers it (C2)
        if rank == 0:
            ct = O.encrypt(P, 11, s, O.encode_acts(P, A))
            data = torch.from_numpy(ct.view(np.int32).copy())
        else:
            data = torch.zeros((n_in // k, 2, 2, N), dtype=torch.int32)
        broadcast_input(data)
        ct = data.numpy().view(np.uint32)
        b0, b1 = row_shards(n_out, k, world)[rank]
        per = shard_slots(n_out, k, world)
        Wt = O.encode_weights(P, W)
        local = O.pcmm(P, Wt, ct, rows=list(range(b0 * k, b1 * k))) if b1 > b0 else np.zeros((0, P.width), np.uint32)
        lb = torch.zeros((per, N), dtype=torch.int32)
        la = torch.zeros((per * k, N), dtype=torch.int32)
        for i in range(b1 - b0):
            rows = local[i * k:(i + 1) * k]
            comp = np.zeros(N, np.uint32)
            for t in range(k):
                comp[t + k * np.arange(d)] = rows[t, :d]
            lb[i] = torch.from_numpy(comp.view(np.int32))
            la[i * k:(i + 1) * k] = torch.from_numpy(rows[:, d:].copy().view(np.int32))
        out_b, out_a = gather_row_shards(lb, la, k, n_out)
        full = O.pcmm(P, Wt, ct)
        assert np.array_equal(out_a.numpy().view(np.uint32), full[:, d:])
        for r in range(n_out // k):
            rows = full[r * k:(r + 1) * k]
            comp = np.zeros(N, np.uint32)
            for t in range(k):
                comp[t + k * np.arange(d)] = rows[t, :d]
            assert np.array_equal(out_b[r].numpy().view(np.uint32), comp)
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_out", [(2, 64), (3, 80)])
def test_row_sharded_pcmm_gathers_exact_output(world, n_out):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_out, 32, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}


def test_rhombus_shards_follow_the_paper():
    """n_in = 4096 -> column split, 4096/8 = 512 input values per rank at 8 GPUs;
    n_in > 4096 -> row split (leaf groups), every rank busy."""
    from paper_2601_18511_b200.sharding import rhombus_shards

    n, rho = 4096, 16
    for n_out, n_in in ((4096, 11008), (14336, 4096), (11008, 4096), (4096, 4096), (4096, 14336)):
        w = 1
        while w * rho < n_in:
            w *= 2
        for world in (1, 2, 4, 8):
            sl = rhombus_shards(n_out, n_in, n, world, window=w)
            assert len(sl) == world and all(s["active"] for s in sl)
            strat = sl[0]["strategy"]
            assert strat == ("cols" if n_in <= n else "rows")
            if strat == "cols":
                spans = [s["cols"] for s in sl]
                assert spans[0][0] == 0 and spans[-1][1] == n_in
                for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
                    assert a1 == b0 and a0 < a1
                for s in sl:
                    assert s["cols"][0] == s["piece0"] * w
                if world == 8 and n_in == 4096:
                    assert all(s["cols"][1] - s["cols"][0] == 512 for s in sl)
            else:
                assert sorted(s["group"] for s in sl) == list(range(world))
                assert all(s["groups"] == world for s in sl)
    sl = rhombus_shards(4096, 11008, n, 3, window=1024)    # 3 ranks: 2 leaf groups, one idle rank
    assert [s["active"] for s in sl] == [True, True, False] and sl[0]["groups"] == 2
    with pytest.raises(ValueError):
        rhombus_shards(4096, 4096, n, 2, strategy="diagonal")
