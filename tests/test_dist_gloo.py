"""Multi-process (world_size 2, gloo, CPU) coverage of the sequence-sharded protocol's host
side: the ranks' page ranges from the C ABI partition the cache; the two
exchanges of the method — an all-gather of per-rank (o, lse) partials merged in rank order,
and an all-gather of per-rank top-k candidates merged into the global selection — reproduce
the unsharded oracle.  The GPU kernels doing the same merges are covered by
tests/test_gpu_shard.py; here the collectives are real (torch.distributed, gloo)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

W = 2


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank: int, port: int, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=W)
        import oracle
        import paper_2510_09883_b200 as d200
        import synth
        from helpers import Shape

        # 1. page ranges from the library partition [0, pages) across the ranks
        shape = Shape(L=2, m=8, g=2, d=64, F=1, delta=[1], k=64, S=4, Lw=32, block=16, dtype="fp32")
        max_seq = 1024
        cfg = shape.delta_config(1, max_seq)
        cfg.shard_world, cfg.shard_rank = W, rank
        lo, hi = d200.shard_range(cfg)
        ranges = [None] * W
        dist.all_gather_object(ranges, (lo, hi))
        pages = -(-max_seq // 16)
        assert ranges[0][0] == 0 and ranges[-1][1] == pages
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))

        # 2. LSE merge of per-rank partials over a real collective
        s, seed, layer = 900, 17, 1
        K = synth.kv_rows(seed, layer, 0, 0, s, shape.g, shape.d, "fp32", "k")
        V = synth.kv_rows(seed, layer, 0, 0, s, shape.g, shape.d, "fp32", "v")
        kv = oracle.SeqKV.from_contiguous(K, V, 16)
        qv = synth.q_rows(seed, layer, 0, s, shape.m, shape.d, "fp32")
        scale = shape.oracle_config().scale
        own = np.arange(min(lo * 16, s), min(hi * 16, s), dtype=np.int64)
        if own.size:
            o_r, lse_r, _ = oracle.decode_heads(qv, kv, own, scale)
        else:
            o_r, lse_r = np.zeros((shape.m, shape.d)), np.full(shape.m, -np.inf)
        got_o = [torch.zeros(shape.m, shape.d, dtype=torch.float64) for _ in range(W)]
        got_l = [torch.zeros(shape.m, dtype=torch.float64) for _ in range(W)]
        dist.all_gather(got_o, torch.from_numpy(np.ascontiguousarray(o_r)))
        dist.all_gather(got_l, torch.from_numpy(np.ascontiguousarray(lse_r)))
        lses = np.stack([x.numpy() for x in got_l])          # [W][m], rank order
        M = lses.max(axis=0)
        LSE = M + np.log(np.exp(lses - M).sum(axis=0))
        O = sum(np.exp(lses[r] - LSE)[:, None] * got_o[r].numpy() for r in range(W))
        o_full, lse_full, alpha = oracle.decode_heads(qv, kv, s, scale, want_alpha=True)
        np.testing.assert_allclose(O, o_full, atol=1e-12, rtol=0)
        np.testing.assert_allclose(LSE, lse_full, atol=1e-12, rtol=0)

        # 3. global selection from per-rank candidates (scores use the MERGED LSE)
        k_units = shape.k // shape.block
        s_t = oracle.token_scores(alpha)                     # alpha uses the global LSE
        S_u = oracle.page_scores(s_t, 16)
        n_units = S_u.size
        units = np.arange(n_units)
        forced = (units < 1) | (units >= (s - shape.Lw) // 16)
        mine = (units >= lo) & (units < hi) & ~forced
        cand = units[mine][np.lexsort((units[mine], -S_u[mine]))][:k_units]   # (key desc, index asc)
        pad = np.full(k_units, -1, np.int64)
        pad[: cand.size] = cand
        keys = np.full(k_units, -np.inf)
        keys[: cand.size] = S_u[cand]
        all_c = [torch.zeros(k_units, dtype=torch.int64) for _ in range(W)]
        all_k = [torch.zeros(k_units, dtype=torch.float64) for _ in range(W)]
        dist.all_gather(all_c, torch.from_numpy(pad))
        dist.all_gather(all_k, torch.from_numpy(keys))
        cu = np.concatenate([c.numpy() for c in all_c])
        ck = np.concatenate([k.numpy() for k in all_k])
        ok = cu >= 0
        cu, ck = cu[ok], ck[ok]
        top = cu[np.lexsort((cu, -ck))][:k_units]
        rho = np.sort(np.concatenate([units[forced], top]))
        expect = oracle.select(S_u, s, 16, shape.S, shape.Lw, k_units)
        assert rho.tolist() == expect.tolist()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc()))
        raise


def test_two_rank_gloo_sharded_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(W)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(W))
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results
