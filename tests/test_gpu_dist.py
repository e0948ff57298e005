"""Sequence sharding across PROCESSES: two ranks, each its own process and its
own libdelta handle (shard_world = 2) holding its page range of every sequence, exchange their
attention partials and top-k candidates through torch.distributed (gloo; both processes share
the one GPU of a gpurun box, so the NCCL transport itself — one GPU per rank — is not what runs
here: the library's external-exchange entry points are).  Checks: both ranks end with identical
outputs, LSEs and plans; the outputs equal a single-process unsharded stack within fp32 merge
rounding and the fp64 oracle within R19; the Delta plans equal the oracle's (planted inputs)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
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


def _exchange(st, which: int):
    """All-gather of this rank's block of exchange region `which` into every rank's receive area."""
    send, recv, nbytes = st.exchange_buffers(which)
    ws = st.workspace
    base = ws.data_ptr()
    mine = ws[send - base: send - base + nbytes].cpu()
    parts = [torch.empty_like(mine) for _ in range(W)]
    dist.all_gather(parts, mine)
    ws[recv - base: recv - base + W * nbytes].copy_(torch.cat(parts).to(ws.device))


def _worker(rank: int, port: int, q, det: int = 0):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=W)
        import synth
        from helpers import Shape, planting_for
        from paper_2510_09883_b200 import ROLE_SELECT, DeltaStack
        from synth import device as sd
        shape = Shape(L=4, m=32, g=8, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=16, dtype="bf16")
        s, seed, B = 1500, 88, 2
        plant = planting_for(shape, s)
        cfg = shape.delta_config(B, 1600)
        cfg.shard_world, cfg.shard_rank, cfg.det_chunks = W, rank, det
        bt = torch.from_numpy(synth.block_table(seed, B, cfg.max_pages))
        st = DeltaStack.allocate(cfg, bt)
        sd.fill_pools(st.kv_pool, st.block_table, seed, s - 1, B, range(shape.L), plant)
        st.set_seq_lens([s - 1] * B)
        qd = torch.empty((shape.L, B, shape.m, shape.d), dtype=torch.bfloat16, device="cuda")
        kd = torch.empty((shape.L, B, shape.g, shape.d), dtype=torch.bfloat16, device="cuda")
        vd = torch.empty_like(kd)
        sd.fill_queries(qd, seed, range(shape.L), [s] * B, plant)
        sd.fill_new_kv(kd, vd, seed, range(shape.L), [s - 1] * B)
        out = torch.empty((shape.L, B, shape.m, shape.d), dtype=torch.float32, device="cuda")
        lse = torch.empty((shape.L, B, shape.m), dtype=torch.float32, device="cuda")
        cap = st.plan_capacity
        plans = {}
        for l in range(shape.L):
            st.append_decode_layer(l, kd[l], vd[l], qd[l], out[l])
            torch.cuda.synchronize()
            _exchange(st, 0)
            st.shard_merge(l, out[l], lse[l])
            if st.role(l) == ROLE_SELECT:
                st.select(l, B)
                torch.cuda.synchronize()
                _exchange(st, 1)
                idx = torch.empty((B, cap), dtype=torch.int32, device="cuda")
                cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
                st.shard_select_merge(l, B, idx, cnt)
                plans[l] = (idx, cnt)
        torch.cuda.synchronize()
        assert st.get_error() == 0
        res = (out.cpu().numpy(), lse.cpu().numpy(),
               {l: [idx[b, : int(cnt[b])].cpu().numpy() for b in range(B)] for l, (idx, cnt) in plans.items()})
        gathered = [None] * W
        dist.all_gather_object(gathered, res)
        if rank == 0:
            q.put(("ok", gathered))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put(("err", f"rank {rank}: {e}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("det", [0, 8], ids=["ranges", "r21-chunks"])
def test_two_process_sequence_sharding(det):
    from helpers import GpuCase, Shape, assert_close_bf16, oracle_step, planting_for
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, det)) for r in range(W)]
    for p in procs:
        p.start()
    status, payload = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
    assert status == "ok", payload
    (out0, lse0, plans0), (out1, lse1, plans1) = payload
    np.testing.assert_array_equal(out0, out1)
    np.testing.assert_array_equal(lse0, lse1)
    assert {l: [p.tolist() for p in v] for l, v in plans0.items()} == {l: [p.tolist() for p in v] for l, v in plans1.items()}
    shape = Shape(L=4, m=32, g=8, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=16, dtype="bf16")
    s, seed = 1500, 88
    plant = planting_for(shape, s)
    ref = GpuCase(shape, seed, batch=2, s_pre=s - 1, max_seq=1600, planting=plant)
    out_u, lse_u, plans_u = ref.step_layers(s)
    if det:  # R21: bitwise equal to one process holding all 8 chunks
        from test_gpu_shard import ShardedStack
        one = ShardedStack(shape, seed, batch=2, s_pre=s - 1, max_seq=1600, W=1, planting=plant, det=det)
        outs1, lses1, plans1 = one.step(*ref.inputs(s))
        np.testing.assert_array_equal(out0, outs1[0])
        np.testing.assert_array_equal(lse0, lses1[0])
        assert [p.tolist() for p in plans0[1]] == [p.tolist() for p in plans1[1][0]]
    np.testing.assert_allclose(out0, out_u, atol=1e-5, rtol=0)
    np.testing.assert_allclose(lse0, lse_u, atol=1e-5, rtol=0)
    for b in range(2):
        assert plans0[1][b].tolist() == plans_u[1][b].tolist()
        ora = oracle_step(shape, seed, b, s, planting=plant)
        for l, (o_out, _lse, units, _k, _t) in ora.items():
            assert_close_bf16(out0[l, b], o_out, f"layer {l} seq {b}")
            if units is not None:
                assert plans0[l][b].tolist() == units.tolist()
