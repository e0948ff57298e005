"""Sequence sharding on one GPU: W handles, each holding its page range of
every sequence, driven layer by layer with the external exchange (the all-gathers done here as
device copies between the handles' workspaces).  The same kernels run as with NCCL; only the
transport differs.  Checks: outputs identical on every rank, equal to the unsharded stack
within fp32 merge rounding and to the fp64 oracle within R19; selections identical (exact)."""
import numpy as np
import pytest

import synth
from helpers import (C0, GpuCase, Shape, assert_close_bf16, assert_close_fp32, oracle_step, planting_for)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


class ShardedStack:
    def __init__(self, shape: Shape, seed: int, batch: int, s_pre: int, max_seq: int, W: int, planting=None,
                 det: int = 0):
        from paper_2510_09883_b200 import DeltaStack
        from synth import device as sd
        self.shape, self.batch, self.W = shape, batch, W
        self.ranks = []
        for r in range(W):
            cfg = shape.delta_config(batch, max_seq)
            cfg.shard_world, cfg.shard_rank, cfg.det_chunks = W, r, det
            bt = torch.from_numpy(synth.block_table(seed, batch, cfg.max_pages))
            st = DeltaStack.allocate(cfg, bt)
            sd.fill_pools(st.kv_pool, st.block_table, seed, s_pre, batch, range(shape.L), planting)
            st.set_seq_lens([s_pre] * batch)
            self.ranks.append(st)

    def _exchange(self, which: int):
        blocks = []
        for st in self.ranks:
            send, recv, nbytes = st.exchange_buffers(which)
            base = st.workspace.data_ptr()
            blocks.append((st.workspace, send - base, recv - base, nbytes))
        for ws_dst, _, roff, nbytes in blocks:
            for r, (ws_src, soff, _, _) in enumerate(blocks):
                ws_dst[roff + r * nbytes: roff + (r + 1) * nbytes].copy_(ws_src[soff: soff + nbytes])

    def step(self, q, k, v):
        from paper_2510_09883_b200 import ROLE_SELECT
        sh, B = self.shape, self.batch
        outs = [torch.empty((sh.L, B, sh.m, sh.d), dtype=torch.float32, device="cuda") for _ in self.ranks]
        lses = [torch.empty((sh.L, B, sh.m), dtype=torch.float32, device="cuda") for _ in self.ranks]
        plans = {}
        cap = self.ranks[0].plan_capacity
        for l in range(sh.L):
            if self.W == 1:  # R21 chunks on one rank: no exchange, the handle merges its chunks
                st = self.ranks[0]
                st.append_decode_layer(l, k[l], v[l], q[l], outs[0][l], lses[0][l])
                if st.role(l) == ROLE_SELECT:
                    idx = torch.empty((B, cap), dtype=torch.int32, device="cuda")
                    cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
                    st.select(l, B, idx_out=idx, count_out=cnt)
                    plans[l] = [(idx, cnt)]
                continue
            for r, st in enumerate(self.ranks):
                st.append_decode_layer(l, k[l], v[l], q[l], outs[r][l])
            self._exchange(0)
            for r, st in enumerate(self.ranks):
                st.shard_merge(l, outs[r][l], lses[r][l])
            if self.ranks[0].role(l) == ROLE_SELECT:
                for st in self.ranks:
                    st.select(l, B)
                self._exchange(1)
                plans[l] = []
                for st in self.ranks:
                    idx = torch.empty((B, cap), dtype=torch.int32, device="cuda")
                    cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
                    st.shard_select_merge(l, B, idx, cnt)
                    plans[l].append((idx, cnt))
        torch.cuda.synchronize()
        for st in self.ranks:
            assert st.get_error() == 0
        host = {l: [[idx[b, : int(cnt[b])].cpu().numpy() for b in range(B)] for idx, cnt in v_]
                for l, v_ in plans.items()}
        return [o.cpu().numpy() for o in outs], [x.cpu().numpy() for x in lses], host


@pytest.mark.parametrize("W", [2, 3])
@pytest.mark.parametrize("shape", [
    C0,
    Shape(L=4, m=32, g=8, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=16, dtype="bf16"),
], ids=["c0-fp32-token", "bf16-page"])
def test_sharded_equals_unsharded_and_oracle(shape, W):
    s = 1500
    plant = planting_for(shape, s)          # planted: the expected selection is known exactly
    seed = 60 + W
    ref = GpuCase(shape, seed, batch=2, s_pre=s - 1, max_seq=1600, planting=plant)
    out_u, lse_u, plans_u = ref.step_layers(s)
    sharded = ShardedStack(shape, seed, batch=2, s_pre=s - 1, max_seq=1600, W=W, planting=plant)
    q, k, v = ref.inputs(s)
    outs, lses, plans = sharded.step(q, k, v)
    for r in range(1, W):                    # every rank ends with the same O, LSE and plan
        np.testing.assert_array_equal(outs[r], outs[0])
        np.testing.assert_array_equal(lses[r], lses[0])
    for l in plans_u:
        for r in range(W):
            for b in range(2):
                assert plans[l][r][b].tolist() == plans_u[l][b].tolist(), f"plan layer {l} rank {r} seq {b}"
    tol = 1e-5   # fp32 rounding of a different merge tree vs the unsharded merge
    np.testing.assert_allclose(outs[0], out_u, atol=tol, rtol=0)
    np.testing.assert_allclose(lses[0], lse_u, atol=tol, rtol=0)
    for b in range(2):
        ora = oracle_step(shape, seed, b, s, planting=plant)
        for l, (o_out, o_lse, units, _keys, _toks) in ora.items():
            if shape.dtype == "fp32":
                assert_close_fp32(outs[0][l, b], o_out, f"layer {l}")
            else:
                assert_close_bf16(outs[0][l, b], o_out, f"layer {l}")
            if units is not None:
                assert plans[l][0][b].tolist() == units.tolist()


def test_shard_with_empty_rank():
    """A context shorter than one rank's share: the last ranks attend nothing (lse = -inf
    partials) and the merge must still give the unsharded result."""
    shape = C0
    s = 300                                  # 19 pages; W = 4 over max_seq 2048 -> 32 pages per rank
    ref = GpuCase(shape, 71, batch=1, s_pre=s - 1, max_seq=2048)
    out_u, _, plans_u = ref.step_layers(s)
    sharded = ShardedStack(shape, 71, batch=1, s_pre=s - 1, max_seq=2048, W=4)
    q, k, v = ref.inputs(s)
    outs, _, plans = sharded.step(q, k, v)
    np.testing.assert_allclose(outs[0], out_u, atol=1e-5, rtol=0)
    assert plans[1][3][0].tolist() == plans_u[1][0].tolist()


@pytest.mark.parametrize("shape", [
    C0,
    Shape(L=4, m=32, g=8, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=16, dtype="bf16"),
], ids=["c0-fp32-token", "bf16-page"])
def test_det_chunks_bitwise_across_world_sizes(shape):
    """R21: with det_chunks = 8 the outputs, LSEs and plans of W = 1, 2, 4, 8 are bitwise
    identical (the same chunk partials, merged in the same fixed order), and still equal the
    unchunked stack within fp32 merge rounding and the fp64 oracle within R19.  Two steps, so the
    second attends the token the first appended through the separate append launch."""
    s, seed, B, C = 1500, 93, 2, 8           # 100 pages, chunks of 13: the last is ragged
    plant = planting_for(shape, s)
    ref = GpuCase(shape, seed, batch=B, s_pre=s - 1, max_seq=1600, planting=plant)
    out_u, lse_u, plans_u = ref.step_layers(s)
    runs = {}
    for W in (1, 2, 4, 8):
        st = ShardedStack(shape, seed, batch=B, s_pre=s - 1, max_seq=1600, W=W, planting=plant, det=C)
        first = st.step(*ref.inputs(s))
        second = st.step(*ref.inputs(s + 1))
        runs[W] = (first, second)
    for W in (2, 4, 8):
        for step in range(2):
            outs, lses, plans = runs[W][step]
            o1, l1, p1 = runs[1][step]
            for r in range(W):
                np.testing.assert_array_equal(outs[r], o1[0], err_msg=f"W={W} rank {r} step {step}")
                np.testing.assert_array_equal(lses[r], l1[0], err_msg=f"W={W} rank {r} step {step}")
                for l in p1:
                    for b in range(B):
                        assert plans[l][r][b].tolist() == p1[l][0][b].tolist()
    (o1, l1, p1), (o2, _, _) = runs[1]
    np.testing.assert_allclose(o1[0], out_u, atol=1e-5, rtol=0)
    np.testing.assert_allclose(l1[0], lse_u, atol=1e-5, rtol=0)
    for b in range(B):
        for l in plans_u:
            assert p1[l][0][b].tolist() == plans_u[l][b].tolist()
        for step, ss, outs in ((0, s, o1), (1, s + 1, o2)):
            ora = oracle_step(shape, seed, b, ss, planting=plant)
            for l, (o_out, _lse, _units, _keys, _toks) in ora.items():
                if shape.dtype == "fp32":
                    assert_close_fp32(outs[0][l, b], o_out, f"step {step} layer {l}")
                else:
                    assert_close_bf16(outs[0][l, b], o_out, f"step {step} layer {l}")


def test_det_chunks_graph_step_equals_layer_calls():
    """R21 chunks inside the captured decode step (delta_decode_step): bitwise equal to the
    same handle driven layer by layer."""
    shape = Shape(L=4, m=32, g=8, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=16, dtype="bf16")
    s, seed = 1500, 94
    a = GpuCase(shape, seed, batch=2, s_pre=s - 1, max_seq=1600)
    b = GpuCase(shape, seed, batch=2, s_pre=s - 1, max_seq=1600)
    for case in (a, b):  # rebuild both handles with det_chunks = 8
        from paper_2510_09883_b200 import DeltaStack
        from synth import device as sd
        case.cfg.det_chunks = 8
        case.stack = DeltaStack.allocate(case.cfg, case.stack.block_table.cpu())
        sd.fill_pools(case.stack.kv_pool, case.stack.block_table, seed, s - 1, 2, range(shape.L), None)
        case.stack.set_seq_lens([s - 1] * 2)
    out_l, lse_l, _ = a.step_layers(s)
    out_g, lse_g = b.step_graph(s)
    np.testing.assert_array_equal(out_g, out_l)
    np.testing.assert_array_equal(lse_g, lse_l)


def test_nccl_loads_and_makes_an_id():
    """The NCCL path loads the library at run time (the copy torch uses) and produces an id;
    the multi-GPU exchange itself needs >= 2 GPUs (bench.py --config c3 under torchrun)."""
    import paper_2510_09883_b200 as d200
    uid = d200.nccl_unique_id()
    assert isinstance(uid, bytes) and len(uid) == 128 and any(uid)
