"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded
synthetic inputs.  Tolerances: R19 (bf16: max-abs 2e-3 and rel-L2 1e-2 per (layer, seq);
fp32: max-abs 1e-5); selections: R20 (exact on planted inputs and whenever the oracle's
boundary gap exceeds 2e-5; top-k exact on any fp32 key buffer)."""
import numpy as np
import pytest

import oracle
import synth
from helpers import (C0, C0_PAGE, C1, GpuCase, Shape, assert_close_bf16, assert_close_fp32, check_plan,
                     oracle_layer, oracle_step, planting_for)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _cmp(shape, gpu, ref, what):
    return assert_close_bf16(gpu, ref, what) if shape.dtype == "bf16" else assert_close_fp32(gpu, ref, what)


def _lse_tol(shape):
    return 2e-4 if shape.dtype == "bf16" else 2e-5


def _check_step(case: GpuCase, s: int, out, lse, plans, layers=None, exact_plans=False):
    sh = case.shape
    for b in range(case.batch):
        ref = oracle_step(sh, case.seed, b, s, layers, case.planting)
        same_plan = {}
        for l, (o_out, o_lse, units, keys, toks) in ref.items():
            if units is not None and l in plans:
                same_plan[l] = check_plan(plans[l][b], units, keys, s, sh, exact_plans)
        roles, gov = oracle.validate_tiers(sh.L, sh.F, sh.delta)
        for l, (o_out, o_lse, units, keys, toks) in ref.items():
            if layers is not None and l not in layers:
                continue
            if roles[l] == oracle.ROLE_SPARSE and not same_plan.get(int(gov[l]), True):
                # near-tie swap at the boundary (R20 iii): the GPU attended its own (valid) plan,
                # so its output is checked against the oracle attending that plan
                toks = oracle.units_to_tokens(np.asarray(plans[int(gov[l])][b]), sh.block, s)
                o_out, o_lse, _ = oracle_layer(sh, case.seed, l, b, s, case.planting, tokens=toks)
            _cmp(sh, out[l, b], o_out, f"layer {l} seq {b}")
            assert np.max(np.abs(lse[l, b] - o_lse)) <= _lse_tol(sh), f"lse layer {l}"


# ---------------------------------------------------------------- generator identity

@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_device_generator_matches_numpy(dtype):
    sh = Shape(L=2, m=8, g=2, d=64, F=1, delta=[1], k=32, S=4, Lw=16, block=16, dtype=dtype)
    plant = planting_for(sh, 100)
    case = GpuCase(sh, 99, batch=2, s_pre=100, max_seq=160, planting=plant)
    kp = case.stack.k_pool.float().cpu().numpy()
    vp = case.stack.v_pool.float().cpu().numpy()
    bt = case.stack.block_table.cpu().numpy()
    for l in range(2):
        for b in range(2):
            K = synth.kv_rows(99, l, b, 0, 100, 2, 64, dtype, "k", plant)
            V = synth.kv_rows(99, l, b, 0, 100, 2, 64, dtype, "v", plant)
            for t in (0, 17, 99):
                np.testing.assert_array_equal(kp[l, bt[b, t // 16], :, t % 16], K[t])
                np.testing.assert_array_equal(vp[l, bt[b, t // 16], :, t % 16], V[t])
    q, k, v = case.inputs(101)
    for l in range(2):
        for b in range(2):
            np.testing.assert_array_equal(q[l, b].float().cpu().numpy(), synth.q_rows(99, l, b, 101, 8, 64, dtype, plant))
            np.testing.assert_array_equal(k[l, b].float().cpu().numpy(),
                                          synth.kv_rows(99, l, b, 100, 101, 2, 64, dtype, "k")[0])


# ---------------------------------------------------------------- C0 (fp32, tiny)

def test_c0_step_token_mode():
    case = GpuCase(C0, 2510, batch=1, s_pre=511, max_seq=640)
    out, lse, plans = case.step_layers(512)
    assert len(plans[1][0]) == 164   # 4 sink + 32 window + 128 salient (R1)
    _check_step(case, 512, out, lse, plans)


def test_c0_multistep_crosses_page_boundary():
    case = GpuCase(C0, 2511, batch=1, s_pre=499, max_seq=640)
    for s in range(500, 521):
        out, lse, plans = case.step_layers(s)
        _check_step(case, s, out, lse, plans)


def test_c0_page_mode():
    case = GpuCase(C0_PAGE, 2512, batch=2, s_pre=511, max_seq=640)
    out, lse, plans = case.step_layers(512)
    assert len(plans[1][0]) == 1 + 2 + 8   # sink page + 2 window pages + k/P (R6)
    _check_step(case, 512, out, lse, plans)


@pytest.mark.parametrize("shape", [C0, C0_PAGE], ids=["token", "page"])
def test_c0_planted_exact_selection(shape):
    plant = planting_for(shape, 512)
    case = GpuCase(shape, 77, batch=2, s_pre=511, max_seq=640, planting=plant)
    out, lse, plans = case.step_layers(512)
    for b in range(2):
        units = synth.planted_units(77, 1, b, plant)
        blk = shape.block
        forced = set(range(0, (shape.S - 1) // blk + 1)) | set(range((512 - shape.Lw) // blk, -(-512 // blk)))
        assert plans[1][b].tolist() == sorted(forced | set(units.tolist()))  # known without any oracle
    _check_step(case, 512, out, lse, plans, exact_plans=True)


# ---------------------------------------------------------------- bf16 tensor-core path

BF16_SMALL = Shape(L=4, m=32, g=8, d=128, F=1, delta=[1], k=512, S=4, Lw=32, block=16, dtype="bf16")


@pytest.mark.parametrize("s", [3001, 4096])
def test_bf16_c1_heads_ragged(s):
    case = GpuCase(BF16_SMALL, 31, batch=2, s_pre=s - 1, max_seq=4160)
    out, lse, plans = case.step_layers(s)
    _check_step(case, s, out, lse, plans)


@pytest.mark.parametrize("shape", [
    Shape(L=3, m=28, g=4, d=128, F=1, delta=[1], k=1024, S=4, Lw=32, block=16, dtype="bf16"),   # Qwen-7B gs=7
    Shape(L=3, m=40, g=8, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=16, dtype="bf16"),    # Qwen3-14B gs=5
    Shape(L=3, m=16, g=2, d=64, F=1, delta=[1], k=64, S=4, Lw=32, block=1, dtype="bf16"),       # d=64, token plan
], ids=["gs7", "gs5", "d64-token"])
def test_bf16_gqa_variants(shape):
    case = GpuCase(shape, 5, batch=3, s_pre=2100, max_seq=2200)
    out, lse, plans = case.step_layers(2101)
    _check_step(case, 2101, out, lse, plans)


def test_bf16_fewhot_precision():
    """Concentrated attention (3 tokens raised by ~+25): exposes bf16-rounded probabilities
    (SURVEY App. B); the hi/lo split of P must keep the error under 2e-3."""
    sh = Shape(L=2, m=32, g=8, d=128, F=2, delta=[], k=0, S=0, Lw=0, block=16, dtype="bf16")
    plant = planting_for(Shape(L=2, m=32, g=8, d=128, F=2, delta=[], k=0, S=4, Lw=32, block=1, dtype="bf16"),
                         4096, "fewhot")
    case = GpuCase(sh, 8, batch=1, s_pre=4095, max_seq=4096, planting=plant)
    out, lse, plans = case.step_layers(4096)
    _check_step(case, 4096, out, lse, plans)


def test_bf16_planted_token_plan_exact():
    sh = Shape(L=3, m=32, g=8, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=1, dtype="bf16")
    plant = planting_for(sh, 3000)
    case = GpuCase(sh, 12, batch=2, s_pre=2999, max_seq=3072, planting=plant)
    out, lse, plans = case.step_layers(3000)
    _check_step(case, 3000, out, lse, plans, exact_plans=True)


# ---------------------------------------------------------------- top-k on fp32 key buffers

@pytest.mark.parametrize("kind", ["iid", "ties", "equal"])
@pytest.mark.parametrize("block,s,k", [(1, 5000, 700), (16, 32768, 2048), (1, 40000, 3000), (16, 300, 4000)])
def test_topk_bitexact_on_key_buffer(kind, block, s, k):
    """R20 (i): the radix select == a correct top-k (key desc, index asc) on the same buffer."""
    sh = Shape(L=2, m=8, g=2, d=64, F=1, delta=[1], k=k, S=4, Lw=32, block=block, dtype="fp32")
    case = GpuCase(sh, 3, batch=2, s_pre=0, max_seq=s)
    case.stack.set_seq_lens([s, s - 7])
    n_units = -(-s // block)
    keys = np.stack([synth.keys_buffer(40 + b, n_units, kind) for b in range(2)]).astype(np.float32)
    kt = torch.from_numpy(keys).cuda()
    cap = case.stack.plan_capacity
    idx = torch.empty((2, cap), dtype=torch.int32, device="cuda")
    cnt = torch.empty((2,), dtype=torch.int32, device="cuda")
    case.stack.select(1, 2, keys_override=kt, idx_out=idx, count_out=cnt)
    torch.cuda.synchronize()
    for b, sb in enumerate([s, s - 7]):
        ref = oracle.select(keys[b].astype(np.float64), sb, block, sh.S, sh.Lw, k // block)
        got = idx[b, : int(cnt[b])].cpu().numpy()
        assert got.tolist() == ref.tolist()
        assert (idx[b, int(cnt[b]):] == -1).all()


# ---------------------------------------------------------------- API-level properties

def test_graph_step_equals_per_layer_calls_bitwise():
    a = GpuCase(BF16_SMALL, 21, batch=2, s_pre=1999, max_seq=2100)
    b = GpuCase(BF16_SMALL, 21, batch=2, s_pre=1999, max_seq=2100)
    for s in (2000, 2001):
        out_a, lse_a, _ = a.step_layers(s)
        out_b, lse_b = b.step_graph(s)
        np.testing.assert_array_equal(out_a, out_b)
        np.testing.assert_array_equal(lse_a, lse_b)


def test_step_host_buffers_equal_device():
    a = GpuCase(BF16_SMALL, 22, batch=1, s_pre=999, max_seq=1100)
    b = GpuCase(BF16_SMALL, 22, batch=1, s_pre=999, max_seq=1100)
    out_a, _ = a.step_graph(1000)
    q, k, v = b.inputs(1000)
    qh, kh, vh = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
    out_h = torch.empty(out_a.shape, dtype=torch.float32).pin_memory()
    st = torch.cuda.Stream()
    b.stack.decode_step_host(qh, kh, vh, out_h, stream=st)
    st.synchronize()
    np.testing.assert_array_equal(out_a, out_h.numpy())


def test_step_host_pipelined_multi_step():
    """Consecutive delta_decode_step_host calls overlap (two staging slots, internal streams):
    every step's host output equals the device-buffer step's, bitwise, and a per-layer call
    after the run is ordered after it."""
    a = GpuCase(BF16_SMALL, 24, batch=2, s_pre=1499, max_seq=1600)
    b = GpuCase(BF16_SMALL, 24, batch=2, s_pre=1499, max_seq=1600)
    st = torch.cuda.Stream()
    outs_h = []
    ref = []
    for s in range(1500, 1505):
        out_a, _ = a.step_graph(s)
        ref.append(out_a)
        q, k, v = b.inputs(s)
        qh, kh, vh = q.cpu().pin_memory(), k.cpu().pin_memory(), v.cpu().pin_memory()
        out_h = torch.empty(out_a.shape, dtype=torch.float32).pin_memory()
        b.stack.decode_step_host(qh, kh, vh, out_h, stream=st)
        outs_h.append((out_h, qh, kh, vh))      # keep the pinned inputs alive until the sync
    st.synchronize()
    for r, (oh, *_) in zip(ref, outs_h):
        np.testing.assert_array_equal(r, oh.numpy())
    # a device-buffer step after the host run continues the same cache
    out_a, _ = a.step_graph(1505)
    out_b, _ = b.step_graph(1505)
    np.testing.assert_array_equal(out_a, out_b)
    assert b.stack.get_error() == 0


def test_deterministic_across_runs():
    outs = []
    for _ in range(2):
        c = GpuCase(BF16_SMALL, 23, batch=2, s_pre=2999, max_seq=3100)
        outs.append(c.step_layers(3000))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    for l in outs[0][2]:
        for b in range(2):
            np.testing.assert_array_equal(outs[0][2][l][b], outs[1][2][l][b])


def test_budget_covering_context_makes_delta_equal_full():
    """k >= s => every sparse layer attends to everything."""
    sh = Shape(L=3, m=32, g=8, d=128, F=1, delta=[1], k=2048, S=4, Lw=32, block=16, dtype="bf16")
    full = Shape(L=3, m=32, g=8, d=128, F=3, delta=[], k=2048, S=4, Lw=32, block=16, dtype="bf16")
    a = GpuCase(sh, 24, batch=1, s_pre=999, max_seq=1024)
    b = GpuCase(full, 24, batch=1, s_pre=999, max_seq=1024)
    out_a, _, plans = a.step_layers(1000)
    out_b, _, _ = b.step_layers(1000)
    assert plans[1][0].tolist() == list(range(63))
    np.testing.assert_allclose(out_a, out_b, atol=1e-6, rtol=0)


def test_standalone_append_then_decode():
    sh = Shape(L=2, m=8, g=2, d=64, F=2, delta=[], k=0, S=0, Lw=0, block=16, dtype="fp32")
    case = GpuCase(sh, 25, batch=2, s_pre=30, max_seq=128)
    ntok = 37
    k_new = torch.stack([torch.from_numpy(synth.kv_rows(25, 0, b, 30, 30 + ntok, 2, 64, "fp32", "k")) for b in range(2)]).cuda()
    v_new = torch.stack([torch.from_numpy(synth.kv_rows(25, 0, b, 30, 30 + ntok, 2, 64, "fp32", "v")) for b in range(2)]).cuda()
    case.stack.append_kv(0, k_new, v_new)
    torch.cuda.synchronize()
    kp = case.stack.k_pool.cpu().numpy()
    bt = case.stack.block_table.cpu().numpy()
    for b in range(2):
        for i in range(ntok):
            t = 30 + i
            np.testing.assert_array_equal(kp[0, bt[b, t // 16], :, t % 16], k_new[b, i].cpu().numpy())
    q = torch.from_numpy(np.stack([synth.q_rows(25, 0, b, 67, 8, 64, "fp32") for b in range(2)])).cuda()
    out = torch.empty((2, 8, 64), dtype=torch.float32, device="cuda")
    case.stack.decode_layer(0, q, out)
    torch.cuda.synchronize()
    for b in range(2):
        ref = oracle_step(sh, 25, b, 67, layers=[0])
        assert_close_fp32(out[b].cpu().numpy(), ref[0][0])


def test_stale_plan_is_a_usage_error():
    from paper_2510_09883_b200 import DeltaError
    case = GpuCase(C0, 26, batch=1, s_pre=300, max_seq=400)
    q, k, v = case.inputs(301)
    out = torch.empty((1, 8, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(DeltaError, match="USAGE"):
        case.stack.append_decode_layer(2, k[2], v[2], q[2], out)   # sparse before its Delta selected


def test_capacity_error_is_sticky():
    case = GpuCase(C0, 27, batch=1, s_pre=64, max_seq=64)
    q, k, v = case.inputs(65)
    out = torch.empty((1, 8, 64), dtype=torch.float32, device="cuda")
    case.stack.append_decode_layer(0, k[0], v[0], q[0], out)
    assert case.stack.get_error() == 4


# ---------------------------------------------------------------- C1 at full size

def test_c1_full_size_planted_graph_step():
    """BASELINE configs[1] (Llama-8B shape, b=1, s=32768, k=2048 page mode) in the launch
    configuration bench.py times (graph-captured step).  Planted inputs make the expected
    selections known a priori; outputs are checked on a sample of layers of every role."""
    s = 32768
    plant = planting_for(C1, s)
    case = GpuCase(C1, 2511, batch=1, s_pre=s - 1, max_seq=s + 64, planting=plant)
    out, lse = case.step_graph(s)
    layers = [0, 1, 2, 3, 16, 17, 25, 31]
    ref = oracle_step(C1, 2511, 0, s, layers, plant)
    for l in layers:
        assert_close_bf16(out[l, 0], ref[l][0], f"C1 layer {l}")
        assert np.max(np.abs(lse[l, 0] - ref[l][1])) <= 2e-4
    # Delta selections: known without the oracle, and the GPU's plans equal them
    for dl in C1.delta:
        units = set(synth.planted_units(2511, dl, 0, plant).tolist())
        expect = units | {0, 2046, 2047}                          # sink page + 2 window pages
        assert set(ref[dl][2].tolist()) == expect, f"oracle plan layer {dl}"
        assert set(_gpu_plan(case, dl, 1)[0].tolist()) == expect, f"GPU plan layer {dl}"


# ---------------------------------------------------------------- the other configs at full size

def _gpu_plan(case: GpuCase, layer: int, batch: int):
    cap = case.stack.plan_capacity
    idx = torch.empty((batch, cap), dtype=torch.int32, device="cuda")
    cnt = torch.empty((batch,), dtype=torch.int32, device="cuda")
    case.stack.copy_plan(layer, batch, idx, cnt)
    torch.cuda.synchronize()
    return [idx[b, : int(cnt[b])].cpu().numpy() for b in range(batch)]


def _gpu_keys(case: GpuCase):
    ptr, n = case.stack.workspace_region(0)
    ws = case.stack.workspace
    off = ptr - ws.data_ptr()
    return ws[off: off + n].view(torch.float32).view(case.cfg.max_batch, -1).cpu().numpy()


def _full_size_sampled(shape: Shape, batch: int, s: int, seqs, layers, seed: int):
    """One graph-captured step at the config's full size and batch, in the launch configuration
    bench.py times (its split counts, merge variants and kernels), on iid inputs; sampled
    (sequence, layer) outputs against the oracle (R19; a sparse layer whose governing plan differs
    from the oracle's only near the boundary is checked against the oracle on the GPU's plan,
    R20 iii), the plans of the sampled sequences (R20 iii), and the last Delta layer's unit keys
    within 1e-5 relative of the oracle's exact S_u (R20 ii)."""
    case = GpuCase(shape, seed, batch=batch, s_pre=s - 1, max_seq=s + 32)
    out, lse = case.step_graph(s)
    assert case.stack.get_error() == 0
    keys = _gpu_keys(case)
    plans = {dl: _gpu_plan(case, dl, batch) for dl in shape.delta}
    roles, gov = oracle.validate_tiers(shape.L, shape.F, shape.delta)
    n_units = -(-s // shape.block)
    for b in seqs:
        ref = oracle_step(shape, seed, b, s, layers + [shape.delta[-1]])
        same = {dl: check_plan(plans[dl][b], ref[dl][2], ref[dl][3], s, shape, False) for dl in ref if ref[dl][2] is not None}
        for l in layers:
            o_out, o_lse = ref[l][0], ref[l][1]
            if roles[l] == oracle.ROLE_SPARSE and not same[int(gov[l])]:
                toks = oracle.units_to_tokens(plans[int(gov[l])][b], shape.block, s)
                o_out, o_lse, _ = oracle_layer(shape, seed, l, b, s, tokens=toks)
            assert_close_bf16(out[l, b], o_out, f"layer {l} seq {b}")
            assert np.max(np.abs(lse[l, b] - o_lse)) <= 2e-4, f"lse layer {l} seq {b}"
        o_keys = ref[shape.delta[-1]][3][:n_units]
        g_keys = keys[b, :n_units].astype(np.float64)
        live = o_keys > 1e-30
        rel = np.abs(g_keys - o_keys)[live] / o_keys[live]
        assert rel.max() <= 1e-5, f"unit keys seq {b}: max rel {rel.max():.3g}"
    del case
    torch.cuda.empty_cache()


C2 = Shape(L=28, m=28, g=4, d=128, F=2, delta=[2, 14, 22], k=4096, S=4, Lw=32, block=16, dtype="bf16")
C4 = Shape(L=40, m=40, g=8, d=128, F=2, delta=[2, 6, 35], k=2048, S=4, Lw=32, block=16, dtype="bf16")


def test_c2_full_size_sampled():
    """BASELINE configs[2] per GPU at W=1: Qwen-7B shape, b=32, 16K context, budget 4K (B*g = 128:
    one global-merge split per (sequence, head) on the full-cache layers, cluster kernel sparse)."""
    _full_size_sampled(C2, 32, 16384, seqs=[0, 13, 31], layers=[0, 2, 3, 14, 21, 27], seed=2512)


def test_c4_full_size_sampled():
    """BASELINE configs[4] per GPU: Qwen3-14B shape, 8 sequences at 32K, budget 2K (B*g = 64)."""
    _full_size_sampled(C4, 8, 32768, seqs=[0, 7], layers=[1, 6, 7, 35, 39], seed=2514)


def test_c3_full_size_sampled():
    """BASELINE configs[3] on one GPU: Llama-8B shape at 128K context (8192 pages), budget 2K."""
    _full_size_sampled(C1, 1, 131072, seqs=[0], layers=[0, 2, 3, 25, 26, 31], seed=2513)


# ---------------------------------------------------------------- tcgen05 / TMEM kernel (opt-in)

@pytest.mark.parametrize("shape,s", [
    (Shape(L=4, m=32, g=8, d=128, F=1, delta=[1], k=512, S=4, Lw=32, block=16, dtype="bf16"), 3001),   # gs 4
    (Shape(L=3, m=28, g=4, d=128, F=1, delta=[1], k=1024, S=4, Lw=32, block=16, dtype="bf16"), 2101),  # gs 7
    (Shape(L=3, m=16, g=2, d=64, F=1, delta=[1], k=64, S=4, Lw=32, block=1, dtype="bf16"), 2101),      # d 64, tokens
], ids=["gs4", "gs7", "d64-token"])
def test_umma_kernel_parity(shape, s, monkeypatch):
    """The tcgen05.mma / TMEM decode kernel (attn_umma.cu, DELTA_TUNE umma=1) against the oracle."""
    monkeypatch.setenv("DELTA_TUNE", "umma=1")
    case = GpuCase(shape, 91, batch=2, s_pre=s - 1, max_seq=s + 64)
    out, lse, plans = case.step_layers(s)
    _check_step(case, s, out, lse, plans)


def test_umma_fewhot_epochs(monkeypatch):
    """Concentrated attention arriving late in the cache forces stabiliser raises (new TMEM
    accumulator epochs) in the tcgen05 kernel; the result must still meet the bound."""
    monkeypatch.setenv("DELTA_TUNE", "umma=1")
    sh = Shape(L=2, m=32, g=8, d=128, F=2, delta=[], k=0, S=0, Lw=0, block=16, dtype="bf16")
    plant = planting_for(Shape(L=2, m=32, g=8, d=128, F=2, delta=[], k=0, S=4, Lw=32, block=1, dtype="bf16"),
                         4096, "fewhot")
    case = GpuCase(sh, 8, batch=1, s_pre=4095, max_seq=4096, planting=plant)
    out, lse, plans = case.step_layers(4096)
    _check_step(case, 4096, out, lse, plans)


# ---------------------------------------------------------------- edge cases

def test_first_token_attends_itself():
    """Degenerate case of Eq.4: the first token of an empty cache (fused append, s = 1) has a
    single key, so softmax = 1 and every head's output is exactly its group's new V row; a
    decode on an empty cache without an append is a sticky USAGE error."""
    shape = Shape(L=2, m=32, g=8, d=128, F=2, delta=[], k=512, S=4, Lw=32, block=16, dtype="bf16")
    case = GpuCase(shape, 91, batch=2, s_pre=0, max_seq=64)
    q, k, v = case.inputs(1)
    out = torch.empty((shape.L, 2, shape.m, shape.d), dtype=torch.float32, device="cuda")
    for l in range(shape.L):
        case.stack.append_decode_layer(l, k[l], v[l], q[l], out[l])
    torch.cuda.synchronize()
    assert case.stack.get_error() == 0
    vf = v.float().cpu().numpy()                           # [L][B][g][d]
    gs = shape.m // shape.g
    for l in range(shape.L):
        for b in range(2):
            expect = np.repeat(vf[l, b], gs, axis=0)          # head j reads group j // gs
            np.testing.assert_array_equal(out[l, b].cpu().numpy(), expect)
    empty = GpuCase(shape, 92, batch=1, s_pre=0, max_seq=64)
    q1, _, _ = empty.inputs(1)
    o1 = torch.empty((1, shape.m, shape.d), dtype=torch.float32, device="cuda")
    empty.stack.decode_layer(0, q1[0], o1)
    assert empty.stack.get_error() == 2                       # DELTA_ERR_USAGE


def test_ragged_batch_lengths():
    """R22: sequences of one call at different lengths (one below the budget, so its plan is
    every page (R12), one across a page boundary, one long), each against the oracle."""
    from synth import device as sd
    from helpers import BF16_MAX_ABS  # noqa: F401
    shape = BF16_SMALL
    seed, lens = 93, [300, 2048, 3001]                     # s after this step's append
    case = GpuCase(shape, seed, batch=3, s_pre=max(lens), max_seq=3100)
    case.stack.set_seq_lens([s - 1 for s in lens])
    q = torch.empty((shape.L, 3, shape.m, shape.d), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((shape.L, 3, shape.g, shape.d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    sd.fill_queries(q, seed, range(shape.L), lens)
    sd.fill_new_kv(k, v, seed, range(shape.L), [s - 1 for s in lens])
    out = torch.empty((shape.L, 3, shape.m, shape.d), dtype=torch.float32, device="cuda")
    cap = case.stack.plan_capacity
    idx = torch.empty((3, cap), dtype=torch.int32, device="cuda")
    cnt = torch.empty((3,), dtype=torch.int32, device="cuda")
    for l in range(shape.L):
        case.stack.append_decode_layer(l, k[l], v[l], q[l], out[l])
        if l == 1:
            case.stack.select(1, 3, idx_out=idx, count_out=cnt)
    torch.cuda.synchronize()
    assert case.stack.get_error() == 0
    o = out.cpu().numpy()
    for b, s in enumerate(lens):
        ref = oracle_step(shape, seed, b, s)
        plan = idx[b, : int(cnt[b])].cpu().numpy()
        same = check_plan(plan, ref[1][2], ref[1][3], s, shape, False)
        if s <= shape.k + shape.S + shape.Lw:
            assert plan.tolist() == list(range(-(-s // 16)))   # budget covers the context
        for l in range(shape.L):
            if l >= 2 and not same:
                continue
            assert_close_bf16(o[l, b], ref[l][0], f"layer {l} seq {b} (s={s})")


def test_gs16_two_head_tiles():
    """The largest GQA group (gs = 16: two 8-head MMA tiles per KV group) against the oracle."""
    shape = Shape(L=3, m=32, g=2, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=16, dtype="bf16")
    case = GpuCase(shape, 95, batch=2, s_pre=1500, max_seq=1600)
    out, lse, plans = case.step_layers(1501)
    _check_step(case, 1501, out, lse, plans)


# ---------------------------------------------------------------- numeric error flag

@pytest.mark.parametrize("where", ["sparse_q", "full_q", "select_cache"])
def test_injected_nan_sets_sticky_numeric_error(where):
    """A NaN in a layer's query (SPARSE: the latency kernel; FULL: the global-merge kernel) or in
    a cached key row of the Delta layer makes that layer's outputs NaN, and the graph-captured step
    raises the sticky DELTA_ERR_NUMERIC flag; delta_get_error reads and clears it, and
    the next clean step leaves it clear."""
    shape = Shape(L=4, m=32, g=8, d=128, F=1, delta=[1], k=512, S=4, Lw=32, block=16, dtype="bf16")
    case = GpuCase(shape, 61, batch=1, s_pre=2999, max_seq=3100)
    assert "sparse_lat" in case.stack.kernel_name(3, 1) and "global" in case.stack.kernel_name(0, 1)
    q, k, v = case.inputs(3000)
    if where == "sparse_q":
        q[3, 0, 5, 7] = float("nan")
    elif where == "full_q":
        q[0, 0, 9, 3] = float("nan")
    else:  # layer 1 (Delta), page 10's physical page, head 2, K row 4
        phys = int(case.stack.block_table[0, 10])
        case.stack.kv_pool[1, phys, 2, 0, 4, 11] = float("nan")
    out = torch.empty((4, 1, 32, 128), dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        case.stack.decode_step(q, k, v, out, stream=st)
    st.synchronize()
    assert case.stack.get_error(stream=st) == 3                       # DELTA_ERR_NUMERIC
    bad_layer = {"sparse_q": 3, "full_q": 0, "select_cache": 1}[where]
    assert torch.isnan(out[bad_layer]).any()
    assert case.stack.get_error(stream=st) == 0                       # read clears it
    q2, k2, v2 = case.inputs(3001)
    if where == "select_cache":
        case.stack.kv_pool[1, phys, 2, 0, 4, 11] = 0.0
    with torch.cuda.stream(st):
        case.stack.decode_step(q2, k2, v2, out, stream=st)
    st.synchronize()
    assert case.stack.get_error(stream=st) == 0
    assert not torch.isnan(out).any()


def test_gmerge_ll_flags_across_split_counts_and_protocols():
    """The global split-K merge's LL flags carry the split count and a per-(b, h, split count)
    launch epoch (combine.cuh): launches with different split counts, and the ticket protocol
    (gll = 0) interleaved with LL launches, reuse the same partial slots — a flag that aliased
    across them would let a merge accept another launch's partials.  Each step checks every
    layer against the oracle."""
    sh = Shape(L=2, m=32, g=8, d=128, F=2, delta=[], k=0, S=0, Lw=0, block=16, dtype="bf16")
    case = GpuCase(sh, 41, batch=1, s_pre=3000, max_seq=3100)
    s = 3000
    for tune in [("nsplit", 18), ("nsplit", 12), ("nsplit", 18), ("gll", 0), ("gll", 1), ("nsplit", 7),
                 ("nsplit", 12)]:
        case.stack.set_tuning(*tune)
        s += 1
        out, lse, plans = case.step_layers(s)
        _check_step(case, s, out, lse, plans)


def test_select_ll_keys_do_not_alias_across_delta_layers():
    """Three Delta layers share the select's LL key buffer; their epochs must never coincide
    (one epoch per sequence, not per layer): several steps through the per-layer ABI and the
    captured step, plans checked against the oracle's."""
    sh = Shape(L=6, m=32, g=8, d=128, F=1, delta=[1, 3, 4], k=256, S=4, Lw=32, block=16, dtype="bf16")
    case = GpuCase(sh, 43, batch=2, s_pre=6000, max_seq=6100)
    for s in (6001, 6002, 6003):
        out, lse, plans = case.step_layers(s)
        _check_step(case, s, out, lse, plans)
    for s in (6004, 6005):
        out, lse = case.step_graph(s)
        ref = [oracle_step(sh, case.seed, b, s) for b in range(case.batch)]
        for b in range(case.batch):
            for l in range(sh.L):
                assert_close_bf16(out[l, b], ref[b][l][0], f"graph step s={s} layer {l} seq {b}")


def test_long_graph_run_then_layer_calls_bitwise():
    """Forty graph-replayed steps with a growing context (the LL merge and select flags cycle
    through many launches and leave stale words behind), then the last step again through the
    per-layer ABI from the same state: bitwise equal outputs and LSEs (same kernels, same inputs)."""
    from paper_2510_09883_b200 import ROLE_SELECT
    sh = Shape(L=6, m=32, g=8, d=128, F=1, delta=[1, 4], k=512, S=4, Lw=32, block=16, dtype="bf16")
    n, s0 = 40, 8000
    case = GpuCase(sh, 47, batch=1, s_pre=s0 - 1, max_seq=s0 + n + 16)
    st = case.stack
    stream = torch.cuda.Stream()
    out = torch.empty((sh.L, 1, sh.m, sh.d), dtype=torch.float32, device="cuda")
    lse = torch.empty((sh.L, 1, sh.m), dtype=torch.float32, device="cuda")
    for i in range(n):
        q, k, v = case.inputs(s0 + i)
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            st.decode_step(q, k, v, out, lse, stream=stream)
        stream.synchronize()
    assert st.get_error() == 0
    g_out, g_lse = out.clone(), lse.clone()
    st.set_seq_lens([s0 + n - 2])
    out2, lse2 = torch.empty_like(out), torch.empty_like(lse)
    for l in range(sh.L):
        st.append_decode_layer(l, k[l], v[l], q[l], out2[l], lse2[l])
        if st.role(l) == ROLE_SELECT:
            st.select(l, 1)
    torch.cuda.synchronize()
    assert st.get_error() == 0
    assert torch.equal(g_out, out2) and torch.equal(g_lse, lse2)
