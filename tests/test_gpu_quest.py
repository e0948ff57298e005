"""GPU parity of the Quest policy (NEXT-1, readings Q1-Q3) against
the fp64 oracle on the same seeded synthetic inputs:
  * page representatives (min/max of bf16 keys) are bit-exact, both rebuilt from the pool and
    maintained by appends across a page boundary;
  * page keys within 1e-5 (relative to max(1, |key|)) of the oracle's exact fp64 keys;
  * the plan equals the oracle's selection on the GPU's own fp32 keys exactly (R20 i), and the
    oracle's own plan whenever its boundary gap exceeds 1e-4 (R20 iii);
  * outputs within the bf16 tolerance of the oracle's attention over tokens(plan) (R19)."""
import numpy as np
import pytest

import oracle
import synth
from helpers import Shape, assert_close_bf16

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

QUEST_SMALL = Shape(L=3, m=32, g=8, d=128, F=1, delta=[], k=512, S=4, Lw=32, block=16, dtype="bf16")
QUEST_GQA = Shape(L=2, m=28, g=4, d=128, F=1, delta=[], k=256, S=4, Lw=32, block=16, dtype="bf16")
QUEST_D64 = Shape(L=2, m=16, g=2, d=64, F=0, delta=[], k=128, S=4, Lw=32, block=16, dtype="bf16")


class QuestCase:
    def __init__(self, shape: Shape, seed: int, batch: int, s_pre: int, max_seq: int):
        from paper_2510_09883_b200 import POLICY_QUEST, DeltaStack
        from synth import device as sd
        self.shape, self.seed, self.batch = shape, seed, batch
        self.cfg = shape.delta_config(batch, max_seq)
        self.cfg.policy = POLICY_QUEST
        bt = torch.from_numpy(synth.block_table(seed, batch, self.cfg.max_pages))
        self.stack = DeltaStack.allocate(self.cfg, bt)
        sd.fill_pools(self.stack.kv_pool, self.stack.block_table, seed, s_pre, batch, range(shape.L))
        self.stack.set_seq_lens([s_pre] * batch)
        self.stack.quest_build_reps(-1, batch)
        self.bt = self.stack.block_table.cpu().numpy()

    def reps(self):
        """[L][phys][g][2][d] float32 view of the library's representatives."""
        ptr, n = self.stack.workspace_region(1)
        ws = self.stack.workspace
        off = ptr - ws.data_ptr()
        c = self.cfg
        r = ws[off: off + n].view(torch.bfloat16).view(c.num_layers, c.phys_pages, c.num_kv_heads, 2, c.head_dim)
        return r.float().cpu().numpy()

    def keys(self):
        ptr, n = self.stack.workspace_region(0)
        ws = self.stack.workspace
        off = ptr - ws.data_ptr()
        return ws[off: off + n].view(torch.float32).view(self.cfg.max_batch, -1).clone()

    def inputs(self, s):
        from synth import device as sd
        sh, B = self.shape, self.batch
        q = torch.empty((sh.L, B, sh.m, sh.d), dtype=torch.bfloat16, device="cuda")
        k = torch.empty((sh.L, B, sh.g, sh.d), dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        sd.fill_queries(q, self.seed, range(sh.L), [s] * B)
        sd.fill_new_kv(k, v, self.seed, range(sh.L), [s - 1] * B)
        return q, k, v

    def step(self, s):
        """Per-layer calls; after each Quest layer copy its keys and plan."""
        from paper_2510_09883_b200 import ROLE_QUEST
        sh, B = self.shape, self.batch
        q, k, v = self.inputs(s)
        out = torch.empty((sh.L, B, sh.m, sh.d), dtype=torch.float32, device="cuda")
        lse = torch.empty((sh.L, B, sh.m), dtype=torch.float32, device="cuda")
        cap = self.stack.plan_capacity
        plans, keys = {}, {}
        for l in range(sh.L):
            self.stack.append_decode_layer(l, k[l], v[l], q[l], out[l], lse[l])
            if self.stack.role(l) == ROLE_QUEST:
                idx = torch.empty((B, cap), dtype=torch.int32, device="cuda")
                cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
                self.stack.copy_plan(l, B, idx, cnt)
                keys[l] = self.keys()
                plans[l] = (idx, cnt)
        torch.cuda.synchronize()
        assert self.stack.get_error() == 0
        hp = {l: [idx[b, : int(cnt[b])].cpu().numpy() for b in range(B)] for l, (idx, cnt) in plans.items()}
        hk = {l: kk.cpu().numpy() for l, kk in keys.items()}
        return out.cpu().numpy(), lse.cpu().numpy(), hp, hk

    def oracle_kv(self, l, b, s):
        sh = self.shape
        K = synth.kv_rows(self.seed, l, b, 0, s, sh.g, sh.d, sh.dtype, "k")
        V = synth.kv_rows(self.seed, l, b, 0, s, sh.g, sh.d, sh.dtype, "v")
        return oracle.SeqKV.from_contiguous(K, V, 16)


def _check_reps(case: QuestCase, s: int):
    reps = case.reps()
    sh = case.shape
    for l in range(sh.F, sh.L):
        for b in range(case.batch):
            ref = oracle.quest_reps(case.oracle_kv(l, b, s), s)     # [pages][g][2][d]
            got = reps[l, case.bt[b, : ref.shape[0]]]                # physical pages of the sequence
            assert np.array_equal(got, ref.astype(np.float32)), f"reps layer {l} seq {b}"


def _check_layer(case: QuestCase, s: int, out, lse, plans, keys):
    sh = case.shape
    ocfg = sh.oracle_config()
    n_pages = -(-s // 16)
    for l in range(sh.F, sh.L):
        for b in range(case.batch):
            kv = case.oracle_kv(l, b, s)
            q = synth.q_rows(case.seed, l, b, s, sh.m, sh.d, sh.dtype)
            o_out, o_lse, o_keys, o_units, _ = oracle.quest_layer(ocfg, kv, q, s)
            g_keys = keys[l][b, :n_pages].astype(np.float64)
            g_units = plans[l][b]
            cand = np.ones(n_pages, bool)
            cand[: (sh.S - 1) // 16 + 1] = False
            cand[max(0, s - sh.Lw) // 16:] = False
            err = np.abs(g_keys - o_keys)[cand] / np.maximum(1.0, np.abs(o_keys[cand]))
            assert err.max() <= 1e-5, f"page keys layer {l} seq {b}: {err.max():.3g}"
            # R20 (i): the plan is exactly the selection rule applied to the GPU's own keys
            host = oracle.select(g_keys, s, 16, sh.S, sh.Lw, sh.k // 16)
            assert np.array_equal(g_units, host), f"plan != top-k of the GPU keys, layer {l} seq {b}"
            # R20 (iii): equal to the oracle's plan unless its boundary is a near tie
            srt = np.sort(o_keys[cand])[::-1]
            kk = sh.k // 16
            if srt.size > kk:
                gap = (srt[kk - 1] - srt[kk]) / max(1.0, abs(srt[kk - 1]))
                if gap > 1e-4:
                    assert np.array_equal(g_units, o_units), f"plan vs oracle layer {l} seq {b} (gap {gap:.3g})"
            # attention over tokens(the GPU plan)
            toks = oracle.units_to_tokens(g_units, 16, s)
            r_out, r_lse, _ = oracle.decode_heads(q, kv, toks, ocfg.scale)
            assert_close_bf16(out[l, b], r_out, f"quest layer {l} seq {b}")
            assert np.max(np.abs(lse[l, b] - r_lse)) <= 2e-4


@pytest.mark.parametrize("shape,s", [(QUEST_SMALL, 3001), (QUEST_GQA, 2101), (QUEST_D64, 777)],
                         ids=["m32g8", "gs7", "d64"])
def test_quest_step_parity(shape, s):
    case = QuestCase(shape, 41, batch=2, s_pre=s - 1, max_seq=s + 64)
    _check_reps(case, s - 1)
    out, lse, plans, keys = case.step(s)
    _check_reps(case, s)
    _check_layer(case, s, out, lse, plans, keys)
    # FULL prefix layers are plain full attention
    for l in range(shape.F):
        for b in range(case.batch):
            kv = case.oracle_kv(l, b, s)
            q = synth.q_rows(case.seed, l, b, s, shape.m, shape.d, shape.dtype)
            r_out, _, _ = oracle.decode_heads(q, kv, s, shape.oracle_config().scale)
            assert_close_bf16(out[l, b], r_out, f"full layer {l}")


def test_quest_reps_maintained_across_page_boundary():
    """Appends 4094 -> 4100 cross the page boundary at 4096: the incrementally maintained reps
    equal the oracle's (a page's first token restarts its min/max)."""
    case = QuestCase(QUEST_SMALL, 43, batch=1, s_pre=4093, max_seq=4160)
    for s in range(4094, 4101):
        out, lse, plans, keys = case.step(s)
        _check_reps(case, s)
    _check_layer(case, 4100, out, lse, plans, keys)


def test_quest_graph_step_equals_per_layer():
    a = QuestCase(QUEST_SMALL, 47, batch=2, s_pre=2999, max_seq=3064)
    b = QuestCase(QUEST_SMALL, 47, batch=2, s_pre=2999, max_seq=3064)
    out_a, lse_a, _, _ = a.step(3000)
    q, k, v = b.inputs(3000)
    out = torch.empty((3, 2, 32, 128), dtype=torch.float32, device="cuda")
    lse = torch.empty((3, 2, 32), dtype=torch.float32, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        b.stack.decode_step(q, k, v, out, lse, stream=st)
    st.synchronize()
    assert np.array_equal(out.cpu().numpy(), out_a) and np.array_equal(lse.cpu().numpy(), lse_a)


def test_quest_budget_covering_context_is_full_attention():
    """R12 with Quest: budget >= context -> every page -> the outputs of full attention."""
    shape = Shape(L=2, m=32, g=8, d=128, F=0, delta=[], k=4096, S=4, Lw=32, block=16, dtype="bf16")
    case = QuestCase(shape, 49, batch=1, s_pre=1999, max_seq=2048)
    out, lse, plans, _ = case.step(2000)
    for l in range(2):
        assert plans[l][0].tolist() == list(range(125))
        kv = case.oracle_kv(l, 0, 2000)
        q = synth.q_rows(case.seed, l, 0, 2000, shape.m, shape.d, shape.dtype)
        r_out, _, _ = oracle.decode_heads(q, kv, 2000, shape.oracle_config().scale)
        assert_close_bf16(out[l, 0], r_out)


def test_quest_config_errors():
    from paper_2510_09883_b200 import POLICY_QUEST, DeltaError, query_sizes
    cfg = QUEST_SMALL.delta_config(1, 1024)
    cfg.policy = POLICY_QUEST
    cfg.select_layers = [1]
    with pytest.raises(DeltaError):
        query_sizes(cfg)
    cfg.select_layers = []
    cfg.select_block = 1
    with pytest.raises(DeltaError):
        query_sizes(cfg)


def test_quest_reps_after_prefill_chunk():
    """A chunk appended by delta_prefill (multi-CTA append: 4 pages per CTA) folds every token
    into its page's min/max: reps bit-exact with the oracle, and the next Quest decode step
    matches the oracle."""
    shape, seed, n0, ntok = QUEST_SMALL, 53, 1000, 300
    case = QuestCase(shape, seed, batch=2, s_pre=n0, max_seq=n0 + ntok + 64)
    for l in range(shape.L):
        q = np.stack([np.stack([synth.q_rows(seed, l, b, n0 + i + 1, shape.m, shape.d, "bf16")
                                for i in range(ntok)]) for b in range(2)])
        kn = np.stack([synth.kv_rows(seed, l, b, n0, n0 + ntok, shape.g, shape.d, "bf16", "k") for b in range(2)])
        vn = np.stack([synth.kv_rows(seed, l, b, n0, n0 + ntok, shape.g, shape.d, "bf16", "v") for b in range(2)])
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).cuda()  # noqa: E731
        out = torch.empty((2, ntok, shape.m, shape.d), dtype=torch.float32, device="cuda")
        case.stack.prefill(l, to(q), to(kn), to(vn), out)
    torch.cuda.synchronize()
    _check_reps(case, n0 + ntok)
    s = n0 + ntok + 1
    out, lse, plans, keys = case.step(s)
    _check_reps(case, s)
    _check_layer(case, s, out, lse, plans, keys)


def test_quest_append_then_decode_scores_the_new_pages():
    """delta_append_kv of more tokens than the window, then an immediate Quest
    delta_decode_layer (no fused append).  The score kernel must read the length counter and the
    representatives after the append completed (no pre-wait reads outside a captured step): every
    page the append opened gets its exact key, and plan and outputs match the oracle."""
    shape, seed, n0, ntok = QUEST_SMALL, 59, 2000, 100   # 100 > n_window = 32: new non-window pages
    case = QuestCase(shape, seed, batch=1, s_pre=n0, max_seq=n0 + ntok + 64)
    s = n0 + ntok
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).cuda()  # noqa: E731
    out = torch.empty((shape.L, 1, shape.m, shape.d), dtype=torch.float32, device="cuda")
    lse = torch.empty((shape.L, 1, shape.m), dtype=torch.float32, device="cuda")
    cap = case.stack.plan_capacity
    plans, keys = {}, {}
    for l in range(shape.L):
        kn = synth.kv_rows(seed, l, 0, n0, s, shape.g, shape.d, "bf16", "k")[None]
        vn = synth.kv_rows(seed, l, 0, n0, s, shape.g, shape.d, "bf16", "v")[None]
        case.stack.append_kv(l, to(kn), to(vn))
        q = to(synth.q_rows(seed, l, 0, s, shape.m, shape.d, "bf16")[None])
        case.stack.decode_layer(l, q, out[l], lse[l])
        if l >= shape.F:
            idx = torch.empty((1, cap), dtype=torch.int32, device="cuda")
            cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
            case.stack.copy_plan(l, 1, idx, cnt)
            keys[l] = case.keys()
            plans[l] = (idx, cnt)
    torch.cuda.synchronize()
    assert case.stack.get_error() == 0
    hp = {l: [idx[0, : int(cnt[0])].cpu().numpy()] for l, (idx, cnt) in plans.items()}
    hk = {l: kk.cpu().numpy() for l, kk in keys.items()}
    _check_reps(case, s)
    _check_layer(case, s, out.cpu().numpy(), lse.cpu().numpy(), hp, hk)
