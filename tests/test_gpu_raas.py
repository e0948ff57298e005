"""GPU parity of the RaaS eviction policy (NEXT-4, readings
RS1-RS4) over a multi-step run against the oracle's per-layer simulation on the same seeded
inputs: every step's attended page set, the page scores (within 1e-5 relative), the eviction
decisions (the oracle replays the GPU's fp32 scores and threshold: exact), and the outputs
(bf16 tolerance); evicted pages never return, sink and recency pages are never evicted."""
import numpy as np
import pytest

import oracle
import synth
from helpers import Shape, assert_close_bf16

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

RA = Shape(L=2, m=32, g=8, d=128, F=1, delta=[], k=128, S=4, Lw=32, block=16, dtype="bf16")


def test_raas_multi_step_parity():
    from paper_2510_09883_b200 import POLICY_RAAS, ROLE_RAAS, DeltaStack
    from synth import device as sd
    shape, seed, n0, steps = RA, 81, 700, 24
    cfg = shape.delta_config(1, n0 + steps + 64)
    cfg.policy = POLICY_RAAS
    bt = torch.from_numpy(synth.block_table(seed, 1, cfg.max_pages))
    st = DeltaStack.allocate(cfg, bt)
    sd.fill_pools(st.kv_pool, st.block_table, seed, n0, 1, range(shape.L))
    st.set_seq_lens([n0])
    st.raas_reset(-1, 1)
    assert st.role(1) == ROLE_RAAS
    ocfg = shape.oracle_config()
    P = 16
    max_pages = cfg.max_pages
    retained = np.zeros(max_pages, np.uint8)
    retained[: -(-n0 // P)] = 1
    last = np.zeros(max_pages, np.int64)
    cap = st.plan_capacity
    idx = torch.empty((1, cap), dtype=torch.int32, device="cuda")
    cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
    ptr, nbytes = st.workspace_region(0)
    ws = st.workspace
    keys = ws[ptr - ws.data_ptr(): ptr - ws.data_ptr() + nbytes].view(torch.float32).view(1, -1)
    evicted_total = set()
    for s in range(n0 + 1, n0 + steps + 1):
        q = torch.empty((shape.L, 1, shape.m, shape.d), dtype=torch.bfloat16, device="cuda")
        k = torch.empty((shape.L, 1, shape.g, shape.d), dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        sd.fill_queries(q, seed, range(shape.L), [s])
        sd.fill_new_kv(k, v, seed, range(shape.L), [s - 1])
        out = torch.empty((shape.L, 1, shape.m, shape.d), dtype=torch.float32, device="cuda")
        for l in range(shape.L):
            st.append_decode_layer(l, k[l], v[l], q[l], out[l])
        st.copy_plan(1, 1, idx, cnt)
        torch.cuda.synchronize()
        g_keys = keys[0].cpu().numpy().astype(np.float64)
        g_plan = idx[0, : int(cnt[0])].cpu().numpy()
        # oracle: the same step on the same rows, replaying the GPU's fp32 scores / threshold
        K = synth.kv_rows(seed, 1, 0, 0, s, shape.g, shape.d, "bf16", "k")
        V = synth.kv_rows(seed, 1, 0, 0, s, shape.g, shape.d, "bf16", "v")
        kv = oracle.SeqKV.from_contiguous(K, V, P)
        qo = synth.q_rows(seed, 1, 0, s, shape.m, shape.d, "bf16")
        ret_before = retained.copy()
        n_pages = -(-s // P)
        # scores of the oracle itself (before replay): compare with the GPU's
        r_tmp, l_tmp = retained.copy(), last.copy()
        o_out, _, pages, S, _ = oracle.raas_layer_step(ocfg, kv, qo, s, r_tmp, l_tmp)
        att = pages
        err = np.abs(g_keys[att] - S[att]) / np.maximum(np.abs(S[att]), 1e-30)
        assert err.max() <= 1e-5, f"page scores step {s}: {err.max():.3g}"
        assert_close_bf16(out[1, 0].cpu().numpy(), o_out, f"raas layer step {s}")
        # replay with the GPU's scores and fp32 threshold: identical eviction decisions
        ev = oracle.raas_layer_step(ocfg, kv, qo, s, retained, last, scores_override=g_keys,
                                    threshold=lambda n: float(np.float32(16.0 / n)))[4]
        exp_plan = np.nonzero(retained[:n_pages])[0].tolist()
        if s % P == 0:                       # the page position s opens joins for the next step
            retained[s // P] = 1
            last[s // P] = s + 1
            exp_plan.append(s // P)
        assert g_plan.tolist() == exp_plan, f"retained set step {s}: gpu {g_plan.tolist()} oracle {exp_plan}"
        ex = oracle.raas_exempt(n_pages, s, P, shape.S, shape.Lw)
        assert not any(ex[u] for u in ev), "an exempt page was evicted"
        evicted_total |= set(ev.tolist())
        assert not (evicted_total & set(g_plan.tolist())), "an evicted page came back"
        assert int(sum(1 for u in g_plan if u < n_pages and not ex[u])) <= shape.k // P
    assert st.get_error() == 0
    assert len(evicted_total) >= -(-n0 // P) - (shape.k // P) - 4   # the initial set shrank to the budget
