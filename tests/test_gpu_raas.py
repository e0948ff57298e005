"""GPU parity of the RaaS eviction policy (NEXT-4, readings
RS1-RS4) over a multi-step run against the oracle's per-layer simulation on the same seeded
inputs: every step's attended page set, the page scores (within 1e-5 relative), the eviction
decisions (the oracle replays the GPU's fp32 scores and threshold: exact), and the outputs
(bf16 tolerance); evicted pages never return, sink and recency pages are never evicted.  Beside
the replay, the oracle's OWN fp64 trajectory (its scores, the exact threshold P/|attended|) must
give the identical retained set at every step where no refresh comparison lies within 1e-5 of
the threshold (R20 iii for RaaS); at a near-threshold step it is re-synchronised to the replay."""
import numpy as np
import pytest

import oracle
import synth
from helpers import Shape, assert_close_bf16

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

RA = Shape(L=2, m=32, g=8, d=128, F=1, delta=[], k=128, S=4, Lw=32, block=16, dtype="bf16")


@pytest.mark.parametrize("batch", [1, 2])
def test_raas_multi_step_parity(batch):
    from paper_2510_09883_b200 import POLICY_RAAS, ROLE_RAAS, DeltaStack
    from synth import device as sd
    shape, seed, n0, steps = RA, 81, 700, 24
    cfg = shape.delta_config(batch, n0 + steps + 64)
    cfg.policy = POLICY_RAAS
    bt = torch.from_numpy(synth.block_table(seed, batch, cfg.max_pages))
    st = DeltaStack.allocate(cfg, bt)
    sd.fill_pools(st.kv_pool, st.block_table, seed, n0, batch, range(shape.L))
    st.set_seq_lens([n0] * batch)
    st.raas_reset(-1, batch)
    assert st.role(1) == ROLE_RAAS
    ocfg = shape.oracle_config()
    P = 16
    max_pages = cfg.max_pages
    retained = np.zeros((batch, max_pages), np.uint8)
    retained[:, : -(-n0 // P)] = 1
    last = np.zeros((batch, max_pages), np.int64)
    cap = st.plan_capacity
    idx = torch.empty((batch, cap), dtype=torch.int32, device="cuda")
    cnt = torch.empty((batch,), dtype=torch.int32, device="cuda")
    ptr, nbytes = st.workspace_region(0)
    ws = st.workspace
    keys = ws[ptr - ws.data_ptr(): ptr - ws.data_ptr() + nbytes].view(torch.float32).view(batch, -1)
    evicted_total = [set() for _ in range(batch)]
    own_ret, own_last = retained.copy(), last.copy()   # the oracle's own fp64 trajectory
    own_checked = own_near = 0
    for s in range(n0 + 1, n0 + steps + 1):
        q = torch.empty((shape.L, batch, shape.m, shape.d), dtype=torch.bfloat16, device="cuda")
        k = torch.empty((shape.L, batch, shape.g, shape.d), dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        sd.fill_queries(q, seed, range(shape.L), [s] * batch)
        sd.fill_new_kv(k, v, seed, range(shape.L), [s - 1] * batch)
        out = torch.empty((shape.L, batch, shape.m, shape.d), dtype=torch.float32, device="cuda")
        for l in range(shape.L):
            st.append_decode_layer(l, k[l], v[l], q[l], out[l])
        st.copy_plan(1, batch, idx, cnt)
        torch.cuda.synchronize()
        for b in range(batch):
            g_keys = keys[b].cpu().numpy().astype(np.float64)
            g_plan = idx[b, : int(cnt[b])].cpu().numpy()
            # oracle: the same step on the same rows, replaying the GPU's fp32 scores / threshold
            K = synth.kv_rows(seed, 1, b, 0, s, shape.g, shape.d, "bf16", "k")
            V = synth.kv_rows(seed, 1, b, 0, s, shape.g, shape.d, "bf16", "v")
            kv = oracle.SeqKV.from_contiguous(K, V, P)
            qo = synth.q_rows(seed, 1, b, s, shape.m, shape.d, "bf16")
            n_pages = -(-s // P)
            r_tmp, l_tmp = retained[b].copy(), last[b].copy()
            o_out, _, pages, S, _ = oracle.raas_layer_step(ocfg, kv, qo, s, r_tmp, l_tmp)
            att = pages
            err = np.abs(g_keys[att] - S[att]) / np.maximum(np.abs(S[att]), 1e-30)
            assert err.max() <= 1e-5, f"page scores step {s} seq {b}: {err.max():.3g}"
            assert_close_bf16(out[1, b].cpu().numpy(), o_out, f"raas layer step {s} seq {b}")
            ret_b, last_b = retained[b], last[b]
            ev = oracle.raas_layer_step(ocfg, kv, qo, s, ret_b, last_b, scores_override=g_keys,
                                        threshold=lambda n: float(np.float32(16.0 / n)))[4]
            exp_plan = np.nonzero(ret_b[:n_pages])[0].tolist()
            if s % P == 0:                   # the page position s opens joins for the next step
                ret_b[s // P] = 1
                last_b[s // P] = s + 1
                exp_plan.append(s // P)
            assert g_plan.tolist() == exp_plan, f"retained set step {s} seq {b}: gpu {g_plan.tolist()} oracle {exp_plan}"
            # the oracle's own trajectory: fp64 scores, exact threshold
            o_ret, o_last = own_ret[b], own_last[b]
            _, _, o_pages, o_S, _ = oracle.raas_layer_step(ocfg, kv, qo, s, o_ret, o_last)
            thr = P / oracle.units_to_tokens(o_pages, P, s).size
            margin = np.min(np.abs(o_S[o_pages] - thr)) / thr
            own_plan = np.nonzero(o_ret[:n_pages])[0].tolist()
            if s % P == 0:
                o_ret[s // P] = 1
                o_last[s // P] = s + 1
                own_plan.append(s // P)
            if margin > 1e-5:
                assert own_plan == g_plan.tolist(), f"oracle's own trajectory differs at step {s} seq {b}"
                own_checked += 1
            else:                              # a refresh decision at the fp32/fp64 boundary
                own_near += 1
                own_ret[b], own_last[b] = ret_b.copy(), last_b.copy()
            ex = oracle.raas_exempt(n_pages, s, P, shape.S, shape.Lw)
            assert not any(ex[u] for u in ev), "an exempt page was evicted"
            evicted_total[b] |= set(ev.tolist())
            assert not (evicted_total[b] & set(g_plan.tolist())), "an evicted page came back"
            assert int(sum(1 for u in g_plan if u < n_pages and not ex[u])) <= shape.k // P
    assert st.get_error() == 0
    assert own_checked >= 0.8 * steps * batch, f"own-trajectory checks {own_checked}, near-threshold {own_near}"
    for b in range(batch):                    # the initial set shrank to the budget
        assert len(evicted_total[b]) >= -(-n0 // P) - (shape.k // P) - 4
