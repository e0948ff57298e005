"""RaaS stack at C1: per-step device time of consecutive graph steps after delta_raas_reset
(the first step attends every page and evicts down to the budget), and the retained count."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402


def main():
    ctx, L, m, g, d = 32768, 32, 32, 8, 128
    steps = 8
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                           max_seq_len=ctx + 64, num_full_prefix=2, select_layers=[], budget_k=2048,
                           n_sink=4, n_window=32, select_block=16, policy=d200.POLICY_RAAS)
    bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
    st = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(st.kv_pool, st.block_table, 7, ctx - 1, 1, range(L))
    st.set_seq_lens([ctx - 1])
    st.raas_reset(-1, 1)
    q = torch.empty((steps, L, 1, m, d), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((steps, L, 1, g, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    for i in range(steps):
        sd.fill_queries(q[i], 7, range(L), [ctx + i])
        sd.fill_new_kv(k[i], v[i], 7, range(L), [ctx - 1 + i])
    out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    cap = st.plan_capacity
    idx = torch.empty((1, cap), dtype=torch.int32, device="cuda")
    cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
    for i in range(steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s):
            ev[0].record(s)
            st.decode_step(q[i], k[i], v[i], out, stream=s)
            ev[1].record(s)
            st.copy_plan(5, 1, idx, cnt, stream=s)
        s.synchronize()
        print(f"step {i}: {ev[0].elapsed_time(ev[1]) * 1e3:9.1f} us, layer-5 retained pages {int(cnt[0])}", flush=True)
    print("error", st.get_error())


if __name__ == "__main__":
    main()
