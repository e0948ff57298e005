"""Quest policy at C1 (Llama-8B shape, 32K): one graph step, then 3 eager Quest layers
(append + reps, page keys, top-k, sparse attention) — for an ncu launch list:
  ncu --metrics gpu__time_duration.sum -k regex:'quest|select|append|attn' python tools/quest_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402


def main():
    ctx = 32768
    L, m, g, d = 32, 32, 8, 128
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                           max_seq_len=ctx + 64, num_full_prefix=2, select_layers=[], budget_k=2048,
                           n_sink=4, n_window=32, select_block=16, policy=d200.POLICY_QUEST)
    bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
    st = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(st.kv_pool, st.block_table, 7, ctx - 1, 1, range(L))
    st.set_seq_lens([ctx - 1])
    st.quest_build_reps(-1, 1)
    q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((L, 1, g, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    sd.fill_queries(q, 7, range(L), [ctx])
    sd.fill_new_kv(k, v, 7, range(L), [ctx - 1])
    out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.decode_step(q, k, v, out, stream=s)
        st.set_seq_lens([ctx - 1], stream=s)
        for l in range(5):
            st.append_decode_layer(l, k[l], v[l], q[l], out[l], stream=s)
    s.synchronize()
    assert st.get_error() == 0
    print("quest probe ok")


if __name__ == "__main__":
    main()
