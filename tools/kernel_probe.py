"""Per-role kernel probe at BASELINE configs[1] (C1) for ncu: one graph-captured decode step
(35 launches: 32 decode + 3 select), then 3 eager launches each of FULL (layer 0),
SELECT decode (layer 2), delta_select (layer 2) and SPARSE (layer 3), in that order.
Profile with:  ncu --set full -k regex:'attn|select' --launch-skip 35 -c 12 python tools/kernel_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402


def main():
    ctx = int(os.environ.get("PROBE_CTX", "32768"))
    L, m, g, d, F, delta = 32, 32, 8, 128, 2, [2, 16, 25]
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                           max_seq_len=ctx + 64, num_full_prefix=F, select_layers=delta, budget_k=2048,
                           n_sink=4, n_window=32, select_block=16)
    bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
    st = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(st.kv_pool, st.block_table, 7, ctx - 1, 1, range(L))
    st.set_seq_lens([ctx - 1])
    q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((L, 1, g, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    sd.fill_queries(q, 7, range(L), [ctx])
    sd.fill_new_kv(k, v, 7, range(L), [ctx - 1])
    out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        st.decode_step(q, k, v, out, stream=s)
        for fn in (lambda: st.decode_layer(0, q[0], out[0], stream=s),
                   lambda: st.decode_layer(2, q[2], out[2], stream=s),
                   lambda: st.select(2, 1, stream=s),
                   lambda: st.decode_layer(3, q[3], out[3], stream=s)):
            for _ in range(3):
                fn()
    s.synchronize()
    assert st.get_error() == 0
    print("probe ok")


if __name__ == "__main__":
    main()
