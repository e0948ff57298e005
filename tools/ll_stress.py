"""Long-run check of the LL protocols (gmerge partial flags, select key epochs): N graph-replayed
C1 steps with the context growing, then the last step repeated through the per-layer ABI from
the same state; outputs and LSEs must be bitwise equal (same kernels, same inputs), and no device
error may be raised.  usage: python tools/ll_stress.py [N]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    ctx, L, m, g, d = 32768, 32, 32, 8, 128
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                           max_seq_len=ctx + n + 64, num_full_prefix=2, select_layers=[2, 16, 25], budget_k=2048,
                           n_sink=4, n_window=32, select_block=16)
    bt = torch.from_numpy(synth.block_table(11, 1, cfg.max_pages))
    st = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(st.kv_pool, st.block_table, 11, ctx - 1, 1, range(L))
    st.set_seq_lens([ctx - 1])
    q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((L, 1, g, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
    lse = torch.empty((L, 1, m), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    for i in range(n):
        sd.fill_queries(q, 11 + i, range(L), [ctx + i])
        sd.fill_new_kv(k, v, 11 + i, range(L), [ctx - 1 + i])
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            st.decode_step(q, k, v, out, lse, stream=s)
        s.synchronize()
    assert st.get_error() == 0
    g_out, g_lse = out.clone(), lse.clone()
    # the last step again through the per-layer ABI, from the state before it
    st.set_seq_lens([ctx - 1 + n - 1])
    out2 = torch.empty_like(out)
    lse2 = torch.empty_like(lse)
    with torch.cuda.stream(s):
        for l in range(L):
            st.append_decode_layer(l, k[l], v[l], q[l], out2[l], lse2[l], stream=s)
            if st.role(l) == d200.ROLE_SELECT:
                st.select(l, 1, stream=s)
    s.synchronize()
    assert st.get_error() == 0
    same_o = torch.equal(g_out, out2)
    same_l = torch.equal(g_lse, lse2)
    print(f"{n} graph steps (s = {ctx}..{ctx + n - 1}); last step re-run through the per-layer ABI: "
          f"outputs bitwise equal {same_o}, LSEs bitwise equal {same_l}; "
          f"max |diff| {float((g_out - out2).abs().max()):.3g}", flush=True)
    assert same_o and same_l


if __name__ == "__main__":
    main()
