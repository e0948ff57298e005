"""How fast can the FULL-layer consumers go when the KV is L2-resident?  Eager back-to-back
decode_layer launches of ONE layer (its pages stay in the 126 MB L2 when they fit) against
launches cycling over all layers (HBM-fed), at several contexts.  Effective TB/s = algorithmic
KV bytes / launch time.  usage: python tools/l2_rate_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402


def main():
    L, m, g, d = 32, 32, 8, 128
    for ctx in [int(x) for x in os.environ.get("PROBE_CTXS", "4096,8192,16384,32768").split(",")]:
        cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                               max_seq_len=ctx + 64, num_full_prefix=L, select_layers=[], budget_k=2048,
                               n_sink=4, n_window=32, select_block=16)
        bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
        st = d200.DeltaStack.allocate(cfg, bt)
        sd.fill_pools(st.kv_pool, st.block_table, 7, ctx, 1, range(L))
        st.set_seq_lens([ctx])
        q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda")
        sd.fill_queries(q, 7, range(L), [ctx])
        out = torch.empty((1, m, d), dtype=torch.float32, device="cuda")
        s = torch.cuda.Stream()
        byt = ctx * g * d * 2 * 2
        res = {}
        for name, layers in (("same", [0] * 64), ("cycle", list(range(L)) * 2)):
            with torch.cuda.stream(s):
                for l in layers[:8]:
                    st.decode_layer(l, q[l], out, stream=s)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for l in layers:
                    st.decode_layer(l, q[l], out, stream=s)
                e1.record(s)
            s.synchronize()
            us = 1e3 * e0.elapsed_time(e1) / len(layers)
            res[name] = (us, byt / us / 1e6)
        assert st.get_error() == 0
        print(f"ctx {ctx:6d} ({byt / 1e6:6.1f} MB/layer): same-layer {res['same'][0]:7.2f} us {res['same'][1]:6.2f} TB/s"
              f" | cycling {res['cycle'][0]:7.2f} us {res['cycle'][1]:6.2f} TB/s", flush=True)
        st.close()


if __name__ == "__main__":
    main()
