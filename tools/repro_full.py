"""Repro: an all-FULL stack (bench's Full baseline) stepped through the CUDA graph."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402

L = int(os.environ.get("REPRO_L", "4"))
ctx = int(os.environ.get("REPRO_CTX", "32768"))
full = int(os.environ.get("REPRO_FULL", "1"))
m, g, d = 32, 8, 128
cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1, max_seq_len=ctx + 64,
                       num_full_prefix=L if full else 1, select_layers=[] if full else [1], budget_k=2048,
                       n_sink=4, n_window=32, select_block=16)
bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
st = d200.DeltaStack.allocate(cfg, bt)
sd.fill_pools(st.kv_pool, st.block_table, 7, ctx - 8, 1, range(L))
st.set_seq_lens([ctx - 8])
q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda")
k = torch.empty((L, 1, g, d), dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
sd.fill_queries(q, 7, range(L), [ctx])
sd.fill_new_kv(k, v, 7, range(L), [ctx - 1])
out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for i in range(int(os.environ.get("REPRO_STEPS", "4"))):
        st.decode_step(q, k, v, out, stream=s)
        s.synchronize()
        print("step", i, "ok", flush=True)
print("err", st.get_error())
