"""Per-CTA phase-A timing of the select kernel inside a graph step at C1 (trace build):
%globaltimer at entry (0), after griddepcontrol.wait (1) and after the CTA's keys are
published (2), for each Delta layer — min / median / max over the CTAs, us relative to the
earliest wait.  usage: python tools/select_cta_probe.py"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["DELTA_LIB_PATH"] = os.environ.get("PROBE_LIB") or os.path.join(ROOT, "build_trace", "libdelta.so")
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402

lib = d200.load_library()
buf = np.zeros(64 * 512 * 12, np.uint64)


def rd():
    assert lib.delta_trace_read_select(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
    return buf.reshape(64, 512, 12).astype(np.int64).copy()


ctx, L, m, g, d = int(os.environ.get('PROBE_CTX', '32768')), 32, 32, 8, 128
cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1, max_seq_len=ctx + 64,
                       num_full_prefix=2, select_layers=[2, 16, 25], budget_k=2048, n_sink=4, n_window=32,
                       select_block=16)
bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
st = d200.DeltaStack.allocate(cfg, bt)
sd.fill_pools(st.kv_pool, st.block_table, 7, ctx - 1, 1, range(L))
q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda")
k = torch.empty((L, 1, g, d), dtype=torch.bfloat16, device="cuda")
v = torch.empty_like(k)
sd.fill_queries(q, 7, range(L), [ctx])
sd.fill_new_kv(k, v, 7, range(L), [ctx - 1])
out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        st.set_seq_lens([ctx - 1])
        st.decode_step(q, k, v, out, stream=s)
s.synchronize()
rd()
st.set_seq_lens([ctx - 1])
with torch.cuda.stream(s):
    st.decode_step(q, k, v, out, stream=s)
s.synchronize()
t = rd()
for l in (2, 16, 25):
    c = t[l + 32, :, :]
    live = c[:, 1] > 0
    c = c[live]
    w0 = c[:, 1].min()
    f = lambda x: f"{(x.min() - w0) / 1e3:6.2f}/{(np.median(x) - w0) / 1e3:6.2f}/{(x.max() - w0) / 1e3:6.2f}"
    print(f"select L{l}: {live.sum()} CTAs  entry {f(c[:, 0])}  waited {f(c[:, 1])}  keys published {f(c[:, 2][c[:, 2] > 0])}"
          f"  | plan done (CTA 0) {(c[0, 5] - w0) / 1e3:6.2f}   (min/med/max us after the first wait)")
