import ctypes, os, sys
sys.argv = ["x"]
os.environ["DELTA_LIB_PATH"] = "build_trace/libdelta.so"
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2510_09883_b200 as d200, synth
from synth import device as sd
lib = d200.load_library()
buf = np.zeros(64 * 160 * 16 * 8, np.int64)
def rd():
    assert lib.delta_trace_read_select_clk(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
    return buf.reshape(64, 160, 16, 8).copy()
ctx = 32768
L, m, g, d = 32, 32, 8, 128
cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1, max_seq_len=ctx + 64,
                       num_full_prefix=2, select_layers=[2, 16, 25], budget_k=2048, n_sink=4, n_window=32, select_block=16)
bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
st = d200.DeltaStack.allocate(cfg, bt)
sd.fill_pools(st.kv_pool, st.block_table, 7, ctx - 1, 1, range(L))
q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda"); k = torch.empty((L, 1, g, d), dtype=torch.bfloat16, device="cuda"); v = torch.empty_like(k)
sd.fill_queries(q, 7, range(L), [ctx]); sd.fill_new_kv(k, v, 7, range(L), [ctx - 1])
out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        st.set_seq_lens([ctx - 1]); st.decode_step(q, k, v, out, stream=s)
s.synchronize(); rd()
st.set_seq_lens([ctx - 1])
with torch.cuda.stream(s):
    st.decode_step(q, k, v, out, stream=s)
s.synchronize()
t = rd()
for l in (2, 16, 25):
    c = t[l + 32][:129, :16, :6] if (t[l + 32] != 0).any() else t[l][:129, :16, :6]
    ok = (c[:, :, 0] > 0) & (c[:, :, 5] > 0)
    dc = np.diff(c[ok].astype(np.float64), axis=1)
    print(f"L{l}: warps {ok.sum()}  cycles med/p90/max: " + "  ".join(f"{n} {np.median(dc[:, i]):.0f}/{np.percentile(dc[:, i], 90):.0f}/{dc[:, i].max():.0f}" for i, n in enumerate(["seqlen", "lse+logits+max", "exp+sum+store", "to_bar", "bar+atomic+bar"])))
