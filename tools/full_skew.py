"""Is the FULL-layer loop skew systematic?  Trace build (make trace), Full stack at C1, graph
replays: per CTA the loop-done stamp (slot 3) relative to its layer's first data (slot 2 min),
and the SM it ran on; then per split index and per SM the mean lateness behind the layer median,
and how consistent it is between the two halves of the layers (correlation).  A systematic skew
(same SMs / splits late in every layer) could be rebalanced statically; a random one cannot.
usage: python tools/full_skew.py"""
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


def main():
    lib = d200.load_library()
    buf = np.zeros(64 * 512 * 12, np.uint64)
    sm = np.zeros(64 * 512, np.uint32)
    ctx, L, m, g, d = 32768, 32, 32, 8, 128
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                           max_seq_len=ctx + 64, num_full_prefix=L, select_layers=[], budget_k=2048,
                           n_sink=4, n_window=32, select_block=16)
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
    late_all, ent, dat, dur = [], [], [], []
    for rep in range(4):
        with torch.cuda.stream(s):
            st.set_seq_lens([ctx - 1])
            st.decode_step(q, k, v, out, stream=s)
        s.synchronize()
        assert lib.delta_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
        assert lib.delta_trace_read_smid(sm.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(sm.nbytes)) == 0
        if rep == 0:
            continue
        tr = buf.reshape(64, 512, 12).astype(np.int64)[:L]
        sid = sm.reshape(64, 512)[:L]
        for l in range(1, L):
            t = tr[l, :144]
            if not (t[:, 3] > 0).all():
                continue
            done = (t[:, 3] - np.median(t[:, 3])) / 1e3
            late_all.append((l, done, sid[l, :144].copy()))
            ent.append((t[:, 0] - np.median(t[:, 0])) / 1e3)
            dat.append((t[:, 2] - np.median(t[:, 2])) / 1e3)
            dur.append((t[:, 3] - t[:, 2]) / 1e3)
    per_split = np.array([d_ for _, d_, _ in late_all])  # [layers][cta]
    half = len(per_split) // 2
    a, b = per_split[:half].mean(0), per_split[half:].mean(0)
    print(f"{len(per_split)} layer samples; loop-done lateness per CTA (us behind the layer median): "
          f"mean of max {per_split.max(1).mean():.2f}, p90 {np.percentile(per_split, 90):.2f}")
    print(f"per CTA index: corr(first half, second half) = {np.corrcoef(a, b)[0, 1]:.3f}; "
          f"slowest CTAs (index: mean us): " +
          ", ".join(f"{i}:{a[i] / 2 + b[i] / 2:.2f}" for i in np.argsort(-(a + b))[:10]))
    E, Dt, U = np.array(ent).mean(0), np.array(dat).mean(0), np.array(dur).mean(0)
    print("per head (18 CTAs each): entry / first data (us vs median) / loop duration (us):")
    for h in range(8):
        sl = slice(18 * h, 18 * h + 18)
        print(f"   head {h}: entry {E[sl].mean():6.2f}  data {Dt[sl].mean():6.2f}  loop {U[sl].mean():6.2f}  late {per_split[:, sl].mean():6.2f}")
    by_sm = {}
    for _, d_, s_ in late_all:
        for x, y in zip(s_, d_):
            by_sm.setdefault(int(x), []).append(y)
    sm_mean = {k_: np.mean(v_) for k_, v_ in by_sm.items()}
    worst = sorted(sm_mean.items(), key=lambda kv: -kv[1])[:12]
    print("per SM mean lateness (worst 12): " + ", ".join(f"sm{k_}:{v_:.2f}" for k_, v_ in worst))
    tpc = {}
    for k_, v_ in sm_mean.items():
        tpc.setdefault(k_ // 2, []).append(v_)
    print("SMs used per layer:", len(set(late_all[0][2].tolist())), "| TPCs with both SMs used:",
          sum(1 for v_ in tpc.values() if len(v_) == 2))


if __name__ == "__main__":
    main()
