"""Per-warp latency anatomy of the SPARSE latency kernel (attn_sparse.cu) inside a graph step
at C1, from the trace build (make trace): per layer, the median / max over CTAs of
  entry, wait done, q loaded, first tile ready, tiles done, states written, epilogue done
relative to the previous layer's last epilogue-done stamp (or the step's first stamp).
usage: python tools/sparse_probe.py   (PROBE_TUNES="auto;snsplit=16" to compare variants)"""
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
NL, NC, NW, NE = 64, 128, 8, 16
sp = np.zeros(NL * NC * NW * NE, np.uint64)
EV = ["entry", "waited", "q", "tile0", "tiles", "states", "done", "pushed", "owner"]
EVI = [0, 1, 2, 3, 4, 5, 6, 12, 13]


def read_sparse():
    assert lib.delta_trace_read_sparse(sp.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(sp.nbytes)) == 0
    return sp.reshape(NL, NC, NW, NE).astype(np.int64).copy()


def main():
    ctx = int(os.environ.get("PROBE_CTX", "32768"))
    L, m, g, d, F, delta = 32, 32, 8, 128, 2, [2, 16, 25]
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                           max_seq_len=ctx + 64, num_full_prefix=F, select_layers=delta, budget_k=2048,
                           n_sink=4, n_window=32, select_block=16)
    bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
    base = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(base.kv_pool, base.block_table, 7, ctx - 1, 1, range(L))
    q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((L, 1, g, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    sd.fill_queries(q, 7, range(L), [ctx])
    sd.fill_new_kv(k, v, 7, range(L), [ctx - 1])
    out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    _, ws_bytes = d200.query_sizes(cfg)
    for tune in os.environ.get("PROBE_TUNES", "auto").split(";"):
        if tune == "auto":
            os.environ.pop("DELTA_TUNE", None)
        else:
            os.environ["DELTA_TUNE"] = tune
        st = d200.DeltaStack(cfg, base.kv_pool, base.block_table,
                             torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda"))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s):
            for _ in range(3):
                st.set_seq_lens([ctx - 1])
                st.decode_step(q, k, v, out, stream=s)
            s.synchronize()
            read_sparse()
            st.set_seq_lens([ctx - 1])
            ev[0].record(s)
            st.decode_step(q, k, v, out, stream=s)
            ev[1].record(s)
        s.synchronize()
        tr = read_sparse()
        assert st.get_error() == 0
        print(f"########## tune: {tune}   step {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us (trace build)")
        print("   layer  ncta  " + "  ".join(f"{e:>13s}" for e in EV) + "   (us after prev layer done: med/max)")
        prev_done = None
        clk = []
        for l in range(L):
            t = tr[l]
            live = t[:, 0, 0] > 0
            if not live.any():
                prev_done = None
                continue
            t = t[live]  # [cta][warp][ev]
            ref = prev_done if prev_done is not None else t[:, 0, 0].min()
            cols = []
            for e in EVI:
                w = t[:, :, e][t[:, :, e] > 0]
                cols.append(f"{(np.median(w) - ref) / 1e3:6.2f}/{(w.max() - ref) / 1e3:6.2f}" if w.size else " " * 13)
            print(f"   L{l:2d}   {int(live.sum()):4d}  " + "  ".join(cols))
            prev_done = t[:, :, 6][t[:, :, 6] > 0].max()
            c = t[:, 0][:, [7, 8, 9, 10, 11, 14, 15]]  # warp 0 of each CTA
            ok = (c > 0).all(axis=1)
            if ok.any():
                clk.append(np.diff(c[ok], axis=1))
        if clk:
            dc = np.concatenate(clk)
            print("   warp-0 epilogue cycles (med / p90 / max):  " + "  ".join(
                f"{n} {np.median(dc[:, i]):.0f}/{np.percentile(dc[:, i], 90):.0f}/{dc[:, i].max():.0f}"
                for i, n in enumerate(["bar1", "states+bar2", "fold+push", "owner_wait", "merge", "tail"])))


if __name__ == "__main__":
    main()
