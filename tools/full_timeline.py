"""Per-layer timeline of a graph-replayed FULL stack (C1 geometry) from the trace build
(make trace): for every layer, CTA entry (min / median), griddepcontrol.wait done, first stage
landed, loop done (median / max) and epilogue done (max), in us from the first CTA entry, and
the gaps between one layer's last loop end and the next layer's first landed stage (HBM idle).
usage: PROBE_TUNES="auto;xm=0" python tools/full_timeline.py"""
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
    ctx, L, m, g, d = 32768, 32, 32, 8, 128
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                           max_seq_len=ctx + 64, num_full_prefix=L, select_layers=[], budget_k=2048,
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
            for i in range(6):
                st.set_seq_lens([ctx - 1])
                if i == 5:
                    ev[0].record(s)
                st.decode_step(q, k, v, out, stream=s)
                if i == 5:
                    ev[1].record(s)
        s.synchronize()
        assert lib.delta_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
        tr = buf.reshape(64, 512, 12).astype(np.int64)[:L].copy()
        t0 = tr[:, :, 0][tr[:, :, 0] > 0].min()
        print(f"########## tune {tune}: step {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us (traced build)")
        print("   layer: entry_min entry_med  wait_med data_min data_med loop_med loop_max  epi_max | idle gap")
        prev_loop_max = None
        gaps = []
        for l in range(L):
            t = tr[l]
            t = t[t[:, 0] > 0]
            f = lambda kk, fn: (fn(t[:, kk][t[:, kk] > 0]) - t0) / 1e3 if (t[:, kk] > 0).any() else float("nan")
            gap = f(2, np.min) - prev_loop_max if prev_loop_max is not None else float("nan")
            if prev_loop_max is not None:
                gaps.append(gap)
            print(f"   L{l:2d}: {f(0, np.min):8.2f} {f(0, np.median):8.2f} {f(1, np.median):8.2f} {f(2, np.min):8.2f} "
                  f"{f(2, np.median):8.2f} {f(3, np.median):8.2f} {f(3, np.max):8.2f} {f(6, np.max):8.2f} | {gap:6.2f}"
                  f" | states {f(10, np.max):8.2f} epi {f(4, np.max):8.2f} stored {f(5, np.max):8.2f} ticket {f(7, np.max):8.2f} staged {f(9, np.max):8.2f}")
            prev_loop_max = f(3, np.max)
        print(f"   median gap (loop_max -> next first data): {np.median(gaps):.2f} us; "
              f"median layer period {np.median(np.diff([ (tr[l][tr[l][:,0]>0][:,3].max()) for l in range(L)]))/1e3:.2f} us")


if __name__ == "__main__":
    main()
