"""Quick A/B timer: device time of the C1 DELTA step (and optionally the Full stack), pure graph
replays on fixed input buffers (one captured graph per stack), CUDA events per step.
usage: python tools/step_time.py [--full] [--steps N]   (DELTA_LIB_PATH / DELTA_TUNE select variants;
PROBE_TUNES="a;b" runs several DELTA_TUNE settings in one process)"""
import argparse
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--config", default="c1", choices=["c1", "c4"])
    a = ap.parse_args()
    ctx = a.ctx
    L, m, g, d, F, delta, B = 32, 32, 8, 128, 2, [2, 16, 25], 1
    if a.config == "c4":  # Qwen3-14B shape, 8 sequences (bench.py c4)
        L, m, g, d, F, delta, B = 40, 40, 8, 128, 2, [2, 6, 35], 8
    mk = lambda sel: d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=B,
                                      max_seq_len=ctx + a.steps + 64, num_full_prefix=F if sel else L,
                                      select_layers=delta if sel else [], budget_k=2048, n_sink=4, n_window=32,
                                      select_block=16)
    cfg = mk(True)
    bt = torch.from_numpy(synth.block_table(7, B, cfg.max_pages))
    base = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(base.kv_pool, base.block_table, 7, ctx - 1, B, range(L))
    q = torch.empty((L, B, m, d), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((L, B, g, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    sd.fill_queries(q, 7, range(L), [ctx] * B)
    sd.fill_new_kv(k, v, 7, range(L), [ctx - 1] * B)
    out = torch.empty((L, B, m, d), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    for tune in os.environ.get("PROBE_TUNES", "auto").split(";"):
        if tune == "auto":
            os.environ.pop("DELTA_TUNE", None)
        else:
            os.environ["DELTA_TUNE"] = tune
        res = {}
        for name, sel in (("delta", True),) + ((("full", False),) if a.full else ()):
            c = mk(sel)
            _, ws = d200.query_sizes(c)
            st = d200.DeltaStack(c, base.kv_pool, base.block_table, torch.zeros(ws, dtype=torch.uint8, device="cuda"))
            st.set_seq_lens([ctx - 1] * B)
            with torch.cuda.stream(s):
                for _ in range(5):
                    st.decode_step(q, k, v, out, stream=s)
            s.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
            with torch.cuda.stream(s):
                ev[0].record(s)
                for i in range(a.steps):
                    st.decode_step(q, k, v, out, stream=s)
                    ev[i + 1].record(s)
            s.synchronize()
            assert st.get_error() == 0
            t = np.array([1e3 * ev[i].elapsed_time(ev[i + 1]) for i in range(a.steps)])
            res[name] = (np.median(t), np.percentile(t, 10), np.percentile(t, 90), t.mean())
            if sel:  # eager select of the first Delta layer, back to back
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s):
                    for _ in range(5):
                        st.select(delta[0], B, stream=s)
                    e0.record(s)
                    for _ in range(50):
                        st.select(delta[0], B, stream=s)
                    e1.record(s)
                s.synchronize()
                print(f"   [{tune}] eager select {1e3 * e0.elapsed_time(e1) / 50:.2f} us", flush=True)
        line = "  ".join(f"{n} p50 {r[0]:7.1f} p10 {r[1]:7.1f} p90 {r[2]:7.1f} mean {r[3]:7.1f} us" for n, r in res.items())
        if "full" in res:
            line += f"  speedup {res['full'][0] / res['delta'][0]:.3f}"
        print(f"[{tune}] {line}", flush=True)


if __name__ == "__main__":
    main()
