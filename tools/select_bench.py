"""Select-kernel microbenchmark at C1 (page mode, 2048 units, k = 128 pages): times, with CUDA
events over back-to-back launches, (a) the full select (phase A scores + phase B top-k) after a
SELECT decode of layer 2, (b) phase B alone through keys_override (one CTA), for each
DELTA_TUNE in SEL_TUNES (';'-separated)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402


def timeit(fn, s, reps=200):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    with torch.cuda.stream(s):
        for _ in range(10):
            fn()
        ev[0].record(s)
        for _ in range(reps):
            fn()
        ev[1].record(s)
    s.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1e3 / reps


def main():
    ctx = int(os.environ.get("SEL_CTX", "32768"))
    L, m, g, d, F, delta = 32, 32, 8, 128, 2, [2, 16, 25]
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                           max_seq_len=ctx + 64, num_full_prefix=F, select_layers=delta, budget_k=2048,
                           n_sink=4, n_window=32, select_block=16)
    bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
    base = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(base.kv_pool, base.block_table, 7, ctx, 1, range(L))
    q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda")
    sd.fill_queries(q, 7, range(L), [ctx])
    out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
    _, ws_bytes = d200.query_sizes(cfg)
    s = torch.cuda.Stream()
    g_ = torch.Generator().manual_seed(3)
    keys = torch.rand((1, cfg.max_pages), generator=g_).mul_(1e-3).cuda()
    for tune in os.environ.get("SEL_TUNES", "auto").split(";"):
        if tune == "auto":
            os.environ.pop("DELTA_TUNE", None)
        else:
            os.environ["DELTA_TUNE"] = tune
        st = d200.DeltaStack(cfg, base.kv_pool, base.block_table,
                             torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda"))
        st.set_seq_lens([ctx])
        with torch.cuda.stream(s):
            st.decode_layer(2, q[2], out[2], stream=s)
        s.synchronize()
        t_full = timeit(lambda: st.select(2, 1, stream=s), s)
        t_b = timeit(lambda: st.select(2, 1, keys_override=keys, stream=s), s)
        assert st.get_error() == 0
        print(f"tune {tune:30s} select (A+B) {t_full:7.2f} us   phase B only {t_b:7.2f} us", flush=True)


if __name__ == "__main__":
    main()
