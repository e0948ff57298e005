"""Prefill throughput (NEXT-3) at the Llama-8B shape (32q/8kv, d = 128, bf16), one layer:
a chunk of NTOK tokens appended to a cache of N0 tokens, CUDA events over REPS calls (the
length counter is reset between calls, so every call attends the same causal triangle).
FLOPs = 4 d m sum_i (N0 + i + 1)  (QK^T and PV, 2 flops per multiply-add)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402


def run(n0, ntok, batch=1, reps=10):
    m, g, d = 32, 8, 128
    cfg = d200.DeltaConfig(num_layers=1, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=batch,
                           max_seq_len=n0 + ntok + 16, num_full_prefix=1, select_layers=[])
    bt = torch.from_numpy(synth.block_table(5, batch, cfg.max_pages))
    st = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(st.kv_pool, st.block_table, 5, n0, batch, range(1))
    q = torch.randn((batch, ntok, m, d), device="cuda").to(torch.bfloat16)
    k = torch.randn((batch, ntok, g, d), device="cuda").to(torch.bfloat16)
    v = torch.randn_like(k)
    out = torch.empty((batch, ntok, m, d), dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()  # inputs were generated on the default stream
    s = torch.cuda.Stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    times = []
    for r in range(reps + 2):
        st.set_seq_lens([n0] * batch, stream=s)
        with torch.cuda.stream(s):
            ev[0].record(s)
            st.prefill(0, q, k, v, out, stream=s)
            ev[1].record(s)
        s.synchronize()
        if r >= 2:
            times.append(ev[0].elapsed_time(ev[1]))
    err = st.get_error()
    if not os.environ.get("PREFILL_IGNORE_ERR"):  # (timing-only experiment builds feed garbage)
        assert err == 0, f"device error {err} at n0={n0} ntok={ntok} batch={batch}"
    ms = sorted(times)[len(times) // 2]
    keys = sum(n0 + i + 1 for i in range(ntok)) * batch
    flops = 4.0 * d * m * keys
    return {"n0": n0, "ntok": ntok, "batch": batch, "ms": round(ms, 4), "tflops": round(flops / (ms * 1e-3) / 1e12, 1)}


if __name__ == "__main__":
    res = [run(0, 4096), run(28672, 4096), run(0, 16384), run(32768 - 512, 512, batch=8)]
    for r in res:
        print(json.dumps(r))
