"""RaaS contrast (SPEC.md:540 acceptance 9; "risking the loss of tokens that may later
become important"): a synthetic trace in which salient pages are ignored early and needed later.
Keys of 8 planted pages (shared by every layer) carry a direction sigma; for
the first PHASE1 decode steps the queries are iid (nothing is salient, RaaS evicts by recency),
afterwards every query is aligned with sigma (the planted pages now hold most of the mass).
Same page budget (k = 256 tokens = 16 pages + sink / window pages) for DELTA (Delta layer 1
governs layers 2-3) and RaaS (every layer >= 1); per step the Eq.9 recall (mean over heads) of
layer 2, measured by the library's delta_attention_recall (RaaS: of its retained set after the
step's eviction)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402

L, M, G, D, S0, PHASE1, PHASE2 = 4, 32, 8, 128, 4096, 8, 8


def run(policy, seed=21):
    raas = policy == "raas"
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=M, num_kv_heads=G, head_dim=D, max_batch=1,
                           max_seq_len=S0 + PHASE1 + PHASE2 + 64, num_full_prefix=1,
                           select_layers=[] if raas else [1], budget_k=256, n_sink=4, n_window=32,
                           select_block=16, policy=d200.POLICY_RAAS if raas else d200.POLICY_DELTA)
    plant = synth.Planting(count=8, block=16, B=1.0, G=1.0, lo=1, hi=(S0 - 64) // 16, shared=True)
    bt = torch.from_numpy(synth.block_table(seed, 1, cfg.max_pages))
    st = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(st.kv_pool, st.block_table, seed, S0, 1, range(L), plant)
    st.set_seq_lens([S0])
    if raas:
        st.raas_reset(-1, 1)
    torch.cuda.synchronize()
    out = torch.empty((L, 1, M, D), dtype=torch.float32, device="cuda")
    rec = torch.empty((1, M), dtype=torch.float32, device="cuda")
    trace = []
    for i in range(PHASE1 + PHASE2):
        s = S0 + 1 + i
        q = torch.empty((L, 1, M, D), dtype=torch.bfloat16, device="cuda")
        k = torch.empty((L, 1, G, D), dtype=torch.bfloat16, device="cuda")
        v = torch.empty_like(k)
        sd.fill_queries(q, seed, range(L), [s], plant if i >= PHASE1 else None)
        sd.fill_new_kv(k, v, seed, range(L), [s - 1])
        torch.cuda.synchronize()
        for layer in range(L):
            st.append_decode_layer(layer, k[layer], v[layer], q[layer], out[layer])
            if not raas and layer == 1:
                st.select(1, 1)
        st.attention_recall(2, q[2], rec)
        torch.cuda.synchronize()
        trace.append(round(float(rec.mean()), 4))
    assert st.get_error() == 0
    return trace


def main():
    for policy in ("delta", "raas"):
        t = run(policy)
        print(json.dumps({"policy": policy, "phase1_steps": PHASE1, "recall_layer2_per_step": t,
                          "phase2_mean": round(sum(t[PHASE1:]) / PHASE2, 4)}), flush=True)


if __name__ == "__main__":
    main()
