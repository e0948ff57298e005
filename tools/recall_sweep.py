"""K x L attention-recall sweep (NEXT-2's Table 1 surrogate, PAPER.md:229-247 axes: salient budget
K and recency window L) on synthetic caches, through the library's Eq.9 instrumentation
(delta_attention_recall): for each (K, L) one decode step of a 4-layer stack (FULL, Delta, two
sparse layers; token-level selection, 32q/8kv, d = 128, s = 8192), and the mean over heads of the
recall of the Delta layer's plan in the Delta layer and in the two sparse layers it governs.
Inputs: iid N(0,1) (no structure: recall ~ budget share); planted (96 salient tokens per
(layer, sequence) with a direction, SURVEY App. B — a different set in every layer, so a Delta
layer's plan cannot serve the layers above it); planted-shared (the same 96 tokens in every
layer: the inter-layer correlation the paper observes, that DELTA relies on).
The same sweep is run for the QUEST policy (per-layer page selection, page budget K rounded up
to pages).  Accuracy itself needs trained weights (out of scope); recall is the paper's own
quality measure for a selection (Eq.9)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402

L, M, G, D, S = 4, 32, 8, 128, 8192


def run(policy, K, Lw, planted, seed=11, shared=False):
    quest = policy == "quest"
    blk = 16 if quest else 1
    k = ((K + 15) // 16) * 16 if quest else K
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=M, num_kv_heads=G, head_dim=D, max_batch=1,
                           max_seq_len=S + 64, num_full_prefix=1, select_layers=[] if quest else [1],
                           budget_k=k, n_sink=4, n_window=Lw, select_block=blk,
                           policy=d200.POLICY_QUEST if quest else d200.POLICY_DELTA)
    plant = synth.Planting(count=96, block=1, B=2.0, G=1.0, lo=4, hi=S - 64, shared=shared) if planted else None
    bt = torch.from_numpy(synth.block_table(seed, 1, cfg.max_pages))
    st = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(st.kv_pool, st.block_table, seed, S - 1, 1, range(L), plant)
    st.set_seq_lens([S - 1])
    if quest:
        st.quest_build_reps(-1, 1)
    q = torch.empty((L, 1, M, D), dtype=torch.bfloat16, device="cuda")
    kk = torch.empty((L, 1, G, D), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(kk)
    sd.fill_queries(q, seed, range(L), [S], plant)
    sd.fill_new_kv(kk, v, seed, range(L), [S - 1])
    torch.cuda.synchronize()
    out = torch.empty((L, 1, M, D), dtype=torch.float32, device="cuda")
    rec = torch.empty((L, 1, M), dtype=torch.float32, device="cuda")
    for layer in range(L):
        st.append_decode_layer(layer, kk[layer], v[layer], q[layer], out[layer])
        if quest and layer >= 1:
            st.attention_recall(layer, q[layer], rec[layer])  # right after the layer (its own plan)
        if not quest and layer == 1:
            st.select(1, 1)                                   # the Delta layer's plan for layers 2, 3
    if not quest:
        for layer in (1, 2, 3):
            st.attention_recall(layer, q[layer], rec[layer])
    torch.cuda.synchronize()
    assert st.get_error() == 0
    return [round(float(rec[layer].mean()), 4) for layer in (1, 2, 3)]


def main():
    rows = []
    for inputs in ("iid", "planted", "planted-shared"):
        for policy in ("delta", "quest"):
            for K in (64, 128, 256):
                for Lw in (1, 8, 16, 32):
                    r = run(policy, K, Lw, inputs != "iid", shared=inputs == "planted-shared")
                    rows.append({"inputs": inputs, "policy": policy, "K": K, "L": Lw,
                                 "recall_layers_1_2_3": r})
                    print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
