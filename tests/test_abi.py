"""The C-ABI boundary, on CPU: the library loads without a GPU, exports every function
include/delta.h declares, and its host-side validation (schedule, shapes, budget) follows
the paper's problem statement."""
import ctypes
import json
import os

import pytest

import paper_2510_09883_b200 as d200
from paper_2510_09883_b200 import DeltaConfig, DeltaError

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_library_loads_and_exports_every_declared_symbol():
    lib = d200.load_library()
    names = d200.declared_functions()
    assert {"delta_create", "delta_append_kv", "delta_decode_layer", "delta_select", "delta_destroy"} <= set(names)
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/delta.h but not exported"
    assert lib.delta_version().decode().startswith("delta-b200")


def test_no_product_dependency_on_oracle():
    """The product path never imports or links the oracle (they share no code)."""
    pkg = os.path.dirname(d200.__file__)
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(root, f)).read()
                for bad in ("import oracle", "from oracle", "delta_oracle", "oracle_"):
                    assert bad not in src, (f, bad)
    syms = os.popen(f"nm -D {d200.binding.LIB_PATH}").read()
    assert "oracle_" not in syms and "delta_create" in syms


def _c1(**kw):
    base = dict(num_layers=32, num_q_heads=32, num_kv_heads=8, head_dim=128, max_batch=1, max_seq_len=32768 + 64,
                num_full_prefix=2, select_layers=[2, 16, 25], budget_k=2048, n_sink=4, n_window=32, select_block=16)
    base.update(kw)
    return DeltaConfig(**base)


def test_query_sizes_c1():
    pool, ws = d200.query_sizes(_c1())
    # kv_pool = L x pages x g x 2 (K, V) x P x d x 2 bytes
    assert pool == 32 * 2052 * 8 * 2 * 16 * 128 * 2
    assert ws > 0 and ws % 256 == 0


@pytest.mark.parametrize("ex", GOLD["tiers"], ids=lambda e: e["cite"][:14])
def test_tier_validation_matches_paper(ex):
    cfg = _c1(num_layers=ex["num_layers"], num_full_prefix=ex["F"], select_layers=ex["delta"])
    if ex["ok"]:
        d200.query_sizes(cfg)
    else:
        with pytest.raises(DeltaError, match="CONFIG"):
            d200.query_sizes(cfg)


@pytest.mark.parametrize("bad", [
    dict(num_kv_heads=7),                       # g must divide m
    dict(head_dim=96),                          # d in {64, 128}
    dict(page_size=8),                          # P = 16
    dict(budget_k=2040),                        # page mode needs P | k (R6)
    dict(select_block=4),                       # token (1) or page (P) granularity
    dict(num_q_heads=64, num_kv_heads=2),       # gs <= 16
    dict(select_layers=[16, 2, 25]),            # ascending
    dict(num_full_prefix=3),                    # Delta layer 2 inside the full prefix
    dict(shard_world=2, shard_rank=2),          # rank outside [0, W)
    dict(shard_world=0),                        # W >= 1
    dict(det_chunks=3, shard_world=2),          # R21: W | C
    dict(det_chunks=-1),
    dict(det_chunks=65),                        # C <= 64
])
def test_config_errors(bad):
    with pytest.raises(DeltaError, match="CONFIG"):
        d200.query_sizes(_c1(**bad))


@pytest.mark.parametrize("policy", [d200.POLICY_QUEST, d200.POLICY_RAAS], ids=["quest", "raas"])
@pytest.mark.parametrize("bad", [
    dict(),                                     # Delta layers are not part of these policies
    dict(select_layers=[], select_block=1),     # they work on pages
    dict(select_layers=[], kv_dtype=d200.DELTA_FP32),
    dict(select_layers=[], shard_world=2, shard_rank=0),
    dict(select_layers=[], det_chunks=8),
], ids=["delta-layers", "token-mode", "fp32", "sharded", "det-chunks"])
def test_policy_config_errors(policy, bad):
    """Quest / RaaS restrictions are CONFIG errors (include/delta.h)."""
    with pytest.raises(DeltaError, match="CONFIG"):
        d200.query_sizes(_c1(policy=policy, **bad))


def test_policy_workspace_sizes():
    """Quest adds the page representatives (L x pages x g x 2 x d bf16); RaaS the per-layer
    plans (one per layer, every page) and last-salient steps."""
    _, ws_delta = d200.query_sizes(_c1())
    _, ws_quest = d200.query_sizes(_c1(policy=d200.POLICY_QUEST, select_layers=[]))
    _, ws_raas = d200.query_sizes(_c1(policy=d200.POLICY_RAAS, select_layers=[]))
    reps = 32 * 2052 * 8 * 2 * 128 * 2
    assert ws_quest - ws_delta >= reps - (1 << 20)
    assert ws_raas > ws_delta
    with pytest.raises(DeltaError, match="CONFIG"):
        d200.query_sizes(_c1(policy=7))


def test_null_handle_calls_are_usage_errors():
    lib = d200.load_library()
    assert lib.delta_decode_layer(None, 0, 1, None, None, None, None) == 2
    assert lib.delta_select(None, 0, 1, None, None, None, None) == 2
    assert lib.delta_layer_role(None, 0) == -1
    assert lib.delta_destroy(None) == 2


def test_shard_ranges_partition_the_pages():
    """Host-only: the ranks' page ranges are contiguous, disjoint and cover ceil(max_seq/P)."""
    for W in (1, 2, 3, 4, 8):
        for max_seq in (16, 1000, 32768 + 64, 131072 + 64):
            pages = -(-max_seq // 16)
            got = [d200.shard_range(_c1(max_seq_len=max_seq, shard_world=W, shard_rank=r)) for r in range(W)]
            assert got[0][0] == 0 and got[-1][1] == pages
            for (lo, hi), (lo2, _) in zip(got, got[1:]):
                assert lo <= hi == lo2


def test_det_chunk_ranges_are_unions_of_fixed_chunks():
    """Host-only (R21): with det_chunks = C a rank's range is the union of its C/W consecutive
    chunks of ceil(pages/C) pages — the same chunk boundaries for every W dividing C."""
    C = 8
    for max_seq in (16, 1000, 1600, 32768 + 64):
        pages = -(-max_seq // 16)
        per = -(-pages // C)
        chunk = [(min(pages, c * per), min(pages, (c + 1) * per)) for c in range(C)]
        for W in (1, 2, 4, 8):
            got = [d200.shard_range(_c1(max_seq_len=max_seq, shard_world=W, shard_rank=r, det_chunks=C))
                   for r in range(W)]
            want = [(chunk[r * C // W][0], chunk[(r + 1) * C // W - 1][1]) for r in range(W)]
            assert got == want, (max_seq, W)
