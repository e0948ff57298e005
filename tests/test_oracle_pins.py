"""Pins for the oracle against what the paper and the mathematics fix (CPU only).

Each test checks the oracle against something OTHER than itself: a worked value the
paper/SPEC prints (tests/golden/spec_examples.json, cited per entry), a closed form, an
invariant, brute-force enumeration, or an independent library routine (scipy).  The
selection of pins is such that a dropped term, wrong sign/index or transposed operand in
any oracle function fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import scipy.special

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ----------------------------------------------------------------- softmax (Eq.4)

@pytest.mark.parametrize("ex", GOLD["softmax"], ids=lambda e: e["cite"][:12])
def test_softmax_worked_examples(ex):
    alpha, _ = oracle.softmax(ex["a"])
    np.testing.assert_allclose(alpha, ex["alpha"], rtol=0, atol=1e-12)  # input 1000+ln2 is rounded to 1 ulp of 1000


def test_softmax_sum_shift_and_library():
    rng = np.random.default_rng(0)
    for _ in range(50):
        a = rng.normal(size=8) * 5
        alpha, lse = oracle.softmax(a)
        assert abs(alpha.sum() - 1.0) < 1e-12
        alpha2, lse2 = oracle.softmax(a + 1e4)
        assert np.max(np.abs(alpha - alpha2)) < 1e-12
        assert abs((lse2 - 1e4) - lse) < 1e-9
        np.testing.assert_allclose(alpha, scipy.special.softmax(a), rtol=1e-13, atol=0)
        assert abs(lse - scipy.special.logsumexp(a)) < 1e-12


def test_softmax_errors():
    with pytest.raises(oracle.OracleError, match="usage"):
        oracle.softmax([])
    with pytest.raises(oracle.OracleError, match="numeric"):
        oracle.softmax([0.0, float("nan")])


# ----------------------------------------------------------------- attend (Eq.4)

def _kv(K, V, P=4):
    return oracle.SeqKV.from_contiguous(np.asarray(K, np.float32)[:, None, :],
                                        np.asarray(V, np.float32)[:, None, :], P)


def test_attend_worked_d2():
    ex = GOLD["attend_d2"]
    kv = _kv(ex["keys"], ex["values"])
    out, lse, alpha = oracle.attend(ex["q"], kv, 0, [0, 1], ex["scale"], want_alpha=True)
    np.testing.assert_allclose(alpha, ex["weights"], atol=1e-15)
    np.testing.assert_allclose(out, ex["out"], atol=1e-15)


def test_attend_single_and_identical_keys():
    rng = np.random.default_rng(1)
    K = rng.normal(size=(3, 8)); V = rng.normal(size=(3, 8))
    kv = _kv(K, V)
    out, _, _ = oracle.attend(rng.normal(size=8), kv, 0, [2], 0.3)
    np.testing.assert_array_equal(out, V[2].astype(np.float32).astype(np.float64))
    K2 = np.stack([K[0], K[0]]); V2 = V[:2]
    out, _, _ = oracle.attend(rng.normal(size=8), _kv(K2, V2), 0, [0, 1], 0.3)
    np.testing.assert_allclose(out, V2.astype(np.float32).astype(np.float64).mean(0), atol=1e-15)


def test_attend_closed_forms_and_gqa_map():
    rng = np.random.default_rng(2)
    s, g, d, m, P = 37, 2, 16, 8, 16
    K = rng.normal(size=(s, g, d)).astype(np.float32)
    V = rng.normal(size=(s, g, d)).astype(np.float32)
    kv = oracle.SeqKV.from_contiguous(K, V, P)
    # q = 0 => uniform weights => O = mean of V over the attended rows (Eq.4)
    out, lse, alpha = oracle.decode_heads(np.zeros((m, d)), kv, s, 0.25, want_alpha=True)
    np.testing.assert_allclose(alpha, 1.0 / s, atol=1e-15)
    assert np.allclose(lse, math.log(s), atol=1e-13)
    gs = m // g
    for j in range(m):
        np.testing.assert_allclose(out[j], V[:, j // gs].astype(np.float64).mean(0), atol=1e-13)
    # V == c per group => O_j = c_phi(j), for any q (phi contiguous, R15)
    Vc = np.zeros_like(V); Vc[:, 0] = 1.5; Vc[:, 1] = -0.25
    kv2 = oracle.SeqKV.from_contiguous(K, Vc, P)
    out, _, _ = oracle.decode_heads(rng.normal(size=(m, d)), kv2, s, 0.25)
    for j in range(m):
        assert np.allclose(out[j], 1.5 if j < gs else -0.25, atol=1e-14)


def test_attend_matches_independent_numpy():
    """Eq.4 written with numpy/scipy (independent library path) on a paged, permuted cache."""
    rng = np.random.default_rng(3)
    s, g, d, m, P = 53, 4, 32, 8, 16
    K = rng.normal(size=(s, g, d)).astype(np.float32)
    V = rng.normal(size=(s, g, d)).astype(np.float32)
    n_pages = -(-s // P)
    bt = rng.permutation(n_pages + 3)[:n_pages].astype(np.int32)
    kp = np.zeros((n_pages + 3, g, P, d), np.float32); vp = np.zeros_like(kp)
    for t in range(s):
        kp[bt[t // P], :, t % P] = K[t]; vp[bt[t // P], :, t % P] = V[t]
    kv = oracle.SeqKV(kp, vp, bt, P)
    q = rng.normal(size=(m, d)).astype(np.float32)
    toks = np.sort(rng.choice(s, 20, replace=False))
    for tokens in (s, toks):
        out, lse, _ = oracle.decode_heads(q, kv, tokens, 0.17)
        tt = np.arange(s) if isinstance(tokens, int) else tokens
        for j in range(m):
            grp = j // (m // g)
            a = 0.17 * (K[tt, grp].astype(np.float64) @ q[j].astype(np.float64))
            w = scipy.special.softmax(a)
            np.testing.assert_allclose(out[j], w @ V[tt, grp].astype(np.float64), rtol=1e-12, atol=1e-13)
            assert abs(lse[j] - scipy.special.logsumexp(a)) < 1e-12


def test_lse_partition_identity():
    """Any partition of the token set merged by LSE weights equals the unsplit result."""
    rng = np.random.default_rng(4)
    s, d = 64, 16
    K = rng.normal(size=(s, d)); V = rng.normal(size=(s, d)); q = rng.normal(size=d)
    kv = _kv(K, V, P=16)
    o_all, l_all, _ = oracle.attend(q, kv, 0, np.arange(s), 0.25)
    cut = 23
    oa, la, _ = oracle.attend(q, kv, 0, np.arange(cut), 0.25)
    ob, lb, _ = oracle.attend(q, kv, 0, np.arange(cut, s), 0.25)
    L = np.logaddexp(la, lb)
    assert abs(L - l_all) < 1e-12
    np.testing.assert_allclose(np.exp(la - L) * oa + np.exp(lb - L) * ob, o_all, atol=1e-13)


# ----------------------------------------------------------------- scores

def test_token_scores_examples_and_invariants():
    ex = GOLD["token_scores"]
    np.testing.assert_array_equal(oracle.token_scores(ex["alpha"]), ex["s_t"])
    rng = np.random.default_rng(5)
    a = rng.random((1, 20))
    np.testing.assert_array_equal(oracle.token_scores(a), a[0])           # single head
    A = rng.random((6, 30))
    np.testing.assert_array_equal(oracle.token_scores(A), oracle.token_scores(A[rng.permutation(6)]))
    np.testing.assert_array_equal(oracle.token_scores(A), A.max(0))


def test_score_sum_bounds():
    """Each alpha_j sums to 1, so 1 <= sum_t s_t <= m (s_t = max_j alpha_j(t))."""
    rng = np.random.default_rng(6)
    s, g, d, m = 200, 2, 16, 8
    kv = oracle.SeqKV.from_contiguous(rng.normal(size=(s, g, d)), rng.normal(size=(s, g, d)), 16)
    _, _, alpha = oracle.decode_heads(rng.normal(size=(m, d)) * 3, kv, s, 0.25, want_alpha=True)
    np.testing.assert_allclose(alpha.sum(1), 1.0, atol=1e-12)
    tot = oracle.token_scores(alpha).sum()
    assert 1.0 - 1e-12 <= tot <= m + 1e-12


@pytest.mark.parametrize("ex", GOLD["page_scores"], ids=lambda e: e["cite"][:12])
def test_page_scores_examples(ex):
    np.testing.assert_allclose(oracle.page_scores(ex["s_t"], ex["P"]), ex["S_u"], rtol=0, atol=1e-16)


def test_page_scores_direct_sum():
    rng = np.random.default_rng(7)
    s_t = rng.random(1000)
    ref = np.add.reduceat(s_t, np.arange(0, 1000, 16))
    np.testing.assert_allclose(oracle.page_scores(s_t, 16), ref, rtol=1e-12)
    np.testing.assert_array_equal(oracle.page_scores(s_t, 1), s_t)


# ----------------------------------------------------------------- selection

@pytest.mark.parametrize("ex", GOLD["select_token"] + GOLD["select_page"], ids=lambda e: e["cite"][:14])
def test_select_worked_examples(ex):
    rho = oracle.select(ex["keys"], ex["s"], ex["block"], ex["n_sink"], ex["n_window"], ex["k_units"])
    assert rho.tolist() == ex["rho"]


def _brute_force(keys, s, block, S, L, k):
    n_units = -(-s // block)
    forced = set()
    if S > 0:
        forced |= set(range(0, (min(S, s) - 1) // block + 1))
    if L > 0:
        forced |= set(range(max(0, s - L) // block, n_units))
    cand = [u for u in range(n_units) if u not in forced]
    if len(cand) <= k:
        return list(range(n_units))
    best, best_sum = None, None
    for comb in itertools.combinations(cand, k):     # lexicographic order of index tuples
        sm = sum(keys[u] for u in comb)
        if best_sum is None or sm > best_sum:        # strict: keep the first (smallest) tuple
            best, best_sum = comb, sm
    return sorted(forced | set(best))


def test_select_exhaustive_bruteforce():
    """Exhaustive max-sum subsets for s <= 14 with small-integer keys (exact sums, many ties):
    the chosen set maximises the key sum and, among maximisers, is the lowest-index one (R9)."""
    rng = np.random.default_rng(8)
    n_checked = 0
    for trial in range(60):
        s = int(rng.integers(1, 15))
        block = int(rng.choice([1, 1, 2, 3]))
        n_units = -(-s // block)
        keys = rng.integers(0, 5, size=n_units).astype(np.float64)
        S = int(rng.integers(0, 3)); L = int(rng.integers(0, 4))
        for k in range(0, n_units + 1):
            got = oracle.select(keys, s, block, S, L, k).tolist()
            assert got == _brute_force(keys, s, block, S, L, k), (s, block, S, L, k, keys)
            n_checked += 1
    assert n_checked > 200


def test_select_invariants():
    rng = np.random.default_rng(9)
    for _ in range(40):
        s = int(rng.integers(1, 300)); S = int(rng.integers(0, 6)); L = int(rng.integers(0, 40))
        keys = rng.random(s)
        prev = None
        for k in range(0, 60, 7):
            rho = oracle.select(keys, s, 1, S, L, k)
            assert np.all(np.diff(rho) > 0)                                   # sorted, unique
            assert set(range(min(S, s))) <= set(rho.tolist())                 # sink kept
            assert set(range(max(0, s - L), s)) <= set(rho.tolist())          # window kept
            assert len(rho) == min(s, k + len(set(range(min(S, s))) | set(range(max(0, s - L), s))))
            if prev is not None:
                assert set(prev.tolist()) <= set(rho.tolist())                # nesting
            prev = rho


def test_select_all_equal_lowest_index_and_page_token_equivalence():
    rho = oracle.select(np.full(50, 0.5), 50, 1, 0, 5, 10)
    assert rho.tolist() == list(range(10)) + list(range(45, 50))
    # page mode with per-page-constant token scores selects the same tokens
    rng = np.random.default_rng(10)
    P, s = 4, 64
    page_keys = rng.permutation(16).astype(np.float64)
    tok_keys = np.repeat(page_keys, P)
    units = oracle.select(page_keys, s, P, 0, 8, 5)
    toks_page = oracle.units_to_tokens(units, P, s)
    toks_tok = oracle.select(tok_keys, s, 1, 0, 8, 20)
    assert toks_page.tolist() == toks_tok.tolist()
    # P = 1 page mode is token mode
    np.testing.assert_array_equal(oracle.select(tok_keys, s, 1, 3, 8, 11),
                                  oracle.units_to_tokens(oracle.select(tok_keys, s, 1, 3, 8, 11), 1, s))


def test_token_reduction_arithmetic():
    ex = GOLD["token_reduction"]
    s, P = ex["s"], ex["P"]
    k = s // 5
    keys = np.random.default_rng(11).random(s // P)
    units = oracle.select(keys, s, P, 0, 0, k // P)
    assert len(oracle.units_to_tokens(units, P, s)) <= ex["bound"]


# ----------------------------------------------------------------- schedule, bytes, paging

@pytest.mark.parametrize("ex", GOLD["tiers"], ids=lambda e: e["cite"][:12])
def test_validate_tiers(ex):
    if not ex["ok"]:
        with pytest.raises(oracle.OracleError, match="configuration"):
            oracle.validate_tiers(ex["num_layers"], ex["F"], ex["delta"])
        return
    roles, gov = oracle.validate_tiers(ex["num_layers"], ex["F"], ex["delta"])
    assert all(roles[l] == 0 for l in range(ex["F"]))
    assert [l for l in range(ex["num_layers"]) if roles[l] == 1] == ex["delta"]
    for rng_s, dl in ex.get("groups", {}).items():
        a, b = map(int, rng_s.split("-"))
        assert all(gov[l] == dl and roles[l] == 2 for l in range(a, b + 1))


@pytest.mark.parametrize("ex", GOLD["kv_bytes"], ids=lambda e: str(e["bytes"]))
def test_kv_bytes(ex):
    assert oracle.kv_bytes(*ex["args"]) == ex["bytes"]


@pytest.mark.parametrize("ex", GOLD["page_of"], ids=lambda e: str(e["t"]))
def test_page_of(ex):
    assert oracle.page_of(ex["t"], ex["P"]) == ex["page"]


@pytest.mark.parametrize("ex", GOLD["recall"], ids=lambda e: str(e["R"]))
def test_recall(ex):
    assert abs(oracle.attention_recall(ex["alpha"], ex["rho"]) - ex["R"]) < 1e-15


def test_append_roundtrip():
    """After N appends, reading every page returns the inputs in order."""
    rng = np.random.default_rng(12)
    P, g, d, N = 16, 2, 8, 37
    n_pages = -(-N // P)
    assert n_pages == 3                                   # ceil(s/P)
    bt = np.array([5, 0, 3], np.int32)
    kv = oracle.SeqKV(np.zeros((6, g, P, d)), np.zeros((6, g, P, d)), bt, P)
    ks = rng.normal(size=(N, g, d)).astype(np.float32); vs = rng.normal(size=(N, g, d)).astype(np.float32)
    for n in range(N):
        kv.append(n, ks[n], vs[n])
    for t in range(N):
        for h in range(g):
            np.testing.assert_array_equal(kv.k_pool[bt[t // P], h, t % P], ks[t, h])
            np.testing.assert_array_equal(kv.v_pool[bt[t // P], h, t % P], vs[t, h])


# ----------------------------------------------------------------- the stack

def _cfg(**kw):
    base = dict(num_layers=4, m=8, g=2, d=64, page_size=16, num_full_prefix=1, select_layers=[1],
                budget_k=128, n_sink=4, n_window=32, select_block=1, scale=0.125)
    base.update(kw)
    return oracle.StackConfig(**base)


def _layers(seed, cfg, s, dtype="fp32", planting=None):
    kvs, qs = [], []
    for l in range(cfg.num_layers):
        K = synth.kv_rows(seed, l, 0, 0, s, cfg.g, cfg.d, dtype, "k", planting)
        V = synth.kv_rows(seed, l, 0, 0, s, cfg.g, cfg.d, dtype, "v", planting)
        kvs.append(oracle.SeqKV.from_contiguous(K, V, cfg.page_size))
        qs.append(synth.q_rows(seed, l, 0, s, cfg.m, cfg.d, dtype, planting))
    return kvs, qs


def test_stack_budget_covers_context_equals_full():
    """k >= s  =>  DELTA stack == Full stack (north star)."""
    s = 150
    cfg = _cfg(budget_k=200)
    kvs, qs = _layers(2510, cfg, s)
    delta = oracle.stack_step(cfg, kvs, qs, s)
    full = oracle.stack_step(_cfg(budget_k=200, num_full_prefix=4, select_layers=[]), kvs, qs, s)
    for l in range(4):
        np.testing.assert_array_equal(delta[l].out, full[l].out)
        np.testing.assert_array_equal(delta[l].lse, full[l].lse)


def test_stack_c0_shapes_and_sparse_set():
    s = 512
    cfg = _cfg()
    kvs, qs = _layers(2510, cfg, s)
    res = oracle.stack_step(cfg, kvs, qs, s)
    assert [r.role for r in res] == [0, 1, 2, 2]
    rho = res[1].units
    assert len(rho) == 164                       # 4 sink + 32 window + 128 salient (R1)
    assert res[2].tokens.tolist() == rho.tolist() == res[3].tokens.tolist()


@pytest.mark.parametrize("block,B,G", [(1, 3.0, 1.0), (16, 1.0, 1.0)])
def test_planted_set_recovered(block, B, G):
    """Planted construction: the expected rho = planted U forced is known WITHOUT any oracle;
    the oracle must select exactly it, with a wide boundary gap."""
    s, cfg = 512, _cfg(select_block=block, budget_k=128)
    k_units = cfg.k_units
    lo = -(-cfg.n_sink // block)
    hi = (s - cfg.n_window) // block
    plant = synth.Planting(count=k_units, block=block, B=B, G=G, lo=lo, hi=hi)
    kvs, qs = _layers(77, cfg, s, "fp32", plant)
    res = oracle.stack_step(cfg, kvs, qs, s)
    planted = synth.planted_units(77, 1, 0, plant)
    n_units = -(-s // block)
    forced = set(range(0, (cfg.n_sink - 1) // block + 1)) | set(range((s - cfg.n_window) // block, n_units))
    assert res[1].units.tolist() == sorted(forced | set(planted.tolist()))
    keys = res[1].unit_keys
    cand = np.array([u for u in range(n_units) if u not in forced])
    ranked = np.sort(keys[cand])[::-1]
    gap = (ranked[k_units - 1] - ranked[k_units]) / ranked[k_units - 1]
    assert gap > 1e-2


# ---------------------------------------------------------------- Quest (NEXT-1)

def _quest_kv(keys_sgd, P=16):
    """A cache whose K rows are keys_sgd [s][g][d] (V = 0), identity block table."""
    K = np.asarray(keys_sgd, np.float32)
    return oracle.SeqKV.from_contiguous(K, np.zeros_like(K), P)


@pytest.mark.parametrize("ex", GOLD["quest_reps"], ids=lambda e: e["cite"])
def test_quest_reps_worked_examples(ex):
    keys = np.asarray(ex["keys"], np.float32)[:, None, :]          # one group
    reps = oracle.quest_reps(_quest_kv(keys, P=16), keys.shape[0])
    assert reps.shape == (1, 1, 2, keys.shape[2])
    assert np.array_equal(reps[0, 0, 0], ex["min"]) and np.array_equal(reps[0, 0, 1], ex["max"])


@pytest.mark.parametrize("ex", GOLD["quest_score"], ids=lambda e: e["cite"])
def test_quest_score_worked_examples(ex):
    reps = np.asarray([[[ex["min"], ex["max"]]]], np.float64)       # [1 page][1 group][2][d]
    got = oracle.quest_scores(np.asarray([ex["q"]], np.float32), reps)
    assert got[0] == ex["score"]


def test_quest_reps_pages_and_partial_last_page():
    """Per-page extrema over exactly the page's filled slots: a 37-token cache has pages of
    16, 16 and 5 tokens; a value planted in slot 5 of the last page (t = 37, not yet written)
    must not count."""
    rng = np.random.default_rng(5)
    s, g, d, P = 37, 2, 8, 16
    K = rng.integers(-50, 50, size=(48, g, d)).astype(np.float32)
    K[37, :, :] = 1000.0                                             # beyond s
    reps = oracle.quest_reps(_quest_kv(K, P), s)
    assert reps.shape == (3, g, 2, d)
    for u, (lo, hi) in enumerate([(0, 16), (16, 32), (32, 37)]):
        for grp in range(g):
            for e in range(d):
                col = [float(K[t, grp, e]) for t in range(lo, hi)]
                assert reps[u, grp, 0, e] == min(col) and reps[u, grp, 1, e] == max(col)


def test_quest_upper_bound_property():
    """quest_score(q, reps(page)) >= max over the page's keys of q . k, for every
    head (m = 1 so the page key is that head's bound), over 2000 random (q, page) draws; and the
    bound is attained when the page holds a single distinct key."""
    rng = np.random.default_rng(6)
    P, d = 16, 16
    for _ in range(2000):
        n = int(rng.integers(1, P + 1))
        K = rng.standard_normal((P, 1, d)).astype(np.float32)
        q = rng.standard_normal((1, d)).astype(np.float32)
        bound = oracle.quest_scores(q, oracle.quest_reps(_quest_kv(K, P), n))[0]
        best = max(float(np.dot(q[0].astype(np.float64), K[t, 0].astype(np.float64))) for t in range(n))
        assert bound >= best - 1e-12
    K = np.repeat(rng.standard_normal((1, 1, d)).astype(np.float32), P, axis=0)
    q = rng.standard_normal((1, d)).astype(np.float32)
    bound = oracle.quest_scores(q, oracle.quest_reps(_quest_kv(K, P), P))[0]
    assert abs(bound - float(np.dot(q[0].astype(np.float64), K[0, 0].astype(np.float64)))) < 1e-12


def test_quest_max_over_heads_and_group_map():
    """Q2 + R15: m = 4 heads over g = 2 groups (heads 0,1 -> group 0; 2,3 -> group 1).  Page 0's
    group-1 keys align with head 3's query, page 1's group-0 keys with head 0's: each page's key
    is the best head's bound, and permuting heads within a group leaves the keys unchanged."""
    d, P = 4, 16
    K = np.zeros((2 * P, 2, d), np.float32)
    K[:P, 1, :] = [0, 0, 5, 0]           # page 0, group 1
    K[P:, 0, :] = [2, 0, 0, 0]           # page 1, group 0
    q = np.zeros((4, d), np.float32)
    q[3] = [0, 0, 1, 0]
    q[0] = [1, 0, 0, 0]
    keys = oracle.quest_scores(q, oracle.quest_reps(_quest_kv(K, P), 2 * P))
    assert keys.tolist() == [5.0, 2.0]
    keys2 = oracle.quest_scores(q[[1, 0, 3, 2]], oracle.quest_reps(_quest_kv(K, P), 2 * P))
    assert keys2.tolist() == keys.tolist()


def test_quest_dominant_page_selected_and_budget_all():
    """a page whose keys all equal q is picked first among the older pages;
    a page budget covering every candidate selects every page (R12)."""
    rng = np.random.default_rng(7)
    P, d, s = 16, 8, 16 * 12
    K = (0.1 * rng.standard_normal((s, 1, d))).astype(np.float32)
    q = rng.standard_normal((1, d)).astype(np.float32)
    K[5 * P:6 * P, 0, :] = q[0]
    kv = _quest_kv(K, P)
    keys = oracle.quest_scores(q, oracle.quest_reps(kv, s))
    units = oracle.select(keys, s, P, 4, 32, 1)                      # sink page 0 + 2 window pages + 1
    assert units.tolist() == [0, 5, 10, 11]
    assert oracle.select(keys, s, P, 4, 32, 9).tolist() == list(range(12))


# ---------------------------------------------------------------- RaaS (NEXT-4)

def _raas(S, step, thr, exempt, cap, retained, last):
    r = np.array(retained, np.uint8)
    l = np.array(last, np.int64)
    ev = oracle.raas_step(np.array(S, float), step, thr, np.array(exempt, np.uint8), cap, r, l)
    return ev.tolist(), r.tolist(), l.tolist()


def test_raas_capacity_covers_all_no_eviction():
    """capacity >= page count -> no eviction; salient pages are refreshed."""
    ev, r, l = _raas([0.5, 0.1, 0.9, 0.0], 7, 0.25, [0, 0, 0, 0], 4, [1, 1, 1, 1], [0, 0, 0, 0])
    assert ev == [] and r == [1, 1, 1, 1] and l == [7, 0, 7, 0]


def test_raas_never_salient_evicted_before_refreshed():
    """a page that never reaches the threshold goes before any refreshed page,
    whatever their indices."""
    ev, r, _ = _raas([0.9, 0.9, 0.0, 0.9], 3, 0.5, [0, 0, 0, 0], 3, [1, 1, 1, 1], [1, 1, 1, 1])
    assert ev == [2] and r == [1, 1, 0, 1]


def test_raas_scripted_five_pages_capacity_three():
    """a scripted score sequence over 5 pages, capacity 3, page 4 exempt (recency).
    Hand simulation of the rule (refresh at >= 0.3, evict smallest (last, index)):
      step 1: S = [.5 .0 .4 .1 .9]: last = [1 0 1 0 0] ; non-exempt {0,1,2,3} > 3 -> evict 1
      step 2: S = [.0 - .6 .5 .9]:  last = [1 - 2 2 0] ; {0,2,3} = 3 -> none
      step 3: S = [.4 - .0 .0 .9]:  last = [3 - 2 2 0] ; none
      step 4: cap 2 (budget shrinks): {0,2,3}: lasts 3,2,2 -> evict 2 (tie 2,2: lowest index)"""
    retained = np.ones(5, np.uint8)
    last = np.zeros(5, np.int64)
    ex = np.array([0, 0, 0, 0, 1], np.uint8)
    evs = []
    for step, S, cap in [(1, [.5, .0, .4, .1, .9], 3), (2, [.0, .0, .6, .5, .9], 3), (3, [.4, .0, .0, .0, .9], 3),
                         (4, [.0, .0, .0, .0, .9], 2)]:
        evs.append(oracle.raas_step(np.array(S), step, 0.3, ex, cap, retained, last).tolist())
    assert evs == [[1], [], [], [2]]
    assert retained.tolist() == [1, 0, 0, 1, 1]
    assert last.tolist() == [3, 0, 2, 2, 4]


def test_raas_invariants_random():
    """retained non-exempt count never exceeds capacity, exempt pages are never
    evicted, evicted pages never come back (200 random steps)."""
    rng = np.random.default_rng(9)
    n, cap = 40, 6
    retained = np.ones(n, np.uint8)
    last = np.zeros(n, np.int64)
    gone = set()
    for step in range(1, 201):
        ex = (rng.random(n) < 0.1).astype(np.uint8)
        ex[-3:] = 1
        before = retained.copy()
        ev = oracle.raas_step(rng.random(n), step, 0.7, ex, cap, retained, last)
        assert all(before[u] and not ex[u] for u in ev)
        assert int(((retained > 0) & (ex == 0)).sum()) <= cap
        gone |= set(ev.tolist())
        assert not any(retained[u] for u in gone)


def test_raas_exempt_pages():
    """RS4 by hand: sink pages overlap [0, S), recency pages overlap [s - L, s)."""
    assert oracle.raas_exempt(10, 150, 16, 4, 32).tolist() == [1, 0, 0, 0, 0, 0, 0, 1, 1, 1]  # 118 // 16 = 7
    assert oracle.raas_exempt(3, 40, 16, 0, 32).tolist() == [1, 1, 1]          # window [8, 40) covers all
    assert oracle.raas_exempt(5, 80, 16, 20, 0).tolist() == [1, 1, 0, 0, 0]   # sink [0, 20): pages 0, 1
    assert oracle.raas_exempt(6, 96, 16, 0, 0).tolist() == [0] * 6
    assert oracle.raas_exempt(0, 0, 16, 4, 32).tolist() == []


def test_raas_layer_step_hand_trajectory():
    """raas_layer_step composition (RS1-RS4) on a tiny sequence whose attention weights are known
    by hand: m = g = d = 1, scale 1, q = [1], K_t = [ln w_t] so alpha_t = w_t / sum(w) over the
    ATTENDED tokens; P = 2, no sink, window L = 2, budget 2 tokens (1 page).  Tokens 2, 3 (page 1)
    weigh 4, every other token 1; V_t = [t].  Start (reset): pages 0-2 retained, last = 0.
      s=7 : token 6 opens page 3 (last 7); attended 0..6, W = 13, S = [2, 8, 2, 1] / 13,
            threshold P/7: page 1 refreshed (last 7); exempt {2, 3}; non-exempt {0, 1}: evict 0
      s=8 : attended 2..7, W = 12, S = [0, 8, 2, 2] / 12, threshold 2/6: page 1 refreshed;
            exempt {3}; non-exempt {1 (last 8), 2 (last 0)}: evict 2
      s=9 : token 8 opens page 4; attended {2,3,6,7,8}, W = 11, S1 = 8/11, S3 = 2/11, S4 = 1/11;
            threshold 2/5: page 1 refreshed; exempt {3, 4}; nothing to evict
      s=10: attended {2,3,6,7,8,9}, W = 12, S1 = 8/12, S3 = S4 = 2/12; exempt {4};
            non-exempt {1 (last 10), 3 (last 7)}: evict 3
      s=11: token 10 opens page 5; attended {2,3,8,9,10}, W = 11; exempt {4, 5}; nothing evicted
    Output = sum_t w_t t / W over the attended tokens (closed form)."""
    P, smax = 2, 11
    w = np.ones(smax)
    w[2:4] = 4.0
    K = np.log(w).astype(np.float32).reshape(smax, 1, 1)
    V = np.arange(smax, dtype=np.float32).reshape(smax, 1, 1)
    cfg = oracle.StackConfig(num_layers=1, m=1, g=1, d=1, page_size=P, num_full_prefix=0, select_layers=[],
                             budget_k=2, n_sink=0, n_window=2, select_block=P, scale=1.0)
    q = np.ones((1, 1), np.float32)
    retained = np.zeros(8, np.uint8)
    retained[:3] = 1
    last = np.zeros(8, np.int64)
    expect = {  # s: (attended pages, page scores by page, evicted, retained after)
        7: ([0, 1, 2, 3], {0: 2 / 13, 1: 8 / 13, 2: 2 / 13, 3: 1 / 13}, [0], [1, 2, 3]),
        8: ([1, 2, 3], {0: 0.0, 1: 8 / 12, 2: 2 / 12, 3: 2 / 12}, [2], [1, 3]),
        9: ([1, 3, 4], {1: 8 / 11, 2: 0.0, 3: 2 / 11, 4: 1 / 11}, [], [1, 3, 4]),
        10: ([1, 3, 4], {1: 8 / 12, 3: 2 / 12, 4: 2 / 12}, [3], [1, 4]),
        11: ([1, 4, 5], {1: 8 / 11, 4: 2 / 11, 5: 1 / 11}, [], [1, 4, 5]),
    }
    for s in range(7, 12):
        kv = oracle.SeqKV.from_contiguous(K[:s], V[:s], P)
        out, lse, pages, S, ev = oracle.raas_layer_step(cfg, kv, q, s, retained, last)
        att, sc, e_ev, e_ret = expect[s]
        assert pages.tolist() == att, f"attended pages at s={s}"
        for u, v in sc.items():
            assert abs(S[u] - v) <= 1e-6, f"S[{u}] at s={s}: {S[u]} vs {v}"
        assert ev.tolist() == e_ev, f"evicted at s={s}"
        assert np.nonzero(retained)[0].tolist() == e_ret, f"retained after s={s}"
        toks = oracle.units_to_tokens(np.array(att), P, s)
        assert abs(out[0, 0] - (w[toks] * toks).sum() / w[toks].sum()) <= 1e-6
    assert last[1] == 11 and last[3] == 7 and last[4] == 9 and last[5] == 11
