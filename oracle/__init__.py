"""ORACLE for DELTA decode-step attention (arXiv 2510.09883) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_2510_09883_b200``) never imports it, and the two share no code.

Thin ctypes wrapper over ``liboracle.so`` (plain fp64 C in ``delta_oracle.c``),
plus :func:`stack_step`, which composes those functions into one decode step of
the three-tier stack (Fig.2 caption PAPER.md:152) exactly in
the order the paper states: append (Eq.7), then per layer full / Delta (full +
score + select) / sparse attention.

Every function's citation and reading (R#) is in ``delta_oracle.h``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

ROLE_FULL, ROLE_SELECT, ROLE_SPARSE = 0, 1, 2


def build() -> str:
    """Compile liboracle.so (gcc, fp64, no fp contraction, no fast-math)."""
    src = os.path.join(_HERE, "delta_oracle.c")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "delta_oracle.h"))
    ):
        cmd = (
            f"gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared "
            f"-o {_LIB_PATH} {src} -lm"
        )
        if os.system(cmd) != 0:
            raise RuntimeError(f"oracle build failed: {cmd}")
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER
        c_i64, c_i32, c_dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.oracle_softmax.argtypes = [P(c_dbl), c_i64, P(c_dbl), P(c_dbl)]
        L.oracle_attend.argtypes = [
            P(ctypes.c_float), ctypes.c_void_p, c_i32, P(c_i64), c_i64, c_dbl,
            P(c_dbl), P(c_dbl), P(c_dbl)]
        L.oracle_decode_heads.argtypes = [
            P(ctypes.c_float), c_i32, ctypes.c_void_p, P(c_i64), c_i64, c_dbl,
            P(c_dbl), P(c_dbl), P(c_dbl), ctypes.c_int]
        L.oracle_token_scores.argtypes = [P(c_dbl), c_i32, c_i64, P(c_dbl)]
        L.oracle_page_scores.argtypes = [P(c_dbl), c_i64, c_i32, P(c_dbl)]
        L.oracle_select.argtypes = [P(c_dbl), c_i64, c_i32, c_i32, c_i32, c_i64, P(c_i64)]
        L.oracle_select.restype = c_i64
        L.oracle_units_to_tokens.argtypes = [P(c_i64), c_i64, c_i32, c_i64, P(c_i64)]
        L.oracle_units_to_tokens.restype = c_i64
        L.oracle_validate_tiers.argtypes = [c_i32, c_i32, c_i32, P(c_i32), P(c_i32), P(c_i32)]
        L.oracle_kv_bytes.argtypes = [ctypes.c_uint64] * 6
        L.oracle_kv_bytes.restype = ctypes.c_uint64
        L.oracle_attention_recall.argtypes = [P(c_dbl), c_i64, P(c_i64), c_i64]
        L.oracle_attention_recall.restype = c_dbl
        L.oracle_quest_reps.argtypes = [ctypes.c_void_p, c_i64, P(c_dbl)]
        L.oracle_quest_scores.argtypes = [P(ctypes.c_float), c_i32, c_i32, c_i32, P(c_dbl), c_i64, P(c_dbl)]
        L.oracle_raas_step.argtypes = [c_i64, P(c_dbl), c_i64, c_dbl, P(ctypes.c_char), c_i64, P(ctypes.c_char),
                                       P(c_i64), P(c_i64)]
        L.oracle_raas_step.restype = c_i64
        L.oracle_page_of.argtypes = [c_i64, c_i32]
        L.oracle_page_of.restype = c_i64
        L.oracle_append.argtypes = [
            P(ctypes.c_float), P(ctypes.c_float), P(c_i32), c_i32, c_i32, c_i32, c_i64,
            P(ctypes.c_float), P(ctypes.c_float)]
        _lib = L
    return _lib


class _SeqKV(ctypes.Structure):
    _fields_ = [
        ("P", ctypes.c_int32), ("g", ctypes.c_int32), ("d", ctypes.c_int32),
        ("k_pool", ctypes.POINTER(ctypes.c_float)), ("v_pool", ctypes.POINTER(ctypes.c_float)),
        ("block_table", ctypes.POINTER(ctypes.c_int32)),
    ]


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class OracleError(RuntimeError):
    pass


def _check(st: int, what: str):
    if st != 0:
        raise OracleError(f"{what}: oracle status {st} "
                          f"({ {1: 'configuration', 2: 'usage', 3: 'numeric'}.get(st, '?') } error)")


# ---------------------------------------------------------------- primitives

def softmax(a) -> tuple[np.ndarray, float]:
    a = np.ascontiguousarray(a, dtype=np.float64)
    alpha = np.empty_like(a)
    lse = ctypes.c_double()
    _check(lib().oracle_softmax(_ptr(a, ctypes.c_double), a.size, _ptr(alpha, ctypes.c_double),
                                ctypes.byref(lse)), "softmax")
    return alpha, lse.value


class SeqKV:
    """One sequence's paged K/V for one layer: pools [phys_pages][g][P][d] float32."""

    def __init__(self, k_pool, v_pool, block_table, P: int):
        self.k_pool = np.ascontiguousarray(k_pool, dtype=np.float32)
        self.v_pool = np.ascontiguousarray(v_pool, dtype=np.float32)
        self.block_table = np.ascontiguousarray(block_table, dtype=np.int32)
        _, g, P2, d = self.k_pool.shape
        assert P2 == P
        self.P, self.g, self.d = P, g, d
        self._s = _SeqKV(P, g, d, _ptr(self.k_pool, ctypes.c_float), _ptr(self.v_pool, ctypes.c_float),
                         _ptr(self.block_table, ctypes.c_int32))

    @classmethod
    def from_contiguous(cls, K, V, P: int):
        """K, V as logical [s][g][d]: lay them into pages with an identity block table."""
        K = np.asarray(K, dtype=np.float32)
        V = np.asarray(V, dtype=np.float32)
        s, g, d = K.shape
        n_pages = max(1, -(-s // P))
        kp = np.zeros((n_pages * P, g, d), np.float32)
        vp = np.zeros((n_pages * P, g, d), np.float32)
        kp[:s] = K
        vp[:s] = V
        # [pages*P][g][d] -> [pages][g][P][d]
        kp = kp.reshape(n_pages, P, g, d).transpose(0, 2, 1, 3)
        vp = vp.reshape(n_pages, P, g, d).transpose(0, 2, 1, 3)
        return cls(kp, vp, np.arange(n_pages, dtype=np.int32), P)

    @property
    def ref(self):
        return ctypes.byref(self._s)

    def append(self, n: int, k_new, v_new):
        """Eq.7 append of token position n (pools are modified in place)."""
        k_new = np.ascontiguousarray(k_new, dtype=np.float32)
        v_new = np.ascontiguousarray(v_new, dtype=np.float32)
        _check(lib().oracle_append(_ptr(self.k_pool, ctypes.c_float), _ptr(self.v_pool, ctypes.c_float),
                                   _ptr(self.block_table, ctypes.c_int32), self.P, self.g, self.d, n,
                                   _ptr(k_new, ctypes.c_float), _ptr(v_new, ctypes.c_float)), "append")


def attend(q, kv: SeqKV, grp: int, tokens, scale: float, want_alpha=False):
    q = np.ascontiguousarray(q, dtype=np.float32)
    toks = np.ascontiguousarray(tokens, dtype=np.int64)
    out = np.empty(kv.d, np.float64)
    lse = ctypes.c_double()
    alpha = np.empty(toks.size, np.float64) if want_alpha else None
    _check(lib().oracle_attend(_ptr(q, ctypes.c_float), kv.ref, grp, _ptr(toks, ctypes.c_int64), toks.size,
                               scale, _ptr(out, ctypes.c_double), ctypes.byref(lse),
                               _ptr(alpha, ctypes.c_double) if want_alpha else None), "attend")
    return out, lse.value, alpha


def decode_heads(q, kv: SeqKV, tokens, scale: float, want_alpha=False, nthreads=0):
    """q [m][d] -> (out [m][d], lse [m], alpha [m][ntok] or None).  tokens=None: all s tokens
    given by ``tokens`` as an int count."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    m, d = q.shape
    if isinstance(tokens, (int, np.integer)):
        ntok, tptr = int(tokens), None
    else:
        toks = np.ascontiguousarray(tokens, dtype=np.int64)
        ntok, tptr = toks.size, _ptr(toks, ctypes.c_int64)
    out = np.empty((m, d), np.float64)
    lse = np.empty(m, np.float64)
    alpha = np.empty((m, ntok), np.float64) if want_alpha else None
    _check(lib().oracle_decode_heads(_ptr(q, ctypes.c_float), m, kv.ref, tptr, ntok, scale,
                                     _ptr(out, ctypes.c_double), _ptr(lse, ctypes.c_double),
                                     _ptr(alpha, ctypes.c_double) if want_alpha else None, nthreads),
           "decode_heads")
    return out, lse, alpha


def token_scores(alpha) -> np.ndarray:
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    m, s = alpha.shape
    out = np.empty(s, np.float64)
    _check(lib().oracle_token_scores(_ptr(alpha, ctypes.c_double), m, s, _ptr(out, ctypes.c_double)),
           "token_scores")
    return out


def page_scores(s_t, P: int) -> np.ndarray:
    s_t = np.ascontiguousarray(s_t, dtype=np.float64)
    out = np.empty(-(-s_t.size // P), np.float64)
    _check(lib().oracle_page_scores(_ptr(s_t, ctypes.c_double), s_t.size, P, _ptr(out, ctypes.c_double)),
           "page_scores")
    return out


def select(unit_keys, s: int, block: int, n_sink: int, n_window: int, k_units: int) -> np.ndarray:
    keys = np.ascontiguousarray(unit_keys, dtype=np.float64)
    n_units = -(-s // block)
    assert keys.size >= n_units
    out = np.empty(max(n_units, 1), np.int64)
    n = lib().oracle_select(_ptr(keys, ctypes.c_double), s, block, n_sink, n_window, k_units,
                            _ptr(out, ctypes.c_int64))
    if n < 0:
        raise OracleError("select: usage error")
    return out[:n].copy()


def units_to_tokens(units, block: int, s: int) -> np.ndarray:
    u = np.ascontiguousarray(units, dtype=np.int64)
    out = np.empty(max(u.size * block, 1), np.int64)
    n = lib().oracle_units_to_tokens(_ptr(u, ctypes.c_int64), u.size, block, s, _ptr(out, ctypes.c_int64))
    return out[:n].copy()


def validate_tiers(num_layers: int, num_full_prefix: int, delta_layers):
    d = np.ascontiguousarray(delta_layers, dtype=np.int32)
    roles = np.empty(num_layers, np.int32)
    gov = np.empty(num_layers, np.int32)
    _check(lib().oracle_validate_tiers(num_layers, num_full_prefix, d.size, _ptr(d, ctypes.c_int32),
                                       _ptr(roles, ctypes.c_int32), _ptr(gov, ctypes.c_int32)),
           "validate_tiers")
    return roles, gov


def kv_bytes(num_layers, seq_len, batch, kv_heads, head_dim, bytes_per_scalar) -> int:
    return int(lib().oracle_kv_bytes(num_layers, seq_len, batch, kv_heads, head_dim, bytes_per_scalar))


def attention_recall(alpha, rho) -> float:
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    r = np.ascontiguousarray(rho, dtype=np.int64)
    return float(lib().oracle_attention_recall(_ptr(a, ctypes.c_double), a.size, _ptr(r, ctypes.c_int64), r.size))


def page_of(t: int, P: int) -> int:
    return int(lib().oracle_page_of(t, P))


def quest_reps(kv: SeqKV, s: int) -> np.ndarray:
    """Quest page representatives [ceil(s/P)][g][2][d] (min row, max row): PAPER.md:205."""
    out = np.empty((-(-s // kv.P), kv.g, 2, kv.d), np.float64)
    _check(lib().oracle_quest_reps(kv.ref, s, _ptr(out, ctypes.c_double)), "quest_reps")
    return out


def quest_scores(q, reps) -> np.ndarray:
    """Quest page keys (readings Q1, Q2): max_j sum_e max(q_je min_e, q_je max_e)."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    reps = np.ascontiguousarray(reps, dtype=np.float64)
    m, d = q.shape
    n_pages, g = reps.shape[0], reps.shape[1]
    out = np.empty(n_pages, np.float64)
    _check(lib().oracle_quest_scores(_ptr(q, ctypes.c_float), m, g, d, _ptr(reps, ctypes.c_double), n_pages,
                                     _ptr(out, ctypes.c_double)), "quest_scores")
    return out


def raas_step(S, step: int, threshold: float, exempt, capacity: int, retained, last):
    """One RaaS refresh + eviction (readings RS1-RS4).  `retained` (uint8) and
    `last` (int64) are updated in place; returns the evicted pages in eviction order."""
    S = np.ascontiguousarray(S, dtype=np.float64)
    ex = np.ascontiguousarray(exempt, dtype=np.uint8)
    assert retained.dtype == np.uint8 and last.dtype == np.int64 and retained.flags.c_contiguous
    out = np.empty(S.size, np.int64)
    n = lib().oracle_raas_step(S.size, _ptr(S, ctypes.c_double), step, threshold, _ptr(ex, ctypes.c_char), capacity,
                               _ptr(retained, ctypes.c_char), _ptr(last, ctypes.c_int64), _ptr(out, ctypes.c_int64))
    assert n >= 0
    return out[:n].copy()


def raas_exempt(n_pages: int, s: int, P: int, n_sink: int, n_window: int) -> np.ndarray:
    """RS4: sink pages (overlapping [0, S)) and recency pages (overlapping [s - L, s))."""
    ex = np.zeros(n_pages, np.uint8)
    if n_sink > 0 and s > 0:
        ex[: (min(n_sink, s) - 1) // P + 1] = 1
    if n_window > 0:
        ex[max(0, s - n_window) // P:] = 1
    return ex


def raas_layer_step(cfg: "StackConfig", kv: SeqKV, q, s: int, retained, last, scores_override=None,
                    threshold=None):
    """One RaaS layer at cache length s (RS1-RS4): the new token's page joins the retained set,
    attention over tokens(retained) (softmax renormalised over them), page scores
    S_u = sum_{t in u} max_j alpha_j(t) over the attended tokens, threshold P / |attended|,
    refresh + eviction of the non-exempt pages beyond k/P.  `retained` / `last` are per page
    arrays with room for ceil(s/P) pages, updated in place.  `scores_override` replaces the
    page scores (to replay a GPU run's fp32 scores).  Returns (out, lse, attended_pages, S, evicted)."""
    P = cfg.page_size
    n_pages = -(-s // P)
    if (s - 1) % P == 0:                       # the appended token opened a page: created now
        retained[(s - 1) // P] = 1
        last[(s - 1) // P] = s
    pages = np.nonzero(retained[:n_pages])[0]
    tokens = units_to_tokens(pages, P, s)
    out, lse, alpha = decode_heads(q, kv, tokens, cfg.scale, want_alpha=True)
    s_t = token_scores(alpha)                  # max over heads of the renormalised weights (R7)
    S = np.zeros(n_pages, np.float64)
    for t, v in zip(tokens, s_t):
        S[t // P] += v
    if scores_override is not None:
        S = np.where(retained[:n_pages] > 0, scores_override[:n_pages], 0.0)
    ex = raas_exempt(n_pages, s, P, cfg.n_sink, cfg.n_window)
    ret = np.ascontiguousarray(retained[:n_pages])
    lst = np.ascontiguousarray(last[:n_pages])
    ev = raas_step(S, s, P / tokens.size if threshold is None else threshold(tokens.size), ex, cfg.budget_k // P,
                   ret, lst)
    retained[:n_pages] = ret
    last[:n_pages] = lst
    return out, lse, pages, S, ev


def quest_layer(cfg: "StackConfig", kv: SeqKV, q, s: int, nthreads=0):
    """One Quest layer (reading Q3): reps -> page keys -> select (same forced set and page
    budget as DELTA) -> attention over tokens(rho).  Returns (out, lse, keys, units, tokens)."""
    assert cfg.select_block == cfg.page_size
    keys = quest_scores(q, quest_reps(kv, s))
    units = select(keys, s, cfg.select_block, cfg.n_sink, cfg.n_window, cfg.k_units)
    tokens = units_to_tokens(units, cfg.select_block, s)
    out, lse, _ = decode_heads(q, kv, tokens, cfg.scale, nthreads=nthreads)
    return out, lse, keys, units, tokens


# ---------------------------------------------------------------- the stack

@dataclass
class StackConfig:
    num_layers: int
    m: int
    g: int
    d: int
    page_size: int
    num_full_prefix: int
    select_layers: list
    budget_k: int
    n_sink: int
    n_window: int
    select_block: int
    scale: float

    @property
    def k_units(self) -> int:
        # R6/R23: k salient tokens -> k/P pages in page mode
        return self.budget_k // self.select_block


@dataclass
class LayerResult:
    role: int
    out: np.ndarray            # [m][d] float64
    lse: np.ndarray            # [m]
    tokens: np.ndarray | None = None    # attended token list (sparse) or None (all)
    unit_keys: np.ndarray | None = None  # Delta layers: s_t (token) or S_u (page)
    units: np.ndarray | None = None      # Delta layers: selected units rho (ascending)


def select_from_alpha(cfg: StackConfig, alpha: np.ndarray, s: int):
    """Delta-layer scoring and selection."""
    s_t = token_scores(alpha)
    keys = s_t if cfg.select_block == 1 else page_scores(s_t, cfg.select_block)
    units = select(keys, s, cfg.select_block, cfg.n_sink, cfg.n_window, cfg.k_units)
    return keys, units


def stack_step(cfg: StackConfig, layers_kv: list, q_layers, s: int, nthreads=0) -> list:
    """One decode step of the three-tier stack for ONE sequence whose cache already
    holds this step's appended token (s tokens).  ``layers_kv[l]`` is a SeqKV and
    ``q_layers[l]`` the [m][d] query of layer l.  Returns a LayerResult per layer.

    Order: FULL layers attend to everything; each Delta layer
    attends to everything (R11), scores and selects rho for THIS step (R13); each
    sparse layer attends to tokens(rho) of the nearest Delta below it (R10)."""
    roles, gov = validate_tiers(cfg.num_layers, cfg.num_full_prefix, cfg.select_layers)
    results = []
    plans = {}
    for l in range(cfg.num_layers):
        kv = layers_kv[l]
        if roles[l] == ROLE_FULL:
            out, lse, _ = decode_heads(q_layers[l], kv, s, cfg.scale, nthreads=nthreads)
            results.append(LayerResult(ROLE_FULL, out, lse))
        elif roles[l] == ROLE_SELECT:
            out, lse, alpha = decode_heads(q_layers[l], kv, s, cfg.scale, want_alpha=True, nthreads=nthreads)
            keys, units = select_from_alpha(cfg, alpha, s)
            plans[l] = units
            results.append(LayerResult(ROLE_SELECT, out, lse, unit_keys=keys, units=units))
        else:
            toks = units_to_tokens(plans[int(gov[l])], cfg.select_block, s)
            out, lse, _ = decode_heads(q_layers[l], kv, toks, cfg.scale, nthreads=nthreads)
            results.append(LayerResult(ROLE_SPARSE, out, lse, tokens=toks))
    return results
