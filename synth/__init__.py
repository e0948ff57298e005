"""Seeded synthetic inputs for DELTA decode attention — shared by the oracle side and the
CUDA side, and holding none of the method's arithmetic.

Counter-based and integer-exact, so the numpy generator here and the CUDA fill kernel in
``synth/csrc/synth_fill.cu`` produce bit-identical values without sharing code with
either the oracle or the product library:

* ``splitmix64`` (Steele/Lea/Flood) keyed by (seed, tag, layer, seq, step);
* each element draws three 64-bit words ``splitmix64(key + 3*i + r)``, r = 0, 1, 2,
  whose twelve 16-bit chunks sum to S (Irwin-Hall of 12 uniforms: mean 393210,
  std 65536), and ``x = (S - 393210) * 2**-16`` -- an exact fp32 value, ~N(0, 1);
* bf16 tensors round x to bf16 with round-to-nearest-even done on the bit pattern.

Element index ``i`` is LOGICAL: K/V row (t, h, e) of sequence ``seq`` in ``layer`` uses
``i = (t*g + h)*d + e``; the query of head j at step position s uses ``i = j*d + e`` with
``step = s``.  The token appended at a decode step is just cache row s-1, so the cache
content is a pure function of (seed, layer, seq, t) and regenerable anywhere.

Planted inputs (SURVEY.md §8(d) "planted"/"few-hot"): for a (layer, seq) a set of
``count`` units (tokens or pages) is chosen among ``[lo, hi)`` as the ``count`` units with
the smallest hash ``splitmix64(key_plant + u)``; every K row of a planted unit gets
``+B*sigma`` and every query head gets ``+G*sigma`` with sigma in {+1,-1}^d from
``splitmix64(key_sigma + e) & 1``.  All additions are exact in fp32 before the final
bf16 rounding (values are multiples of 2**-16 below 2**4).
"""
from __future__ import annotations

from dataclasses import dataclass

import os

import numpy as np

M64 = (1 << 64) - 1
TAG_K, TAG_V, TAG_Q, TAG_PLANT, TAG_SIGMA, TAG_KEYS, TAG_BT = 1, 2, 3, 4, 5, 6, 7
IH_MEAN = 6 * 65535  # 393210


def splitmix64_int(x: int) -> int:
    z = (x + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 on uint64 (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def stream_key(seed: int, tag: int, layer: int = 0, seq: int = 0, step: int = 0) -> int:
    k = splitmix64_int(seed & M64)
    k = splitmix64_int(k ^ tag)
    k = splitmix64_int(k ^ (layer & M64))
    k = splitmix64_int(k ^ (seq & M64))
    k = splitmix64_int(k ^ (step & M64))
    return k


def normal_f32(key: int, idx: np.ndarray) -> np.ndarray:
    """Irwin-Hall(12) approx N(0,1), exact multiples of 2**-16, as float32.  Large requests are
    split into chunks evaluated on a thread pool (numpy releases the GIL; the values are the same
    element by element)."""
    idx = np.asarray(idx).astype(np.uint64)
    if idx.size >= (1 << 21):
        from concurrent.futures import ThreadPoolExecutor
        flat = idx.reshape(-1)
        nchunk = min(32, max(1, (os.cpu_count() or 1) * 2))
        bounds = np.linspace(0, flat.size, nchunk + 1).astype(np.int64)
        out = np.empty(flat.size, np.float32)

        def work(i):
            out[bounds[i]:bounds[i + 1]] = _normal_f32(key, flat[bounds[i]:bounds[i + 1]])

        with ThreadPoolExecutor(max_workers=nchunk) as ex:
            list(ex.map(work, range(nchunk)))
        return out.reshape(idx.shape)
    return _normal_f32(key, idx)


def _normal_f32(key: int, idx: np.ndarray) -> np.ndarray:
    base = np.uint64(key)
    with np.errstate(over="ignore"):
        S = np.zeros(idx.shape, np.int64)
        for r in range(3):
            w = splitmix64(base + idx * np.uint64(3) + np.uint64(r))
            for c in range(4):
                S += ((w >> np.uint64(16 * c)) & np.uint64(0xFFFF)).astype(np.int64)
    return ((S - IH_MEAN).astype(np.float32) * np.float32(2.0 ** -16)).astype(np.float32)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 (ties to even), returned as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    u = (u + np.uint64(0x7FFF) + lsb) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """Upper 16 bits of bf16-representable float32 values (as uint16)."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


@dataclass(frozen=True)
class Planting:
    """Planted salient units for one (layer, seq).  ``block`` is 1 (tokens) or P (pages)."""
    count: int
    block: int
    B: float          # K boost (multiple of 0.5)
    G: float          # Q boost (multiple of 0.5)
    lo: int           # first eligible unit
    hi: int           # one past the last eligible unit
    shared: bool = False  # the same units in every layer (inter-layer correlation)


def planted_units(seed: int, layer: int, seq: int, p: Planting) -> np.ndarray:
    if p is None or p.count <= 0:
        return np.zeros(0, np.int64)
    units = np.arange(p.lo, p.hi, dtype=np.int64)
    assert units.size >= p.count, "planting region too small"
    key_layer = 0 if p.shared else layer
    h = splitmix64(np.uint64(stream_key(seed, TAG_PLANT, key_layer, seq)) + units.astype(np.uint64))
    order = np.lexsort((units, h))  # smallest hash, ties by index
    return np.sort(units[order[: p.count]])


def sigma(seed: int, layer: int, seq: int, d: int) -> np.ndarray:
    w = splitmix64(np.uint64(stream_key(seed, TAG_SIGMA, layer, seq)) + np.arange(d, dtype=np.uint64))
    return np.where((w & np.uint64(1)) == 1, 1.0, -1.0).astype(np.float32)


def _finish(x: np.ndarray, dtype: str) -> np.ndarray:
    return round_bf16(x) if dtype == "bf16" else x.astype(np.float32)


def kv_rows(seed: int, layer: int, seq: int, t0: int, t1: int, g: int, d: int, dtype: str,
            which: str, planting: Planting | None = None) -> np.ndarray:
    """Logical cache rows t0..t1-1 of K (which='k') or V ('v'): float32 [t1-t0][g][d]."""
    tag = TAG_K if which == "k" else TAG_V
    key = stream_key(seed, tag, layer, seq)
    n = t1 - t0
    idx = np.arange(t0 * g * d, t1 * g * d, dtype=np.uint64)
    x = normal_f32(key, idx).reshape(n, g, d)
    if which == "k" and planting is not None and planting.count > 0:
        x = round_bf16(x) if dtype == "bf16" else x
        units = planted_units(seed, layer, seq, planting)
        sg = sigma(seed, layer, seq, d)
        t = np.arange(t0, t1)
        mask = np.isin(t // planting.block, units)
        x = x.copy()
        x[mask] = x[mask] + np.float32(planting.B) * sg[None, None, :]
    return _finish(x, dtype)


def q_rows(seed: int, layer: int, seq: int, s: int, m: int, d: int, dtype: str,
           planting: Planting | None = None) -> np.ndarray:
    """Query [m][d] of (layer, seq) at the step whose cache holds s tokens."""
    key = stream_key(seed, TAG_Q, layer, seq, s)
    x = normal_f32(key, np.arange(m * d, dtype=np.uint64)).reshape(m, d)
    if planting is not None and planting.count > 0:
        x = round_bf16(x) if dtype == "bf16" else x
        x = x + np.float32(planting.G) * sigma(seed, layer, seq, d)[None, :]
    return _finish(x, dtype)


def block_table(seed: int, batch: int, pages_per_seq: int) -> np.ndarray:
    """A seeded permutation of physical pages [batch*pages_per_seq] dealt to sequences:
    realistic scattered paging, deterministic.  Returns int32 [batch][pages_per_seq]."""
    n = batch * pages_per_seq
    h = splitmix64(np.uint64(stream_key(seed, TAG_BT)) + np.arange(n, dtype=np.uint64))
    perm = np.argsort(h, kind="stable").astype(np.int32)
    return perm.reshape(batch, pages_per_seq)


def keys_buffer(seed: int, n: int, kind: str = "iid") -> np.ndarray:
    """Selection-key buffers for the top-k unit tests (fed through keys_override).
    kind: 'iid' (N(0,1)-like fp32), 'ties' (16 distinct values incl. +-0 and subnormals),
    'equal' (all one value)."""
    key = stream_key(seed, TAG_KEYS)
    x = normal_f32(key, np.arange(n, dtype=np.uint64))
    if kind == "iid":
        return x
    if kind == "ties":
        vals = np.array([0.0, -0.0, 1e-40, -1e-40, 1.5e-45, 0.25, 0.5, 1.0, 1.0 + 2 ** -23, 2.0,
                         3.0, -1.0, -2.5, 7.0, 1e30, -1e30], dtype=np.float32)
        w = splitmix64(np.uint64(key) + np.arange(n, dtype=np.uint64))
        return vals[(w % np.uint64(16)).astype(np.int64)]
    if kind == "equal":
        return np.full(n, 0.5, np.float32)
    raise ValueError(kind)


def build_seq_pools(seed: int, layer: int, seq: int, s: int, g: int, d: int, P: int, dtype: str,
                    bt_row: np.ndarray, n_phys: int, planting: Planting | None = None):
    """Host pools [n_phys][g][P][d] float32 holding this sequence's rows 0..s-1 at the
    physical pages bt_row (other pages zero).  Test infrastructure (layout only)."""
    K = kv_rows(seed, layer, seq, 0, s, g, d, dtype, "k", planting)
    V = kv_rows(seed, layer, seq, 0, s, g, d, dtype, "v", planting)
    kp = np.zeros((n_phys, g, P, d), np.float32)
    vp = np.zeros((n_phys, g, P, d), np.float32)
    for u in range(-(-s // P)):
        t0, t1 = u * P, min(s, (u + 1) * P)
        kp[bt_row[u], :, : t1 - t0, :] = K[t0:t1].transpose(1, 0, 2)
        vp[bt_row[u], :, : t1 - t0, :] = V[t0:t1].transpose(1, 0, 2)
    return kp, vp
