"""Device-side fills with the seeded generator of synth/__init__.py (libsynth.so).

Bit-identical to the numpy generator (checked by tests/test_gpu_parity.py).  Used by the
GPU tests and bench.py to build caches of the paper's shapes directly in HBM.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import TAG_K, TAG_Q, TAG_V, Planting, planted_units, sigma

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsynth.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} missing: run `make`")
        L = ctypes.CDLL(_LIB)
        vp, i32 = ctypes.c_void_p, ctypes.c_int
        L.synth_fill_pool.argtypes = [vp, i32, ctypes.c_uint64, i32, i32, i32, i32, i32, i32, i32, i32, i32, vp, i32,
                                      vp, i32, i32, vp, ctypes.c_float, i32, i32, vp]
        L.synth_fill_rows.argtypes = [vp, i32, ctypes.c_uint64, i32, i32, i32, i32, vp, i32, i32, i32, vp, vp, vp,
                                      ctypes.c_float, vp]
        _lib = L
    return _lib


def _stream():
    return torch.cuda.current_stream().cuda_stream


def plant_tables(seed, layers, batch, d, planting: Planting | None, n_units: int, device):
    """(mask [nl][batch][n_units] uint8, sigma [nl][batch][d] f32) on device, or (None, None)."""
    if planting is None or planting.count <= 0:
        return None, None
    mask = np.zeros((len(layers), batch, n_units), np.uint8)
    sg = np.zeros((len(layers), batch, d), np.float32)
    for i, l in enumerate(layers):
        for b in range(batch):
            mask[i, b, planted_units(seed, l, b, planting)] = 1
            sg[i, b] = sigma(seed, l, b, d)
    return torch.from_numpy(mask).to(device), torch.from_numpy(sg).to(device)


def fill_pools(kv_pool, block_table, seed: int, s_fill: int, batch: int, layers, planting=None):
    """Fill logical rows t < s_fill of sequences [0,batch) for the given (contiguous) layers of a
    pool [L][phys][g][2][P][d] (K rows then V rows per (page, head))."""
    L_, phys, g, two, P, d = kv_pool.shape
    assert two == 2
    bf16 = 1 if kv_pool.dtype == torch.bfloat16 else 0
    layers = list(layers)
    l0, nl = layers[0], len(layers)
    assert layers == list(range(l0, l0 + nl))
    n_units = -(-s_fill // (planting.block if planting else 1)) if planting else 1
    mask, sg = plant_tables(seed, layers, batch, d, planting, max(n_units, 1), kv_pool.device)
    for slot, tag in ((0, TAG_K), (1, TAG_V)):
        use_plant = planting is not None and tag == TAG_K and mask is not None
        st = lib().synth_fill_pool(kv_pool.data_ptr(), bf16, seed, tag, l0, nl, batch, s_fill, g, d, P, phys,
                                   block_table.data_ptr(), block_table.shape[1],
                                   mask.data_ptr() if use_plant else None,
                                   planting.block if use_plant else 1, mask.shape[2] if use_plant else 1,
                                   sg.data_ptr() if use_plant else None,
                                   float(planting.B) if use_plant else 0.0, 2, slot, _stream())
        assert st == 0, f"synth_fill_pool failed: {st}"


def fill_queries(out, seed: int, layers, s_per_seq, planting=None):
    """out [nl][batch][m][d]: queries of each layer at the step whose cache holds s tokens."""
    nl, batch, m, d = out.shape
    layers = list(layers)
    bf16 = 1 if out.dtype == torch.bfloat16 else 0
    steps = torch.tensor(list(s_per_seq), dtype=torch.int32, device=out.device)
    planted = sg = None
    if planting is not None and planting.count > 0:
        planted = torch.ones((nl, batch), dtype=torch.uint8, device=out.device)
        sg = torch.from_numpy(np.stack([np.stack([sigma(seed, l, b, d) for b in range(batch)]) for l in layers])
                              ).to(out.device)
    st = lib().synth_fill_rows(out.data_ptr(), bf16, seed, TAG_Q, layers[0], nl, batch, steps.data_ptr(), 1, m, d,
                               None, planted.data_ptr() if planted is not None else None,
                               sg.data_ptr() if sg is not None else None,
                               float(planting.G) if planted is not None else 0.0, _stream())
    assert st == 0


def fill_new_kv(k_out, v_out, seed: int, layers, pos_per_seq):
    """k_out, v_out [nl][batch][g][d]: cache rows at position pos (the token appended this step)."""
    nl, batch, g, d = k_out.shape
    layers = list(layers)
    bf16 = 1 if k_out.dtype == torch.bfloat16 else 0
    offs = torch.tensor([int(p) * g * d for p in pos_per_seq], dtype=torch.int64, device=k_out.device)
    for out, tag in ((k_out, TAG_K), (v_out, TAG_V)):
        st = lib().synth_fill_rows(out.data_ptr(), bf16, seed, tag, layers[0], nl, batch, offs.data_ptr(), 0, g, d,
                                   offs.data_ptr(), None, None, 0.0, _stream())
        assert st == 0
