"""GPU parity of the chunked prefill (NEXT-3): after appending ntok tokens at positions
n0 .. n0+ntok-1, query i attends causally to tokens t <= n0 + i (Eq.4 with the causal mask,
PAPER.md:61-67), against the oracle's decode_heads over the first n0 + i + 1
tokens, on the same seeded rows; and the cache the prefill wrote serves a following decode step."""
import numpy as np
import pytest

import oracle
import synth
from helpers import GpuCase, Shape, assert_close_bf16

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

PF = Shape(L=3, m=32, g=8, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=16, dtype="bf16")
PF_GS7 = Shape(L=2, m=28, g=4, d=128, F=1, delta=[1], k=256, S=4, Lw=32, block=16, dtype="bf16")
PF_D64 = Shape(L=2, m=16, g=2, d=64, F=1, delta=[1], k=128, S=4, Lw=32, block=16, dtype="bf16")


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).cuda()


def _run_prefill(shape, seed, batch, n0, ntok, layer):
    case = GpuCase(shape, seed, batch=batch, s_pre=n0, max_seq=n0 + ntok + 64)
    q = np.stack([np.stack([synth.q_rows(seed, layer, b, n0 + i + 1, shape.m, shape.d, "bf16")
                            for i in range(ntok)]) for b in range(batch)])
    kn = np.stack([synth.kv_rows(seed, layer, b, n0, n0 + ntok, shape.g, shape.d, "bf16", "k") for b in range(batch)])
    vn = np.stack([synth.kv_rows(seed, layer, b, n0, n0 + ntok, shape.g, shape.d, "bf16", "v") for b in range(batch)])
    out = torch.empty((batch, ntok, shape.m, shape.d), dtype=torch.float32, device="cuda")
    lse = torch.empty((batch, ntok, shape.m), dtype=torch.float32, device="cuda")
    case.stack.prefill(layer, _bf16(q), _bf16(kn), _bf16(vn), out, lse)
    torch.cuda.synchronize()
    assert case.stack.get_error() == 0
    return case, q, out.cpu().numpy(), lse.cpu().numpy()


@pytest.mark.parametrize("shape,n0,ntok", [(PF, 1000, 37), (PF, 0, 50), (PF_GS7, 333, 40), (PF_D64, 517, 33)],
                         ids=["m32g8", "from-empty", "gs7", "d64"])
def test_prefill_causal_parity(shape, n0, ntok):
    batch, layer, seed = 2, 0, 71
    case, q, out, lse = _run_prefill(shape, seed, batch, n0, ntok, layer)
    scale = shape.oracle_config().scale
    for b in range(batch):
        K = synth.kv_rows(seed, layer, b, 0, n0 + ntok, shape.g, shape.d, "bf16", "k")
        V = synth.kv_rows(seed, layer, b, 0, n0 + ntok, shape.g, shape.d, "bf16", "v")
        kv = oracle.SeqKV.from_contiguous(K, V, 16)
        for i in range(ntok):
            r_out, r_lse, _ = oracle.decode_heads(q[b, i], kv, n0 + i + 1, scale)
            assert_close_bf16(out[b, i], r_out, f"seq {b} token {i}")
            assert np.max(np.abs(lse[b, i] - r_lse)) <= 2e-4


def test_prefill_then_decode_step():
    """The rows the prefill appended are the cache a decode step then reads (every layer
    prefilled, then one DELTA step through the per-layer ABI against the oracle)."""
    shape, seed, batch, n0, ntok = PF, 73, 1, 900, 99
    case = GpuCase(shape, seed, batch=batch, s_pre=n0, max_seq=n0 + ntok + 64)
    for layer in range(shape.L):
        q = np.stack([np.stack([synth.q_rows(seed, layer, b, n0 + i + 1, shape.m, shape.d, "bf16")
                                for i in range(ntok)]) for b in range(batch)])
        kn = np.stack([synth.kv_rows(seed, layer, b, n0, n0 + ntok, shape.g, shape.d, "bf16", "k")
                       for b in range(batch)])
        vn = np.stack([synth.kv_rows(seed, layer, b, n0, n0 + ntok, shape.g, shape.d, "bf16", "v")
                       for b in range(batch)])
        out = torch.empty((batch, ntok, shape.m, shape.d), dtype=torch.float32, device="cuda")
        case.stack.prefill(layer, _bf16(q), _bf16(kn), _bf16(vn), out)
    s = n0 + ntok + 1
    out, lse, plans = case.step_layers(s)
    from helpers import oracle_step
    ref = oracle_step(shape, seed, 0, s)
    for l in range(shape.F):                    # full layers: no plan near-tie ambiguity
        assert_close_bf16(out[l, 0], ref[l][0], f"layer {l}")
