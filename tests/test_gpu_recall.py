"""GPU parity of the attention-recall diagnostic (Eq.9; NEXT-2): the fraction of
a layer's exact full-attention mass kept by the plan it attended, per head, against the oracle's
`attention_recall` (pinned by the SPEC examples) on the oracle's own full-attention weights."""
import numpy as np
import pytest

import oracle
import synth
from helpers import GpuCase, Shape, oracle_layer, planting_for
from test_gpu_quest import QUEST_SMALL, QuestCase

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SHAPE = Shape(L=4, m=32, g=8, d=128, F=1, delta=[1], k=512, S=4, Lw=32, block=16, dtype="bf16")


def _oracle_recall(shape, seed, layer, seq, s, units, planting=None):
    _, _, alpha = oracle_layer(shape, seed, layer, seq, s, planting, want_alpha=True)
    toks = oracle.units_to_tokens(np.asarray(units, np.int64), shape.block, s)
    return np.array([oracle.attention_recall(alpha[j], toks) for j in range(shape.m)])


@pytest.mark.parametrize("kind", ["iid", "planted"])
def test_recall_delta_layers(kind):
    s = 3001
    planting = planting_for(SHAPE, s) if kind == "planted" else None
    case = GpuCase(SHAPE, 61, batch=2, s_pre=s - 1, max_seq=s + 63, planting=planting)
    q, _, _ = case.inputs(s)
    out, lse, plans = case.step_layers(s)
    rec = torch.empty((4, 2, SHAPE.m), dtype=torch.float32, device="cuda")
    for l in (1, 2, 3):                        # the Delta layer and the two sparse layers it governs
        case.stack.attention_recall(l, q[l], rec[l])
    torch.cuda.synchronize()
    assert case.stack.get_error() == 0
    got = rec.cpu().numpy()
    for l in (1, 2, 3):
        for b in range(2):
            ref = _oracle_recall(SHAPE, 61, l, b, s, plans[1][b], planting)
            assert np.max(np.abs(got[l, b] - ref)) <= 1e-4, f"recall layer {l} seq {b}"
    if kind == "planted":   # the planted set holds most of the mass of the Delta layer
        assert got[1].mean() > 0.5


def test_recall_quest_layer():
    s = 2101
    case = QuestCase(QUEST_SMALL, 63, batch=1, s_pre=s - 1, max_seq=s + 63)
    q, k, v = case.inputs(s)
    out = torch.empty((3, 1, 32, 128), dtype=torch.float32, device="cuda")
    rec = torch.empty((1, 32), dtype=torch.float32, device="cuda")
    cap = case.stack.plan_capacity
    idx = torch.empty((1, cap), dtype=torch.int32, device="cuda")
    cnt = torch.empty((1,), dtype=torch.int32, device="cuda")
    for l in range(2):
        case.stack.append_decode_layer(l, k[l], v[l], q[l], out[l])
    case.stack.copy_plan(1, 1, idx, cnt)
    case.stack.attention_recall(1, q[1], rec)
    torch.cuda.synchronize()
    units = idx[0, : int(cnt[0])].cpu().numpy()
    ref = _oracle_recall(QUEST_SMALL, 63, 1, 0, s, units)
    assert np.max(np.abs(rec.cpu().numpy()[0] - ref)) <= 1e-4
