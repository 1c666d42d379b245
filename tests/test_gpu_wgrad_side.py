"""dW_h reduced partly on a side stream while the per-timestep backward recurrence runs
(MLSTM_WGRAD_SIDE=chunks,ch,pairs; mlstm.cu enqueue_train_a): chunk j = timesteps [T-(j+1)ch, T-j*ch)
is reduced into an fp32 partial as soon as the BPTT has produced its dZ rows, and dW_h's main GEMM over
the remaining timesteps adds it before the single fp16 rounding.  dW_h = sum over (t, b) of dZ^T M
(the weight gradient of z_t = W_x x_t + W_h m_t, P:36 mLSTM, summed over the window's timesteps, P:132
TBTT), so the split changes only the fp32 summation order."""
import numpy as np
import pytest

from gpu_helpers import TOL, compare_grads, inputs, make_model, oracle_step, oracle_theta, split, to_dev

pytestmark = pytest.mark.gpu


def _step(monkeypatch, side, h, e, B, T, recurrence=2, **kw):
    if side:
        monkeypatch.setenv("MLSTM_WGRAD_SIDE", side)
    else:
        monkeypatch.delenv("MLSTM_WGRAD_SIDE", raising=False)
    m = make_model(h, e, B, T, "mixed", recurrence=recurrence, **kw)
    r = m.train_step(to_dev(inputs(B, T)))
    g = m.get_grads().astype(np.float64)
    m.close()
    return r, g


@pytest.mark.parametrize("h,B,T,side,recurrence", [(1024, 16, 16, "3,4,3", 2), (256, 16, 9, "2,3,1", 2),
                                                     (1024, 256, 10, "2,3,2", 3)])
def test_side_chunks_match_oracle(monkeypatch, h, B, T, side, recurrence):
    """All 8 gradients against the fp64 oracle (north_star mixed tolerances) with part of dW_h on the side
    stream: several chunks, a ragged main range (T not a multiple of ch), one pair, the persistent forward."""
    e = 64
    r, g = _step(monkeypatch, side, h, e, B, T, recurrence)
    assert np.isfinite(r["loss_nats"]) and not r["skipped"]
    loss_ref, g_ref, _, _ = oracle_step(oracle_theta(h, e), inputs(B, T), h, e)
    assert abs(r["loss_nats"] - loss_ref) / loss_ref <= TOL["mixed"]["loss_rel"]
    rep = compare_grads(g, g_ref, h, e, "mixed")
    for n, v in rep.items():
        assert v >= TOL["mixed"]["grad_cos"], (n, v, rep)


@pytest.mark.parametrize("h,B,T,side,micro", [(1024, 16, 16, "3,4,3", 0), (4096, 256, 8, "1,4,10", 0),
                                               (512, 64, 12, "2,5,2", 16)])
def test_side_chunks_change_only_dW_h_summation_order(monkeypatch, h, B, T, side, micro):
    """Against the same step without side chunks: every other gradient bitwise equal (the side stream
    writes nothing else), dW_h within one fp16 rounding (rel 2^-9; abs 1e-3 of the largest entry where
    the sum cancels) -- also at the C3 width and rows per GPU, and with micro-batches (each pass of the
    step's graph A forks and joins its own side chunks; the fp32 accumulation across passes follows)."""
    e = 64
    kw = {"micro_batch": micro} if micro else {}
    r0, g0 = _step(monkeypatch, None, h, e, B, T, **kw)
    r1, g1 = _step(monkeypatch, side, h, e, B, T, **kw)
    assert r0["loss_nats"] == r1["loss_nats"]
    G0, G1 = split(g0, h, e), split(g1, h, e)
    for n in G0:
        if n != "W_h":
            assert np.array_equal(G0[n], G1[n]), n
    a, b = G1["W_h"], G0["W_h"]
    scale = np.abs(b).max()
    assert scale > 0
    # fp32 sums in another order: one fp16 rounding apart, or a few ulps where the sum cancels
    bad = np.abs(a - b) > 2.0 ** -9 * np.abs(b) + 1e-3 * scale
    assert not bad.any(), (int(bad.sum()), float(np.abs(a - b).max()), scale)

