"""GPU tests of the C-ABI step contract (include/mlstm.h): MLSTM_ASYNC result delivery through the
pinned ring and mlstm_sync, and the divergence detector (MLSTM_EDIVERGED)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_1808_01371_b200 as M  # noqa: E402
from gpu_helpers import inputs, make_model, oracle_theta, to_dev  # noqa: E402

FIELDS = ("loss_nats", "bpc", "lr", "loss_scale", "skipped", "step", "applied")


@pytest.mark.parametrize("n_async", [3, 11])
def test_async_results_are_delivered_in_order(n_async):
    """n_async MLSTM_ASYNC steps (11 > the 8-slot ring: the 9th..11th deliver the oldest early), then
    mlstm_sync: every result equals the one the same step returns synchronously, bit for bit."""
    h, e, B, T = 128, 64, 8, 6
    batches = [inputs(B, T, k=k) for k in range(n_async)]
    ref = make_model(h, e, B, T, "mixed")
    want = [ref.train_step(to_dev(by)) for by in batches]
    ref.close()
    m = make_model(h, e, B, T, "mixed")
    devs = [to_dev(by) for by in batches]
    outs = [m.train_step_async(d) for d in devs]
    m.sync()
    got = [o.as_dict() for o in outs]
    for k, (g, w) in enumerate(zip(got, want)):
        assert g["step"] == k
        for f in FIELDS:
            assert g[f] == w[f], (k, f, g[f], w[f])
    # a later synchronous step continues the same trajectory
    r = m.train_step(to_dev(inputs(B, T, k=n_async)))
    assert r["step"] == n_async
    m.close()


def test_nonfinite_loss_trips_divergence_detector():
    """A NaN in the decoder weights makes every loss non-finite (and every step skipped); after
    diverge_patience such steps in a row the step returns MLSTM_EDIVERGED, also when the steps were
    enqueued with MLSTM_ASYNC (reported by the delivering call)."""
    h, e, B, T = 64, 64, 4, 5
    for asynchronous in (False, True):
        m = make_model(h, e, B, T, "mixed", diverge_patience=3)
        th = oracle_theta(h, e).astype(np.float32)
        th[-300] = np.nan  # inside W_dec
        m.set_params(th)
        by = to_dev(inputs(B, T))
        if not asynchronous:
            for _ in range(2):
                r = m.train_step(by)
                assert not np.isfinite(r["loss_nats"]) and r["skipped"] == 1
            with pytest.raises(M.MlstmError) as ei:
                m.train_step(by)
        else:
            outs = [m.train_step_async(by) for _ in range(3)]
            with pytest.raises(M.MlstmError) as ei:
                m.sync()
            assert all(o.skipped == 1 for o in outs)
        assert ei.value.status == M.MLSTM_EDIVERGED
        m.close()


def test_finite_steps_reset_the_divergence_run():
    """Two non-finite steps, then finite ones: the run restarts, no MLSTM_EDIVERGED."""
    h, e, B, T = 64, 64, 4, 5
    m = make_model(h, e, B, T, "mixed", diverge_patience=3)
    th = oracle_theta(h, e).astype(np.float32)
    bad = th.copy()
    bad[-300] = np.nan
    by = to_dev(inputs(B, T))
    m.set_params(bad)
    for _ in range(2):
        m.train_step(by)
    m.set_params(th)
    for _ in range(4):
        r = m.train_step(by)
        assert np.isfinite(r["loss_nats"])
    m.close()
