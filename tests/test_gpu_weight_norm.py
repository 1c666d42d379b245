"""GPU parity of the weight-normalised step (Q24) against the oracle,
through the C ABI: init, one step (loss, dv and dg of every row, the Adam update) in fp32 and mixed
mode, and a 10-step fp32 trace."""
import numpy as np
import pytest

from gpu_helpers import TOL, make_model, inputs, to_dev, rel_l2, cosine
import oracle.mlstm_oracle as O

pytestmark = pytest.mark.gpu


def _compare(g_gpu, g_ref, h, e, precision):
    G, Gg = O.wn_split(np.asarray(g_gpu, dtype=np.float64), h, e)
    R, Rg = O.wn_split(g_ref, h, e)
    rep = {n: (rel_l2 if precision == "fp32" else cosine)(G[n], R[n]) for n in O.PARAM_NAMES}
    rep.update({"g_" + n: (rel_l2 if precision == "fp32" else cosine)(Gg[n], Rg[n]) for n in O.WN_NAMES})
    return rep


def test_init_matches_oracle():
    h, e, B, T = 128, 64, 4, 8
    m = make_model(h, e, B, T, "mixed", push_oracle=False, weight_norm=1)
    got = m.get_params().astype(np.float64)
    ref = O.wn_init(h, e, seed=0x5EED)
    assert got.size == ref.size == O.wn_param_count(h, e)
    base = O.param_count(h, e)
    assert np.array_equal(got[:base], ref[:base])              # v: the plain counter-based init
    assert np.allclose(got[base:], ref[base:], rtol=2e-7, atol=0)  # gains: ||v|| (fp64 sums, fp32)


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
@pytest.mark.parametrize("h,e,B,T", [(64, 64, 4, 16), (128, 64, 130, 5)])
def test_step_matches_oracle(h, e, B, T, precision):
    m = make_model(h, e, B, T, precision, weight_norm=1)
    theta0 = O.wn_init(h, e, seed=0x5EED)          # oracle values in, pushed through the ABI
    m.set_params(theta0)
    by = inputs(B, T)
    res = m.train_step(to_dev(by))
    z = np.zeros((B, h))
    alpha = 65536.0
    loss_ref, g_ref, _, _ = O.wn_loss_and_grads(theta0, h, e, by, z, z, scale=alpha)
    g_ref = g_ref / alpha
    loss_ref /= B * T
    tol = TOL[precision]
    assert abs(res["loss_nats"] - loss_ref) / loss_ref <= tol["loss_rel"], (res, loss_ref)
    assert not res["skipped"]
    rep = _compare(m.get_grads(), g_ref, h, e, precision)
    for n, v in rep.items():
        if precision == "fp32":
            assert v <= tol["grad_rel_l2"], (n, v, rep)
        else:
            assert v >= tol["grad_cos"], (n, v, rep)
    # Adam on (v, g) with the GPU's own gradients
    theta1 = m.get_params().astype(np.float64)
    st = O.AdamState(np.zeros_like(theta0), np.zeros_like(theta0))
    th_ref, _ = O.adam_apply(theta0.astype(np.float32).astype(np.float64), m.get_grads().astype(np.float64), st,
                             O.lr_at(3e-3, 0, 100_000))
    assert rel_l2(theta1 - theta0, th_ref - theta0) < 1e-3


def test_ten_step_fp32_trace():
    h, e, B, T = 64, 64, 4, 16
    m = make_model(h, e, B, T, "fp32", weight_norm=1)
    st = O.new_train_state(h, e, B, seed=0x5EED, weight_norm=True)
    m.set_params(st.theta)                         # identical starting point, oracle -> GPU
    for k in range(10):
        by = inputs(B, T, k=k)
        r = m.train_step(to_dev(by))
        ro = O.train_step(st, by)
        assert abs(r["loss_nats"] - ro["loss_nats"]) <= 1e-4 * ro["loss_nats"], (k, r, ro)
    assert rel_l2(m.get_params().astype(np.float64), st.theta) < 1e-4
