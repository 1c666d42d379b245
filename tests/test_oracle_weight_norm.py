"""Pins of the oracle's weight normalisation (P:149-150 [§VI]), all -m "not gpu".

Each pin is fixed by something other than the oracle itself: SPEC's worked examples, central
finite differences of the loss through (v, g), the invariances the parameterisation implies, and
the function-preserving initialisation."""
import numpy as np
import pytest

from oracle import mlstm_oracle as O


def test_spec_worked_examples():
    """v row (3,4) with g=1 -> (0.6, 0.8); with g=5 -> (3, 4)."""
    v = np.array([[3.0, 4.0]])
    assert np.allclose(O.weight_norm_build(v, np.array([1.0])), [[0.6, 0.8]], atol=1e-15)
    assert np.allclose(O.weight_norm_build(v, np.array([5.0])), [[3.0, 4.0]], atol=1e-15)


def _rand_wn(h, e, rng):
    P = {n: rng.uniform(-0.6, 0.6, size=s) for n, s in O.param_shapes(h, e).items()}
    gains = {n: rng.uniform(0.5, 1.5, size=O.param_shapes(h, e)[n][0]) for n in O.WN_NAMES}
    return O.wn_join(P, gains)


@pytest.mark.parametrize("seed", [0, 1])
def test_wn_backward_matches_central_finite_differences(seed):
    """d loss / d(v, g) for every v and g entry of the 4 normalised matrices (and spot checks of the
    rest) against central differences in fp64."""
    rng = np.random.default_rng(300 + seed)
    h, e, B, T = 4, 3, 2, 4
    flat = _rand_wn(h, e, rng)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    h0 = rng.standard_normal((B, h)) * 0.5
    c0 = rng.standard_normal((B, h)) * 0.5
    scale, denom = 4.0, B * T
    _, g, _, _ = O.wn_loss_and_grads(flat, h, e, by, h0, c0, scale=scale)

    def f(x):
        P, gains = O.wn_split(x, h, e)
        return O.forward(O.wn_effective(P, gains), by, h0, c0)[0] * scale / denom

    base = O.param_count(h, e)
    offs, off = {}, 0
    for n in O.PARAM_NAMES:
        offs[n] = off
        off += int(np.prod(O.param_shapes(h, e)[n]))
    idx = []
    for n in O.WN_NAMES:
        idx += list(range(offs[n], offs[n] + int(np.prod(O.param_shapes(h, e)[n]))))
    idx += list(range(base, O.wn_param_count(h, e)))          # every gain
    idx += [offs["b"], offs["W_dec"] + 5, offs["b_dec"] + 7]  # untouched tensors still flow through
    eps = 1e-6
    num = np.empty(len(idx))
    for k, q in enumerate(idx):
        xp, xm = flat.copy(), flat.copy()
        xp[q] += eps
        xm[q] -= eps
        num[k] = (f(xp) - f(xm)) / (2 * eps)
    ana = g[idx]
    err = np.abs(num - ana).max() / np.abs(ana).max()
    assert err < 1e-5, err


def test_scale_invariance_in_v_and_orthogonal_dv():
    """w depends on v_i only through its direction: scaling a row of v leaves the loss unchanged,
    so the gradient w.r.t. v_i is orthogonal to v_i."""
    rng = np.random.default_rng(7)
    h, e, B, T = 8, 4, 3, 3
    flat = _rand_wn(h, e, rng)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    z = np.zeros((B, h))
    l0, g, _, _ = O.wn_loss_and_grads(flat, h, e, by, z, z)
    P, gains = O.wn_split(flat, h, e)
    P2 = {n: P[n].copy() for n in P}
    c = rng.uniform(0.2, 5.0, size=(4 * h, 1))
    P2["W_h"] = P2["W_h"] * c
    P2["W_mx"] = P2["W_mx"] * 3.0
    l1, _, _, _ = O.wn_loss_and_grads(O.wn_join(P2, gains), h, e, by, z, z)
    assert abs(l1 - l0) <= 1e-12 * abs(l0)
    G, _ = O.wn_split(g, h, e)
    for n in O.WN_NAMES:
        dots = (G[n] * P[n]).sum(axis=1)
        assert np.abs(dots).max() <= 1e-12 * (np.abs(G[n]).max() * np.abs(P[n]).max() * P[n].shape[1]), n


def test_init_is_function_preserving():
    """g_i = ||v_i|| at init: the effective weights equal the plain init up to fp32 rounding of g."""
    h, e = 16, 8
    flat = O.wn_init(h, e, seed=0x5EED)
    assert flat.size == O.wn_param_count(h, e) == O.param_count(h, e) + 10 * h
    P, gains = O.wn_split(flat, h, e)
    plain = O.init_params(h, e, seed=0x5EED)
    W = O.wn_effective(P, gains)
    for n in O.PARAM_NAMES:
        assert np.allclose(W[n], plain[n], rtol=1e-7, atol=0), n
    for n in O.WN_NAMES:
        assert np.array_equal(gains[n], gains[n].astype(np.float32).astype(np.float64))


def test_wn_train_step_reduces_loss_on_repeated_batch():
    """One trajectory property of the whole wn step (Adam on v and g): a few steps on one batch
    lower its loss."""
    h, e, B, T = 8, 8, 4, 6
    st = O.new_train_state(h, e, B, seed=1, weight_norm=True)
    rng = np.random.default_rng(3)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    losses = []
    for _ in range(6):
        st.h_state[:] = 0.0
        st.c_state[:] = 0.0
        losses.append(O.train_step(st, by, lr0=1e-2)["loss_nats"])
    assert losses[-1] < losses[0]
