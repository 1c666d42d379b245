"""Pins for the fp64 oracle against what the paper and mathematics fix (not against itself).

Each test names the passage it follows.  All CPU-only (-m "not gpu").
"""
import csv
import math
import os

import numpy as np
import pytest
import torch

from oracle import mlstm_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand_params(h, e, rng, scale=0.5):
    P = {}
    for n, s in O.param_shapes(h, e).items():
        P[n] = rng.standard_normal(s) * scale
    return P


def _read_csv(name):
    with open(os.path.join(GOLD, name)) as f:
        rows = [r for r in f if not r.startswith("#")]
    return list(csv.DictReader(rows))


# ---------------------------------------------------------------- init (Q12) ----------

def test_splitmix64_matches_published_reference():
    with open(os.path.join(GOLD, "splitmix64_seed0.txt")) as f:
        ref = [int(l, 16) for l in f if l.strip() and not l.startswith("#")]
    got = O.splitmix64(0, np.arange(3, dtype=np.uint64))
    assert [int(v) for v in got] == ref


def test_init_ranges_and_biases():
    h, e = 16, 8
    P = O.init_params(h, e, seed=1234)
    for n, s in O.param_shapes(h, e).items():
        if len(s) == 1:
            assert np.all(P[n] == 0.0)
        else:
            bound = 1.0 / math.sqrt(s[1])
            assert np.abs(P[n]).max() <= bound
            assert np.abs(P[n]).max() > 0.8 * bound            # actually spans the range
            assert np.all(P[n].astype(np.float32).astype(np.float64) == P[n])   # fp32 values
    assert O.param_count(4096, 64) == 86_278_400


# ---------------------------------------------------------------- forward -------------

def test_forward_reduces_to_torch_lstm_when_mx_is_one():
    """If E has a constant-1 column selected by W_mx, mx == 1 and m == W_mh h, so the mLSTM is an
    LSTM with W_hh = W_h W_mh (library routine torch.nn.LSTM, fp64)."""
    rng = np.random.default_rng(0)
    h, e, B, T = 6, 5, 3, 7
    P = _rand_params(h, e, rng)
    P["E"][:, 0] = 1.0
    P["W_mx"][:] = 0.0
    P["W_mx"][:, 0] = 1.0
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    h0 = rng.standard_normal((B, h)) * 0.3
    c0 = rng.standard_normal((B, h)) * 0.3
    _, cache, (hT, cT) = O.forward(P, by, h0, c0)

    lstm = torch.nn.LSTM(e, h, batch_first=True).double()
    perm = np.concatenate([np.arange(0, h), np.arange(h, 2 * h), np.arange(3 * h, 4 * h),
                           np.arange(2 * h, 3 * h)])        # ours (i,f,o,u) -> torch (i,f,g,o)
    with torch.no_grad():
        lstm.weight_ih_l0.copy_(torch.from_numpy(P["W_x"][perm]))
        lstm.weight_hh_l0.copy_(torch.from_numpy((P["W_h"] @ P["W_mh"])[perm]))
        lstm.bias_ih_l0.copy_(torch.from_numpy(P["b"][perm]))
        lstm.bias_hh_l0.zero_()
        x = torch.from_numpy(P["E"][by[:, :T]])
        out, (hn, cn) = lstm(x, (torch.from_numpy(h0)[None], torch.from_numpy(c0)[None]))
    ours = np.stack(cache.hs[1:], axis=1)
    assert np.abs(out.numpy() - ours).max() < 1e-12
    assert np.abs(cn[0].numpy() - cT).max() < 1e-12
    # logits and loss against torch's cross-entropy on the same hidden states
    y = torch.from_numpy(ours) @ torch.from_numpy(P["W_dec"]).T + torch.from_numpy(P["b_dec"])
    ce = torch.nn.functional.cross_entropy(y.reshape(-1, 256), torch.from_numpy(by[:, 1:].astype(np.int64)).reshape(-1),
                                           reduction="sum")
    loss_sum, _, _ = O.forward(P, by, h0, c0)
    assert abs(loss_sum - ce.item()) < 1e-10 * abs(ce.item())


def test_forward_is_an_lstm_with_input_dependent_transition():
    """The multiplicative LSTM (P:36, P:55 defer to Krause et al. 2016; reading Q1) is an LSTM whose
    recurrent matrix depends on the current input: W_hh(x_t) = W_h diag(W_mx x_t) W_mh.  Pinned step by
    step against the library cell torch.nn.LSTMCell (fp64), fed per row and timestep with that
    transition.  General E and W_mx (no constant column), so dropping the mx factor, transposing W_mx,
    or gathering mx with another byte or unit changes the transition and fails."""
    rng = np.random.default_rng(11)
    h, e, B, T = 5, 4, 3, 6
    P = _rand_params(h, e, rng)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    h0 = rng.standard_normal((B, h)) * 0.3
    c0 = rng.standard_normal((B, h)) * 0.3
    loss_sum, cache, (hT, cT) = O.forward(P, by, h0, c0)
    perm = np.concatenate([np.arange(0, h), np.arange(h, 2 * h), np.arange(3 * h, 4 * h),
                           np.arange(2 * h, 3 * h)])        # ours (i,f,o,u) -> torch (i,f,g,o)
    cell = torch.nn.LSTMCell(e, h).double()
    ref_loss = 0.0
    with torch.no_grad():
        cell.weight_ih.copy_(torch.from_numpy(P["W_x"][perm]))
        cell.bias_ih.copy_(torch.from_numpy(P["b"][perm]))
        cell.bias_hh.zero_()
        for b in range(B):
            hb, cb = torch.from_numpy(h0[b:b + 1]), torch.from_numpy(c0[b:b + 1])
            for t in range(T):
                x = torch.from_numpy(P["E"][by[b, t]][None])
                w_hh = P["W_h"] @ np.diag(P["W_mx"] @ P["E"][by[b, t]]) @ P["W_mh"]
                cell.weight_hh.copy_(torch.from_numpy(w_hh[perm]))
                hb, cb = cell(x, (hb, cb))
                assert np.abs(hb.numpy()[0] - cache.hs[t + 1][b]).max() < 1e-12
                assert np.abs(cb.numpy()[0] - cache.c[t + 1][b]).max() < 1e-12
                y = hb @ torch.from_numpy(P["W_dec"]).T + torch.from_numpy(P["b_dec"])
                ref_loss += torch.nn.functional.cross_entropy(y, torch.tensor([int(by[b, t + 1])]),
                                                              reduction="sum").item()
    assert abs(loss_sum - ref_loss) < 1e-10 * abs(ref_loss)


def test_mixed_step_overflow_decision_uses_fp16_gradients():
    """the step is skipped when the (alpha-scaled) fp16 weight gradients overflow.  Far from the
    binary16 threshold the decision is fixed: alpha = 1 keeps every scaled gradient well inside 65504
    (applied); alpha = 2^40 pushes them past 65520 (skipped, alpha halves, masters and Adam state
    untouched).  fp32 mode (no fp16 buffer) applies both."""
    h, e, B, T = 8, 4, 2, 5
    rng = np.random.default_rng(12)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    for alpha, skip_mixed in ((1.0, False), (2.0 ** 40, True)):
        for precision, want in (("mixed", skip_mixed), ("fp32", False)):
            st = O.new_train_state(h, e, B, seed=3, scaler=O.ScalerState(alpha=alpha, alpha_max=2.0 ** 50))
            theta0 = st.theta.copy()
            r = O.train_step(st, by, precision=precision)
            g_scaled = np.abs(r["grads"]).max() * alpha
            assert (g_scaled < 65504 / 4) if alpha == 1.0 else (g_scaled > 4 * 65520)
            assert r["skipped"] == want
            assert np.array_equal(st.theta, theta0) == want
            assert st.scaler.alpha == (alpha / 2 if want else alpha)


def test_forward_zero_weights_closed_form():
    """All weights and biases zero: i=f=o=1/2, u=0 => c_t = c_{t-1}/2, h_t = tanh(c_t)/2."""
    h, e, B, T = 4, 3, 2, 5
    P = {n: np.zeros(s) for n, s in O.param_shapes(h, e).items()}
    rng = np.random.default_rng(1)
    c0 = rng.standard_normal((B, h))
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    _, cache, (hT, cT) = O.forward(P, by, np.zeros((B, h)), c0)
    for t in range(T):
        c = c0 * 0.5 ** (t + 1)
        assert np.array_equal(cache.c[t + 1], c)
        assert np.abs(cache.hs[t + 1] - 0.5 * np.tanh(c)).max() < 1e-15


def test_uniform_logits_give_8_bpc_and_closed_form_dy():
    """W_dec = 0, b_dec = 0 => loss = ln 256 nats = 8 bits exactly per char,
    and dL/db_dec = (n/256 - count_v)/(B*T)."""
    rng = np.random.default_rng(2)
    h, e, B, T = 5, 4, 3, 6
    P = _rand_params(h, e, rng)
    P["W_dec"][:] = 0.0
    P["b_dec"][:] = 0.0
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    loss_sum, g, _, _ = O.loss_and_grads(P, by, np.zeros((B, h)), np.zeros((B, h)))
    L = loss_sum / (B * T)
    assert abs(L - math.log(256)) < 1e-14
    assert abs(O.bpc_from_nats(L) - 8.0) < 1e-13
    counts = np.bincount(by[:, 1:].ravel(), minlength=256)
    expect = (B * T / 256.0 - counts) / (B * T)
    assert np.abs(g["b_dec"] - expect).max() < 1e-15


def test_state_carry_two_windows_equal_one_long_window():
    """TBTT state persistence: forward over 2T == two T-windows with carried state."""
    rng = np.random.default_rng(3)
    h, e, B, T = 5, 4, 2, 6
    P = _rand_params(h, e, rng)
    s = rng.integers(0, 256, size=(B, 2 * T + 1)).astype(np.uint8)
    z = np.zeros((B, h))
    _, c_long, st_long = O.forward(P, s, z, z)
    _, c1, st1 = O.forward(P, s[:, :T + 1], z, z)
    _, c2, st2 = O.forward(P, s[:, T:], *st1)
    assert np.array_equal(np.stack(c_long.logits), np.stack(c1.logits + c2.logits))
    assert np.array_equal(st_long[0], st2[0]) and np.array_equal(st_long[1], st2[1])


def test_reset_zeroes_state_rows():
    rng = np.random.default_rng(4)
    h, e, B, T = 4, 3, 3, 4
    P = _rand_params(h, e, rng)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    h0, c0 = rng.standard_normal((B, h)), rng.standard_normal((B, h))
    r = np.array([0, 1, 0], dtype=np.uint8)
    _, ca, _ = O.forward(P, by, h0, c0, reset=r)
    h0z, c0z = h0.copy(), c0.copy()
    h0z[1] = 0
    c0z[1] = 0
    _, cb, _ = O.forward(P, by, h0z, c0z)
    assert np.array_equal(np.stack(ca.logits), np.stack(cb.logits))


# ---------------------------------------------------------------- backward ------------

@pytest.mark.parametrize("seed", [0, 1, 2])
def test_backward_matches_central_finite_differences(seed):
    """Every one of the 8 parameter tensors against central differences in fp64."""
    rng = np.random.default_rng(100 + seed)
    h, e, B, T = 4, 3, 2, 5
    P = _rand_params(h, e, rng, scale=0.6)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    by[:, 2] = by[:, 0]                                   # a repeated byte exercises np.add.at
    h0 = rng.standard_normal((B, h)) * 0.5
    c0 = rng.standard_normal((B, h)) * 0.5
    denom, scale = B * T * 3, 8.0
    _, g, _, _ = O.loss_and_grads(P, by, h0, c0, n_global_rows=3 * B, scale=scale)

    def f(PP):
        return O.forward(PP, by, h0, c0)[0] * scale / denom

    eps = 1e-6
    for n in O.PARAM_NAMES:
        if n == "E":
            idx = sorted(set(by[:, :T].ravel().tolist()))[:3]
            coords = [(v, j) for v in idx for j in range(e)]
        else:
            coords = list(np.ndindex(P[n].shape))
        num = np.zeros(len(coords))
        ana = np.zeros(len(coords))
        for k, cidx in enumerate(coords):
            Pp = {m: P[m].copy() for m in P}
            Pm = {m: P[m].copy() for m in P}
            Pp[n][cidx] += eps
            Pm[n][cidx] -= eps
            num[k] = (f(Pp) - f(Pm)) / (2 * eps)
            ana[k] = g[n][cidx]
        err = np.abs(num - ana).max() / max(np.abs(ana).max(), 1e-12)
        assert err < 1e-5, (n, err)


def test_embedding_gradient_support_is_input_bytes():
    """dE rows are nonzero exactly for bytes used as inputs (bytes[:, :T]); others exactly 0 (Q21)."""
    rng = np.random.default_rng(5)
    h, e, B, T = 4, 3, 3, 6
    P = _rand_params(h, e, rng)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    _, g, _, _ = O.loss_and_grads(P, by, np.zeros((B, h)), np.zeros((B, h)))
    nz = set(np.nonzero(np.abs(g["E"]).sum(axis=1))[0].tolist())
    assert nz == set(by[:, :T].ravel().tolist())


def test_loss_scale_invariance_fp64():
    """Gradients of alpha*L divided by alpha equal gradients of L."""
    rng = np.random.default_rng(6)
    h, e, B, T = 4, 3, 2, 4
    P = _rand_params(h, e, rng)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    z = np.zeros((B, h))
    _, g1, _, _ = O.loss_and_grads(P, by, z, z, scale=1.0)
    _, g2, _, _ = O.loss_and_grads(P, by, z, z, scale=1024.0)
    for n in O.PARAM_NAMES:
        assert np.array_equal(g1[n] * 1024.0, g2[n])


# ---------------------------------------------------------------- optimiser / schedule -

def test_adam_matches_torch_optim_adam_fp64():
    rng = np.random.default_rng(7)
    theta = rng.standard_normal(50)
    p = torch.nn.Parameter(torch.from_numpy(theta.copy()))
    opt = torch.optim.Adam([p], lr=3e-3, betas=(0.9, 0.999), eps=1e-8)
    st = O.AdamState(np.zeros(50), np.zeros(50))
    th = theta.copy()
    for k in range(12):
        g = rng.standard_normal(50) * (k + 1)
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        th, st = O.adam_apply(th, g, st, 3e-3)
    assert np.abs(th - p.detach().numpy()).max() < 1e-14
    assert st.tau == 12


def test_adam_first_step_closed_form_and_lr_zero():
    g = np.array([0.5, -2.0, 1e-3])
    st = O.AdamState(np.zeros(3), np.zeros(3))
    th, _ = O.adam_apply(np.zeros(3), g, st, 1e-3)
    assert np.abs(th - (-1e-3 * g / (np.abs(g) + 1e-8))).max() < 1e-18
    th0 = np.array([1.0, 2.0, 3.0])
    th1, _ = O.adam_apply(th0, g, st, 0.0)
    assert np.array_equal(th0, th1)


def test_lr_schedule_values_from_paper():
    """start at 3e-3, linear decay to zero over 100,000 iterations."""
    assert O.lr_at(3e-3, 0, 100_000) == 3e-3
    assert abs(O.lr_at(3e-3, 50_000, 100_000) - 1.5e-3) < 1e-18
    assert O.lr_at(3e-3, 100_000, 100_000) == 0.0
    assert O.lr_at(3e-3, 250_000, 100_000) == 0.0
    vals = [O.lr_at(3e-3, i, 100_000) for i in range(0, 120_000, 977)]
    assert all(a >= b for a, b in zip(vals, vals[1:]))


def test_scale_lr_reproduces_lr_scale_table():
    """Tab. lr_scale: rules from 5e-4 at batch 128."""
    for row in _read_csv("lr_scale_table.csv"):
        got = O.scale_lr(5e-4, row["rule"], int(row["batch"]))
        printed = float(row["printed_lr"])
        two_sig = float(f"{got:.2g}")
        if row["note"] == "Q17":
            assert abs(got - 5.657e-3) < 1e-6 and two_sig != printed
        else:
            assert two_sig == printed, (row, got)
    assert O.scale_lr(5e-4, "none", 32768) == 5e-4


def test_speedup_arithmetic_matches_gpu_scale_table():
    rows = _read_csv("gpu_scale_table.csv")
    t1 = {r["column"]: float(r["s_per_iter"]) for r in rows if r["gpus"] == "1"}
    for r in rows:
        s = O.speedup(int(r["gpus"]), t1[r["column"]], float(r["s_per_iter"]))
        agrees = abs(s - float(r["printed_speedup"])) < 0.1      # the table prints 1 decimal (7.96 -> "7.9")
        assert agrees == bool(int(r["formula_agrees"])), (r, s)
    assert abs(O.speedup(128, 0.81, 0.91) - 113.9) < 0.05       # the printed 109x (Q20)


# ---------------------------------------------------------------- scaler / overflow ----

def test_scaler_spec_traces():
    a, s = O.scaler_step(O.ScalerState(alpha=2.0 ** 16), True)
    assert (a, s.alpha, s.clean) == (False, 2.0 ** 15, 0)
    a, s = O.scaler_step(O.ScalerState(alpha=2.0 ** 14, clean=1999), False)
    assert (a, s.alpha, s.clean) == (True, 2.0 ** 15, 0)
    a, s = O.scaler_step(O.ScalerState(alpha=1.0), True)                  # S:204 clamp
    assert (a, s.alpha) == (False, 1.0)


def test_scaler_properties_random_sequences():
    rng = np.random.default_rng(8)
    for _ in range(200):
        st = O.ScalerState(alpha=2.0 ** int(rng.integers(0, 25)), growth_interval=int(rng.integers(1, 6)))
        clean_run = 0
        for ov in rng.random(60) < rng.random():
            prev = st.alpha
            apply, st = O.scaler_step(st, bool(ov))
            assert apply == (not ov)
            assert 1.0 <= st.alpha <= 2.0 ** 24 and math.log2(st.alpha) == int(math.log2(st.alpha))
            if ov:
                clean_run = 0
                assert st.alpha == max(prev / 2, 1.0)
            else:
                clean_run += 1
                if clean_run == st.growth_interval:
                    assert st.alpha == min(prev * 2, 2.0 ** 24)
                    clean_run = 0
                else:
                    assert st.alpha == prev


def test_fp16_overflow_thresholds():
    """IEEE binary16 RNE: 65504 is the max finite; 65519.99 rounds to it; 65520 rounds to inf (Q13)."""
    assert O.to_fp16(65504.0) == 65504.0
    assert O.to_fp16(65519.99) == 65504.0
    assert np.isinf(O.to_fp16(65520.0))
    assert O.to_fp16(2.0 ** -25) == 0.0                         # tie to even
    assert not O.overflow(O.to_fp16([1.0, -65504.0, 65519.99]))
    assert O.overflow(O.to_fp16([1.0, 65520.0]))
    assert O.overflow(np.array([0.0, np.nan], dtype=np.float16))


def test_skipped_step_leaves_masters_bitwise_unchanged():
    rng = np.random.default_rng(9)
    h, e, B, T = 4, 64, 2, 3
    st = O.new_train_state(h, e, B, seed=3)
    by = rng.integers(0, 256, size=(B, T + 1)).astype(np.uint8)
    th0 = st.theta.copy()
    m0 = st.adam.m.copy()
    out = O.train_step(st, by, grads_hook=lambda g: g * np.inf)   # force an overflow
    assert out["skipped"] and np.array_equal(st.theta, th0) and np.array_equal(st.adam.m, m0)
    assert st.adam.tau == 0 and st.it == 1 and st.scaler.alpha == 2.0 ** 15
    out = O.train_step(st, by)
    assert not out["skipped"] and st.adam.tau == 1 and not np.array_equal(st.theta, th0)
    assert out["lr"] == O.lr_at(3e-3, 1, 100_000)


def test_random_init_loss_is_about_8_bits():
    """Random init => BPC ~ 8 (north_star: "uniform-init loss ~ 8 bits/char")."""
    from synth import bytestream
    h, e, B, T = 64, 64, 4, 16
    P = O.init_params(h, e, seed=0x5EED)
    by = bytestream.window(np.arange(B), 0, T)
    loss, _, _ = O.forward(P, by, np.zeros((B, h)), np.zeros((B, h)))
    bpc = O.bpc_from_nats(loss / (B * T))
    assert 7.5 < bpc < 8.5
