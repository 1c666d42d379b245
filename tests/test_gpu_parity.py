"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical seeded inputs.

Sizes span several tiles and a ragged tail (B = 130 > 128 rows, h = 128 > 64 columns) and the
BASELINE.json parity configs C1 (h=64, T=16, B=4) and C2 (h=1024, T=64, B=128).
"""
import math

import numpy as np
import pytest

from oracle import mlstm_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

from gpu_helpers import (TOL, oracle_theta, compare_grads, cosine, inputs, make_model, oracle_step, rel_l2, split,  # noqa: E402
                         to_dev)

CASES = [
    # (name, h, e, B, T)
    ("C1", 64, 64, 4, 16),
    ("ragged", 128, 64, 130, 5),
    ("C2", 1024, 64, 128, 64),
]


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
def test_init_matches_oracle_bitwise(precision):
    h, e = 128, 64
    m = make_model(h, e, 8, 4, precision, seed=1234, push_oracle=False)
    got = m.get_params()
    ref = O.flatten(O.init_params(h, e, 1234)).astype(np.float32)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
@pytest.mark.parametrize("name,h,e,B,T", CASES)
def test_train_step_parity(name, h, e, B, T, precision):
    m = make_model(h, e, B, T, precision)
    theta0 = oracle_theta(h, e)
    by = inputs(B, T)
    res = m.train_step(to_dev(by))
    loss_ref, g_ref, (hT, cT), _ = oracle_step(theta0, by, h, e)
    loss_rel = abs(res["loss_nats"] - loss_ref) / abs(loss_ref)
    g = m.get_grads().astype(np.float64)
    rep = compare_grads(g, g_ref, h, e, precision)
    tol = TOL[precision]
    assert loss_rel <= tol["loss_rel"], (loss_rel, res, loss_ref)
    assert res["skipped"] == 0 and res["step"] == 0 and res["applied"] == 1
    assert abs(res["bpc"] - res["loss_nats"] / math.log(2)) < 1e-12
    for n, v in rep.items():
        if precision == "fp32":
            assert v <= tol["grad_rel_l2"], (n, v, rep)
        else:
            assert v >= tol["grad_cos"], (n, v, rep)
    # persisted state = final (h, c) of the window
    hs, cs = m.get_state(0)
    htol = 1e-5 if precision == "fp32" else 2e-3
    assert np.abs(hs - hT).max() <= htol and np.abs(cs - cT).max() <= 10 * htol
    # the Adam update the GPU applied equals the oracle's Adam on the GPU's own gradients
    theta1 = m.get_params().astype(np.float64)
    st = O.AdamState(np.zeros_like(theta0), np.zeros_like(theta0))
    th_ref, _ = O.adam_apply(theta0, g, st, O.lr_at(3e-3, 0, 100_000))
    upd, upd_ref = theta1 - theta0, th_ref - theta0
    assert rel_l2(upd, upd_ref) < 1e-3


def test_multi_step_trace_fp32_tracks_oracle():
    """100 steps (forward, BPTT, scaler, Adam, schedule, persisted state) vs the oracle loop
    (SURVEY 8(d) C4 validation (i): fp32-mode loss trace within rel 1e-3 per step; first 10 steps 1e-4)."""
    h, e, B, T = 64, 64, 4, 16
    m = make_model(h, e, B, T, "fp32")
    st = O.new_train_state(h, e, B, seed=0x5EED)
    assert np.array_equal(st.theta.astype(np.float32), m.get_params())
    worst = 0.0
    for k in range(100):
        by = inputs(B, T, k=k)
        r = m.train_step(to_dev(by))
        ro = O.train_step(st, by)
        rel = abs(r["loss_nats"] - ro["loss_nats"]) / ro["loss_nats"]
        worst = max(worst, rel)
        assert rel <= (1e-4 if k < 10 else 1e-3), (k, r, ro)
        assert r["lr"] == pytest.approx(ro["lr"], rel=1e-12) and r["loss_scale"] == ro["alpha"]
        assert bool(r["skipped"]) == ro["skipped"]
        if k == 9:
            assert rel_l2(m.get_params().astype(np.float64), st.theta) < 1e-4
    assert rel_l2(m.get_params().astype(np.float64), st.theta) < 1e-3, worst


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
def test_byte_indexing_bit_exact(precision):
    h, e, B, T = 64, 64, 6, 9
    m = make_model(h, e, B, T, precision)
    # a tiny W_dec (logit noise ~1e-5) and distinct b_dec make the 256 logits of every row distinct
    # by ~1e-2, so the target index of each per-position loss is identifiable from its value
    P = split(oracle_theta(h, e), h, e)
    P["W_dec"] *= 1e-3
    P["b_dec"][:] = np.arange(256) * 1e-2
    m.set_params(O.flatten(P))
    by = inputs(B, T, kind="uniform")
    m.train_step(to_dev(by))
    # X = E_w[bytes] exactly as the kernels index it
    x = m.debug_dump("x", T * B * e).reshape(T, B, e)
    E = m.get_params()[: 256 * e].reshape(256, e)  # masters after the update == E_w's source
    # one-hot of the input bytes (drives S = onehot^T dG, i.e. dE, dW_x, dW_mx, db)
    oh = m.debug_dump("onehot", 256 * T * B).reshape(256, T, B)
    ref = (np.arange(256)[:, None, None] == by[:, :T].T[None]).astype(np.float32)
    assert np.array_equal(oh, ref)
    # target shift: each per-position loss equals lse(y) - y[bytes[b, t+1]] and no other index
    y = m.debug_dump("logits", T * B * 256).reshape(T, B, 256).astype(np.float64)
    lr = m.debug_dump("loss_rows", T * B).reshape(T, B).astype(np.float64)
    lse = np.log(np.exp(y - y.max(-1, keepdims=True)).sum(-1)) + y.max(-1)
    cand = lse[..., None] - y
    best = np.abs(cand - lr[..., None]).argmin(-1)
    assert np.array_equal(best, by[:, 1:].T)
    # dE support: nonzero rows exactly the bytes used as inputs
    g = split(m.get_grads(), h, e)
    nz = set(np.nonzero(np.abs(g["E"]).sum(1))[0].tolist())
    assert nz == set(by[:, :T].ravel().tolist())
    # X rows equal the working copy of E (fp16 RNE of the masters in mixed mode) at those bytes
    Ew = E.astype(np.float16).astype(np.float32) if precision == "mixed" else E
    assert np.array_equal(x, Ew[by[:, :T].T])


@pytest.mark.parametrize("precision,recurrence", [("fp32", 0), ("mixed", 0), ("mixed", 1)])
def test_hot_path_gather_of_mx(precision, recurrence):
    """The byte gather the hot path performs (P:36 m = (W_mx x_t) . (W_mh h_{t-1}); x_t = E[s_t]): the
    m_t and a_t rows the recurrence stashed, against (i) the oracle's m_t, a_t on the same parameters,
    bytes and carried state, and (ii) the table row of the byte at (b, t): in fp32 mode m_t is exactly
    tab[s_t, :h] * a_t (one fp32 multiply), so a wrong byte, row or unit fails bit for bit."""
    h, e = (64, 64) if recurrence == 0 else (256, 64)
    B, T = (6, 5) if recurrence == 0 else (256, 3)
    m = make_model(h, e, B, T, precision, recurrence=recurrence)
    assert m.uses_recur() == (recurrence == 1)
    theta0 = oracle_theta(h, e)
    rng = np.random.default_rng(5)
    h0 = rng.uniform(-0.9, 0.9, (B, h)).astype(np.float32)
    c0 = rng.uniform(-1.0, 1.0, (B, h)).astype(np.float32)
    if precision == "mixed":
        h0 = h0.astype(np.float16).astype(np.float32)
    m.set_state(h0, c0)
    by = inputs(B, T, kind="uniform")
    m.train_step(to_dev(by))
    mm = m.debug_dump("m", T * B * h).reshape(T, B, h).astype(np.float64)
    aa = m.debug_dump("a", T * B * h).reshape(T, B, h).astype(np.float64)
    tab = m.debug_dump("tab", 256 * 5 * h).reshape(256, 5 * h)
    _, cache, _ = O.forward(split(theta0, h, e), by, h0.astype(np.float64), c0.astype(np.float64))
    tol = 1e-5 if precision == "fp32" else 2e-2
    for t in range(T):
        ref_a, ref_m = cache.a[t], cache.m[t]
        assert np.abs(aa[t] - ref_a).max() <= tol * max(1.0, np.abs(ref_a).max()), t
        assert np.abs(mm[t] - ref_m).max() <= tol * max(1.0, np.abs(ref_m).max()), t
    mx = tab[by[:, :T].T, :h].astype(np.float64)  # [T][B][h]: the table row of each input byte
    if precision == "fp32":
        assert np.array_equal(mm.astype(np.float32), (mx.astype(np.float32) * aa.astype(np.float32)))
    else:  # m rounded to fp16 from fp32 a; a itself stored in fp16
        assert np.abs(mm - mx * aa).max() <= 2e-3 * max(1.0, np.abs(mm).max())
    m.close()


def test_overflow_predicate_bit_exact():
    m = make_model(64, 64, 4, 4, "mixed")
    rng = np.random.default_rng(0)
    for trial in range(20):
        n = int(rng.integers(1, 5000))
        vals = rng.standard_normal(n) * 1000
        k = int(rng.integers(0, 4))
        for _ in range(k):
            vals[rng.integers(0, n)] = rng.choice([65504.0, 65519.99, 65520.0, -65520.0, np.inf, np.nan, 7e4])
        h16 = O.to_fp16(vals)
        t16 = torch.from_numpy(h16).cuda()
        assert m.check_overflow(t16) == O.overflow(h16)
        t32 = torch.from_numpy(vals.astype(np.float32)).cuda()
        assert m.check_overflow(t32) == O.overflow(vals.astype(np.float32))


def test_loss_scale_overflow_decisions_and_replay():
    """alpha = 2^24 must overflow the fp16 gradients at this size, alpha = 1 must not (far from the
    threshold); the GPU's alpha trace equals the oracle scaler replayed on the GPU's
    overflow flags."""
    h, e, B, T = 64, 64, 4, 16
    m = make_model(h, e, B, T, "mixed", scale_growth_interval=2)
    st = O.ScalerState(alpha=2.0 ** 24, growth_interval=2)
    m.set_opt_state(alpha=2.0 ** 24)
    theta = m.get_params()
    skipped = []
    for k in range(8):
        r = m.train_step(to_dev(inputs(B, T, k=k)))
        assert r["loss_scale"] == st.alpha
        apply, st = O.scaler_step(st, bool(r["skipped"]))
        skipped.append(r["skipped"])
        if r["skipped"]:
            assert np.array_equal(m.get_params(), theta)
        theta = m.get_params()
    assert skipped[0] == 1
    assert m.get_opt_state()["alpha"] == st.alpha
    m2 = make_model(h, e, B, T, "mixed")
    m2.set_opt_state(alpha=1.0)
    assert m2.train_step(to_dev(inputs(B, T)))["skipped"] == 0


def test_long_scaler_replay_with_injected_overflows():
    """64 steps with overflows injected at random steps (W_dec scaled by 1e9 for that step only:
    the fp16 gradients overflow at any alpha >= 1).  Every injected step is skipped with the parameters
    untouched, and the GPU's alpha trace equals the oracle scaler (reading Q9) replayed on the
    GPU's own skip flags, growth every 3 clean steps included."""
    h, e, B, T = 64, 64, 4, 16
    m = make_model(h, e, B, T, "mixed", scale_growth_interval=3, scale_init=2.0 ** 10, scale_max=2.0 ** 24)
    st = O.ScalerState(alpha=2.0 ** 10, growth_interval=3, alpha_max=2.0 ** 24)
    rng = np.random.default_rng(7)
    flags = rng.random(64) < 0.3
    n_skipped = 0
    for k, inject in enumerate(flags):
        good = m.get_params()
        if inject:
            bad = split(good, h, e)
            bad["W_dec"] = bad["W_dec"] * 1e9
            m.set_params(O.flatten(bad))
        r = m.train_step(to_dev(inputs(B, T, k=k)))
        assert r["loss_scale"] == st.alpha, (k, r["loss_scale"], st.alpha)
        if inject:
            assert r["skipped"] == 1, k
            m.set_params(good)  # the skipped step left the masters untouched: restore the unscaled decoder
        if r["skipped"]:
            assert np.array_equal(m.get_params(), good)
        n_skipped += r["skipped"]
        _, st = O.scaler_step(st, bool(r["skipped"]))
        assert m.get_opt_state()["alpha"] == st.alpha, k
    assert n_skipped >= flags.sum()


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
def test_loss_scale_invariance(precision):
    """the unscaled gradients do not depend on alpha while nothing under- or overflows.  Scaling
    by a power of two is exact in binary floating point, so in fp32 mode alpha = 1 and alpha = 2^10
    give bitwise-identical unscaled gradients.  In mixed mode alpha = 2^8 and 2^12 agree to cosine
    1 - 1e-5 per tensor, while alpha = 1 loses the small fp16 gradients to underflow -- the reason the
    paper scales the loss -- and is measurably further from the fp64 oracle than alpha = 2^10."""
    h, e, B, T = 128, 64, 8, 12
    alphas = (1.0, 2.0 ** 10) if precision == "fp32" else (1.0, 2.0 ** 8, 2.0 ** 10, 2.0 ** 12)
    grads = {}
    for alpha in alphas:
        m = make_model(h, e, B, T, precision)
        m.set_opt_state(alpha=alpha)
        r = m.train_step(to_dev(inputs(B, T)))
        assert r["loss_scale"] == alpha and not r["skipped"]
        grads[alpha] = m.get_grads().astype(np.float64)
        m.close()
    if precision == "fp32":
        assert np.array_equal(grads[1.0], grads[2.0 ** 10])
        return
    rep = compare_grads(grads[2.0 ** 12], grads[2.0 ** 8], h, e, "mixed")
    assert min(rep.values()) >= 0.99999, rep
    _, g_ref, _, _ = oracle_step(oracle_theta(h, e), inputs(B, T), h, e)
    lo = compare_grads(grads[1.0], g_ref, h, e, "mixed")
    hi = compare_grads(grads[2.0 ** 10], g_ref, h, e, "mixed")
    assert min(hi.values()) >= TOL["mixed"]["grad_cos"], hi
    assert min(hi.values()) > min(lo.values()), (lo, hi)


@pytest.mark.parametrize("alpha", [1.0, 2.0 ** 24, 2.0 ** 40])
def test_mixed_skip_decision_matches_oracle(alpha):
    """End-to-end loss-scale decision (SURVEY 8(c) bit-exact #4): the GPU's skip on one mixed
    step equals the oracle's mixed-mode decision (fp16 round trip of the alpha-scaled gradients) on
    the same parameters and bytes, at alpha = 1 (scaled gradients < 0.2: applied), 2^24 (max 1.8e6,
    27x past 65520: skipped) and 2^40 (skipped); both then hold the same halved / unchanged alpha."""
    h, e, B, T = 64, 64, 4, 16
    m = make_model(h, e, B, T, "mixed", scale_max=2.0 ** 50)
    m.set_opt_state(alpha=alpha)
    by = inputs(B, T)
    r = m.train_step(to_dev(by))
    st = O.new_train_state(h, e, B, seed=0x5EED, scaler=O.ScalerState(alpha=alpha, alpha_max=2.0 ** 50))
    ro = O.train_step(st, by, precision="mixed")
    assert r["loss_scale"] == alpha == ro["alpha"]
    assert bool(r["skipped"]) == ro["skipped"] == (alpha > 1.0)
    assert m.get_opt_state()["alpha"] == st.scaler.alpha
    assert abs(r["loss_nats"] - ro["loss_nats"]) <= TOL["mixed"]["loss_rel"] * ro["loss_nats"]


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
def test_eval_matches_oracle(precision):
    h, e, B, T = 128, 64, 16, 12
    m = make_model(h, e, B, T, precision)
    P = split(oracle_theta(h, e), h, e)
    by = inputs(B, T, kind="markov")
    nats, tok, bpc = m.eval(to_dev(by))
    ref, tok_ref, _ = O.evaluate(P, by, np.zeros((B, h)), np.zeros((B, h)))
    assert tok == tok_ref
    tol = 1e-5 if precision == "fp32" else 5e-3
    assert abs(nats - ref) / ref <= tol
    assert abs(bpc - O.bpc_from_nats(ref / tok)) <= tol * 8


def test_state_carry_two_windows_bitwise():
    """Eval over [T] then [T] with persisted state == the state after the same bytes in one model
    run twice (determinism) and equals the oracle's carried state."""
    h, e, B, T = 128, 64, 8, 6
    s = inputs(B, 2 * T)
    w1, w2 = s[:, :T + 1], s[:, T:]
    outs = []
    for _ in range(2):
        m = make_model(h, e, B, T, "fp32")
        m.eval(to_dev(w1))
        m.eval(to_dev(w2))
        outs.append(m.get_state(1))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    P = split(oracle_theta(h, e), h, e)
    _, _, (hT, cT) = O.forward(P, s, np.zeros((B, h)), np.zeros((B, h)))
    assert np.abs(outs[0][0] - hT).max() < 1e-5


def test_reset_rows_start_from_zero_state():
    h, e, B, T = 64, 64, 4, 8
    m = make_model(h, e, B, T, "fp32")
    rng = np.random.default_rng(3)
    h0, c0 = rng.standard_normal((B, h)).astype(np.float32), rng.standard_normal((B, h)).astype(np.float32)
    m.set_state(h0, c0)
    by = inputs(B, T)
    reset = np.array([0, 1, 0, 1], dtype=np.uint8)
    theta0 = oracle_theta(h, e)
    r = m.train_step(to_dev(by), to_dev(reset))
    h0r, c0r = h0.astype(np.float64), c0.astype(np.float64)
    h0r[reset == 1] = 0
    c0r[reset == 1] = 0
    loss_ref, _, _, _ = oracle_step(theta0, by, h, e, h0r, c0r)
    assert abs(r["loss_nats"] - loss_ref) / loss_ref < 1e-5


def test_host_entry_point_matches_device_entry_point():
    h, e, B, T = 64, 64, 4, 16
    by = inputs(B, T)
    a = make_model(h, e, B, T, "mixed")
    b = make_model(h, e, B, T, "mixed")
    ra = a.train_step(to_dev(by))
    rb = b.train_step_host(by)
    assert ra == rb
    assert np.array_equal(a.get_params(), b.get_params())


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
def test_micro_batches_equal_one_batch(precision):
    """Micro-batching (4096 rows/GPU as 1024-row micro-batches) accumulates gradients in
    fp32 across micro-batches: the step equals one un-split step on the same rows (fp32 mode to
    fp32 rounding; mixed mode to the per-micro-batch fp16 rounding of the gradients), and the
    persisted state of every row is carried."""
    h, e, B, T = 128, 64, 12, 6
    by0 = inputs(B, T, k=0)
    by1 = inputs(B, T, k=1)
    whole = make_model(h, e, B, T, precision)
    split = make_model(h, e, B, T, precision, micro_batch=4)
    for by in (by0, by1):
        ra, rb = whole.train_step(to_dev(by)), split.train_step(to_dev(by))
        assert abs(ra["loss_nats"] - rb["loss_nats"]) <= 1e-6 * ra["loss_nats"]
        ga, gb = whole.get_grads().astype(np.float64), split.get_grads().astype(np.float64)
        if precision == "fp32":
            assert rel_l2(gb, ga) < 1e-5
        else:
            rep = compare_grads(gb, ga, h, e, "mixed")
            assert min(rep.values()) > 0.9999, rep
    ha, ca = whole.get_state(0)
    hb, cb = split.get_state(0)
    assert np.abs(ha - hb).max() < (1e-6 if precision == "fp32" else 2e-3)
    assert rel_l2(split.get_params().astype(np.float64), whole.get_params().astype(np.float64)) < 1e-4


@pytest.mark.parametrize("plan", ["pair", "split", "single", "persist", "pair512"])
@pytest.mark.parametrize("h,B,T", [(512, 256, 4), (512, 200, 3), (1024, 256, 2)])
def test_forced_tile_plans_match_oracle(plan, h, B, T, monkeypatch):
    """Every tcgen05 tile plan (CTA pair, cluster split-K, single CTA, persistent pairs) on every GEMM,
    forced at a size the oracle finishes quickly (full-size shapes select them on their own);
    B=200 leaves a ragged last M tile."""
    if plan == "pair512":  # weight gradients on 256 x 512 pair tiles (two N=256 MMAs per k-step)
        if h % 512:
            pytest.skip("needs N % 512 == 0")
        monkeypatch.setenv("MLSTM_WGRAD512", "1")
        plan = "pair"
    else:
        monkeypatch.setenv("MLSTM_WGRAD512", "0")
    monkeypatch.setenv("MLSTM_FORCE_PLAN", plan)
    if plan == "persist":  # two resident pairs: every pair walks several tiles (TMEM double buffer)
        monkeypatch.setenv("MLSTM_PERSIST_PAIRS", "2")
    e = 64
    m = make_model(h, e, B, T, "mixed")
    theta0 = oracle_theta(h, e)
    by = inputs(B, T)
    res = m.train_step(to_dev(by))
    loss_ref, g_ref, (hT, cT), _ = oracle_step(theta0, by, h, e)
    assert abs(res["loss_nats"] - loss_ref) / loss_ref <= TOL["mixed"]["loss_rel"]
    rep = compare_grads(m.get_grads().astype(np.float64), g_ref, h, e, "mixed")
    assert min(rep.values()) >= TOL["mixed"]["grad_cos"], rep
    hs, cs = m.get_state(0)
    assert np.abs(hs - hT).max() <= 2e-3 and np.abs(cs - cT).max() <= 2e-2
    nats, tokens, _ = m.eval(to_dev(inputs(B, T, k=1)))
    assert np.isfinite(nats) and tokens == B * T


def test_multi_step_trace_mixed_tracks_oracle():
    """10 mixed-precision steps at C2's width (fp16 storage, loss scaling, Adam on fp32 masters)
    against the fp64 oracle loop: the loss stays within the north_star bound at every step."""
    h, e, B, T = 1024, 64, 64, 16
    m = make_model(h, e, B, T, "mixed")
    st = O.new_train_state(h, e, B, seed=0x5EED)
    for k in range(10):
        by = inputs(B, T, k=k)
        r = m.train_step(to_dev(by))
        ro = O.train_step(st, by)
        assert abs(r["loss_nats"] - ro["loss_nats"]) <= TOL["mixed"]["loss_rel"] * ro["loss_nats"], (k, r, ro)
        assert bool(r["skipped"]) == ro["skipped"] and r["loss_scale"] == ro["alpha"]
    assert cosine(m.get_params().astype(np.float64) - oracle_theta(h, e), st.theta - oracle_theta(h, e)) > 0.99


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
@pytest.mark.parametrize("h,B,T", [(64, 4, 1), (64, 1, 5), (128, 3, 2)])
def test_degenerate_shapes_match_oracle(h, B, T, precision):
    """Degenerate cases of the method: a one-timestep window (no recurrent backward at all), a single
    row, and a tiny ragged batch."""
    e = 64
    m = make_model(h, e, B, T, precision)
    theta0 = oracle_theta(h, e)
    by = inputs(B, T)
    res = m.train_step(to_dev(by))
    loss_ref, g_ref, (hT, cT), _ = oracle_step(theta0, by, h, e)
    tol = TOL[precision]
    assert abs(res["loss_nats"] - loss_ref) / loss_ref <= tol["loss_rel"]
    rep = compare_grads(m.get_grads().astype(np.float64), g_ref, h, e, precision)
    for n, v in rep.items():
        assert (v <= tol["grad_rel_l2"]) if precision == "fp32" else (v >= tol["grad_cos"]), (n, v, rep)


def test_eval_partial_batch_and_reset_with_micro_batches():
    """Eval over Be < micro-batch rows equals the oracle on those rows; reset masks that fall in the
    second micro-batch zero exactly those rows' state (micro-batched step vs the oracle)."""
    h, e, B, T = 64, 64, 8, 6
    m = make_model(h, e, B, T, "fp32", micro_batch=4)
    by = inputs(B, T)
    nats, tok, _ = m.eval(to_dev(by[:3]))
    P = split(oracle_theta(h, e), h, e)
    ref, tok_ref, _ = O.evaluate(P, by[:3], np.zeros((3, h)), np.zeros((3, h)))
    assert tok == tok_ref and abs(nats - ref) / ref <= 1e-5
    rng = np.random.default_rng(5)
    h0, c0 = rng.standard_normal((B, h)).astype(np.float32), rng.standard_normal((B, h)).astype(np.float32)
    m.set_state(h0, c0)
    reset = np.array([0, 0, 0, 0, 1, 0, 1, 0], dtype=np.uint8)
    r = m.train_step(to_dev(by), to_dev(reset))
    h0r, c0r = h0.astype(np.float64), c0.astype(np.float64)
    h0r[reset == 1] = 0
    c0r[reset == 1] = 0
    loss_ref, _, (hT, _), _ = oracle_step(oracle_theta(h, e), by, h, e, h0r, c0r)
    assert abs(r["loss_nats"] - loss_ref) / loss_ref < 1e-5
    hs, _ = m.get_state(0)
    assert np.abs(hs - hT).max() < 1e-5
