"""Plain fp64 CPU oracle for the mixed-precision mLSTM training step of arXiv 1808.01371.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It shares no code, headers, tables or constants with the CUDA path in
``paper_1808_01371_b200/`` and never imports it.

Everything is written out in the paper's order and notation, in float64 NumPy,
with explicit Python loops over time.  Citations are ``P:L`` = line L of the
paper's PAPER.md (section in brackets) and ``S:L`` = line L of SPEC.md.  Where
the paper is silent the reading is the one listed in DESIGN.md "Readings"
(Q-numbers follow SURVEY.md §8c).

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``):
  * forward      -- torch.nn.LSTM special case (mx == 1); torch.nn.LSTMCell with the mLSTM's
                    input-dependent transition W_h diag(W_mx x_t) W_mh (pins mx and its byte
                    indexing); zero-weight closed form, uniform-logit ln(256) closed form, TBTT
                    state-carry identity.
  * backward     -- central finite differences on tiny models (all 8 tensors).
  * dE support   -- nonzero embedding-gradient rows == bytes present.
  * adam         -- torch.optim.Adam (fp64), first-step closed form, lr=0 identity.
  * lr schedule  -- values printed in P:302-307 and Tab. lr_scale.
  * scaler       -- SPEC traces S:202-204 and the state-machine properties S:216-218.
  * overflow     -- IEEE binary16 thresholds (65504 finite, 65520 -> inf); the mixed-mode step
                    decision (fp16 round trip of the scaled gradients) at alpha far below / above them.
  * init         -- SplitMix64 published reference outputs.
  * speedup      -- Tab. gpu_scale arithmetic.
  * weight norm  -- S:129-130 worked examples, finite differences through (v, g), scale
                    invariance in v, dv orthogonal to v, function-preserving init.
No function is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

V = 256  # byte-level vocabulary ("character-level")

# --------------------------------------------------------------------------------------
# Parameters: canonical layout
#   E[256 x e] | W_mx[h x e] | W_mh[h x h] | W_x[4h x e] | W_h[4h x h] | b[4h] | W_dec[256 x h] | b_dec[256]
# Gate blocks inside 4h are ordered i, f, o, u, each h rows.
# --------------------------------------------------------------------------------------

PARAM_NAMES = ("E", "W_mx", "W_mh", "W_x", "W_h", "b", "W_dec", "b_dec")


def param_shapes(h: int, e: int):
    return {
        "E": (V, e),
        "W_mx": (h, e),
        "W_mh": (h, h),
        "W_x": (4 * h, e),
        "W_h": (4 * h, h),
        "b": (4 * h,),
        "W_dec": (V, h),
        "b_dec": (V,),
    }


def param_count(h: int, e: int) -> int:
    """P = 5h^2 + 5he + 4h + 256e + 256h + 256 (SURVEY symbols table)."""
    return sum(int(np.prod(s)) for s in param_shapes(h, e).values())


def flatten(params: dict) -> np.ndarray:
    return np.concatenate([np.asarray(params[n], dtype=np.float64).ravel() for n in PARAM_NAMES])


def unflatten(flat: np.ndarray, h: int, e: int) -> dict:
    out, off = {}, 0
    for n in PARAM_NAMES:
        s = param_shapes(h, e)[n]
        cnt = int(np.prod(s))
        out[n] = np.asarray(flat[off:off + cnt], dtype=np.float64).reshape(s).copy()
        off += cnt
    return out


# --------------------------------------------------------------------------------------
# Initialisation (paper silent; reading Q12): U(-1/sqrt(cols), +1/sqrt(cols)) per matrix,
# biases zero.  Counter-based SplitMix64 so any implementation reproduces it bit-exactly:
#   z = seed + (q+1)*0x9E3779B97F4A7C15 (mod 2^64); z = (z^(z>>30))*0xBF58476D1CE4E5B9;
#   z = (z^(z>>27))*0x94D049BB133111EB; z ^= z>>31;  u = (z>>11)*2^-53;
#   w = RNE_fp32(s*(2u-1)) computed in fp64, q = canonical flat index.
# --------------------------------------------------------------------------------------

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(seed: int, q: np.ndarray) -> np.ndarray:
    """The SplitMix64 output for counter q (q=0 is the generator's first output)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (np.asarray(q, dtype=np.uint64) + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def init_params(h: int, e: int, seed: int) -> dict:
    """Returns fp32-representable values (stored as float64) in the canonical layout."""
    out, off = {}, 0
    for n in PARAM_NAMES:
        s = param_shapes(h, e)[n]
        cnt = int(np.prod(s))
        if len(s) == 1:
            out[n] = np.zeros(s)
        else:
            q = np.arange(off, off + cnt, dtype=np.uint64)
            u = (splitmix64(seed, q) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
            scale = 1.0 / math.sqrt(s[1])
            out[n] = (scale * (2.0 * u - 1.0)).astype(np.float32).astype(np.float64).reshape(s)
        off += cnt
    return out


# --------------------------------------------------------------------------------------
# Forward: mLSTM (reading Q1) + byte decoder + softmax cross-entropy
# --------------------------------------------------------------------------------------

def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


@dataclass
class ForwardCache:
    bytes_: np.ndarray
    x: list = field(default_factory=list)
    mx: list = field(default_factory=list)
    a: list = field(default_factory=list)
    m: list = field(default_factory=list)
    i: list = field(default_factory=list)
    f: list = field(default_factory=list)
    o: list = field(default_factory=list)
    u: list = field(default_factory=list)
    c: list = field(default_factory=list)      # c[t+1] = C_t ; c[0] = c0
    hs: list = field(default_factory=list)     # hs[t+1] = H_t ; hs[0] = h0
    p: list = field(default_factory=list)      # softmax probabilities, per t [B,256]
    logits: list = field(default_factory=list)
    loss_t: list = field(default_factory=list)  # per-position CE in nats, per t [B]


def forward(P: dict, bytes_: np.ndarray, h0: np.ndarray, c0: np.ndarray, reset=None):
    """One TBTT window.  bytes_ is [B, T+1] uint8: inputs = [:, :T], targets = [:, 1:] (reading Q6).

    Returns (loss_sum_nats, cache, (h_T, c_T)).  State rows with reset[b] set start from zero.
    """
    bytes_ = np.asarray(bytes_)
    Bn, T1 = bytes_.shape
    T = T1 - 1
    h = np.array(h0, dtype=np.float64, copy=True)
    c = np.array(c0, dtype=np.float64, copy=True)
    if reset is not None:
        r = np.asarray(reset).astype(bool)
        h[r] = 0.0
        c[r] = 0.0
    H = P["W_mh"].shape[0]
    cache = ForwardCache(bytes_=bytes_)
    cache.hs.append(h)
    cache.c.append(c)
    loss_sum = 0.0
    for t in range(T):
        x = P["E"][bytes_[:, t]]                       # X = E[s_t]           (byte embedding)
        mx = x @ P["W_mx"].T                           # W_mx x
        a = h @ P["W_mh"].T                            # W_mh h_{t-1}
        m = mx * a                                     # m = (W_mx x) . (W_mh h_{t-1})
        z = x @ P["W_x"].T + m @ P["W_h"].T + P["b"]   # z = W_x x + W_h m + b
        zi, zf, zo, zu = z[:, :H], z[:, H:2 * H], z[:, 2 * H:3 * H], z[:, 3 * H:]
        i, f, o, u = sigmoid(zi), sigmoid(zf), sigmoid(zo), np.tanh(zu)
        c = f * c + i * u                              # c_t = f . c_{t-1} + i . u
        h = o * np.tanh(c)                             # h_t = o . tanh(c_t)
        y = h @ P["W_dec"].T + P["b_dec"]              # logits (fp32 in the paper)
        ymax = y.max(axis=1, keepdims=True)
        ez = np.exp(y - ymax)
        se = ez.sum(axis=1, keepdims=True)
        lse = ymax[:, 0] + np.log(se[:, 0])            # max-subtracted logsumexp (Q16)
        tgt = bytes_[:, t + 1]
        lt = lse - y[np.arange(Bn), tgt]
        loss_sum += float(lt.sum())
        for lst, val in ((cache.x, x), (cache.mx, mx), (cache.a, a), (cache.m, m), (cache.i, i),
                         (cache.f, f), (cache.o, o), (cache.u, u), (cache.c, c), (cache.hs, h),
                         (cache.p, ez / se), (cache.logits, y), (cache.loss_t, lt)):
            lst.append(val)
    return loss_sum, cache, (h, c)


# --------------------------------------------------------------------------------------
# Backward: BPTT inside the window, truncated at the window start (TBTT)
# --------------------------------------------------------------------------------------

def backward(P: dict, cache: ForwardCache, denom: float, scale: float = 1.0) -> dict:
    """Gradient of scale * (sum of per-position CE) / denom w.r.t. every parameter.

    denom = B_g * T (mean over all global positions, reading Q7); scale = loss scale alpha
    ("multiplying the training loss by a scalar").  The incoming state (h0, c0) is
    treated as a constant (TBTT), so dh and dc entering step 0 are dropped.
    """
    bytes_ = cache.bytes_
    Bn, T1 = bytes_.shape
    T = T1 - 1
    H = P["W_mh"].shape[0]
    g = {n: np.zeros_like(P[n]) for n in PARAM_NAMES}
    dh_rec = np.zeros((Bn, H))
    dc_next = np.zeros((Bn, H))
    w = scale / denom
    for t in range(T - 1, -1, -1):
        tgt = bytes_[:, t + 1]
        dy = cache.p[t].copy()
        dy[np.arange(Bn), tgt] -= 1.0                   # softmax - onehot
        dy *= w
        h_t = cache.hs[t + 1]
        g["W_dec"] += dy.T @ h_t
        g["b_dec"] += dy.sum(axis=0)
        dh = dy @ P["W_dec"] + dh_rec
        i, f, o, u = cache.i[t], cache.f[t], cache.o[t], cache.u[t]
        c_t, c_prev = cache.c[t + 1], cache.c[t]
        k = np.tanh(c_t)
        dzo = dh * k * o * (1.0 - o)
        dc = dc_next + dh * o * (1.0 - k * k)
        dzi = dc * u * i * (1.0 - i)
        dzf = dc * c_prev * f * (1.0 - f)
        dzu = dc * i * (1.0 - u * u)
        dc_next = dc * f
        dz = np.concatenate([dzi, dzf, dzo, dzu], axis=1)
        x, mx, a, m = cache.x[t], cache.mx[t], cache.a[t], cache.m[t]
        h_prev = cache.hs[t]
        g["W_h"] += dz.T @ m
        g["W_x"] += dz.T @ x
        g["b"] += dz.sum(axis=0)
        dm = dz @ P["W_h"]
        da = dm * mx
        dmx = dm * a
        g["W_mh"] += da.T @ h_prev
        g["W_mx"] += dmx.T @ x
        dx = dz @ P["W_x"] + dmx @ P["W_mx"]
        np.add.at(g["E"], bytes_[:, t], dx)            # dE[s_t] += W_x^T dz + W_mx^T dmx
        dh_rec = da @ P["W_mh"]
    return g


def loss_and_grads(P: dict, bytes_, h0, c0, n_global_rows: int | None = None, scale: float = 1.0,
                   reset=None):
    """Forward + backward for one window; returns (loss_sum, grads, (hT, cT), cache)."""
    bytes_ = np.asarray(bytes_)
    Bn, T1 = bytes_.shape
    Bg = Bn if n_global_rows is None else n_global_rows
    loss_sum, cache, state = forward(P, bytes_, h0, c0, reset=reset)
    grads = backward(P, cache, denom=Bg * (T1 - 1), scale=scale)
    return loss_sum, grads, state, cache


def bpc_from_nats(l: float) -> float:
    """BPC = l * log2(e)."""
    return l / math.log(2.0)


# --------------------------------------------------------------------------------------
# Mixed-precision bookkeeping: fp16 overflow predicate and the dynamic loss scaler
# --------------------------------------------------------------------------------------

def to_fp16(x) -> np.ndarray:
    """IEEE binary16, round-to-nearest-even, overflow -> inf (reading Q13)."""
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float64).astype(np.float16)


def overflow(buf) -> bool:
    """"checking for an overflow in the weight gradients": any non-finite element."""
    return bool(not np.all(np.isfinite(np.asarray(buf))))


@dataclass
class ScalerState:
    alpha: float = 2.0 ** 16          # "starting at a large value" (Q9)
    clean: int = 0
    growth_interval: int = 2000
    alpha_min: float = 1.0
    alpha_max: float = 2.0 ** 24


def scaler_step(st: ScalerState, overflowed: bool) -> tuple[bool, ScalerState]:
    """Returns (apply_update, new_state).  Overflow: skip and halve. Otherwise count clean
    steps; after growth_interval of them double alpha ("tries to increase alpha after a
    sufficient number of iterations")."""
    s = ScalerState(st.alpha, st.clean, st.growth_interval, st.alpha_min, st.alpha_max)
    if overflowed:
        s.alpha = max(s.alpha / 2.0, s.alpha_min)
        s.clean = 0
        return False, s
    s.clean += 1
    if s.clean == s.growth_interval:
        s.alpha = min(s.alpha * 2.0, s.alpha_max)
        s.clean = 0
    return True, s


# --------------------------------------------------------------------------------------
# Optimiser and LR schedule (P:153 Adam; P:302-307 schedule; P:107-109, P:153 scaling rules)
# --------------------------------------------------------------------------------------

def lr_at(lr0: float, it: int, decay_iters: int) -> float:
    """"Set an initial learning rate of 3e-3. Linearly decay learning rate to zero over 100,000
    iterations"."""
    return lr0 * max(0.0, 1.0 - it / decay_iters)


def scale_lr(base_lr: float, rule: str, batch: int, ref_batch: int = 128) -> float:
    """Linear rule eps ~ B, sqrt rule eps ~ sqrt(B), from 5e-4 at batch 128."""
    r = batch / ref_batch
    if rule == "none":
        return base_lr
    if rule == "linear":
        return base_lr * r
    if rule == "sqrt":
        return base_lr * math.sqrt(r)
    raise ValueError(rule)


@dataclass
class AdamState:
    m: np.ndarray
    v: np.ndarray
    tau: int = 0


def adam_apply(theta: np.ndarray, g: np.ndarray, st: AdamState, lr: float,
               beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8):
    """Kingma & Ba Adam with bias correction (Q11).  tau counts applied updates only."""
    tau = st.tau + 1
    m = beta1 * st.m + (1.0 - beta1) * g
    v = beta2 * st.v + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** tau)
    vhat = v / (1.0 - beta2 ** tau)
    theta_new = theta - lr * mhat / (np.sqrt(vhat) + eps)
    return theta_new, AdamState(m, v, tau)


# --------------------------------------------------------------------------------------
# One full training step: forward, CE, BPTT, (allreduce), overflow
# check, scaler, unscale, Adam, schedule.  ``grads_hook`` lets a DP test sum grads across ranks.
# --------------------------------------------------------------------------------------

@dataclass
class TrainState:
    h: int
    e: int
    theta: np.ndarray                 # flat fp64 masters, canonical layout
    adam: AdamState
    scaler: ScalerState
    it: int = 0                       # LR clock: advances every step incl. skipped (Q10)
    h_state: np.ndarray | None = None
    c_state: np.ndarray | None = None
    weight_norm: bool = False         # theta in the wn layout (v, gains)


def new_train_state(h: int, e: int, B: int, seed: int, scaler: ScalerState | None = None,
                    weight_norm: bool = False) -> TrainState:
    theta = wn_init(h, e, seed) if weight_norm else flatten(init_params(h, e, seed))
    return TrainState(h, e, theta, AdamState(np.zeros_like(theta), np.zeros_like(theta)),
                      scaler or ScalerState(), 0, np.zeros((B, h)), np.zeros((B, h)), weight_norm)


def train_step(st: TrainState, bytes_, lr0=3e-3, decay_iters=100_000, n_global_rows=None,
               reset=None, grads_hook=None, loss_hook=None, beta1=0.9, beta2=0.999, eps=1e-8,
               precision: str = "fp32"):
    """Returns a dict {loss_nats, bpc, skipped, alpha, lr, grads (unscaled, flat)}; mutates st.

    precision="mixed": the overflow check runs on the alpha-scaled weight gradients as they exist in
    the mixed-precision step, i.e. rounded to IEEE binary16 ("FP16 ... weight gradients" sent in
    the allreduce; "checking for an overflow in the weight gradients"; readings Q8, Q13).  The
    update itself still uses the fp64 gradients (the oracle is the exact reference).  "fp32": the
    check runs on the fp64 values (fp32 parity mode has no fp16 buffer to overflow)."""
    bytes_ = np.asarray(bytes_)
    Bn, T1 = bytes_.shape
    Bg = Bn if n_global_rows is None else n_global_rows
    alpha = st.scaler.alpha
    if st.weight_norm:
        loss_sum, gflat, (hT, cT), _ = wn_loss_and_grads(st.theta, st.h, st.e, bytes_, st.h_state, st.c_state,
                                                         Bg, alpha, reset=reset)
    else:
        P = unflatten(st.theta, st.h, st.e)
        loss_sum, grads, (hT, cT), _ = loss_and_grads(P, bytes_, st.h_state, st.c_state, Bg, alpha,
                                                     reset=reset)
        gflat = flatten(grads)                  # alpha-scaled, mean over global positions
    if grads_hook is not None:
        gflat = grads_hook(gflat)               # e.g. SUM allreduce across ranks (Q7)
    if loss_hook is not None:
        loss_sum = loss_hook(loss_sum)
    ovf = overflow(to_fp16(gflat) if precision == "mixed" else gflat)
    apply, st.scaler = scaler_step(st.scaler, ovf)
    lr = lr_at(lr0, st.it, decay_iters)
    g_unscaled = gflat / alpha                  # "The division by alpha occurs on the gradients of
    if apply:                                   #  these master copies"
        st.theta, st.adam = adam_apply(st.theta, g_unscaled, st.adam, lr, beta1, beta2, eps)
    st.it += 1
    st.h_state, st.c_state = hT, cT             # persisted, detached
    loss_nats = loss_sum / (Bg * (T1 - 1))
    return {"loss_nats": loss_nats, "bpc": bpc_from_nats(loss_nats), "skipped": not apply,
            "alpha": alpha, "lr": lr, "grads": g_unscaled}


def evaluate(P: dict, bytes_, h0, c0, reset=None, valid=None):
    """Forward-only BPC over one window with persisted state: (nats_sum, tokens, (hT,cT)).
    Rows with valid[b] == 0 (idle data-loader rows) are not counted; their state restarts at zero."""
    Bn, T1 = np.asarray(bytes_).shape
    if valid is None:
        loss_sum, cache, state = forward(P, bytes_, h0, c0, reset=reset)
        return loss_sum, Bn * (T1 - 1), state
    valid = np.asarray(valid).astype(bool)
    reset = (np.zeros(Bn, bool) if reset is None else np.asarray(reset).astype(bool)) | ~valid
    loss_sum, cache, state = forward(P, bytes_, h0, c0, reset=reset)
    counted = float(np.stack(cache.loss_t, axis=0)[:, valid].sum())
    return counted, int(valid.sum()) * (T1 - 1), state


# --------------------------------------------------------------------------------------
# Weight normalisation (P:149-150 [§VI "Weight Normalization"]: applied "to the LSTM parameters
# only ... the 4 hidden->hidden and input->hidden parameters", not to biases; Salimans & Kingma
# 2016; S:124-131 weight_norm_build).  Row-wise over output units: w_i = g_i v_i / ||v_i||_2.
# Parameters become v (in the W slots of the canonical layout) and one gain per row, appended
# after b_dec in the order g_mx[h] | g_mh[h] | g_x[4h] | g_h[4h] (reading Q24).  Init: v as the
# plain init, g_i = ||v_i|| (function-preserving; paper silent).
# --------------------------------------------------------------------------------------

WN_NAMES = ("W_mx", "W_mh", "W_x", "W_h")


def wn_gain_count(h: int) -> int:
    return h + h + 4 * h + 4 * h


def wn_param_count(h: int, e: int) -> int:
    return param_count(h, e) + wn_gain_count(h)


def wn_split(flat: np.ndarray, h: int, e: int):
    """Flat wn layout -> (dict of the 8 tensors with v in the W slots, dict of gains)."""
    base = param_count(h, e)
    P = unflatten(flat[:base], h, e)
    gains, off = {}, base
    for n in WN_NAMES:
        rows = param_shapes(h, e)[n][0]
        gains[n] = np.asarray(flat[off:off + rows], dtype=np.float64).copy()
        off += rows
    return P, gains


def wn_join(P: dict, gains: dict) -> np.ndarray:
    return np.concatenate([flatten(P)] + [np.asarray(gains[n], dtype=np.float64).ravel() for n in WN_NAMES])


def weight_norm_build(v: np.ndarray, g: np.ndarray) -> np.ndarray:
    """w_i = g_i * v_i / ||v_i||_2 per row (S:124 weight_norm_build; P:132 the norm in fp32 or wider)."""
    v = np.asarray(v, dtype=np.float64)
    norm = np.sqrt((v * v).sum(axis=1))
    return (np.asarray(g, dtype=np.float64) / norm)[:, None] * v


def weight_norm_backward(v: np.ndarray, g: np.ndarray, dw: np.ndarray):
    """Chain rule through w = g v/||v||: dg_i = dw_i . v_i / ||v_i||,
    dv_i = (g_i / ||v_i||) (dw_i - (dg_i / ||v_i||) v_i)   (Salimans & Kingma 2016, eq. 3)."""
    v = np.asarray(v, dtype=np.float64)
    dw = np.asarray(dw, dtype=np.float64)
    norm = np.sqrt((v * v).sum(axis=1))
    dg = (dw * v).sum(axis=1) / norm
    dv = (np.asarray(g, dtype=np.float64) / norm)[:, None] * (dw - (dg / norm)[:, None] * v)
    return dv, dg


def wn_effective(P: dict, gains: dict) -> dict:
    """The plain parameter dict the mLSTM runs with: W = weight_norm_build(v, g) for WN_NAMES."""
    out = {n: np.asarray(P[n], dtype=np.float64).copy() for n in PARAM_NAMES}
    for n in WN_NAMES:
        out[n] = weight_norm_build(P[n], gains[n])
    return out


def wn_init(h: int, e: int, seed: int) -> np.ndarray:
    """Flat wn parameters: v = the plain init (Q12), g_i = RNE_fp32(||v_i||) computed in fp64."""
    P = init_params(h, e, seed)
    gains = {n: np.sqrt((P[n] * P[n]).sum(axis=1)).astype(np.float32).astype(np.float64) for n in WN_NAMES}
    return wn_join(P, gains)


def wn_loss_and_grads(flat: np.ndarray, h: int, e: int, bytes_, h0, c0, n_global_rows=None, scale=1.0,
                      reset=None):
    """Forward + backward with weight normalisation; grads flat in the wn layout (dv, dg)."""
    P, gains = wn_split(flat, h, e)
    loss_sum, gw, state, cache = loss_and_grads(wn_effective(P, gains), bytes_, h0, c0, n_global_rows, scale,
                                                reset=reset)
    dg = {}
    for n in WN_NAMES:
        gw[n], dg[n] = weight_norm_backward(P[n], gains[n], gw[n])
    return loss_sum, wn_join(gw, dg), state, cache


# --------------------------------------------------------------------------------------
# Reporting arithmetic (Tab. gpu_scale caption P:232)
# --------------------------------------------------------------------------------------

def speedup(n: int, t1: float, tn: float) -> float:
    """Relative speedup of n data-parallel workers at fixed per-worker batch: n * t1 / tn."""
    return n * t1 / tn


def flops_per_char(h: int, e: int) -> float:
    """Dense algorithmic work per character: 6 * (5h^2 + 5he + 256h) (fwd, dW and dX of every
    matmul)."""
    return 6.0 * (5 * h * h + 5 * h * e + V * h)
