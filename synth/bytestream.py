"""Seeded synthetic byte streams shaped like the paper's workload (Amazon reviews).

Input generation only: this module holds none of the method's arithmetic and is the one
piece shared by the oracle-side tests and the CUDA-side tests/bench.

kind="markov" (default): an order-2 Markov source over a 97-symbol alphabet (95 printable ASCII
bytes, '\\n', '\\t').  Unigram preference is Zipf-like; each 2-byte context allows 8 successors
drawn without replacement by that preference, with Dirichlet(0.5) probabilities; '\\n' is
forced into every context's successor set with a small probability so its stationary frequency
is roughly 1/488 (one "review" per ~488 bytes: 40 GB / 82 M reviews).  Its exact entropy
rate is computed by power iteration over the 97^2 contexts (`entropy_rate_bits`).
kind="uniform": iid bytes, entropy exactly 8 bits/char.

Every global row r is its own stream.  Row r's k-th window is bytes [k*T, k*T + T] of its stream
(T+1 bytes; consecutive windows overlap by one byte, so targets continue across windows -- the
contiguity the paper needs for TBTT state persistence).  Rows are independent of how they
are assigned to ranks, so an N-rank run sees exactly the rows a 1-rank run would.
"""
from __future__ import annotations

import numpy as np

ALPHABET = np.array(list(range(32, 127)) + [10, 9], dtype=np.uint8)  # 97 symbols
NSYM = len(ALPHABET)
NSUCC = 8
_MASK = (1 << 64) - 1


def _mix64(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _uniforms(row_keys: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """Counter-based U[0,1) per (row, position)."""
    with np.errstate(over="ignore"):
        z = row_keys + (pos.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
    return (_mix64(z) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


class MarkovSource:
    """The transition structure (shared by all rows) of the order-2 source."""

    def __init__(self, seed: int = 0x5EED):
        rng = np.random.Generator(np.random.PCG64(seed))
        pref = 1.0 / np.arange(1, NSYM + 1) ** 1.1           # Zipf-like unigram preference
        pref = pref[rng.permutation(NSYM)]
        nl = int(np.where(ALPHABET == 10)[0][0])
        pref[nl] = 0.0
        pref /= pref.sum()
        succ = np.zeros((NSYM * NSYM, NSUCC), dtype=np.int64)
        prob = np.zeros((NSYM * NSYM, NSUCC))
        for ctx in range(NSYM * NSYM):
            s = rng.choice(NSYM, size=NSUCC - 1, replace=False, p=pref)
            p = rng.dirichlet(np.full(NSUCC - 1, 0.5))
            succ[ctx, :NSUCC - 1] = s
            prob[ctx, :NSUCC - 1] = p * (1.0 - 1.0 / 488.0)
            succ[ctx, NSUCC - 1] = nl
            prob[ctx, NSUCC - 1] = 1.0 / 488.0
        self.succ = succ
        self.cdf = np.cumsum(prob, axis=1)
        self.cdf[:, -1] = 1.0
        self.prob = prob

    def entropy_rate_bits(self, iters: int = 400) -> float:
        """H = sum_ctx pi(ctx) H(next | ctx), pi by power iteration over contexts (a,b)->(b,c)."""
        n = NSYM * NSYM
        pi = np.full(n, 1.0 / n)
        ctx_b = np.arange(n) % NSYM
        for _ in range(iters):
            nxt = np.zeros(n)
            dest = ctx_b[:, None] * NSYM + self.succ          # new context (b, c)
            np.add.at(nxt, dest.ravel(), (pi[:, None] * self.prob).ravel())
            pi = nxt
        p = self.prob
        hctx = -(np.where(p > 0, p * np.log2(np.where(p > 0, p, 1.0)), 0.0)).sum(axis=1)
        return float((pi * hctx).sum())


_SOURCES: dict[int, MarkovSource] = {}


def source(seed: int = 0x5EED) -> MarkovSource:
    if seed not in _SOURCES:
        _SOURCES[seed] = MarkovSource(seed)
    return _SOURCES[seed]


def row_keys(rows: np.ndarray, seed: int) -> np.ndarray:
    with np.errstate(over="ignore"):
        return _mix64(np.uint64(seed) ^ rows.astype(np.uint64))


def stream(rows, start: int, length: int, seed: int = 0x5EED, kind: str = "markov") -> np.ndarray:
    """Bytes [start, start+length) of each listed global row's stream: uint8 [len(rows), length]."""
    rows = np.asarray(rows, dtype=np.int64)
    keys = row_keys(rows, seed)
    if kind == "uniform":
        pos = np.arange(start, start + length, dtype=np.uint64)
        u = _uniforms(keys[:, None], pos[None, :])
        return np.minimum((u * 256).astype(np.int64), 255).astype(np.uint8)
    if kind != "markov":
        raise ValueError(kind)
    src = source(seed)
    n = len(rows)
    # Symbol indices: run the chain from position 0 (cheap, vectorised over rows).
    a = np.zeros(n, dtype=np.int64)
    b = np.zeros(n, dtype=np.int64)
    out = np.empty((n, length), dtype=np.uint8)
    for p in range(start + length):
        u = _uniforms(keys, np.full(n, p, dtype=np.uint64))
        ctx = a * NSYM + b
        k = (u[:, None] >= src.cdf[ctx]).sum(axis=1)
        k = np.minimum(k, NSUCC - 1)
        c = src.succ[ctx, k]
        if p >= start:
            out[:, p - start] = ALPHABET[c]
        a, b = b, c
    return out


def window(rows, k: int, T: int, seed: int = 0x5EED, kind: str = "markov") -> np.ndarray:
    """The k-th TBTT window (T+1 bytes) of each row: uint8 [len(rows), T+1]."""
    return stream(rows, k * T, T + 1, seed=seed, kind=kind)


def windows(rows, k0: int, count: int, T: int, seed: int = 0x5EED, kind: str = "markov") -> np.ndarray:
    """Windows k0 .. k0+count-1 in one pass: uint8 [count, len(rows), T+1]."""
    s = stream(rows, k0 * T, count * T + 1, seed=seed, kind=kind)
    return np.stack([s[:, j * T: j * T + T + 1] for j in range(count)])
