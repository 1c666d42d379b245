"""Held-out BPC through the data pipeline: evaluation shards from the
library's loader, every window through mlstm_eval with the loader's reset masks, against the
oracle's evaluate() carried over the oracle pipeline's windows."""
import numpy as np
import pytest

from gpu_helpers import make_model, oracle_theta
from oracle import data_oracle as D
import oracle.mlstm_oracle as O
import paper_1808_01371_b200 as M
from synth import bytestream

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("mixed", 5e-3)])
def test_heldout_bpc_matches_oracle(precision, tol):
    h, e, B, T = 64, 64, 8, 16
    # >= 8 x 1002 records so the 1/1002 validation split fills B = 8 evaluation shards
    stream = bytestream.stream(np.arange(64), 0, 5000).tobytes()
    cuts = np.cumsum(np.random.default_rng(0).integers(20, 50, size=9000))
    recs = [stream[a:b] for a, b in zip(np.r_[0, cuts[:-1]], cuts) if b <= len(stream)]
    seed = 3
    corpus = M.Corpus(recs, seed=seed)
    _, va, _ = D.split_corpus(recs, seed)
    loader = M.Loader(corpus, M.MLSTM_SPLIT_VAL, M.MLSTM_SHARDS_EVAL, B, T, seed=seed + 1)
    m = make_model(h, e, B, T, precision)
    bpc = M.heldout_bpc(m, loader)
    # oracle: the same windows, state carried within a shard and zeroed at a shard start
    P = O.unflatten(oracle_theta(h, e), h, e)
    hs, cs = np.zeros((B, h)), np.zeros((B, h))
    nats = tokens = 0.0
    for rows, reset, valid in D.minibatches(D.make_shards(va, B, "eval", seed + 1), B, T):
        by = np.frombuffer(b"".join(rows), dtype=np.uint8).reshape(B, T + 1)
        n, tok, (hs, cs) = O.evaluate(P, by, hs, cs, reset=np.array(reset), valid=np.array(valid))
        nats += n
        tokens += tok
    ref = nats / tokens / np.log(2.0)
    assert tokens > 0 and abs(bpc - ref) <= tol * ref, (bpc, ref)
