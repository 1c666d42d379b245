"""Frozen-feature transfer mechanism ("final cell state ... logistic
regression"): the GPU's final cell states over multi-window texts equal the oracle's, and a
scikit-learn logistic regression trains on them.  The paper's accuracies need trained weights and
the SST / IMDB data (out of scope); only the mechanism is checked."""
import numpy as np
import pytest

from gpu_helpers import make_model, oracle_theta
import oracle.mlstm_oracle as O
import paper_1808_01371_b200 as M
from synth import bytestream

pytestmark = pytest.mark.gpu


def test_cell_features_match_oracle_and_feed_a_classifier():
    from sklearn.linear_model import LogisticRegression
    h, e, B, T, k = 128, 64, 32, 8, 3
    m = make_model(h, e, B, T, "fp32")
    # two "classes": the order-2 Markov source and iid bytes
    a = bytestream.stream(np.arange(B // 2), 0, k * T + 1)
    b = bytestream.stream(np.arange(B // 2), 0, k * T + 1, kind="uniform")
    texts = [r.tobytes() for r in a] + [r.tobytes() for r in b]
    feats = M.cell_features(m, texts)
    P = O.unflatten(oracle_theta(h, e), h, e)
    by = np.frombuffer(b"".join(texts), dtype=np.uint8).reshape(B, k * T + 1)
    _, _, (_, cT) = O.forward(P, by, np.zeros((B, h)), np.zeros((B, h)))
    assert np.abs(feats - cT).max() <= 1e-5 * max(1.0, np.abs(cT).max())
    y = np.r_[np.zeros(B // 2), np.ones(B // 2)]
    clf = LogisticRegression(max_iter=2000).fit(feats, y)
    p = clf.predict_proba(feats)
    assert p.shape == (B, 2) and np.allclose(p.sum(1), 1.0)
