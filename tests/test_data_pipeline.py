"""Shard-contiguous TBTT data pipeline: the plain-Python
oracle against the paper's / SPEC's worked examples and properties, and the library's C ABI
(include/mlstm_data.h) against the oracle byte for byte.  CPU only."""
import numpy as np
import pytest

from oracle import data_oracle as D
import paper_1808_01371_b200 as M


def _records(n, seed, lo=3, hi=40):
    rng = np.random.default_rng(seed)
    return [bytes(rng.integers(32, 127, size=int(rng.integers(lo, hi))).astype(np.uint8)) for _ in range(n)]


# ---------------------------------------------------------------- oracle pins -----------

@pytest.mark.parametrize("n,sizes", [(1002, (1000, 1, 1)), (2004, (2000, 2, 2)), (3, (1, 1, 1))])
def test_split_ratio_examples(n, sizes):
    """1002 records -> 1000/1/1, 2004 -> 2000/2/2; tiny corpora keep every split non-empty."""
    tr, va, te = D.split_corpus(_records(n, 0), seed=5)
    assert (len(tr), len(va), len(te)) == sizes


def test_split_is_a_deterministic_partition():
    recs = [bytes([i % 256, i // 256]) for i in range(5000)]
    a = D.split_corpus(recs, 9)
    assert a == D.split_corpus(recs, 9)                               # S:331 determinism
    assert sorted(a[0] + a[1] + a[2]) == sorted(recs)                  # disjoint and exhaustive
    assert D.split_corpus(recs, 10) != a
    with pytest.raises(ValueError):
        D.split_corpus(recs[:2], 0)


@pytest.mark.parametrize("kind,B,count", [("train", 256, 1000), ("train", 2048, 2048), ("eval", 16, 16)])
def test_shard_counts(kind, B, count):
    """max(1000, B) training shards, B evaluation shards."""
    recs = _records(2100, 1)
    sh = D.make_shards(recs, B, kind, seed=3)
    assert len(sh) == count
    # every record in exactly one shard, records joined by one newline each
    assert sum(len(s) for s in sh) == sum(len(r) for r in recs) + len(recs) - count
    with pytest.raises(ValueError):
        D.make_shards(recs[:10], 16, "eval", 0)


def test_records_joined_with_newline():
    """S:363 "Record boundaries inside a shard are joined with a newline delimiter": a one-shard split
    of three records is their newline-joined concatenation in the seeded round-robin order."""
    recs = [b"ab", b"cde", b"f"]
    order = D.seeded_shuffle(list(range(3)), 4)
    assert D.make_shards(recs, 1, "eval", seed=4) == [b"\n".join(recs[i] for i in order)]


def test_tiny_minibatch_enumeration():
    """S:345 (windows of T+1 bytes overlapping by one byte, Q6): shards 'abcdefghi', 'jklmnopqr', B=2,
    T=4 -> batch 1 rows ('abcde', 'jklmn') with reset on both, batch 2 ('efghi', 'nopqr') without."""
    out = list(D.minibatches([b"abcdefghi", b"jklmnopqr"], B=2, T=4))
    assert out == [([b"abcde", b"jklmn"], [1, 1], [1, 1]), ([b"efghi", b"nopqr"], [0, 0], [1, 1])]
    # B=1, one shard -> sequential windows
    assert [r[0][0] for r in D.minibatches([b"0123456789"], B=1, T=3)] == [b"0123", b"3456", b"6789"]
    # S:347 "epoch ends when all shards are consumed": with three shards and two rows, row 0 takes the
    # third shard after its first and the epoch runs on with row 1 idle until that shard is done
    out = list(D.minibatches([b"abcde", b"fghij", b"klmnopqrs"], B=2, T=4))
    assert [o[0][0] for o in out] == [b"abcde", b"klmno", b"opqrs"]
    assert [o[2] for o in out] == [[1, 1], [1, 0], [1, 0]]
    assert [o[1] for o in out] == [[1, 1], [1, 1], [0, 1]]


def test_contiguity_coverage_and_target_alignment():
    """each row's consecutive windows are contiguous ranges of one shard (until a reset), and
    over one epoch every shard byte but its tail (< T+1 bytes) is an input exactly once."""
    shards = D.make_shards(_records(1500, 2, 50, 400), 4, "eval", seed=1)
    B, T = 4, 16
    seen = {i: [] for i in range(len(shards))}
    cur = [None] * B
    nxt = 0
    for rows, reset, valid in D.minibatches(shards, B, T):
        for j in range(B):
            if not valid[j]:
                assert rows[j] == bytes(T + 1) and reset[j] == 1
                continue
            if reset[j]:
                cur[j] = nxt
                nxt += 1
            seen[cur[j]].append(rows[j])
    assert nxt == len(shards)  # every shard was taken
    for i, wins in seen.items():
        s = shards[i]
        # reconstruction: windows overlap by one byte and tile a prefix of the shard; the rest is a
        # tail shorter than one window
        recon = wins[0] + b"".join(w[1:] for w in wins[1:]) if wins else b""
        assert s.startswith(recon)
        assert len(s) - len(recon) < T + 1 if wins else len(s) < T + 1


# ---------------------------------------------------------------- library vs oracle ------

@pytest.mark.parametrize("B,T,kind,seed", [(4, 8, "eval", 7), (16, 32, "train", 11), (3, 5, "train", 0)])
def test_library_loader_matches_oracle(B, T, kind, seed):
    recs = _records(3100, seed, 2, 90)
    tr, va, te = D.split_corpus(recs, seed)
    c = M.Corpus(recs, seed=seed)
    assert c.split_sizes() == (len(tr), len(va), len(te))
    split = tr if kind == "train" else va
    if kind == "eval" and len(va) < B:
        split, sid = tr, M.MLSTM_SPLIT_TRAIN
    else:
        sid = M.MLSTM_SPLIT_TRAIN if kind == "train" else M.MLSTM_SPLIT_VAL
    shards = D.make_shards(split, B, kind, seed + 1)
    L = M.Loader(c, sid, M.MLSTM_SHARDS_TRAIN if kind == "train" else M.MLSTM_SHARDS_EVAL, B, T, seed=seed + 1)
    assert L.num_shards() == len(shards)
    for i in (0, 1, len(shards) - 1):
        assert L.shard(i) == shards[i]
    n = 0
    for (rows, reset, valid), got in zip(D.minibatches(shards, B, T), L):
        assert got[0].tobytes() == b"".join(rows) and got[1].tolist() == reset and got[2].tolist() == valid
        n += 1
        if n == 400:
            break
    if n < 400:  # both ended the epoch at the same batch
        assert L.next() is None
    L.rewind()                                                           # same shards, same order
    first = L.next()
    rows, reset, valid = next(iter(D.minibatches(shards, B, T)))
    assert first[0].tobytes() == b"".join(rows) and first[1].tolist() == reset


def test_library_rejects_bad_arguments():
    with pytest.raises(M.MlstmError):
        M.Corpus([b"a", b"b"])
    c = M.Corpus(_records(50, 0))
    with pytest.raises(M.MlstmError):
        M.Loader(c, M.MLSTM_SPLIT_TRAIN, M.MLSTM_SHARDS_TRAIN, 4, 8)     # 48 records < 1000 shards
    L = M.Loader(c, M.MLSTM_SPLIT_TRAIN, M.MLSTM_SHARDS_EVAL, 4, 8)
    assert L.num_shards() == 4
