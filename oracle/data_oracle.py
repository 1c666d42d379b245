"""Plain-Python oracle of the shard-contiguous TBTT data pipeline.

TEST INFRASTRUCTURE ONLY (same rules as mlstm_oracle.py: only tests/, __graft_entry__.smoke() and
bench.py's reference legs may import it; it shares no code with the library).

Follows P:143-147 [§VI "Data Sharding"] and S:325-357 step by step:
  split 1000:1:1 after a seeded shuffle; B eval shards / max(1000, B) train shards dealt round-robin
  after a second seeded shuffle, records joined with a newline inside a shard; minibatch row j
  continues its shard window by window (windows of T+1 bytes overlapping by one byte, reading Q6) and
  takes the next unassigned shard with reset = 1 when fewer than T+1 bytes remain; a row that finds no
  unassigned shard idles (valid = 0) and the epoch ends when every shard is consumed.
Shuffles: Fisher-Yates, i = n-1 .. 1, j = splitmix64(seed, n-1-i) mod (i+1) (reading Q25).
Pins: tests/test_data_pipeline.py (S:329-330, S:337-339, S:345-347 examples; contiguity, coverage,
determinism properties).
"""
from __future__ import annotations

M64 = (1 << 64) - 1


def splitmix64(seed: int, q: int) -> int:
    z = (seed + (q + 1) * 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def seeded_shuffle(items: list, seed: int) -> list:
    v = list(items)
    n = len(v)
    for i in range(n - 1, 0, -1):
        j = splitmix64(seed, n - 1 - i) % (i + 1)
        v[i], v[j] = v[j], v[i]
    return v


def split_corpus(records: list[bytes], seed: int):
    """(train, val, test) record lists in the ratio 1000:1:1; each split non-empty."""
    if len(records) < 3:
        raise ValueError("insufficient data: fewer than 3 records")
    recs = seeded_shuffle(records, seed)
    held = max(1, int(round(len(recs) / 1002.0)))
    ntrain = len(recs) - 2 * held
    if ntrain < 1:
        raise ValueError("insufficient data for a 1000:1:1 split")
    return recs[:ntrain], recs[ntrain:ntrain + held], recs[ntrain + held:]


def make_shards(split: list[bytes], B: int, kind: str, seed: int) -> list[bytes]:
    """B shards for evaluation, max(1000, B) for training; round-robin after a shuffle."""
    nshards = B if kind == "eval" else max(1000, B)
    if len(split) < nshards:
        raise ValueError("shards exceed records: lower B")
    order = seeded_shuffle(list(range(len(split))), seed)
    parts = [[] for _ in range(nshards)]
    for i, r in enumerate(order):
        parts[i % nshards].append(split[r])
    return [b"\n".join(p) for p in parts]  # "record boundaries inside a shard are joined with a newline"


def minibatches(shards: list[bytes], B: int, T: int):
    """Yields (rows: list of B byte strings of length T+1, reset: list of B ints, valid: list of B ints)
    until every shard is consumed (row j of batch i+1 continues row j of batch i within a shard;
    S:347 "epoch ends when all shards are consumed").  A row without an unassigned shard is idle for
    the rest of the epoch: valid 0, T+1 zero bytes, reset 1."""
    IDLE = -1
    shard_of, pos, nxt = [None] * B, [0] * B, 0
    while True:
        rows, reset, valid = [], [], []
        new_shard_of, new_pos = list(shard_of), list(pos)
        for j in range(B):
            r = 0
            while new_shard_of[j] != IDLE and (new_shard_of[j] is None
                                               or new_pos[j] + T + 1 > len(shards[new_shard_of[j]])):
                if nxt >= len(shards):
                    new_shard_of[j] = IDLE
                    break
                new_shard_of[j], new_pos[j], r = nxt, 0, 1
                nxt += 1
            if new_shard_of[j] == IDLE:
                rows.append(bytes(T + 1))
                reset.append(1)
                valid.append(0)
                continue
            s = shards[new_shard_of[j]]
            rows.append(s[new_pos[j]:new_pos[j] + T + 1])
            reset.append(r)
            valid.append(1)
            new_pos[j] += T
        if not any(valid):
            return
        shard_of, pos = new_shard_of, new_pos
        yield rows, reset, valid
