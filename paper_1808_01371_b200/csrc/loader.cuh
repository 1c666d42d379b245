// loader.cuh -- host-side shard-contiguous TBTT data pipeline (include/mlstm_data.h; SURVEY NEXT #2;
// P:143-147 [§VI "Data Sharding"]).  Included by mlstm.cu (one translation unit, so it
// shares the thread-local error message); no device code.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/mlstm_data.h"

struct mlstm_corpus {
  std::vector<std::vector<uint8_t>> records;  // shuffled order
  int64_t n[3] = {0, 0, 0};                   // train, val, test record counts (in that order)
};

struct mlstm_loader {
  std::vector<std::vector<uint8_t>> shards;
  int B = 0, T = 0;
  std::vector<int64_t> shard_of, pos;  // per row: current shard (-1 = none yet) and window start
  int64_t next_shard = 0;
  bool first = true;
};

namespace {

uint64_t splitmix64_host(uint64_t seed, uint64_t q) {
  uint64_t z = seed + (q + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Fisher-Yates: for i = n-1 .. 1 (draw index d = n-1-i), swap(v[i], v[splitmix64(seed, d) % (i+1)]).
template <typename V>
void seeded_shuffle(V& v, uint64_t seed) {
  const int64_t n = (int64_t)v.size();
  for (int64_t i = n - 1; i >= 1; --i) {
    const uint64_t j = splitmix64_host(seed, (uint64_t)(n - 1 - i)) % (uint64_t)(i + 1);
    std::swap(v[i], v[j]);
  }
}

}  // namespace

extern "C" {

mlstm_status mlstm_corpus_create(const uint8_t* data, const int64_t* offsets, int64_t nrecords, uint64_t seed,
                                 mlstm_corpus** out) {
  if (!out || !offsets || (nrecords > 0 && !data)) return fail(MLSTM_EINVAL, "corpus: null argument");
  if (nrecords < 3) return fail(MLSTM_EINVAL, "corpus: fewer than 3 records (one per split needed)");
  if (offsets[0] != 0) return fail(MLSTM_EINVAL, "corpus: offsets[0] must be 0");
  for (int64_t r = 0; r < nrecords; ++r)
    if (offsets[r + 1] < offsets[r]) return fail(MLSTM_EINVAL, "corpus: offsets must be non-decreasing");
  auto* c = new mlstm_corpus;
  c->records.resize(nrecords);
  for (int64_t r = 0; r < nrecords; ++r) c->records[r].assign(data + offsets[r], data + offsets[r + 1]);
  seeded_shuffle(c->records, seed);
  // 1000 : 1 : 1; proportional rounding with every split non-empty
  const int64_t held = std::max<int64_t>(1, (int64_t)std::llround((double)nrecords / 1002.0));
  c->n[1] = c->n[2] = held;
  c->n[0] = nrecords - 2 * held;
  if (c->n[0] < 1) {
    delete c;
    return fail(MLSTM_EINVAL, "corpus: too few records for a 1000:1:1 split");
  }
  *out = c;
  return MLSTM_OK;
}

mlstm_status mlstm_corpus_split_sizes(const mlstm_corpus* c, int64_t out[3]) {
  if (!c || !out) return fail(MLSTM_EINVAL, "null argument");
  for (int i = 0; i < 3; ++i) out[i] = c->n[i];
  return MLSTM_OK;
}

void mlstm_corpus_destroy(mlstm_corpus* c) { delete c; }

mlstm_status mlstm_loader_create(const mlstm_corpus* c, int32_t split, int32_t kind, int32_t B, int32_t T,
                                 uint64_t seed, mlstm_loader** out) {
  if (!c || !out) return fail(MLSTM_EINVAL, "loader: null argument");
  if (split < 0 || split > 2 || (kind != MLSTM_SHARDS_TRAIN && kind != MLSTM_SHARDS_EVAL) || B < 1 || T < 1)
    return fail(MLSTM_EINVAL, "loader: bad split / kind / B / T");
  // the split's records (train first, then val, then test in the corpus order)
  const int64_t begin = split == 0 ? 0 : (split == 1 ? c->n[0] : c->n[0] + c->n[1]);
  std::vector<int64_t> idx(c->n[split]);
  for (int64_t i = 0; i < c->n[split]; ++i) idx[i] = begin + i;
  const int64_t nshards = kind == MLSTM_SHARDS_EVAL ? B : std::max<int64_t>(1000, B);
  if ((int64_t)idx.size() < nshards)
    return fail(MLSTM_EINVAL, "loader: fewer records than shards (lower B or use a larger corpus)");
  seeded_shuffle(idx, seed);
  auto* L = new mlstm_loader;
  L->shards.resize(nshards);
  for (int64_t i = 0; i < (int64_t)idx.size(); ++i) {  // round-robin after the shuffle
    const auto& rec = c->records[idx[i]];
    auto& sh = L->shards[i % nshards];
    if (!sh.empty()) sh.push_back('\n');  // record boundaries joined with a newline
    sh.insert(sh.end(), rec.begin(), rec.end());
  }
  L->B = B;
  L->T = T;
  mlstm_loader_rewind(L);
  *out = L;
  return MLSTM_OK;
}

int64_t mlstm_loader_num_shards(const mlstm_loader* L) { return L ? (int64_t)L->shards.size() : 0; }

mlstm_status mlstm_loader_shard(const mlstm_loader* L, int64_t i, uint8_t* out, int64_t cap, int64_t* len) {
  if (!L || i < 0 || i >= (int64_t)L->shards.size() || (cap > 0 && !out)) return fail(MLSTM_EINVAL, "bad shard");
  const auto& s = L->shards[i];
  if (cap > 0) memcpy(out, s.data(), (size_t)std::min<int64_t>(cap, (int64_t)s.size()));
  if (len) *len = (int64_t)s.size();
  return MLSTM_OK;
}

mlstm_status mlstm_loader_rewind(mlstm_loader* L) {
  if (!L) return fail(MLSTM_EINVAL, "null loader");
  L->shard_of.assign(L->B, -1);
  L->pos.assign(L->B, 0);
  L->next_shard = 0;
  L->first = true;
  return MLSTM_OK;
}

mlstm_status mlstm_loader_next(mlstm_loader* L, uint8_t* bytes, uint8_t* reset, uint8_t* valid, int32_t* end) {
  if (!L || !bytes || !reset || !end) return fail(MLSTM_EINVAL, "loader_next: null argument");
  const int64_t W = (int64_t)L->T + 1;
  // plan the batch first so that an end of epoch leaves the outputs and cursors untouched
  std::vector<int64_t> sh(L->shard_of), ps(L->pos);
  std::vector<uint8_t> rs(L->B, 0), ok(L->B, 1);
  int64_t next = L->next_shard;
  int nvalid = 0;
  for (int j = 0; j < L->B; ++j) {
    if (sh[j] == -2) {  // this row ran out of shards earlier in the epoch
      ok[j] = 0;
      continue;
    }
    while (sh[j] < 0 || ps[j] + W > (int64_t)L->shards[sh[j]].size()) {  // needs a (new) shard
      if (next >= (int64_t)L->shards.size()) {  // none left: the row idles for the rest of the epoch
        sh[j] = -2;
        ok[j] = 0;
        break;
      }
      sh[j] = next++;
      ps[j] = 0;
      rs[j] = 1;
    }
    nvalid += ok[j];
  }
  if (nvalid == 0) {  // every shard consumed ("epoch ends when all shards are consumed")
    *end = 1;
    return MLSTM_OK;
  }
  for (int j = 0; j < L->B; ++j) {
    if (ok[j]) {
      memcpy(bytes + (size_t)j * W, L->shards[sh[j]].data() + ps[j], (size_t)W);
      ps[j] += L->T;  // consecutive windows overlap by one byte (Q6)
    } else {
      memset(bytes + (size_t)j * W, 0, (size_t)W);
      rs[j] = 1;
    }
    reset[j] = rs[j];
    if (valid) valid[j] = ok[j];
  }
  L->shard_of = sh;
  L->pos = ps;
  L->next_shard = next;
  L->first = false;
  *end = 0;
  return MLSTM_OK;
}

void mlstm_loader_destroy(mlstm_loader* L) { delete L; }

}  // extern "C"
