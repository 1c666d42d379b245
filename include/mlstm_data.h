/*
 * mlstm_data.h -- C ABI of the shard-contiguous TBTT data pipeline in libmlstm.so:
 * the 1000:1:1 corpus split, the training / evaluation shards and the minibatch iterator whose
 * rows are contiguous across consecutive minibatches, so the hidden state persists across TBTT
 * windows (P:143-147 [§VI "Data Sharding"]).  Host-only code: no GPU needed.
 *
 * Conventions: plain C types; every call returns an mlstm_status (mlstm.h) and reports failures
 * through mlstm_last_error(); MLSTM_EINVAL on bad arguments, with no side effects.  Objects are
 * owned by the caller and freed with the matching *_destroy.
 *
 * Determinism (reading Q25): every shuffle is a Fisher-Yates pass whose i-th draw is
 * splitmix64(seed', i) mod (n_remaining), the same counter-based generator as the parameter init
 * (Q12), so a plain reimplementation reproduces every split, shard and minibatch byte for byte.
 */
#ifndef MLSTM_DATA_H_
#define MLSTM_DATA_H_

#include <stdint.h>

#include "mlstm.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mlstm_corpus mlstm_corpus; /* a copy of the records and their 1000:1:1 split    */
typedef struct mlstm_loader mlstm_loader; /* one split's shards and the B row cursors            */

enum { MLSTM_SPLIT_TRAIN = 0, MLSTM_SPLIT_VAL = 1, MLSTM_SPLIT_TEST = 2 };
enum { MLSTM_SHARDS_TRAIN = 0, MLSTM_SHARDS_EVAL = 1 };

/* Copies nrecords records (record r = data[offsets[r] .. offsets[r+1]), offsets has nrecords+1
 * entries, non-decreasing, offsets[0] = 0), shuffles them with `seed` and splits them train / val /
 * test in the ratio 1000 : 1 : 1: n_val = n_test = max(1, round(n / 1002)), n_train = the
 * rest.  Fewer than 3 records: MLSTM_EINVAL. */
mlstm_status mlstm_corpus_create(const uint8_t* data, const int64_t* offsets, int64_t nrecords, uint64_t seed,
                                 mlstm_corpus** out);
/* Records per split: out[MLSTM_SPLIT_TRAIN], out[MLSTM_SPLIT_VAL], out[MLSTM_SPLIT_TEST]. */
mlstm_status mlstm_corpus_split_sizes(const mlstm_corpus* corpus, int64_t out[3]);
void mlstm_corpus_destroy(mlstm_corpus* corpus);

/* Shards of one split: B shards for evaluation (kind MLSTM_SHARDS_EVAL), max(1000, B) for
 * training; the split's records are shuffled with `seed` and dealt round-robin, each shard is the
 * concatenation of its records joined with a newline.  Windows hold T+1 bytes (T inputs + the next byte as the last
 * target) and consecutive windows of a row overlap by one byte (Q6).  Fewer records than shards:
 * MLSTM_EINVAL. */
mlstm_status mlstm_loader_create(const mlstm_corpus* corpus, int32_t split, int32_t kind, int32_t B, int32_t T,
                                 uint64_t seed, mlstm_loader** out);
int64_t mlstm_loader_num_shards(const mlstm_loader* loader);
/* Shard i's bytes (test access): copies min(cap, length) bytes to out, length to *len. */
mlstm_status mlstm_loader_shard(const mlstm_loader* loader, int64_t i, uint8_t* out, int64_t cap, int64_t* len);
/* The next minibatch: host bytes [B][T+1], reset [B] and valid [B] (valid may be NULL).  Row j
 * continues its shard from the previous minibatch; when fewer than T+1 bytes remain, row j takes the
 * next unassigned shard (in row order) and reset[j] = 1 (the hidden state restarts at zero at a shard
 * start).  The first minibatch of an epoch has every reset set.  A row that finds no unassigned
 * shard idles for the rest of the epoch: valid[j] = 0, zero bytes, reset[j] = 1 (pass reset = 2 for
 * such rows to mlstm_eval so they are not counted).  When no row is valid -- every shard consumed
 * (S:347), so every shard byte except a tail shorter than T+1 was an input exactly once -- *end = 1
 * and the outputs are left untouched (end of epoch, not an error). */
mlstm_status mlstm_loader_next(mlstm_loader* loader, uint8_t* bytes, uint8_t* reset, uint8_t* valid, int32_t* end);
/* Back to the start of the epoch: the same shards in the same order ("used for all training epochs
 * with no further shuffling"). */
mlstm_status mlstm_loader_rewind(mlstm_loader* loader);
void mlstm_loader_destroy(mlstm_loader* loader);

/* Held-out BPC over one epoch of an evaluation loader, accumulated in the library: rewinds the
 * loader and runs every minibatch through mlstm_eval from the eval-slot state (reset = the loader's
 * reset, 2 for idle rows), stopping after max_batches (< 0: the whole epoch).  Outputs (host, any may
 * be NULL): nats_sum and tokens summed over the batches and all ranks, bpc = nats_sum / tokens / ln 2.
 * The loader's B and T must equal the context's batch (rows per micro-batch) and seq_len, else
 * MLSTM_EINVAL.  Collective when world > 1: every rank calls it with loaders yielding equally many
 * batches. */
mlstm_status mlstm_heldout_bpc(mlstm_ctx* ctx, mlstm_loader* loader, int64_t max_batches, double* nats_sum,
                               int64_t* tokens, double* bpc);

#ifdef __cplusplus
}
#endif

#endif /* MLSTM_DATA_H_ */
