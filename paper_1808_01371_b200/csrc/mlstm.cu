// mlstm.cu -- host orchestrator and C ABI of libmlstm.so (include/mlstm.h).
//
// One context per rank.  A train step is enqueued on the caller's stream as two CUDA graphs
// (recorded on first use): A = forward + CE + BPTT + weight gradients, B = overflow check +
// scaler + Adam + cast + state carry, with the NCCL fp16 SUM allreduce of the gradient arena
// between them when world > 1.  See DESIGN.md for the data layout and kernel list.
#include <cudaTypedefs.h>
#include <nccl.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <type_traits>
#include <vector>

#include "../../include/mlstm.h"
#include "gemm.cuh"
#include "kernels.cuh"
#include "recur.cuh"

using namespace mlstm;

namespace mlstm {  // trace tags of the fused epilogues (mlstm_trace_read)
template <typename S> struct EpiTag<EpiF1<S>> { static constexpr int value = 1; };
template <typename S> struct EpiTag<EpiF2<S>> { static constexpr int value = 2; };
template <typename S> struct EpiTag<EpiF2IO<S>> { static constexpr int value = 2; };
template <typename S> struct EpiTag<EpiF1IO<S>> { static constexpr int value = 1; };
template <typename S> struct EpiTag<EpiB1IO<S>> { static constexpr int value = 3; };
template <typename S> struct EpiTag<EpiB1<S>> { static constexpr int value = 3; };
template <typename S> struct EpiTag<EpiB2<S>> { static constexpr int value = 4; };
template <typename S> struct EpiTag<EpiY<S>> { static constexpr int value = 5; };
template <typename S> struct EpiTag<EpiDHdec<S>> { static constexpr int value = 6; };
template <typename S> struct EpiTag<EpiTab<S>> { static constexpr int value = 7; };
template <typename S> struct EpiTag<EpiWgrad<S>> { static constexpr int value = 8; };
template <> struct EpiTag<EpiPartial> { static constexpr int value = 9; };
// epilogues that run on MN-major operands (the weight-gradient GEMMs)
template <class E> constexpr bool kMNEpi = false;
template <typename S> constexpr bool kMNEpi<EpiWgrad<S>> = true;
template <> constexpr bool kMNEpi<EpiPartial> = true;
template <> constexpr bool kMNEpi<EpiWacc> = true;
// epilogues of the backward recurrence's GEMMs, whose B operand (a weight) may be read MN-major
// straight from its row-major working copy (K-major A, MN-major B)
template <class E> constexpr bool kBMNEpi = false;
template <typename S> constexpr bool kBMNEpi<EpiB1IO<S>> = true;
template <typename S> constexpr bool kBMNEpi<EpiB1<S>> = true;
template <typename S> constexpr bool kBMNEpi<EpiB2<S>> = true;
}  // namespace mlstm

namespace {

thread_local std::string g_err;

enum Phase { PH_PREP, PH_TAB, PH_FWD, PH_DEC, PH_CE, PH_DHDEC, PH_BWD, PH_WGRAD, PH_ALLREDUCE, PH_OPT, NPH };
const char* kPhaseNames[NPH] = {"prep", "tab", "fwd_rec", "decoder", "ce", "dhdec",
                                "bwd_rec", "wgrad", "allreduce", "optimizer"};

struct Opd {  // K-major operand view: [zdim][rows][K], element strides ld (row) and zstride
  const void* ptr;
  long rows, K, ld, zdim, zstride;
  uint32_t pol = 0;     // L2 policy code for its TMA loads (ptx::make_policy)
  bool weight = false;  // a parameter copy: not written by any kernel of the step before the optimiser
  bool mn = false;      // MN-major instead: element (r, k) at z*zstride + k*ld + r  ([K][rows] in memory)
};
constexpr uint32_t kPolFirst = 1u << 8;
inline uint32_t pol_last(float frac) { return (2u << 8) | (uint32_t)(frac * 255.f + 0.5f); }

struct Plan {
  int bn, splits;
  bool pair;     // CTA-pair (cta_group::2) 256-row tiles
  bool cluster;  // K split over the CTAs of a cluster, reduced in-kernel (1-CTA 128 x 256 tiles)
  bool persist = false;  // pair tiles walked by a persistent grid (more tiles than pairs fit)
};
constexpr long kSplitScratchFloats = 160L * 128 * 256;  // >= tiles * S partials of any cluster-split plan

long rup(long x, long m) { return (x + m - 1) / m * m; }
constexpr int kAsyncRing = 8;  // MLSTM_ASYNC steps in flight before the oldest is delivered

}  // namespace

struct mlstm_ctx {
  mlstm_config cfg{};
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;   // caller's stream: every launch and graph launch goes here
  cudaStream_t cap = nullptr;      // private stream graphs are recorded on (the caller's may be
                                   // the legacy default stream, which cannot be captured)
  bool mixed = true, tc = true;
  int h = 0, e = 0, B = 0, T = 0, Bp = 0;  // B = rows per micro-batch
  int Bfull = 0, nmb = 1;                    // rows per rank, micro-batches per step
  long P = 0, Kt = 0;
  ParamOffsets po{};
  uint8_t* ws = nullptr;
  size_t ws_bytes = 0;
  // buffers that are not in Net
  float *adam_m = nullptr, *adam_v = nullptr;
  uint8_t *bytes = nullptr, *reset = nullptr;
  int32_t* scratch_flag = nullptr;
  double* eval_tok = nullptr;  // token count of the last mlstm_eval (device, summed over ranks)
  DevState* st = nullptr;
  DevState* st_host = nullptr;  // pinned ring: slots [0, kAsyncRing) for MLSTM_ASYNC steps, slot kAsyncRing for
                                // synchronous ones (each step copies its DevState into its own slot)
  struct Pending {
    mlstm_step_result* out;
    int slot;
  };
  std::vector<Pending> pending;  // MLSTM_ASYNC steps not yet delivered, in step order
  int ring_next = 0;
  cudaEvent_t ring_ev[8] = {};
  int nblk_ce = 0;
  long part_elems = 0;
  int seg_splits = 1;
  float l2_wmh = 0.f, l2_wh = 0.f;  // evict_last fractions of the recurrent weights
  float* split_scratch = nullptr;
  bool pdl = true;                    // programmatic dependent launch of the GEMMs (MLSTM_PDL=0 disables)
  float pf_fwd = 0.f, pf_bwd = 0.f;   // L2 prefetch of the next W_h / W_h^T (MLSTM_PF_FWD/BWD; neutral,
                                      // profiles/r01_l2_prefetch.log)
  bool pf_stash = true;               // backward: prefetch the next epilogue's stash blocks (MLSTM_PF_STASH)
  Net<__half> nh{};
  Net<float> nf{};
  ncclComm_t comm = nullptr;
  // N>1: the gradient allreduce runs on a high-priority stream in buckets that start as soon as
  // the weight-gradient GEMM producing them finishes (W_h, then W_mh, then the rest), overlapping
  // the remaining weight-gradient work; MLSTM_AR_OVERLAP=0 reduces after graph A.
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_wh = nullptr, ev_wmh = nullptr, ev_a_end = nullptr, ev_comm = nullptr, ev_wh_a = nullptr,
              ev_wdec = nullptr;
  bool ar_overlap = true;
  int force_plan = 0;          // MLSTM_FORCE_PLAN (test instrument), applied while this ctx enqueues
  bool wgrad512 = true;        // weight gradients on 256 x 512 pair tiles (MLSTM_WGRAD512=0: 256 x 256)
  bool raster_group = true;    // weight-gradient GEMMs in bands of 8 M-tiles (MLSTM_RASTER_GROUP=0: N-fastest)
  // dW_h over the last side_chunks x side_ch timesteps on a low-priority side stream, on side_pairs CTA
  // pairs, while the per-timestep backward recurrence (128 CTAs) still runs
  // (MLSTM_WGRAD_SIDE=chunks[,ch[,pairs[,pol]]]; measured a wash under the power cap, DESIGN 9.1: off by default)
  int side_chunks = 0, side_ch = 32, side_pairs = 10, side_pol = 1;  // side_pol 1: operands evict_first
  cudaStream_t side = nullptr;
  cudaEvent_t side_ev[17] = {};  // [0, side_chunks): chunk j's dZ rows are final; [16]: side stream done
  float* wpart = nullptr;        // fp32 [4h][h] partial of dW_h over the side chunks
  int tc2p_pairs = 0;            // > 0: grid of the persistent pair engine for the launch being enqueued
  int prio = 0;                  // launch priority attribute of the GEMM being enqueued (0: none)
  int prio_hi = 0, prio_lo = 0;
  // persistent dataflow recurrence (recur.cuh): mlstm_config.recurrence = 1 (or MLSTM_RECUR=1)
  int recur_env = 1;
  int recur_ok = -1;
  bool recur_fwd_only = false;  // recurrence = 3: persistent forward, per-timestep BPTT
  bool bwd_needs_transposes = true;  // decided while recording graph A (enqueue_train_a)
  int rc_wkm = 0;                 // MLSTM_RC_WKM=1: persistent BPTT reads the transposed (K-major) weights
  int rc_exp = 0;                 // MLSTM_RC_EXP: 64 = no per-k-block trace records (see RcPolicy::exp)
  int rc_rotate = 1;              // MLSTM_RC_ROTATE
  int rc_pf_dist = 0;             // MLSTM_RC_PF: weight k-blocks prefetched into L2 ahead of the ring
  int rc_flag_lanes = 32;  // MLSTM_RC_FLAG_LANES: activation flags acquired in parallel (1 = serial)           // decided once per ctx (shape + co-residency), see recur_on()
  float* rc_scratch = nullptr;
  uint32_t* rc_flags = nullptr;
  int async_epi = 2;  // recurrent epilogue row I/O: 0 per-thread LSU, 1 bulk copies, 2 staged + coalesced (MLSTM_ASYNC_EPI)
  bool overlap_now() const { return world > 1 && ar_overlap && nmb == 1; }
  cudaGraphExec_t gA = nullptr, gB = nullptr;
  std::map<std::tuple<const void*, long, long, long, long, long, int>, CUtensorMap> maps;
  mlstm_status failed = MLSTM_OK;
  bool have_last = false;
  DevState last{};
  int nonfinite_run = 0;
  // profiling
  bool profile = false;
  cudaEvent_t ev[NPH + 1] = {};
  double phase_ms[NPH] = {};
  int32_t phase_launches[NPH] = {};
  int cur_phase = 0;
  int launches = 0;
  bool counting = false;
};

namespace {

mlstm_status fail(mlstm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define CUDA_OR_FAIL(ctx, x)                                                                   \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      if (ctx) (ctx)->failed = MLSTM_ECUDA;                                                    \
      return fail(MLSTM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));               \
    }                                                                                          \
  } while (0)

#define NCCL_OR_FAIL(ctx, x)                                                                   \
  do {                                                                                         \
    ncclResult_t r_ = (x);                                                                     \
    if (r_ != ncclSuccess) {                                                                   \
      if (ctx) (ctx)->failed = MLSTM_ENCCL;                                                    \
      return fail(MLSTM_ENCCL, std::string(#x) + ": " + ncclGetErrorString(r_));               \
    }                                                                                          \
  } while (0)

// ------------------------------------------------------------------ workspace layout
struct Carver {
  uint8_t* base;
  size_t off = 0;
  template <typename X>
  X* take(long count) {
    off = rup((long)off, 256);
    X* p = base ? reinterpret_cast<X*>(base + off) : nullptr;
    off += (size_t)count * sizeof(X);
    return p;
  }
};

int grid_for(long n, int threads = 256, int cap = 148 * 16) {
  long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

// Tile-N and split-K choice shared by the workspace layout and the launches.
// Engine choice (measured with mlstm_gemm_bench, profiles/r01_gemm_sweep.log): tcgen05 issue
// rate per k-block is nearly flat in N, so wide (BN = 256) tiles matter most; the CTA-pair engine
// (256 x 256 per pair) halves per-SM operand traffic and wins whenever it can fill ~60 pairs,
// with split-K where allowed.  Otherwise one CTA per 128-row tile with the widest BN that still
// fills ~120 SMs.
// Test instrument (MLSTM_FORCE_PLAN=pair|split|single): take one tile plan wherever it is legal, so
// small parity tests cover the plans that only full-size shapes select on their own.
int g_force_plan = 0;
int g_max_pairs = 74;  // CTA pairs resident at once (148 SMs); MLSTM_PERSIST_PAIRS overrides (tests)

Plan plan_gemm(bool tc, long M, long N, long K, bool allow_split) {
  Plan p{64, 1, false, false};
  const long kb = (K + 63) / 64;
  const long pairs = ((M + 255) / 256) * ((N + 255) / 256);
  if (tc && g_force_plan == 1 && M > 128) return Plan{256, 1, true, false, pairs > g_max_pairs};
  if (tc && g_force_plan == 4 && M > 128) return Plan{256, 1, true, false, true};
  if (tc && g_force_plan == 2 && kb >= 8) {
    const int sp = kb >= 16 ? 4 : 2;
    if (((M + 127) / 128) * ((N + 255) / 256) * sp <= 160) return Plan{256, sp, false, true};
  }
  if (tc && g_force_plan == 3) allow_split = false;
  if (tc && g_force_plan != 0) goto single;
  if (tc && M > 128 && pairs >= 60) return Plan{256, 1, true, false, pairs > g_max_pairs};
  if (tc) {
    const long mt = (M + 127) / 128;
    // 128 x 256 tiles with the K loop split over a cluster of S <= 4 CTAs when 256-wide tiles
    // alone cannot fill the GPU (measured: N=64 tiles issue MMAs at ~1/4 of the N=256 rate)
    const long tiles = mt * ((N + 255) / 256);
    int sp = 1;
    while (tiles * sp < 100 && sp < 4 && kb / (sp * 2) >= 4) sp *= 2;
    if (sp > 1 && tiles * sp <= 160) return Plan{256, sp, false, true};
  }
single:
  if (tc) {
    const long mt = (M + 127) / 128;
    for (int bn : {256, 128, 64}) {
      if (mt * ((N + bn - 1) / bn) >= 120 || bn == 64) {
        p.bn = bn;
        break;
      }
    }
  }
  if (allow_split) {
    const long tiles = ((M + 127) / 128) * ((N + p.bn - 1) / p.bn);
    while (tiles * p.splits < 148 && kb / (p.splits * 2) >= 4) p.splits *= 2;
  }
  return p;
}

// Shapes the persistent dataflow recurrence (recur.cuh) covers: mixed precision on tcgen05, 256 rows
// per micro-batch (one CTA pair along M), h a multiple of 256 with h/64 pairs resident at once.
bool recur_shape_ok(const mlstm_ctx* c) {
  return c->recur_env != 0 && c->tc && c->mixed && c->B == 256 && c->h % 256 == 0 && c->h / 32 <= 148 &&
         c->force_plan == 0;
}

template <typename S>
void carve(mlstm_ctx* c, Carver& cv, Net<S>& n) {
  const int h = c->h, e = c->e, B = c->B, T = c->T;
  const long P = c->P;
  n.h = h; n.e = e; n.B = B; n.T = T; n.Bp = c->Bp;
  n.Bfull = c->Bfull; n.nmb = c->nmb;
  n.po = c->po;
  n.master = cv.take<float>(P);
  c->adam_m = cv.take<float>(P);
  c->adam_v = cv.take<float>(P);
  n.arena = cv.take<S>(P);
  n.E_w = cv.take<S>(256L * e);
  n.Wcat_w = cv.take<S>(5L * h * e);
  n.Wmh_w = cv.take<S>((long)h * h);
  n.Wh_w = cv.take<S>(4L * h * h);
  n.Wdec_w = cv.take<S>(256L * h);
  n.WmhT = cv.take<S>((long)h * h);
  n.WhT = cv.take<S>(4L * h * h);
  n.WdecT = cv.take<S>(256L * h);
  c->bytes = cv.take<uint8_t>((long)B * (T + 1));
  c->reset = cv.take<uint8_t>(B);
  n.bytes = c->bytes;
  n.reset = c->reset;
  n.tab = cv.take<float>(256L * 5 * h);
  n.XZT = c->tc ? cv.take<S>(4L * h * 256) : nullptr;
  n.OHR = cv.take<S>((long)T * B * 256);
  n.Hrm = cv.take<S>((long)(T + 1) * B * h);
  n.Crm = cv.take<float>((long)(T + 1) * B * h);
  n.Mrm = cv.take<S>((long)T * B * h);
  n.Astash = cv.take<S>((long)T * B * h);
  n.Gates = cv.take<S>((long)T * B * 4 * h);
  n.Y = cv.take<float>((long)T * B * 256);
  n.lossrow = cv.take<float>((long)T * B);
  n.dY = cv.take<S>((long)T * B * 256);
  // tcgen05 path: dH_dec,t = dY_t W_dec enters the B2 accumulator as a second K segment (no buffer)
  n.dHdec = c->tc ? nullptr : cv.take<float>((long)T * B * h);
  n.G5 = cv.take<S>((long)T * B * 5 * h);
  n.dA = cv.take<S>((long)T * B * h);
  n.dC = cv.take<float>((long)B * h);
  // split-K partial buffer: the largest split GEMM among the weight gradients
  long part = 64;
  const long K = c->Kt;
  const long shapes[4][2] = {{4L * h, h}, {h, h}, {256, h}, {256, 5L * h}};
  g_force_plan = c->force_plan;  // size for the plans this ctx will take
  for (auto& s : shapes) {
    Plan p = plan_gemm(c->tc, s[0], s[1], K, true);
    if (p.splits > 1 && !p.pair && !p.cluster) part = std::max(part, (long)p.splits * s[0] * s[1]);
  }
  g_force_plan = 0;
  c->seg_splits = (int)std::max(1L, std::min(64L, (5L * h) / 512));
  part = std::max(part, (long)c->seg_splits * 256 * e);
  part = std::max(part, 5L * h * e);
  c->part_elems = part;
  n.part = cv.take<float>(part);
  c->split_scratch = c->tc ? cv.take<float>(kSplitScratchFloats) : nullptr;
  if (recur_shape_ok(c)) {
    c->rc_scratch = cv.take<float>(rc_scratch_floats(h));
    c->rc_flags = cv.take<uint32_t>(kRcFlagWords(h / 64));
  }
  n.Scan = cv.take<float>(256L * 5 * h);
  n.hstate = cv.take<S>(2L * c->Bfull * h);
  n.cstate = cv.take<float>(2L * c->Bfull * h);
  n.gacc = c->nmb > 1 ? cv.take<float>(P) : nullptr;
  n.wn_norm = c->po.wn ? cv.take<float>(10L * h) : nullptr;
  c->nblk_ce = (int)(((long)T * B + 31) / 32);
  n.loss_part = cv.take<double>(c->nblk_ce);
  n.colsum_part = cv.take<float>((long)c->nblk_ce * 256);
  n.st = cv.take<DevState>(1);
  c->st = n.st;
  c->scratch_flag = cv.take<int32_t>(4);
  c->eval_tok = cv.take<double>(2);
}

mlstm_status validate(const mlstm_config* cfg) {
  if (!cfg) return fail(MLSTM_EINVAL, "null config");
  if (cfg->hidden <= 0 || cfg->hidden % 64) return fail(MLSTM_EINVAL, "hidden must be a positive multiple of 64");
  if (cfg->embed <= 0 || cfg->embed % 64) return fail(MLSTM_EINVAL, "embed must be a positive multiple of 64");
  if (cfg->vocab != 256) return fail(MLSTM_EINVAL, "vocab must be 256 (byte level)");
  if (cfg->seq_len <= 0 || cfg->batch <= 0) return fail(MLSTM_EINVAL, "seq_len and batch must be positive");
  if (cfg->micro_batch < 0 || (cfg->micro_batch > 0 && cfg->batch % cfg->micro_batch != 0))
    return fail(MLSTM_EINVAL, "micro_batch must be 0 (= batch) or divide batch");
  if (cfg->weight_norm != 0 && cfg->weight_norm != 1) return fail(MLSTM_EINVAL, "weight_norm must be 0 or 1 (Q24)");
  if (cfg->precision != MLSTM_FP32 && cfg->precision != MLSTM_MIXED) return fail(MLSTM_EINVAL, "bad precision");
  if (cfg->recurrence < 0 || cfg->recurrence > 3) return fail(MLSTM_EINVAL, "recurrence must be 0, 1, 2 or 3");
  if (!(cfg->decay_iters > 0) || !(cfg->lr0 >= 0)) return fail(MLSTM_EINVAL, "bad LR schedule");
  if (!(cfg->scale_min > 0) || !(cfg->scale_max >= cfg->scale_min) || !(cfg->scale_init >= cfg->scale_min) ||
      !(cfg->scale_init <= cfg->scale_max) || cfg->scale_growth_interval <= 0)
    return fail(MLSTM_EINVAL, "bad loss-scale settings");
  return MLSTM_OK;
}

void set_dims(mlstm_ctx* c, const mlstm_config* cfg) {
  c->cfg = *cfg;
  // 1: persistent forward + BPTT; 3: persistent forward, per-timestep BPTT; 0 (default), 2: per-timestep
  c->recur_env = (cfg->recurrence == 1 || cfg->recurrence == 3) ? 1 : 0;
  c->recur_fwd_only = cfg->recurrence == 3;
  c->h = cfg->hidden;
  c->e = cfg->embed;
  c->Bfull = cfg->batch;
  c->B = cfg->micro_batch > 0 ? cfg->micro_batch : cfg->batch;  // rows per micro-batch
  c->nmb = c->Bfull / c->B;
  c->T = cfg->seq_len;
  c->Bp = c->B;
  c->Kt = (long)c->T * c->B;  // K of the weight-gradient GEMMs: every (t, b) of the micro-batch
  c->po.set(c->h, c->e, cfg->weight_norm);
  c->P = c->po.P;
  c->mixed = cfg->precision == MLSTM_MIXED;
  if (const char* v = getenv("MLSTM_L2_WMH")) c->l2_wmh = (float)atof(v);  // tuning knobs
  if (const char* v = getenv("MLSTM_PDL")) c->pdl = v[0] != '0';
  if (const char* v = getenv("MLSTM_PF_FWD")) c->pf_fwd = (float)atof(v);
  if (const char* v = getenv("MLSTM_PF_BWD")) c->pf_bwd = (float)atof(v);
  if (const char* v = getenv("MLSTM_PF_STASH")) c->pf_stash = v[0] != '0';
  if (const char* v = getenv("MLSTM_L2_WH")) c->l2_wh = (float)atof(v);
  if (const char* v = getenv("MLSTM_AR_OVERLAP")) c->ar_overlap = v[0] != '0';
  if (const char* v = getenv("MLSTM_ASYNC_EPI")) c->async_epi = atoi(v);
  if (const char* v = getenv("MLSTM_WGRAD512")) c->wgrad512 = v[0] != '0';
  if (const char* v = getenv("MLSTM_RASTER_GROUP")) c->raster_group = v[0] != '0';
  if (const char* v = getenv("MLSTM_WGRAD_SIDE")) {
    int a = 0, b = 32, d = 10, q = 1;
    sscanf(v, "%d,%d,%d,%d", &a, &b, &d, &q);
    c->side_pol = q;
    c->side_chunks = std::max(0, std::min(16, a));
    c->side_ch = std::max(1, b);
    c->side_pairs = std::max(1, std::min(74, d));
  }
  if (const char* v = getenv("MLSTM_RECUR")) c->recur_env = atoi(v);
  if (const char* v = getenv("MLSTM_RC_EXP")) c->rc_exp = atoi(v);
  if (const char* v = getenv("MLSTM_RC_WKM")) c->rc_wkm = atoi(v) != 0;
  if (const char* v = getenv("MLSTM_RC_ROTATE")) c->rc_rotate = atoi(v) != 0;
  if (const char* v = getenv("MLSTM_RC_PF")) c->rc_pf_dist = std::max(0, atoi(v));
  if (const char* v = getenv("MLSTM_RC_FLAG_LANES")) c->rc_flag_lanes = std::max(1, std::min(32, atoi(v)));
  {
    const char* v = getenv("MLSTM_FORCE_PLAN");
    const std::string fp = v ? v : "";
    c->force_plan = fp == "pair" ? 1 : fp == "split" ? 2 : fp == "single" ? 3 : fp == "persist" ? 4 : 0;
    const char* pp = getenv("MLSTM_PERSIST_PAIRS");
    g_max_pairs = pp ? std::max(1, atoi(pp)) : 74;
  }
  const char* dbg = getenv("MLSTM_DEBUG_SIMT_GEMM");  // test instrument: mixed mode on the SIMT engine
  c->tc = c->mixed && !(dbg && dbg[0] == '1');
}

size_t layout_bytes(mlstm_ctx* c) {
  Carver cv{nullptr};
  if (c->mixed) {
    Net<__half> n{};
    carve(c, cv, n);
  } else {
    Net<float> n{};
    carve(c, cv, n);
  }
  return cv.off + 256;
}

// ------------------------------------------------------------------ launches
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool get_encoder() {
  if (g_encode) return true;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn)
    return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

const CUtensorMap* get_map(mlstm_ctx* c, const Opd& o, int box_rows) {
  if (o.mn) box_rows = -1;  // MN-major maps always use 64 x 64 boxes
  auto key = std::make_tuple(o.ptr, o.rows, o.K, o.ld, o.zdim, o.zstride, box_rows);
  auto it = c->maps.find(key);
  if (it != c->maps.end()) return &it->second;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)(o.mn ? o.rows : o.K), (cuuint64_t)(o.mn ? o.K : o.rows), (cuuint64_t)o.zdim};
  cuuint64_t strides[2] = {(cuuint64_t)o.ld * 2, (cuuint64_t)o.zstride * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)(o.mn ? 64 : box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, const_cast<void*>(o.ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    char buf[256];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d) rows=%ld K=%ld ld=%ld", (int)r, o.rows, o.K, o.ld);
    g_err = buf;
    return nullptr;
  }
  return &(c->maps[key] = m);
}

void count_launch(mlstm_ctx* c) {
  if (c->counting) {
    c->launches++;
    c->phase_launches[c->cur_phase]++;
  }
}

// Launches one tcgen05 GEMM kernel: cluster dims for the pair / split engines and, when enabled,
// programmatic dependent launch (the kernel waits on griddepcontrol before reading its inputs).
template <typename Kern, typename... Args>
cudaError_t launch_gemm(mlstm_ctx* c, Kern kern, dim3 grid, int smem, int cluster, Args... args) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[3];
  int na = 0;
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (c->pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (c->prio != 0) {  // graph nodes keep it (instantiated with cudaGraphInstantiateFlagUseNodePriority)
    at[na].id = cudaLaunchAttributePriority;
    at[na].val.priority = c->prio;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  e = cudaLaunchKernelEx(&cfg, kern, args...);
  count_launch(c);
  return e;
}

template <int BN, class Epi, int MN = 0>
cudaError_t launch_tc(mlstm_ctx* c, const CUtensorMap* ma, const CUtensorMap* mb, const CUtensorMap* ma2,
                      const CUtensorMap* mb2, Seg2 sg, int M, int N, int K, int az, int bz,
                      uint32_t pa, uint32_t pb, int flags, int splits, PrefetchJob pj,
                      const Epi& epi) {
  const int kb = (K + 63) / 64, kbps = (kb + splits - 1) / splits;
  return launch_gemm(c, gemm_tc_kernel<BN, Epi, MN>, dim3((N + BN - 1) / BN, (M + 127) / 128, splits), TcCfg<BN>::SMEM,
                     1, *ma, *mb, *ma2, *mb2, sg, M, N, K, az, bz, kbps, pa, pb, flags, pj, epi);
}

template <int S, class Epi, int MN = 0>
cudaError_t launch_tc1s(mlstm_ctx* c, const CUtensorMap* ma, const CUtensorMap* mb, const CUtensorMap* ma2,
                        const CUtensorMap* mb2, Seg2 sg, int M, int N, int K, int az,
                        int bz, uint32_t pa, uint32_t pb, int flags, PrefetchJob pj,
                        const Epi& epi) {
  const int kb = (K + 63) / 64, kbps = (kb + S - 1) / S;
  if ((long)S * ((N + 255) / 256) * ((M + 127) / 128) * 128 * 256 > kSplitScratchFloats)
    return cudaErrorInvalidConfiguration;  // the split-K partials would not fit the scratch
  return launch_gemm(c, gemm_tc1s_kernel<S, Epi, MN>, dim3(S * ((N + 255) / 256), (M + 127) / 128, 1), TcCfg<256>::SMEM,
                     S, *ma, *mb, *ma2, *mb2, sg, M, N, K, az, bz, kbps, pa, pb, flags, pj, c->split_scratch, epi);
}

template <int BN, class Epi, int MN = 0>
cudaError_t launch_tc2(mlstm_ctx* c, const CUtensorMap* ma, const CUtensorMap* mb, const CUtensorMap* ma2,
                       const CUtensorMap* mb2, Seg2 sg, int M, int N, int K, int az,
                       int bz, uint32_t pa, uint32_t pb, int flags, int splits, PrefetchJob pj,
                       const Epi& epi) {
  const int kb = (K + 63) / 64, kbps = (kb + splits - 1) / splits;
  return launch_gemm(c, gemm_tc2_kernel<BN, Epi, MN>, dim3(2 * ((N + BN - 1) / BN), (M + 255) / 256, splits),
                     Tc2Cfg<BN>::SMEM, 2, *ma, *mb, *ma2, *mb2, sg, M, N, K, az, bz, kbps, pa, pb, flags, pj, epi);
}

template <int BN, class Epi, int MN = 0>
cudaError_t launch_tc2p(mlstm_ctx* c, const CUtensorMap* ma, const CUtensorMap* mb, const CUtensorMap* ma2,
                        const CUtensorMap* mb2, Seg2 sg, int M, int N, int K, int az, int bz, uint32_t pa,
                        uint32_t pb, int flags, PrefetchJob pj, const Epi& epi) {
  const int tiles = ((M + 255) / 256) * ((N + BN - 1) / BN);
  const int npairs = std::min(tiles, c->tc2p_pairs > 0 ? c->tc2p_pairs : g_max_pairs);
  return launch_gemm(c, gemm_tc2p_kernel<BN, Epi, MN>, dim3(2 * npairs, 1, 1), Tc2Cfg<BN>::SMEM, 2, *ma, *mb, *ma2,
                     *mb2, sg, M, N, K, az, bz, 0, pa, pb, flags, pj, epi);
}

// Engine dispatch for one plan (MN: 0 both operands K-major, 1 both MN-major, 2 K-major A with
// MN-major B; MN-major B needs at least 64 B rows per CTA, so pair tiles of BN = 64 are refused).
template <int MN, class Epi>
cudaError_t dispatch_tc(mlstm_ctx* c, const Plan& p, const CUtensorMap* ma, const CUtensorMap* mb,
                        const CUtensorMap* ma2, const CUtensorMap* mb2, Seg2 sg, int M, int N, int K, int az, int bz,
                        uint32_t pa, uint32_t pb, int gflags, PrefetchJob pj, const Epi& epi) {
  if (p.cluster)
    return p.splits == 2 ? launch_tc1s<2, Epi, MN>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, pj, epi)
                         : launch_tc1s<4, Epi, MN>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, pj, epi);
  if (p.pair && p.persist && p.splits == 1)
    return launch_tc2p<256, Epi, MN>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, pj, epi);
  if constexpr (kMNEpi<Epi>) {
    if (p.pair && p.bn == 512)
      return launch_tc2<512, Epi, MN>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, p.splits, pj, epi);
  }
  if (p.pair) {
    if (MN == 1 || p.bn == 256)
      return launch_tc2<256, Epi, MN>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, p.splits, pj, epi);
    if constexpr (MN != 1) {
      if (p.bn == 128)
        return launch_tc2<128, Epi, MN>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, p.splits, pj, epi);
      if constexpr (MN == 0)
        return launch_tc2<64, Epi>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, p.splits, pj, epi);
      return cudaErrorInvalidValue;
    }
  }
  switch (p.bn) {
    case 256: return launch_tc<256, Epi, MN>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, p.splits, pj, epi);
    case 128: return launch_tc<128, Epi, MN>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, p.splits, pj, epi);
    default: return launch_tc<64, Epi, MN>(c, ma, mb, ma2, mb2, sg, M, N, K, az, bz, pa, pb, gflags, p.splits, pj, epi);
  }
}

// Whether the plan p can read an MN-major B operand (dispatch_tc<2>).
inline bool bmn_plan_ok(const Plan& p) { return !(p.pair && !p.cluster && !(p.persist && p.splits == 1) && p.bn < 128); }

// D[M x N] = A[az] . B[bz]^T, fused epilogue.  `splits` > 1 only with a partial epilogue.
// Optional L2 prefetch of the next GEMM's weight operand (see l2_prefetch in gemm.cuh).
struct Prefetch {
  PrefetchJob job{{nullptr, nullptr, nullptr, nullptr}, {0, 0, 0, 0}};
  int n = 0;
  void add(const void* p, long bytes) {
    if (n < 4 && bytes > 0) {
      job.base[n] = static_cast<const uint8_t*>(p);
      job.bytes[n] = bytes / 16 * 16;
      ++n;
    }
  }
};

// Optional second K segment (A2[az2] . B2^T added into the same accumulator; tcgen05 engines only).
struct Segment {
  const Opd* A2 = nullptr;
  int az2 = 0;
  const Opd* B2 = nullptr;
  int K2 = 0;
};

template <typename S, class Epi>
mlstm_status gemm(mlstm_ctx* c, const Opd& A, int az, const Opd& B, int bz, int M, int N, int K, Plan p,
                  const Epi& epi, const Prefetch& pf = Prefetch{}, const Segment& seg = Segment{}) {
  if constexpr (std::is_same<S, __half>::value) {
    if (c->tc) {
    const CUtensorMap* ma = get_map(c, A, 128);
    const int bbox = p.pair ? (p.bn == 512 ? 128 : p.bn / 2) : p.bn;  // B rows per TMA box (K-major)
    const CUtensorMap* mb = get_map(c, B, bbox);
    if (!ma || !mb) {
      c->failed = MLSTM_ECUDA;
      return MLSTM_ECUDA;
    }
    cudaError_t e;
    const int gflags = B.weight ? (kGemmStaticB | kGemmRasterM) : (A.mn && c->raster_group ? kGemmRasterG : 0);
    const PrefetchJob pj = pf.job;
    const CUtensorMap* ma2 = seg.A2 ? get_map(c, *seg.A2, 128) : ma;
    const CUtensorMap* mb2 = seg.B2 ? get_map(c, *seg.B2, bbox) : mb;
    if (!ma2 || !mb2) {
      c->failed = MLSTM_ECUDA;
      return MLSTM_ECUDA;
    }
    const Seg2 sg{seg.A2 ? (K + 63) / 64 : (1 << 30), seg.az2, 0};
    const int Kt = seg.A2 ? ((K + 63) / 64) * 64 + seg.K2 : K;  // the kernels' K runs over both segments
    if ((A.mn && !B.mn) || (A.mn && seg.A2) || (seg.B2 && seg.B2->mn != B.mn))
      return fail(MLSTM_EINVAL, "gemm: unsupported operand majors / MN segment");
    if constexpr (kMNEpi<Epi>) {
      if (A.mn) {
        if (p.pair && p.bn < 128) return fail(MLSTM_EINVAL, "gemm: MN-major pair tiles need BN >= 128");
        e = dispatch_tc<1>(c, p, ma, mb, ma2, mb2, sg, M, N, Kt, az, bz, A.pol, B.pol, gflags, pj, epi);
      } else {
        e = dispatch_tc<0>(c, p, ma, mb, ma2, mb2, sg, M, N, Kt, az, bz, A.pol, B.pol, gflags, pj, epi);
      }
    } else if constexpr (kBMNEpi<Epi>) {
      if (A.mn) return fail(MLSTM_EINVAL, "gemm: MN-major A only for weight-gradient epilogues");
      if (B.mn && !bmn_plan_ok(p)) return fail(MLSTM_EINVAL, "gemm: MN-major B needs pair tiles of BN >= 128");
      e = B.mn ? dispatch_tc<2>(c, p, ma, mb, ma2, mb2, sg, M, N, Kt, az, bz, A.pol, B.pol, gflags, pj, epi)
               : dispatch_tc<0>(c, p, ma, mb, ma2, mb2, sg, M, N, Kt, az, bz, A.pol, B.pol, gflags, pj, epi);
    } else {
      if (A.mn || B.mn) return fail(MLSTM_EINVAL, "gemm: MN-major operands only for weight-gradient / BPTT epilogues");
      e = dispatch_tc<0>(c, p, ma, mb, ma2, mb2, sg, M, N, Kt, az, bz, A.pol, B.pol, gflags, pj, epi);
    }
    CUDA_OR_FAIL(c, e);
    return MLSTM_OK;
    }
  }
  const S* a = static_cast<const S*>(A.ptr) + (long)az * A.zstride;
  const S* b = static_cast<const S*>(B.ptr) + (long)bz * B.zstride;
  const int kps = (int)rup((K + p.splits - 1) / p.splits, 32);
  dim3 grid((N + 63) / 64, (M + 127) / 128, p.splits);
  gemm_simt_kernel<S, Epi><<<grid, 128, 0, c->stream>>>(a, A.ld, b, B.ld, M, N, K, kps, A.mn ? 1 : 0, epi);
  count_launch(c);
  CUDA_OR_FAIL(c, cudaGetLastError());
  return MLSTM_OK;
}

#define RET_IF(x)                         \
  do {                                    \
    mlstm_status s_ = (x);                \
    if (s_ != MLSTM_OK) return s_;        \
  } while (0)

#define LAUNCH(c, ...)                        \
  do {                                        \
    __VA_ARGS__;                              \
    count_launch(c);                          \
    CUDA_OR_FAIL(c, cudaGetLastError());      \
  } while (0)

void phase(mlstm_ctx* c, int ph) {
  c->cur_phase = ph;
  // External: inside stream capture this becomes an event-record node that fires when the graph
  // runs (a plain record would only be an intra-graph dependency marker).
  if (c->profile) cudaEventRecordWithFlags(c->ev[ph], c->stream, cudaEventRecordExternal);
}

template <typename S>
Net<S>& net(mlstm_ctx* c);
template <>
Net<__half>& net<__half>(mlstm_ctx* c) {
  return c->nh;
}
template <>
Net<float>& net<float>(mlstm_ctx* c) {
  return c->nf;
}

// ------------------------------------------------------------------ persistent recurrence
cudaLaunchConfig_t recur_cfg(mlstm_ctx* c, cudaLaunchAttribute* at, bool coop) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c->h / 32, 1, 1);  // h/64 CTA pairs
  cfg.blockDim = dim3(kRcThreads);
  cfg.dynamicSmemBytes = kRcSmem;
  cfg.stream = c->stream;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = coop ? 2 : 1;
  return cfg;
}

// Whether this ctx runs the recurrence on the persistent dataflow kernels (recur.cuh): the shape
// predicate plus co-residency of all h/64 CTA pairs, decided once.
bool recur_on(mlstm_ctx* c) {
  if (c->recur_ok >= 0) return c->recur_ok != 0;
  c->recur_ok = 0;
  if (!recur_shape_ok(c) || !c->rc_scratch) return false;
  for (const void* kern : {(const void*)fwd_recur_kernel, (const void*)bwd_recur_kernel<false>,
                           (const void*)bwd_recur_kernel<true>}) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kRcSmem) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    cudaLaunchAttribute at[2];
    cudaLaunchConfig_t cfg = recur_cfg(c, at, false);
    cfg.gridDim = dim3(2, 1, 1);
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess || mc < c->h / 64) {
      cudaGetLastError();
      if (getenv("MLSTM_RECUR_DEBUG")) fprintf(stderr, "recur off: max active clusters %d < %d\n", mc, c->h / 64);
      return false;
    }
  }
  c->recur_ok = 1;
  return true;
}

RcPolicy recur_policy(mlstm_ctx* c) {
  // the per-timestep activation chunks are re-read by every pair within microseconds (normal); the
  // split GEMM's weight (W_mh, 2h^2 bytes) and the segment operands (XZT / W_dec) are re-read every
  // timestep (evict_last); W_h (8h^2 bytes, more than L2) streams (evict_first unless MLSTM_L2_WH)
  const uint32_t wide = c->l2_wh > 0 ? pol_last(c->l2_wh) : kPolFirst;
  return RcPolicy{0u, pol_last(1.f), wide, pol_last(1.f), c->rc_flag_lanes, c->rc_pf_dist, c->rc_rotate, c->rc_exp};
}

mlstm_status launch_fwd_recur(mlstm_ctx* c) {
  Net<__half>& n = c->nh;
  const int h = c->h, B = c->B, T = c->T;
  const Opd H{n.Hrm, B, h, h, T + 1, (long)B * h};
  const Opd M{n.Mrm, B, h, h, T, (long)B * h};
  const Opd OH{n.OHR, B, 256, 256, T, (long)B * 256};
  const Opd Wmh{n.Wmh_w, h, h, h, 1, (long)h * h};
  const Opd Wh{n.Wh_w, 4L * h, h, h, 1, 4L * h * h};
  const Opd XZ{n.XZT, 4L * h, 256, 256, 1, 4L * h * 256};
  const CUtensorMap *mH = get_map(c, H, 128), *mM = get_map(c, M, 128), *mO = get_map(c, OH, 128),
                    *mW1 = get_map(c, Wmh, 128), *mW2 = get_map(c, Wh, 128), *mX = get_map(c, XZ, 128);
  if (!mH || !mM || !mO || !mW1 || !mW2 || !mX) {
    c->failed = MLSTM_ECUDA;
    return MLSTM_ECUDA;
  }
  CUDA_OR_FAIL(c, cudaMemsetAsync(c->rc_flags, 0, sizeof(uint32_t) * kRcFlagWords(h / 64), c->stream));
  cudaLaunchAttribute at[2];
  cudaLaunchConfig_t cfg = recur_cfg(c, at, true);
  CUDA_OR_FAIL(c, cudaLaunchKernelEx(&cfg, fwd_recur_kernel, *mH, *mM, *mO, *mW1, *mW2, *mX, n, c->rc_scratch,
                                     c->rc_flags, recur_policy(c)));
  count_launch(c);
  return MLSTM_OK;
}

mlstm_status launch_bwd_recur(mlstm_ctx* c) {
  Net<__half>& n = c->nh;
  const int h = c->h, B = c->B, T = c->T;
  const Opd dZ{n.G5 + h, B, 4L * h, 5L * h, T, 5L * B * h};
  const Opd dA{n.dA, B, h, h, T, (long)B * h};
  const Opd dY{n.dY, B, 256, 256, T, (long)B * 256};
  const CUtensorMap *mZ = get_map(c, dZ, 128), *mA = get_map(c, dA, 128), *mY = get_map(c, dY, 128);
  const CUtensorMap *mW2, *mW1, *mD;
  if (c->rc_wkm) {  // K-major from the transposed working copies (element (unit n, k) at n * K + k)
    mW2 = get_map(c, Opd{n.WhT, h, 4L * h, 4L * h, 1, 4L * h * h}, 128);
    mW1 = get_map(c, Opd{n.WmhT, h, h, h, 1, (long)h * h}, 128);
    mD = get_map(c, Opd{n.WdecT, h, 256, 256, 1, 256L * h}, 128);
  } else {  // MN-major straight from the row-major working copies: element (unit n, k) at k*h + n
    mW2 = get_map(c, Opd{n.Wh_w, h, 4L * h, h, 1, 4L * h * h, 0, true, true}, 64);
    mW1 = get_map(c, Opd{n.Wmh_w, h, h, h, 1, (long)h * h, 0, true, true}, 64);
    mD = get_map(c, Opd{n.Wdec_w, h, 256, h, 1, 256L * h, 0, true, true}, 64);
  }
  if (!mZ || !mA || !mY || !mW2 || !mW1 || !mD) {
    c->failed = MLSTM_ECUDA;
    return MLSTM_ECUDA;
  }
  CUDA_OR_FAIL(c, cudaMemsetAsync(c->rc_flags, 0, sizeof(uint32_t) * kRcFlagWords(h / 64), c->stream));
  cudaLaunchAttribute at[2];
  cudaLaunchConfig_t cfg = recur_cfg(c, at, true);
  if (c->rc_wkm)
    CUDA_OR_FAIL(c, cudaLaunchKernelEx(&cfg, bwd_recur_kernel<true>, *mZ, *mA, *mY, *mW2, *mW1, *mD, n, c->rc_scratch,
                                       c->rc_flags, recur_policy(c)));
  else
    CUDA_OR_FAIL(c, cudaLaunchKernelEx(&cfg, bwd_recur_kernel<false>, *mZ, *mA, *mY, *mW2, *mW1, *mD, n, c->rc_scratch,
                                       c->rc_flags, recur_policy(c)));
  count_launch(c);
  return MLSTM_OK;
}

// Recomputes the transposed working copies from the row-major ones.
template <typename S>
mlstm_status enqueue_transposes(mlstm_ctx* c) {
  Net<S>& n = net<S>(c);
  const int h = c->h;
  dim3 blk(32, 8);
  if constexpr (std::is_same<S, __half>::value) {  // h is a multiple of 64
    // the backward reads W_h, W_mh, W_dec MN-major (persistent kernel, or per-timestep plans that allow it)
    if (!c->bwd_needs_transposes && !(recur_on(c) && c->rc_wkm)) return MLSTM_OK;
    LAUNCH(c, (transpose64_kernel<<<dim3(h / 64, h / 64), blk, 0, c->stream>>>(n.Wmh_w, n.WmhT, h, h)));
    LAUNCH(c, (transpose64_kernel<<<dim3(h / 64, 4 * h / 64), blk, 0, c->stream>>>(n.Wh_w, n.WhT, 4 * h, h)));
    LAUNCH(c, (transpose64_kernel<<<dim3(h / 64, 256 / 64), blk, 0, c->stream>>>(n.Wdec_w, n.WdecT, 256, h)));
    return MLSTM_OK;
  }
  LAUNCH(c, (transpose_kernel<S><<<dim3((h + 31) / 32, (h + 31) / 32), blk, 0, c->stream>>>(n.Wmh_w, n.WmhT, h, h)));
  LAUNCH(c, (transpose_kernel<S><<<dim3((h + 31) / 32, (4 * h + 31) / 32), blk, 0, c->stream>>>(n.Wh_w, n.WhT, 4 * h, h)));
  LAUNCH(c, (transpose_kernel<S><<<dim3((h + 31) / 32, 256 / 32), blk, 0, c->stream>>>(n.Wdec_w, n.WdecT, 256, h)));
  return MLSTM_OK;
}

template <typename S>
mlstm_status enqueue_cast(mlstm_ctx* c) {
  Net<S>& n = net<S>(c);
  LAUNCH(c, (cast_working_kernel<S><<<grid_for(c->P), 256, 0, c->stream>>>(n)));
  if (c->po.wn) LAUNCH(c, (wn_norm_kernel<S><<<grid_for(10L * c->h * 32), 256, 0, c->stream>>>(n)));
  return enqueue_transposes<S>(c);
}

// Input projection table + forward recurrence over T steps (+ decoder logits).
template <typename S>
mlstm_status enqueue_forward(mlstm_ctx* c, int slot) {
  Net<S>& n = net<S>(c);
  const int h = c->h, e = c->e, B = c->B, T = c->T;
  phase(c, PH_PREP);
  LAUNCH(c, (state_in_kernel<S><<<grid_for((long)B * h), 256, 0, c->stream>>>(n, slot)));
  const bool fold = n.XZT != nullptr;  // tcgen05 path: W_x x + b enters F2 as a second K segment
  if (fold) LAUNCH(c, (onehot_kernel<S><<<grid_for((long)T * B), 256, 0, c->stream>>>(n)));
  phase(c, PH_TAB);
  {
    Opd A{n.E_w, 256, e, e, 1, 256L * e};
    Opd Bo{n.Wcat_w, 5L * h, e, e, 1, 5L * h * e, 0, true};
    RET_IF(gemm<S>(c, A, 0, Bo, 0, 256, 5 * h, e, plan_gemm(c->tc, 256, 5 * h, e, false), EpiTab<S>{n}));
  }
  phase(c, PH_FWD);
  // L2 policy: the recurrent weights are re-read every timestep -- keep W_mh and a fraction of
  // W_h resident (evict_last); the activations are read once (evict_first).
  const Opd Hprev{n.Hrm, B, h, h, T + 1, (long)B * h, kPolFirst};
  const Opd Wmh{n.Wmh_w, h, h, h, 1, (long)h * h, pol_last(c->l2_wmh), true};
  const Opd Mt{n.Mrm, B, h, h, T, (long)B * h, kPolFirst};  // m_t = slot t
  const Opd Wh{n.Wh_w, 4L * h, h, h, 1, 4L * h * h, pol_last(c->l2_wh), true};
  const Plan p1 = plan_gemm(c->tc, B, h, h, false), p2 = plan_gemm(c->tc, B, 4 * h, h + 256, false);
  // tcgen05 path: W_x x_t + b enters F2's accumulator as a second K segment, one-hot(bytes_t) x
  // (W_x E + b)^T (exact selection of one table row; the table is rounded to fp16)
  const Opd OH{n.OHR, B, 256, 256, T, (long)B * 256, kPolFirst};
  const Opd XZ{n.XZT, 4L * h, 256, 256, 1, 4L * h * 256, 0, true};
  Segment seg2;
  if (fold) {
    seg2.A2 = &OH;
    seg2.B2 = &XZ;
    seg2.K2 = 256;
  }
  // F1 (light on HBM) prefetches into L2 the first k-blocks of every W_h tile F2 will stream
  Prefetch pf1;
  if (c->pf_fwd > 0 && c->tc) pf1.add(n.Wh_w, (long)(c->pf_fwd * 8.0 * h * h));
  bool rc = false;
  if constexpr (std::is_same<S, __half>::value) rc = recur_on(c);
  if (rc) RET_IF(launch_fwd_recur(c));
  for (int t = 0; t < (rc ? 0 : T); ++t) {
    if (fold && c->async_epi)
      RET_IF(gemm<S>(c, Hprev, t, Wmh, 0, B, h, h, p1, EpiF1IO<S>{{n, t}}, pf1));
    else
      RET_IF(gemm<S>(c, Hprev, t, Wmh, 0, B, h, h, p1, EpiF1<S>{n, t}, pf1));
    seg2.az2 = t;
    if (fold && c->async_epi)  // tcgen05 path (W_x x + b folded): async row I/O epilogue
      RET_IF(gemm<S>(c, Mt, t, Wh, 0, B, 4 * h, h, p2, EpiF2IO<S>{{n, t, 1}, c->async_epi}, Prefetch{}, seg2));
    else
      RET_IF(gemm<S>(c, Mt, t, Wh, 0, B, 4 * h, h, p2, EpiF2<S>{n, t, fold ? 1 : 0}, Prefetch{}, seg2));
  }
  phase(c, PH_DEC);
  {
    Opd A{n.Hrm + (long)B * h, (long)T * B, h, h, 1, (long)T * B * h};
    Opd Bo{n.Wdec_w, 256, h, h, 1, 256L * h, 0, true};
    RET_IF(gemm<S>(c, A, 0, Bo, 0, T * B, 256, h, plan_gemm(c->tc, (long)T * B, 256, h, false), EpiY<S>{n}));
  }
  return MLSTM_OK;
}

template <typename S>
mlstm_status enqueue_train_a(mlstm_ctx* c) {
  Net<S>& n = net<S>(c);
  const int h = c->h, B = c->B, T = c->T;
  const long Kt = c->Kt;
  RET_IF(enqueue_forward<S>(c, MLSTM_SLOT_TRAIN));
  // the one-hot and the dC reset belong to the prep phase logically; they run here, off the
  // forward's critical path
  if (!n.XZT) LAUNCH(c, (onehot_kernel<S><<<grid_for((long)T * B), 256, 0, c->stream>>>(n)));
  CUDA_OR_FAIL(c, cudaMemsetAsync(n.dC, 0, sizeof(float) * (size_t)B * h, c->stream));
  phase(c, PH_CE);
  const double denom = (double)c->Bfull * c->world * T;  // B_g * T (Q7): all rows of all ranks
  LAUNCH(c, (ce_kernel<S><<<c->nblk_ce, 256, 0, c->stream>>>(n, B, (float)(1.0 / denom), 1)));
  LAUNCH(c, (ce_reduce_kernel<S><<<1 + 256, 256, 0, c->stream>>>(n, c->nblk_ce, 1)));
  phase(c, PH_DHDEC);
  const Opd dYs{n.dY, B, 256, 256, T, (long)B * 256, kPolFirst};  // dY_s = rows of timestep s
  const Opd WdecT{n.WdecT, h, 256, 256, 1, 256L * h, 0, true};
  if (n.dHdec) {  // SIMT path: dH_dec for all timesteps in one GEMM
    Opd A{n.dY, (long)T * B, 256, 256, 1, (long)T * B * 256};
    RET_IF(gemm<S>(c, A, 0, WdecT, 0, T * B, h, 256, plan_gemm(c->tc, (long)T * B, h, 256, false), EpiDHdec<S>{n}));
  }
  // dW_dec = dY^T H needs only the forward and the CE: it runs before BPTT, and with several ranks its
  // allreduce bucket (W_dec, b_dec: SURVEY 8(e) "bucket 0") overlaps the backward
  struct W {
    Opd A, B;
    long M, N, off;
    int mode;
  };
  // every operand MN-major: the row-major [T*B][cols] stashes the recurrence wrote, K = (t, b)
  auto mn = [&](const void* p, long cols, long ld) { return Opd{p, cols, Kt, ld, 1, 0, 0, false, true}; };
  const W ws[4] = {
      {mn(n.G5 + h, 4L * h, 5L * h), mn(n.Mrm, h, h), 4L * h, h, c->po.Wh, 1},      // dW_h = dZ^T M
      {mn(n.dA, h, h), mn(n.Hrm, h, h), h, h, c->po.Wmh, 0},                         // dW_mh = dA^T H_{t-1}
      {mn(n.dY, 256, 256), mn(n.Hrm + (long)B * h, h, h), 256, h, c->po.Wdec, 0},    // dW_dec = dY^T H
      {mn(n.OHR, 256, 256), mn(n.G5, 5L * h, 5L * h), 256, 5L * h, 0, 2},          // S = onehot^T [dMX|dZ]
  };
  // dW_h side chunks (MLSTM_WGRAD_SIDE): chunk j = timesteps [T - (j+1) ch, T - j ch), reduced on the side
  // stream as soon as the backward has produced its dZ rows; dW_h's main GEMM then covers K = [0, Kmain)
  // and adds the side partial in its epilogue
  int nside = 0;
  if constexpr (std::is_same<S, __half>::value) {
    const int ch = c->side_ch;
    if (c->side_chunks > 0 && c->tc && !n.dHdec && !(recur_on(c) && !c->recur_fwd_only) && h % 256 == 0)
      nside = std::max(0, std::min(c->side_chunks, (T - 1) / ch));
    const Plan pm = plan_gemm(c->tc, 4L * h, h, (long)(T - nside * ch) * B, true);
    if (!(pm.splits == 1 || pm.pair || pm.cluster)) nside = 0;  // the split-K finaliser has no partial input
  }
  const long Kmain = (long)(T - nside * c->side_ch) * B;
  // one weight-gradient job (plan, optional dW_h row halves, split-K finaliser, bucket event)
  auto run_w = [&](int wi) -> mlstm_status {
    W w = ws[wi];
    const long Kw = (wi == 0) ? Kmain : Kt;
    const float* acc = (wi == 0 && nside > 0) ? c->wpart : nullptr;
    if (wi == 0) {
      w.A.K = Kw;
      w.B.K = Kw;
    }
    Plan p = plan_gemm(c->tc, w.M, w.N, Kw, true);
    if (c->wgrad512 && p.pair && w.N % 512 == 0) {  // 256 x 512 pair tiles (MLSTM_WGRAD512)
      p.bn = 512;
      p.persist = false;
    }
    if (wi == 0 && c->overlap_now() && p.pair && p.splits == 1) {
      // dW_h in two row halves: the first half's allreduce starts while the second computes
      // (internal rows [0, 2h) are units [0, h/2) of every gate: 4 contiguous canonical ranges)
      for (int half = 0; half < 2; ++half) {
        Opd Ah = mn(n.G5 + h + (long)half * 2 * h, 2L * h, 5L * h);
        Ah.K = Kw;
        RET_IF(gemm<S>(c, Ah, 0, w.B, 0, 2 * h, (int)w.N, (int)Kw, p,
                       EpiWgrad<S>{n, w.off, w.mode, (int)w.N, half * 2 * h, acc}));
        if (half == 0) CUDA_OR_FAIL(c, cudaEventRecordWithFlags(c->ev_wh_a, c->stream, cudaEventRecordExternal));
      }
    } else if (p.splits == 1 || p.pair || p.cluster) {
      RET_IF(gemm<S>(c, w.A, 0, w.B, 0, (int)w.M, (int)w.N, (int)Kw, p,
                     EpiWgrad<S>{n, w.off, w.mode, (int)w.N, 0, acc}));
    } else {
      if (acc) return fail(MLSTM_EINVAL, "wgrad side chunks need a single-pass dW_h plan");
      RET_IF(gemm<S>(c, w.A, 0, w.B, 0, (int)w.M, (int)w.N, (int)Kt, p, EpiPartial{n.part, w.N, w.M * w.N}));
      LAUNCH(c, (wgrad_finalize_kernel<S><<<grid_for(w.M * w.N), 256, 0, c->stream>>>(n, n.part, p.splits, (int)w.M,
                                                                                        (int)w.N, w.off, w.mode)));
    }
    // bucket boundaries of the overlapped allreduce (external event nodes in the graph)
    if (c->overlap_now() && wi < 3)
      CUDA_OR_FAIL(c, cudaEventRecordWithFlags(wi == 0 ? c->ev_wh : (wi == 1 ? c->ev_wmh : c->ev_wdec), c->stream,
                                               cudaEventRecordExternal));
    return MLSTM_OK;
  };
  RET_IF(run_w(2));
  // side chunk j of dW_h: fork from the capture stream once its dZ rows exist, run on side_pairs pairs
  // at the lowest priority (the recurrence's GEMMs carry the highest)
  auto enqueue_side = [&](int j) -> mlstm_status {
    const long lo = (long)T - (long)(j + 1) * c->side_ch, Kc = (long)c->side_ch * B;
    CUDA_OR_FAIL(c, cudaEventRecord(c->side_ev[j], c->stream));
    CUDA_OR_FAIL(c, cudaStreamWaitEvent(c->side, c->side_ev[j], 0));
    const uint32_t pol = c->side_pol ? kPolFirst : 0;  // keep the recurrence's L2-resident weights
    const Opd A{n.G5 + h + lo * B * 5L * h, 4L * h, Kc, 5L * h, 1, 0, pol, false, true};
    const Opd Bm{n.Mrm + lo * B * (long)h, h, Kc, h, 1, 0, pol, false, true};
    cudaStream_t keep = c->stream;
    const bool pdl = c->pdl;
    const int prio = c->prio;
    c->stream = c->side;
    c->pdl = false;
    c->prio = 0;
    c->tc2p_pairs = c->side_pairs;
    const mlstm_status r =
        gemm<S>(c, A, 0, Bm, 0, 4 * h, h, (int)Kc, Plan{256, 1, true, false, true}, EpiWacc{c->wpart, h, j == 0});
    c->stream = keep;
    c->pdl = pdl;
    c->prio = prio;
    c->tc2p_pairs = 0;
    return r;
  };
  if (nside > 0) c->prio = c->prio_hi;
  phase(c, PH_BWD);
  bool rc = false;
  if constexpr (std::is_same<S, __half>::value) rc = recur_on(c) && !c->recur_fwd_only;
  const Plan p1 = plan_gemm(c->tc, B, h, 4 * h, false), p2 = plan_gemm(c->tc, B, h, h, false);
  const Plan p0 = plan_gemm(c->tc, B, h, 256, false);
  // the per-timestep backward reads W_h, W_mh, W_dec MN-major straight from the row-major working
  // copies (no transposed copies) whenever its tile plans allow it (tensor-core path)
  const bool bmn = c->tc && !rc && !n.dHdec && bmn_plan_ok(p0) && bmn_plan_ok(p1) && bmn_plan_ok(p2);
  c->bwd_needs_transposes = !rc && !bmn;
  const Opd WdecB = bmn ? Opd{n.Wdec_w, h, 256, h, 1, 256L * h, 0, true, true} : WdecT;
  if (rc) {
    RET_IF(launch_bwd_recur(c));
  } else if (n.dHdec) {
    LAUNCH(c, (gate_bwd_last_kernel<S><<<grid_for((long)B * h / 16), 256, 0, c->stream>>>(n)));
  } else {  // gate backward of the last timestep: dH = dY_{T-1} W_dec only (TBTT: no recurrent term)
    RET_IF(gemm<S>(c, dYs, T - 1, WdecB, 0, B, h, 256, p0, EpiB2<S>{n, T - 1}));
  }
  Segment segd;  // B2's second K segment: + dY_{t-1} W_dec
  if (!n.dHdec && !rc) {
    segd.A2 = &dYs;
    segd.B2 = &WdecB;
    segd.K2 = 256;
  }
  {
    const Opd dZ{n.G5 + h, B, 4L * h, 5L * h, T, 5L * B * h, kPolFirst};  // dZ_t = slot t, cols [h, 5h)
    const Opd WhT = bmn ? Opd{n.Wh_w, h, 4L * h, h, 1, 4L * h * h, pol_last(c->l2_wh), true, true}
                        : Opd{n.WhT, h, 4L * h, 4L * h, 1, 4L * h * h, pol_last(c->l2_wh), true};
    const Opd dA{n.dA, B, h, h, T, (long)B * h, kPolFirst};
    const Opd WmhT = bmn ? Opd{n.Wmh_w, h, h, h, 1, (long)h * h, pol_last(c->l2_wmh), true, true}
                         : Opd{n.WmhT, h, h, h, 1, (long)h * h, pol_last(c->l2_wmh), true};
    // B2 prefetches into L2 the first k-blocks (of each K split) of the W_h^T tiles B1 streams next
    const size_t es = sizeof(S);
    for (int t = rc ? -1 : T - 1; t >= 0; --t) {
      // B1(t) prefetches what B2's gate backward of step t-1 reads (written long ago by the
      // forward: gates, c_{t-1} and c_{t-2} (adjacent blocks), dH_dec); B2 prefetches the a-stash
      // block the next B1 reads.
      Prefetch pb1, pb2;
      if (c->pf_stash && c->tc && t > 0) {
        const long BH = (long)B * h;
        pb1.add(n.Gates + (long)(t - 1) * 4 * BH, 4 * BH * (long)es);
        pb1.add(n.Crm + (long)(t - 1) * BH, 2 * BH * 4L);
        if (n.dHdec) pb1.add(n.dHdec + (long)(t - 1) * BH, BH * 4L);
        pb2.add(n.Astash + (long)(t - 1) * BH, BH * (long)es);
      }
      if (c->pf_bwd > 0 && c->tc && !bmn) pb2.add(n.WhT, (long)(c->pf_bwd * 8.0 * h * h));
      if (c->tc && c->async_epi)
        RET_IF(gemm<S>(c, dZ, t, WhT, 0, B, h, 4 * h, p1, EpiB1IO<S>{{n, t}}, pb1));
      else
        RET_IF(gemm<S>(c, dZ, t, WhT, 0, B, h, 4 * h, p1, EpiB1<S>{n, t}, pb1));
      segd.az2 = t - 1;
      if (t > 0) RET_IF(gemm<S>(c, dA, t, WmhT, 0, B, h, h, p2, EpiB2<S>{n, t - 1}, pb2, segd));
      const int done = T - (t - 1);  // timesteps [t-1, T) have their dZ rows now
      if (nside > 0 && t > 0 && done % c->side_ch == 0 && done / c->side_ch <= nside)
        RET_IF(enqueue_side(done / c->side_ch - 1));
    }
  }
  c->prio = 0;
  phase(c, PH_WGRAD);
  {
    if (nside > 0) {  // join the side stream: dW_h's main GEMM adds its partial
      CUDA_OR_FAIL(c, cudaEventRecord(c->side_ev[16], c->side));
      CUDA_OR_FAIL(c, cudaStreamWaitEvent(c->stream, c->side_ev[16], 0));
    }
    for (int wi : {0, 1, 3}) RET_IF(run_w(wi));
    // dE = S [W_mx; W_x] (M=256, N=e, K=5h) and [dW_mx; dW_x] = S^T E (M=5h, N=e, K=256)
    {
      const int sp = c->seg_splits;
      const int kps = (int)rup((5L * h + sp - 1) / sp, 32);
      LAUNCH(c, (seg_gemm_kernel<S, 0><<<dim3((c->e + 63) / 64, 4, sp), 256, 0, c->stream>>>(n, n.part, 256, c->e,
                                                                                               5 * h, kps)));
      LAUNCH(c, (seg_finalize_kernel<S, 0><<<grid_for(256L * c->e), 256, 0, c->stream>>>(n, n.part, sp, 256, c->e)));
      LAUNCH(c, (seg_gemm_kernel<S, 1><<<dim3((c->e + 63) / 64, (5 * h + 63) / 64, 1), 256, 0, c->stream>>>(
                     n, n.part, 5 * h, c->e, 256, 256)));
      LAUNCH(c, (seg_finalize_kernel<S, 1><<<grid_for(5L * h * c->e), 256, 0, c->stream>>>(n, n.part, 1, 5 * h, c->e)));
    }
    LAUNCH(c, (db_kernel<S><<<grid_for(4L * h), 256, 0, c->stream>>>(n)));
    if (c->nmb > 1) LAUNCH(c, (grad_accum_kernel<S><<<grid_for(c->P), 256, 0, c->stream>>>(n)));
  }
  // persist this micro-batch's final (h, c) rows (TBTT state carry)
  LAUNCH(c, (state_out_kernel<S><<<grid_for((long)B * h), 256, 0, c->stream>>>(n, MLSTM_SLOT_TRAIN)));
  return MLSTM_OK;
}

template <typename S>
mlstm_status enqueue_train_b(mlstm_ctx* c) {
  Net<S>& n = net<S>(c);
  const mlstm_config& cf = c->cfg;
  phase(c, PH_OPT);
  if (c->po.wn) LAUNCH(c, (wn_grad_kernel<S><<<grid_for(10L * c->h * 32), 256, 0, c->stream>>>(n)));
  // overflow predicate: with one rank every writer of the gradient arena already flagged a
  // non-finite fp16 value; after a SUM allreduce finite values can still overflow, so the reduced
  // buffer (identical on every rank) is scanned
  if (c->world > 1)
    LAUNCH(c, (overflow_kernel<S><<<grid_for(c->P), 256, 0, c->stream>>>(n.arena, c->P, &c->st->overflow)));
  LAUNCH(c, (adam_kernel<S><<<grid_for(c->P), 256, 0, c->stream>>>(n, c->adam_m, c->adam_v, (float)cf.beta1,
                                                                   (float)cf.beta2, (float)cf.eps, cf.lr0,
                                                                   (long)cf.decay_iters)));
  if (c->po.wn) LAUNCH(c, (wn_norm_kernel<S><<<grid_for(10L * c->h * 32), 256, 0, c->stream>>>(n)));
  RET_IF(enqueue_transposes<S>(c));
  LAUNCH(c, (scaler_kernel<<<1, 1, 0, c->stream>>>(c->st, cf.scale_min, cf.scale_max, cf.scale_growth_interval,
                                                   cf.lr0, (long)cf.decay_iters)));
  return MLSTM_OK;
}

template <typename S>
mlstm_status record_graph(mlstm_ctx* c, mlstm_status (*fn)(mlstm_ctx*), cudaGraphExec_t* out) {
  cudaGraph_t g = nullptr;
  cudaStream_t user = c->stream;
  c->stream = c->cap;
  cudaError_t eb = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
  if (eb != cudaSuccess) {
    c->stream = user;
    CUDA_OR_FAIL(c, eb);
  }
  mlstm_status s = fn(c);
  cudaError_t e = cudaStreamEndCapture(c->stream, &g);
  c->stream = user;
  if (s != MLSTM_OK) {
    if (g) cudaGraphDestroy(g);
    return s;
  }
  CUDA_OR_FAIL(c, e);
  CUDA_OR_FAIL(c, cudaGraphInstantiate(out, g, c->side_chunks > 0 ? cudaGraphInstantiateFlagUseNodePriority : 0));
  cudaGraphDestroy(g);
  return MLSTM_OK;
}

template <typename S>
mlstm_status build_graphs(mlstm_ctx* c) {
  if (c->gA) cudaGraphExecDestroy(c->gA);
  if (c->gB) cudaGraphExecDestroy(c->gB);
  c->gA = c->gB = nullptr;
  g_force_plan = c->force_plan;
  c->counting = true;
  c->launches = 0;
  memset(c->phase_launches, 0, sizeof c->phase_launches);
  mlstm_status s = record_graph<S>(c, enqueue_train_a<S>, &c->gA);
  if (s == MLSTM_OK) s = record_graph<S>(c, enqueue_train_b<S>, &c->gB);
  c->counting = false;
  g_force_plan = 0;
  return s;
}

void accumulate_phases(mlstm_ctx* c, int from, int to) {
  float ms;
  for (int p = from; p < to; ++p)
    if (cudaEventElapsedTime(&ms, c->ev[p], c->ev[p + 1]) == cudaSuccess) c->phase_ms[p] += ms;
}

// Whether graph A splits dW_h into row halves (and records ev_wh_a): the same test the wgrad loop
// applies (overlapped allreduce, CTA-pair plan without split-K).
template <typename S>
bool wh_split_ok(mlstm_ctx* c) {
  if (!c->overlap_now() || !c->tc) return false;
  g_force_plan = c->force_plan;
  Plan p = plan_gemm(c->tc, 4L * c->h, c->h, c->Kt, true);
  g_force_plan = 0;
  return p.pair && p.splits == 1;
}

// The gradient allreduce's buckets as element ranges of the canonical fp16 arena,
// in the order they are reduced, each tagged with the event it waits for: kAfterWdec = dW_dec (run
// before BPTT; its bucket also carries b_dec, reduced by the CE), kAfterWhA = the first half of dW_h
// (internal rows [0, 2h) = units [0, h/2) of every gate: four contiguous canonical ranges), kAfterWh =
// dW_h, kAfterWmh = dW_mh, kAfterA = the end of graph A (E, W_mx, W_x, b: the per-byte sums and db;
// with weight norm the gain slots too).  Without overlap (world 1, micro-batches, or
// MLSTM_AR_OVERLAP=0): one range, the whole arena, after graph A.
enum { kAfterWdec = 0, kAfterWhA = 1, kAfterWh = 2, kAfterWmh = 3, kAfterA = 4 };
struct ArRange {
  int64_t off, count;
  int32_t after;
};
std::vector<ArRange> allreduce_plan(mlstm_ctx* c) {
  std::vector<ArRange> r;
  const ParamOffsets& po = c->po;
  if (!c->overlap_now()) {
    r.push_back({0, c->P, kAfterA});
    return r;
  }
  r.push_back({po.Wdec, po.bdec + 256 - po.Wdec, kAfterWdec});
  const long hh = c->h;
  if (wh_split_ok<__half>(c)) {
    for (int half = 0; half < 2; ++half)
      for (int g = 0; g < 4; ++g)
        r.push_back({po.Wh + ((long)g * hh + half * (hh / 2)) * hh, (hh / 2) * hh, half == 0 ? kAfterWhA : kAfterWh});
  } else {
    r.push_back({po.Wh, po.b - po.Wh, kAfterWh});
  }
  r.push_back({po.Wmh, po.Wx - po.Wmh, kAfterWmh});
  r.push_back({0, po.Wmh, kAfterA});
  r.push_back({po.Wx, po.Wh - po.Wx, kAfterA});
  r.push_back({po.b, po.Wdec - po.b, kAfterA});
  if (po.P > po.bdec + 256) r.push_back({po.bdec + 256, po.P - po.bdec - 256, kAfterA});
  return r;
}

// One step: for each micro-batch, copy its rows of the input (host or device) into the step
// buffers and run graph A (forward, BPTT, weight gradients, fp32 accumulation across micro-batches);
// then the allreduce and graph B (overflow check, scaler, Adam, cast) once.
template <typename S>
mlstm_status run_train(mlstm_ctx* c, const uint8_t* bytes, const uint8_t* reset, cudaMemcpyKind kind, int slot) {
  if (!c->gA) RET_IF(build_graphs<S>(c));
  Net<S>& n = net<S>(c);
  const size_t rowb = (size_t)(c->T + 1);
  for (int i = 0; i < c->nmb; ++i) {
    set_microbatch_kernel<<<1, 1, 0, c->stream>>>(c->st, i);
    CUDA_OR_FAIL(c, cudaGetLastError());
    CUDA_OR_FAIL(c, cudaMemcpyAsync(c->bytes, bytes + (size_t)i * c->B * rowb, (size_t)c->B * rowb, kind, c->stream));
    if (reset) CUDA_OR_FAIL(c, cudaMemcpyAsync(c->reset, reset + (size_t)i * c->B, c->B, kind, c->stream));
    else CUDA_OR_FAIL(c, cudaMemsetAsync(c->reset, 0, c->B, c->stream));
    CUDA_OR_FAIL(c, cudaGraphLaunch(c->gA, c->stream));
    if (c->profile) {
      CUDA_OR_FAIL(c, cudaEventRecord(c->ev[PH_ALLREDUCE], c->stream));
      if (i + 1 < c->nmb) {  // earlier micro-batches: fold their phase times in now
        CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
        accumulate_phases(c, PH_PREP, PH_ALLREDUCE);
      }
    }
  }
  if (c->world > 1) {
    c->cur_phase = PH_ALLREDUCE;
    const ncclDataType_t dt = c->mixed ? ncclFloat16 : ncclFloat32;
    if (c->overlap_now()) {
      // fp16 SUM in buckets on the comm stream (allreduce_plan); each group of buckets waits for the
      // GEMM that wrote it, the last group carries the loss sum
      S* a = n.arena;
      cudaStream_t cs = c->comm_stream;
      CUDA_OR_FAIL(c, cudaEventRecord(c->ev_a_end, c->stream));
      const cudaEvent_t after_ev[5] = {c->ev_wdec, c->ev_wh_a, c->ev_wh, c->ev_wmh, c->ev_a_end};
      const std::vector<ArRange> plan = allreduce_plan(c);
      for (size_t k = 0; k < plan.size();) {
        const int32_t after = plan[k].after;
        CUDA_OR_FAIL(c, cudaStreamWaitEvent(cs, after_ev[after], 0));
        NCCL_OR_FAIL(c, ncclGroupStart());
        for (; k < plan.size() && plan[k].after == after; ++k)
          NCCL_OR_FAIL(c, ncclAllReduce(a + plan[k].off, a + plan[k].off, (size_t)plan[k].count, dt, ncclSum, c->comm, cs));
        if (k == plan.size())
          NCCL_OR_FAIL(c, ncclAllReduce(&c->st->loss_sum, &c->st->loss_sum, 1, ncclFloat64, ncclSum, c->comm, cs));
        NCCL_OR_FAIL(c, ncclGroupEnd());
      }
      CUDA_OR_FAIL(c, cudaEventRecord(c->ev_comm, cs));
      CUDA_OR_FAIL(c, cudaStreamWaitEvent(c->stream, c->ev_comm, 0));
    } else {
      NCCL_OR_FAIL(c, ncclAllReduce(n.arena, n.arena, (size_t)c->P, dt, ncclSum, c->comm, c->stream));
      NCCL_OR_FAIL(c, ncclAllReduce(&c->st->loss_sum, &c->st->loss_sum, 1, ncclFloat64, ncclSum, c->comm, c->stream));
    }
  }
  CUDA_OR_FAIL(c, cudaGraphLaunch(c->gB, c->stream));
  if (c->profile) CUDA_OR_FAIL(c, cudaEventRecord(c->ev[NPH], c->stream));
  CUDA_OR_FAIL(c, cudaMemcpyAsync(c->st_host + slot, c->st, sizeof(DevState), cudaMemcpyDeviceToHost, c->stream));
  return MLSTM_OK;
}

mlstm_status ctx_ok(mlstm_ctx* c) {
  if (!c) return fail(MLSTM_EINVAL, "null context");
  if (c->failed != MLSTM_OK) return fail(c->failed, "context failed earlier: " + g_err);
  return MLSTM_OK;
}

void fill_result(mlstm_ctx* c, const DevState& s, mlstm_step_result* out) {
  c->last = s;
  c->have_last = true;
  if (!out) return;
  const double denom = (double)c->Bfull * c->world * c->T;
  out->loss_nats = s.loss_sum / denom;
  out->bpc = out->loss_nats / std::log(2.0);
  out->lr = s.lr_used;
  out->loss_scale = s.alpha_used;
  out->skipped = s.skipped;
  out->step = s.it - 1;
  out->applied = s.tau;
}

// Result delivery + divergence detector for one completed step, in step order.  A step
// counts towards divergence when its loss is non-finite (whether or not the update was skipped --
// a NaN loss makes the gradients non-finite, so such steps are always skipped) or when it was
// skipped at the minimum loss scale (alpha cannot back off any further).
mlstm_status deliver(mlstm_ctx* c, int slot, mlstm_step_result* out) {
  const DevState s = c->st_host[slot];
  fill_result(c, s, out);
  if (c->profile) accumulate_phases(c, PH_PREP, NPH);
  const bool bad = !std::isfinite(s.loss_sum) || (s.skipped && s.alpha_used <= c->cfg.scale_min);
  if (bad) {
    if (++c->nonfinite_run >= c->cfg.diverge_patience)
      return fail(MLSTM_EDIVERGED, "diverged: diverge_patience consecutive steps with a non-finite loss or an "
                                   "overflow at the minimum loss scale");
  } else {
    c->nonfinite_run = 0;
  }
  return MLSTM_OK;
}

// Delivers every outstanding MLSTM_ASYNC result (oldest first); the first failure is returned
// after all of them were delivered.
mlstm_status drain_pending(mlstm_ctx* c) {
  mlstm_status first = MLSTM_OK;
  for (const auto& p : c->pending) {
    CUDA_OR_FAIL(c, cudaEventSynchronize(c->ring_ev[p.slot]));
    const mlstm_status s = deliver(c, p.slot, p.out);
    if (first == MLSTM_OK) first = s;
  }
  c->pending.clear();
  return first;
}

mlstm_status after_step(mlstm_ctx* c, mlstm_step_result* out) {
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  return deliver(c, kAsyncRing, out);
}

template <typename S>
mlstm_status run_eval(mlstm_ctx* c, int Be, double* nats, double* tok) {
  Net<S>& n = net<S>(c);
  g_force_plan = c->force_plan;
  const mlstm_status fs = enqueue_forward<S>(c, MLSTM_SLOT_EVAL);
  g_force_plan = 0;
  RET_IF(fs);
  LAUNCH(c, (ce_kernel<S><<<c->nblk_ce, 256, 0, c->stream>>>(n, Be, 0.f, 0)));
  LAUNCH(c, (ce_reduce_kernel<S><<<1, 256, 0, c->stream>>>(n, c->nblk_ce, 0)));
  LAUNCH(c, (eval_tokens_kernel<S><<<1, 256, 0, c->stream>>>(n, Be, c->eval_tok)));
  LAUNCH(c, (state_out_kernel<S><<<grid_for((long)c->B * c->h), 256, 0, c->stream>>>(n, MLSTM_SLOT_EVAL)));
  if (c->world > 1) {
    NCCL_OR_FAIL(c, ncclAllReduce(&c->st->loss_sum, &c->st->loss_sum, 1, ncclFloat64, ncclSum, c->comm, c->stream));
    NCCL_OR_FAIL(c, ncclAllReduce(c->eval_tok, c->eval_tok, 1, ncclFloat64, ncclSum, c->comm, c->stream));
  }
  CUDA_OR_FAIL(c, cudaMemcpyAsync(nats, &c->st->loss_sum, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_FAIL(c, cudaMemcpyAsync(tok, c->eval_tok, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  return MLSTM_OK;
}

// One evaluation window from device (D2D) or host (H2D) buffers; nats and tokens over all ranks.
mlstm_status eval_window(mlstm_ctx* c, const uint8_t* bytes, int32_t Be, const uint8_t* reset, cudaMemcpyKind kind,
                         double* nats, double* tok) {
  CUDA_OR_FAIL(c, cudaMemsetAsync(c->bytes, 0, (size_t)c->B * (c->T + 1), c->stream));
  CUDA_OR_FAIL(c, cudaMemcpyAsync(c->bytes, bytes, (size_t)Be * (c->T + 1), kind, c->stream));
  CUDA_OR_FAIL(c, cudaMemsetAsync(c->reset, 0, c->B, c->stream));
  if (reset) CUDA_OR_FAIL(c, cudaMemcpyAsync(c->reset, reset, Be, kind, c->stream));
  set_microbatch_kernel<<<1, 1, 0, c->stream>>>(c->st, 0);
  CUDA_OR_FAIL(c, cudaGetLastError());
  return c->mixed ? run_eval<__half>(c, Be, nats, tok) : run_eval<float>(c, Be, nats, tok);
}

float half_bits_to_float(uint16_t b) {
  __half_raw r;
  r.x = b;
  return __half2float(__half(r));
}

// Copies `count` S elements at `dev` into host floats.
mlstm_status read_floats(mlstm_ctx* c, const void* dev, long count, float* host) {
  if (c->mixed) {
    std::vector<uint16_t> tmp(count);
    CUDA_OR_FAIL(c, cudaMemcpyAsync(tmp.data(), dev, count * 2, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
    for (long i = 0; i < count; ++i) host[i] = half_bits_to_float(tmp[i]);
  } else {
    CUDA_OR_FAIL(c, cudaMemcpyAsync(host, dev, count * 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  }
  return MLSTM_OK;
}

mlstm_status write_floats(mlstm_ctx* c, void* dev, long count, const float* host) {
  if (c->mixed) {
    std::vector<uint16_t> tmp(count);
    for (long i = 0; i < count; ++i) {
      __half_raw r = __half(__float2half_rn(host[i]));
      tmp[i] = r.x;
    }
    CUDA_OR_FAIL(c, cudaMemcpyAsync(dev, tmp.data(), count * 2, cudaMemcpyHostToDevice, c->stream));
  } else {
    CUDA_OR_FAIL(c, cudaMemcpyAsync(dev, host, count * 4, cudaMemcpyHostToDevice, c->stream));
  }
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  return MLSTM_OK;
}

const void* hstate_ptr(mlstm_ctx* c) { return c->mixed ? (const void*)c->nh.hstate : (const void*)c->nf.hstate; }
float* cstate_ptr(mlstm_ctx* c) { return c->mixed ? c->nh.cstate : c->nf.cstate; }

}  // namespace

// ====================================================================== C ABI
extern "C" {

void mlstm_default_config(mlstm_config* cfg) {
  if (!cfg) return;
  memset(cfg, 0, sizeof *cfg);
  cfg->hidden = 4096;
  cfg->embed = 64;
  cfg->vocab = 256;
  cfg->seq_len = 256;
  cfg->batch = 256;
  cfg->micro_batch = 0;
  cfg->precision = MLSTM_MIXED;
  cfg->weight_norm = 0;
  cfg->seed = 0x5EED;
  cfg->lr0 = 3e-3;
  cfg->decay_iters = 100000;
  cfg->beta1 = 0.9;
  cfg->beta2 = 0.999;
  cfg->eps = 1e-8;
  cfg->scale_init = 65536.f;
  cfg->scale_min = 1.f;
  cfg->scale_max = 16777216.f;
  cfg->scale_growth_interval = 2000;
  cfg->diverge_patience = 50;
}

int64_t mlstm_param_count(const mlstm_config* cfg) {
  if (!cfg) return 0;
  ParamOffsets po;
  po.set(cfg->hidden, cfg->embed, cfg->weight_norm);
  return po.P;
}

size_t mlstm_workspace_bytes(const mlstm_config* cfg) {
  if (validate(cfg) != MLSTM_OK) return 0;
  mlstm_ctx tmp;
  set_dims(&tmp, cfg);
  return layout_bytes(&tmp);
}

mlstm_status mlstm_allreduce_plan(const mlstm_config* cfg, int32_t world, int64_t* out, int32_t cap, int32_t* n) {
  RET_IF(validate(cfg));
  if (world < 1 || !n || (cap > 0 && !out)) return fail(MLSTM_EINVAL, "bad arguments");
  mlstm_ctx tmp;
  set_dims(&tmp, cfg);
  tmp.world = world;
  const std::vector<ArRange> plan = allreduce_plan(&tmp);
  *n = (int32_t)plan.size();
  if ((int32_t)plan.size() > cap) return fail(MLSTM_EINVAL, "cap smaller than the number of buckets");
  for (size_t k = 0; k < plan.size(); ++k) {
    out[3 * k] = plan[k].off;
    out[3 * k + 1] = plan[k].count;
    out[3 * k + 2] = plan[k].after;
  }
  return MLSTM_OK;
}

mlstm_status mlstm_nccl_unique_id(uint8_t out[128]) {
  if (!out) return fail(MLSTM_EINVAL, "null out");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(MLSTM_ENCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  memcpy(out, &id, 128);
  return MLSTM_OK;
}

mlstm_status mlstm_init(const mlstm_config* cfg, void* workspace, size_t workspace_bytes, void* cuda_stream,
                        const uint8_t* nccl_id, int rank, int world, mlstm_ctx** out) {
  if (!out) return fail(MLSTM_EINVAL, "null out");
  *out = nullptr;
  RET_IF(validate(cfg));
  if (world < 1 || rank < 0 || rank >= world) return fail(MLSTM_EINVAL, "bad rank/world");
  if (world > 1 && !nccl_id) return fail(MLSTM_EINVAL, "nccl_id required when world > 1");
  if (!workspace || (reinterpret_cast<uintptr_t>(workspace) & 255))
    return fail(MLSTM_EINVAL, "workspace must be non-null and 256-byte aligned");
  int dev = 0;
  cudaDeviceProp prop;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess)
    return fail(MLSTM_ECUDA, "no CUDA device");
  if (prop.major != 10 || prop.minor != 0)
    return fail(MLSTM_ECUDA, "libmlstm is built for sm_100a (B200); device is sm_" + std::to_string(prop.major) +
                                 std::to_string(prop.minor));
  mlstm_ctx* c = new mlstm_ctx();
  set_dims(c, cfg);
  const size_t need = layout_bytes(c);
  if (workspace_bytes < need) {
    delete c;
    return fail(MLSTM_ENOMEM, "workspace too small: need " + std::to_string(need));
  }
  if (c->tc && !get_encoder()) {
    delete c;
    return fail(MLSTM_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
  }
  c->rank = rank;
  c->world = world;
  c->stream = static_cast<cudaStream_t>(cuda_stream);
  c->ws = static_cast<uint8_t*>(workspace);
  c->ws_bytes = workspace_bytes;
  Carver cv{c->ws};
  if (c->mixed) carve(c, cv, c->nh);
  else carve(c, cv, c->nf);
  auto bail = [&](mlstm_status s) {
    mlstm_destroy(c);
    return s;
  };
  if (cudaMallocHost(&c->st_host, sizeof(DevState) * (kAsyncRing + 1)) != cudaSuccess)
    return bail(fail(MLSTM_ECUDA, "cudaMallocHost"));
  for (int i = 0; i < kAsyncRing; ++i)
    if (cudaEventCreateWithFlags(&c->ring_ev[i], cudaEventDisableTiming) != cudaSuccess)
      return bail(fail(MLSTM_ECUDA, "cudaEventCreate"));
  if (cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(MLSTM_ECUDA, "cudaStreamCreate"));
  if (c->side_chunks > 0) {
    cudaDeviceGetStreamPriorityRange(&c->prio_lo, &c->prio_hi);
    if (cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, c->prio_lo) != cudaSuccess)
      return bail(fail(MLSTM_ECUDA, "cudaStreamCreateWithPriority"));
    for (cudaEvent_t& ev : c->side_ev)
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(MLSTM_ECUDA, "cudaEventCreate"));
    if (cudaMalloc(&c->wpart, sizeof(float) * 4 * (size_t)c->h * c->h) != cudaSuccess)
      return bail(fail(MLSTM_ECUDA, "cudaMalloc wpart"));
  }
  for (int i = 0; i <= NPH; ++i)
    if (cudaEventCreate(&c->ev[i]) != cudaSuccess) return bail(fail(MLSTM_ECUDA, "cudaEventCreate"));
  // zero everything (pads of the transposed stashes must stay zero), then init
  if (cudaMemsetAsync(c->ws, 0, need - 256, c->stream) != cudaSuccess) return bail(fail(MLSTM_ECUDA, "memset"));
  DevState s0{};
  s0.alpha = cfg->scale_init;
  s0.alpha_used = cfg->scale_init;
  if (cudaMemcpyAsync(c->st, &s0, sizeof s0, cudaMemcpyHostToDevice, c->stream) != cudaSuccess)
    return bail(fail(MLSTM_ECUDA, "memcpy state"));
  float* master = c->mixed ? c->nh.master : c->nf.master;
  init_params_kernel<<<grid_for(c->P), 256, 0, c->stream>>>(master, c->po, c->h, c->e, cfg->seed);
  if (c->po.wn) wn_init_gain_kernel<<<grid_for(10L * c->h * 32), 256, 0, c->stream>>>(master, c->po, c->h, c->e);
  if (cudaGetLastError() != cudaSuccess) return bail(fail(MLSTM_ECUDA, "init kernel"));
  mlstm_status s = c->mixed ? enqueue_cast<__half>(c) : enqueue_cast<float>(c);
  if (s != MLSTM_OK) return bail(s);
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(fail(MLSTM_ECUDA, "init sync"));
  if (world > 1) {
    ncclUniqueId id;
    memcpy(&id, nccl_id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
    if (r != ncclSuccess) return bail(fail(MLSTM_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    if (cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi) != cudaSuccess)
      return bail(fail(MLSTM_ECUDA, "cudaStreamCreateWithPriority"));
    for (cudaEvent_t* ev : {&c->ev_wh, &c->ev_wmh, &c->ev_a_end, &c->ev_comm, &c->ev_wh_a, &c->ev_wdec})
      if (cudaEventCreateWithFlags(ev, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(MLSTM_ECUDA, "cudaEventCreate"));
  }
  *out = c;
  return MLSTM_OK;
}

mlstm_status mlstm_train_step(mlstm_ctx* c, const uint8_t* bytes, const uint8_t* reset, uint32_t flags,
                              mlstm_step_result* out) {
  RET_IF(ctx_ok(c));
  if (!bytes) return fail(MLSTM_EINVAL, "null bytes");
  if (flags & MLSTM_ASYNC) {
    mlstm_status first = MLSTM_OK;
    if ((int)c->pending.size() == kAsyncRing) {  // ring full: deliver the oldest
      const auto p = c->pending.front();
      CUDA_OR_FAIL(c, cudaEventSynchronize(c->ring_ev[p.slot]));
      c->pending.erase(c->pending.begin());
      first = deliver(c, p.slot, p.out);
    }
    const int slot = c->ring_next;
    c->ring_next = (c->ring_next + 1) % kAsyncRing;
    RET_IF(c->mixed ? run_train<__half>(c, bytes, reset, cudaMemcpyDeviceToDevice, slot)
                    : run_train<float>(c, bytes, reset, cudaMemcpyDeviceToDevice, slot));
    CUDA_OR_FAIL(c, cudaEventRecord(c->ring_ev[slot], c->stream));
    c->pending.push_back({out, slot});
    return first;
  }
  const mlstm_status prev = drain_pending(c);
  RET_IF(c->mixed ? run_train<__half>(c, bytes, reset, cudaMemcpyDeviceToDevice, kAsyncRing)
                  : run_train<float>(c, bytes, reset, cudaMemcpyDeviceToDevice, kAsyncRing));
  const mlstm_status s = after_step(c, out);
  return prev != MLSTM_OK ? prev : s;
}

mlstm_status mlstm_sync(mlstm_ctx* c) {
  RET_IF(ctx_ok(c));
  return drain_pending(c);
}

mlstm_status mlstm_train_step_host(mlstm_ctx* c, const uint8_t* bytes_host, const uint8_t* reset_host,
                                   mlstm_step_result* out) {
  RET_IF(ctx_ok(c));
  if (!bytes_host) return fail(MLSTM_EINVAL, "null bytes");
  const mlstm_status prev = drain_pending(c);
  RET_IF(c->mixed ? run_train<__half>(c, bytes_host, reset_host, cudaMemcpyHostToDevice, kAsyncRing)
                  : run_train<float>(c, bytes_host, reset_host, cudaMemcpyHostToDevice, kAsyncRing));
  const mlstm_status s = after_step(c, out);
  return prev != MLSTM_OK ? prev : s;
}

mlstm_status mlstm_eval(mlstm_ctx* c, const uint8_t* bytes, int32_t Be, const uint8_t* reset, double* nats_sum,
                        int64_t* tokens, double* bpc) {
  RET_IF(ctx_ok(c));
  if (!bytes || Be <= 0 || Be > c->B) return fail(MLSTM_EINVAL, "eval needs bytes and 0 < Be <= batch");
  double nats = 0, tok = 0;
  RET_IF(eval_window(c, bytes, Be, reset, cudaMemcpyDeviceToDevice, &nats, &tok));
  if (nats_sum) *nats_sum = nats;
  if (tokens) *tokens = (int64_t)tok;
  if (bpc) *bpc = tok > 0 ? nats / tok / std::log(2.0) : 0.0;
  return MLSTM_OK;
}

double mlstm_lr_at(double lr0, int64_t it, int64_t decay_iters) {
  if (decay_iters <= 0) return 0.0;
  return lr0 * std::fmax(0.0, 1.0 - (double)it / (double)decay_iters);
}

double mlstm_scale_lr(double base_lr, int rule, int64_t batch, int64_t ref_batch) {
  if (ref_batch <= 0) ref_batch = 128;
  const double r = (double)batch / (double)ref_batch;
  switch (rule) {
    case MLSTM_LR_LINEAR: return base_lr * r;
    case MLSTM_LR_SQRT: return base_lr * std::sqrt(r);
    default: return base_lr;
  }
}

double mlstm_bpc_from_nats(double nats) { return nats / std::log(2.0); }

mlstm_status mlstm_get_params(mlstm_ctx* c, float* host_out) {
  RET_IF(ctx_ok(c));
  if (!host_out) return fail(MLSTM_EINVAL, "null out");
  float* master = c->mixed ? c->nh.master : c->nf.master;
  CUDA_OR_FAIL(c, cudaMemcpyAsync(host_out, master, sizeof(float) * c->P, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  return MLSTM_OK;
}

mlstm_status mlstm_set_params(mlstm_ctx* c, const float* host_in) {
  RET_IF(ctx_ok(c));
  if (!host_in) return fail(MLSTM_EINVAL, "null in");
  float* master = c->mixed ? c->nh.master : c->nf.master;
  CUDA_OR_FAIL(c, cudaMemcpyAsync(master, host_in, sizeof(float) * c->P, cudaMemcpyHostToDevice, c->stream));
  RET_IF(c->mixed ? enqueue_cast<__half>(c) : enqueue_cast<float>(c));
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  return MLSTM_OK;
}

mlstm_status mlstm_get_grads(mlstm_ctx* c, float* host_out) {
  RET_IF(ctx_ok(c));
  if (!host_out) return fail(MLSTM_EINVAL, "null out");
  if (!c->have_last) return fail(MLSTM_ESTATE, "no train step has completed");
  const void* arena = c->mixed ? (const void*)c->nh.arena : (const void*)c->nf.arena;
  RET_IF(read_floats(c, arena, c->P, host_out));
  const float inv = 1.f / c->last.alpha_used;
  for (long i = 0; i < c->P; ++i) host_out[i] *= inv;
  return MLSTM_OK;
}

mlstm_status mlstm_get_state(mlstm_ctx* c, int slot, float* h_out, float* c_out) {
  RET_IF(ctx_ok(c));
  if (slot != 0 && slot != 1) return fail(MLSTM_EINVAL, "bad slot");
  const long BH = (long)c->Bfull * c->h;
  const size_t es = c->mixed ? 2 : 4;
  if (h_out) RET_IF(read_floats(c, (const uint8_t*)hstate_ptr(c) + es * slot * BH, BH, h_out));
  if (c_out) {
    CUDA_OR_FAIL(c, cudaMemcpyAsync(c_out, cstate_ptr(c) + slot * BH, 4 * BH, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  }
  return MLSTM_OK;
}

mlstm_status mlstm_set_state(mlstm_ctx* c, int slot, const float* h_in, const float* c_in) {
  RET_IF(ctx_ok(c));
  if (slot != 0 && slot != 1) return fail(MLSTM_EINVAL, "bad slot");
  const long BH = (long)c->Bfull * c->h;
  const size_t es = c->mixed ? 2 : 4;
  if (h_in) RET_IF(write_floats(c, (uint8_t*)hstate_ptr(c) + es * slot * BH, BH, h_in));
  if (c_in) {
    CUDA_OR_FAIL(c, cudaMemcpyAsync(cstate_ptr(c) + slot * BH, c_in, 4 * BH, cudaMemcpyHostToDevice, c->stream));
    CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  }
  return MLSTM_OK;
}

mlstm_status mlstm_get_opt_state(mlstm_ctx* c, float* m_out, float* v_out, int64_t* tau, float* alpha,
                                 int32_t* clean_steps, int64_t* it) {
  RET_IF(ctx_ok(c));
  if (m_out) CUDA_OR_FAIL(c, cudaMemcpyAsync(m_out, c->adam_m, 4 * c->P, cudaMemcpyDeviceToHost, c->stream));
  if (v_out) CUDA_OR_FAIL(c, cudaMemcpyAsync(v_out, c->adam_v, 4 * c->P, cudaMemcpyDeviceToHost, c->stream));
  DevState s;
  CUDA_OR_FAIL(c, cudaMemcpyAsync(&s, c->st, sizeof s, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  if (tau) *tau = s.tau;
  if (alpha) *alpha = s.alpha;
  if (clean_steps) *clean_steps = s.clean;
  if (it) *it = s.it;
  return MLSTM_OK;
}

mlstm_status mlstm_set_opt_state(mlstm_ctx* c, const float* m_in, const float* v_in, int64_t tau, float alpha,
                                 int32_t clean_steps, int64_t it) {
  RET_IF(ctx_ok(c));
  if (!(alpha >= c->cfg.scale_min && alpha <= c->cfg.scale_max) || tau < 0 || it < 0 || clean_steps < 0)
    return fail(MLSTM_EINVAL, "bad optimiser state");
  if (m_in) CUDA_OR_FAIL(c, cudaMemcpyAsync(c->adam_m, m_in, 4 * c->P, cudaMemcpyHostToDevice, c->stream));
  if (v_in) CUDA_OR_FAIL(c, cudaMemcpyAsync(c->adam_v, v_in, 4 * c->P, cudaMemcpyHostToDevice, c->stream));
  DevState s;
  CUDA_OR_FAIL(c, cudaMemcpyAsync(&s, c->st, sizeof s, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  s.tau = tau;
  s.alpha = alpha;
  s.clean = clean_steps;
  s.it = it;
  CUDA_OR_FAIL(c, cudaMemcpyAsync(c->st, &s, sizeof s, cudaMemcpyHostToDevice, c->stream));
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  return MLSTM_OK;
}

mlstm_status mlstm_debug_dump(mlstm_ctx* c, const char* name, float* host_out, size_t n) {
  RET_IF(ctx_ok(c));
  if (!name || !host_out) return fail(MLSTM_EINVAL, "null argument");
  const long B = c->B, T = c->T, h = c->h, e = c->e;
  const std::string nm(name);
  auto need = [&](long k) { return (size_t)k <= n; };
  if (nm == "x") {
    const long cnt = T * B * e;
    if (!need(cnt)) return fail(MLSTM_EINVAL, "buffer too small");
    float* tmp = nullptr;
    CUDA_OR_FAIL(c, cudaMalloc(&tmp, cnt * 4));
    if (c->mixed) gather_x_kernel<__half><<<grid_for(cnt), 256, 0, c->stream>>>(c->nh, tmp);
    else gather_x_kernel<float><<<grid_for(cnt), 256, 0, c->stream>>>(c->nf, tmp);
    cudaError_t e1 = cudaMemcpyAsync(host_out, tmp, cnt * 4, cudaMemcpyDeviceToHost, c->stream);
    cudaError_t e2 = cudaStreamSynchronize(c->stream);
    cudaFree(tmp);
    CUDA_OR_FAIL(c, e1);
    CUDA_OR_FAIL(c, e2);
    return MLSTM_OK;
  }
  if (nm == "logits" || nm == "loss_rows" || nm == "c" || nm == "tab") {
    const float* src;
    long cnt;
    if (nm == "logits") src = c->mixed ? c->nh.Y : c->nf.Y, cnt = T * B * 256;
    else if (nm == "loss_rows") src = c->mixed ? c->nh.lossrow : c->nf.lossrow, cnt = T * B;
    else if (nm == "c") src = (c->mixed ? c->nh.Crm : c->nf.Crm) + B * h, cnt = T * B * h;
    else src = c->mixed ? c->nh.tab : c->nf.tab, cnt = 256 * 5 * h;
    if (!need(cnt)) return fail(MLSTM_EINVAL, "buffer too small");
    CUDA_OR_FAIL(c, cudaMemcpyAsync(host_out, src, cnt * 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
    return MLSTM_OK;
  }
  if (nm == "m" || nm == "a") {  // the stashes the recurrence wrote: m_t = mx_t * a_t and a_t, [T][B][h]
    const long cnt = T * B * h;
    if (!need(cnt)) return fail(MLSTM_EINVAL, "buffer too small");
    const void* src = nm == "m" ? (c->mixed ? (const void*)c->nh.Mrm : (const void*)c->nf.Mrm)
                                : (c->mixed ? (const void*)c->nh.Astash : (const void*)c->nf.Astash);
    return read_floats(c, src, cnt, host_out);
  }
  if (nm == "h") {
    const long cnt = T * B * h;
    if (!need(cnt)) return fail(MLSTM_EINVAL, "buffer too small");
    const size_t es = c->mixed ? 2 : 4;
    const void* src = c->mixed ? (const void*)c->nh.Hrm : (const void*)c->nf.Hrm;
    return read_floats(c, (const uint8_t*)src + es * B * h, cnt, host_out);
  }
  if (nm == "onehot") {  // [256][T][B]
    const long cnt = 256 * T * B;
    if (!need(cnt)) return fail(MLSTM_EINVAL, "buffer too small");
    std::vector<float> all(cnt);  // OHR is [T][B][256]
    const uint8_t* base = c->mixed ? (const uint8_t*)c->nh.OHR : (const uint8_t*)c->nf.OHR;
    RET_IF(read_floats(c, base, cnt, all.data()));
    for (int v = 0; v < 256; ++v)
      for (long t = 0; t < T; ++t)
        for (long b = 0; b < B; ++b) host_out[(v * T + t) * B + b] = all[(t * B + b) * 256 + v];
    return MLSTM_OK;
  }
  return fail(MLSTM_EINVAL, "unknown dump name");
}

mlstm_status mlstm_check_overflow(mlstm_ctx* c, const void* device_buf, int64_t n, int dtype, int32_t* flag) {
  RET_IF(ctx_ok(c));
  if (!device_buf || !flag || n < 0 || (dtype != 0 && dtype != 1)) return fail(MLSTM_EINVAL, "bad arguments");
  CUDA_OR_FAIL(c, cudaMemsetAsync(c->scratch_flag, 0, 4, c->stream));
  if (dtype == 0)
    overflow_kernel<__half><<<grid_for(n), 256, 0, c->stream>>>((const __half*)device_buf, n, c->scratch_flag);
  else
    overflow_kernel<float><<<grid_for(n), 256, 0, c->stream>>>((const float*)device_buf, n, c->scratch_flag);
  CUDA_OR_FAIL(c, cudaGetLastError());
  CUDA_OR_FAIL(c, cudaMemcpyAsync(flag, c->scratch_flag, 4, cudaMemcpyDeviceToHost, c->stream));
  CUDA_OR_FAIL(c, cudaStreamSynchronize(c->stream));
  return MLSTM_OK;
}

mlstm_status mlstm_profile_enable(mlstm_ctx* c, int enable) {
  RET_IF(ctx_ok(c));
  if ((enable != 0) != c->profile) {
    c->profile = enable != 0;
    if (c->gA) cudaGraphExecDestroy(c->gA);
    if (c->gB) cudaGraphExecDestroy(c->gB);
    c->gA = c->gB = nullptr;
  }
  memset(c->phase_ms, 0, sizeof c->phase_ms);
  return MLSTM_OK;
}

mlstm_status mlstm_phase_times(mlstm_ctx* c, double* ms_out, int32_t* launches_out, int32_t* n_phases) {
  RET_IF(ctx_ok(c));
  if (n_phases) *n_phases = NPH;
  for (int i = 0; i < NPH; ++i) {
    if (ms_out) ms_out[i] = c->phase_ms[i];
    if (launches_out) launches_out[i] = c->phase_launches[i];
  }
  return MLSTM_OK;
}

const char* mlstm_phase_name(int phase) { return (phase >= 0 && phase < NPH) ? kPhaseNames[phase] : ""; }

int32_t mlstm_launches_per_step(mlstm_ctx* c) {
  if (!c) return 0;
  if (!c->gA) {
    mlstm_status s = c->mixed ? build_graphs<__half>(c) : build_graphs<float>(c);
    if (s != MLSTM_OK) return -1;
  }
  return c->launches;
}

int32_t mlstm_recurrence_kind(mlstm_ctx* c) {
  if (!c) return -1;
  return recur_on(c) ? (c->recur_fwd_only ? 3 : 1) : 0;
}

mlstm_status mlstm_gemm_bench(int engine, int M, int N, int K, int bn, int iters, double* ms) {
  if (!ms || M <= 0 || N <= 0 || K <= 0 || iters <= 0 || engine < 1 || engine > 3 ||
      (bn != 0 && bn != 64 && bn != 128 && bn != 256 && !(bn == 512 && engine == 2)) || N % 64 || K % 8)
    return fail(MLSTM_EINVAL, "bad gemm_bench arguments");
  if (!get_encoder()) return fail(MLSTM_ECUDA, "cuTensorMapEncodeTiled unavailable");
  mlstm_ctx c;
  c.tc = true;
  if (cudaMalloc(&c.split_scratch, sizeof(float) * kSplitScratchFloats) != cudaSuccess)
    return fail(MLSTM_ECUDA, "cudaMalloc");
  __half *A = nullptr, *B = nullptr;
  float* D = nullptr;
  cudaEvent_t e0, e1;
  auto cleanup = [&]() {
    cudaFree(c.split_scratch);
    cudaFree(A);
    cudaFree(B);
    cudaFree(D);
  };
  if (cudaMalloc(&A, 2L * M * K) != cudaSuccess || cudaMalloc(&B, 2L * N * K) != cudaSuccess ||
      cudaMalloc(&D, 4L * M * N) != cudaSuccess) {
    cleanup();
    return fail(MLSTM_ECUDA, "cudaMalloc");
  }
  const long nA = (long)M * K, nB = (long)N * K;
  // random operands: constant bit patterns draw less tensor-core power and overstate throughput
  random_half_kernel<<<grid_for(nA), 256>>>(A, nA, 1);
  random_half_kernel<<<grid_for(nB), 256>>>(B, nB, 2);
  Opd oa{A, M, K, K, 1, nA}, ob{B, N, K, K, 1, nB, 0, true};
  Plan p = plan_gemm(true, M, N, K, false);
  if (engine != 3) {
    p.cluster = false;
    p.pair = engine == 2;
    p.splits = 1;
    if (bn) p.bn = bn;
    if (bn == 512) p.persist = false;
  }
  EpiPartial epi{D, N, (long)M * N};
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mlstm_status st = gemm<__half>(&c, oa, 0, ob, 0, M, N, K, p, epi);
  if (st == MLSTM_OK) {
    cudaEventRecord(e0);
    for (int i = 0; i < iters && st == MLSTM_OK; ++i) st = gemm<__half>(&c, oa, 0, ob, 0, M, N, K, p, epi);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float t = 0;
    cudaEventElapsedTime(&t, e0, e1);
    *ms = t / iters;
    if (e != cudaSuccess) st = fail(MLSTM_ECUDA, cudaGetErrorString(e));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cleanup();
  return st;
}

namespace {
TraceRec* g_trace_host_buf = nullptr;
}

mlstm_status mlstm_trace_enable(int capacity) {
  if (g_trace_host_buf) {
    cudaFree(g_trace_host_buf);
    g_trace_host_buf = nullptr;
  }
  TraceRec* p = nullptr;
  unsigned int cap = capacity > 0 ? (unsigned int)capacity : 0u, zero = 0;
  if (cap && cudaMalloc(&p, sizeof(TraceRec) * cap) != cudaSuccess) return fail(MLSTM_ECUDA, "cudaMalloc trace");
  g_trace_host_buf = p;
  if (cudaMemcpyToSymbol(g_trace, &p, sizeof p) != cudaSuccess ||
      cudaMemcpyToSymbol(g_trace_cap, &cap, sizeof cap) != cudaSuccess ||
      cudaMemcpyToSymbol(g_trace_n, &zero, sizeof zero) != cudaSuccess)
    return fail(MLSTM_ECUDA, "trace symbols");
  return MLSTM_OK;
}

mlstm_status mlstm_trace_read(uint64_t* out, int capacity, int* n) {
  if (!out || !n) return fail(MLSTM_EINVAL, "null argument");
  unsigned int cnt = 0, zero = 0;
  if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpyFromSymbol(&cnt, g_trace_n, sizeof cnt) != cudaSuccess)
    return fail(MLSTM_ECUDA, "trace count");
  unsigned int cap = 0;
  cudaMemcpyFromSymbol(&cap, g_trace_cap, sizeof cap);
  cnt = std::min(cnt, cap);
  cnt = std::min(cnt, (unsigned int)std::max(capacity, 0));
  if (cnt && cudaMemcpy(out, g_trace_host_buf, sizeof(TraceRec) * cnt, cudaMemcpyDeviceToHost) != cudaSuccess)
    return fail(MLSTM_ECUDA, "trace copy");
  cudaMemcpyToSymbol(g_trace_n, &zero, sizeof zero);
  *n = (int)cnt;
  return MLSTM_OK;
}

const char* mlstm_last_error(void) { return g_err.c_str(); }

void mlstm_destroy(mlstm_ctx* c) {
  if (!c) return;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->gA) cudaGraphExecDestroy(c->gA);
  if (c->gB) cudaGraphExecDestroy(c->gB);
  for (int i = 0; i <= NPH; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  if (c->st_host) cudaFreeHost(c->st_host);
  for (cudaEvent_t e : c->ring_ev)
    if (e) cudaEventDestroy(e);
  if (c->cap) cudaStreamDestroy(c->cap);
  if (c->comm) ncclCommDestroy(c->comm);
  for (cudaEvent_t ev : {c->ev_wh, c->ev_wmh, c->ev_a_end, c->ev_comm, c->ev_wh_a, c->ev_wdec})
    if (ev) cudaEventDestroy(ev);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->side) cudaStreamDestroy(c->side);
  for (cudaEvent_t ev : c->side_ev)
    if (ev) cudaEventDestroy(ev);
  if (c->wpart) cudaFree(c->wpart);
  delete c;
}

}  // extern "C"

#include "loader.cuh"

extern "C" {

mlstm_status mlstm_heldout_bpc(mlstm_ctx* c, mlstm_loader* L, int64_t max_batches, double* nats_sum, int64_t* tokens,
                               double* bpc) {
  RET_IF(ctx_ok(c));
  if (!L) return fail(MLSTM_EINVAL, "null loader");
  if (L->B != c->B || L->T != c->T) return fail(MLSTM_EINVAL, "loader B / T differ from the context's batch / seq_len");
  RET_IF(mlstm_loader_rewind(L));
  const size_t W = (size_t)c->T + 1;
  std::vector<uint8_t> by((size_t)c->B * W), rs(c->B), ok(c->B);
  double nats = 0, tok = 0;
  for (int64_t k = 0; max_batches < 0 || k < max_batches; ++k) {
    int32_t end = 0;
    RET_IF(mlstm_loader_next(L, by.data(), rs.data(), ok.data(), &end));
    if (end) break;
    for (int b = 0; b < c->B; ++b)
      if (!ok[b]) rs[b] = 2;  // idle row: state reset, no tokens
    double n = 0, t = 0;
    RET_IF(eval_window(c, by.data(), c->B, rs.data(), cudaMemcpyHostToDevice, &n, &t));
    nats += n;
    tok += t;
  }
  if (nats_sum) *nats_sum = nats;
  if (tokens) *tokens = (int64_t)tok;
  if (bpc) *bpc = tok > 0 ? nats / tok / std::log(2.0) : 0.0;
  return MLSTM_OK;
}

}  // extern "C"
