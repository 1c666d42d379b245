// recur.cuh -- the recurrence (BASELINE north_star kernels (b), (c-1))
// as two persistent dataflow kernels: one launch runs all T timesteps of the forward, one all T
// timesteps of BPTT.
//
// Work mapping (B = 256 rows per micro-batch, h a multiple of 256, P = h/64 CTA pairs, one pair per
// two SMs for the whole launch).  Activations are the MMA A operand (M = 256 batch rows over the CTA
// pair, cta_group::2; CTA rank r holds rows [128r, +128)); weights are the B operand (N = 256 rows
// per pair, 128 per CTA).  Pair p owns
//   * the 256-wide N tile of a "wide" GEMM with its full K:     F2 (z = W_h m, gates)  rows [256p, +256)
//   * split z = p % 4 of an N = h GEMM's tile n1 = p / 4:        F1 (a = W_mh h)  units [256 n1, +256),
//                                                                K range [z h/4, +h/4)
//   and in the backward the two N = h GEMMs B1 (dM = dZ W_h, K = 4h) and B2 (dH = dA W_mh + dY W_dec).
// Every timestep's contraction therefore reads the same weight rows on the same SM: the TMA
// producer streams a pair's weight k-blocks continuously (they do not depend on t) and runs up to the
// ring depth ahead of the activations, which it loads only once the producing CTA has published them.
//
// Synchronisation: no grid barrier.  Each 64-column activation chunk (64 units x 128 rows of one
// rank) has a monotonic readiness flag in global memory written with release semantics by the one
// epilogue that produces it (after its coalesced stores and a named barrier); the consumer's
// producer thread acquires it, orders the async proxy after it (fence.proxy.async) and issues the TMA
// load.  K-split partials of the N = h GEMMs are exchanged through an L2 scratch with per-split flags
// and summed in fixed order z = 0..3 (deterministic; every CTA keeps its own slice in TMEM).
//
// Per-pair state that never leaves the SM: the forward cell state c (fp32 registers of the F2
// epilogue threads, 32 per thread) and the backward cell-gradient carry dc (registers of the B2
// epilogue threads).  TMEM: columns [0,256) accumulate the split GEMM (F1 / B1), [256,512) the wide
// GEMM (F2 / B2), so the next contraction's independent K segment (the one-hot input projection in
// F2, dY W_dec in B2) runs while the other accumulator's epilogue is still reducing.
//
// Launched with cluster dims (2,1,1) and the cooperative attribute (all pairs co-resident).
// Roles (352 threads): warp 0 lane 0 = weight TMA producer, warp 10 = activation TMA producer (both
// CTAs; the activation warp polls readiness flags with all lanes), warp 1 lane 0 of the leader CTA =
// tcgen05.mma issuer, warps 2..9 = epilogue (two warps per TMEM lane quarter: q = warp & 3 owns
// rows [32q, +32), grp = (warp - 2) >> 2 takes half of each 64-column slice).
#pragma once
#include "gemm.cuh"
#include "epilogues.cuh"

namespace mlstm {

constexpr int kRcStages = 5;
constexpr int kRcActWarp = 10;                // activation producer (after the 8 epilogue warps)
constexpr int kRcThreads = kGemmThreads + 32;
constexpr int kRcTile = 128 * 64 * 2;  // one 128-row x 64-K fp16 operand tile (per CTA, per stage)
constexpr int kRcWin = 8192;           // staging window of one epilogue warp
constexpr int kRcSmem = kRcStages * 2 * kRcTile + kEpiWarps * kRcWin + 1024 + 256;

struct RcPolicy {  // L2 policy codes (ptx::make_policy) of the operand streams
  uint32_t act, w_split, w_wide, w_seg;
  int flag_lanes;  // activation flags the producer warp acquires in parallel (1 = one at a time)
  int pf_dist;     // weight k-blocks prefetched into L2 ahead of the ring (0 = off)
  int rotate;      // 1: each pair starts its K loop at its own chunk (spreads the L2 reads); 0: all pairs
                   // read the shared activation chunks in the same order (same lines requested together)
  int exp;         // bit 6: no per-k-block trace records (the timing experiments of round 2 --
                   // operand substitution, skipped loads, no flags, bare epilogue -- are recorded in
                   // profiles/r02_recur_timing_experiments.log and were removed)
};

// One operand k-block of the producer's stream: its readiness flag (null = no dependency, e.g. a
// weight-only or input-only segment) and the value that flag must reach.
struct RcBlk {
  int t, kind, j;
  const uint32_t* flag;
  uint32_t target;
};

// Optional timeline (mlstm_trace_enable; tools/trace_recur.py): each CTA reserves T + per TraceRec
// records -- one per timestep {tag = 1000 + t (fwd) / 2000 + u (bwd), cta, 10 event times in ns} and
// one per k-block of the sampled timestep {tag = 3000 / 4000 + i, cta, weight issued, activation
// issued, stage full (MMA thread)}.
constexpr int kRcTraceStep = 8;
constexpr int kRcTraceBlk = 160;  // >= k-blocks per timestep (h <= 4736)
struct RcTrace {
  uint32_t base;
  int T, idx0, per, tag;
  __device__ __forceinline__ bool on() const { return base != 0xffffffffu; }
  __device__ __forceinline__ void step(int t, int slot) const {
    if (on()) g_trace[base + t].v[slot] = ptx::globaltimer();
  }
  __device__ __forceinline__ void step_tag(int t, int tg) const {
    if (on()) {
      g_trace[base + t].v[0] = (uint64_t)tg;
      g_trace[base + t].v[1] = blockIdx.x;
    }
  }
  // detail record of timestep t (tag + 2000 + t): sub-phases of the epilogues
  __device__ __forceinline__ void det(int t, int slot) const {
    if (on() && t >= 0) {
      TraceRec& rr = g_trace[base + T + t];
      rr.v[slot] = ptx::globaltimer();
      rr.v[0] = (uint64_t)(tag + 2000 + t);
      rr.v[1] = blockIdx.x;
    }
  }
  __device__ __forceinline__ void blk_val(int idx, int slot, uint64_t v) const {
    const int i = idx - idx0;
    if (on() && i >= 0 && i < per) g_trace[base + 2 * T + i].v[slot] = v;
  }
  __device__ __forceinline__ uint64_t now() const { return on() ? ptx::globaltimer() : 0; }
  __device__ __forceinline__ void blk(int idx, int slot) const {
    const int i = idx - idx0;
    if (on() && i >= 0 && i < per) {
      TraceRec& rr = g_trace[base + 2 * T + i];
      rr.v[slot] = ptx::globaltimer();
      if (slot == 2) {
        rr.v[0] = (uint64_t)(tag + i);
        rr.v[1] = blockIdx.x;
      }
    }
  }
};
__device__ __forceinline__ uint32_t rc_trace_reserve(int n) {
  if (!g_trace) return 0xffffffffu;
  const uint32_t base = atomicAdd(&g_trace_n, (uint32_t)n);
  return base + (uint32_t)n <= g_trace_cap ? base : 0xffffffffu;
}

struct RcLayout {
  uint8_t *sA, *sB, *win;
  uint64_t *full, *empty, *accf, *acce;
  uint32_t* tmem_slot;
  __device__ __forceinline__ explicit RcLayout(uint8_t* raw) {
    uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    sA = s;
    sB = s + kRcStages * kRcTile;
    win = s + 2 * kRcStages * kRcTile;
    full = reinterpret_cast<uint64_t*>(win + kEpiWarps * kRcWin);
    empty = full + kRcStages;
    accf = empty + kRcStages;
    acce = accf + 2;
    tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
  }
};

// Flag words (reset to 0 before each launch), P = pairs:
//   [0, 2P)   chunk flags X[p][r]  (fwd: H_t of pair p;  bwd: unused)
//   [2P, 4P)  chunk flags Y[p][r]  (fwd: M_t chunk p;   bwd: dA_t chunk p)
//   [4P, 6P)  split partial flags of the first N = h GEMM  [(n1, r)][z]  (fwd F1, bwd B1)
//   [6P, 8P)  split partial flags of the second            [(n1, r)][z]  (bwd B2)
//   [8P, 16P) bwd: dZ_s chunk flags [(p, r)][c], c = the pair's 64-column chunk (16 units x 4 gates),
//             published per chunk so B1 starts on the first chunks while the rest are computed
constexpr int kRcFlagWords(int P) { return 16 * P; }
// Split-K scratch: per (GEMM, timestep parity) region, per (tile n1, rank r) group
// [zsrc 4][zdst 4][16 float4 column groups][128 rows].  Alternating parities keep a fast CTA's next
// partial from overwriting one a slow peer has not read yet (the flags order t before t + 2).
constexpr long kRcGroupF4 = 16L * 16 * 128;
inline long rc_scratch_floats(int h) { return 4L * 4 * (h / 256) * 2 * kRcGroupF4; }

// Barrier setup shared by both kernels: full (2 arrivals of the leader's producer: weights and
// activations, bytes of both CTAs), empty (MMA commit, multicast), accf (MMA commit, multicast),
// acce (one arrive per epilogue warp of both CTAs); 512 TMEM columns for the pair.
__device__ __forceinline__ void rc_setup(const RcLayout& L) {
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int s = 0; s < kRcStages; ++s) {
      ptx::mbar_init(&L.full[s], 2);
      ptx::mbar_init(&L.empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&L.accf[a], 1);
      ptx::mbar_init(&L.acce[a], 2 * kEpiWarps);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc2(L.tmem_slot, 512);
    ptx::tmem_relinquish2();
  }
}

// One k-block on the MMA thread: 4 x (M=256, N=256, K=16) into accumulator `d`.
template <bool BMN>
__device__ __forceinline__ void rc_consume(const RcLayout& L, uint32_t it, uint32_t d, bool acc, const RcTrace& tr) {
  constexpr uint32_t idesc = ptx::idesc_f16_f32_ab(256, 256, false, BMN);
  const int s = it % kRcStages;
  ptx::mbar_wait(&L.full[s], (it / kRcStages) & 1);
  ptx::tc_fence_after();
  tr.blk((int)it, 4);
  const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(L.sA + s * kRcTile));
  const uint32_t sb = ptx::smem_u32(L.sB + s * kRcTile);
  const uint64_t bd = BMN ? ptx::sdesc_mnmajor_sw128(sb) : ptx::sdesc_kmajor_sw128(sb);
  constexpr int bstep = BMN ? (2048 >> 4) : (32 >> 4);
#pragma unroll
  for (int k = 0; k < 4; ++k) ptx::mma_f16_2sm(d, ad + 2 * k, bd + bstep * k, idesc, (acc || k > 0) ? 1u : 0u);
  ptx::mma_commit_2sm_mc(&L.empty[s], 0x3);
}

// Epilogue warp gave back its accumulator columns: one arrive per warp on the leader's barrier.
__device__ __forceinline__ void rc_release_acc(uint64_t* acce_local, bool leader, int lane) {
  ptx::tc_fence_before();
  __syncwarp();
  if (lane == 0) {
    if (leader) ptx::mbar_arrive(acce_local);
    else ptx::mbar_arrive_remote(ptx::mapa_shared(ptx::smem_u32(acce_local), 0));
  }
}

__device__ __forceinline__ void rc_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// After every epilogue thread stored its piece of a chunk: publish `val` (gpu-scope release).
__device__ __forceinline__ void rc_publish(uint32_t* flag, uint32_t val, int tid) {
  rc_bar();
  if (tid == 0) {
    ptx::fence_acq_rel_gpu();
    ptx::st_relaxed_gpu(flag, val);
  }
}

// Split-K exchange of the 128 x 256 fp32 accumulator at TMEM column `col0` among the 4 CTAs
// (z = 0..3, same rank) of one tile: the 3 foreign 64-column slices go to the L2 scratch
// grp_scratch[zsrc][zdst][16 float4 column groups][128 rows], this CTA's flag is published, the
// peers' flags are awaited, and `out` receives this thread's 32 columns [64z + 32grp, +32) of its
// own slice summed over z = 0..3 in order (its own partial straight from TMEM).
__device__ __forceinline__ void rc_reduce(uint32_t tmem, int col0, float4* grp_scratch, int z, int q, int grp,
                                          int lane, int tid, uint32_t* pflags, uint32_t val, uint64_t* acce,
                                          bool leader, float* out, const RcTrace& tr, int trt, int slot0) {
  const int rl = q * 32 + lane;
  const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16) + col0;
#pragma unroll 1
  for (int zd = 0; zd < 4; ++zd) {
    if (zd == z) continue;
    float v[32];
    ptx::tmem_ld16(trow + 64 * zd + 32 * grp, v);
    ptx::tmem_ld16(trow + 64 * zd + 32 * grp + 16, v + 16);
    ptx::tmem_ld_wait();
    float4* dst = grp_scratch + ((z * 4 + zd) * 16 + 8 * grp) * 128 + rl;
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[i * 128] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  }
  if (tid == 0) tr.det(trt, slot0);
  float own[32];
  ptx::tmem_ld16(trow + 64 * z + 32 * grp, own);
  ptx::tmem_ld16(trow + 64 * z + 32 * grp + 16, own + 16);
  ptx::tmem_ld_wait();
  rc_release_acc(acce, leader, lane);
  rc_bar();
  if (tid == 0) {
    tr.det(trt, slot0 + 1);
    ptx::fence_acq_rel_gpu();
    ptx::st_relaxed_gpu(pflags + z, val);
#pragma unroll 1
    for (int zz = 0; zz < 4; ++zz)
      if (zz != z) ptx::spin_until_geq(pflags + zz, val);
    tr.det(trt, slot0 + 2);
  }
  rc_bar();
#pragma unroll
  for (int i = 0; i < 32; ++i) out[i] = 0.f;
#pragma unroll 1
  for (int zz = 0; zz < 4; ++zz) {
    if (zz == z) {
#pragma unroll
      for (int i = 0; i < 32; ++i) out[i] += own[i];
      continue;
    }
    const float4* src = grp_scratch + ((zz * 4 + z) * 16 + 8 * grp) * 128 + rl;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float4 p = __ldcg(src + i * 128);
      out[4 * i] += p.x;
      out[4 * i + 1] += p.y;
      out[4 * i + 2] += p.z;
      out[4 * i + 3] += p.w;
    }
  }
  if (tid == 0) tr.det(trt, slot0 + 3);
}

// Stage 16*NG values of this lane's row (converted to fp16) at w + lane*pitch.
template <int NG>
__device__ __forceinline__ void rc_stage_h(uint8_t* w, int pitch, int lane, const float* v) {
  __half* d = reinterpret_cast<__half*>(w + lane * pitch);
#pragma unroll
  for (int g = 0; g < NG; ++g) st16(d + 16 * g, v + 16 * g);
}

// Producer loop guard: a dependency that makes no progress for ~10 s traps instead of hanging.
__device__ __forceinline__ void rc_watchdog(bool progress, uint64_t& idle_since) {
  if (progress) {
    idle_since = 0;
    return;
  }
  const uint64_t now = ptx::globaltimer();
  if (idle_since == 0) idle_since = now;
  else if (now - idle_since > 10000000000ull) __trap();
}

// Two producers per CTA, so that neither stream waits behind the other's issue overhead.  The
// k-block stream is `pre` prologue blocks followed by `per` blocks per step; `dec(u, i)` maps step u
// (-1 = prologue) and block i to its operands.  Both producers walk it with incremental cursors (no
// divisions on the issue path).
struct RcCursor {
  int u, i, per;
  __device__ __forceinline__ RcCursor(int idx, int pre, int per_) : per(per_) {
    if (idx < pre) {
      u = -1;
      i = idx;
    } else {
      u = (idx - pre) / per;
      i = (idx - pre) - u * per;
    }
  }
  __device__ __forceinline__ void next(int pre) {
    if (u < 0) {
      if (++i == pre) {
        u = 0;
        i = 0;
      }
    } else if (++i == per) {
      i = 0;
      ++u;
    }
  }
};

// Weights (warp 0, lane 0): the weight k-blocks do not depend on the recurrence; each is loaded as
// soon as its ring stage is free (HW-sleeping mbarrier wait), optionally with block wi + pf_dist
// prefetched into L2 at the same time.  (Measured alternative: one thread issuing both operands of
// each stage ran at 0.88 us per F2 k-block against 0.55 us for the two producers here.)
template <class Dec, class IssueW, class PrefW>
__device__ __forceinline__ void rc_weights(const RcLayout& L, int total, int pre, int per, bool leader, int pf_dist,
                                           const RcTrace& tr, Dec dec, IssueW issue_w, PrefW prefetch_w) {
  if (pf_dist > 0) {
    RcCursor pc(0, pre, per);
#pragma unroll 1
    for (int i = 0; i < min(pf_dist, total); ++i, pc.next(pre)) prefetch_w(dec(pc.u, pc.i));
  }
  RcCursor c(0, pre, per), pc(pf_dist, pre, per);
  int s = 0;
  uint32_t ph = 1;
#pragma unroll 1
  for (int wi = 0; wi < total; ++wi, c.next(pre)) {
    if (wi >= kRcStages) ptx::mbar_wait(&L.empty[s], ph);
    const RcBlk b = dec(c.u, c.i);
    if (leader) ptx::mbar_arrive_expect_tx(&L.full[s], 2 * kRcTile);
    issue_w(s, b);
    if (tr.on()) tr.blk(wi, 2);
    if (pf_dist > 0 && wi + pf_dist < total) {
      prefetch_w(dec(pc.u, pc.i));
      pc.next(pre);
    }
    if (++s == kRcStages) {
      s = 0;
      ph ^= 1;
    }
  }
}

// Activations (warp kRcActWarp, all lanes; lane 0 issues): an activation k-block is loaded into its
// stage once the flag of the CTA that produces it says it is published.  Readiness is learned in
// windows, ahead of need: the lanes acquire the flags of the next `flag_lanes` blocks in parallel
// and extend the known-published prefix, lane 0 orders the async proxy after the acquires with one
// fence.proxy.async and then issues every known block on its own (no warp synchronisation per
// block) -- a few L2 round trips per timestep instead of one acquire + one warp barrier per block.
template <class Dec, class IssueA>
__device__ __forceinline__ void rc_acts(const RcLayout& L, int total, int pre, int per, int lane, bool leader,
                                        int flag_lanes, const RcTrace& tr, Dec dec, IssueA issue_a) {
  int ai = 0, known = 0;  // activation blocks [0, known) are published and fenced; [0, ai) issued
  uint64_t idle_since = 0;
  RcCursor c(0, pre, per);
  int s = 0;
  uint32_t ph = 1;
#pragma unroll 1
  while (ai < total) {
    if (known < min(total, ai + kRcStages)) {  // learn readiness of the blocks after `known`
      const int n = min(total - known, flag_lanes);
      bool ready = true;
      if (lane < n) {
        const RcCursor q(known + lane, pre, per);
        const RcBlk b = dec(q.u, q.i);
        if (b.flag) ready = ptx::ld_acquire_gpu(b.flag) >= b.target;
      }
      const unsigned waiting = __ballot_sync(0xffffffffu, !ready);
      const int k = min(waiting ? __ffs(waiting) - 1 : 32, n);
      if (k > 0) {
        __syncwarp();
        if (lane == 0) ptx::fence_proxy_async_global();
        known += k;
      }
      if (lane == 0) rc_watchdog(k > 0 || known > ai, idle_since);
      if (known == ai) continue;
    }
    if (lane == 0) {
#pragma unroll 1
      for (int a = ai; a < known; ++a, c.next(pre)) {
        if (a >= kRcStages) ptx::mbar_wait(&L.empty[s], ph);
        const RcBlk b = dec(c.u, c.i);
        if (leader) ptx::mbar_arrive_expect_tx(&L.full[s], 2 * kRcTile);
        issue_a(s, b);
        if (tr.on()) tr.blk(a, 3);
        if (++s == kRcStages) {
          s = 0;
          ph ^= 1;
        }
      }
    }
    ai = known;
    __syncwarp();
  }
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// =============================================================================================
// Forward: for t = 0..T-1   F1(t): a_t = H_{t-1} W_mh^T (split z of tile n1), m_t = mx_t * a_t
//                            F2(t): z_t = onehot(x_t) (W_x E + b)^T + M_t W_h^T; gates, c, h
// =============================================================================================
__global__ void __launch_bounds__(kRcThreads, 1)
    fwd_recur_kernel(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmM,
                     const __grid_constant__ CUtensorMap tmOH, const __grid_constant__ CUtensorMap tmWmh,
                     const __grid_constant__ CUtensorMap tmWh, const __grid_constant__ CUtensorMap tmXZ, Net<__half> n,
                     float* __restrict__ scratch, uint32_t* __restrict__ flags, RcPolicy pol) {
  extern __shared__ uint8_t smem_raw[];
  const RcLayout L(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = (int)ptx::cluster_ctarank();
  const bool leader = r == 0;
  const int p = blockIdx.x >> 1, P = gridDim.x >> 1;
  const int n1 = p >> 2, z = p & 3;
  const int h = n.h, B = n.B, T = n.T;
  const int nF1 = h / 256, nF2 = h / 64, per = nF1 + 4 + nF2;
  uint32_t* fH = flags;           // [P][2]
  uint32_t* fM = flags + 2 * P;   // [P][2]
  uint32_t* fP = flags + 4 * P;   // [(n1, r)][4]
  __shared__ uint32_t tr_base_s;
  if (threadIdx.x == 0) tr_base_s = rc_trace_reserve(2 * T + kRcTraceBlk);
  rc_setup(L);
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmH);
    ptx::prefetch_tmap(&tmM);
    ptx::prefetch_tmap(&tmOH);
    ptx::prefetch_tmap(&tmWmh);
    ptx::prefetch_tmap(&tmWh);
    ptx::prefetch_tmap(&tmXZ);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *L.tmem_slot;
  const RcTrace tr{tr_base_s, T, kRcTraceStep * per, (pol.exp & 64) ? 0 : per, 3000};

  if (warp == 0 || warp == kRcActWarp) {
    {  // ----------------------------------------------------------- TMA producers (weights, activations)
      const uint64_t pact = ptx::make_policy(pol.act), pw1 = ptx::make_policy(pol.w_split),
                     pw2 = ptx::make_policy(pol.w_wide), pws = ptx::make_policy(pol.w_seg);
      const uint32_t bar0 = ptx::mapa_shared(ptx::smem_u32(&L.full[0]), 0);
      // k-block idx -> (t, kind, chunk): per timestep nF1 H chunks of F1 (K range z), the 4 one-hot
      // segment blocks of F2, then nF2 M chunks of F2 (each stream starts at its own chunk)
      auto dec = [&](int u, int i) {
        RcBlk b;
        b.t = u;
        b.flag = nullptr;
        if (i < nF1) {
          b.kind = 0;
          int jj = i + n1 * pol.rotate;
          if (jj >= nF1) jj -= nF1;
          b.j = z * nF1 + jj;
          if (b.t > 0) {
            b.flag = &fH[2 * b.j + r];
            b.target = (uint32_t)b.t;
          }
        } else if (i < nF1 + 4) {
          b.kind = 1;
          b.j = i - nF1;
        } else {
          b.kind = 2;
          int jj = i - nF1 - 4 + p * pol.rotate;
          if (jj >= nF2) jj -= nF2;
          b.j = jj;
          b.flag = &fM[2 * b.j + r];
          b.target = (uint32_t)(b.t + 1);
        }
        return b;
      };
      auto issue_w = [&](int s, const RcBlk& b) {
        uint8_t* dst = L.sB + s * kRcTile;
        if (b.kind == 0) ptx::tma_load_3d_2sm(dst, &tmWmh, bar0 + 8 * s, 64 * b.j, 256 * n1 + 128 * r, 0, pw1);
        else if (b.kind == 1) ptx::tma_load_3d_2sm(dst, &tmXZ, bar0 + 8 * s, 64 * b.j, 256 * p + 128 * r, 0, pws);
        else ptx::tma_load_3d_2sm(dst, &tmWh, bar0 + 8 * s, 64 * b.j, 256 * p + 128 * r, 0, pw2);
      };
      auto issue_a = [&](int s, const RcBlk& b) {
        uint8_t* dst = L.sA + s * kRcTile;
        if (b.kind == 0) ptx::tma_load_3d_2sm(dst, &tmH, bar0 + 8 * s, 64 * b.j, 128 * r, b.t, pact);
        else if (b.kind == 1) ptx::tma_load_3d_2sm(dst, &tmOH, bar0 + 8 * s, 64 * b.j, 128 * r, b.t, pact);
        else ptx::tma_load_3d_2sm(dst, &tmM, bar0 + 8 * s, 64 * b.j, 128 * r, b.t, pact);
      };
      auto prefetch_w = [&](const RcBlk& b) {
        if (b.kind == 0) ptx::tma_prefetch_3d(&tmWmh, 64 * b.j, 256 * n1 + 128 * r, 0, pw1);
        else if (b.kind == 1) ptx::tma_prefetch_3d(&tmXZ, 64 * b.j, 256 * p + 128 * r, 0, pws);
        else ptx::tma_prefetch_3d(&tmWh, 64 * b.j, 256 * p + 128 * r, 0, pw2);
      };
      if (warp == 0) {
        if (lane == 0)
          rc_weights(L, T * per, 0, per, leader, pol.pf_dist, tr, dec, issue_w, prefetch_w);
      } else {
        rc_acts(L, T * per, 0, per, lane, leader, pol.flag_lanes, tr, dec, issue_a);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ------------------------------------------------- MMA issuer
      uint32_t it = 0;
#pragma unroll 1
      for (int t = 0; t < T; ++t) {
        if (t > 0) {
          ptx::mbar_wait(&L.acce[0], (t - 1) & 1);
          ptx::tc_fence_after();
        }
        tr.step(t, 2);
#pragma unroll 1
        for (int i = 0; i < nF1; ++i) {
          rc_consume<false>(L, it++, tmem, i > 0, tr);
          if (i == 0) tr.step(t, 3);
        }
        ptx::mma_commit_2sm_mc(&L.accf[0], 0x3);
        tr.step(t, 4);
        if (t > 0) {
          ptx::mbar_wait(&L.acce[1], (t - 1) & 1);
          ptx::tc_fence_after();
        }
#pragma unroll 1
        for (int i = 0; i < 4 + nF2; ++i) {
          rc_consume<false>(L, it++, tmem + 256, i > 0, tr);
          if (i == 4) tr.step(t, 5);
        }
        ptx::mma_commit_2sm_mc(&L.accf[1], 0x3);
        tr.step(t, 6);
      }
    }
  } else {  // ---------------------------------------------------------------- epilogue warps
    const int q = warp & 3, grp = (warp - 2) >> 2, tid = threadIdx.x - 64;
    const int rl = q * 32 + lane, b = 128 * r + rl, b0 = 128 * r + 32 * q;
    uint8_t* w = L.win + (warp - 2) * kRcWin;
    const long region = (long)(h / 256) * 2 * kRcGroupF4;  // one (kind, parity) region
    float4* gscr = reinterpret_cast<float4*>(scratch) + (long)(n1 * 2 + r) * kRcGroupF4;
    const int u1 = 64 * p + 32 * grp;  // F1 units of this thread: [u1, u1 + 32)
    // F2 units of this thread: chunks c = grp, grp + 2 of the pair's 64 units, 16 each
    float cst[32];  // cell state c_{t-1} of those units (fp32, lives in registers for all T)
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) ld16(n.Crm + (long)b * h + 64 * p + 16 * (grp + 2 * cc), cst + 16 * cc);
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      const int byte = n.byte_at(b, t);
      // ---------------------------------------------- F1 epilogue: split-K reduce, m = mx * a
      const float* mxp = n.tab + (long)byte * 5 * h + u1;
      // this thread's 32 mx values land in its slot of the staging window while the split-K partials
      // are exchanged (off the critical path; the m staging below uses the window's first half)
      float* mxs = reinterpret_cast<float*>(w + 4096 + lane * 128);
#pragma unroll
      for (int k = 0; k < 8; ++k) ptx::cp_async16(mxs + 4 * k, mxp + 4 * k);
      ptx::mbar_wait(&L.accf[0], t & 1);
      ptx::tc_fence_after();
      if (tid == 0) {
        tr.step_tag(t, 1000 + t);
        tr.step(t, 7);
      }
      float a[32];
      rc_reduce(tmem, 0, gscr + (t & 1) * region, z, q, grp, lane, tid, fP + (n1 * 2 + r) * 4, (uint32_t)(t + 1),
                &L.acce[0], leader, a, tr, t, 2);
      if (tid == 0) tr.step(t, 8);
      {
        float m[32];
        ptx::cp_async_wait_all();
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float x[16];
          ld16(mxs + 16 * g, x);
#pragma unroll
          for (int i = 0; i < 16; ++i) m[16 * g + i] = x[i] * a[16 * g + i];
        }
        rc_stage_h<2>(w, 80, lane, m);
        warp_rows_out(reinterpret_cast<uint8_t*>(n.Mrm + ((long)t * B + b0) * h + u1), 2L * h, w, 80, 64, 32, lane);
        __syncwarp();
      }
      rc_publish(&fM[2 * p + r], (uint32_t)(t + 1), tid);
      if (tid == 0) tr.step(t, 9);
      rc_stage_h<2>(w, 80, lane, a);
      warp_rows_out(reinterpret_cast<uint8_t*>(n.Astash + ((long)t * B + b0) * h + u1), 2L * h, w, 80, 64, 32, lane);
      __syncwarp();
      // ---------------------------------------------- F2 epilogue: gates, cell update, hidden state
      ptx::mbar_wait(&L.accf[1], t & 1);
      ptx::tc_fence_after();
      if (tid == 0) tr.step(t, 10);
      uint32_t gpk[2][32];  // fp16 gate pairs of both chunks (stored after h is published)
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        float v[64];
        const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + 256 + 64 * (grp + 2 * cc);
        ptx::tmem_ld16(ta, v);
        ptx::tmem_ld16(ta + 16, v + 16);
        ptx::tmem_ld16(ta + 32, v + 32);
        ptx::tmem_ld16(ta + 48, v + 48);
        ptx::tmem_ld_wait();
        float hv[16];
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const float gi = act_sigmoid<__half>(v[jj]), gf = act_sigmoid<__half>(v[16 + jj]);
          const float go = act_sigmoid<__half>(v[32 + jj]), gu = act_tanh<__half>(v[48 + jj]);
          v[jj] = gi;
          v[16 + jj] = gf;
          v[32 + jj] = go;
          v[48 + jj] = gu;
          const float cn = gf * cst[16 * cc + jj] + gi * gu;  // c_t = f c_{t-1} + i u   (fp32)
          cst[16 * cc + jj] = cn;
          hv[jj] = go * act_tanh<__half>(cn);  // h_t = o tanh(c_t)
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          __half2 hh = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
          gpk[cc][i] = *reinterpret_cast<uint32_t*>(&hh);
        }
        rc_stage_h<1>(w + cc * 1536, 48, lane, hv);
      }
      rc_release_acc(&L.acce[1], leader, lane);
      if (tid == 0) tr.det(t, 6);
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
        warp_rows_out(reinterpret_cast<uint8_t*>(n.Hrm + ((long)(t + 1) * B + b0) * h + 64 * p + 16 * (grp + 2 * cc)),
                      2L * h, w + cc * 1536, 48, 32, 32, lane);
      if (tid == 0) tr.det(t, 7);
      rc_publish(&fH[2 * p + r], (uint32_t)(t + 1), tid);
      if (tid == 0) tr.step(t, 11);
      // stashes for BPTT: gates (internal order) and c_t
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int c = grp + 2 * cc;
        __syncwarp();
        uint4* gs = reinterpret_cast<uint4*>(w + 3072 + lane * 144);
#pragma unroll
        for (int k = 0; k < 8; ++k) gs[k] = make_uint4(gpk[cc][4 * k], gpk[cc][4 * k + 1], gpk[cc][4 * k + 2], gpk[cc][4 * k + 3]);
        warp_rows_out(reinterpret_cast<uint8_t*>(n.Gates + ((long)t * B + b0) * 4 * h + 256 * p + 64 * c), 8L * h,
                      w + 3072, 144, 128, 32, lane);
        __syncwarp();
        st16(reinterpret_cast<float*>(w + 3072 + lane * 80), cst + 16 * cc);
        warp_rows_out(reinterpret_cast<uint8_t*>(n.Crm + ((long)(t + 1) * B + b0) * h + 64 * p + 16 * c), 4L * h,
                      w + 3072, 80, 64, 32, lane);
      }
      __syncwarp();
      if (tid == 0) tr.det(t, 8);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, 512);
  }
}

// =============================================================================================
// Backward (TBTT over the window): prologue B2(T): dH_{T-1} = dY_{T-1} W_dec -> gate backward
// of step T-1; then for t = T-1..0:
//   B1(t): dM_t = dZ_t W_h (split z of tile n1, K = 4h)  ->  dA_t = dM * mx_t, dMX_t = dM * a_t
//   B2(t), t >= 1: dH_{t-1} = dY_{t-1} W_dec + dA_t W_mh  ->  gate backward of step t-1 (dZ_{t-1}, dc)
// Weights are read MN-major straight from the row-major working copies (no transposed copies).
// Flag values: dZ_s -> T - s, dA_t -> T - t, B1(t) partials -> T - t, B2(t) partials -> T - t + 1.
// =============================================================================================
// WKM: the weights come K-major from the transposed working copies (one 128-row TMA box per stage)
// instead of MN-major from the row-major ones (two 64 x 64 boxes per stage; no transposes needed).
template <bool WKM>
__global__ void __launch_bounds__(kRcThreads, 1)
    bwd_recur_kernel(const __grid_constant__ CUtensorMap tmDZ, const __grid_constant__ CUtensorMap tmDA,
                     const __grid_constant__ CUtensorMap tmDY, const __grid_constant__ CUtensorMap tmWh,
                     const __grid_constant__ CUtensorMap tmWmh, const __grid_constant__ CUtensorMap tmWdec,
                     Net<__half> n, float* __restrict__ scratch, uint32_t* __restrict__ flags, RcPolicy pol) {
  extern __shared__ uint8_t smem_raw[];
  const RcLayout L(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = (int)ptx::cluster_ctarank();
  const bool leader = r == 0;
  const int p = blockIdx.x >> 1, P = gridDim.x >> 1;
  const int n1 = p >> 2, z = p & 3;
  const int h = n.h, B = n.B, T = n.T;
  const int nB1 = h / 64, nB2 = h / 256, per = nB1 + 1 + nB2;
  uint32_t* fA = flags + 2 * P;   // [P][2]  dA_t chunk p
  uint32_t* fP1 = flags + 4 * P;  // [(n1, r)][4]
  uint32_t* fP2 = flags + 6 * P;  // [(n1, r)][4]
  uint32_t* fZc = flags + 8 * P;  // [(p, r)][4 chunks]
  __shared__ uint32_t tr_base_s;
  if (threadIdx.x == 0) tr_base_s = rc_trace_reserve(2 * T + kRcTraceBlk);
  rc_setup(L);
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmDZ);
    ptx::prefetch_tmap(&tmDA);
    ptx::prefetch_tmap(&tmDY);
    ptx::prefetch_tmap(&tmWh);
    ptx::prefetch_tmap(&tmWmh);
    ptx::prefetch_tmap(&tmWdec);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *L.tmem_slot;
  const RcTrace tr{tr_base_s, T, 1 + kRcTraceStep * per, (pol.exp & 64) ? 0 : per, 4000};
  const int total = 1 + T * per - (1 + nB2);  // no B2(0)

  if (warp == 0 || warp == kRcActWarp) {
    {  // ----------------------------------------------------------- TMA producers (weights, activations)
      const uint64_t pact = ptx::make_policy(pol.act), pw1 = ptx::make_policy(pol.w_split),
                     pw2 = ptx::make_policy(pol.w_wide), pws = ptx::make_policy(pol.w_seg);
      const uint32_t bar0 = ptx::mapa_shared(ptx::smem_u32(&L.full[0]), 0);
      // idx -> (t, kind, chunk): kind 0 = B1 dZ chunk, 1 = B2 segment dY_{t-1}, 2 = B2 dA chunk
      auto dec = [&](int u, int i) {
        RcBlk b;
        b.flag = nullptr;
        if (u < 0) {  // prologue B2(T): the dY_{T-1} W_dec segment only
          b.t = T;
          b.kind = 1;
          b.j = z;
          return b;
        }
        b.t = T - 1 - u;
        if (i < nB1) {
          // the K range's 64-column dZ chunks: first the ones each producer publishes first (its c = 0, 2
          // chunks, written by the first pass of the gate backward), then the c = 1, 3 ones
          b.kind = 0;
          const int half = i >= (nB1 >> 1), ii = i - half * (nB1 >> 1);
          int pp = (ii >> 1) + n1 * pol.rotate;  // producer pair within the K range (nB1 / 4 of them)
          if (pp >= (nB1 >> 2)) pp -= nB1 >> 2;
          b.j = z * nB1 + 4 * pp + 2 * (ii & 1) + half;
          b.flag = &fZc[((b.j >> 2) * 2 + r) * 4 + (b.j & 3)];
          b.target = (uint32_t)(T - b.t);
        } else if (i == nB1) {
          b.kind = 1;
          b.j = z;
        } else {
          b.kind = 2;
          int jj = i - nB1 - 1 + n1 * pol.rotate;
          if (jj >= nB2) jj -= nB2;
          b.j = z * nB2 + jj;
          b.flag = &fA[2 * b.j + r];
          b.target = (uint32_t)(T - b.t);
        }
        return b;
      };
      auto issue_w = [&](int s, const RcBlk& b) {
        uint8_t* dst = L.sB + s * kRcTile;
        const int u0 = 256 * n1 + 128 * r;  // this CTA's 128 output units
        const CUtensorMap* tm = b.kind == 0 ? &tmWh : (b.kind == 1 ? &tmWdec : &tmWmh);
        const uint64_t pw = b.kind == 0 ? pw2 : (b.kind == 1 ? pws : pw1);
        if constexpr (WKM) {
          ptx::tma_load_3d_2sm(dst, tm, bar0 + 8 * s, 64 * b.j, u0, 0, pw);
        } else {  // MN-major boxes of 64 units
#pragma unroll
          for (int i = 0; i < 2; ++i) ptx::tma_load_3d_2sm(dst + i * 8192, tm, bar0 + 8 * s, u0 + 64 * i, 64 * b.j, 0, pw);
        }
      };
      auto issue_a = [&](int s, const RcBlk& b) {
        uint8_t* dst = L.sA + s * kRcTile;
        if (b.kind == 0) ptx::tma_load_3d_2sm(dst, &tmDZ, bar0 + 8 * s, 64 * b.j, 128 * r, b.t, pact);
        else if (b.kind == 1) ptx::tma_load_3d_2sm(dst, &tmDY, bar0 + 8 * s, 64 * b.j, 128 * r, b.t - 1, pact);
        else ptx::tma_load_3d_2sm(dst, &tmDA, bar0 + 8 * s, 64 * b.j, 128 * r, b.t, pact);
      };
      auto prefetch_w = [&](const RcBlk& b) {
        const int u0 = 256 * n1 + 128 * r;
        const CUtensorMap* tm = b.kind == 0 ? &tmWh : (b.kind == 1 ? &tmWdec : &tmWmh);
        const uint64_t pw = b.kind == 0 ? pw2 : (b.kind == 1 ? pws : pw1);
        if constexpr (WKM) {
          ptx::tma_prefetch_3d(tm, 64 * b.j, u0, 0, pw);
        } else {
#pragma unroll
          for (int i = 0; i < 2; ++i) ptx::tma_prefetch_3d(tm, u0 + 64 * i, 64 * b.j, 0, pw);
        }
      };
      if (warp == 0) {
        if (lane == 0) rc_weights(L, total, 1, per, leader, pol.pf_dist, tr, dec, issue_w, prefetch_w);
      } else {
        rc_acts(L, total, 1, per, lane, leader, pol.flag_lanes, tr, dec, issue_a);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ------------------------------------------------- MMA issuer
      uint32_t it = 0;
      rc_consume<!WKM>(L, it++, tmem + 256, false, tr);  // B2(T): dY_{T-1} W_dec
      ptx::mma_commit_2sm_mc(&L.accf[1], 0x3);
#pragma unroll 1
      for (int u = 0; u < T; ++u) {
        const int t = T - 1 - u;
        if (u > 0) {
          ptx::mbar_wait(&L.acce[0], (u - 1) & 1);
          ptx::tc_fence_after();
        }
        tr.step(u, 2);
#pragma unroll 1
        for (int i = 0; i < nB1; ++i) {
          rc_consume<!WKM>(L, it++, tmem, i > 0, tr);
          if (i == 0) tr.step(u, 3);
        }
        ptx::mma_commit_2sm_mc(&L.accf[0], 0x3);
        tr.step(u, 4);
        if (t == 0) break;
        ptx::mbar_wait(&L.acce[1], u & 1);  // use u of the wide accumulator (use 0 = prologue)
        ptx::tc_fence_after();
#pragma unroll 1
        for (int i = 0; i < 1 + nB2; ++i) {
          rc_consume<!WKM>(L, it++, tmem + 256, i > 0, tr);
          if (i == 1) tr.step(u, 5);
        }
        ptx::mma_commit_2sm_mc(&L.accf[1], 0x3);
        tr.step(u, 6);
      }
    }
  } else {  // ---------------------------------------------------------------- epilogue warps
    const int q = warp & 3, grp = (warp - 2) >> 2, tid = threadIdx.x - 64;
    const int rl = q * 32 + lane, b = 128 * r + rl, b0 = 128 * r + 32 * q;
    uint8_t* w = L.win + (warp - 2) * kRcWin;
    const long region = (long)(h / 256) * 2 * kRcGroupF4;  // one (kind, parity) region
    float4* gscr1 = reinterpret_cast<float4*>(scratch) + (long)(n1 * 2 + r) * kRcGroupF4;
    float4* gscr2 = gscr1 + 2 * region;
    const int u1 = 64 * p + 32 * grp;  // this thread's 32 units in both reductions
    float dcs[32];                     // dc carry (TBTT: zero at the window end)
#pragma unroll
    for (int i = 0; i < 32; ++i) dcs[i] = 0.f;
    // B2(t) epilogue: dH of step s = t - 1 -> gate backward -> dZ_s, dc
    float ccar[32];  // c_s of the next gate backward: this one's c_{s-1}, carried in registers
    auto b2_epi = [&](int t, int use) {
      const int s = t - 1;
      const long BH = (long)B * h;
      const __half* gates = n.Gates + ((long)s * B + b) * 4 * h + (u1 >> 4) * 64;
      const float* cs = n.Crm + (long)(s + 1) * BH + (long)b * h + u1;
      const float* cp = n.Crm + (long)s * BH + (long)b * h + u1;
      prefetch_l2(gates);
      prefetch_l2(gates + 64);
      if (t == T) prefetch_l2(cs);
      prefetch_l2(cp);
      ptx::mbar_wait(&L.accf[1], use & 1);
      ptx::tc_fence_after();
      if (tid == 0 && t < T) tr.step(T - 1 - t, 10);
      float dh[32];
      rc_reduce(tmem, 256, gscr2 + (t & 1) * region, z, q, grp, lane, tid, fP2 + (n1 * 2 + r) * 4,
                (uint32_t)(T - t + 1), &L.acce[1], leader, dh, tr, t < T ? T - 1 - t : -1, 6);
      if (t == T) {
        ld16(cs, ccar);
        ld16(cs + 16, ccar + 16);
      }
#pragma unroll
      for (int g = 0; g < 2; ++g) {  // two groups of 16 units = two 64-column internal chunks
        float gi[16], gf[16], go[16], gu[16], cpv[16];
        ld16(gates + 64 * g, gi);
        ld16(gates + 64 * g + 16, gf);
        ld16(gates + 64 * g + 32, go);
        ld16(gates + 64 * g + 48, gu);
        ld16(cp + 16 * g, cpv);
        float dz[64];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float kk = act_tanh<__half>(ccar[16 * g + k]);
          const float i = gi[k], f = gf[k], o = go[k], u = gu[k], d = dh[16 * g + k];
          dz[32 + k] = d * kk * o * (1.f - o);                    // dZ_o
          const float dc = dcs[16 * g + k] + d * o * (1.f - kk * kk);
          dz[k] = dc * u * i * (1.f - i);                         // dZ_i
          dz[16 + k] = dc * cpv[k] * f * (1.f - f);               // dZ_f
          dz[48 + k] = dc * i * (1.f - u * u);                    // dZ_u
          dcs[16 * g + k] = dc * f;                               // dc carry to step s-1
          ccar[16 * g + k] = cpv[k];                              // c_{s-1} is the next step's c_s
        }
        if (tid == 0 && t < T && g == 0) tr.det(T - 1 - t, 11);
        rc_stage_h<4>(w, 144, lane, dz);
        warp_rows_out(reinterpret_cast<uint8_t*>(n.G5 + ((long)s * B + b0) * 5 * h + h + (u1 >> 4) * 64 + 64 * g),
                      10L * h, w, 144, 128, 32, lane);
        __syncwarp();
        // chunk c = 2 grp + g (all 128 rows of this rank) is complete once the four warps of this
        // group stored it: publish it on its own flag (B1 of the next timestep may start on it)
        asm volatile("bar.sync %0, 128;" ::"r"(2 + grp) : "memory");
        if (warp == 2 + 4 * grp && lane == 0) {
          ptx::fence_acq_rel_gpu();
          ptx::st_relaxed_gpu(&fZc[(p * 2 + r) * 4 + 2 * grp + g], (uint32_t)(T - s));
        }
      }
      if (tid == 0 && t < T) {
        tr.det(T - 1 - t, 10);
        tr.step(T - 1 - t, 11);
      }
    };
    b2_epi(T, 0);
#pragma unroll 1
    for (int u = 0; u < T; ++u) {
      const int t = T - 1 - u;
      // ---------------------------------------------- B1 epilogue: dA = dM * mx, dMX = dM * a
      const int byte = n.byte_at(b, t);
      const float* mxp = n.tab + (long)byte * 5 * h + u1;
      const __half* ap = n.Astash + ((long)t * B + b) * h + u1;
      // mx (32 fp32) and a (32 fp16) of this thread land in the window during the exchange
      float* mxs = reinterpret_cast<float*>(w + lane * 128);
      __half* as_ = reinterpret_cast<__half*>(w + 32 * 128 + lane * 64);
#pragma unroll
      for (int k = 0; k < 8; ++k) ptx::cp_async16(mxs + 4 * k, mxp + 4 * k);
#pragma unroll
      for (int k = 0; k < 4; ++k) ptx::cp_async16(as_ + 8 * k, ap + 8 * k);
      ptx::mbar_wait(&L.accf[0], u & 1);
      ptx::tc_fence_after();
      if (tid == 0) {
        tr.step_tag(u, 2000 + u);
        tr.step(u, 7);
      }
      float dm[32];
      rc_reduce(tmem, 0, gscr1 + (t & 1) * region, z, q, grp, lane, tid, fP1 + (n1 * 2 + r) * 4, (uint32_t)(T - t),
                &L.acce[0], leader, dm, tr, u, 2);
      if (tid == 0) tr.step(u, 8);
      {
        float da[32], dmx[32];
        ptx::cp_async_wait_all();
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float x[16], av[16];
          ld16(mxs + 16 * g, x);
          ld16(as_ + 16 * g, av);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            da[16 * g + i] = dm[16 * g + i] * x[i];
            dmx[16 * g + i] = dm[16 * g + i] * av[i];
          }
        }
        __syncwarp();  // every lane has read its mx / a slot before the staging below overwrites them
        rc_stage_h<2>(w, 80, lane, da);
        warp_rows_out(reinterpret_cast<uint8_t*>(n.dA + ((long)t * B + b0) * h + u1), 2L * h, w, 80, 64, 32, lane);
        __syncwarp();
        if (t > 0) rc_publish(&fA[2 * p + r], (uint32_t)(T - t), tid);
        if (tid == 0) tr.step(u, 9);
        rc_stage_h<2>(w, 80, lane, dmx);
        warp_rows_out(reinterpret_cast<uint8_t*>(n.G5 + ((long)t * B + b0) * 5 * h + u1), 10L * h, w, 80, 64, 32,
                      lane);
        __syncwarp();
      }
      if (t > 0) b2_epi(t, u + 1);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, 512);
  }
}

}  // namespace mlstm
