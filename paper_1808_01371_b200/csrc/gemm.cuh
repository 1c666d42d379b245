// gemm.cuh -- the GEMM engines every contraction of the step runs on.
//
//   D[M x N] = A[M x K] . B[N x K]^T   (both operands K-major, i.e. row-major with K contiguous),
//   fp32 accumulation, result handed to a fused epilogue functor 16*NG columns at a time:
//       epi.run<NG>(row, col0, v)   with v[i] = D[row][col0 + i], i < 16*NG.
//
// tcgen05 engines (mixed precision, fp16 operands).  Warp roles: warp 0 TMA producer, warp 1 TMEM
// allocator + single-thread MMA issuer, warps 2..9 epilogue (two warps per TMEM lane quarter, so
// the memory-heavy fused epilogues -- on the recurrence's critical path -- get 8 warps).
//   * gemm_tc_kernel   one CTA per 128 x BN tile (M=128 tcgen05.mma).
//   * gemm_tc2_kernel  a CTA pair (cluster of 2, cta_group::2) per 256 x BN tile: each CTA stages
//                      its 128 rows of A and BN/2 rows of B, halving per-SM operand traffic.
//   * gemm_tc1s_kernel one CTA per 128 x 256 tile with the K loop split S ways over a cluster of S
//                      CTAs, reduced in-kernel through an L2 scratch in fixed order.
//   Pipeline: TMA (128B swizzle) -> STAGES-deep mbarrier ring -> MMA into a TMEM fp32 accumulator
//   -> tcgen05.ld by the epilogue warps.  Measured engine choice: profiles/r01_gemm_sweep.log.
// SIMT engine (fp32 parity mode, "single precision"): plain FFMA, 128 x 64 tile.
#pragma once
#include "net.cuh"
#include "ptx.cuh"

namespace mlstm {

constexpr int kEpiWarps = 8;
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;
constexpr int kGemmStaticB = 1;  // B operand is a weight untouched by the preceding kernels
constexpr int kGemmRasterM = 2;  // launch order M-fastest (CTAs running together share a B tile)
constexpr int kGemmRasterG = 4;  // grouped raster: bands of 8 M-tiles, N-fastest inside a band (L2 reuse
                                 // of both operands across the CTAs resident together)

// ---- optional intra-kernel timeline (mlstm_trace_enable): one record per CTA,
// {tag, cta, t_start, t_first_tma, t_first_full, t_acc_ready, t_reduced, t_end} in ns.
struct TraceRec {
  uint64_t v[12];
};
__device__ TraceRec* g_trace = nullptr;
__device__ unsigned int g_trace_n = 0;
__device__ unsigned int g_trace_cap = 0;
__device__ __forceinline__ void trace_flush(const uint64_t* ts, int tag) {
  TraceRec* tr = g_trace;
  if (!tr) return;
  const unsigned int i = atomicAdd(&g_trace_n, 1u);
  if (i >= g_trace_cap) return;
  TraceRec r;
  r.v[0] = (uint64_t)tag;
  r.v[1] = blockIdx.x + (uint64_t)gridDim.x * (blockIdx.y + (uint64_t)gridDim.y * blockIdx.z);
  for (int k = 0; k < 10; ++k) r.v[2 + k] = ts[k];
  tr[i] = r;
}
template <class Epi>
struct EpiTag {
  static constexpr int value = 0;
};
template <class E, class = void>
struct HasTile {  // epilogue with a cooperative tile() form (used by the split-K engine)
  static constexpr bool value = false;
};
template <class E>
struct HasTile<E, decltype(void(E::kTile))> {
  static constexpr bool value = E::kTile;
};

template <class E, class = void>
struct HasPreC {  // row-I/O epilogue whose per-row input can be loaded into registers before the accumulator
  static constexpr bool value = false;
};
template <class E>
struct HasPreC<E, decltype(void(E::kPreC))> {
  static constexpr bool value = E::kPreC;
};

template <class E, class = void>
struct HasAsyncIO {
  static constexpr bool value = false;
};
template <class E>
struct HasAsyncIO<E, decltype(void(E::kAsyncIO))> {
  static constexpr bool value = E::kAsyncIO;
};

template <int BN>
struct TcCfg {  // one CTA per 128 x BN tile
  static constexpr int BM = 128, BK = 64, BNT = BN;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 512;
  static_assert(STAGES * STAGE_BYTES >= kEpiWarps * kWarpStageBytes, "epilogue staging windows");
};
#ifndef MLSTM_F2_PREC
#define MLSTM_F2_PREC 1  // F2 epilogue: c_{t-1} into registers during the main loop (0: bulk copy after it)
#endif
#ifndef MLSTM_TC2_STAGES256
#define MLSTM_TC2_STAGES256 6  // ring depth of the 256 x 256 CTA-pair tiles (A/B builds override)
#endif
template <int BN>
struct Tc2Cfg {  // CTA pair per 256 x BN tile: per CTA 128 rows of A, BN/2 rows of B
  // BN = 512: two N = 256 MMAs per k-step into TMEM columns [0,256) and [256,512); each CTA holds
  // the two 128-row B blocks of its rank ([r*128, +128) of each 256-wide half)
  static constexpr int BM = 128, BK = 64, BNT = BN;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 512 ? 4 : BN == 256 ? MLSTM_TC2_STAGES256 : (BN == 128 ? 8 : 10);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 512;
  static_assert(STAGES * STAGE_BYTES >= kEpiWarps * kWarpStageBytes, "epilogue staging windows");
};

// Shared-memory carve-up common to the tcgen05 kernels.
template <class C>
struct SmemLayout {
  uint8_t *sA, *sB;
  uint64_t *full, *empty, *accf, *epibar;
  uint32_t* tmem_slot;
  __device__ __forceinline__ explicit SmemLayout(uint8_t* smem_raw) {
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    sA = smem;
    sB = smem + C::STAGES * C::A_BYTES;
    full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
    empty = full + C::STAGES;
    accf = empty + C::STAGES;
    tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
    epibar = accf + 2;  // kEpiWarps epilogue load barriers
  }
  __device__ __forceinline__ EpiIO io(int ew, int row0, int M, int lane) const {
    return EpiIO{sA + ew * kWarpStageBytes, epibar + ew, row0, max(0, min(32, M - row0)), lane};
  }
};

// Barrier init (thread 0), TMEM allocation (warp 1) and descriptor prefetch (warp 0).
template <class C, bool PAIR>
__device__ __forceinline__ void gemm_setup(const SmemLayout<C>& L, const CUtensorMap* tmA, const CUtensorMap* tmB,
                                           int ncols) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&L.full[s], 1);   // one arrive.expect_tx per phase (the pair leader's in PAIR mode)
      ptx::mbar_init(&L.empty[s], 1);  // the MMA commit (multicast to both CTAs in PAIR mode)
    }
    ptx::mbar_init(L.accf, 1);
#pragma unroll 1
    for (int w = 0; w < kEpiWarps; ++w) ptx::mbar_init(&L.epibar[w], 32);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    if (PAIR) {
      ptx::tmem_alloc2(L.tmem_slot, ncols);
      ptx::tmem_relinquish2();
    } else {
      ptx::tmem_alloc(L.tmem_slot, ncols);
      ptx::tmem_relinquish();
    }
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(tmA);
    ptx::prefetch_tmap(tmB);
  }
}

// TMA producer (one thread).  With kGemmStaticB the B operand (a weight) does not depend on the
// preceding kernel: its first stages are fetched before the grid-dependency wait (overlapping the
// previous kernel's tail under programmatic dependent launch); the A operand after it.
// PAIR: both CTAs load their halves and count bytes on the leader's barrier (bar_leader0 = its
// full[0] in shared::cluster space); only the leader arrives, with both CTAs' byte count -- the
// peer's bytes may land first (transiently negative tx-count); the peer cannot run a phase ahead
// because it waits on its own empty barrier, released by the same multicast commit.  (A
// release.cluster remote arrive here would fence every prior TMA and serialise the pipeline.)
// K runs over two segments: k-blocks [0, kb_seg0) from (A, B), then from (A2, B2) -- used to fold
// a one-hot x table product (input projection + bias) into the recurrent GEMM's accumulator.
struct Seg2 {
  int kb_seg0;  // k-blocks of the first segment
  int az2, bz2;
};

// MN (operand majors): 0 = both K-major; 1 = both MN-major ([K][M] / [K][N] in memory, the
// weight-gradient GEMMs D = A^T B over a long K = T*B): each stage is one 64-row K block loaded as
// 64-wide MN boxes; 2 = K-major A, MN-major B (the backward recurrence reading the row-major weight
// working copies directly, no transposed copies).
__host__ __device__ constexpr bool a_mn(int mn) { return mn == 1; }
__host__ __device__ constexpr bool b_mn(int mn) { return mn != 0; }
template <class C, bool PAIR, int MN = 0>
__device__ __forceinline__ void gemm_produce(const SmemLayout<C>& L, const CUtensorMap* tmA, const CUtensorMap* tmB,
                                             const CUtensorMap* tmA2, const CUtensorMap* tmB2, Seg2 sg, int nkb,
                                             int kb0, int m0, int nb0, int az, int bz, uint32_t polA,
                                             uint32_t polB, int flags, bool leader, uint32_t bar_leader0,
                                             uint64_t* trace_slot, int part = 0) {
  // part 0: everything; part 1: only the static-B stages (issued by the barrier-initialising thread
  // before the CTA-wide setup barrier, so the weight stream starts while TMEM is being allocated);
  // part 2: everything but those stages.
  const uint64_t pa = ptx::make_policy(polA), pb = ptx::make_policy(polB);
  const uint32_t tx = PAIR ? 2 * C::STAGE_BYTES : C::STAGE_BYTES;
  auto loadA = [&](int s, int kb) {
    if constexpr (a_mn(MN)) {
#pragma unroll
      for (int i = 0; i < C::BM / 64; ++i) {
        uint8_t* dst = L.sA + s * C::A_BYTES + i * 8192;
        if (PAIR) ptx::tma_load_3d_2sm(dst, tmA, bar_leader0 + s * 8, m0 + 64 * i, kb * C::BK, az, pa);
        else ptx::tma_load_3d(dst, tmA, &L.full[s], m0 + 64 * i, kb * C::BK, az, pa);
      }
      return;
    }
    const bool s2 = kb >= sg.kb_seg0;
    const CUtensorMap* m = s2 ? tmA2 : tmA;
    const int k = (s2 ? kb - sg.kb_seg0 : kb) * C::BK, z = s2 ? sg.az2 : az;
    if (PAIR) ptx::tma_load_3d_2sm(L.sA + s * C::A_BYTES, m, bar_leader0 + s * 8, k, m0, z, pa);
    else ptx::tma_load_3d(L.sA + s * C::A_BYTES, m, &L.full[s], k, m0, z, pa);
  };
  auto loadB = [&](int s, int kb) {
    if constexpr (b_mn(MN)) {
      static_assert(C::B_BYTES % 8192 == 0, "MN-major B needs 64-wide boxes per CTA");
      const bool s2 = kb >= sg.kb_seg0;  // second K segment (MN == 2 only; never for MN == 1)
      const CUtensorMap* m = s2 ? tmB2 : tmB;
      const int k = (s2 ? kb - sg.kb_seg0 : kb) * C::BK, z = s2 ? sg.bz2 : bz;
#pragma unroll
      for (int i = 0; i < C::B_BYTES / 8192; ++i) {
        uint8_t* dst = L.sB + s * C::B_BYTES + i * 8192;
        const int col = C::BNT == 512 ? nb0 + (i >> 1) * 256 + (i & 1) * 64 : nb0 + 64 * i;
        if (PAIR) ptx::tma_load_3d_2sm(dst, m, bar_leader0 + s * 8, col, k, z, pb);
        else ptx::tma_load_3d(dst, m, &L.full[s], col, k, z, pb);
      }
      return;
    }
    if constexpr (C::BNT == 512) {  // two 128-row boxes, N offsets 0 and 256 (no second segment)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        uint8_t* dst = L.sB + s * C::B_BYTES + i * 16384;
        if (PAIR) ptx::tma_load_3d_2sm(dst, tmB, bar_leader0 + s * 8, kb * C::BK, nb0 + 256 * i, bz, pb);
        else ptx::tma_load_3d(dst, tmB, &L.full[s], kb * C::BK, nb0 + 256 * i, bz, pb);
      }
      return;
    }
    const bool s2 = kb >= sg.kb_seg0;
    const CUtensorMap* m = s2 ? tmB2 : tmB;
    const int k = (s2 ? kb - sg.kb_seg0 : kb) * C::BK, z = s2 ? sg.bz2 : bz;
    if (PAIR) ptx::tma_load_3d_2sm(L.sB + s * C::B_BYTES, m, bar_leader0 + s * 8, k, nb0, z, pb);
    else ptx::tma_load_3d(L.sB + s * C::B_BYTES, m, &L.full[s], k, nb0, z, pb);
  };
  const int pre = (flags & kGemmStaticB) ? min(C::STAGES, nkb) : 0;
  if (part != 2)
    for (int i = 0; i < pre; ++i) {
      if (leader) ptx::mbar_arrive_expect_tx(&L.full[i], tx);
      loadB(i, kb0 + i);
    }
  if (part == 1) return;
  ptx::pdl_wait();
  if (trace_slot) *trace_slot = ptx::globaltimer();
  for (int i = 0; i < pre; ++i) loadA(i, kb0 + i);
#pragma unroll 1
  for (int i = pre; i < nkb; ++i) {
    const int s = i % C::STAGES;
    const uint32_t ph = (i / C::STAGES) & 1;
    ptx::mbar_wait(&L.empty[s], ph ^ 1);
    if (leader) ptx::mbar_arrive_expect_tx(&L.full[s], tx);
    loadA(s, kb0 + i);
    loadB(s, kb0 + i);
  }
}

// MMA issuer (one thread of the leader CTA): BK/16 tcgen05.mma per stage, commit frees the stage;
// the final commit signals the accumulator.  PAIR: M = 256 over the CTA pair, commits multicast.
template <class C, bool PAIR, int MMA_N, int MN = 0>
__device__ __forceinline__ void gemm_mma(const SmemLayout<C>& L, uint32_t tmem, int nkb, uint16_t pair_mask,
                                         uint64_t* trace_slot) {
  constexpr int MN_ = MMA_N > 256 ? 256 : MMA_N;  // BN = 512: two N = 256 MMAs per k-step
  constexpr uint32_t idesc = ptx::idesc_f16_f32_ab(PAIR ? 256 : 128, MN_, a_mn(MN), b_mn(MN));
  // descriptor start-address step per K = 16: one 128-byte swizzle row group (MN-major) or 32 bytes
  constexpr int akstep = a_mn(MN) ? 2048 >> 4 : 32 >> 4, bkstep = b_mn(MN) ? 2048 >> 4 : 32 >> 4;
#pragma unroll 1
  for (int i = 0; i < nkb; ++i) {
    const int s = i % C::STAGES;
    const uint32_t ph = (i / C::STAGES) & 1;
    ptx::mbar_wait(&L.full[s], ph);
    ptx::tc_fence_after();
    if (trace_slot && i == 0) *trace_slot = ptx::globaltimer();
    const uint32_t sa = ptx::smem_u32(L.sA + s * C::A_BYTES), sb = ptx::smem_u32(L.sB + s * C::B_BYTES);
    const uint64_t ad = a_mn(MN) ? ptx::sdesc_mnmajor_sw128(sa) : ptx::sdesc_kmajor_sw128(sa);
    const uint64_t bd = b_mn(MN) ? ptx::sdesc_mnmajor_sw128(sb) : ptx::sdesc_kmajor_sw128(sb);
#pragma unroll
    for (int k = 0; k < C::BK / 16; ++k) {
      if (PAIR) ptx::mma_f16_2sm(tmem, ad + akstep * k, bd + bkstep * k, idesc, (i | k) != 0 ? 1u : 0u);
      else ptx::mma_f16(tmem, ad + akstep * k, bd + bkstep * k, idesc, (i | k) != 0 ? 1u : 0u);
      if constexpr (MMA_N == 512) {  // second half: B block at +16 KB, accumulator columns +256
        const uint64_t bd2 = bd + (16384 >> 4);
        if (PAIR) ptx::mma_f16_2sm(tmem + 256, ad + akstep * k, bd2 + bkstep * k, idesc, (i | k) != 0 ? 1u : 0u);
        else ptx::mma_f16(tmem + 256, ad + akstep * k, bd2 + bkstep * k, idesc, (i | k) != 0 ? 1u : 0u);
      }
    }
    if (PAIR) ptx::mma_commit_2sm_mc(&L.empty[s], pair_mask);
    else ptx::mma_commit(&L.empty[s]);
  }
  if (PAIR) ptx::mma_commit_2sm_mc(L.accf, pair_mask);
  else ptx::mma_commit(L.accf);
}

// 64 accumulator columns of this thread's TMEM lane (zeros if the CTA had no k-blocks).
__device__ __forceinline__ void tmem_chunk(uint32_t tmem, int q, int c, bool have, float* v) {
  if (have) {
    const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + c * 64;
    ptx::tmem_ld16(ta, v);
    ptx::tmem_ld16(ta + 16, v + 16);
    ptx::tmem_ld16(ta + 32, v + 32);
    ptx::tmem_ld16(ta + 48, v + 48);
    ptx::tmem_ld_wait();
  } else {
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = 0.f;
  }
}

// Tile epilogue on a one-tile-per-CTA engine: the 128 x BN accumulator goes through shared memory
// in 64-column slices (stageT[128][68] fp32 in the idle stages, then epi.tile() with its scratch
// behind it), so tile epilogues (coalesced, batched) also run on the CTA-pair / 1-CTA plans that
// large batches select.  Epilogue warps only (256 threads, named barrier 1).
template <int BN, class Epi, class C>
__device__ __forceinline__ void tile_epilogue(const SmemLayout<C>& L, uint32_t tmem, bool have, int m0, int n0, int M,
                                              int N, const Epi& epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = warp & 3, grp = (warp - 2) >> 2, tid = threadIdx.x - 64;
  float* stageT = reinterpret_cast<float*>(L.sA);
  uint8_t* scratch = reinterpret_cast<uint8_t*>(stageT + 128 * 68);
  const int rows = min(128, M - m0);
#pragma unroll 1
  for (int c = 0; c < BN / 64; ++c) {
    float v[32];
    if (have) {
      const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + c * 64 + grp * 32;
      ptx::tmem_ld16(ta, v);
      ptx::tmem_ld16(ta + 16, v + 16);
      ptx::tmem_ld_wait();
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.f;
    }
    float4* d = reinterpret_cast<float4*>(stageT + (q * 32 + lane) * 68 + grp * 32);
#pragma unroll
    for (int i = 0; i < 8; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    asm volatile("bar.sync 1, 256;" ::: "memory");
    const int c0 = n0 + c * 64;
    if (rows > 0 && c0 < N) epi.tile(stageT, 68, m0, c0, min(64, N - c0), rows, scratch, tid);
    asm volatile("bar.sync 1, 256;" ::: "memory");
  }
}

// L2 prefetch job for the NEXT kernel's inputs: up to 4 contiguous regions (a weight's first row
// blocks, or activation-stash blocks the next fused epilogue reads), split evenly over this grid's
// CTAs, one bulk prefetch per CTA and region, issued by the producer thread after its own loads
// (the TMA unit is a FIFO: queued ahead of them the prefetches would delay this kernel's mainloop).
struct PrefetchJob {
  const uint8_t* base[4];
  long bytes[4];
};
__device__ __forceinline__ void l2_prefetch(const PrefetchJob& pj) {
  const long G = (long)gridDim.x * gridDim.y * gridDim.z;
  const long lin = blockIdx.x + (long)gridDim.x * (blockIdx.y + (long)gridDim.y * blockIdx.z);
  const uint64_t pol = ptx::policy_evict_last();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (pj.bytes[r] <= 0) continue;
    const long chunk = ((pj.bytes[r] + G - 1) / G + 15) / 16 * 16;
    const long off = lin * chunk;
    if (off >= pj.bytes[r]) continue;
    ptx::bulk_prefetch_l2(pj.base[r] + off, (uint32_t)min(chunk, pj.bytes[r] - off), pol);
  }
}

// Epilogue warps' common start: wait for the accumulator, then for the preceding grid (inputs
// of the fused epilogue), and let the next kernel's prologue start.
__device__ __forceinline__ void epi_begin(uint64_t* accf, bool have, uint64_t* trace_slot) {
  if (have) {
    ptx::mbar_wait(accf, 0);
    ptx::tc_fence_after();
  }
  if (trace_slot && threadIdx.x == 64) *trace_slot = ptx::globaltimer();
  ptx::pdl_wait();
  if (threadIdx.x == 64) ptx::pdl_trigger();
}

#define MLSTM_TRACE_BEGIN()                                  \
  __shared__ uint64_t tr_ts[10];                             \
  const bool tracing = g_trace != nullptr;                   \
  if (tracing && threadIdx.x == 0) {                         \
    for (int k = 1; k < 10; ++k) tr_ts[k] = 0;               \
    tr_ts[0] = ptx::globaltimer();                           \
  }
#define MLSTM_TRACE_SLOT(i) (tracing ? &tr_ts[i] : nullptr)
#define MLSTM_TRACE_END()                                    \
  if (tracing && threadIdx.x == 0) {                         \
    tr_ts[5] = ptx::globaltimer();                           \
    trace_flush(tr_ts, EpiTag<Epi>::value);                  \
  }

// ---------------------------------------------------------------------------------------------
template <int BN, class Epi, int MN = 0>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2, Seg2 sg, int M,
                   int N, int K, int az, int bz, int kb_per_split, uint32_t polA, uint32_t polB, int flags,
                   PrefetchJob pj, Epi epi) {
  using C = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  const SmemLayout<C> L(smem_raw);
  MLSTM_TRACE_BEGIN();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // kGemmRasterM: M-fastest raster -- CTAs launched together share their B (weight) tile, so a
  // multi-wave per-timestep GEMM streams each weight tile from HBM once (its A operand is small and
  // L2-resident).  Otherwise N-fastest (weight gradients: both operands stream along a long K).
  const int lin = blockIdx.x + gridDim.x * blockIdx.y;
  const bool rm = flags & kGemmRasterM;
  const int m0 = (rm ? lin % gridDim.y : blockIdx.y) * C::BM, n0 = (rm ? lin / gridDim.y : blockIdx.x) * BN;
  const int total_kb = (K + C::BK - 1) / C::BK;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = max(0, min(kb_per_split, total_kb - kb0));
  gemm_setup<C, false>(L, &tmA, &tmB, BN);
  if (threadIdx.x == 0 && nkb > 0)  // the barrier-initialising thread starts the weight stream
    gemm_produce<C, false, MN>(L, &tmA, &tmB, &tmA2, &tmB2, sg, nkb, kb0, m0, n0, az, bz, polA, polB, flags, true, 0,
                               nullptr, 1);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *L.tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      if (nkb > 0)
        gemm_produce<C, false, MN>(L, &tmA, &tmB, &tmA2, &tmB2, sg, nkb, kb0, m0, n0, az, bz, polA, polB, flags, true,
                                   0, MLSTM_TRACE_SLOT(1), 2);
      l2_prefetch(pj);
    }
  } else if (warp == 1) {
    if (lane == 0 && nkb > 0) gemm_mma<C, false, BN, MN>(L, tmem, nkb, 0, MLSTM_TRACE_SLOT(2));
  } else {
    const int q = warp & 3, grp = (warp - 2) >> 2;
    const int row = m0 + q * 32 + lane;
    if constexpr (HasTile<Epi>::value) {
      epi_begin(L.accf, nkb > 0, MLSTM_TRACE_SLOT(3));
      tile_epilogue<BN>(L, tmem, nkb > 0, m0, n0, M, N, epi);
    } else if constexpr (HasPreC<Epi>::value && MLSTM_F2_PREC) {
      // the epilogue's per-row input (F2: c_{t-1}) is loaded into registers while the main loop runs,
      // so no load latency sits between the accumulator and the outputs
      const EpiIO io = L.io(warp - 2, m0 + q * 32, M, lane);
      constexpr int NC = (BN / 64 + 1) / 2;  // chunks per epilogue warp (c = grp, grp + 2, ...)
      float4 cpre[NC][4];
      ptx::pdl_wait();
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int c = grp + 2 * i;
        if (c < BN / 64 && n0 + c * 64 < N) epi.preload_c(io, n0 + c * 64, cpre[i]);
      }
      epi_begin(L.accf, nkb > 0, MLSTM_TRACE_SLOT(3));
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int c = grp + 2 * i;
        if (c >= BN / 64) break;
        float v[64];
        tmem_chunk(tmem, q, c, nkb > 0, v);
        const int col0 = n0 + c * 64;
        if (col0 < N) epi.template run_io_c<4>(io, i, col0, v, cpre[i]);
      }
      ptx::bulk_wait_read0();
    } else if constexpr (HasAsyncIO<Epi>::value) {
      const EpiIO io = L.io(warp - 2, m0 + q * 32, M, lane);
      epi_begin(L.accf, nkb > 0, MLSTM_TRACE_SLOT(3));
      for (int c = grp, slot = 0; c < BN / 64; c += 2, ++slot)
        if (n0 + c * 64 < N) epi.io_issue(io, slot, n0 + c * 64);
      ptx::mbar_arrive(io.bar);
#pragma unroll 1
      for (int c = grp, slot = 0; c < BN / 64; c += 2, ++slot) {
        float v[64];
        tmem_chunk(tmem, q, c, nkb > 0, v);
        const int col0 = n0 + c * 64;
        if (col0 < N) epi.template run_io<4>(io, slot, col0, v);
      }
      ptx::bulk_wait_read0();
    } else {
      epi_begin(L.accf, nkb > 0, MLSTM_TRACE_SLOT(3));
#pragma unroll 1
      for (int c = grp; c < BN / 64; c += 2) {
        float v[64];
        tmem_chunk(tmem, q, c, nkb > 0, v);
        const int col0 = n0 + c * 64;
        if (row < M && col0 < N) epi.template run<4>(row, col0, v);
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  MLSTM_TRACE_END();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, BN);
  }
}

// ---------------------------------------------------------------------------------------------
template <int BN, class Epi, int MN = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2, Seg2 sg, int M,
                    int N, int K, int az, int bz, int kb_per_split, uint32_t polA, uint32_t polB, int flags,
                    PrefetchJob pj, Epi epi) {
  using C = Tc2Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  const SmemLayout<C> L(smem_raw);
  MLSTM_TRACE_BEGIN();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int lin = (blockIdx.x >> 1) + (gridDim.x >> 1) * blockIdx.y;  // raster: see gemm_tc_kernel
  const bool rm = flags & kGemmRasterM;
  int mi = rm ? lin % gridDim.y : blockIdx.y, ni = rm ? lin / gridDim.y : (blockIdx.x >> 1);
  if (flags & kGemmRasterG) {  // bands of 8 M-tiles, M-fastest inside a band
    const int nt = gridDim.x >> 1, band = lin / (8 * nt), in = lin - band * 8 * nt;
    const int bm = min(8, (int)gridDim.y - band * 8);
    mi = band * 8 + in % bm;
    ni = in / bm;
  }
  const int n0 = ni * BN;
  const int m0 = mi * 256 + rank * 128;
  const int total_kb = (K + C::BK - 1) / C::BK;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = max(0, min(kb_per_split, total_kb - kb0));
  gemm_setup<C, true>(L, &tmA, &tmB, BN);
  // the leader's own static-B stages can start before the cluster barrier (they complete on its own
  // barriers); the peer's signal the leader's barriers, so they wait for it
  if (leader && threadIdx.x == 0 && nkb > 0)
    gemm_produce<C, true, MN>(L, &tmA, &tmB, &tmA2, &tmB2, sg, nkb, kb0, m0, n0, az, bz, polA, polB, flags, true,
                              ptx::mapa_shared(ptx::smem_u32(&L.full[0]), 0), nullptr, 1);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *L.tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      if (nkb > 0)
        gemm_produce<C, true, MN>(L, &tmA, &tmB, &tmA2, &tmB2, sg, nkb, kb0, m0, n0 + rank * (BN == 512 ? 128 : BN / 2), az, bz, polA, polB, flags,
                              leader, ptx::mapa_shared(ptx::smem_u32(&L.full[0]), 0), MLSTM_TRACE_SLOT(1),
                              leader ? 2 : 0);
      l2_prefetch(pj);
    }
  } else if (warp == 1) {
    if (leader && lane == 0 && nkb > 0) gemm_mma<C, true, BN, MN>(L, tmem, nkb, 0x3, MLSTM_TRACE_SLOT(2));
  } else {
    const int q = warp & 3, grp = (warp - 2) >> 2;
    const int row = m0 + q * 32 + lane;
    if constexpr (HasTile<Epi>::value) {
      epi_begin(L.accf, nkb > 0, MLSTM_TRACE_SLOT(3));
      tile_epilogue<BN>(L, tmem, nkb > 0, m0, n0, M, N, epi);
    } else if constexpr (HasPreC<Epi>::value && MLSTM_F2_PREC) {
      // the epilogue's per-row input (F2: c_{t-1}) is loaded into registers while the main loop runs,
      // so no load latency sits between the accumulator and the outputs
      const EpiIO io = L.io(warp - 2, m0 + q * 32, M, lane);
      constexpr int NC = (BN / 64 + 1) / 2;  // chunks per epilogue warp (c = grp, grp + 2, ...)
      float4 cpre[NC][4];
      ptx::pdl_wait();
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int c = grp + 2 * i;
        if (c < BN / 64 && n0 + c * 64 < N) epi.preload_c(io, n0 + c * 64, cpre[i]);
      }
      epi_begin(L.accf, nkb > 0, MLSTM_TRACE_SLOT(3));
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int c = grp + 2 * i;
        if (c >= BN / 64) break;
        float v[64];
        tmem_chunk(tmem, q, c, nkb > 0, v);
        const int col0 = n0 + c * 64;
        if (col0 < N) epi.template run_io_c<4>(io, i, col0, v, cpre[i]);
      }
      ptx::bulk_wait_read0();
    } else if constexpr (HasAsyncIO<Epi>::value) {
      const EpiIO io = L.io(warp - 2, m0 + q * 32, M, lane);
      epi_begin(L.accf, nkb > 0, MLSTM_TRACE_SLOT(3));
      for (int c = grp, slot = 0; c < BN / 64; c += 2, ++slot)
        if (n0 + c * 64 < N) epi.io_issue(io, slot, n0 + c * 64);
      ptx::mbar_arrive(io.bar);
#pragma unroll 1
      for (int c = grp, slot = 0; c < BN / 64; c += 2, ++slot) {
        float v[64];
        tmem_chunk(tmem, q, c, nkb > 0, v);
        const int col0 = n0 + c * 64;
        if (col0 < N) epi.template run_io<4>(io, slot, col0, v);
      }
      ptx::bulk_wait_read0();
    } else {
      epi_begin(L.accf, nkb > 0, MLSTM_TRACE_SLOT(3));
#pragma unroll 1
      for (int c = grp; c < BN / 64; c += 2) {
        float v[64];
        tmem_chunk(tmem, q, c, nkb > 0, v);
        const int col0 = n0 + c * 64;
        if (row < M && col0 < N) epi.template run<4>(row, col0, v);
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  MLSTM_TRACE_END();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, BN);
  }
}

// ---------------------------------------------------------------------------------------------
// Persistent CTA-pair engine for GEMMs with more 256 x BN tiles than pairs fit on the GPU: the grid
// holds min(tiles, max_pairs) pairs and pair p walks tiles p, p + npairs, ...  The TMEM accumulator
// is double-buffered (2 x BN columns), so the epilogue of tile i overlaps the main loop of tile
// i+1; the stage ring and its phases run on across tiles.  Barriers (leader CTA unless noted):
// acc_full[b] (MMA commit, multicast to both CTAs) and acc_empty[b] (one arrive per epilogue warp
// of both CTAs, the peer's remotely).  Epilogues run in their row form (run<NG>).
template <int BN, class Epi, int MN = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm_tc2p_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2, Seg2 sg,
                     int M, int N, int K, int az, int bz, int unused, uint32_t polA, uint32_t polB, int flags,
                     PrefetchJob pj, Epi epi) {
  using C = Tc2Cfg<BN>;
  static_assert(2 * BN <= 512, "two accumulators must fit in TMEM");
  extern __shared__ uint8_t smem_raw[];
  const SmemLayout<C> L(smem_raw);
  uint64_t* acc_full = L.epibar;       // [2]
  uint64_t* acc_empty = L.epibar + 2;  // [2]
  MLSTM_TRACE_BEGIN();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int mt = (M + 255) / 256, nt = (N + BN - 1) / BN, ntiles = mt * nt;
  const int pid = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  const bool rm = flags & kGemmRasterM;
  const int total_kb = (K + C::BK - 1) / C::BK;
  auto tile_m = [&](int tile) { return (rm ? tile % mt : tile / nt) * 256 + (int)rank * 128; };
  auto tile_n = [&](int tile) { return (rm ? tile / mt : tile % nt) * BN; };
  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&L.full[s], 1);
      ptx::mbar_init(&L.empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&acc_full[b], 1);
      ptx::mbar_init(&acc_empty[b], 2 * kEpiWarps);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc2(L.tmem_slot, 2 * BN);
    ptx::tmem_relinquish2();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *L.tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pa = ptx::make_policy(polA), pb = ptx::make_policy(polB);
      const uint32_t tx = 2 * C::STAGE_BYTES;
      const uint32_t bar0 = ptx::mapa_shared(ptx::smem_u32(&L.full[0]), 0);
      ptx::pdl_wait();
      if (tracing) tr_ts[1] = ptx::globaltimer();
      int it = 0;
#pragma unroll 1
      for (int tile = pid; tile < ntiles; tile += npairs) {
        const int m0 = tile_m(tile), nb0 = tile_n(tile) + (int)rank * (BN / 2);
#pragma unroll 1
        for (int kb = 0; kb < total_kb; ++kb, ++it) {
          const int s = it % C::STAGES;
          if (it >= C::STAGES) ptx::mbar_wait(&L.empty[s], ((it / C::STAGES) & 1) ^ 1);
          if (leader) ptx::mbar_arrive_expect_tx(&L.full[s], tx);
          uint8_t* da = L.sA + s * C::A_BYTES;
          uint8_t* db = L.sB + s * C::B_BYTES;
          const bool s2 = kb >= sg.kb_seg0;  // second K segment (never with MN == 1)
          const int k = (s2 ? kb - sg.kb_seg0 : kb) * C::BK;
          if constexpr (a_mn(MN)) {
#pragma unroll
            for (int i = 0; i < C::BM / 64; ++i)
              ptx::tma_load_3d_2sm(da + i * 8192, &tmA, bar0 + s * 8, m0 + 64 * i, kb * C::BK, az, pa);
          } else {
            ptx::tma_load_3d_2sm(da, s2 ? &tmA2 : &tmA, bar0 + s * 8, k, m0, s2 ? sg.az2 : az, pa);
          }
          if constexpr (b_mn(MN)) {
            static_assert(C::B_BYTES % 8192 == 0, "MN-major B needs 64-wide boxes per CTA");
#pragma unroll
            for (int i = 0; i < C::B_BYTES / 8192; ++i)
              ptx::tma_load_3d_2sm(db + i * 8192, s2 ? &tmB2 : &tmB, bar0 + s * 8, nb0 + 64 * i, k, s2 ? sg.bz2 : bz,
                                   pb);
          } else {
            ptx::tma_load_3d_2sm(db, s2 ? &tmB2 : &tmB, bar0 + s * 8, k, nb0, s2 ? sg.bz2 : bz, pb);
          }
        }
      }
      l2_prefetch(pj);
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_f16_f32_ab(256, BN, a_mn(MN), b_mn(MN));
      constexpr int akstep = a_mn(MN) ? 2048 >> 4 : 32 >> 4, bkstep = b_mn(MN) ? 2048 >> 4 : 32 >> 4;
      int it = 0, lt = 0;
#pragma unroll 1
      for (int tile = pid; tile < ntiles; tile += npairs, ++lt) {
        const int b = lt & 1, use = lt >> 1;
        if (use > 0) ptx::mbar_wait(&acc_empty[b], (use - 1) & 1);
        ptx::tc_fence_after();
        const uint32_t td = tmem + b * BN;
#pragma unroll 1
        for (int kb = 0; kb < total_kb; ++kb, ++it) {
          const int s = it % C::STAGES;
          ptx::mbar_wait(&L.full[s], (it / C::STAGES) & 1);
          ptx::tc_fence_after();
          if (tracing && it == 0) tr_ts[2] = ptx::globaltimer();
          const uint32_t sa = ptx::smem_u32(L.sA + s * C::A_BYTES), sb = ptx::smem_u32(L.sB + s * C::B_BYTES);
          const uint64_t ad = a_mn(MN) ? ptx::sdesc_mnmajor_sw128(sa) : ptx::sdesc_kmajor_sw128(sa);
          const uint64_t bd = b_mn(MN) ? ptx::sdesc_mnmajor_sw128(sb) : ptx::sdesc_kmajor_sw128(sb);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k)
            ptx::mma_f16_2sm(td, ad + akstep * k, bd + bkstep * k, idesc, (kb | k) != 0 ? 1u : 0u);
          ptx::mma_commit_2sm_mc(&L.empty[s], 0x3);
        }
        ptx::mma_commit_2sm_mc(&acc_full[b], 0x3);
      }
    }
  } else {
    const int q = warp & 3, grp = (warp - 2) >> 2;
    const uint32_t empty_addr0 = ptx::mapa_shared(ptx::smem_u32(&acc_empty[0]), 0);
    int lt = 0;
#pragma unroll 1
    for (int tile = pid; tile < ntiles; tile += npairs, ++lt) {
      const int b = lt & 1, use = lt >> 1;
      ptx::mbar_wait(&acc_full[b], use & 1);
      ptx::tc_fence_after();
      if (lt == 0) {
        if (tracing && threadIdx.x == 64) tr_ts[3] = ptx::globaltimer();
        ptx::pdl_wait();
      }
      if (tile + npairs >= ntiles && threadIdx.x == 64) ptx::pdl_trigger();  // last tile of this pair
      const int m0 = tile_m(tile), n0 = tile_n(tile);
      const int row = m0 + q * 32 + lane;
#pragma unroll 1
      for (int c = grp; c < BN / 64; c += 2) {
        float v[64];
        tmem_chunk(tmem + b * BN, q, c, true, v);
        const int col0 = n0 + c * 64;
        if (row < M && col0 < N) epi.template run<4>(row, col0, v);
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&acc_empty[b]);
        else ptx::mbar_arrive_remote(empty_addr0 + b * 8);
      }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  MLSTM_TRACE_END();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, 2 * BN);
  }
}

// ---------------------------------------------------------------------------------------------
// Split-K over a cluster of S CTAs (rank z = K split).  Each CTA writes its fp32 partial to an
// L2-resident scratch laid out [z][float4 column group (64)][row (128)] (lanes = rows: coalesced);
// after the cluster barrier (release/acquire at cluster scope orders those writes) CTA z sums
// columns [z*256/S, (z+1)*256/S) of its 128 rows over the S partials in fixed order z' = 0..S-1
// (deterministic) and runs the fused epilogue on that slice -- the 256 epilogue threads each take
// half a row of the slice, or a whole row when the epilogue needs full 64-column chunks.
template <int S, class Epi, int MN = 0>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tc1s_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2, Seg2 sg, int M,
                     int N, int K, int az, int bz, int kb_per_split, uint32_t polA, uint32_t polB, int flags,
                     PrefetchJob pj, float* __restrict__ scratch,
                     Epi epi) {
  constexpr int BN = 256;
  using C = TcCfg<BN>;
  constexpr int SLICE = BN / S;
  constexpr bool HALF_ROWS = Epi::kMinGroups <= SLICE / 32;  // can a thread take half a row?
  constexpr int WIDTH = HALF_ROWS ? SLICE / 2 : SLICE;       // columns per thread
  constexpr int PIECE = WIDTH > 64 ? 64 : WIDTH;             // columns per epilogue call
  constexpr int NG = PIECE / 16;
  static_assert(WIDTH % PIECE == 0 && NG >= Epi::kMinGroups, "epilogue granularity");
  // the cooperative tile epilogue stages the reduced slice (fp32) and its own scratch in the idle
  // pipeline stages, which hold them only for 64-column slices; wider slices use the row epilogue
  constexpr bool kUseTile = HasTile<Epi>::value && SLICE <= 64;
  extern __shared__ uint8_t smem_raw[];
  const SmemLayout<C> L(smem_raw);
  MLSTM_TRACE_BEGIN();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = (int)ptx::cluster_ctarank();
  const int tile_n = blockIdx.x / S;
  const int n0 = tile_n * BN, m0 = blockIdx.y * C::BM;
  const int total_kb = (K + C::BK - 1) / C::BK;
  const int kb0 = z * kb_per_split;
  const int nkb = max(0, min(kb_per_split, total_kb - kb0));
  float* part = scratch + ((long)(blockIdx.y * (gridDim.x / S) + tile_n) * S) * (128L * BN);
  float* stageT = reinterpret_cast<float*>(L.sA);  // tile-epilogue staging: the stages are idle by then
  gemm_setup<C, false>(L, &tmA, &tmB, BN);
  if (threadIdx.x == 0 && nkb > 0)  // the barrier-initialising thread starts the weight stream
    gemm_produce<C, false, MN>(L, &tmA, &tmB, &tmA2, &tmB2, sg, nkb, kb0, m0, n0, az, bz, polA, polB, flags, true, 0,
                               nullptr, 1);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *L.tmem_slot;
  if (warp == 0) {
    if (lane == 0) {
      if (nkb > 0)
        gemm_produce<C, false, MN>(L, &tmA, &tmB, &tmA2, &tmB2, sg, nkb, kb0, m0, n0, az, bz, polA, polB, flags, true,
                                   0, MLSTM_TRACE_SLOT(1), 2);
      l2_prefetch(pj);
    }
  } else if (warp == 1) {
    if (lane == 0 && nkb > 0) gemm_mma<C, false, BN, MN>(L, tmem, nkb, 0, MLSTM_TRACE_SLOT(2));
  } else {
    const int q = warp & 3, grp = (warp - 2) >> 2;
    const int rl = q * 32 + lane;
    epi_begin(L.accf, nkb > 0, MLSTM_TRACE_SLOT(3));
    if constexpr (HasAsyncIO<Epi>::value && !kUseTile) {
      // the reduction phase's rows/columns of this thread (tid mapping below); loads land in the
      // idle stages while the partials are exchanged
      const int tid = threadIdx.x - 64, hh = tid >> 7;
      const EpiIO io = L.io(warp - 2, m0 + q * 32, M, lane);
      if (HALF_ROWS || hh == 0)
        for (int j = 0; j < WIDTH / PIECE; ++j) {
          const int col0 = n0 + z * SLICE + (HALF_ROWS ? hh * WIDTH : 0) + j * PIECE;
          if (col0 < N) epi.io_issue(io, j, col0);
        }
      ptx::mbar_arrive(io.bar);
    }
    float4* dst = reinterpret_cast<float4*>(part + (long)z * 128 * BN) + rl;
#pragma unroll 1
    for (int c = grp; c < BN / 64; c += 2) {
      if (c * 64 >= z * SLICE && c * 64 < (z + 1) * SLICE) continue;  // own slice: re-read from TMEM
      float v[64];
      tmem_chunk(tmem, q, c, nkb > 0, v);
#pragma unroll
      for (int i = 0; i < 16; ++i)
        dst[(c * 16 + i) * 128] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // all S partials of the tile are written (cluster-scope release/acquire)
  if (tracing && threadIdx.x == 0) tr_ts[4] = ptx::globaltimer();
  if (warp >= 2) {
    const int tid = threadIdx.x - 64;
    const int q = warp & 3, rl = q * 32 + lane, hh = tid >> 7;  // TMEM lane quarter of this warp
    const int row = m0 + rl;
    if (HALF_ROWS || hh == 0) {
#pragma unroll 1
      for (int j = 0; j < WIDTH / PIECE; ++j) {
        const int cl = z * SLICE + (HALF_ROWS ? hh * WIDTH : 0) + j * PIECE;
        float v[PIECE];
#pragma unroll
        for (int i = 0; i < PIECE; ++i) v[i] = 0.f;
#pragma unroll 1
        for (int zz = 0; zz < S; ++zz) {
          if (zz == z) {  // this CTA's own partial is still in TMEM
            if (nkb > 0) {
              float o[PIECE];
              const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + cl;
#pragma unroll
              for (int i = 0; i < PIECE / 16; ++i) ptx::tmem_ld16(ta + 16 * i, o + 16 * i);
              ptx::tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < PIECE; ++i) v[i] += o[i];
            }
            continue;
          }
          const float4* src = reinterpret_cast<const float4*>(part + (long)zz * 128 * BN) + (cl / 4) * 128 + rl;
#pragma unroll
          for (int i = 0; i < PIECE / 4; ++i) {
            const float4 p = __ldcg(src + i * 128);
            v[4 * i] += p.x;
            v[4 * i + 1] += p.y;
            v[4 * i + 2] += p.z;
            v[4 * i + 3] += p.w;
          }
        }
        const int col0 = n0 + cl;
        if constexpr (HasAsyncIO<Epi>::value && !kUseTile) {
          if (col0 < N) epi.template run_io<NG>(L.io(warp - 2, m0 + rl - lane, M, lane), j, col0, v);
        } else if constexpr (kUseTile) {
          float4* d = reinterpret_cast<float4*>(stageT + rl * (SLICE + 4) + (cl - z * SLICE));
#pragma unroll
          for (int i = 0; i < PIECE / 4; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        } else {
          if (row < M && col0 < N) epi.template run<NG>(row, col0, v);
        }
      }
    }
    if constexpr (HasAsyncIO<Epi>::value && !kUseTile) ptx::bulk_wait_read0();
    if (tracing && threadIdx.x == 64) tr_ts[6] = ptx::globaltimer();
    if constexpr (kUseTile) {
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (tracing && threadIdx.x == 64) tr_ts[7] = ptx::globaltimer();
      const int c0 = n0 + z * SLICE;
      if (m0 < M && c0 < N)
        epi.tile(stageT, SLICE + 4, m0, c0, min(SLICE, N - c0), min(128, M - m0),
                 reinterpret_cast<uint8_t*>(stageT + 128 * (SLICE + 4)), tid);
      if (tracing && threadIdx.x == 64) tr_ts[8] = ptx::globaltimer();
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  MLSTM_TRACE_END();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, BN);
  }
}

// ---------------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ float ld_as_float(const T* p) {
  return static_cast<float>(*p);
}
template <>
__device__ __forceinline__ float ld_as_float<__half>(const __half* p) {
  return __half2float(*p);
}

// SIMT engine: 128 x 64 output tile, 128 threads, thread t owns row m0 + t.  K is consumed in
// chunks of 32 staged through shared memory; k runs in ascending order inside each split.
template <typename T, class Epi>
__global__ void __launch_bounds__(128)
    gemm_simt_kernel(const T* __restrict__ A, long lda, const T* __restrict__ B, long ldb, int M, int N, int K,
                     int k_per_split, int mn, Epi epi) {
  __shared__ float As[32][129];
  __shared__ __align__(16) float Bs[32][64];
  const int tid = threadIdx.x;
  const int m0 = blockIdx.y * 128, n0 = blockIdx.x * 64;
  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(K, kbeg + k_per_split);
  float acc[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) acc[i] = 0.f;
#pragma unroll 1
  for (int kk = kbeg; kk < kend; kk += 32) {
#pragma unroll 4
    for (int i = tid; i < 128 * 32; i += 128) {
      // mn: operands MN-major (element (r, k) at k * ld + r), lanes along r
      const int r = mn ? (i & 127) : (i >> 5), k = mn ? (i >> 7) : (i & 31), gr = m0 + r, gk = kk + k;
      As[k][r] = (gr < M && gk < kend) ? ld_as_float(A + (mn ? (long)gk * lda + gr : (long)gr * lda + gk)) : 0.f;
    }
#pragma unroll 4
    for (int i = tid; i < 64 * 32; i += 128) {
      const int n = mn ? (i & 63) : (i >> 5), k = mn ? (i >> 6) : (i & 31), gn = n0 + n, gk = kk + k;
      Bs[k][n] = (gn < N && gk < kend) ? ld_as_float(B + (mn ? (long)gk * ldb + gn : (long)gn * ldb + gk)) : 0.f;
    }
    __syncthreads();
#pragma unroll 2
    for (int k = 0; k < 32; ++k) {
      const float a = As[k][tid];
      const float4* b4 = reinterpret_cast<const float4*>(&Bs[k][0]);
#pragma unroll
      for (int n = 0; n < 16; ++n) {
        const float4 bb = b4[n];
        acc[4 * n + 0] = fmaf(a, bb.x, acc[4 * n + 0]);
        acc[4 * n + 1] = fmaf(a, bb.y, acc[4 * n + 1]);
        acc[4 * n + 2] = fmaf(a, bb.z, acc[4 * n + 2]);
        acc[4 * n + 3] = fmaf(a, bb.w, acc[4 * n + 3]);
      }
    }
    __syncthreads();
  }
  const int row = m0 + tid;
  if (row < M && n0 < N) epi.template run<4>(row, n0, acc);
}

}  // namespace mlstm
