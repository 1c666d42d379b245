// gemm.cuh -- the two GEMM engines every contraction of the step runs on.
//
//   D[M x N] = A[M x K] . B[N x K]^T   (both operands K-major, i.e. row-major with K contiguous),
//   fp32 accumulation, result handed to a fused epilogue functor 64 columns at a time:
//       epi(row, col0, float (&v)[64])   with v[i] = D[row][col0 + i].
//
// * gemm_tc_kernel (mixed precision, fp16 operands): TMA (128B swizzle) -> multi-stage mbarrier
//   ring in shared memory -> single-thread tcgen05.mma (M=128, N=BN, K=16) into a TMEM fp32
//   accumulator -> 4 epilogue warps tcgen05.ld their 32 TMEM lanes (one accumulator row per
//   thread).  Warp roles: warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer, warps 2-5
//   epilogue.  One output tile per CTA; optional split-K over blockIdx.z.
// * gemm_simt_kernel (fp32 parity mode, "single precision"): plain FFMA, 128 x 64 tile,
//   one output row per thread, fixed ascending-k accumulation -- same epilogue interface.
#pragma once
#include "ptx.cuh"

namespace mlstm {

// ---- optional intra-kernel timeline (mlstm_trace_enable): one record per CTA,
// {tag, cta, t_start, t_first_tma, t_first_full, t_acc_ready, t_reduced, t_end} in ns.
struct TraceRec {
  uint64_t v[8];
};
__device__ TraceRec* g_trace = nullptr;
__device__ unsigned int g_trace_n = 0;
__device__ unsigned int g_trace_cap = 0;
struct Trace {
  uint64_t t[6];
  __device__ __forceinline__ void mark(int i) { t[i] = ptx::globaltimer(); }
};
__device__ __forceinline__ void trace_flush(const uint64_t* ts, int tag) {
  TraceRec* tr = g_trace;
  if (!tr) return;
  const unsigned int i = atomicAdd(&g_trace_n, 1u);
  if (i >= g_trace_cap) return;
  TraceRec r;
  r.v[0] = (uint64_t)tag;
  r.v[1] = blockIdx.x + (uint64_t)gridDim.x * (blockIdx.y + (uint64_t)gridDim.y * blockIdx.z);
  for (int k = 0; k < 6; ++k) r.v[2 + k] = ts[k];
  tr[i] = r;
}
__device__ __forceinline__ void epi_bar_() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
template <class E, class = void>
struct IsTile {  // epilogue with a cooperative tile() member (see epilogues.cuh)
  static constexpr bool value = false;
};
template <class E>
struct IsTile<E, decltype(void(E::kTile))> {
  static constexpr bool value = E::kTile;
};

// Stages a 128 x (64*nchunk) fp32 accumulator tile from TMEM into shared memory (row stride ldt):
// thread = TMEM lane = tile row.
__device__ __forceinline__ void stage_tmem_rows(float* T, int ldt, uint32_t tmem, int q, int lane, int nchunk,
                                                bool have) {
  const int rl = q * 32 + lane;
#pragma unroll 1
  for (int c = 0; c < nchunk; ++c) {
    float v[64];
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
    float4* dst = reinterpret_cast<float4*>(T + rl * ldt + c * 64);
#pragma unroll
    for (int i = 0; i < 16; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
  }
}

template <class Epi>
struct EpiTag {
  static constexpr int value = 0;
};

template <int BN>
struct TcCfg {
  static constexpr int BM = 128, BK = 64;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN, class Epi>
__global__ void __launch_bounds__(192, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                   int N, int K, int az, int bz, int kb_per_split, uint32_t polA, uint32_t polB, Epi epi) {
  using C = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accf = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  __shared__ uint64_t tr_ts[6];
  const bool tracing = g_trace != nullptr;
  if (tracing && threadIdx.x == 0) {
    for (int k = 1; k < 6; ++k) tr_ts[k] = 0;
    tr_ts[0] = ptx::globaltimer();
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * C::BM, n0 = blockIdx.x * BN;
  const int total_kb = (K + C::BK - 1) / C::BK;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = max(0, min(kb_per_split, total_kb - kb0));

  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(tmem_slot, BN);
    ptx::tmem_relinquish();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && nkb > 0) {
      const uint64_t pa = ptx::make_policy(polA), pb = ptx::make_policy(polB);
#pragma unroll 1
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        ptx::mbar_wait(&empty[s], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
        const int kc = (kb0 + i) * C::BK;
        if (tracing && i == 0) tr_ts[1] = ptx::globaltimer();
        ptx::tma_load_3d(sA + s * C::A_BYTES, &tmA, &full[s], kc, m0, az, pa);
        ptx::tma_load_3d(sB + s * C::B_BYTES, &tmB, &full[s], kc, n0, bz, pb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nkb > 0) {
      constexpr uint32_t idesc = ptx::idesc_f16_f32(C::BM, BN);
#pragma unroll 1
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        ptx::mbar_wait(&full[s], ph);
        ptx::tc_fence_after();
        if (tracing && i == 0) tr_ts[2] = ptx::globaltimer();
        const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sA + s * C::A_BYTES));
        const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sB + s * C::B_BYTES));
#pragma unroll
        for (int k = 0; k < C::BK / 16; ++k)
          ptx::mma_f16(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0 ? 1u : 0u);
        ptx::mma_commit(&empty[s]);
      }
      ptx::mma_commit(accf);
    }
  } else {
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = m0 + q * 32 + lane;
    if (nkb > 0) {
      ptx::mbar_wait(accf, 0);
      ptx::tc_fence_after();
    }
    if (tracing && threadIdx.x == 64) tr_ts[3] = ptx::globaltimer();
    if constexpr (IsTile<Epi>::value) {
      float* T = reinterpret_cast<float*>(smem);  // the pipeline stages are idle now
      constexpr int ldt = BN + 4;
      stage_tmem_rows(T, ldt, tmem, q, lane, BN / 64, nkb > 0);
      ptx::tc_fence_before();
      epi_bar_();
      const int rows = min(128, M - (row - q * 32 - lane));
      if (rows > 0 && n0 < N)
        epi.tile(T, ldt, row - q * 32 - lane, n0, min(BN, N - n0), rows,
                 reinterpret_cast<uint8_t*>(T + 128 * ldt), (int)threadIdx.x - 64);
    } else {
#pragma unroll 1
    for (int c = 0; c < BN / 64; ++c) {
      float v[64];
      if (nkb > 0) {
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
      const int col0 = n0 + c * 64;
      if (row < M && col0 < N) epi(row, col0, v);
    }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (tracing && threadIdx.x == 0) {
    tr_ts[5] = ptx::globaltimer();
    trace_flush(tr_ts, EpiTag<Epi>::value);
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, BN);
  }
}


// ---------------------------------------------------------------------------------------------
// gemm_tc2_kernel: the same contract with a CTA pair (cluster of 2, tcgen05 cta_group::2) per
// 256 x BN output tile.  Each CTA stages its 128 rows of A and BN/2 rows of B per k-block, so a
// CTA pulls (128 + BN/2) x 64 x 2 bytes per 256 x BN x 64 of MMA work: half the operand traffic per
// FLOP of the 1-CTA tile -- the L2 -> SM path is what bounds these GEMMs.  Both CTAs' TMA loads
// count on the leader's full barrier; the leader's single thread issues the M=256 MMA; its commit
// multicasts to both CTAs' empty / accumulator barriers; each CTA's epilogue reads its own TMEM.
template <int BN>
struct Tc2Cfg {
  static constexpr int BM = 128, BK = 64;  // rows per CTA
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / 2) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 6 : (BN == 128 ? 8 : 10);
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <int BN, class Epi>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                    int N, int K, int az, int bz, int kb_per_split, uint32_t polA, uint32_t polB, Epi epi) {
  using C = Tc2Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accf = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  __shared__ uint64_t tr_ts[6];
  const bool tracing = g_trace != nullptr;
  if (tracing && threadIdx.x == 0) {
    for (int k = 1; k < 6; ++k) tr_ts[k] = 0;
    tr_ts[0] = ptx::globaltimer();
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;
  const int n0 = (blockIdx.x >> 1) * BN;
  const int m0 = blockIdx.y * 256 + rank * 128;
  const int total_kb = (K + C::BK - 1) / C::BK;
  const int kb0 = blockIdx.z * kb_per_split;
  const int nkb = max(0, min(kb_per_split, total_kb - kb0));

  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);   // leader's arrive.expect_tx covers both CTAs' bytes
      ptx::mbar_init(&empty[s], 1);  // leader's multicast commit
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc2(tmem_slot, BN);
    ptx::tmem_relinquish2();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && nkb > 0) {
      const uint64_t pa = ptx::make_policy(polA), pb = ptx::make_policy(polB);
      const uint32_t full_leader0 = ptx::mapa_shared(ptx::smem_u32(&full[0]), 0);
#pragma unroll 1
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        ptx::mbar_wait(&empty[s], ph ^ 1);
        // Only the leader arrives (with both CTAs' byte count).  The peer's bytes may land first and
        // drive the tx-count transiently negative; the phase cannot complete before the leader's
        // arrive, and the peer cannot run a phase ahead (it waits on its own empty barrier, released
        // by the same commit).  A release.cluster remote arrive here would fence every prior TMA.
        if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * C::STAGE_BYTES);
        const int kc = (kb0 + i) * C::BK;
        if (tracing && i == 0) tr_ts[1] = ptx::globaltimer();
        ptx::tma_load_3d_2sm(sA + s * C::A_BYTES, &tmA, full_leader0 + s * 8, kc, m0, az, pa);
        ptx::tma_load_3d_2sm(sB + s * C::B_BYTES, &tmB, full_leader0 + s * 8, kc, n0 + rank * (BN / 2), bz, pb);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0 && nkb > 0) {
      constexpr uint32_t idesc = ptx::idesc_f16_f32(256, BN);
#pragma unroll 1
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        ptx::mbar_wait(&full[s], ph);
        ptx::tc_fence_after();
        if (tracing && i == 0) tr_ts[2] = ptx::globaltimer();
        const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sA + s * C::A_BYTES));
        const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sB + s * C::B_BYTES));
#pragma unroll
        for (int k = 0; k < C::BK / 16; ++k)
          ptx::mma_f16_2sm(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0 ? 1u : 0u);
        ptx::mma_commit_2sm_mc(&empty[s], 0x3);
      }
      ptx::mma_commit_2sm_mc(accf, 0x3);
    }
  } else {
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    if (nkb > 0) {
      ptx::mbar_wait(accf, 0);
      ptx::tc_fence_after();
    }
    if (tracing && threadIdx.x == 64) tr_ts[3] = ptx::globaltimer();
    if constexpr (IsTile<Epi>::value) {
      float* T = reinterpret_cast<float*>(smem);  // the pipeline stages are idle now
      constexpr int ldt = BN + 4;
      stage_tmem_rows(T, ldt, tmem, q, lane, BN / 64, nkb > 0);
      ptx::tc_fence_before();
      epi_bar_();
      const int rows = min(128, M - (row - q * 32 - lane));
      if (rows > 0 && n0 < N)
        epi.tile(T, ldt, row - q * 32 - lane, n0, min(BN, N - n0), rows,
                 reinterpret_cast<uint8_t*>(T + 128 * ldt), (int)threadIdx.x - 64);
    } else {
#pragma unroll 1
    for (int c = 0; c < BN / 64; ++c) {
      float v[64];
      if (nkb > 0) {
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
      const int col0 = n0 + c * 64;
      if (row < M && col0 < N) epi(row, col0, v);
    }
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (tracing && threadIdx.x == 0) {
    tr_ts[5] = ptx::globaltimer();
    trace_flush(tr_ts, EpiTag<Epi>::value);
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, BN);
  }
}

// ---------------------------------------------------------------------------------------------
// gemm_tc2s_kernel: CTA-pair 256 x 256 tiles with the K loop split S ways across S pairs of one
// cluster (2S CTAs; cluster rank r: row half r & 1, K-split r >> 1).  Used where the output is too
// small to fill the machine with 256-wide tiles (the per-timestep GEMMs with N = h).  After the
// mainloop every CTA stages its fp32 partial in its own (now idle) pipeline shared memory; after a
// cluster barrier, CTA r reduces columns [z*256/S, (z+1)*256/S) of its 128 rows over the S
// partials through DSMEM in fixed order z = 0..S-1 (deterministic) and runs the fused epilogue on
// that slice -- so the epilogue work stays spread over all 2S CTAs.
template <int S, class Epi>
__global__ void __launch_bounds__(192, 1)
    gemm_tc2s_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                     int N, int K, int az, int bz, int kb_per_split, uint32_t polA, uint32_t polB, Epi epi) {
  constexpr int BN = 256;
  using C = Tc2Cfg<BN>;
  constexpr int SLICE = BN / S;
  constexpr int LDS = BN + 4;  // staging row stride in floats (odd number of 16-byte units)
  static_assert(128 * LDS * 4 <= C::STAGES * C::STAGE_BYTES, "staging must fit in the pipeline smem");
  static_assert(SLICE % 64 == 0, "slice is a whole number of epilogue chunks");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  float* stage = reinterpret_cast<float*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accf = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  __shared__ uint64_t tr_ts[6];
  const bool tracing = g_trace != nullptr;
  if (tracing && threadIdx.x == 0) {
    for (int k = 1; k < 6; ++k) tr_ts[k] = 0;
    tr_ts[0] = ptx::globaltimer();
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const uint32_t half = rank & 1u, z = rank >> 1, pair_leader = rank & ~1u;
  const bool leader = half == 0;
  const int n0 = (blockIdx.x / (2 * S)) * BN;
  const int m0 = blockIdx.y * 256 + half * 128;
  const int total_kb = (K + C::BK - 1) / C::BK;
  const int kb0 = z * kb_per_split;
  const int nkb = max(0, min(kb_per_split, total_kb - kb0));

  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc2(tmem_slot, BN);
    ptx::tmem_relinquish2();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && nkb > 0) {
      const uint64_t pa = ptx::make_policy(polA), pb = ptx::make_policy(polB);
      const uint32_t full_leader0 = ptx::mapa_shared(ptx::smem_u32(&full[0]), pair_leader);
#pragma unroll 1
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        ptx::mbar_wait(&empty[s], ph ^ 1);
        if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * C::STAGE_BYTES);
        const int kc = (kb0 + i) * C::BK;
        if (tracing && i == 0) tr_ts[1] = ptx::globaltimer();
        ptx::tma_load_3d_2sm(sA + s * C::A_BYTES, &tmA, full_leader0 + s * 8, kc, m0, az, pa);
        ptx::tma_load_3d_2sm(sB + s * C::B_BYTES, &tmB, full_leader0 + s * 8, kc, n0 + half * (BN / 2), bz, pb);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0 && nkb > 0) {
      constexpr uint32_t idesc = ptx::idesc_f16_f32(256, BN);
      const uint16_t mask = static_cast<uint16_t>(3u << pair_leader);
#pragma unroll 1
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        ptx::mbar_wait(&full[s], ph);
        ptx::tc_fence_after();
        if (tracing && i == 0) tr_ts[2] = ptx::globaltimer();
        const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sA + s * C::A_BYTES));
        const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sB + s * C::B_BYTES));
#pragma unroll
        for (int k = 0; k < C::BK / 16; ++k)
          ptx::mma_f16_2sm(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0 ? 1u : 0u);
        ptx::mma_commit_2sm_mc(&empty[s], mask);
      }
      ptx::mma_commit_2sm_mc(accf, mask);
    }
  } else {
    // stage this CTA's fp32 partial (128 rows x 256 cols) in its own shared memory
    const int q = warp & 3;
    const int rl = q * 32 + lane;
    if (nkb > 0) {
      ptx::mbar_wait(accf, 0);
      ptx::tc_fence_after();
    }
    if (tracing && threadIdx.x == 64) tr_ts[3] = ptx::globaltimer();
#pragma unroll 1
    for (int c = 0; c < BN / 64; ++c) {
      float v[64];
      if (nkb > 0) {
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
      float4* dst = reinterpret_cast<float4*>(stage + rl * LDS + c * 64);
#pragma unroll
      for (int i = 0; i < 16; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // every partial of the cluster is staged
  if (tracing && threadIdx.x == 0) tr_ts[4] = ptx::globaltimer();
  if (warp >= 2) {
    const int q = warp & 3;
    const int rl = q * 32 + lane;
    const int row = m0 + rl;
    const uint32_t my = ptx::smem_u32(stage + rl * LDS + z * SLICE);
#pragma unroll 1
    for (int j = 0; j < SLICE / 64; ++j) {
      float v[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = 0.f;
#pragma unroll 1
      for (int zz = 0; zz < S; ++zz) {
        const uint32_t src = ptx::mapa_shared(my, 2 * zz + half) + j * 256;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float4 p = ptx::ld_dsmem_f4(src + 16 * i);
          v[4 * i] += p.x;
          v[4 * i + 1] += p.y;
          v[4 * i + 2] += p.z;
          v[4 * i + 3] += p.w;
        }
      }
      const int col0 = n0 + z * SLICE + j * 64;
      if (row < M && col0 < N) epi(row, col0, v);
    }
  }
  ptx::cluster_sync();  // no CTA leaves while others still read its staging buffer
  if (tracing && threadIdx.x == 0) {
    tr_ts[5] = ptx::globaltimer();
    trace_flush(tr_ts, EpiTag<Epi>::value);
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, BN);
  }
}

// ---------------------------------------------------------------------------------------------
// gemm_tc1s_kernel: one CTA per 128 x 256 tile (full-rate M=128, N=256 tcgen05.mma) with the K
// loop split S ways over the S CTAs of a cluster (cluster rank z = K split).  Used when 256-wide
// tiles alone cannot fill the machine (the per-timestep GEMMs with N = h).  Each CTA writes its
// fp32 partial to an L2-resident scratch; after the cluster barrier (release/acquire at cluster
// scope orders those writes) CTA z sums columns [z*256/S, (z+1)*256/S) of its 128 rows over the S
// partials in fixed order z' = 0..S-1 (deterministic) and runs the fused epilogue on that slice,
// so the epilogue work stays spread over all S CTAs of the tile.
template <int S, class Epi>
__global__ void __launch_bounds__(192, 1)
    gemm_tc1s_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                     int N, int K, int az, int bz, int kb_per_split, uint32_t polA, uint32_t polB,
                     float* __restrict__ scratch, Epi epi) {
  constexpr int BN = 256;
  using C = TcCfg<BN>;
  constexpr int SLICE = BN / S;
  static_assert(SLICE % 64 == 0, "slice is a whole number of epilogue chunks");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accf = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  __shared__ uint64_t tr_ts[6];
  const bool tracing = g_trace != nullptr;
  if (tracing && threadIdx.x == 0) {
    for (int k = 1; k < 6; ++k) tr_ts[k] = 0;
    tr_ts[0] = ptx::globaltimer();
  }

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = (int)ptx::cluster_ctarank();
  const int tile_n = blockIdx.x / S;
  const int n0 = tile_n * BN, m0 = blockIdx.y * C::BM;
  const int total_kb = (K + C::BK - 1) / C::BK;
  const int kb0 = z * kb_per_split;
  const int nkb = max(0, min(kb_per_split, total_kb - kb0));
  float* stage_T = reinterpret_cast<float*>(smem);  // tile-epilogue staging (stages idle by then)
  // this tile's S partials: scratch[(tile * S + z')][128][256]
  float* part = scratch + ((long)(blockIdx.y * (gridDim.x / S) + tile_n) * S) * (128L * BN);

  if (threadIdx.x == 0) {
#pragma unroll 1
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(accf, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc(tmem_slot, BN);
    ptx::tmem_relinquish();
  }
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0 && nkb > 0) {
      const uint64_t pa = ptx::make_policy(polA), pb = ptx::make_policy(polB);
#pragma unroll 1
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        ptx::mbar_wait(&empty[s], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full[s], C::STAGE_BYTES);
        const int kc = (kb0 + i) * C::BK;
        if (tracing && i == 0) tr_ts[1] = ptx::globaltimer();
        ptx::tma_load_3d(sA + s * C::A_BYTES, &tmA, &full[s], kc, m0, az, pa);
        ptx::tma_load_3d(sB + s * C::B_BYTES, &tmB, &full[s], kc, n0, bz, pb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nkb > 0) {
      constexpr uint32_t idesc = ptx::idesc_f16_f32(C::BM, BN);
#pragma unroll 1
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t ph = (i / C::STAGES) & 1;
        ptx::mbar_wait(&full[s], ph);
        ptx::tc_fence_after();
        if (tracing && i == 0) tr_ts[2] = ptx::globaltimer();
        const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sA + s * C::A_BYTES));
        const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sB + s * C::B_BYTES));
#pragma unroll
        for (int k = 0; k < C::BK / 16; ++k)
          ptx::mma_f16(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) != 0 ? 1u : 0u);
        ptx::mma_commit(&empty[s]);
      }
      ptx::mma_commit(accf);
    }
  } else {
    const int q = warp & 3;
    const int rl = q * 32 + lane;
    if (nkb > 0) {
      ptx::mbar_wait(accf, 0);
      ptx::tc_fence_after();
    }
    if (tracing && threadIdx.x == 64) tr_ts[3] = ptx::globaltimer();
    // partial layout [z][float4 column group (64)][row (128)]: lanes (= rows) write consecutive
    // 16-byte vectors, fully coalesced; the reducer reads with the same mapping
    float4* dst = reinterpret_cast<float4*>(part + (long)z * 128 * BN) + rl;
#pragma unroll 1
    for (int c = 0; c < BN / 64; ++c) {
      float v[64];
      if (nkb > 0) {
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
#pragma unroll
      for (int i = 0; i < 16; ++i) dst[(c * 16 + i) * 128] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // all S partials of the tile are written (cluster-scope release/acquire)
  if (tracing && threadIdx.x == 0) tr_ts[4] = ptx::globaltimer();
  if (warp >= 2) {
    const int q = warp & 3;
    const int rl = q * 32 + lane;
    const int row = m0 + rl;
#pragma unroll 1
    for (int j = 0; j < SLICE / 64; ++j) {
      const int cl = z * SLICE + j * 64;
      float v[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = 0.f;
#pragma unroll 1
      for (int zz = 0; zz < S; ++zz) {
        const float4* src = reinterpret_cast<const float4*>(part + (long)zz * 128 * BN) + (cl / 4) * 128 + rl;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float4 p = __ldcg(src + i * 128);
          v[4 * i] += p.x;
          v[4 * i + 1] += p.y;
          v[4 * i + 2] += p.z;
          v[4 * i + 3] += p.w;
        }
      }
      const int col0 = n0 + cl;
      if constexpr (IsTile<Epi>::value) {
        float4* dst = reinterpret_cast<float4*>(stage_T + rl * (SLICE + 4) + j * 64);
#pragma unroll
        for (int i = 0; i < 16; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      } else {
        if (row < M && col0 < N) epi(row, col0, v);
      }
    }
    if constexpr (IsTile<Epi>::value) {
      epi_bar_();
      const int rows = min(128, M - m0);
      const int c0 = n0 + z * SLICE;
      if (rows > 0 && c0 < N)
        epi.tile(stage_T, SLICE + 4, m0, c0, min(SLICE, N - c0), rows,
                 reinterpret_cast<uint8_t*>(stage_T + 128 * (SLICE + 4)), (int)threadIdx.x - 64);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (tracing && threadIdx.x == 0) {
    tr_ts[5] = ptx::globaltimer();
    trace_flush(tr_ts, EpiTag<Epi>::value);
  }
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, BN);
  }
}

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
                     int k_per_split, Epi epi) {
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
      const int r = i >> 5, k = i & 31, gr = m0 + r, gk = kk + k;
      As[k][r] = (gr < M && gk < kend) ? ld_as_float(A + (long)gr * lda + gk) : 0.f;
    }
#pragma unroll 4
    for (int i = tid; i < 64 * 32; i += 128) {
      const int n = i >> 5, k = i & 31, gn = n0 + n, gk = kk + k;
      Bs[k][n] = (gn < N && gk < kend) ? ld_as_float(B + (long)gn * ldb + gk) : 0.f;
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
  if constexpr (IsTile<Epi>::value) {
    extern __shared__ float simt_dyn[];
    float* T = simt_dyn;
    float4* dst = reinterpret_cast<float4*>(T + tid * 68);
#pragma unroll
    for (int i = 0; i < 16; ++i) dst[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
    __syncthreads();
    const int rows = min(128, M - m0);
    if (rows > 0 && n0 < N)
      epi.tile(T, 68, m0, n0, min(64, N - n0), rows, reinterpret_cast<uint8_t*>(T + 128 * 68), tid);
  } else {
    if (row < M && n0 < N) epi(row, n0, acc);
  }
}

}  // namespace mlstm
