// bwd_persist.cuh -- the backward recurrence as ONE persistent kernel.
//
// The per-timestep form launches B1(t) (dM = dZ_t W_h, epilogue dA, dMX) and B2(t) (dH = dA_t W_mh
// + dY_{t-1} W_dec, epilogue: gate backward of step t-1) as two split-K cluster GEMMs per timestep.
// Here the same 128 CTAs (clusters of S = 4 along the K split, 128 x 256 tiles) stay resident for
// all 2T-1 phases B1(T-1), B2(T-1), B1(T-2), ..., B1(0):
//   * the TMA producer streams the next phase's weight stages (W_h^T / W_mh^T do not depend on the
//     recurrence) while the current epilogue runs, then waits for the grid-wide phase barrier
//     before loading the activation operand the previous phase wrote;
//   * the stage ring, its mbarrier phases and the TMEM accumulator carry over from phase to phase;
//   * the split-K partials go through the L2 scratch as in gemm_tc1s_kernel, synchronised by a
//     per-tile counter among the epilogue warps (the producer / MMA warps never block on it);
//   * the grid barrier is a monotonically increasing arrival counter plus a generation word in
//     global memory (release/acquire at gpu scope); the cooperative launch guarantees co-residency.
// Every spin is bounded: a barrier that does not complete within ~seconds traps instead of hanging.
#pragma once
#include "gemm.cuh"
#include "epilogues.cuh"

namespace mlstm {

using ptx::ld_acquire_gpu;
using ptx::st_release_gpu;
using ptx::spin_until_geq;
using ptx::fence_proxy_async_global;

constexpr int kBwdSyncWords = 2;  // [0] grid arrivals, [1] grid generation; then one counter per tile

template <int S>
__global__ void __launch_bounds__(kGemmThreads, 1)
    bwd_persist_kernel(const __grid_constant__ CUtensorMap tA1, const __grid_constant__ CUtensorMap tB1,
                       const __grid_constant__ CUtensorMap tA2, const __grid_constant__ CUtensorMap tB2,
                       const __grid_constant__ CUtensorMap tA2s, const __grid_constant__ CUtensorMap tB2s,
                       Net<__half> n, float* __restrict__ scratch, uint32_t* __restrict__ sync) {
  constexpr int BN = 256, SLICE = BN / S, WIDTH = SLICE / 2;  // both epilogues take half rows
  static_assert(SLICE <= 64, "B2's tile epilogue needs 64-column slices");
  using C = TcCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  const SmemLayout<C> L(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int z = (int)ptx::cluster_ctarank();
  const int tile_n = blockIdx.x / S, ntn = gridDim.x / S;
  const int n0 = tile_n * BN, m0 = blockIdx.y * C::BM;
  const int M = n.B, N = n.h, T = n.T;
  const int kb1 = 4 * N / C::BK, kb2a = N / C::BK, kb2 = kb2a + 256 / C::BK;
  const int kbps1 = (kb1 + S - 1) / S, kbps2 = (kb2 + S - 1) / S;
  const int nphase = 2 * T - 1;
  const int tile_id = blockIdx.y * ntn + tile_n;
  const uint32_t ncta = gridDim.x * gridDim.y;
  float* part = scratch + (long)tile_id * S * 128 * BN;
  auto phase = [&](int k, bool& b1, int& t, int& kb0, int& nkb) {
    b1 = !(k & 1);
    t = T - 1 - (k >> 1);
    const int kbps = b1 ? kbps1 : kbps2, tot = b1 ? kb1 : kb2;
    kb0 = z * kbps;
    nkb = max(0, min(kbps, tot - kb0));
  };
  gemm_setup<C, false>(L, &tA1, &tB1, BN);
  if (threadIdx.x == 32) {
    ptx::prefetch_tmap(&tA2);
    ptx::prefetch_tmap(&tB2);
    ptx::prefetch_tmap(&tA2s);
    ptx::prefetch_tmap(&tB2s);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *L.tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------------------- TMA producer
      const uint64_t pa = ptx::make_policy(1u << 8), pb = ptx::make_policy(0);
      auto loadA = [&](bool b1, int t, int s, int kb) {
        uint8_t* dst = L.sA + s * C::A_BYTES;
        if (b1) ptx::tma_load_3d(dst, &tA1, &L.full[s], kb * C::BK, m0, t, pa);
        else if (kb < kb2a) ptx::tma_load_3d(dst, &tA2, &L.full[s], kb * C::BK, m0, t, pa);
        else ptx::tma_load_3d(dst, &tA2s, &L.full[s], (kb - kb2a) * C::BK, m0, t - 1, pa);
      };
      auto loadB = [&](bool b1, int s, int kb) {
        uint8_t* dst = L.sB + s * C::B_BYTES;
        if (b1) ptx::tma_load_3d(dst, &tB1, &L.full[s], kb * C::BK, n0, 0, pb);
        else if (kb < kb2a) ptx::tma_load_3d(dst, &tB2, &L.full[s], kb * C::BK, n0, 0, pb);
        else ptx::tma_load_3d(dst, &tB2s, &L.full[s], (kb - kb2a) * C::BK, n0, 0, pb);
      };
      int it = 0;
#pragma unroll 1
      for (int k = 0; k < nphase; ++k) {
        bool b1;
        int t, kb0, nkb;
        phase(k, b1, t, kb0, nkb);
        const int pre = min(C::STAGES, nkb);
        // weights first: they do not depend on the previous phase
        for (int i = 0; i < pre; ++i) {
          const int j = it + i, s = j % C::STAGES;
          if (j >= C::STAGES) ptx::mbar_wait(&L.empty[s], ((j / C::STAGES) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&L.full[s], C::STAGE_BYTES);
          loadB(b1, s, kb0 + i);
        }
        {  // warm L2 with the stash the coming epilogues read (written by the forward long ago)
          const long BH = (long)M * N;
          PrefetchJob pj{{nullptr, nullptr, nullptr, nullptr}, {0, 0, 0, 0}};
          if (b1 && t > 0) {  // B2's gate backward of step t-1: gates_{t-1}, c_{t-1}, c_{t-2}
            pj.base[0] = reinterpret_cast<const uint8_t*>(n.Gates + (long)(t - 1) * 4 * BH);
            pj.bytes[0] = 4 * BH * 2;
            pj.base[1] = reinterpret_cast<const uint8_t*>(n.Crm + (long)(t - 1) * BH);
            pj.bytes[1] = 2 * BH * 4;
          } else if (!b1 && t > 0) {  // B1(t-1)'s a-stash block
            pj.base[0] = reinterpret_cast<const uint8_t*>(n.Astash + (long)(t - 1) * BH);
            pj.bytes[0] = BH * 2;
          }
          l2_prefetch(pj);
        }
        if (k > 0) {  // the activations of this phase were written by every CTA in phase k-1
          spin_until_geq(&sync[1], (uint32_t)k);
          fence_proxy_async_global();
        }
        for (int i = 0; i < pre; ++i) loadA(b1, t, (it + i) % C::STAGES, kb0 + i);
#pragma unroll 1
        for (int i = pre; i < nkb; ++i) {
          const int j = it + i, s = j % C::STAGES;
          ptx::mbar_wait(&L.empty[s], ((j / C::STAGES) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&L.full[s], C::STAGE_BYTES);
          loadA(b1, t, s, kb0 + i);
          loadB(b1, s, kb0 + i);
        }
        it += nkb;
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // -------------------------------------------------------- MMA issuer
      constexpr uint32_t idesc = ptx::idesc_f16_f32(128, BN);
      int it = 0;
#pragma unroll 1
      for (int k = 0; k < nphase; ++k) {
        bool b1;
        int t, kb0, nkb;
        phase(k, b1, t, kb0, nkb);
#pragma unroll 1
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % C::STAGES;
          ptx::mbar_wait(&L.full[s], (it / C::STAGES) & 1);
          ptx::tc_fence_after();
          const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(L.sA + s * C::A_BYTES));
          const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(L.sB + s * C::B_BYTES));
#pragma unroll
          for (int kk = 0; kk < C::BK / 16; ++kk)
            ptx::mma_f16(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (i | kk) != 0 ? 1u : 0u);
          ptx::mma_commit(&L.empty[s]);
        }
        ptx::mma_commit(L.accf);
      }
    }
  } else {  // ------------------------------------------------------------------- epilogue warps
    const int q = warp & 3, grp = (warp - 2) >> 2, tid = threadIdx.x - 64;
    const int rl = tid & 127, hh = tid >> 7;
    float* stageT = reinterpret_cast<float*>(L.sA);  // A stages are idle during the epilogue
#pragma unroll 1
    for (int k = 0; k < nphase; ++k) {
      bool b1;
      int t, kb0, nkb;
      phase(k, b1, t, kb0, nkb);
      ptx::mbar_wait(L.accf, k & 1);
      ptx::tc_fence_after();
      {  // this CTA's fp32 partial -> L2 scratch [z][float4 column group][row]
        float4* dst = reinterpret_cast<float4*>(part + (long)z * 128 * BN) + (q * 32 + lane);
#pragma unroll 1
        for (int c = grp; c < BN / 64; c += 2) {
          float v[64];
          tmem_chunk(tmem, q, c, nkb > 0, v);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            dst[(c * 16 + i) * 128] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
      ptx::tc_fence_before();
      // the S CTAs of this tile have written their partials (per-tile counter, epilogue warps only)
      epi_bar256();
      if (tid == 0) {
        __threadfence();
        atomicAdd(&sync[kBwdSyncWords + tile_id], 1u);
        spin_until_geq(&sync[kBwdSyncWords + tile_id], (uint32_t)(S * (k + 1)));
      }
      epi_bar256();
      // fixed-order sum over the S partials of this thread's half-row slice
      const int cl = z * SLICE + hh * WIDTH;
      float acc[WIDTH];
#pragma unroll
      for (int i = 0; i < WIDTH; ++i) acc[i] = 0.f;
#pragma unroll 1
      for (int zz = 0; zz < S; ++zz) {
        const float4* src = reinterpret_cast<const float4*>(part + (long)zz * 128 * BN) + (cl / 4) * 128 + rl;
#pragma unroll
        for (int i = 0; i < WIDTH / 4; ++i) {
          const float4 p = __ldcg(src + i * 128);
          acc[4 * i] += p.x;
          acc[4 * i + 1] += p.y;
          acc[4 * i + 2] += p.z;
          acc[4 * i + 3] += p.w;
        }
      }
      if (b1) {  // dA = dM * mx, dMX = dM * a (row outputs staged in this warp's window)
        const EpiIO io{L.sA + (warp - 2) * 8192, L.epibar + (warp - 2), m0 + rl - lane,
                       max(0, min(32, M - (m0 + rl - lane))), lane};
        if (n0 + cl < N) EpiB1IO<__half>{{n, t}}.template run_io<WIDTH / 16>(io, 0, n0 + cl, acc);
      } else {  // gate backward of step t-1 on the reduced tile
        float4* d = reinterpret_cast<float4*>(stageT + rl * (SLICE + 4) + hh * WIDTH);
#pragma unroll
        for (int i = 0; i < WIDTH / 4; ++i) d[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
        epi_bar256();
        const int c0 = n0 + z * SLICE;
        if (m0 < M && c0 < N)
          EpiB2<__half>{n, t - 1}.tile(stageT, SLICE + 4, m0, c0, min(SLICE, N - c0), min(128, M - m0),
                                        reinterpret_cast<uint8_t*>(stageT + 128 * (SLICE + 4)), tid);
      }
      // phase done on this CTA: its outputs are visible, its shared-memory staging is free again
      ptx::fence_proxy_async_smem();
      epi_bar256();
      if (tid == 0) {
        __threadfence();
        const uint32_t old = atomicAdd(&sync[0], 1u);
        if (old + 1 == ncta * (uint32_t)(k + 1)) st_release_gpu(&sync[1], (uint32_t)(k + 1));
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, BN);
  }
}

}  // namespace mlstm
