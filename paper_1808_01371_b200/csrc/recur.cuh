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
// Roles (320 threads): warp 0 lane 0 = TMA producer (both CTAs), warp 1 lane 0 of the leader CTA =
// tcgen05.mma issuer, warps 2..9 = epilogue (two warps per TMEM lane quarter: q = warp & 3 owns
// rows [32q, +32), grp = (warp - 2) >> 2 takes half of each 64-column slice).
#pragma once
#include "gemm.cuh"
#include "epilogues.cuh"

namespace mlstm {

constexpr int kRcStages = 5;
constexpr int kRcTile = 128 * 64 * 2;  // one 128-row x 64-K fp16 operand tile (per CTA, per stage)
constexpr int kRcWin = 8192;           // staging window of one epilogue warp
constexpr int kRcSmem = kRcStages * 2 * kRcTile + kEpiWarps * kRcWin + 1024 + 256;

struct RcPolicy {  // L2 policy codes (ptx::make_policy) of the operand streams
  uint32_t act, w_split, w_wide, w_seg;
};

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
//   [0, 2P)   chunk flags X[p][r]  (fwd: H_t of pair p;  bwd: dZ_s of pair p)
//   [2P, 4P)  chunk flags Y[p][r]  (fwd: M_t chunk p;   bwd: dA_t chunk p)
//   [4P, 6P)  split partial flags of the first N = h GEMM  [(n1, r)][z]  (fwd F1, bwd B1)
//   [6P, 8P)  split partial flags of the second            [(n1, r)][z]  (bwd B2)
constexpr int kRcFlagWords(int P) { return 8 * P; }
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
__device__ __forceinline__ void rc_consume(const RcLayout& L, uint32_t it, uint32_t d, bool acc) {
  constexpr uint32_t idesc = ptx::idesc_f16_f32_ab(256, 256, false, BMN);
  const int s = it % kRcStages;
  ptx::mbar_wait(&L.full[s], (it / kRcStages) & 1);
  ptx::tc_fence_after();
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
    __threadfence();
    ptx::st_release_gpu(flag, val);
  }
}

// Split-K exchange of the 128 x 256 fp32 accumulator at TMEM column `col0` among the 4 CTAs
// (z = 0..3, same rank) of one tile: the 3 foreign 64-column slices go to the L2 scratch
// grp_scratch[zsrc][zdst][16 float4 column groups][128 rows], this CTA's flag is published, the
// peers' flags are awaited, and `out` receives this thread's 32 columns [64z + 32grp, +32) of its
// own slice summed over z = 0..3 in order (its own partial straight from TMEM).
__device__ __forceinline__ void rc_reduce(uint32_t tmem, int col0, float4* grp_scratch, int z, int q, int grp,
                                          int lane, int tid, uint32_t* pflags, uint32_t val, uint64_t* acce,
                                          bool leader, float* out) {
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
  float own[32];
  ptx::tmem_ld16(trow + 64 * z + 32 * grp, own);
  ptx::tmem_ld16(trow + 64 * z + 32 * grp + 16, own + 16);
  ptx::tmem_ld_wait();
  rc_release_acc(acce, leader, lane);
  rc_bar();
  if (tid == 0) {
    __threadfence();
    ptx::st_release_gpu(pflags + z, val);
#pragma unroll 1
    for (int zz = 0; zz < 4; ++zz)
      if (zz != z) ptx::spin_until_geq(pflags + zz, val);
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

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// =============================================================================================
// Forward: for t = 0..T-1   F1(t): a_t = H_{t-1} W_mh^T (split z of tile n1), m_t = mx_t * a_t
//                            F2(t): z_t = onehot(x_t) (W_x E + b)^T + M_t W_h^T; gates, c, h
// =============================================================================================
__global__ void __launch_bounds__(kGemmThreads, 1)
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

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------------------ TMA producer
      const uint64_t pact = ptx::make_policy(pol.act), pw1 = ptx::make_policy(pol.w_split),
                     pw2 = ptx::make_policy(pol.w_wide), pws = ptx::make_policy(pol.w_seg);
      const uint32_t bar0 = ptx::mapa_shared(ptx::smem_u32(&L.full[0]), 0);
      const int total = T * per;
      // k-block idx -> (t, kind, chunk)
      auto decode = [&](int idx, int& t, int& kind, int& j) {
        t = idx / per;
        const int i = idx - t * per;
        if (i < nF1) {
          kind = 0;
          j = z * nF1 + (i + n1) % nF1;
        } else if (i < nF1 + 4) {
          kind = 1;
          j = i - nF1;
        } else {
          kind = 2;
          j = (i - nF1 - 4 + p) % nF2;
        }
      };
      int wi = 0, ai = 0;
      uint64_t idle_since = 0;
#pragma unroll 1
      while (ai < total) {
        bool progress = false;
        // weights: as far ahead as free stages allow (they do not depend on the recurrence)
#pragma unroll 1
        while (wi < total && wi < ai + kRcStages) {
          const int s = wi % kRcStages;
          if (wi >= kRcStages && !ptx::mbar_test(&L.empty[s], ((wi / kRcStages) & 1) ^ 1)) break;
          int t, kind, j;
          decode(wi, t, kind, j);
          if (leader) ptx::mbar_arrive_expect_tx(&L.full[s], 2 * kRcTile);
          uint8_t* dst = L.sB + s * kRcTile;
          if (kind == 0) ptx::tma_load_3d_2sm(dst, &tmWmh, bar0 + 8 * s, 64 * j, 256 * n1 + 128 * r, 0, pw1);
          else if (kind == 1) ptx::tma_load_3d_2sm(dst, &tmXZ, bar0 + 8 * s, 64 * j, 256 * p + 128 * r, 0, pws);
          else ptx::tma_load_3d_2sm(dst, &tmWh, bar0 + 8 * s, 64 * j, 256 * p + 128 * r, 0, pw2);
          ++wi;
          progress = true;
        }
        // activations: once their producer published them
        if (ai < wi) {
          int t, kind, j;
          decode(ai, t, kind, j);
          bool ready = true;
          if (kind == 0 && t > 0) ready = ptx::ld_acquire_gpu(&fH[2 * j + r]) >= (uint32_t)t;
          else if (kind == 2) ready = ptx::ld_acquire_gpu(&fM[2 * j + r]) >= (uint32_t)(t + 1);
          if (ready) {
            if (kind != 1) ptx::fence_proxy_async_global();
            const int s = ai % kRcStages;
            if (leader) ptx::mbar_arrive_expect_tx(&L.full[s], 2 * kRcTile);
            uint8_t* dst = L.sA + s * kRcTile;
            if (kind == 0) ptx::tma_load_3d_2sm(dst, &tmH, bar0 + 8 * s, 64 * j, 128 * r, t, pact);
            else if (kind == 1) ptx::tma_load_3d_2sm(dst, &tmOH, bar0 + 8 * s, 64 * j, 128 * r, t, pact);
            else ptx::tma_load_3d_2sm(dst, &tmM, bar0 + 8 * s, 64 * j, 128 * r, t, pact);
            ++ai;
            progress = true;
          }
        }
        rc_watchdog(progress, idle_since);
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
#pragma unroll 1
        for (int i = 0; i < nF1; ++i) rc_consume<false>(L, it++, tmem, i > 0);
        ptx::mma_commit_2sm_mc(&L.accf[0], 0x3);
        if (t > 0) {
          ptx::mbar_wait(&L.acce[1], (t - 1) & 1);
          ptx::tc_fence_after();
        }
#pragma unroll 1
        for (int i = 0; i < 4 + nF2; ++i) rc_consume<false>(L, it++, tmem + 256, i > 0);
        ptx::mma_commit_2sm_mc(&L.accf[1], 0x3);
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
      prefetch_l2(mxp);
      ptx::mbar_wait(&L.accf[0], t & 1);
      ptx::tc_fence_after();
      float a[32];
      rc_reduce(tmem, 0, gscr + (t & 1) * region, z, q, grp, lane, tid, fP + (n1 * 2 + r) * 4, (uint32_t)(t + 1),
                &L.acce[0], leader, a);
      {
        float m[32];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float x[16];
          ld16(mxp + 16 * g, x);
#pragma unroll
          for (int i = 0; i < 16; ++i) m[16 * g + i] = x[i] * a[16 * g + i];
        }
        rc_stage_h<2>(w, 80, lane, m);
        warp_rows_out(reinterpret_cast<uint8_t*>(n.Mrm + ((long)t * B + b0) * h + u1), 2L * h, w, 80, 64, 32, lane);
        __syncwarp();
      }
      rc_publish(&fM[2 * p + r], (uint32_t)(t + 1), tid);
      rc_stage_h<2>(w, 80, lane, a);
      warp_rows_out(reinterpret_cast<uint8_t*>(n.Astash + ((long)t * B + b0) * h + u1), 2L * h, w, 80, 64, 32, lane);
      __syncwarp();
      // ---------------------------------------------- F2 epilogue: gates, cell update, hidden state
      ptx::mbar_wait(&L.accf[1], t & 1);
      ptx::tc_fence_after();
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
#pragma unroll
      for (int cc = 0; cc < 2; ++cc)
        warp_rows_out(reinterpret_cast<uint8_t*>(n.Hrm + ((long)(t + 1) * B + b0) * h + 64 * p + 16 * (grp + 2 * cc)),
                      2L * h, w + cc * 1536, 48, 32, 32, lane);
      rc_publish(&fH[2 * p + r], (uint32_t)(t + 1), tid);
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
__global__ void __launch_bounds__(kGemmThreads, 1)
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
  uint32_t* fZ = flags;           // [P][2]  dZ_s of units [64p, +64)
  uint32_t* fA = flags + 2 * P;   // [P][2]  dA_t chunk p
  uint32_t* fP1 = flags + 4 * P;  // [(n1, r)][4]
  uint32_t* fP2 = flags + 6 * P;  // [(n1, r)][4]
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
  const int total = 1 + T * per - (1 + nB2);  // no B2(0)

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------------------ TMA producer
      const uint64_t pact = ptx::make_policy(pol.act), pw1 = ptx::make_policy(pol.w_split),
                     pw2 = ptx::make_policy(pol.w_wide), pws = ptx::make_policy(pol.w_seg);
      const uint32_t bar0 = ptx::mapa_shared(ptx::smem_u32(&L.full[0]), 0);
      // idx -> (t, kind, chunk): kind 0 = B1 dZ chunk, 1 = B2 segment dY_{t-1}, 2 = B2 dA chunk
      auto decode = [&](int idx, int& t, int& kind, int& j) {
        if (idx == 0) {  // prologue B2(T): the dY_{T-1} W_dec segment only
          t = T;
          kind = 1;
          j = z;
          return;
        }
        const int u = (idx - 1) / per, i = (idx - 1) - u * per;
        t = T - 1 - u;
        if (i < nB1) {
          kind = 0;
          j = z * nB1 + (i + n1) % nB1;
        } else if (i == nB1) {
          kind = 1;
          j = z;
        } else {
          kind = 2;
          j = z * nB2 + (i - nB1 - 1 + n1) % nB2;
        }
      };
      int wi = 0, ai = 0;
      uint64_t idle_since = 0;
#pragma unroll 1
      while (ai < total) {
        bool progress = false;
#pragma unroll 1
        while (wi < total && wi < ai + kRcStages) {
          const int s = wi % kRcStages;
          if (wi >= kRcStages && !ptx::mbar_test(&L.empty[s], ((wi / kRcStages) & 1) ^ 1)) break;
          int t, kind, j;
          decode(wi, t, kind, j);
          if (leader) ptx::mbar_arrive_expect_tx(&L.full[s], 2 * kRcTile);
          uint8_t* dst = L.sB + s * kRcTile;
          const int u0 = 256 * n1 + 128 * r;  // this CTA's 128 output units (MN-major boxes of 64)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (kind == 0) ptx::tma_load_3d_2sm(dst + i * 8192, &tmWh, bar0 + 8 * s, u0 + 64 * i, 64 * j, 0, pw2);
            else if (kind == 1)
              ptx::tma_load_3d_2sm(dst + i * 8192, &tmWdec, bar0 + 8 * s, u0 + 64 * i, 64 * j, 0, pws);
            else ptx::tma_load_3d_2sm(dst + i * 8192, &tmWmh, bar0 + 8 * s, u0 + 64 * i, 64 * j, 0, pw1);
          }
          ++wi;
          progress = true;
        }
        if (ai < wi) {
          int t, kind, j;
          decode(ai, t, kind, j);
          bool ready = true;
          if (kind == 0) ready = ptx::ld_acquire_gpu(&fZ[2 * (j >> 2) + r]) >= (uint32_t)(T - t);
          else if (kind == 2) ready = ptx::ld_acquire_gpu(&fA[2 * j + r]) >= (uint32_t)(T - t);
          if (ready) {
            if (kind != 1) ptx::fence_proxy_async_global();
            const int s = ai % kRcStages;
            if (leader) ptx::mbar_arrive_expect_tx(&L.full[s], 2 * kRcTile);
            uint8_t* dst = L.sA + s * kRcTile;
            if (kind == 0) ptx::tma_load_3d_2sm(dst, &tmDZ, bar0 + 8 * s, 64 * j, 128 * r, t, pact);
            else if (kind == 1) ptx::tma_load_3d_2sm(dst, &tmDY, bar0 + 8 * s, 64 * j, 128 * r, t - 1, pact);
            else ptx::tma_load_3d_2sm(dst, &tmDA, bar0 + 8 * s, 64 * j, 128 * r, t, pact);
            ++ai;
            progress = true;
          }
        }
        rc_watchdog(progress, idle_since);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {  // ------------------------------------------------- MMA issuer
      uint32_t it = 0;
      rc_consume<true>(L, it++, tmem + 256, false);  // B2(T): dY_{T-1} W_dec
      ptx::mma_commit_2sm_mc(&L.accf[1], 0x3);
#pragma unroll 1
      for (int u = 0; u < T; ++u) {
        const int t = T - 1 - u;
        if (u > 0) {
          ptx::mbar_wait(&L.acce[0], (u - 1) & 1);
          ptx::tc_fence_after();
        }
#pragma unroll 1
        for (int i = 0; i < nB1; ++i) rc_consume<true>(L, it++, tmem, i > 0);
        ptx::mma_commit_2sm_mc(&L.accf[0], 0x3);
        if (t == 0) break;
        ptx::mbar_wait(&L.acce[1], u & 1);  // use u of the wide accumulator (use 0 = prologue)
        ptx::tc_fence_after();
#pragma unroll 1
        for (int i = 0; i < 1 + nB2; ++i) rc_consume<true>(L, it++, tmem + 256, i > 0);
        ptx::mma_commit_2sm_mc(&L.accf[1], 0x3);
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
    auto b2_epi = [&](int t, int use) {
      const int s = t - 1;
      const long BH = (long)B * h;
      const __half* gates = n.Gates + ((long)s * B + b) * 4 * h + (u1 >> 4) * 64;
      const float* cs = n.Crm + (long)(s + 1) * BH + (long)b * h + u1;
      const float* cp = n.Crm + (long)s * BH + (long)b * h + u1;
      prefetch_l2(gates);
      prefetch_l2(gates + 64);
      prefetch_l2(cs);
      prefetch_l2(cp);
      ptx::mbar_wait(&L.accf[1], use & 1);
      ptx::tc_fence_after();
      float dh[32];
      rc_reduce(tmem, 256, gscr2 + (t & 1) * region, z, q, grp, lane, tid, fP2 + (n1 * 2 + r) * 4,
                (uint32_t)(T - t + 1), &L.acce[1], leader, dh);
#pragma unroll
      for (int g = 0; g < 2; ++g) {  // two groups of 16 units = two 64-column internal chunks
        float gi[16], gf[16], go[16], gu[16], c[16], cpv[16];
        ld16(gates + 64 * g, gi);
        ld16(gates + 64 * g + 16, gf);
        ld16(gates + 64 * g + 32, go);
        ld16(gates + 64 * g + 48, gu);
        ld16(cs + 16 * g, c);
        ld16(cp + 16 * g, cpv);
        float dz[64];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const float kk = act_tanh<__half>(c[k]);
          const float i = gi[k], f = gf[k], o = go[k], u = gu[k], d = dh[16 * g + k];
          dz[32 + k] = d * kk * o * (1.f - o);                    // dZ_o
          const float dc = dcs[16 * g + k] + d * o * (1.f - kk * kk);
          dz[k] = dc * u * i * (1.f - i);                         // dZ_i
          dz[16 + k] = dc * cpv[k] * f * (1.f - f);               // dZ_f
          dz[48 + k] = dc * i * (1.f - u * u);                    // dZ_u
          dcs[16 * g + k] = dc * f;                               // dc carry to step s-1
        }
        rc_stage_h<4>(w, 144, lane, dz);
        warp_rows_out(reinterpret_cast<uint8_t*>(n.G5 + ((long)s * B + b0) * 5 * h + h + (u1 >> 4) * 64 + 64 * g),
                      10L * h, w, 144, 128, 32, lane);
        __syncwarp();
      }
      rc_publish(&fZ[2 * p + r], (uint32_t)(T - s), tid);
    };
    b2_epi(T, 0);
#pragma unroll 1
    for (int u = 0; u < T; ++u) {
      const int t = T - 1 - u;
      // ---------------------------------------------- B1 epilogue: dA = dM * mx, dMX = dM * a
      const int byte = n.byte_at(b, t);
      const float* mxp = n.tab + (long)byte * 5 * h + u1;
      const __half* ap = n.Astash + ((long)t * B + b) * h + u1;
      prefetch_l2(mxp);
      prefetch_l2(ap);
      ptx::mbar_wait(&L.accf[0], u & 1);
      ptx::tc_fence_after();
      float dm[32];
      rc_reduce(tmem, 0, gscr1 + (t & 1) * region, z, q, grp, lane, tid, fP1 + (n1 * 2 + r) * 4, (uint32_t)(T - t),
                &L.acce[0], leader, dm);
      {
        float da[32];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float x[16];
          ld16(mxp + 16 * g, x);
#pragma unroll
          for (int i = 0; i < 16; ++i) da[16 * g + i] = dm[16 * g + i] * x[i];
        }
        rc_stage_h<2>(w, 80, lane, da);
        warp_rows_out(reinterpret_cast<uint8_t*>(n.dA + ((long)t * B + b0) * h + u1), 2L * h, w, 80, 64, 32, lane);
        __syncwarp();
      }
      if (t > 0) rc_publish(&fA[2 * p + r], (uint32_t)(T - t), tid);
      {
        float dmx[32];
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          float av[16];
          ld16(ap + 16 * g, av);
#pragma unroll
          for (int i = 0; i < 16; ++i) dmx[16 * g + i] = dm[16 * g + i] * av[i];
        }
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
