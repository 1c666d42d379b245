// stream_bench.cu -- the recurrence's streaming core in isolation (tools only; not part of the library):
// CTA pairs (cta_group::2) stream 256 x 64 A and 256 x 64 B k-blocks through an S-stage ring into
// M = N = 256, K = 64 tcgen05 MMAs (the F2 / B1 inner loop), stages released by the MMA commit
// multicast to both CTAs.  Variants: one producer thread issuing both boxes of a stage, or two
// producers (weights / activations) issuing one each; A from a small L2-resident buffer shared by all
// pairs (the activations), B from a per-pair slab of a 134 MB tensor (W_h).  Reports us per k-block.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1808_01371_b200/csrc
//        tools/stream_bench.cu -o tools/stream_bench.bin -lcuda
#include <cudaTypedefs.h>

#include <cstdio>
#include <vector>

#include "recur.cuh"

using namespace mlstm;

constexpr int kTile = 16384;
constexpr int kMaxS = 6;

struct Cfg {
  int stages, producers, iters, kblocks, b_shared, spin, maps;
};

__global__ void __launch_bounds__(384, 1) stream_bench(const __grid_constant__ CUtensorMap tA,
                                                       const __grid_constant__ CUtensorMap tB,
                                                       const __grid_constant__ CUtensorMap tA2,
                                                       const __grid_constant__ CUtensorMap tB2, Cfg cfg,
                                                       unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;
  uint8_t* sB = sm + kMaxS * kTile;
  __shared__ uint64_t full[kMaxS], empty[kMaxS], done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r = ptx::cluster_ctarank();
  const bool leader = r == 0;
  const int S = cfg.stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], cfg.producers);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(&done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    ptx::tmem_alloc2(&tslot, 256);
    ptx::tmem_relinquish2();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = tslot;
  const int pair = blockIdx.x >> 1;
  const uint32_t bar0 = ptx::mapa_shared(ptx::smem_u32(&full[0]), 0);
  const uint64_t pol = ptx::make_policy(0);
  unsigned long long t0 = 0, t1 = 0;
  auto issueA = [&](int s, int i) {
    // spin = 2: rotated A order per pair (each pair at a different chunk at a given time)
    const int ka = cfg.spin == 2 ? (i + pair) % 64 : i % 64;
    ptx::tma_load_3d_2sm(sA + s * kTile, (cfg.maps && (i & 1)) ? &tA2 : &tA, bar0 + 8 * s, 64 * ka, 128 * r, 0, pol);
  };
  auto issueB = [&](int s, int i) {
    const int row = cfg.b_shared ? 128 * r : 256 * pair + 128 * r;
    ptx::tma_load_3d_2sm(sB + s * kTile, (cfg.maps && (i & 1)) ? &tB2 : &tB, bar0 + 8 * s, 64 * (i % cfg.kblocks),
                         row, 0, pol);
  };
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < cfg.iters; ++i) {
      const int s = i % S;
      if (i >= S) ptx::mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
      if (cfg.producers == 1) {
        if (leader) ptx::mbar_arrive_expect_tx(&full[s], 4 * kTile);
        issueB(s, i);
        issueA(s, i);
      } else {
        if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * kTile);
        issueB(s, i);
      }
    }
  } else if (warp == 2 && lane == 0 && cfg.producers == 2) {
    for (int i = 0; i < cfg.iters; ++i) {
      const int s = i % S;
      if (i >= S) ptx::mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
      if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * kTile);
      issueA(s, i);
    }
  } else if (warp == 1 && lane == 0 && leader) {
    constexpr uint32_t idesc = ptx::idesc_f16_f32_ab(256, 256, false, false);
    t0 = ptx::globaltimer();
    for (int i = 0; i < cfg.iters; ++i) {
      const int s = i % S;
      ptx::mbar_wait(&full[s], (i / S) & 1);
      ptx::tc_fence_after();
      const uint64_t ad = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sA + s * kTile));
      const uint64_t bd = ptx::sdesc_kmajor_sw128(ptx::smem_u32(sB + s * kTile));
#pragma unroll
      for (int k = 0; k < 4; ++k) ptx::mma_f16_2sm(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) ? 1u : 0u);
      ptx::mma_commit_2sm_mc(&empty[s], 0x3);
    }
    ptx::mma_commit_2sm_mc(&done, 0x3);
    ptx::mbar_wait(&done, 0);
    t1 = ptx::globaltimer();
    out[2 * pair] = t0;
    out[2 * pair + 1] = t1;
  }
  if (!leader && threadIdx.x == 64) ptx::mbar_wait(&done, 0);
  if (cfg.spin == 1 && warp >= 4) ptx::mbar_wait(&done, 0);  // idle "epilogue" warps sleeping on a barrier
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, 256);
  }
}


// The same streaming core built from the library's own pieces (RcLayout, rc_setup, rc_weights,
// rc_acts, rc_consume): the difference to stream_bench isolates their overheads.
__global__ void __launch_bounds__(kRcThreads, 1) lib_core(const __grid_constant__ CUtensorMap tA,
                                                          const __grid_constant__ CUtensorMap tB, int iters,
                                                          unsigned long long* out, int storm, uint32_t* flag) {
  extern __shared__ uint8_t smem_raw[];
  const RcLayout L(smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = (int)ptx::cluster_ctarank();
  const bool leader = r == 0;
  const int p = blockIdx.x >> 1;
  rc_setup(L);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *L.tmem_slot;
  const RcTrace tr{0xffffffffu, 1, 0, 1, 0};
  const int per = 64;
  if (warp == 0 || warp == kRcActWarp) {
    const uint64_t pact = ptx::make_policy(0), pw = ptx::make_policy(0);
    const uint32_t bar0 = ptx::mapa_shared(ptx::smem_u32(&L.full[0]), 0);
    auto dec = [&](int u, int i) {
      RcBlk b;
      b.t = u;
      b.kind = 2;
      b.j = i;
      b.flag = nullptr;
      return b;
    };
    auto issue_w = [&](int s, const RcBlk& b) {
      ptx::tma_load_3d_2sm(L.sB + s * kRcTile, &tB, bar0 + 8 * s, 64 * b.j, 256 * p + 128 * r, 0, pw);
    };
    auto issue_a = [&](int s, const RcBlk& b) {
      ptx::tma_load_3d_2sm(L.sA + s * kRcTile, &tA, bar0 + 8 * s, 64 * b.j, 128 * r, 0, pact);
    };
    auto prefetch_w = [&](const RcBlk&) {};
    if (warp == 0) {
      if (lane == 0) rc_weights(L, iters, 0, per, leader, 0, tr, dec, issue_w, prefetch_w);
    } else {
      rc_acts(L, iters, 0, per, lane, leader, 32, tr, dec, issue_a);
    }
  } else if (warp == 1 && leader && lane == 0) {
    const unsigned long long t0 = ptx::globaltimer();
    for (int it = 0; it < iters; ++it) rc_consume<false>(L, it, tmem, it > 0, tr);
    ptx::mma_commit_2sm_mc(&L.accf[0], 0x3);
    ptx::mbar_wait(&L.accf[0], 0);
    out[2 * p] = t0;
    out[2 * p + 1] = ptx::globaltimer();
  }
  if (warp >= 2 && warp < kRcActWarp) {
    if (storm && warp == 2 && lane == 0) {  // an epilogue thread spinning on an acquire flag (CCTL.IVALL)
      while (!ptx::mbar_test(&L.accf[0], 0)) (void)ptx::ld_acquire_gpu(flag);
    }
    ptx::mbar_wait(&L.accf[0], 0);
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc2(tmem, 512);
  }
}

static CUtensorMap make_map(void* p, long rows, long cols) {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)rows * cols * 2};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)(
      &m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

int main() {
  void *a, *b;
  const long arows = 256, acols = 4096, brows = 16384, bcols = 4096;
  cudaMalloc(&a, arows * acols * 2);
  cudaMalloc(&b, brows * bcols * 2);
  cudaMemset(a, 0, arows * acols * 2);
  cudaMemset(b, 0, brows * bcols * 2);
  const CUtensorMap ta = make_map(a, arows, acols), tb = make_map(b, brows, bcols);
  const CUtensorMap ta2 = make_map(a, arows, acols), tb2 = make_map(b, brows, bcols);
  const int smem = 2 * kMaxS * kTile + 1024;
  cudaFuncSetAttribute(stream_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, 2 * 128 * sizeof(unsigned long long));
  std::vector<unsigned long long> h(256);
  printf("%-52s %10s\n", "variant (64 pairs, 4096 k-blocks)", "us/kblock");
  for (int variant = 0; variant < 3; variant += 2)
    for (int prod : {2})
      for (int S : {5}) {
        const int bs = 0, spin = variant, maps = 0;
        Cfg cfg{S, prod, 4096, 64, bs, spin, maps};
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(128);
        lc.blockDim = dim3(128);
        lc.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&lc, stream_bench, ta, tb, ta2, tb2, cfg, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e == cudaSuccess) e = cudaGetLastError();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(h.data(), d, 2 * 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double us = 0;
        for (int p = 0; p < 64; ++p) us += (double)(h[2 * p + 1] - h[2 * p]) / 1e3;
        us /= 64;
        char name[128];
        snprintf(name, sizeof name, "%d prod, %d st, HBM B%s%s", prod, S, spin == 2 ? ", A rotated per pair" : "",
                 maps ? ", alternating maps" : "");
        printf("%-52s %10.3f\n", name, us / cfg.iters);
      }
  uint32_t* flag;
  cudaMalloc(&flag, 4);
  cudaMemset(flag, 0, 4);
  for (int storm : {0, 1})
    for (int smem_kb : {200, 226}) {
      const int sm = smem_kb * 1024 < kRcSmem ? kRcSmem : smem_kb * 1024;
      cudaFuncSetAttribute(lib_core, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(128);
      lc.blockDim = dim3(kRcThreads);
      lc.dynamicSmemBytes = sm;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&lc, lib_core, ta, tb, 4096, d, storm, flag);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("lib_core error %s\n", cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h.data(), d, 2 * 64 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double us = 0;
      for (int p = 0; p < 64; ++p) us += (double)(h[2 * p + 1] - h[2 * p]) / 1e3;
      char name[128];
      snprintf(name, sizeof name, "library core, %d KB smem%s", sm / 1024, storm ? ", acquire-spinning thread" : "");
      printf("%-52s %10.3f\n", name, us / 64 / 4096);
    }
  return 0;
}
