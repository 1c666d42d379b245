// tma_bench.cu -- microbenchmark of TMA load throughput per SM on the recurrence's operand shapes
// (tools only; not part of the library).  One producer thread per CTA streams 64 x R fp16 boxes
// (128-byte rows, SW128) from a [rows x 4096] tensor into a ring of S stages; one consumer thread
// releases each stage as soon as it is full.  Reports bytes per microsecond per CTA and the mean
// duration of the TMA issue instruction.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1808_01371_b200/csrc
//        tools/tma_bench.cu -o /tmp/tma_bench -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cudaTypedefs.h>

#include "ptx.cuh"

using namespace mlstm;

constexpr int S = 6;

struct Cfg {
  int boxes;   // boxes per stage (1 or 2: A then B)
  int shared;  // 1: every CTA reads the same rows (L2-hot); 0: CTA c reads rows [128c, +128) (+ B rows)
  int pair;    // 0: 1-CTA loads; 1: 2-SM loads (cta_group::2), both CTAs arrive on the leader's barrier;
               // 2: 1-CTA loads in both CTAs, the peer forwards its local completion to the leader;
               // 3: 2-SM loads, the leader's arrive expects both CTAs' bytes (the GEMM engine's form)
  int kblocks; // k-blocks per row before wrapping
  int iters;
};

__global__ void __launch_bounds__(96, 1) tma_bench(const __grid_constant__ CUtensorMap tA,
                                                   const __grid_constant__ CUtensorMap tB, Cfg cfg,
                                                   unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S], empty[S], pfull[S];
  const int tile = 16384;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t rank = cfg.pair ? ptx::cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      ptx::mbar_init(&full[s], (cfg.pair == 1 || cfg.pair == 2 || cfg.pair == 4) ? 2 : 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&pfull[s], 1);
    }
    ptx::fence_barrier_init();
  }
  if (cfg.pair) ptx::cluster_sync();
  else __syncthreads();
  const int cta = blockIdx.x;
  const int row0 = cfg.shared ? 0 : 128 * cta;
  unsigned long long issue_ns = 0, t_begin = 0, t_end = 0;
  const uint32_t bytes = cfg.boxes * tile * (cfg.pair ? 2 : 1);
  if (warp == 0 && lane == 0) {
    const uint32_t bar0 = cfg.pair ? ptx::mapa_shared(ptx::smem_u32(&full[0]), 0) : ptx::smem_u32(&full[0]);
    const uint64_t pol = ptx::make_policy(0);
    t_begin = ptx::globaltimer();
    for (int i = 0; i < cfg.iters; ++i) {
      const int s = i % S;
      if (i >= S) ptx::mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
      const long long c0 = clock64();
      const int kb = i % cfg.kblocks;
      uint8_t* dst = sm + s * cfg.boxes * tile;
      if (cfg.pair == 1 || cfg.pair == 3) {
        if (rank == 0) ptx::mbar_arrive_expect_tx(&full[s], bytes);
        else if (cfg.pair == 1) ptx::mbar_arrive_remote(bar0 + 8 * s);
        ptx::tma_load_3d_2sm(dst, &tA, bar0 + 8 * s, 64 * kb, row0, 0, pol);
        if (cfg.boxes == 2) ptx::tma_load_3d_2sm(dst + tile, &tB, bar0 + 8 * s, 64 * kb, row0, 0, pol);
      } else if (cfg.pair == 4) {
        ptx::mbar_arrive_expect_tx(&full[s], tile);
        ptx::tma_load_3d(dst, &tA, &full[s], 64 * kb, row0, 0, pol);
      } else {
        uint64_t* fb = (cfg.pair == 2 && rank == 1) ? &pfull[s] : &full[s];
        ptx::mbar_arrive_expect_tx(fb, cfg.boxes * tile);
        ptx::tma_load_3d(dst, &tA, fb, 64 * kb, row0, 0, pol);
        if (cfg.boxes == 2) ptx::tma_load_3d(dst + tile, &tB, fb, 64 * kb, row0, 0, pol);
      }
      issue_ns += clock64() - c0;
    }
  } else if (warp == 2 && lane == 0 && cfg.pair == 4) {  // second producer: box B of every stage
    const uint64_t pol = ptx::make_policy(0);
    long long iss = 0;
    for (int i = 0; i < cfg.iters; ++i) {
      const int s = i % S;
      if (i >= S) ptx::mbar_wait(&empty[s], ((i / S) & 1) ^ 1);
      const long long c0 = clock64();
      ptx::mbar_arrive_expect_tx(&full[s], tile);
      ptx::tma_load_3d(sm + s * cfg.boxes * tile + tile, &tB, &full[s], 64 * (i % cfg.kblocks), row0, 0, pol);
      iss += clock64() - c0;
    }
    out[3 * 256 + cta] = iss;
  } else if (warp == 1 && lane == 0) {
    if (rank == 0) {
      for (int i = 0; i < cfg.iters; ++i) {
        const int s = i % S;
        ptx::mbar_wait(&full[s], (i / S) & 1);
        ptx::mbar_arrive(&empty[s]);
        if (cfg.pair) ptx::mbar_arrive_remote(ptx::mapa_shared(ptx::smem_u32(&empty[s]), 1));
      }
      t_end = ptx::globaltimer();
    } else if (cfg.pair == 2) {  // forward the peer's local completion to the leader's barrier
      const uint32_t bar0 = ptx::mapa_shared(ptx::smem_u32(&full[0]), 0);
      for (int i = 0; i < cfg.iters; ++i) {
        const int s = i % S;
        ptx::mbar_wait(&pfull[s], (i / S) & 1);
        ptx::mbar_arrive_remote(bar0 + 8 * s);
      }
    }
  }
  if (warp == 0 && lane == 0) {
    out[3 * cta + 0] = issue_ns;
    out[3 * cta + 1] = t_begin;
  }
  if (warp == 1 && lane == 0 && rank == 0) out[3 * cta + 2] = t_end;
  if (cfg.pair) ptx::cluster_sync();
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

static CUtensorMap make_map(void* p, long rows, long cols) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, (cuuint64_t)rows * cols * 2};
  cuuint32_t box[3] = {64, 128, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return m;
}

int main() {
  const long rows = 16384, cols = 4096;
  void *a, *b;
  cudaMalloc(&a, rows * cols * 2);
  cudaMalloc(&b, rows * cols * 2);
  cudaMemset(a, 0, rows * cols * 2);
  cudaMemset(b, 0, rows * cols * 2);
  const CUtensorMap ta = make_map(a, rows, cols), tb = make_map(b, rows, cols);
  const int smem = S * 2 * 16384 + 1024;
  cudaFuncSetAttribute(tma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d_out;
  cudaMalloc(&d_out, 4 * 256 * sizeof(unsigned long long));
  std::vector<unsigned long long> h(4 * 256);
  printf("%-44s %10s %12s %12s\n", "variant", "ctas", "GB/s per CTA", "issue cyc");
  for (int grid : {128})
    for (int pair : {0, 4, 3})
      for (int boxes : {2})
        for (int shared : {0, 1}) {
          Cfg cfg{boxes, shared, pair, 64, 4096};
          cudaLaunchConfig_t lc{};
          lc.gridDim = dim3(grid);
          lc.blockDim = dim3(96);
          lc.dynamicSmemBytes = smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = 2;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          lc.attrs = at;
          lc.numAttrs = 1;
          for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&lc, tma_bench, ta, tb, cfg, d_out);
          cudaError_t e = cudaDeviceSynchronize();
          if (e == cudaSuccess) e = cudaGetLastError();
          if (e != cudaSuccess) {
            printf("error %s\n", cudaGetErrorString(e));
            return 1;
          }
          cudaMemcpy(h.data(), d_out, 4 * 256 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
          double gbs = 0, iss = 0;
          int n = 0;
          for (int c = 0; c < grid; ++c) {
            const int lead = pair ? (c & ~1) : c;
            const double us = ((double)h[3 * lead + 2] - (double)h[3 * c + 1]) / 1e3;
            if (c == 0 && !(us > 0)) printf("  raw: issue %llu begin %llu end %llu\n", h[0], h[1], h[2]);
            gbs += (double)cfg.iters * boxes * 16384 / us / 1e3;
            iss += (double)h[3 * c] / cfg.iters;
            if (pair == 4) iss += (double)h[3 * 256 + c] / cfg.iters / 1e6;  // second producer: printed below
            ++n;
          }
          char name[128];
          const char* pn[5] = {"1-CTA", "2-SM both arrive", "1-CTA + fwd", "2-SM leader tx", "1-CTA 2 producers"};
          snprintf(name, sizeof name, "%s %d box/stage %s", pn[pair], boxes,
                   shared ? "same rows (L2-hot)" : "own rows (DRAM)");
          printf("%-44s %10d %12.1f %12.0f", name, grid, gbs / n, iss / n);
          if (pair == 4) printf("   (producer B: %.0f cyc)", (double)h[3 * 256] / cfg.iters);
          printf("\n");
        }
  return 0;
}
