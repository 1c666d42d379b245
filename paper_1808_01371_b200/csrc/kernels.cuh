// kernels.cuh -- the non-GEMM kernels of the step.
//   (d)  ce_kernel / ce_reduce_kernel: fused softmax cross-entropy + BPC partials + dY over the
//        256-byte vocabulary, warp-shuffle reductions, fp32 logits, fp32/fp64 sums.
//   (e)  overflow_kernel + adam_kernel + scaler_kernel: overflow check on the reduced fp16
//        gradients, skip-and-halve / grow loss scaling, unscale + Adam on fp32
//        masters with the linear LR decay, fp16 working-copy cast.
//   plus init (Q12), state carry / reset, one-hot, TBTT gate backward of the last
//   step, weight-gradient finalisation and the per-byte segmented-sum reductions (dE, dW_x, db).
#pragma once
#include "epilogues.cuh"

namespace mlstm {

// ------------------------------------------------------------------ init (reading Q12)
__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t q) {
  uint64_t z = seed + (q + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_params_kernel(float* master, ParamOffsets po, int h, int e, uint64_t seed) {
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < po.P; q += (long)gridDim.x * blockDim.x) {
    int cols = 0;  // fan-in of the matrix holding q; 0 for biases
    if (q < po.Wmx) cols = e;
    else if (q < po.Wmh) cols = e;
    else if (q < po.Wx) cols = h;
    else if (q < po.Wh) cols = e;
    else if (q < po.b) cols = h;
    else if (q < po.Wdec) cols = 0;
    else if (q < po.bdec) cols = h;
    float w = 0.f;
    if (cols) {
      const double u = (double)(splitmix64_at(seed, (uint64_t)q) >> 11) * 0x1.0p-53;
      const double s = 1.0 / sqrt((double)cols);
      w = __double2float_rn(s * (2.0 * u - 1.0));
    }
    master[q] = w;
  }
}

// Write one master value into the fp16 (S) working copies the GEMMs read (gate-interleaved rows
// for W_x and W_h, see net.cuh).  Biases have no working copy: epilogues read the fp32 masters.
template <typename S>
__device__ __forceinline__ void store_working(const Net<S>& n, long q, float val) {
  const ParamOffsets& po = n.po;
  const int h = n.h, e = n.e;
  if (q < po.Wmx) {
    n.E_w[q] = to_s<S>(val);
  } else if (q < po.Wmh) {
    n.Wcat_w[q - po.Wmx] = to_s<S>(val);
  } else if (q < po.Wx) {
    n.Wmh_w[q - po.Wmh] = to_s<S>(val);
  } else if (q < po.Wh) {
    const long r = (q - po.Wx) / e, c = (q - po.Wx) % e;
    n.Wcat_w[((long)h + int_row((int)(r / h), (int)(r % h))) * e + c] = to_s<S>(val);
  } else if (q < po.b) {
    const long r = (q - po.Wh) / h, c = (q - po.Wh) % h;
    n.Wh_w[(long)int_row((int)(r / h), (int)(r % h)) * h + c] = to_s<S>(val);
  } else if (q >= po.Wdec && q < po.bdec) {
    n.Wdec_w[q - po.Wdec] = to_s<S>(val);
  }
}

// ------------------------------------------------------------------ weight normalisation (Q24)
// One warp per normalised row (W_mx, W_mh, W_x, W_h; w_r = g_r v_r / ||v_r||).
__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// g_r = RNE_fp32(||v_r||) with the squared sum in fp64 (function-preserving init).
__global__ void wn_init_gain_kernel(float* master, ParamOffsets po, int h, int e) {
  const int lane = threadIdx.x & 31;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < 10 * h; r += (gridDim.x * blockDim.x) >> 5) {
    long off, gi;
    int len;
    po.wn_row(h, e, r, off, len, gi);
    double ss = 0.0;
    for (int j = lane; j < len; j += 32) ss += (double)master[off + j] * master[off + j];
#pragma unroll
    for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) master[gi] = __double2float_rn(sqrt(ss));
  }
}

// ||v_r|| (fp32 squared sum; rounded to fp16 in mixed mode, "the final norm value is output
// in FP16") and the effective weights g_r v_r / ||v_r|| into the working copies.
template <typename S>
__global__ void wn_norm_kernel(Net<S> n) {
  const int lane = threadIdx.x & 31, h = n.h, e = n.e;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < 10 * h; r += (gridDim.x * blockDim.x) >> 5) {
    long off, gi;
    int len;
    n.po.wn_row(h, e, r, off, len, gi);
    float ss = 0.f;
    for (int j = lane; j < len; j += 32) ss = fmaf(n.master[off + j], n.master[off + j], ss);
    float nrm = sqrtf(warp_sum(ss));
    if (sizeof(S) == 2) nrm = __half2float(__float2half_rn(nrm));
    if (lane == 0) n.wn_norm[r] = nrm;
    const float sc = n.master[gi] / nrm;
    for (int j = lane; j < len; j += 32) store_working(n, off + j, n.master[off + j] * sc);
  }
}

// After the allreduce: the gradient w.r.t. w in the arena becomes (dv, dg) in place
// (dg_r = dw_r . v_r / ||v_r||, dv_r = (g_r / ||v_r||)(dw_r - (dg_r / ||v_r||) v_r)), alpha-scaled.
template <typename S>
__global__ void wn_grad_kernel(Net<S> n) {
  const int lane = threadIdx.x & 31, h = n.h, e = n.e;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < 10 * h; r += (gridDim.x * blockDim.x) >> 5) {
    long off, gi;
    int len;
    n.po.wn_row(h, e, r, off, len, gi);
    float dot = 0.f;
    for (int j = lane; j < len; j += 32) dot = fmaf(to_f(n.arena[off + j]), n.master[off + j], dot);
    const float nrm = n.wn_norm[r];
    const float dg = warp_sum(dot) / nrm, sc = n.master[gi] / nrm, k = dg / nrm;
    bool bad = false;
    for (int j = lane; j < len; j += 32) {
      const float gv = sc * (to_f(n.arena[off + j]) - k * n.master[off + j]);
      n.arena[off + j] = to_s<S>(gv);
      bad |= s_nonfinite<S>(gv);
    }
    if (lane == 0) {
      n.arena[gi] = to_s<S>(dg);
      bad |= s_nonfinite<S>(dg);
    }
    if (bad) n.st->overflow = 1;
  }
}

// Four consecutive parameters q..q+3 (never straddling a tensor or a row: P, e, h are multiples of
// 64) into the working copies with one vector store; 32-bit index arithmetic within a tensor.
template <typename S>
__device__ __forceinline__ void store_working4(const Net<S>& n, long q, const float* val) {
  const ParamOffsets& po = n.po;
  const int h = n.h, e = n.e;
  S* dst = nullptr;
  if (q < po.Wmx) {
    dst = n.E_w + q;
  } else if (q < po.Wmh) {
    dst = n.Wcat_w + (q - po.Wmx);
  } else if (q < po.Wx) {
    dst = n.Wmh_w + (q - po.Wmh);
  } else if (q < po.Wh) {
    const unsigned o = (unsigned)(q - po.Wx), r = o / (unsigned)e, c = o - r * (unsigned)e;
    dst = n.Wcat_w + ((long)h + int_row((int)(r / h), (int)(r % h))) * e + c;
  } else if (q < po.b) {
    const unsigned o = (unsigned)(q - po.Wh), r = o / (unsigned)h, c = o - r * (unsigned)h;
    dst = n.Wh_w + (long)int_row((int)(r / h), (int)(r % h)) * h + c;
  } else if (q >= po.Wdec && q < po.bdec) {
    dst = n.Wdec_w + (q - po.Wdec);
  }
  if (dst) st4(dst, make_float4(val[0], val[1], val[2], val[3]));
}

template <typename S>
__global__ void cast_working_kernel(Net<S> n) {
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n.po.P; q += (long)gridDim.x * blockDim.x)
    store_working(n, q, n.master[q]);
}

// dst[c][r] = src[r][c], src [R x C] row-major.
template <typename S>
__global__ void transpose_kernel(const S* __restrict__ src, S* __restrict__ dst, int R, int C) {
  __shared__ S tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < R && c < C) tile[i][threadIdx.x] = src[(long)r * C + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < R && c < C) dst[(long)c * R + r] = tile[threadIdx.x][i];
  }
}

// fp16 fast path: 64 x 64 tiles, half2 vectors on both sides (R, C multiples of 64), 32 x 8 threads.
__global__ void transpose64_kernel(const __half* __restrict__ src, __half* __restrict__ dst, int R, int C) {
  __shared__ __half tile[64][66];
  const int c0 = blockIdx.x * 64, r0 = blockIdx.y * 64;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int i = ty; i < 64; i += 8)
    *reinterpret_cast<__half2*>(&tile[i][2 * tx]) =
        *reinterpret_cast<const __half2*>(src + (long)(r0 + i) * C + c0 + 2 * tx);
  __syncthreads();
#pragma unroll
  for (int i = ty; i < 64; i += 8) {
    __half2 o;
    o.x = tile[2 * tx][i];
    o.y = tile[2 * tx + 1][i];
    *reinterpret_cast<__half2*>(dst + (long)(c0 + i) * R + r0 + 2 * tx) = o;
  }
}

// ------------------------------------------------------------------ state carry
template <typename S>
__global__ void state_in_kernel(Net<S> n, int slot) {
  const long BH = (long)n.B * n.h;
  // this micro-batch's rows of the persisted state
  const long so = (long)slot * n.Bfull * n.h + (long)n.st->mb * BH;
  if (blockIdx.x == 0 && threadIdx.x == 0) n.st->overflow = 0;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < BH; i += (long)gridDim.x * blockDim.x) {
    const int b = (int)(i / n.h), j = (int)(i % n.h);
    const bool rst = n.reset[b] != 0;
    const S hv = rst ? to_s<S>(0.f) : n.hstate[so + i];
    const float cv = rst ? 0.f : n.cstate[so + i];
    n.Hrm[i] = hv;
    n.Crm[i] = cv;
  }
}

template <typename S>
__global__ void state_out_kernel(Net<S> n, int slot) {
  const long BH = (long)n.B * n.h;
  const long so = (long)slot * n.Bfull * n.h + (long)n.st->mb * BH;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < BH; i += (long)gridDim.x * blockDim.x) {
    n.hstate[so + i] = n.Hrm[(long)n.T * BH + i];
    n.cstate[so + i] = n.Crm[(long)n.T * BH + i];
  }
}

// Sets the micro-batch index the following kernels work on.
__global__ void set_microbatch_kernel(DevState* st, int mb) { st->mb = mb; }

// Micro-batch gradient accumulation in fp32 (the paper accumulates into fp32 masters):
// gacc = (mb == 0 ? 0 : gacc) + g; after the last micro-batch the sum goes back to the fp16 arena
// (the allreduce payload; an fp16 overflow of the sum is caught by the overflow check).
template <typename S>
__global__ void grad_accum_kernel(Net<S> n) {
  const int mb = n.st->mb;
  const bool first = mb == 0, last = mb == n.nmb - 1;
  for (long q = blockIdx.x * (long)blockDim.x + threadIdx.x; q < n.po.P; q += (long)gridDim.x * blockDim.x) {
    const float g = (first ? 0.f : n.gacc[q]) + to_f(n.arena[q]);
    if (last) {
      n.arena[q] = to_s<S>(g);
      if (s_nonfinite<S>(g)) n.st->overflow = 1;
    } else {
      n.gacc[q] = g;
    }
  }
}

// One-hot of the input bytes, row-major: OHR[t][b][v] = [bytes[b][t] == v] (exact in fp16).
template <typename S>
__global__ void onehot_kernel(Net<S> n) {
  const long TB = (long)n.T * n.B;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < TB; i += (long)gridDim.x * blockDim.x) {
    const int t = (int)(i / n.B), b = (int)(i % n.B);
    const int v0 = n.byte_at(b, t);
    S* row = n.OHR + i * 256;
    for (int v = 0; v < 256; v += 4)
      st4(row + v, make_float4(v == v0 ? 1.f : 0.f, v + 1 == v0 ? 1.f : 0.f, v + 2 == v0 ? 1.f : 0.f,
                               v + 3 == v0 ? 1.f : 0.f));
  }
}

// ------------------------------------------------------------------ (d) softmax cross-entropy
// Block = 8 warps = 32 logit rows (row r = t*B + b); one warp per row, 8 logits per lane.
// loss_r = logsumexp(y_r) - y_r[target] (max-subtracted, fp32);  dY = (softmax - onehot) *
// alpha / (B_g T) (Q7).  Emits dY row-major and transposed (for dW_dec), per-block loss
// and column sums (for db_dec), all in fixed order (deterministic).
template <typename S>
__global__ void __launch_bounds__(256) ce_kernel(Net<S> n, int Be, float inv_denom, int with_grad) {
  __shared__ float tile[32][257];
  __shared__ float rl[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long R = (long)n.T * n.B;
  const long r0 = (long)blockIdx.x * 32;
  const float coef = with_grad ? n.st->alpha * inv_denom : 0.f;
#pragma unroll 1
  for (int i = 0; i < 4; ++i) {
    const int lr = warp * 4 + i;
    const long r = r0 + lr;
    const int t = r < R ? (int)(r / n.B) : 0;
    const int b = r < R ? (int)(r % n.B) : 0;
    // evaluation: rows with reset == 2 are idle loader rows (no tokens counted)
    const bool valid = r < R && b < Be && (with_grad || n.reset[b] != 2);
    float y[8];
    if (valid) {
      const float4 a = reinterpret_cast<const float4*>(n.Y + r * 256)[lane];
      const float4 c = reinterpret_cast<const float4*>(n.Y + r * 256 + 128)[lane];
      y[0] = a.x; y[1] = a.y; y[2] = a.z; y[3] = a.w;
      y[4] = c.x; y[5] = c.y; y[6] = c.z; y[7] = c.w;
    } else {
#pragma unroll
      for (int k = 0; k < 8; ++k) y[k] = 0.f;
    }
    float mx = y[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) mx = fmaxf(mx, y[k]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float ex[8], se = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      ex[k] = expf(y[k] - mx);
      se += ex[k];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const int tgt = valid ? n.byte_at(b, t + 1) : 0;
    const int within = tgt & 127, owner = within >> 2, comp = (tgt >> 7) * 4 + (within & 3);
    float sel = y[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) sel = (k == comp) ? y[k] : sel;
    const float yt = __shfl_sync(0xffffffffu, sel, owner);
    const float loss = valid ? (mx + logf(se)) - yt : 0.f;
    if (lane == 0) {
      rl[lr] = loss;
      if (r < R) n.lossrow[r] = loss;
    }
    if (with_grad) {
      const float inv = 1.f / se;
      float g[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int col = (k < 4) ? lane * 4 + k : 128 + lane * 4 + (k - 4);
        float p = ex[k] * inv;
        if (col == tgt) p -= 1.f;
        g[k] = valid ? p * coef : 0.f;
        tile[lr][col] = g[k];
      }
      if (r < R) {
        S* drow = n.dY + r * 256;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          drow[lane * 4 + k] = to_s<S>(g[k]);
          drow[128 + lane * 4 + k] = to_s<S>(g[4 + k]);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < 32; ++i) s += (double)rl[i];
    n.loss_part[blockIdx.x] = s;
  }
  if (with_grad) {
    {
      const int v = threadIdx.x;
      float s = 0.f;
      for (int i = 0; i < 32; ++i) s += tile[i][v];
      n.colsum_part[(long)blockIdx.x * 256 + v] = s;
    }
  }
}

// Final fixed-order reductions of the CE partials: block 0 sums the loss partials into
// st->loss_sum; with_grad: block 1 + v sums column v of the db_dec partials (strided per thread,
// then a fixed-shape tree: deterministic).  Grid = 1 + 256 * with_grad blocks of 256 threads.
// Evaluation token count: T positions per row b < Be whose reset flag is not 2 (idle loader rows).
template <typename S>
__global__ void eval_tokens_kernel(Net<S> n, int Be, double* tok) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  int mine = 0;
  for (int b = threadIdx.x; b < Be; b += blockDim.x) mine += n.reset[b] != 2;
  atomicAdd(&cnt, mine);
  __syncthreads();
  if (threadIdx.x == 0) *tok = (double)cnt * n.T;
}

template <typename S>
__global__ void __launch_bounds__(256) ce_reduce_kernel(Net<S> n, int nblk, int with_grad) {
  __shared__ double red[256];
  double s = 0.0;
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i < nblk; i += 256) s += n.loss_part[i];
  } else {
    const int v = blockIdx.x - 1;
    for (int i = threadIdx.x; i < nblk; i += 256) s += (double)n.colsum_part[(long)i * 256 + v];
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) n.st->loss_sum = (n.st->mb == 0 ? 0.0 : n.st->loss_sum) + red[0];
    else {
      n.arena[n.po.bdec + blockIdx.x - 1] = to_s<S>((float)red[0]);
      if (s_nonfinite<S>((float)red[0])) n.st->overflow = 1;
    }
  }
}

// ------------------------------------------------------------------ (c-1) TBTT start of BPTT
// Gate backward of the last step s = T-1: dH = dH_dec only, dC carry = 0 (memset before).
template <typename S>
__global__ void gate_bwd_last_kernel(Net<S> n) {
  const int nblk = n.h / 16;
  const long total = (long)n.B * nblk;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int b = (int)(i / nblk), j0 = (int)(i % nblk) * 16;
    const int s = n.T - 1;
    float dh[16];
    ld16(n.dHdec + ((long)s * n.B + b) * n.h + j0, dh);
    gate_bwd16(n, s, b, j0, dh);
  }
}

// ------------------------------------------------------------------ (c-2) weight gradients
// Store modes: 0 = identity into the arena at `off`; 1 = W_h rows internal -> canonical;
// 2 = per-byte segmented sums into Scan[256][5h] with canonical columns.
__device__ __forceinline__ long wgrad_col_canon(int mode, int c, int h) {
  return (mode == 2 && c >= h) ? (long)h + canon_of_int(c - h, h) : c;
}

template <typename S>
struct EpiWgrad {
  static constexpr int kMinGroups = 1;  // 16-column groups one call must cover
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  Net<S> n;
  long off;
  int mode;
  int N;
  int row0 = 0;  // first output row of this launch (dW_h split into row halves for the allreduce)
  const float* acc = nullptr;  // fp32 partial of the K range the side stream reduced (EpiWacc), added first
  template <int NG>
  __device__ __forceinline__ void run(int row_, int col0, const float* v_) const {
    const int row = row_ + row0;
    float w[16 * NG];
    const float* v = v_;
    if (acc) {
      const float4* a = reinterpret_cast<const float4*>(acc + (long)row * N + col0);
#pragma unroll
      for (int q = 0; q < 4 * NG; ++q) {
        const float4 x = a[q];
        w[4 * q] = v_[4 * q] + x.x;
        w[4 * q + 1] = v_[4 * q + 1] + x.y;
        w[4 * q + 2] = v_[4 * q + 2] + x.z;
        w[4 * q + 3] = v_[4 * q + 3] + x.w;
      }
      v = w;
    }
    if (mode == 2) {
      float* dst = n.Scan + (long)row * 5 * n.h;
#pragma unroll
      for (int i = 0; i < 16 * NG; ++i) dst[wgrad_col_canon(2, col0 + i, n.h)] = v[i];
      return;
    }
    const long r = (mode == 1) ? canon_of_int(row, n.h) : row;
    S* dst = n.arena + off + r * N + col0;
#pragma unroll
    for (int q = 0; q < NG; ++q) st16(dst + 16 * q, v + 16 * q);
    bool bad = false;  // overflow predicate at the writer (the separate scan runs only when world > 1)
#pragma unroll
    for (int i = 0; i < 16 * NG; ++i) bad |= s_nonfinite<S>(v[i]);
    if (bad) n.st->overflow = 1;
  }
};

// fp32 partial of a weight gradient over one K range (a chunk of timesteps), reduced on the side stream
// while the backward recurrence still runs: [M][N] internal rows, the first chunk stores, later ones add
// (the side stream runs them in order); EpiWgrad adds the result to the remaining K range's sum.
struct EpiWacc {
  static constexpr int kMinGroups = 1;
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  float* part;
  int N;
  int first;
  template <int NG>
  __device__ __forceinline__ void run(int row, int col0, const float* v) const {
    float4* d = reinterpret_cast<float4*>(part + (long)row * N + col0);
#pragma unroll
    for (int q = 0; q < 4 * NG; ++q) {
      float4 x = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
      if (!first) {
        const float4 o = d[q];
        x.x += o.x;
        x.y += o.y;
        x.z += o.z;
        x.w += o.w;
      }
      d[q] = x;
    }
  }
};

template <typename S>
__global__ void wgrad_finalize_kernel(Net<S> n, const float* __restrict__ part, int splits, int M, int N, long off,
                                      int mode) {
  const long MN = (long)M * N;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < MN; i += (long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[z * MN + i];
    const int row = (int)(i / N), col = (int)(i % N);
    if (mode == 2) {
      n.Scan[(long)row * 5 * n.h + wgrad_col_canon(2, col, n.h)] = s;
    } else {
      const long r = (mode == 1) ? canon_of_int(row, n.h) : row;
      n.arena[off + r * N + col] = to_s<S>(s);
      if (s_nonfinite<S>(s)) n.st->overflow = 1;
    }
  }
}

// Small fp32 SIMT GEMM for the per-byte segmented-sum products (fp32 operands: S holds sums of up
// to B*T alpha-scaled gradients and may exceed the fp16 range).  part[z] = sum_k A(m, k) B(k, n)
// over split z; 64 x 64 tile, 256 threads x (4 x 4) outputs, K staged 32 at a time.
//   MODE 0 (dE):    A(m=v, k=r) = Scan[v][r],  B(k=r, n=c) = [W_mx; W_x]_canonical[r][c]
//   MODE 1 (dWcat): A(m=r, k=v) = Scan[v][r],  B(k=v, n=c) = E[v][c]
template <typename S, int MODE>
__global__ void __launch_bounds__(256) seg_gemm_kernel(Net<S> n, float* __restrict__ part, int M, int N, int K,
                                                       int k_per_split) {
  __shared__ float As[32][64 + 4];
  __shared__ float Bs[32][64 + 4];
  const int h = n.h, e = n.e, R = 5 * h;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int kbeg = blockIdx.z * k_per_split, kend = min(K, kbeg + k_per_split);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  for (int k0 = kbeg; k0 < kend; k0 += 32) {
    for (int i = threadIdx.x; i < 32 * 64; i += 256) {
      int kk, mm;
      if (MODE == 0) { mm = i >> 5; kk = i & 31; }   // Scan[v][r] with v = m: coalesce over k
      else { kk = i >> 6; mm = i & 63; }             // Scan[v][r] with r = m: coalesce over m
      const int gm = m0 + mm, gk = k0 + kk;
      float a = 0.f;
      if (gm < M && gk < kend) a = (MODE == 0) ? n.Scan[(long)gm * R + gk] : n.Scan[(long)gk * R + gm];
      As[kk][mm] = a;
    }
    for (int i = threadIdx.x; i < 32 * 64; i += 256) {
      const int kk = i >> 6, nn = i & 63, gk = k0 + kk, gn = n0 + nn;
      float bv = 0.f;
      if (gk < kend && gn < N) {
        if (MODE == 0) {
          const long wrow = (gk < h) ? gk : (long)h + int_row((gk - h) / h, (gk - h) % h);
          bv = to_f(n.Wcat_w[wrow * e + gn]);
        } else {
          bv = to_f(n.E_w[(long)gk * e + gn]);
        }
      }
      Bs[kk][nn] = bv;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      float a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* dst = part + (long)blockIdx.z * M * N;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gm = m0 + ty * 4 + i, gn = n0 + tx * 4 + j;
      if (gm < M && gn < N) dst[(long)gm * N + gn] = acc[i][j];
    }
}

// Sums the split-K partials in order and stores dE (MODE 0) or [dW_mx; dW_x] (MODE 1) in the arena.
template <typename S, int MODE>
__global__ void seg_finalize_kernel(Net<S> n, const float* __restrict__ part, int splits, int M, int N) {
  const long MN = (long)M * N;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < MN; i += (long)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += part[z * MN + i];
    const int r = (int)(i / N), c = (int)(i % N);
    long dst;
    if (MODE == 0) dst = n.po.E + i;
    else dst = (r < n.h) ? n.po.Wmx + (long)r * n.e + c : n.po.Wx + (long)(r - n.h) * n.e + c;
    n.arena[dst] = to_s<S>(s);
    if (s_nonfinite<S>(s)) n.st->overflow = 1;
  }
}

// db = sum_v S_x[v].
template <typename S>
__global__ void db_kernel(Net<S> n) {
  const int h = n.h;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < 4 * h; r += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int v = 0; v < 256; ++v) s += n.Scan[(long)v * 5 * h + h + r];
    n.arena[n.po.b + r] = to_s<S>(s);
    if (s_nonfinite<S>(s)) n.st->overflow = 1;
  }
}

// ------------------------------------------------------------------ (e) optimiser
__device__ __forceinline__ bool nonfinite_bits(__half x) {
  return (__half_as_ushort(x) & 0x7C00u) == 0x7C00u;
}
__device__ __forceinline__ bool nonfinite_bits(float x) {
  return (__float_as_uint(x) & 0x7F800000u) == 0x7F800000u;
}

// "checking for an overflow in the weight gradients": any inf/NaN in the buffer.
template <typename S>
__global__ void overflow_kernel(const S* __restrict__ buf, long count, int32_t* flag) {
  bool bad = false;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x)
    bad |= nonfinite_bits(buf[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

// Unscale + Adam on fp32 masters + fp16 working-copy cast; a no-op when the step overflowed.
template <typename S>
__device__ __forceinline__ void load4(const S* p, float* g);
template <>
__device__ __forceinline__ void load4<__half>(const __half* p, float* g) {
  const uint2 w = *reinterpret_cast<const uint2*>(p);
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
  g[0] = a.x; g[1] = a.y; g[2] = b.x; g[3] = b.y;
}
template <>
__device__ __forceinline__ void load4<float>(const float* p, float* g) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  g[0] = v.x; g[1] = v.y; g[2] = v.z; g[3] = v.w;
}

// Unscale + Adam on fp32 masters + fp16 working-copy cast, 4 consecutive parameters per thread
// (P, e, h are multiples of 64, so a group never straddles a tensor or a row); a no-op when the
// step overflowed.
template <typename S>
__global__ void adam_kernel(Net<S> n, float* __restrict__ m, float* __restrict__ v, float beta1, float beta2,
                            float eps, double lr0, long decay) {
  const DevState* st = n.st;
  if (st->overflow) return;
  const float inv_alpha = 1.f / st->alpha;  // alpha is a power of two: exact
  const long tau = st->tau + 1;
  const double lr = lr0 * fmax(0.0, 1.0 - (double)st->it / (double)decay);
  const float bc1 = (float)(1.0 - pow((double)beta1, (double)tau));
  const float bc2 = (float)(1.0 - pow((double)beta2, (double)tau));
  const float lrf = (float)lr;
  const long P4 = n.po.P / 4;
  for (long q4 = blockIdx.x * (long)blockDim.x + threadIdx.x; q4 < P4; q4 += (long)gridDim.x * blockDim.x) {
    const long q = q4 * 4;
    float g[4];
    load4<S>(n.arena + q, g);
    float4 mm = reinterpret_cast<const float4*>(m)[q4];
    float4 vv = reinterpret_cast<const float4*>(v)[q4];
    float4 th = reinterpret_cast<const float4*>(n.master)[q4];
    float* mp = &mm.x;
    float* vp = &vv.x;
    float* tp = &th.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float gi = g[i] * inv_alpha;
      mp[i] = beta1 * mp[i] + (1.f - beta1) * gi;
      vp[i] = beta2 * vp[i] + (1.f - beta2) * gi * gi;
      tp[i] = tp[i] - lrf * (mp[i] / bc1) / (sqrtf(vp[i] / bc2) + eps);
    }
    reinterpret_cast<float4*>(m)[q4] = mm;
    reinterpret_cast<float4*>(v)[q4] = vv;
    reinterpret_cast<float4*>(n.master)[q4] = th;
    // normalised rows get their working copies from wn_norm_kernel once the whole row is updated
    if (!(n.po.wn && q >= n.po.Wmx && q < n.po.b)) store_working4(n, q, tp);
  }
}

// Loss-scale state machine + LR clock / Adam count (Q10).  One thread.
__global__ void scaler_kernel(DevState* st, float smin, float smax, int interval, double lr0, long decay) {
  const int ovf = st->overflow;
  st->alpha_used = st->alpha;
  st->lr_used = lr0 * fmax(0.0, 1.0 - (double)st->it / (double)decay);
  st->skipped = ovf;
  if (ovf) {
    st->alpha = fmaxf(st->alpha * 0.5f, smin);
    st->clean = 0;
  } else {
    st->tau += 1;
    st->clean += 1;
    if (st->clean >= interval) {
      st->alpha = fminf(st->alpha * 2.f, smax);
      st->clean = 0;
    }
  }
  st->it += 1;
}

// Debug: X = E_w[bytes] as the kernels index it ([T][B][e], fp32).
template <typename S>
__global__ void gather_x_kernel(Net<S> n, float* out) {
  const long total = (long)n.T * n.B * n.e;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const long tb = i / n.e;
    const int c = (int)(i % n.e), t = (int)(tb / n.B), b = (int)(tb % n.B);
    out[i] = to_f(n.E_w[(long)n.byte_at(b, t) * n.e + c]);
  }
}

// Deterministic pseudo-random fp16 fill in [-1, 1) (benchmark operands: realistic bit toggling).
__global__ void random_half_kernel(__half* p, long count, uint64_t seed) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x) {
    const double u = (double)(splitmix64_at(seed, (uint64_t)i) >> 11) * 0x1.0p-53;
    p[i] = __float2half_rn((float)(2.0 * u - 1.0));
  }
}

template <typename S>
__global__ void to_float_kernel(const S* __restrict__ src, float* __restrict__ dst, long count) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x)
    dst[i] = to_f(src[i]);
}
template <typename S>
__global__ void from_float_kernel(const float* __restrict__ src, S* __restrict__ dst, long count) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x)
    dst[i] = to_s<S>(src[i]);
}

}  // namespace mlstm
