// net.cuh -- device view of the step's HBM layout and the small helpers every kernel shares.
//
// Notation follows the paper / SURVEY §8a: h hidden width, e embedding width, B rows per rank,
// T TBTT window, S the storage type (__half in mixed mode, float in fp32 mode).
//
// Internal gate order.  The 4h gate rows of W_h / W_x (canonical order i | f | o | u, each h rows)
// are stored interleaved in blocks of 16 units: internal row r = (j/16)*64 + g*16 + j%16 for gate
// g in {i,f,o,u} and unit j.  A 64-column chunk of any gate-producing GEMM therefore holds all
// four gates of 16 units, so the gate nonlinearity and cell update fuse into that GEMM's
// epilogue with no cross-thread exchange (one TMEM lane = one batch row).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>
#include "ptx.cuh"

namespace mlstm {

// Async row I/O for epilogues that declare kAsyncIO: after the main loop the pipeline stages are
// idle, so each epilogue warp gets a private staging window there (kWarpStage bytes) plus an
// mbarrier for its loads.  Inputs come in by per-row bulk copies (issued before the accumulator is
// read, so their latency overlaps the TMEM loads / split-K reduction); outputs are written to the
// window and leave by per-row bulk copies -- no 32-line LSU wavefronts per warp instruction.
constexpr int kWarpStageBytes = 24 * 1024;
struct EpiIO {
  uint8_t* buf;   // this warp's staging window (16-byte aligned)
  uint64_t* bar;  // this warp's load barrier (count 32: every lane arrives once per launch)
  int row0;       // accumulator row of lane 0
  int nvalid;     // rows of this warp inside M: lane < nvalid
  int lane;
  __device__ __forceinline__ bool valid() const { return lane < nvalid; }
};

__host__ __device__ __forceinline__ int int_row(int g, int j) { return (j >> 4) * 64 + g * 16 + (j & 15); }
__host__ __device__ __forceinline__ int canon_of_int(int r, int h) {
  return ((r >> 4) & 3) * h + (r >> 6) * 16 + (r & 15);
}

// Canonical flat parameter offsets (include/mlstm.h).
struct ParamOffsets {
  long E, Wmx, Wmh, Wx, Wh, b, Wdec, bdec, P;
  long g;  // weight normalisation (Q24): gains g_mx[h] | g_mh[h] | g_x[4h] | g_h[4h] appended at `g`
  int wn;  // weight normalisation on?
  __host__ __device__ void set(int h, int e, int weight_norm = 0) {
    E = 0;
    Wmx = E + 256L * e;
    Wmh = Wmx + (long)h * e;
    Wx = Wmh + (long)h * h;
    Wh = Wx + 4L * h * e;
    b = Wh + 4L * h * h;
    Wdec = b + 4L * h;
    bdec = Wdec + 256L * h;
    g = bdec + 256;
    wn = weight_norm;
    P = g + (weight_norm ? 10L * h : 0);
  }
  // normalised row r in [0, 10h): its first element, length and gain index (canonical order)
  __host__ __device__ void wn_row(int h, int e, int r, long& off, int& len, long& gi) const {
    if (r < h) { off = Wmx + (long)r * e; len = e; }
    else if (r < 2 * h) { off = Wmh + (long)(r - h) * h; len = h; }
    else if (r < 6 * h) { off = Wx + (long)(r - 2 * h) * e; len = e; }
    else { off = Wh + (long)(r - 6 * h) * h; len = h; }
    gi = g + r;
  }
};

// Device-resident scalar state: loss-scale state machine, LR clock and Adam count (Q10).
struct DevState {
  double loss_sum;     // global sum of per-position CE of the last step (after allreduce)
  double lr_used;      // LR the last step used
  float alpha;         // current loss scale
  float alpha_used;    // loss scale the last step's backward used
  int32_t overflow;    // set by the overflow scan of the reduced gradients
  int32_t clean;       // clean steps since the last growth / backoff
  int64_t it;          // LR clock: advances every step (incl. skipped)
  int64_t tau;         // applied Adam updates
  int32_t skipped;     // last step skipped?
  int32_t mb;          // micro-batch index being processed (rows [mb*B, (mb+1)*B) of the rank's batch)
};

template <typename S>
struct Net {
  int h, e, B, T, Bp;
  int Bfull, nmb;  // rows per rank and micro-batches per step (B = Bfull / nmb rows per micro-batch)
  ParamOffsets po;
  const uint8_t* bytes;  // [B][T+1]
  const uint8_t* reset;  // [B] or null
  float* master;         // fp32 masters, canonical (biases are read from here)
  S* arena;              // gradient buckets, canonical layout (fp16 in mixed mode)
  // fp16 (S) working copies
  S *E_w, *Wcat_w, *Wmh_w, *Wh_w, *Wdec_w, *WmhT, *WhT, *WdecT;
  // activations / stash
  float* tab;     // [256][5h]: cols [0,h) = W_mx E^T (mx table), [h,5h) = W_x E^T in internal order
  S* XZT;         // [4h][256] (W_x E^T + b)^T in internal row order: F2's second K segment (mixed mode)
  S* OHR;         // [T][B][256] one-hot of the input bytes: F2's second A segment (tcgen05 path) and the
                  // MN-major A operand of the per-byte sums S = onehot^T [dMX | dZ]
  S* Hrm;         // [(T+1)][B][h]; block 0 = h0, block t+1 = H_t
  float* Crm;     // [(T+1)][B][h]
  S* Mrm;         // [T][B][h] m_t: A operand of F2 at t; MN-major B operand of dW_h = dZ^T M
  S* Astash;      // [T][B][h] a_t = W_mh h_{t-1}
  S* Gates;       // [T][B][4h] i,f,o,u activations, internal order
  float* Y;       // [T*B][256] logits (fp32)
  float* lossrow; // [T*B]
  S* dY;          // [T*B][256]
  float* dHdec;   // [T*B][h] (SIMT path only; null when B2 folds dY W_dec into its K loop)
  S* G5;          // [T][B][5h]: cols [0,h) dMX, [h,5h) dZ (internal order); dZ_t is B1's A operand,
                  // the whole stash the MN-major operand of dW_h (dZ) and of the per-byte sums
  S* dA;          // [T][B][h] dA_t: B2's A operand at t; MN-major A operand of dW_mh
  float* dC;      // [B][h] dc carry
  float* part;    // split-K partials
  float* Scan;    // [256][5h] per-byte segmented sums, canonical columns
  S* hstate;      // [2][Bfull][h]  persisted h per slot
  float* cstate;  // [2][Bfull][h]  persisted c per slot
  float* gacc;    // [P] fp32 gradient accumulator across micro-batches (nmb > 1)
  float* wn_norm; // [10h] ||v_r|| of the normalised rows (fp32 sum; fp16-rounded in mixed mode)
  double* loss_part;
  float* colsum_part;
  DevState* st;
  __device__ __forceinline__ int byte_at(int b, int t) const { return bytes[(long)b * (T + 1) + t]; }
};

template <typename S>
__device__ __forceinline__ S to_s(float x);
template <>
__device__ __forceinline__ __half to_s<__half>(float x) {
  return __float2half_rn(x);
}
template <>
__device__ __forceinline__ float to_s<float>(float x) {
  return x;
}
// Whether the fp32 value v is non-finite once stored as S (the overflow predicate of P:126 applied at
// the writer): binary16 RNE sends |v| >= 65520 to inf (65504 is the largest finite), NaN stays NaN.
template <typename S>
__device__ __forceinline__ bool s_nonfinite(float v);
template <>
__device__ __forceinline__ bool s_nonfinite<__half>(float v) {
  return !(fabsf(v) < 65520.f);
}
template <>
__device__ __forceinline__ bool s_nonfinite<float>(float v) {
  return !(fabsf(v) <= 3.402823466e38f);
}
__device__ __forceinline__ float to_f(__half x) { return __half2float(x); }
__device__ __forceinline__ float to_f(float x) { return x; }

// Contiguous stores / loads of 16 values (rows are 16-element aligned by construction).
__device__ __forceinline__ void st16(__half* dst, const float* v) {
  uint4 w[2];
  __half2* p = reinterpret_cast<__half2*>(w);
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
  reinterpret_cast<uint4*>(dst)[0] = w[0];
  reinterpret_cast<uint4*>(dst)[1] = w[1];
}
__device__ __forceinline__ void st16(float* dst, const float* v) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}
__device__ __forceinline__ void ld16(const __half* src, float* v) {
  uint4 w[2];
  w[0] = reinterpret_cast<const uint4*>(src)[0];
  w[1] = reinterpret_cast<const uint4*>(src)[1];
  const __half2* p = reinterpret_cast<const __half2*>(w);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float2 f = __half22float2(p[i]);
    v[2 * i] = f.x;
    v[2 * i + 1] = f.y;
  }
}
__device__ __forceinline__ void ld16(const float* src, float* v) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 f = reinterpret_cast<const float4*>(src)[i];
    v[4 * i] = f.x;
    v[4 * i + 1] = f.y;
    v[4 * i + 2] = f.z;
    v[4 * i + 3] = f.w;
  }
}

// 4 consecutive values (8-byte fp16 / 16-byte fp32 vectors; callers keep them aligned).
__device__ __forceinline__ float4 ld4(const __half* p) {
  const uint2 w = *reinterpret_cast<const uint2*>(p);
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&w.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&w.y));
  return make_float4(a.x, a.y, b.x, b.y);
}
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(__half* p, float4 v) {
  uint2 w;
  *reinterpret_cast<__half2*>(&w.x) = __floats2half2_rn(v.x, v.y);
  *reinterpret_cast<__half2*>(&w.y) = __floats2half2_rn(v.z, v.w);
  *reinterpret_cast<uint2*>(p) = w;
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
// 4 values to shared memory at a 2-element-aligned address (fp16: two 4-byte stores).
__device__ __forceinline__ void st4s(__half* p, float4 v) {
  reinterpret_cast<__half2*>(p)[0] = __floats2half2_rn(v.x, v.y);
  reinterpret_cast<__half2*>(p)[1] = __floats2half2_rn(v.z, v.w);
}
__device__ __forceinline__ void st4s(float* p, float4 v) {
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
  p[3] = v.w;
}

__device__ __forceinline__ float sigmoidf_(float x) { return 1.f / (1.f + expf(-x)); }

// Gate nonlinearities.  Mixed mode (S = __half): the hardware tanh.approx.f32 (MUFU, max relative
// error ~2^-11, below the fp16 resolution the gates are stored at) and sigma(x) = tanh(x/2)/2 + 1/2.
// fp32 parity mode (S = float): IEEE expf/tanhf.
__device__ __forceinline__ float tanh_approx(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <typename S>
__device__ __forceinline__ float act_tanh(float x) {
  return tanhf(x);
}
template <>
__device__ __forceinline__ float act_tanh<__half>(float x) {
  return tanh_approx(x);
}
template <typename S>
__device__ __forceinline__ float act_sigmoid(float x) {
  return sigmoidf_(x);
}
template <>
__device__ __forceinline__ float act_sigmoid<__half>(float x) {
  return fmaf(0.5f, tanh_approx(0.5f * x), 0.5f);
}

}  // namespace mlstm
