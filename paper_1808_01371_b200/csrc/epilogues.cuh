// epilogues.cuh -- the fused GEMM epilogues of the step.
//
// Every functor is called by one thread for one accumulator row and 64 consecutive columns:
//   (row, col0, v[0..63]) with v = fp32 accumulator values.  Rows of the per-timestep GEMMs are
//   batch rows b; columns are hidden units (N = h) or internal gate rows (N = 4h).
#pragma once
#include "net.cuh"

#ifndef MLSTM_TILE_EPI
#define MLSTM_TILE_EPI 0  // row epilogues measured faster (profiles/r01_epilogue_ab.log)
#endif

namespace mlstm {

// (a) input-projection table: tab[v][:] = [W_mx E[v] | W_x E[v]]  (the per-token input GEMM of
// every timestep, done once per step for the 256 possible bytes; gathered by byte below).
template <typename S>
struct EpiTab {
  Net<S> n;
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const {
    float* dst = n.tab + (long)row * 5 * n.h + col0;
#pragma unroll
    for (int q = 0; q < 4; ++q) st16(dst + 16 * q, v + 16 * q);
  }
};


// ---------------------------------------------------------------------------------------------
// Tile epilogues.  The recurrent GEMMs' epilogues are memory-heavy elementwise work on the
// critical path of the recurrence, so they run cooperatively on the whole output tile: the kernel
// stages the fp32 accumulator tile T[rows][ncols] (row stride ldt) in shared memory; each of the
// 128 epilogue threads then owns one hidden-unit column u (lanes along units: coalesced global
// traffic) and walks the tile's rows in batches of NB with every load of a batch issued before
// any of its stores (memory-level parallelism).  Transposed stash writes go through a second
// shared-memory pass with lanes along batch rows.  `sm` = free shared memory, tid in [0,128),
// bar 1 syncs the 128 threads.
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
constexpr int kNB = 8;

// Byte ids of the tile's rows at timestep t, staged once: sb[r] = bytes[m0 + r][t].
template <typename S>
__device__ __forceinline__ void stage_bytes(const Net<S>& n, uint8_t* sb, int m0, int t, int rows, int tid) {
  if (tid < rows) sb[tid] = (uint8_t)n.byte_at(m0 + tid, t);
  epi_bar();
}

// F1: m = mx * a  ->  M_t (row-major), a_t stash, m_t^T stash.  U = units in this block (<= 64).
template <typename S>
__device__ __forceinline__ void tile_f1_blk(const Net<S>& n, int t, const float* T, int ldt, int m0, int n0, int U,
                                            int rows, uint8_t* sm, int tid) {
  const int h = n.h, ldm = U + 2;
  const uint8_t* sb = sm;
  S* Ms = reinterpret_cast<S*>(sm + 128);
  const int u = tid % U, rp = tid / U, RS = 128 / U, j = n0 + u;
  if (rp < RS) {
    const float* tabc = n.tab + j;
    for (int r0 = rp; r0 < rows; r0 += RS * kNB) {
      float a[kNB], mx[kNB];
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int r = min(r0 + k * RS, rows - 1);
        a[k] = T[r * ldt + u];
        mx[k] = __ldg(tabc + (long)sb[r] * 5 * h);
      }
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int r = r0 + k * RS;
        if (r >= rows) break;
        const long b = m0 + r;
        const float m = mx[k] * a[k];
        n.Mscr[b * h + j] = to_s<S>(m);
        n.Astash[((long)t * n.B + b) * h + j] = to_s<S>(a[k]);
        Ms[r * ldm + u] = to_s<S>(m);
      }
    }
  }
  epi_bar();
  if (tid < rows) {
    const long kc = n.kcol(t, m0 + tid);
    for (int uu = 0; uu < U; ++uu) n.MT[(long)(n0 + uu) * n.ldK + kc] = Ms[tid * ldm + uu];
  }
}

// F2: z = acc + W_x x + b -> gates, c_t, h_t (+ h_t^T).  Tile columns are internal gate rows:
// ncols = 4 * units, units <= 64.
template <typename S>
__device__ __forceinline__ void tile_f2(const Net<S>& n, int t, const float* T, int ldt, int m0, int n0, int ncols,
                                        int rows, uint8_t* sm, int tid) {
  const int h = n.h, U = ncols / 4, j0 = (n0 >> 6) * 16, ldm = U + 2;
  uint8_t* sb = sm;
  S* Hs = reinterpret_cast<S*>(sm + 128);
  stage_bytes(n, sb, m0, t, rows, tid);
  const int u = tid % U, rp = tid / U, RS = 128 / U, j = j0 + u;
  const int cb = (u >> 4) * 64 + (u & 15);  // tile column of gate i of unit u
  if (rp < RS) {
    const float* bias = n.master + n.po.b;
    const float bi = bias[j], bf = bias[h + j], bo = bias[2 * h + j], bu = bias[3 * h + j];
    const float* tabx = n.tab + h + n0 + cb;
    for (int r0 = rp; r0 < rows; r0 += RS * kNB) {
      float zi[kNB], zf[kNB], zo[kNB], zu[kNB], cp[kNB];
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int r = min(r0 + k * RS, rows - 1);
        const float* xz = tabx + (long)sb[r] * 5 * h;
        const float* tr = T + r * ldt + cb;
        zi[k] = tr[0] + __ldg(xz) + bi;
        zf[k] = tr[16] + __ldg(xz + 16) + bf;
        zo[k] = tr[32] + __ldg(xz + 32) + bo;
        zu[k] = tr[48] + __ldg(xz + 48) + bu;
        cp[k] = n.Crm[((long)t * n.B + m0 + r) * h + j];
      }
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int r = r0 + k * RS;
        if (r >= rows) break;
        const float gi = act_sigmoid<S>(zi[k]), gf = act_sigmoid<S>(zf[k]), go = act_sigmoid<S>(zo[k]), gu = act_tanh<S>(zu[k]);
        const float cv = gf * cp[k] + gi * gu;  // c_t = f c_{t-1} + i u   (fp32)
        const float hv = go * act_tanh<S>(cv);  // h_t = o tanh(c_t)
        const long row = (long)t * n.B + m0 + r;
        S* gr = n.Gates + row * 4 * h + n0 + cb;
        gr[0] = to_s<S>(gi);
        gr[16] = to_s<S>(gf);
        gr[32] = to_s<S>(go);
        gr[48] = to_s<S>(gu);
        n.Crm[(row + n.B) * h + j] = cv;
        n.Hrm[(row + n.B) * h + j] = to_s<S>(hv);
        Hs[r * ldm + u] = to_s<S>(hv);
      }
    }
  }
  epi_bar();
  if (tid < rows) {
    const long kc = n.kcol(t + 1, m0 + tid);
    for (int uu = 0; uu < U; ++uu) n.HT[(long)(j0 + uu) * n.ldH + kc] = Hs[tid * ldm + uu];
  }
}

// B1: dM = acc -> dA = dM * mx (row-major + transposed), dMX = dM * a (transposed).
template <typename S>
__device__ __forceinline__ void tile_b1_blk(const Net<S>& n, int t, const float* T, int ldt, int m0, int n0, int U,
                                            int rows, uint8_t* sm, int tid) {
  const int h = n.h, ldm = U + 2;
  const uint8_t* sb = sm;
  S* As = reinterpret_cast<S*>(sm + 128);
  S* Xs = As + 128 * ldm;
  const int u = tid % U, rp = tid / U, RS = 128 / U, j = n0 + u;
  if (rp < RS) {
    const float* tabc = n.tab + j;
    for (int r0 = rp; r0 < rows; r0 += RS * kNB) {
      float dm[kNB], mx[kNB], a[kNB];
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int r = min(r0 + k * RS, rows - 1);
        dm[k] = T[r * ldt + u];
        mx[k] = __ldg(tabc + (long)sb[r] * 5 * h);
        a[k] = to_f(n.Astash[((long)t * n.B + m0 + r) * h + j]);
      }
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int r = r0 + k * RS;
        if (r >= rows) break;
        const float da = dm[k] * mx[k];
        n.dAscr[(long)(m0 + r) * h + j] = to_s<S>(da);
        As[r * ldm + u] = to_s<S>(da);
        Xs[r * ldm + u] = to_s<S>(dm[k] * a[k]);
      }
    }
  }
  epi_bar();
  if (tid < rows) {
    const long kc = n.kcol(t, m0 + tid);
    for (int uu = 0; uu < U; ++uu) {
      const long o = (long)(n0 + uu) * n.ldK + kc;
      n.dAT[o] = As[tid * ldm + uu];
      n.dGT[o] = Xs[tid * ldm + uu];
    }
  }
}

// B2: dH = acc + dH_dec -> gate backward of step s (dZ row-major + transposed, dc carry).
template <typename S>
__device__ __forceinline__ void tile_b2_blk(const Net<S>& n, int s, const float* T, int ldt, int m0, int n0, int U,
                                            int rows, uint8_t* sm, int tid) {
  const int h = n.h, ldz = 4 * U + 2;
  S* Zs = reinterpret_cast<S*>(sm);
  const int u = tid % U, rp = tid / U, RS = 128 / U, j = n0 + u;
  const long gcol = (long)(j >> 4) * 64 + (j & 15);
  if (rp < RS) {
    for (int r0 = rp; r0 < rows; r0 += RS * kNB) {
      float dh[kNB], gi[kNB], gf[kNB], go[kNB], gu[kNB], c[kNB], cp[kNB], dcn[kNB];
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int r = min(r0 + k * RS, rows - 1);
        const long row = (long)s * n.B + m0 + r;
        const S* g = n.Gates + row * 4 * h + gcol;
        dh[k] = T[r * ldt + u] + n.dHdec[row * h + j];
        gi[k] = to_f(g[0]);
        gf[k] = to_f(g[16]);
        go[k] = to_f(g[32]);
        gu[k] = to_f(g[48]);
        c[k] = n.Crm[(row + n.B) * h + j];
        cp[k] = n.Crm[row * h + j];
        dcn[k] = n.dC[(long)(m0 + r) * h + j];
      }
#pragma unroll
      for (int k = 0; k < kNB; ++k) {
        const int r = r0 + k * RS;
        if (r >= rows) break;
        const float kk = act_tanh<S>(c[k]);
        const float i = gi[k], f = gf[k], o = go[k], uu = gu[k];
        const float dzo = dh[k] * kk * o * (1.f - o);
        const float dc = dcn[k] + dh[k] * o * (1.f - kk * kk);
        const float dzi = dc * uu * i * (1.f - i);
        const float dzf = dc * cp[k] * f * (1.f - f);
        const float dzu = dc * i * (1.f - uu * uu);
        const long b = m0 + r;
        n.dC[b * h + j] = dc * f;
        S* zr = n.dZscr + b * 4 * h + gcol;
        zr[0] = to_s<S>(dzi);
        zr[16] = to_s<S>(dzf);
        zr[32] = to_s<S>(dzo);
        zr[48] = to_s<S>(dzu);
        S* zs = Zs + r * ldz + u;
        zs[0] = to_s<S>(dzi);
        zs[U] = to_s<S>(dzf);
        zs[2 * U] = to_s<S>(dzo);
        zs[3 * U] = to_s<S>(dzu);
      }
    }
  }
  epi_bar();
  if (tid < rows) {
    const long kc = n.kcol(s, m0 + tid);
    for (int gu = 0; gu < 4 * U; ++gu) {
      const int g = gu / U, uu = gu - g * U;
      n.dGT[((long)h + int_row(g, n0 + uu)) * n.ldK + kc] = Zs[tid * ldz + gu];
    }
  }
}

// Column sub-blocks keep the second-pass shared memory bounded (see tile_smem_bytes).
template <typename S>
__device__ __forceinline__ void tile_f1(const Net<S>& n, int t, const float* T, int ldt, int m0, int n0, int ncols,
                                        int rows, uint8_t* sm, int tid) {
  stage_bytes(n, sm, m0, t, rows, tid);
  for (int c = 0; c < ncols; c += 64) {
    if (c) epi_bar();
    tile_f1_blk(n, t, T + c, ldt, m0, n0 + c, min(64, ncols - c), rows, sm, tid);
  }
}
template <typename S>
__device__ __forceinline__ void tile_b1(const Net<S>& n, int t, const float* T, int ldt, int m0, int n0, int ncols,
                                        int rows, uint8_t* sm, int tid) {
  stage_bytes(n, sm, m0, t, rows, tid);
  for (int c = 0; c < ncols; c += 64) {
    if (c) epi_bar();
    tile_b1_blk(n, t, T + c, ldt, m0, n0 + c, min(64, ncols - c), rows, sm, tid);
  }
}
template <typename S>
__device__ __forceinline__ void tile_b2(const Net<S>& n, int s, const float* T, int ldt, int m0, int n0, int ncols,
                                        int rows, uint8_t* sm, int tid) {
  for (int c = 0; c < ncols; c += 32) {
    if (c) epi_bar();
    tile_b2_blk(n, s, T + c, ldt, m0, n0 + c, min(32, ncols - c), rows, sm, tid);
  }
}

// Shared memory a tile epilogue needs: the fp32 tile (row stride ncols + 4) plus its second-pass
// buffer (bytes + F1/F2: 128 x 66, B1: 2 x 128 x 66, B2: 128 x 130 elements of S; <= 68 KB fp32).
__host__ __device__ constexpr int tile_smem_bytes(int ncols) { return 128 * (ncols + 4) * 4 + 128 + 2 * 128 * 66 * 4; }

// (b) forward GEMM 1, A_t = H_{t-1} W_mh^T:  m_t = mx_t * a_t  (multiplicative intermediate).
template <typename S>
struct EpiF1 {
  Net<S> n;
  int t;
  static constexpr bool kTile = MLSTM_TILE_EPI;
  __device__ __forceinline__ void tile(const float* T, int ldt, int m0, int n0, int ncols, int rows, uint8_t* sm,
                                       int tid) const {
    tile_f1(n, t, T, ldt, m0, n0, ncols, rows, sm, tid);
  }
  __device__ __forceinline__ void operator()(int b, int col0, float (&v)[64]) const {
    const float* mx = n.tab + (long)n.byte_at(b, t) * 5 * n.h + col0;
    S* mrow = n.Mscr + (long)b * n.h + col0;
    S* arow = n.Astash + ((long)t * n.B + b) * n.h + col0;
    const long kc = n.kcol(t, b);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float x[16], m[16];
      ld16(mx + 16 * q, x);
#pragma unroll
      for (int i = 0; i < 16; ++i) m[i] = x[i] * v[16 * q + i];
      st16(mrow + 16 * q, m);
      st16(arow + 16 * q, v + 16 * q);
#pragma unroll
      for (int i = 0; i < 16; ++i) n.MT[(long)(col0 + 16 * q + i) * n.ldK + kc] = to_s<S>(m[i]);
    }
  }
};

// (b) forward GEMM 2, Z_t = M_t W_h^T (+ W_x x_t + b): gates, cell update, hidden state.
template <typename S>
struct EpiF2 {
  Net<S> n;
  int t;
  static constexpr bool kTile = MLSTM_TILE_EPI;
  __device__ __forceinline__ void tile(const float* T, int ldt, int m0, int n0, int ncols, int rows, uint8_t* sm,
                                       int tid) const {
    tile_f2(n, t, T, ldt, m0, n0, ncols, rows, sm, tid);
  }
  __device__ __forceinline__ void operator()(int b, int col0, float (&v)[64]) const {
    const int h = n.h;
    const int j0 = (col0 >> 6) * 16;
    const float* xz = n.tab + (long)n.byte_at(b, t) * 5 * h + h + col0;
    const float* bias = n.master + n.po.b;
    float xv[64];
#pragma unroll
    for (int q = 0; q < 4; ++q) ld16(xz + 16 * q, xv + 16 * q);
    float cprev[16];
    ld16(n.Crm + ((long)t * n.B + b) * h + j0, cprev);
    float gi[16], gf[16], go[16], gu[16], cv[16], hv[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int j = j0 + jj;
      const float zi = v[jj] + xv[jj] + bias[j];
      const float zf = v[16 + jj] + xv[16 + jj] + bias[h + j];
      const float zo = v[32 + jj] + xv[32 + jj] + bias[2 * h + j];
      const float zu = v[48 + jj] + xv[48 + jj] + bias[3 * h + j];
      gi[jj] = act_sigmoid<S>(zi);
      gf[jj] = act_sigmoid<S>(zf);
      go[jj] = act_sigmoid<S>(zo);
      gu[jj] = act_tanh<S>(zu);
      cv[jj] = gf[jj] * cprev[jj] + gi[jj] * gu[jj];  // c_t = f c_{t-1} + i u   (fp32)
      hv[jj] = go[jj] * act_tanh<S>(cv[jj]);                 // h_t = o tanh(c_t)
    }
    S* grow = n.Gates + ((long)t * n.B + b) * 4 * h + col0;
    st16(grow, gi);
    st16(grow + 16, gf);
    st16(grow + 32, go);
    st16(grow + 48, gu);
    st16(n.Hrm + ((long)(t + 1) * n.B + b) * h + j0, hv);
    st16(n.Crm + ((long)(t + 1) * n.B + b) * h + j0, cv);
    const long kc = n.kcol(t + 1, b);
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) n.HT[(long)(j0 + jj) * n.ldH + kc] = to_s<S>(hv[jj]);
  }
};

// (d) decoder logits Y = H W_dec^T + b_dec, fp32 ("operating on FP32 logits").
template <typename S>
struct EpiY {
  Net<S> n;
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const {
    const float* bd = n.master + n.po.bdec + col0;
    float* dst = n.Y + (long)row * 256 + col0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float o[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) o[i] = v[16 * q + i] + bd[16 * q + i];
      st16(dst + 16 * q, o);
    }
  }
};

// dH from the decoder: dH_dec = dY W_dec.
template <typename S>
struct EpiDHdec {
  Net<S> n;
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const {
    float* dst = n.dHdec + (long)row * n.h + col0;
#pragma unroll
    for (int q = 0; q < 4; ++q) st16(dst + 16 * q, v + 16 * q);
  }
};

// (c-1) backward gate step for timestep s and 16 units j0..j0+15 of row b, given dH (the sum of
// the decoder and recurrent contributions).  TBTT: dC carry starts at zero for s = T-1.
template <typename S>
__device__ __forceinline__ void gate_bwd16(const Net<S>& n, int s, int b, int j0, const float* dh) {
  const int h = n.h;
  const long gofs = ((long)s * n.B + b) * 4 * h + (long)(j0 >> 4) * 64;
  float gi[16], gf[16], go[16], gu[16], c[16], cp[16], dcn[16];
  ld16(n.Gates + gofs, gi);
  ld16(n.Gates + gofs + 16, gf);
  ld16(n.Gates + gofs + 32, go);
  ld16(n.Gates + gofs + 48, gu);
  ld16(n.Crm + ((long)(s + 1) * n.B + b) * h + j0, c);
  ld16(n.Crm + ((long)s * n.B + b) * h + j0, cp);
  ld16(n.dC + (long)b * h + j0, dcn);
  float dzi[16], dzf[16], dzo[16], dzu[16], dcnew[16];
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) {
    const float k = act_tanh<S>(c[jj]);
    const float i = gi[jj], f = gf[jj], o = go[jj], u = gu[jj];
    dzo[jj] = dh[jj] * k * o * (1.f - o);
    const float dc = dcn[jj] + dh[jj] * o * (1.f - k * k);
    dzi[jj] = dc * u * i * (1.f - i);
    dzf[jj] = dc * cp[jj] * f * (1.f - f);
    dzu[jj] = dc * i * (1.f - u * u);
    dcnew[jj] = dc * f;
  }
  st16(n.dC + (long)b * h + j0, dcnew);
  S* zrow = n.dZscr + (long)b * 4 * h + (long)(j0 >> 4) * 64;
  st16(zrow, dzi);
  st16(zrow + 16, dzf);
  st16(zrow + 32, dzo);
  st16(zrow + 48, dzu);
  const long kc = n.kcol(s, b);
  const long r0 = (long)h + (long)(j0 >> 4) * 64;
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) {
    n.dGT[(r0 + jj) * n.ldK + kc] = to_s<S>(dzi[jj]);
    n.dGT[(r0 + 16 + jj) * n.ldK + kc] = to_s<S>(dzf[jj]);
    n.dGT[(r0 + 32 + jj) * n.ldK + kc] = to_s<S>(dzo[jj]);
    n.dGT[(r0 + 48 + jj) * n.ldK + kc] = to_s<S>(dzu[jj]);
  }
}

// (c-1) backward GEMM 1, dM_t = dZ_t W_h:  dA = dM * mx,  dMX = dM * a.
template <typename S>
struct EpiB1 {
  Net<S> n;
  int t;
  static constexpr bool kTile = MLSTM_TILE_EPI;
  __device__ __forceinline__ void tile(const float* T, int ldt, int m0, int n0, int ncols, int rows, uint8_t* sm,
                                       int tid) const {
    tile_b1(n, t, T, ldt, m0, n0, ncols, rows, sm, tid);
  }
  __device__ __forceinline__ void operator()(int b, int col0, float (&v)[64]) const {
    const float* mx = n.tab + (long)n.byte_at(b, t) * 5 * n.h + col0;
    const S* arow = n.Astash + ((long)t * n.B + b) * n.h + col0;
    S* darow = n.dAscr + (long)b * n.h + col0;
    const long kc = n.kcol(t, b);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float x[16], a[16], da[16], dmx[16];
      ld16(mx + 16 * q, x);
      ld16(arow + 16 * q, a);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        da[i] = v[16 * q + i] * x[i];
        dmx[i] = v[16 * q + i] * a[i];
      }
      st16(darow + 16 * q, da);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const long r = col0 + 16 * q + i;
        n.dAT[r * n.ldK + kc] = to_s<S>(da[i]);
        n.dGT[r * n.ldK + kc] = to_s<S>(dmx[i]);
      }
    }
  }
};

// (c-1) backward GEMM 2, dH_rec = dA_t W_mh, fused with the gate backward of step s = t-1.
template <typename S>
struct EpiB2 {
  Net<S> n;
  int s;
  static constexpr bool kTile = MLSTM_TILE_EPI;
  __device__ __forceinline__ void tile(const float* T, int ldt, int m0, int n0, int ncols, int rows, uint8_t* sm,
                                       int tid) const {
    tile_b2(n, s, T, ldt, m0, n0, ncols, rows, sm, tid);
  }
  __device__ __forceinline__ void operator()(int b, int col0, float (&v)[64]) const {
    const float* dhd = n.dHdec + ((long)s * n.B + b) * n.h + col0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float dh[16];
      ld16(dhd + 16 * q, dh);
#pragma unroll
      for (int i = 0; i < 16; ++i) dh[i] += v[16 * q + i];
      gate_bwd16(n, s, b, col0 + 16 * q, dh);
    }
  }
};

// (c-2) split-K partial of a weight-gradient GEMM: part[z][row][col] (fp32).
struct EpiPartial {
  float* part;
  long ldo;
  long split_stride;
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const {
    float* dst = part + (long)blockIdx.z * split_stride + (long)row * ldo + col0;
#pragma unroll
    for (int q = 0; q < 4; ++q) st16(dst + 16 * q, v + 16 * q);
  }
};

}  // namespace mlstm
