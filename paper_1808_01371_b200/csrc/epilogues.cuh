// epilogues.cuh -- the fused GEMM epilogues of the step.
//
// Every functor is called by one thread for one accumulator row and 64 consecutive columns:
//   (row, col0, v[0..63]) with v = fp32 accumulator values.  Rows of the per-timestep GEMMs are
//   batch rows b; columns are hidden units (N = h) or internal gate rows (N = 4h).
#pragma once
#include "net.cuh"

namespace mlstm {

// (a) input-projection table: tab[v][:] = [W_mx E[v] | W_x E[v]]  (the per-token input GEMM of
// every timestep, done once per step for the 256 possible bytes; gathered by byte below).
template <typename S>
struct EpiTab {
  static constexpr int kMinGroups = 1;  // 16-column groups one call must cover
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  Net<S> n;
  template <int NG>
  __device__ __forceinline__ void run(int row, int col0, const float* v) const {
    float* dst = n.tab + (long)row * 5 * n.h + col0;
#pragma unroll
    for (int q = 0; q < NG; ++q) st16(dst + 16 * q, v + 16 * q);
    if (n.XZT && col0 >= n.h) {  // transposed fp16 (W_x E + b) for the folded F2 (lanes = bytes)
      const float* bias = n.master + n.po.b;
#pragma unroll
      for (int i = 0; i < 16 * NG; ++i) {
        const int r = col0 - n.h + i;
        n.XZT[(long)r * 256 + row] = to_s<S>(v[i] + bias[canon_of_int(r, n.h)]);
      }
    }
  }
};



// (b) forward GEMM 1, A_t = H_{t-1} W_mh^T:  m_t = mx_t * a_t  (multiplicative intermediate).
template <typename S>
struct EpiF1 {
  static constexpr int kMinGroups = 1;  // 16-column groups one call must cover
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  Net<S> n;
  int t;
  template <int NG>
  __device__ __forceinline__ void run(int b, int col0, const float* v) const {
    const float* mx = n.tab + (long)n.byte_at(b, t) * 5 * n.h + col0;
    S* mrow = n.Mrm + ((long)t * n.B + b) * n.h + col0;
    S* arow = n.Astash + ((long)t * n.B + b) * n.h + col0;
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      float x[16], m[16];
      ld16(mx + 16 * q, x);
#pragma unroll
      for (int i = 0; i < 16; ++i) m[i] = x[i] * v[16 * q + i];
      st16(mrow + 16 * q, m);
      st16(arow + 16 * q, v + 16 * q);
    }
  }
};

// (b) forward GEMM 2, Z_t = M_t W_h^T (+ W_x x_t + b): gates, cell update, hidden state.  With
// `folded` the GEMM's second K segment (one-hot x (W_x E + b)^T) already added W_x x_t + b.
template <typename S>
struct EpiF2 {  // one call = 4 gates x 16 units: NG must be 4
  static constexpr int kMinGroups = 4;  // 16-column groups one call must cover
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  Net<S> n;
  int t;
  int folded;
  template <int NG>
  __device__ __forceinline__ void run(int b, int col0, const float* v) const {
    const int h = n.h;
    const int j0 = (col0 >> 6) * 16;
    const float* bias = n.master + n.po.b;
    float xv[64];
    if (folded) {
#pragma unroll
      for (int i = 0; i < 64; ++i) xv[i] = 0.f;
    } else {
      const float* xz = n.tab + (long)n.byte_at(b, t) * 5 * h + h + col0;
#pragma unroll
      for (int q = 0; q < 4; ++q) ld16(xz + 16 * q, xv + 16 * q);
    }
    float cprev[16];
    ld16(n.Crm + ((long)t * n.B + b) * h + j0, cprev);
    float gi[16], gf[16], go[16], gu[16], cv[16], hv[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int j = j0 + jj;
      const float zi = v[jj] + (folded ? 0.f : xv[jj] + bias[j]);
      const float zf = v[16 + jj] + (folded ? 0.f : xv[16 + jj] + bias[h + j]);
      const float zo = v[32 + jj] + (folded ? 0.f : xv[32 + jj] + bias[2 * h + j]);
      const float zu = v[48 + jj] + (folded ? 0.f : xv[48 + jj] + bias[3 * h + j]);
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
  }
};

// Async-I/O form of EpiF2 (tcgen05 engines; W_x x + b always folded there).  Per warp and slot
// (one 64-column call): c_{t-1} rows come in by bulk copy; gates, c_t and h_t rows are staged in
// the warp's window with 16-byte row padding (conflict-free) and leave by bulk copy.
// Warp-cooperative store of 32 staged rows (row r of the warp at src + r*spitch, `bytes` per row)
// to dst + r*dpitch (elements of 16 bytes): consecutive lanes take consecutive 16-byte pieces of a
// row, so one warp instruction writes 512/bytes full rows instead of touching 32 lines.
__device__ __forceinline__ void warp_rows_out(uint8_t* dst, long dpitch, const uint8_t* src, int spitch, int bytes,
                                              int nvalid, int lane) {
  const int per = bytes >> 4;
  __syncwarp();
  for (int k = lane; k < 32 * per; k += 32) {
    const int r = k / per, i = k - r * per;
    if (r < nvalid)
      *reinterpret_cast<uint4*>(dst + r * dpitch + i * 16) = *reinterpret_cast<const uint4*>(src + r * spitch + i * 16);
  }
}

// Stage this lane's 16*NG-value row piece (converted to S) in the warp window and store the warp's
// rows coalesced: dst0 = the row of lane 0, consecutive rows `pitch` elements apart.
template <int NG, typename S>
__device__ __forceinline__ void stage_rows_out(const EpiIO& io, S* dst0, long pitch, const float* vals) {
  constexpr int BYTES = 16 * NG * (int)sizeof(S);
  S* w = reinterpret_cast<S*>(io.buf + io.lane * (BYTES + 16));
#pragma unroll
  for (int q = 0; q < NG; ++q) st16(w + 16 * q, vals + 16 * q);
  warp_rows_out(reinterpret_cast<uint8_t*>(dst0), pitch * (long)sizeof(S), io.buf, BYTES + 16, BYTES, io.nvalid,
                io.lane);
  __syncwarp();
}

// Row-I/O forms of EpiF1 / EpiB1: same loads, outputs staged and stored coalesced.
template <typename S>
struct EpiF1IO : EpiF1<S> {
  static constexpr bool kAsyncIO = true;
  __device__ __forceinline__ void io_issue(const EpiIO&, int, int) const {}
  template <int NG>
  __device__ __forceinline__ void run_io(const EpiIO& io, int, int col0, const float* v) const {
    const Net<S>& n = this->n;
    const int t = this->t, b = io.row0 + io.lane;
    float m[16 * NG];
    if (io.valid()) {
      const float* mx = n.tab + (long)n.byte_at(b, t) * 5 * n.h + col0;
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        float x[16];
        ld16(mx + 16 * q, x);
#pragma unroll
        for (int i = 0; i < 16; ++i) m[16 * q + i] = x[i] * v[16 * q + i];
      }
    }
    const long r0 = (long)t * n.B + io.row0;
    stage_rows_out<NG>(io, n.Mrm + r0 * n.h + col0, n.h, m);
    stage_rows_out<NG>(io, n.Astash + r0 * n.h + col0, n.h, v);
  }
};

template <typename S>
struct EpiF2IO : EpiF2<S> {
  static constexpr bool kAsyncIO = true;
  int out_mode;  // 1: per-row bulk copies out; 2: warp-cooperative coalesced stores
  static constexpr int kCp = 0, kG = 32 * 80, kC = kG + 32 * 144, kH = kC + 32 * 80, kSlot = kH + 32 * 48;
  static_assert(2 * kSlot <= kWarpStageBytes, "staging window");
  __device__ __forceinline__ void io_issue(const EpiIO& io, int slot, int col0) const {
    const Net<S>& n = this->n;
    if (!io.valid()) return;
    const int b = io.row0 + io.lane, j0 = (col0 >> 6) * 16;
    ptx::mbar_expect_tx(io.bar, 64);
    ptx::bulk_g2s(io.buf + slot * kSlot + kCp + io.lane * 80, n.Crm + ((long)this->t * n.B + b) * n.h + j0, 64,
                  io.bar);
  }
  // c_{t-1} of this lane's row and chunk straight into registers (issued by the epilogue warps while the
  // main loop still runs; c_{t-1} was written two launches earlier, see gemm_tc2_kernel)
  static constexpr bool kPreC = true;
  __device__ __forceinline__ void preload_c(const EpiIO& io, int col0, float4 (&c)[4]) const {
    const Net<S>& n = this->n;
    if (!io.valid()) return;
    const float4* src =
        reinterpret_cast<const float4*>(n.Crm + ((long)this->t * n.B + io.row0 + io.lane) * n.h + (col0 >> 6) * 16);
#pragma unroll
    for (int k = 0; k < 4; ++k) c[k] = src[k];
  }
  template <int NG>
  __device__ __forceinline__ void run_io(const EpiIO& io, int slot, int col0, const float* v) const {
    ptx::mbar_wait(io.bar, 0);
    const float4* cp = reinterpret_cast<const float4*>(io.buf + slot * kSlot + kCp + io.lane * 80);
    const float4 c[4] = {cp[0], cp[1], cp[2], cp[3]};
    run_io_c<NG>(io, slot, col0, v, c);
  }
  template <int NG>
  __device__ __forceinline__ void run_io_c(const EpiIO& io, int slot, int col0, const float* v,
                                           const float4 (&cp)[4]) const {
    static_assert(NG == 4, "one call = 4 gates x 16 units");
    const Net<S>& n = this->n;
    const int h = n.h, t = this->t, j0 = (col0 >> 6) * 16, lane = io.lane;
    const int b = io.row0 + lane;
    uint8_t* sb = io.buf + slot * kSlot;
    __align__(16) S gs[64];
    __align__(16) float cv[16];
    __align__(16) S hv[16];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 c4 = cp[k];
      const float cpv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int jj = 4 * k + e;
        const float gi = act_sigmoid<S>(v[jj]), gf = act_sigmoid<S>(v[16 + jj]);
        const float go = act_sigmoid<S>(v[32 + jj]), gu = act_tanh<S>(v[48 + jj]);
        gs[jj] = to_s<S>(gi);
        gs[16 + jj] = to_s<S>(gf);
        gs[32 + jj] = to_s<S>(go);
        gs[48 + jj] = to_s<S>(gu);
        cv[jj] = gf * cpv[e] + gi * gu;               // c_t = f c_{t-1} + i u   (fp32)
        hv[jj] = to_s<S>(go * act_tanh<S>(cv[jj]));  // h_t = o tanh(c_t)
      }
    }
    uint4* sg = reinterpret_cast<uint4*>(sb + kG + lane * 144);
    uint4* sc = reinterpret_cast<uint4*>(sb + kC + lane * 80);
    uint4* sh = reinterpret_cast<uint4*>(sb + kH + lane * 48);
#pragma unroll
    for (int k = 0; k < 8; ++k) sg[k] = reinterpret_cast<const uint4*>(gs)[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) sc[k] = reinterpret_cast<const uint4*>(cv)[k];
#pragma unroll
    for (int k = 0; k < 2; ++k) sh[k] = reinterpret_cast<const uint4*>(hv)[k];
    if (out_mode == 1) {
      ptx::fence_proxy_async_smem();
      if (io.valid()) {
        ptx::bulk_s2g(n.Gates + ((long)t * n.B + b) * 4 * h + col0, sg, 128);
        ptx::bulk_s2g(n.Crm + ((long)(t + 1) * n.B + b) * h + j0, sc, 64);
        ptx::bulk_s2g(n.Hrm + ((long)(t + 1) * n.B + b) * h + j0, sh, 32);
      }
      ptx::bulk_commit();
    } else {
      const int b0 = io.row0;
      warp_rows_out(reinterpret_cast<uint8_t*>(n.Gates + ((long)t * n.B + b0) * 4 * h + col0), 8L * h, sb + kG, 144,
                    128, io.nvalid, lane);
      warp_rows_out(reinterpret_cast<uint8_t*>(n.Crm + ((long)(t + 1) * n.B + b0) * h + j0), 4L * h, sb + kC, 80, 64,
                    io.nvalid, lane);
      warp_rows_out(reinterpret_cast<uint8_t*>(n.Hrm + ((long)(t + 1) * n.B + b0) * h + j0), 2L * h, sb + kH, 48, 32,
                    io.nvalid, lane);
    }
  }
};

// (d) decoder logits Y = H W_dec^T + b_dec, fp32 ("operating on FP32 logits").
template <typename S>
struct EpiY {
  static constexpr int kMinGroups = 1;  // 16-column groups one call must cover
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  Net<S> n;
  template <int NG>
  __device__ __forceinline__ void run(int row, int col0, const float* v) const {
    const float* bd = n.master + n.po.bdec + col0;
    float* dst = n.Y + (long)row * 256 + col0;
#pragma unroll
    for (int q = 0; q < NG; ++q) {
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
  static constexpr int kMinGroups = 1;  // 16-column groups one call must cover
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  Net<S> n;
  template <int NG>
  __device__ __forceinline__ void run(int row, int col0, const float* v) const {
    float* dst = n.dHdec + (long)row * n.h + col0;
#pragma unroll
    for (int q = 0; q < NG; ++q) st16(dst + 16 * q, v + 16 * q);
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
  S* zrow = n.G5 + ((long)s * n.B + b) * 5 * h + h + (long)(j0 >> 4) * 64;
  st16(zrow, dzi);
  st16(zrow + 16, dzf);
  st16(zrow + 32, dzo);
  st16(zrow + 48, dzu);
}

// (c-1) backward GEMM 1, dM_t = dZ_t W_h:  dA = dM * mx,  dMX = dM * a.
template <typename S>
struct EpiB1 {
  static constexpr int kMinGroups = 1;  // 16-column groups one call must cover
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  Net<S> n;
  int t;
  template <int NG>
  __device__ __forceinline__ void run(int b, int col0, const float* v) const {
    const float* mx = n.tab + (long)n.byte_at(b, t) * 5 * n.h + col0;
    const S* arow = n.Astash + ((long)t * n.B + b) * n.h + col0;
    S* darow = n.dA + ((long)t * n.B + b) * n.h + col0;
    S* mxrow = n.G5 + ((long)t * n.B + b) * 5 * n.h + col0;  // dMX block of the stash row
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      float x[16], a[16], da[16], dmx[16];
      ld16(mx + 16 * q, x);
      ld16(arow + 16 * q, a);
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        da[i] = v[16 * q + i] * x[i];
        dmx[i] = v[16 * q + i] * a[i];
      }
      st16(darow + 16 * q, da);
      st16(mxrow + 16 * q, dmx);
    }
  }
};


template <typename S>
struct EpiB1IO : EpiB1<S> {
  static constexpr bool kAsyncIO = true;
  __device__ __forceinline__ void io_issue(const EpiIO&, int, int) const {}
  template <int NG>
  __device__ __forceinline__ void run_io(const EpiIO& io, int, int col0, const float* v) const {
    const Net<S>& n = this->n;
    const int t = this->t, b = io.row0 + io.lane;
    float da[16 * NG], dmx[16 * NG];
    if (io.valid()) {
      const float* mx = n.tab + (long)n.byte_at(b, t) * 5 * n.h + col0;
      const S* arow = n.Astash + ((long)t * n.B + b) * n.h + col0;
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        float x[16], a[16];
        ld16(mx + 16 * q, x);
        ld16(arow + 16 * q, a);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          da[16 * q + i] = v[16 * q + i] * x[i];
          dmx[16 * q + i] = v[16 * q + i] * a[i];
        }
      }
    }
    const long r0 = (long)t * n.B + io.row0;
    stage_rows_out<NG>(io, n.dA + r0 * n.h + col0, n.h, da);
    stage_rows_out<NG>(io, n.G5 + r0 * 5 * n.h + col0, 5L * n.h, dmx);
  }
};

// Cooperative tile form of the gate backward (used by the split-K engine, whose reduced fp32 tile
// T[rows][U] (row stride ldt, columns = hidden units n0..n0+U) sits in shared memory).  The row-
// per-thread form touches 32 cache lines per warp instruction, which makes the L1 wavefront rate,
// not DRAM, the bound; here 16 lanes x 4 units cover 64 units of one row (two rows per warp
// instruction, 8/16-byte vectors) and each thread batches RB rows' loads before any store.
// 256 threads, tid in [0, 256).
__device__ __forceinline__ void epi_bar256() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <typename S>
__device__ __forceinline__ void b2_tile(const Net<S>& n, int s, const float* T, int ldt, int m0, int n0, int U,
                                        int rows, uint8_t* sm, int tid) {
  constexpr int RB = 4;
  const int h = n.h, ng = U / 4, rpi = 256 / ng;
  const int ug = tid % ng, rr = tid / ng;
  const int u0 = 4 * ug, j = n0 + u0;
  const long gcol = (long)(j >> 4) * 64 + (j & 15);  // internal column of gate i of unit j
  if (rr < rpi) {
    for (int rb = rr; rb < rows; rb += rpi * RB) {
      float4 dh[RB], gi[RB], gf[RB], go[RB], gu[RB], c[RB], cp[RB], dcn[RB];
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int r = min(rb + k * rpi, rows - 1);
        const long row = (long)s * n.B + m0 + r;
        const float4 t4 = *reinterpret_cast<const float4*>(T + r * ldt + u0);
        const float4 d4 = n.dHdec ? ld4(n.dHdec + row * h + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        dh[k] = make_float4(t4.x + d4.x, t4.y + d4.y, t4.z + d4.z, t4.w + d4.w);
        const S* g = n.Gates + row * 4 * h + gcol;
        gi[k] = ld4(g);
        gf[k] = ld4(g + 16);
        go[k] = ld4(g + 32);
        gu[k] = ld4(g + 48);
        c[k] = ld4(n.Crm + (row + n.B) * h + j);
        cp[k] = ld4(n.Crm + row * h + j);
        dcn[k] = ld4(n.dC + (long)(m0 + r) * h + j);

      }
#pragma unroll
      for (int k = 0; k < RB; ++k) {
        const int r = rb + k * rpi;
        if (r >= rows) break;
        float dzi[4], dzf[4], dzo[4], dzu[4], dcw[4];
        const float* DH = &dh[k].x;
        const float *I = &gi[k].x, *F = &gf[k].x, *O = &go[k].x, *UU = &gu[k].x;
        const float *CC = &c[k].x, *CP = &cp[k].x, *DC = &dcn[k].x;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float kk = act_tanh<S>(CC[i]);
          dzo[i] = DH[i] * kk * O[i] * (1.f - O[i]);
          const float dc = DC[i] + DH[i] * O[i] * (1.f - kk * kk);
          dzi[i] = dc * UU[i] * I[i] * (1.f - I[i]);
          dzf[i] = dc * CP[i] * F[i] * (1.f - F[i]);
          dzu[i] = dc * I[i] * (1.f - UU[i] * UU[i]);
          dcw[i] = dc * F[i];
        }
        const long b = m0 + r;
        st4(n.dC + b * h + j, make_float4(dcw[0], dcw[1], dcw[2], dcw[3]));
        S* zr = n.G5 + ((long)s * n.B + b) * 5 * h + h + gcol;
        st4(zr, make_float4(dzi[0], dzi[1], dzi[2], dzi[3]));
        st4(zr + 16, make_float4(dzf[0], dzf[1], dzf[2], dzf[3]));
        st4(zr + 32, make_float4(dzo[0], dzo[1], dzo[2], dzo[3]));
        st4(zr + 48, make_float4(dzu[0], dzu[1], dzu[2], dzu[3]));
      }
    }
  }
}

// (c-1) backward GEMM 2, dH_rec = dA_t W_mh, fused with the gate backward of step s = t-1.
template <typename S>
struct EpiB2 {
  static constexpr int kMinGroups = 1;  // 16-column groups one call must cover
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  Net<S> n;
  int s;
  static constexpr bool kTile = true;  // the split-K engine calls tile()
  __device__ __forceinline__ void tile(const float* T, int ldt, int m0, int n0, int U, int rows, uint8_t* sm,
                                       int tid) const {
    b2_tile(n, s, T, ldt, m0, n0, U, rows, sm, tid);
  }
  template <int NG>
  __device__ __forceinline__ void run(int b, int col0, const float* v) const {
    // dH = dH_rec + dH_dec; on the tcgen05 path dH_dec is already in the accumulator (dHdec null)
    const float* dhd = n.dHdec ? n.dHdec + ((long)s * n.B + b) * n.h + col0 : nullptr;
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      float dh[16];
      if (dhd) ld16(dhd + 16 * q, dh);
#pragma unroll
      for (int i = 0; i < 16; ++i) dh[i] = (dhd ? dh[i] : 0.f) + v[16 * q + i];
      gate_bwd16(n, s, b, col0 + 16 * q, dh);
    }
  }
};

// (c-2) split-K partial of a weight-gradient GEMM: part[z][row][col] (fp32).
struct EpiPartial {
  static constexpr int kMinGroups = 1;  // 16-column groups one call must cover
  __device__ __forceinline__ void operator()(int row, int col0, float (&v)[64]) const { run<4>(row, col0, v); }
  float* part;
  long ldo;
  long split_stride;
  template <int NG>
  __device__ __forceinline__ void run(int row, int col0, const float* v) const {
    float* dst = part + (long)blockIdx.z * split_stride + (long)row * ldo + col0;
#pragma unroll
    for (int q = 0; q < NG; ++q) st16(dst + 16 * q, v + 16 * q);
  }
};

}  // namespace mlstm
