// tcgen05 (kind::tf32) implicit-GEMM engine shared by the convolution and
// inner-product layers ("rotates (multiply W)"
// convolution).
//
//   D[m][n] = sum_k A(m, k) * B(n, k)      fp32 storage, TF32 operands, fp32 accumulate
//
// One CTA computes a 128 x BN output tile (optionally one K-split of it):
//   warps 0-7 : producers — gather 16-byte chunks with cp.async (zero-filled
//               outside the operand) straight into the UMMA canonical layouts,
//               one stage of BK = 32 fp32 (128 B) per step; then the epilogue
//               (TMEM -> registers -> global; warp w reads TMEM lanes
//               32*(w%4).. and column half w/4).
//   warp 8    : TMEM allocation and the single MMA-issuing thread.
// Operands are "loaders": each maps a (row, k) of the GEMM onto the layer's
// native tensor (NHWC activations, KRSC / [d_v][d_h] weights), so the im2col
// of the convolution is never materialised.  A loader is K-major (4
// consecutive k contiguous in memory) or MN-major (4 consecutive rows
// contiguous); tcgen05 kind::tf32 accepts both from shared memory
// (instruction-descriptor bits 15/16); MN-major tf32 must use the
// SWIZZLE_128B_BASE32B layout (32-byte swizzle granules, 4-line atoms).
//
// Producer threads own fixed tile rows (K-major) or a fixed MN chunk
// (MN-major) for the whole K loop, so address bases are computed once (loader
// State); per stage a chunk costs a handful of integer ops.  In the weight
// gradient the K index is the output pixel: each warp decomposes its 4 pixels
// of the stage once (lanes 0-3) and broadcasts them with shuffles.
//
// Bias gradients are fused into the weight-gradient GEMMs: the A operand gets
// one extra "ones" row (index `ones_row`), whose output row is sum_k B(n, k) =
// column sums of dy, routed by the epilogue to the bias-gradient buffer.
#pragma once
#include <type_traits>
#include <cuda.h>

#include "sg_common.cuh"

namespace sg {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 32;  // fp32 elements = 128 bytes = one swizzle row
constexpr int GEMM_PRODUCERS = 256;

// {1, 0, 0, 0}: source of the ones-row chunk (global memory, cp.async source).
__device__ __align__(16) static const float g_one4[4] = {1.f, 0.f, 0.f, 0.f};

// ---------------------------------------------------------------------------
// Blocked row-major matrix view: element (i, j) at p[(j / cb) * bs + i * ld + j % cb].
// cb >= cols means a plain row-major matrix.  Column blocking is how a tensor
// gathered along the feature dimension by NCCL is laid out ([K][rows][cols/K]).
struct MatView {
  const float* p;
  long long ld, bs;
  int cb, rows, cols;
  FastDiv fcb;  // divides by cb (blocked views)
  __device__ __forceinline__ long long col_off(int j) const {
    if (cb >= cols) return j;
    int blk = fcb.div(j);
    return (long long)blk * bs + (j - blk * cb);
  }
};

// Chunk placement of one stage (T tile rows x BK).
//   K-major (SWIZZLE_128B): thread t covers k-chunk (t & 7) of rows (t >> 3) + 32 i,
//     i < T/32; row r at (r >> 3) * 1024 + (r & 7) * 128, chunk c at c ^ (r & 7).
//   MN-major (SWIZZLE_128B_BASE32B): thread t covers row chunk (t % (T/4)) * 4 of
//     k-lines t / (T/4) + (1024/T) i, i < T/32; k-line kr of MN-atom a at
//     a*(BK*128) + kr*128, 32-byte granule g at g ^ (kr & 3) (LBO = BK*128, SBO = 512).
template <int T>
struct Place {
  static constexpr int N = T / 32;          // chunks per thread per stage
  static constexpr int CPR = T / 4;         // MN-major chunks per k-line
  static constexpr int KSTEP = GEMM_PRODUCERS / CPR;
  static __device__ __forceinline__ int krow(int tid, int i) { return (tid >> 3) + 32 * i; }
  static __device__ __forceinline__ uint32_t kdst(uint32_t sm, int tid, int i) {
    const int kc = tid & 7, r7 = (tid >> 3) & 7;
    return sm + ((tid >> 6) << 10) + (r7 << 7) + ((kc ^ r7) << 4) + i * 4096;
  }
  static __device__ __forceinline__ int mn(int tid) { return (tid % CPR) * 4; }
  static __device__ __forceinline__ int kr(int tid, int i) { return tid / CPR + KSTEP * i; }
  static __device__ __forceinline__ uint32_t mdst(uint32_t sm, int tid, int i) {
    const int m = mn(tid), k = kr(tid, i);
    return sm + (m >> 5) * (GEMM_BK * 128) + ((m & 4) << 2) + k * 128 + ((((m & 31) >> 3) ^ (k & 3)) << 5);
  }
};

// ---------------------------------------------------------------- loaders --
// K-major dense operand: op(r, k) = M(r, k).
struct LdDenseK {
  static constexpr int kMN = 0;
  static constexpr bool kTMA = false;
  MatView m;
  template <int T>
  struct State {
    const float* base[Place<T>::N];
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      int r = row0 + Place<T>::krow(tid, i);
      s.base[i] = r < m.rows ? m.p + (long long)r * m.ld : nullptr;
    }
  }
  template <int T>
  __device__ __forceinline__ void load(const State<T>& s, uint32_t sm, int k0, int tid) const {
    const int k = k0 + (tid & 7) * 4;  // multiple of 4; column blocks are multiples of 4 wide
    const int nv = m.cols - k;
    const int nb = nv <= 0 ? 0 : (nv >= 4 ? 16 : nv * 4);
    const long long off = nb ? m.col_off(k) : 0;
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      const bool ok = nb && s.base[i];
      cp_async16(Place<T>::kdst(sm, tid, i), ok ? s.base[i] + off : m.p, ok ? nb : 0);
    }
  }
};

// MN-major dense operand: op(r, k) = M(k, r) (4 consecutive r contiguous).
// ones_row >= 0 (a multiple of 4): that row chunk reads {1, 0, 0, 0}.
struct LdDenseMN {
  static constexpr int kMN = 1;
  static constexpr bool kTMA = false;
  MatView m;
  int ones_row;
  template <int T>
  struct State {
    const float* col;  // &M(0, this thread's column chunk), or g_one4
    long long ld;      // 0 for the ones chunk
    int nb;
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    const int r = row0 + Place<T>::mn(tid);
    s.nb = 0;
    s.col = m.p;
    s.ld = m.ld;
    if (r < m.cols) {
      const int nv = m.cols - r;
      s.nb = (nv >= 4 ? 4 : nv) * 4;
      s.col = m.p + m.col_off(r);
    } else if (r == ones_row) {
      s.nb = 16;
      s.col = g_one4;
      s.ld = 0;
    }
  }
  template <int T>
  __device__ __forceinline__ void load(const State<T>& s, uint32_t sm, int k0, int tid) const {
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      const int k = k0 + Place<T>::kr(tid, i);
      const bool ok = s.nb && k < m.rows;
      cp_async16(Place<T>::mdst(sm, tid, i), ok ? s.col + (long long)k * s.ld : m.p, ok ? s.nb : 0);
    }
  }
};

struct ConvGeom {
  int N, H, W, C;       // input (C multiple of 4)
  int Co, R, S;         // filter
  int Ho, Wo, st, pad;  // output
  FastDiv fC, fS, fCo, fHoWo, fWo, fHW, fW;
};

// Convolution forward, A(m, k): m = (n, oh, ow), k = (r, s, c); x NHWC.
struct LdConvFwdA {
  static constexpr int kMN = 0;
  static constexpr bool kTMA = false;
  const float* x;
  ConvGeom g;
  template <int T>
  struct State {
    const float* base[Place<T>::N];  // x at (n, oh*st - p, ow*st - p, 0) (may point outside x)
    int h0[Place<T>::N], w0[Place<T>::N];
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    const int Mtot = g.N * g.Ho * g.Wo;
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      const int m = row0 + Place<T>::krow(tid, i);
      if (m < Mtot) {
        const int n = g.fHoWo.div(m), rem = m - n * g.Ho * g.Wo;
        const int oh = g.fWo.div(rem), ow = rem - oh * g.Wo;
        s.h0[i] = oh * g.st - g.pad;
        s.w0[i] = ow * g.st - g.pad;
        s.base[i] = x + (((long long)n * g.H + s.h0[i]) * g.W + s.w0[i]) * g.C;
      } else {
        s.h0[i] = -(1 << 28);
        s.w0[i] = 0;
        s.base[i] = x;
      }
    }
  }
  template <int T>
  __device__ __forceinline__ void load(const State<T>& s, uint32_t sm, int k0, int tid) const {
    const int k = k0 + (tid & 7) * 4;
    const bool kok = k < g.R * g.S * g.C;
    const int rs = g.fC.div(k), c = k - rs * g.C;
    const int r = g.fS.div(rs), sc = rs - r * g.S;
    const int off = (r * g.W + sc) * g.C + c;
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      const int h = s.h0[i] + r, w = s.w0[i] + sc;
      const bool ok = kok && (unsigned)h < (unsigned)g.H && (unsigned)w < (unsigned)g.W;
      cp_async16(Place<T>::kdst(sm, tid, i), ok ? s.base[i] + off : x, ok ? 16 : 0);
    }
  }
};

// Convolution data gradient, A(m, k): m = (n, h, w) over the input,
// k = (r, s, co); value dy[n][(h+p-r)/st][(w+p-s)/st][co] when integral & in range.
struct LdConvDgradA {
  static constexpr int kMN = 0;
  static constexpr bool kTMA = false;
  const float* dy;
  ConvGeom g;
  template <int T>
  struct State {
    const float* base[Place<T>::N];  // stride 1: dy at (n, h+p, w+p, 0)
    int hp[Place<T>::N], wp[Place<T>::N], n[Place<T>::N];
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    const int Mtot = g.N * g.H * g.W;
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      const int m = row0 + Place<T>::krow(tid, i);
      if (m < Mtot) {
        const int n = g.fHW.div(m), rem = m - n * g.H * g.W;
        const int h = g.fW.div(rem), w = rem - h * g.W;
        s.hp[i] = h + g.pad;
        s.wp[i] = w + g.pad;
        s.n[i] = n;
        s.base[i] = dy + (((long long)n * g.Ho + s.hp[i]) * g.Wo + s.wp[i]) * g.Co;
      } else {
        s.hp[i] = -(1 << 28);
        s.wp[i] = 0;
        s.n[i] = 0;
        s.base[i] = dy;
      }
    }
  }
  template <int T>
  __device__ __forceinline__ void load(const State<T>& s, uint32_t sm, int k0, int tid) const {
    const int k = k0 + (tid & 7) * 4;
    const bool kok = k < g.R * g.S * g.Co;
    const int rs = g.fCo.div(k), co = k - rs * g.Co;
    const int r = g.fS.div(rs), sc = rs - r * g.S;
    if (g.st == 1) {
      const int off = co - (r * g.Wo + sc) * g.Co;
#pragma unroll
      for (int i = 0; i < Place<T>::N; ++i) {
        const int oh = s.hp[i] - r, ow = s.wp[i] - sc;
        const bool ok = kok && (unsigned)oh < (unsigned)g.Ho && (unsigned)ow < (unsigned)g.Wo;
        cp_async16(Place<T>::kdst(sm, tid, i), ok ? s.base[i] + off : dy, ok ? 16 : 0);
      }
    } else {
#pragma unroll
      for (int i = 0; i < Place<T>::N; ++i) {
        int oh = s.hp[i] - r, ow = s.wp[i] - sc;
        bool ok = kok && oh >= 0 && ow >= 0 && oh % g.st == 0 && ow % g.st == 0;
        oh /= g.st;
        ow /= g.st;
        ok = ok && oh < g.Ho && ow < g.Wo;
        cp_async16(Place<T>::kdst(sm, tid, i),
                   ok ? dy + (((long long)s.n[i] * g.Ho + oh) * g.Wo + ow) * g.Co + co : dy, ok ? 16 : 0);
      }
    }
  }
};

// Convolution data gradient, B(c, k) = W[co][r][s][c] with k = (r, s, co); MN-major (c contiguous).
struct LdConvDgradB {
  static constexpr int kMN = 1;
  static constexpr bool kTMA = false;
  const float* Wt;
  ConvGeom g;
  template <int T>
  struct State {
    int c;
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    s.c = row0 + Place<T>::mn(tid);
  }
  template <int T>
  __device__ __forceinline__ void load(const State<T>& s, uint32_t sm, int k0, int tid) const {
    const int RS = g.R * g.S;
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      const int k = k0 + Place<T>::kr(tid, i);
      const bool ok = s.c < g.C && k < RS * g.Co;
      const int rs = g.fCo.div(k), co = k - rs * g.Co;
      cp_async16(Place<T>::mdst(sm, tid, i), ok ? Wt + ((long long)co * RS + rs) * g.C + s.c : Wt, ok ? 16 : 0);
    }
  }
};

// Convolution weight gradient, A(kg, m) = x[n][oh*st-p+r][ow*st-p+s][c] with
// kg = (r, s, c) the GEMM row and m = (n, oh, ow) the reduction index; MN-major.
// Row ones_row (= R*S*C) is the ones row of the fused bias gradient.
struct LdConvWgradA {
  static constexpr int kMN = 1;
  static constexpr bool kTMA = false;
  const float* x;
  ConvGeom g;
  int ones_row;
  template <int T>
  struct State {
    int r, s, off;  // off = (r*W + s)*C + c
    int mode;       // 0 outside, 1 data, 2 ones
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    const int kg = row0 + Place<T>::mn(tid);
    s.mode = 0;
    s.r = s.s = s.off = 0;
    if (kg < g.R * g.S * g.C) {
      const int rs = g.fC.div(kg), c = kg - rs * g.C;
      s.r = g.fS.div(rs);
      s.s = rs - s.r * g.S;
      s.off = (s.r * g.W + s.s) * g.C + c;
      s.mode = 1;
    } else if (kg == ones_row) {
      s.mode = 2;
    }
  }
  template <int T>
  __device__ __forceinline__ void load(const State<T>& s, uint32_t sm, int k0, int tid) const {
    // The k-lines (pixels) of this thread are warp-uniform when 32 | T/4 (T = 128):
    // lanes 0..N-1 decompose pixel k0 + kr(tid, lane), the warp shares them.
    static_assert(Place<T>::CPR % 32 == 0 || Place<T>::CPR < 32, "mapping");
    const int Mtot = g.N * g.Ho * g.Wo;
    const int lane = tid & 31;
    if constexpr (Place<T>::CPR % 32 == 0) {
      int poff = 0, ph0 = -(1 << 28), pw0 = 0;
      if (lane < Place<T>::N) {
        const int m = k0 + Place<T>::kr(tid - lane, lane);
        if (m < Mtot) {
          const int n = g.fHoWo.div(m), rem = m - n * g.Ho * g.Wo;
          const int oh = g.fWo.div(rem), ow = rem - oh * g.Wo;
          ph0 = oh * g.st - g.pad;
          pw0 = ow * g.st - g.pad;
          poff = ((n * g.H + ph0) * g.W + pw0) * g.C;
        }
      }
#pragma unroll
      for (int i = 0; i < Place<T>::N; ++i) {
        const int off = __shfl_sync(0xffffffffu, poff, i);
        const int h = __shfl_sync(0xffffffffu, ph0, i) + s.r;
        const int w = __shfl_sync(0xffffffffu, pw0, i) + s.s;
        bool ok = s.mode == 1 && (unsigned)h < (unsigned)g.H && (unsigned)w < (unsigned)g.W;
        const float* src = x + off + s.off;
        if (s.mode == 2) {
          ok = k0 + Place<T>::kr(tid, i) < Mtot;
          src = g_one4;
        }
        cp_async16(Place<T>::mdst(sm, tid, i), ok ? src : x, ok ? 16 : 0);
      }
    } else {
#pragma unroll
      for (int i = 0; i < Place<T>::N; ++i) {
        const int m = k0 + Place<T>::kr(tid, i);
        bool ok = m < Mtot && s.mode != 0;
        const float* src = g_one4;
        if (s.mode == 1) {
          const int n = g.fHoWo.div(m), rem = m - n * g.Ho * g.Wo;
          const int oh = g.fWo.div(rem), ow = rem - oh * g.Wo;
          const int h0 = oh * g.st - g.pad, w0 = ow * g.st - g.pad;
          ok = ok && (unsigned)(h0 + s.r) < (unsigned)g.H && (unsigned)(w0 + s.s) < (unsigned)g.W;
          src = x + ((n * g.H + h0) * g.W + w0) * g.C + s.off;
        }
        cp_async16(Place<T>::mdst(sm, tid, i), ok ? src : x, ok ? 16 : 0);
      }
    }
  }
};

// ------------------------------------------- shared-memory im2col loaders --
// The implicit-GEMM gathers re-read every input element R*S times from L2 (and
// with C = 4 a filter tap is one 16-byte granule, so the gather is pure
// latency).  These loaders stage the zero-padded input image of the current
// sample in a per-CTA shared-memory scratch once (cp.async, restaged when the
// sample changes; all producer threads in lock step via named barrier 2) and
// build each operand tile from it with ld.shared / st.shared.  Requires
// C % 4 == 0, every tile / k-block inside one image, and the padded image
// within kIm2colScratch bytes.
constexpr int kIm2colScratch = 64 * 1024;

__device__ __forceinline__ void producer_bar_sync() { asm volatile("bar.sync 2, 256;" ::: "memory"); }
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}

// Padded image of sample n, float4 granules: (ph, pw, c4) at ((ph*Wp + pw)*C4 + c4)
// = x[n][ph - pad][pw - pad][4 c4 .. 4 c4 + 3] (0 outside), ph < Hp = (Ho-1)*st + R,
// pw < Wp = (Wo-1)*st + S.
struct SmemImage {
  const float* x;
  ConvGeom g;
  int Hp, Wp, C4;
  FastDiv fWpC4, fC4;
  __device__ __forceinline__ void restage(int& staged, uint32_t scr, int n, int tid) const {
    if (n == staged) return;
    producer_bar_sync();  // every producer is done reading the previous image
    // all copies in flight at once (cp.async, zero-fill outside the image)
    const float4* x4 = reinterpret_cast<const float4*>(x) + (size_t)n * g.H * g.W * C4;
    const int total = Hp * Wp * C4;
    for (int i = tid; i < total; i += GEMM_PRODUCERS) {
      const int ph = fWpC4.div(i), r1 = i - ph * Wp * C4;
      const int pw = fC4.div(r1), c4 = r1 - pw * C4;
      const int ih = ph - g.pad, iw = pw - g.pad;
      const bool in = (unsigned)ih < (unsigned)g.H && (unsigned)iw < (unsigned)g.W;
      cp_async16(scr + i * 16, in ? x4 + (ih * g.W + iw) * C4 + c4 : x4, in ? 16 : 0);
    }
    cp_async_commit();
    cp_async_wait<0>();
    producer_bar_sync();
    staged = n;
  }
};

// Convolution forward A(m = (n, oh, ow), k = (r, s, c)), K-major.
struct LdConvFwdSmemA {
  static constexpr int kMN = 0;
  static constexpr bool kTMA = false;
  static constexpr int kScratch = kIm2colScratch;
  SmemImage im;
  template <int T>
  struct State {
    uint32_t scr;
    int pix[Place<T>::N];  // granule offset of (oh*st, ow*st, 0), -1 past the end
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    const ConvGeom& g = im.g;
    const int Mtot = g.N * g.Ho * g.Wo;
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      const int m = row0 + Place<T>::krow(tid, i);
      s.pix[i] = -1;
      if (m < Mtot) {
        const int n = g.fHoWo.div(m), rem = m - n * g.Ho * g.Wo;
        const int oh = g.fWo.div(rem), ow = rem - oh * g.Wo;
        s.pix[i] = (oh * g.st * im.Wp + ow * g.st) * im.C4;
      }
    }
  }
  template <int T>
  __device__ __forceinline__ void prepare(State<T>& s, int& staged, uint32_t scr, int row0, int k0, int tid) const {
    s.scr = scr;
    const int Mtot = im.g.N * im.g.Ho * im.g.Wo;
    im.restage(staged, scr, im.g.fHoWo.div(row0 < Mtot ? row0 : Mtot - 1), tid);
  }
  template <int T>
  __device__ __forceinline__ void load(const State<T>& s, uint32_t sm, int k0, int tid) const {
    const ConvGeom& g = im.g;
    const int k = k0 + (tid & 7) * 4;  // k = (r*S + s)*C + c, c % 4 == 0
    const bool kok = k < g.R * g.S * g.C;
    const int tap = g.fC.div(k), c4 = (k - tap * g.C) >> 2;
    const int r = g.fS.div(tap), sc = tap - r * g.S;
    const int off = (r * im.Wp + sc) * im.C4 + c4;
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (kok && s.pix[i] >= 0) v = lds4(s.scr + (s.pix[i] + off) * 16);
      sts4(Place<T>::kdst(sm, tid, i), v);
    }
  }
};

// Convolution weight gradient A(kg = (r, s, c), m = pixel), MN-major, with the
// bias-gradient ones row at kg = ones_row.
struct LdConvWgradSmemA {
  static constexpr int kMN = 1;
  static constexpr bool kTMA = false;
  static constexpr int kScratch = kIm2colScratch;
  SmemImage im;
  int ones_row;
  template <int T>
  struct State {
    uint32_t scr;
    int off;   // granule offset of (r, s, c4)
    int mode;  // 0 zero, 1 data, 2 ones
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    const ConvGeom& g = im.g;
    const int kg = row0 + Place<T>::mn(tid);  // multiple of 4
    s.mode = 0;
    s.off = 0;
    if (kg < g.R * g.S * g.C) {
      const int tap = g.fC.div(kg), c4 = (kg - tap * g.C) >> 2;
      const int r = g.fS.div(tap), sc = tap - r * g.S;
      s.off = (r * im.Wp + sc) * im.C4 + c4;
      s.mode = 1;
    } else if (kg == ones_row) {
      s.mode = 2;
    }
  }
  template <int T>
  __device__ __forceinline__ void prepare(State<T>& s, int& staged, uint32_t scr, int row0, int k0, int tid) const {
    s.scr = scr;
    const int Mtot = im.g.N * im.g.Ho * im.g.Wo;
    im.restage(staged, scr, im.g.fHoWo.div(k0 < Mtot ? k0 : Mtot - 1), tid);
  }
  template <int T>
  __device__ __forceinline__ void load(const State<T>& s, uint32_t sm, int k0, int tid) const {
    const ConvGeom& g = im.g;
    const int Mtot = g.N * g.Ho * g.Wo;
    const int HoWo = g.Ho * g.Wo;
#pragma unroll
    for (int i = 0; i < Place<T>::N; ++i) {
      const int p = k0 + Place<T>::kr(tid, i);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p < Mtot) {
        if (s.mode == 1) {
          const int rem = p - g.fHoWo.div(p) * HoWo;
          const int oh = g.fWo.div(rem), ow = rem - oh * g.Wo;
          v = lds4(s.scr + ((oh * g.st * im.Wp + ow * g.st) * im.C4 + s.off) * 16);
        } else if (s.mode == 2) {
          v.x = 1.f;
        }
      }
      sts4(Place<T>::mdst(sm, tid, i), v);
    }
  }
};

// Loaders whose scratch holds per-sample state want contiguous work ranges.
template <class T, class = void>
struct ContiguousOf {
  static constexpr bool value = false;
};
template <class T>
struct ContiguousOf<T, std::void_t<decltype(T::kScratch)>> {
  static constexpr bool value = true;
};

// Scratch bytes a loader needs (0 unless it declares kScratch).
template <class T, class = void>
struct ScratchOf {
  static constexpr int value = 0;
};
template <class T>
struct ScratchOf<T, std::void_t<decltype(T::kScratch)>> {
  static constexpr int value = T::kScratch;
};

// Producer warps issuing the A operand's TMA boxes (kIssueWarps parts, each part
// issued by its own warp, the B operand by one more warp); 1 unless declared.
template <class T, class = void>
struct IssueWarpsOf {
  static constexpr int value = 1;
};
template <class T>
struct IssueWarpsOf<T, std::void_t<decltype(T::kIssueWarps)>> {
  static constexpr int value = T::kIssueWarps;
};

// ------------------------------------------------------------ TMA loaders --
// One elected producer thread issues cp.async.bulk.tensor per operand per stage
// (tensor maps encoded on the host after the tile shape is chosen; layouts
// validated by tools/tma_test.cu).  Whole MN atoms past the data (`valid`) are
// constant: prefilled once per stage buffer with zeros and the ones row.

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

// Constant MN atoms: rows [valid, ...) are zero, except row ones_row (= 1).
template <int T>
__device__ __forceinline__ void prefill_const_atoms(uint32_t sm, int row0, int valid, int ones_row, int t, int nt) {
#pragma unroll 1
  for (int a = 0; a < T / 32; ++a) {
    const int r0 = row0 + 32 * a;
    if (r0 < valid) continue;
    // 32 k-lines x 128 B; the ones row sits at MN position (ones_row - r0)
    for (int i = t; i < 32 * 32; i += nt) {
      const int kr = i >> 5, mn = i & 31;
      const float v = (r0 + mn == ones_row) ? 1.f : 0.f;
      const uint32_t addr = sm + a * (GEMM_BK * 128) + kr * 128 + ((((mn >> 3) ^ (kr & 3))) << 5) + (mn & 7) * 4;
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
    }
  }
}

// K-major tile of a (possibly column-blocked) row-major matrix; box {32, T}.
struct TmaK {
  static constexpr int kMN = 0;
  static constexpr bool kTMA = true;
  CUtensorMap map;
  int blocked, cb;  // blocked: 3-D map {cb, rows, nblk}
  template <int T>
  __device__ __forceinline__ bool needs_prefill(int) const {
    return false;
  }
  template <int T>
  __device__ __forceinline__ void prefill(uint32_t, int, int, int) const {}
  template <int T>
  __device__ __forceinline__ void issue(uint32_t sm, int row0, int k0, uint32_t bar) const {
    mbar_expect_tx(bar, T * 128);
    if (blocked)
      tma_load_3d(sm, &map, k0 % cb, row0, k0 / cb, bar);
    else
      tma_load_2d(sm, &map, k0, row0, bar);
  }
};

// MN-major tile of M(k, mn) (mn contiguous), one {32 mn, 32 k} box per MN atom.
struct TmaMN {
  static constexpr int kMN = 1;
  static constexpr bool kTMA = true;
  CUtensorMap map;
  int blocked, cb;      // blocked along mn: 3-D map {cb, rows, nblk}
  int valid, ones_row;  // atoms starting at >= valid are constant (prefilled)
  int atoms;            // whole tile in one box: 3-D view {32, rows, cols/32}, box {32, 32, T/32}
  template <int T>
  __device__ __forceinline__ bool needs_prefill(int row0) const {
    return !atoms && row0 + T > valid;
  }
  template <int T>
  __device__ __forceinline__ void prefill(uint32_t sm, int row0, int t, int nt) const {
    prefill_const_atoms<T>(sm, row0, valid, ones_row, t, nt);
  }
  template <int T>
  __device__ __forceinline__ void issue(uint32_t sm, int mn0, int k0, uint32_t bar) const {
    if (atoms) {
      mbar_expect_tx(bar, T * 128);
      tma_load_3d(sm, &map, 0, k0, mn0 >> 5, bar);
      return;
    }
    int n = 0;
#pragma unroll
    for (int a = 0; a < T / 32; ++a) n += (mn0 + 32 * a < valid);
    mbar_expect_tx(bar, n * 32 * 128);
#pragma unroll
    for (int a = 0; a < T / 32; ++a) {
      const int mn = mn0 + 32 * a;
      if (mn >= valid) continue;
      if (blocked)
        tma_load_3d(sm + a * (GEMM_BK * 128), &map, mn % cb, k0, mn / cb, bar);
      else
        tma_load_2d(sm + a * (GEMM_BK * 128), &map, mn, k0, bar);
    }
  }
};

// im2col A operand of the convolution forward (fwd) or data gradient (dgrad,
// stride 1, taps flipped): 128 pixels of the walk x 32 channels at one tap.
struct TmaIm2col {
  static constexpr int kMN = 0;
  static constexpr bool kTMA = true;
  CUtensorMap map;
  int C, R, S, gH, gW;  // channels of the mapped tensor; walk grid gH x gW
  int st, lo;           // window origin of walk pixel (y, x): (y*st + lo, x*st + lo)
  int flip;
  FastDiv fC, fS, fHW, fW;
  template <int T>
  __device__ __forceinline__ bool needs_prefill(int) const {
    return false;
  }
  template <int T>
  __device__ __forceinline__ void prefill(uint32_t, int, int, int) const {}
  template <int T>
  __device__ __forceinline__ void issue(uint32_t sm, int m0, int k0, uint32_t bar) const {
    const int rs = fC.div(k0), c0 = k0 - rs * C;
    int r = fS.div(rs), s = rs - r * S;
    if (flip) {
      r = R - 1 - r;
      s = S - 1 - s;
    }
    const int n = fHW.div(m0), rem = m0 - n * gH * gW;
    const int y = fW.div(rem), x = rem - y * gW;
    mbar_expect_tx(bar, T * 128);  // one box of T pixels (encoded for the tile height)
    tma_load_im2col(sm, &map, c0, x * st + lo, y * st + lo, n, s, r, bar);
  }
};

// Data-gradient B(c, k = (rs, co)) = W[co][rs][c]: 3-D map {C, RS, Co}, box
// {32, 1, 32} per 32-channel atom, or (atoms4) the whole tile as ONE box of the
// 4-D view {32, RS, Co, C/32}, box {32, 1, 32, BN/32} (atom-consecutive in shared
// memory, channels past C zero-filled): one TMA issue per stage instead of BN/32.
struct TmaDgradB {
  static constexpr int kMN = 1;
  static constexpr bool kTMA = true;
  CUtensorMap map;
  int C, Co;
  int atoms4;
  FastDiv fCo;
  template <int T>
  __device__ __forceinline__ bool needs_prefill(int) const {
    return false;
  }
  template <int T>
  __device__ __forceinline__ void prefill(uint32_t, int, int, int) const {}
  template <int T>
  __device__ __forceinline__ void issue(uint32_t sm, int c0, int k0, uint32_t bar) const {
    const int rs = fCo.div(k0), co0 = k0 - rs * Co;
    if (atoms4) {
      mbar_expect_tx(bar, T * 128);
      tma_load_4d(sm, &map, 0, rs, co0, c0 >> 5, bar);
      return;
    }
    int n = 0;
#pragma unroll
    for (int a = 0; a < T / 32; ++a) n += (c0 + 32 * a < C);
    mbar_expect_tx(bar, n * 32 * 128);
#pragma unroll
    for (int a = 0; a < T / 32; ++a)
      if (c0 + 32 * a < C) tma_load_3d(sm + a * (GEMM_BK * 128), &map, c0 + 32 * a, rs, co0, bar);
  }
};

// Weight-gradient A(kg = (rs, c), m = pixel): im2col map with 32-pixel x
// 32-channel boxes (one per MN atom of 32 kg), C % 32 == 0; kg >= valid constant.
struct TmaWgradA {
  static constexpr int kMN = 1;
  static constexpr bool kTMA = true;
  // one 32-pixel im2col box per 32-channel atom: the issue of a box costs ~200
  // cycles of the issuing thread (tools/gemm_trace.py), so the 4 atoms of a
  // stage are issued by 4 producer warps side by side
  static constexpr int kIssueWarps = 4;
  CUtensorMap map;
  int C, S, Ho, Wo, st, pad;
  int valid, ones_row;
  FastDiv fC, fS, fHoWo, fWo;
  template <int T>
  __device__ __forceinline__ bool needs_prefill(int row0) const {
    return row0 + T > valid;
  }
  template <int T>
  __device__ __forceinline__ void prefill(uint32_t sm, int row0, int t, int nt) const {
    prefill_const_atoms<T>(sm, row0, valid, ones_row, t, nt);
  }
  template <int T>
  __device__ __forceinline__ void issue(uint32_t sm, int kg0, int k0, uint32_t bar) const {
    const int n = fHoWo.div(k0), rem = k0 - n * Ho * Wo;
    const int oh = fWo.div(rem), ow = rem - oh * Wo;
    int cnt = 0;
#pragma unroll
    for (int a = 0; a < T / 32; ++a) cnt += (kg0 + 32 * a < valid);
    mbar_expect_tx(bar, cnt * 32 * 128);
#pragma unroll
    for (int a = 0; a < T / 32; ++a) {
      const int kg = kg0 + 32 * a;
      if (kg >= valid) continue;
      const int rs = fC.div(kg), c0 = kg - rs * C;
      const int r = fS.div(rs), s = rs - r * S;
      tma_load_im2col(sm + a * (GEMM_BK * 128), &map, c0, ow * st - pad, oh * st - pad, n, s, r, bar);
    }
  }
  // atoms a = part, part + kIssueWarps, ... of the stage (own expect_tx)
  template <int T>
  __device__ __forceinline__ void issue_part(uint32_t sm, int kg0, int k0, uint32_t bar, int part) const {
    const int n = fHoWo.div(k0), rem = k0 - n * Ho * Wo;
    const int oh = fWo.div(rem), ow = rem - oh * Wo;
    int cnt = 0;
    for (int a = part; a < T / 32; a += kIssueWarps) cnt += (kg0 + 32 * a < valid);
    if (cnt) mbar_expect_tx(bar, cnt * 32 * 128);
    for (int a = part; a < T / 32; a += kIssueWarps) {
      const int kg = kg0 + 32 * a;
      if (kg >= valid) continue;
      const int rs = fC.div(kg), c0 = kg - rs * C;
      const int r = fS.div(rs), s = rs - r * S;
      tma_load_im2col(sm + a * (GEMM_BK * 128), &map, c0, ow * st - pad, oh * st - pad, n, s, r, bar);
    }
  }
};

// ---------------------------------------------------------------------------
// Epilogue parameters.  Output element (m, n) goes to out(m, n) (trans = 0) or
// out(n, m) (trans = 1) of a blocked row-major view for m < mvalid; row
// m == xrow goes to xout[n] (fused bias gradient); other rows are dropped.
// With ws != nullptr the CTA writes its raw K-split partial to
// ws[split][m][n] (ld = ws_ld) instead.
struct EpiArgs {
  float* p;
  long long ld, bs;
  int cb, trans;
  const float* bias;  // indexed by n (bias_on_m = 0) or by m
  int bias_on_m;
  int relu;
  int rn;  // round the stored outputs to TF32 (reading A19: the output is a GEMM operand)
  int mvalid, xrow;
  float* xout;
  float* ws;
  long long ws_ld, ws_split_stride;
  int* cnt;  // split-K tile counters (zero between GEMMs); null: separate reduce kernel
};

__device__ __forceinline__ float* out_at(const EpiArgs& e, int i, int j, int cols) {
  if (e.cb >= cols) return e.p + (long long)i * e.ld + j;
  int blk = j / e.cb;
  return e.p + (long long)blk * e.bs + (long long)i * e.ld + (j - blk * e.cb);
}

template <class LA, class LB>
struct GemmArgs {
  LA a;
  LB b;
  int M, N, K;
  int kb_per_split;  // k-blocks of one work item (a K split)
  EpiArgs epi;
  int async_arrive;  // cp.async producers: mbarrier arrive on copy completion (else LAG-delayed arrive)
};

// Shared-memory descriptor of the kk-th K=8 step of a stage tile, per operand
// layout: 0 K-major SWIZZLE_128B, 1 MN-major SWIZZLE_128B_BASE32B, 2 K-major
// no-swizzle (16-byte K chunks of T rows at 2 KB), 3 MN-major no-swizzle
// (16-byte MN chunks of 32 k-lines at 512 B).
template <int T, int LAYOUT>
__device__ __forceinline__ uint64_t tile_desc(uint32_t sm, int kk) {
  if constexpr (LAYOUT == 0) {
    return umma_desc_sw128(sm + kk * 32, 16, 1024);
  } else if constexpr (LAYOUT == 1) {
    return umma_desc_mn_sw128_32b(sm + kk * 8 * 128, GEMM_BK * 128, 512);
  } else if constexpr (LAYOUT == 2) {
    return umma_desc_noswz(sm + kk * 2 * (T * 16), T * 16, 128);
  } else {
    return umma_desc_noswz(sm + kk * 128, 128, GEMM_BK * 16);
  }
}

// MT = M tiles of 128 rows per CTA work item (2: a 256-row tile, both halves
// sharing the B stage: twice the MMA work per B box for narrow N).
template <int BN, int SCRATCH = 0, int MT = 1>
constexpr int gemm_stages() {
  // default depth; with a loader scratch as many stages as fit 225 KB
  constexpr int d = MT == 2 ? 5 : BN <= 32 ? 8 : BN <= 64 ? 7 : BN <= 128 ? 6 : BN <= 192 ? 5 : 4;
  constexpr int fit = (225 * 1024 - SCRATCH) / ((MT * GEMM_BM + BN) * GEMM_BK * 4);
  return d < fit ? d : fit;
}

template <int BN, int STAGES, int SCRATCH = 0, int MT = 1>
constexpr int gemm_smem_bytes() {
  return STAGES * (MT * GEMM_BM * GEMM_BK * 4 + BN * GEMM_BK * 4) + SCRATCH + 1024 /*align*/ + 256 /*barriers*/;
}

// Second counter block of the split-K workspace head (re-arm counters).
constexpr int kSplitDone = 256;

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Final epilogue of 4 consecutive columns (col0 .. col0+3, guarded by N).
__device__ __forceinline__ void epi_store4(const EpiArgs& e, int row, int col0, float4 v4, int N) {
  const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int col = col0 + j;
    if (col >= N) break;
    float o = v[j];
    if (row >= e.mvalid) {
      if (row == e.xrow) e.xout[col] = o;
      continue;
    }
    if (e.bias) o += e.bias_on_m ? e.bias[row] : e.bias[col];
    if (e.relu) o = fmaxf(o, 0.f);
    if (e.rn) o = tf32_rna(o);
    if (e.trans)
      *out_at(e, col, row, e.mvalid) = o;
    else
      *out_at(e, row, col, N) = o;
  }
}

// Final epilogue of 16 consecutive accumulator columns of one row: bias, ReLU,
// plain / transposed / column-blocked store, or the bias-gradient row (xrow).
__device__ __forceinline__ void epi_store16(const EpiArgs& e, int row, int col0, const float (&v)[16], int N,
                                            bool plain_vec) {
  if (row >= e.mvalid) {
    if (row == e.xrow) {
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (col0 + i < N) e.xout[col0 + i] = v[i];
    }
    return;
  }
  if (plain_vec && col0 + 15 < N) {
    float* dst = e.p + (long long)row * e.ld + col0;
#pragma unroll
    for (int i = 0; i < 16; i += 4) {
      float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      if (e.bias) {
        o.x += e.bias[col0 + i];
        o.y += e.bias[col0 + i + 1];
        o.z += e.bias[col0 + i + 2];
        o.w += e.bias[col0 + i + 3];
      }
      if (e.relu) {
        o.x = fmaxf(o.x, 0.f);
        o.y = fmaxf(o.y, 0.f);
        o.z = fmaxf(o.z, 0.f);
        o.w = fmaxf(o.w, 0.f);
      }
      *reinterpret_cast<float4*>(dst + i) = tf32_rna4_if(o, e.rn);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int col = col0 + i;
    if (col >= N) break;
    float o = v[i];
    if (e.bias) o += e.bias_on_m ? e.bias[row] : e.bias[col];
    if (e.relu) o = fmaxf(o, 0.f);
    if (e.rn) o = tf32_rna(o);
    if (e.trans)
      *out_at(e, col, row, e.mvalid) = o;
    else
      *out_at(e, row, col, N) = o;
  }
}

// Optional per-role timeline of CTA 0 (build variant -D SG_GEMM_TRACE; read with
// sg_debug_gemm_trace): rows = producer start / end of a k-block, MMA operands
// ready / issued, epilogue accumulator ready / released per tile, kernel start.
#ifdef SG_GEMM_TRACE
__device__ long long g_gemm_trace[7][256];
#define SG_TRACE(row, idx)                                                            \
  do {                                                                                \
    if (blockIdx.x == 0 && (idx) < 256) g_gemm_trace[row][idx] = (long long)clock64(); \
  } while (0)
#else
#define SG_TRACE(row, idx) \
  do {                     \
  } while (0)
#endif

// Persistent warp-specialised kernel.  Work items = (M tile, N tile, K split),
// strided over the CTAs; the operand pipeline runs across work items without
// draining, and the accumulator is double-buffered in TMEM so the epilogue of
// one item overlaps the main loop of the next.
//   warps 0-7  : producers (cp.async: all 256 threads; TMA: warp 0, lane 0 issues)
//   warp 8     : MMA issuer (lane 0)
//   warps 9-16 : epilogue (TMEM lane group warp % 4; column half (warp - 9) / 4)
constexpr int GEMM_EPI_WARPS = 8;
constexpr int GEMM_ALL_THREADS = GEMM_PRODUCERS + 32 + GEMM_EPI_WARPS * 32;

struct WorkDecode {
  int mt, nt, splits;
  __device__ __forceinline__ void get(int w, int& mi, int& ni, int& si) const {
    // M tile fastest: CTAs running side by side share the B tile (and its L2 lines)
    mi = w % mt;
    const int r = w / mt;
    ni = r % nt;
    si = r / nt;
  }
};

template <int BN, int STAGES, class LA, class LB, int MT = 1>
__global__ void __launch_bounds__(GEMM_ALL_THREADS, 1) gemm_tc_kernel(const __grid_constant__ GemmArgs<LA, LB> args) {
  constexpr int TM = MT * GEMM_BM;  // rows of a work item
  constexpr int A_HALF = GEMM_BM * GEMM_BK * 4;
  constexpr int A_BYTES = MT * A_HALF;
  constexpr int B_BYTES = BN * GEMM_BK * 4;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // two accumulator buffers, allocation rounded up to a power of two (BN = 192: 512)
  constexpr int ACC = MT * BN;  // accumulator columns of one work item
  constexpr int TMEM_COLS = 2 * ACC <= 32 ? 32 : 2 * ACC <= 64 ? 64 : 2 * ACC <= 128 ? 128 : 2 * ACC <= 256 ? 256 : 512;
  static_assert(2 * ACC <= 512, "TMEM");
  static_assert(MT == 1 || (LA::kTMA && ScratchOf<LA>::value == 0), "256-row tiles: TMA operands only");
  constexpr int LAG = STAGES > 2 ? STAGES - 2 : 1;
  constexpr int MMA_WARP = GEMM_PRODUCERS / 32;
  constexpr int EPI_WARP0 = MMA_WARP + 1;
  static_assert(BN % 32 == 0 && BN <= 256, "BN");
  static_assert(GEMM_EPI_WARPS * 32 == 256, "epi_bar_sync() counts 256 threads");
  static_assert(LA::kTMA == LB::kTMA, "both operands TMA or both cp.async");
  constexpr bool TMA = LA::kTMA;

  constexpr int SCRATCH = ScratchOf<LA>::value;
  static_assert(ScratchOf<LB>::value == 0, "scratch is an A-operand feature");
  // TMA producer warps: the A operand's parts, then one warp for B (box issues of
  // the two operands overlap)
  constexpr int NA_ISSUE = IssueWarpsOf<LA>::value;
  constexpr int NPW = NA_ISSUE + 1;
  static_assert(NPW * 32 <= GEMM_PRODUCERS, "issue warps");

  extern __shared__ uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t scratch = sbase + STAGES * STAGE_BYTES;  // loader scratch (SCRATCH bytes)
  const uint32_t bar_base = scratch + SCRATCH;
  // full[s] at bar_base + 8s, empty[s] at +8(STAGES+s), tfull[b] at +16 STAGES + 8b,
  // tempty[b] at +16 STAGES + 16 + 8b, tmem slot after.
  const uint32_t tfull_bar = bar_base + 16 * STAGES;
  const uint32_t tempty_bar = tfull_bar + 16;
  const uint32_t tmem_slot = tempty_bar + 16;
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));

  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;  // warp-uniform role
  const int nkb_total = (args.K + GEMM_BK - 1) / GEMM_BK;
  const WorkDecode wd{(args.M + TM - 1) / TM, (args.N + BN - 1) / BN,
                      (nkb_total + args.kb_per_split - 1) / (args.kb_per_split > 0 ? args.kb_per_split : 1)};
  const int nwork = wd.mt * wd.nt * (wd.splits > 0 ? wd.splits : 1);
  // work items of this CTA: strided (neighbouring CTAs share operand tiles in
  // L2) or, for loaders that keep per-sample state, one contiguous range
  // (the loops stay "w = blockIdx.x; w < nwork_it; w += gridDim.x"; a stateful
  // loader remaps the j-th item of CTA b to item b*per + j and skips the tail)
  constexpr bool CONTIG = ContiguousOf<LA>::value;
  const int per_cta = CONTIG ? (nwork + (int)gridDim.x - 1) / (int)gridDim.x : 0;
  const int nwork_it = CONTIG ? per_cta * (int)gridDim.x : nwork;
  auto work_of = [&](int w) {
    return CONTIG ? (w % (int)gridDim.x) * per_cta + w / (int)gridDim.x : w;
  };
  auto kb_range = [&](int si, int& kb0, int& nkb) {
    kb0 = si * args.kb_per_split;
    int e = kb0 + args.kb_per_split;
    if (e > nkb_total) e = nkb_total;
    nkb = e - kb0;
  };

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_base + 8 * s, TMA ? NPW : GEMM_PRODUCERS);  // TMA issuing warps / every producer thread
      mbar_init(bar_base + 8 * (STAGES + s), 1);              // tcgen05.commit
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull_bar + 8 * b, 1);                        // tcgen05.commit
      mbar_init(tempty_bar + 8 * b, GEMM_EPI_WARPS * 32);     // every epilogue thread
    }
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc<TMEM_COLS>(tmem_slot);
  if constexpr (TMA) {
    if (tid == 0) {
      prefetch_tmap(&args.a.map);
      prefetch_tmap(&args.b.map);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;
  // the prologue above overlapped the previous kernel; its outputs are read below
  pdl_entry();
  if (tid == 0) SG_TRACE(6, 0);

  if (warp < MMA_WARP) {
    // ------------------------------- producers -------------------------------
    if constexpr (TMA) {
      if (warp < NPW) {
        int it = 0;
        int tagA[STAGES], tagB[STAGES];  // row0 the stage's constant atoms were written for
#pragma unroll
        for (int s = 0; s < STAGES; ++s) tagA[s] = tagB[s] = -1;
        for (int w = blockIdx.x; w < nwork_it; w += gridDim.x) {
          if (CONTIG && work_of(w) >= nwork) break;
          int mi, ni, si, kb0, nkb;
          wd.get(work_of(w), mi, ni, si);
          kb_range(si, kb0, nkb);
          const int m0 = mi * TM, n0 = ni * BN;
          for (int j = 0; j < nkb; ++j, ++it) {
            const int s = it % STAGES;
            const int round = it / STAGES;
            if (round > 0) mbar_wait(bar_base + 8 * (STAGES + s), (round - 1) & 1);
            if (lane == 0 && warp == 0) SG_TRACE(0, it);
            const uint32_t sa = sbase + s * STAGE_BYTES;
            // constant operand atoms (zeros / the bias ones-row) are written by warp 0
            bool wrote = false;
#pragma unroll
            for (int q = 0; q < STAGES; ++q) {
              if (q != s || warp != 0) continue;
              // (a tag names the row0 whose constant atoms the stage holds; a tile
              // without constant atoms lets TMA overwrite them, clearing the tag)
              if (!args.a.template needs_prefill<TM>(m0)) {
                tagA[q] = -1;
              } else if (tagA[q] != m0) {
                args.a.template prefill<TM>(sa, m0, lane, 32);
                tagA[q] = m0;
                wrote = true;
              }
              if (!args.b.template needs_prefill<BN>(n0)) {
                tagB[q] = -1;
              } else if (tagB[q] != n0) {
                args.b.template prefill<BN>(sa + A_BYTES, n0, lane, 32);
                tagB[q] = n0;
                wrote = true;
              }
            }
            if (wrote) {
              fence_proxy_async_smem();
              __syncwarp();
            }
            if (lane == 0) {
              const uint32_t full = bar_base + 8 * s;
              const int k0 = (kb0 + j) * GEMM_BK;
              if (warp < NA_ISSUE) {
                if constexpr (NA_ISSUE == 1)
                  args.a.template issue<TM>(sa, m0, k0, full);
                else
                  args.a.template issue_part<TM>(sa, m0, k0, full, warp);
              } else {
                args.b.template issue<BN>(sa + A_BYTES, n0, k0, full);
              }
              mbar_arrive(full);  // after this warp's expect_tx (the phase needs all NPW arrivals)
              if (warp == 0) SG_TRACE(1, it);
            }
            __syncwarp();
          }
        }
      }
    } else {
      int it = 0;
      int staged = -1;  // sample whose padded image is in the scratch (smem im2col loaders)
      (void)staged;
      for (int w = blockIdx.x; w < nwork_it; w += gridDim.x) {
        if (CONTIG && work_of(w) >= nwork) break;
        int mi, ni, si, kb0, nkb;
        wd.get(work_of(w), mi, ni, si);
        kb_range(si, kb0, nkb);
        typename LA::template State<GEMM_BM> sa_st;
        typename LB::template State<BN> sb_st;
        args.a.template init<GEMM_BM>(sa_st, mi * GEMM_BM, tid);
        args.b.template init<BN>(sb_st, ni * BN, tid);
        for (int j = 0; j < nkb; ++j, ++it) {
          const int s = it % STAGES;
          const int round = it / STAGES;
          if (round > 0) mbar_wait(bar_base + 8 * (STAGES + s), (round - 1) & 1);
          if (tid == 0) SG_TRACE(0, it);
          const uint32_t sa = sbase + s * STAGE_BYTES;
          const int k0 = (kb0 + j) * GEMM_BK;
          if constexpr (SCRATCH > 0) args.a.template prepare<GEMM_BM>(sa_st, staged, scratch, mi * GEMM_BM, k0, tid);
          args.a.template load<GEMM_BM>(sa_st, sa, k0, tid);
          args.b.template load<BN>(sb_st, sa + A_BYTES, k0, tid);
          if (args.async_arrive) {
            // the barrier counts this thread's arrival once its copies have
            // landed; the MMA warp fences them into the async proxy
            cp_async_mbar_arrive_noinc(bar_base + 8 * s);
            if (tid == 0) SG_TRACE(1, it);
            continue;
          }
          cp_async_commit();
          if (it >= LAG) {
            // this thread's copies of stage it-LAG have landed: make them visible
            // to the tensor-core (async) proxy, then release the stage.
            cp_async_wait<LAG>();
            fence_proxy_async_smem();
            mbar_arrive(bar_base + 8 * ((it - LAG) % STAGES));
          }
        }
      }
      if (args.async_arrive) {
        cp_async_wait_all();
      } else {
        cp_async_wait<0>();
        fence_proxy_async_smem();
        for (int j = (it > LAG ? it - LAG : 0); j < it; ++j) mbar_arrive(bar_base + 8 * (j % STAGES));
      }
    }
  } else if (warp == MMA_WARP) {
    // ------- MMA issuer: the whole warp runs the loop, elect.sync picks the issuing lane -------
    constexpr uint32_t idesc = idesc_tf32(GEMM_BM, BN, LA::kMN & 1, LB::kMN & 1);
    int it = 0, local = 0;
    for (int w = blockIdx.x; w < nwork_it; w += gridDim.x, ++local) {
      if (CONTIG && work_of(w) >= nwork) break;
      int mi, ni, si, kb0, nkb;
      wd.get(work_of(w), mi, ni, si);
      kb_range(si, kb0, nkb);
      const int b = local & 1;
      const int use = local >> 1;  // how many times buffer b was used before
      if (use > 0) mbar_wait(tempty_bar + 8 * b, (use - 1) & 1);
      tc_fence_after();
      const uint32_t acc = tmem + b * ACC;
      for (int j = 0; j < nkb; ++j, ++it) {
        const int s = it % STAGES;
#ifdef SG_MMA_BACKOFF
        mbar_wait_sleep(bar_base + 8 * s, (it / STAGES) & 1);
#else
        mbar_wait(bar_base + 8 * s, (it / STAGES) & 1);
#endif
        if (lane == 0) SG_TRACE(2, it);
        if constexpr (!TMA) {
          if (args.async_arrive) fence_proxy_async_smem();  // producers' generic-proxy writes -> tensor core
        }
        tc_fence_after();
        {
          const uint32_t sa = sbase + s * STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < GEMM_BK / 8; ++kk) {
            const uint64_t bd = tile_desc<BN, LB::kMN>(sa + A_BYTES, kk);  // kMN also names the smem layout
#pragma unroll
            for (int h = 0; h < MT; ++h) {  // 128-row halves of the A stage, one accumulator each
              const uint64_t ad = tile_desc<GEMM_BM, LA::kMN>(sa + h * A_HALF, kk);
              mma_tf32_warp(acc + h * BN, ad, bd, idesc, (j | kk) ? 1u : 0u);
            }
          }
          mma_commit_warp(bar_base + 8 * (STAGES + s));
          if (lane == 0) SG_TRACE(3, it);
        }
        __syncwarp();
      }
      mma_commit_warp(tfull_bar + 8 * b);
      __syncwarp();
    }
  } else {
    // ---------------------------------- epilogue ----------------------------------
    const int lg = warp & 3;  // TMEM lane group this warp may access
    // MT = 1: the two warp quads take the column halves; MT = 2: quad g takes
    // all columns of the 128-row half g
    constexpr int HALF = MT == 1 ? BN / 2 : BN;
    const int quad = (warp - EPI_WARP0) >> 2;
    const int cbeg = MT == 1 ? quad * HALF : 0;
    const int rhalf = MT == 1 ? 0 : quad;
    const EpiArgs& e = args.epi;
    const bool plain_vec = !e.trans && e.cb >= args.N && (e.ld & 3) == 0 && !e.bias_on_m;
    int local = 0;
    for (int w = blockIdx.x; w < nwork_it; w += gridDim.x, ++local) {
      if (CONTIG && work_of(w) >= nwork) break;
      int mi, ni, si, kb0, nkb;
      wd.get(work_of(w), mi, ni, si);
      kb_range(si, kb0, nkb);
      const int b = local & 1;
#ifdef SG_EPI_BACKOFF
      mbar_wait_sleep(tfull_bar + 8 * b, (local >> 1) & 1);
#else
      mbar_wait(tfull_bar + 8 * b, (local >> 1) & 1);
#endif
      if (warp == EPI_WARP0 && lane == 0) SG_TRACE(4, local);
      tc_fence_after();
      const int m0 = mi * TM, n0 = ni * BN;
      const int row = m0 + rhalf * GEMM_BM + lg * 32 + lane;
      const uint32_t tb = tmem + b * ACC + rhalf * BN + ((uint32_t)(lg * 32) << 16);
#pragma unroll 1
      for (int c0 = cbeg; c0 < cbeg + HALF; c0 += 16) {
        if (n0 + c0 >= args.N) break;
        float v[16];
        if (nkb > 0) {
          tmem_ld16(tb + c0, v);
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = 0.f;
        }
        if (row >= args.M) continue;
        if (e.ws) {
          float* dst = e.ws + (long long)si * e.ws_split_stride + (long long)row * e.ws_ld + n0 + c0;
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            if (n0 + c0 + i + 3 < args.N) {
              *reinterpret_cast<float4*>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            } else {
              for (int t = 0; t < 4; ++t)
                if (n0 + c0 + i + t < args.N) dst[i + t] = v[i + t];
            }
          }
          continue;
        }
        epi_store16(e, row, n0 + c0, v, args.N, plain_vec);
      }
      // this buffer's accumulator has been read: release it to the MMA warp
      tc_fence_before();
      mbar_arrive(tempty_bar + 8 * b);
      if (warp == EPI_WARP0 && lane == 0) SG_TRACE(5, local);
      if (e.ws && e.cnt) {
        // Cooperative split-K reduction.  The planner keeps tiles x splits <= the
        // grid, so every split of a tile is a resident CTA with exactly this one
        // work item: once all S partials of the tile are written (tile counter),
        // split si sums rows [si*BM/S, (si+1)*BM/S) of the tile over the splits in
        // ascending order and applies the epilogue (deterministic).
        const int t = mi + wd.mt * ni, S = wd.splits;
        __threadfence();
        epi_bar_sync();
        if (warp == EPI_WARP0 && lane == 0) {
          atomicAdd(e.cnt + t, 1);
          while (ld_acquire_gpu(e.cnt + t) < S) __nanosleep(32);
        }
        epi_bar_sync();
        __threadfence();
        const int r_b = m0 + si * TM / S;
        const int r_e = min(m0 + (si + 1) * TM / S, args.M);
        constexpr int C4 = BN / 4;
        const int et = (warp - EPI_WARP0) * 32 + lane;
        for (int idx = et; idx < (r_e - r_b) * C4; idx += GEMM_EPI_WARPS * 32) {
          const int r = r_b + idx / C4, c = n0 + (idx % C4) * 4;
          if (c >= args.N) continue;
          const float* src = e.ws + (long long)r * e.ws_ld + c;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int s2 = 0; s2 < S; ++s2) {
            const float4 u = __ldcg(reinterpret_cast<const float4*>(src + (long long)s2 * e.ws_split_stride));
            acc.x += u.x;
            acc.y += u.y;
            acc.z += u.z;
            acc.w += u.w;
          }
          epi_store4(e, r, c, acc, args.N);
        }
        // re-arm both counters once every split has finished its slice
        epi_bar_sync();
        if (warp == EPI_WARP0 && lane == 0) {
          if (atomicAdd(e.cnt + kSplitDone + t, 1) == S - 1) {
            e.cnt[t] = 0;
            e.cnt[kSplitDone + t] = 0;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
  }
}

}  // namespace sg
