// tcgen05 (kind::tf32) implicit-GEMM engine shared by the convolution and
// inner-product layers ("rotates (multiply W)"
// convolution).
//
//   D[m][n] = sum_k A(m, k) * B(n, k)      fp32 storage, TF32 operands, fp32 accumulate
//
// One CTA computes a 128 x BN output tile (optionally one K-split of it):
//   warps 0-3 : producers — gather 16-byte chunks with cp.async (zero-filled
//               outside the operand) straight into the UMMA canonical layouts,
//               one stage of BK = 32 fp32 (128 B) per step; then the epilogue
//               (TMEM -> registers -> global).
//   warp 4    : TMEM allocation and the single MMA-issuing thread.
// Operands are "loaders": each maps a (row, k) of the GEMM onto the layer's
// native tensor (NHWC activations, KRSC / [d_v][d_h] weights), so the im2col
// of the convolution is never materialised.  A loader is K-major (4
// consecutive k contiguous in memory) or MN-major (4 consecutive rows
// contiguous); tcgen05 kind::tf32 accepts both from shared memory
// (instruction-descriptor bits 15/16); MN-major tf32 must use the
// SWIZZLE_128B_BASE32B layout (32-byte swizzle granules, 4-line atoms).
//
// Every producer thread handles fixed tile rows (K-major) or a fixed MN chunk
// (MN-major) for the whole K loop, so per-row / per-column address bases are
// computed once (loader State) and a stage costs a few integer ops per chunk;
// the remaining divisions use multiply-shift FastDiv.
//
// Bias gradients are fused into the weight-gradient GEMMs: the A operand gets
// one extra "ones" row (index `ones_row`), whose output row is sum_k B(n, k) =
// column sums of dy, routed by the epilogue to the bias-gradient buffer.
#pragma once
#include "sg_common.cuh"

namespace sg {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 32;  // fp32 elements = 128 bytes = one swizzle row
constexpr int GEMM_THREADS = 160;

// {1, 0, 0, 0}: source of the ones-row chunk (global memory, cp.async source).
__device__ __align__(16) static const float g_one4[4] = {1.f, 0.f, 0.f, 0.f};

// Unsigned division by a runtime constant via multiply-high (n < 2^31).
struct FastDiv {
  int d;
  uint32_t mul, shr;
  __device__ __forceinline__ int div(int n) const {
    return (int)((__umulhi((uint32_t)n, mul) + (uint32_t)n) >> shr);
  }
};
inline FastDiv make_fastdiv(int d) {
  FastDiv f;
  f.d = d < 1 ? 1 : d;
  if (f.d == 1) {
    f.mul = 0;
    f.shr = 0;
    return f;
  }
  uint32_t l = 0;
  while ((1ull << l) < (unsigned long long)f.d) ++l;
  f.mul = (uint32_t)(((1ull << 32) * ((1ull << l) - (unsigned long long)f.d)) / (unsigned long long)f.d + 1);
  f.shr = l;
  return f;
}

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

// Thread -> chunk mapping of one stage (see load_stage):
//   K-major tile of T rows: thread t covers k-chunk (t & 7) of rows (t >> 3) + 16 i, i < T/16.
//   MN-major tile of T rows: thread t covers row chunk (t % (T/4)) * 4 of k-lines
//   t / (T/4) + (512/T) i, i < T/16.
template <int T>
struct MNMap {
  static constexpr int CPR = T / 4;
  static constexpr int KSTEP = 128 / CPR;
  static __device__ __forceinline__ int mn(int tid) { return (tid % CPR) * 4; }
  static __device__ __forceinline__ int kr(int tid, int i) { return tid / CPR + KSTEP * i; }
};

// ---------------------------------------------------------------- loaders --
// K-major dense operand: op(r, k) = M(r, k).
struct LdDenseK {
  static constexpr int kMN = 0;
  MatView m;
  template <int T>
  struct State {
    const float* base[T / 16];
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
#pragma unroll
    for (int i = 0; i < T / 16; ++i) {
      int r = row0 + (tid >> 3) + 16 * i;
      s.base[i] = r < m.rows ? m.p + (long long)r * m.ld : nullptr;
    }
  }
  template <int T>
  __device__ __forceinline__ const float* src(const State<T>& s, int i, int k, int& nb) const {
    // k is a multiple of 4; column blocks are multiples of 4 wide
    if (!s.base[i] || k >= m.cols) {
      nb = 0;
      return m.p;
    }
    int nv = m.cols - k;
    nb = (nv >= 4 ? 4 : nv) * 4;
    return s.base[i] + m.col_off(k);
  }
};

// MN-major dense operand: op(r, k) = M(k, r) (4 consecutive r contiguous).
// ones_row >= 0 (a multiple of 4): rows ones_row.. read {1, 0, 0, 0}.
struct LdDenseMN {
  static constexpr int kMN = 1;
  MatView m;
  int ones_row;
  template <int T>
  struct State {
    long long coff;
    int nb;  // bytes of this thread's row chunk (0 = outside)
    bool ones;
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    int r = row0 + MNMap<T>::mn(tid);
    s.ones = (r == ones_row);
    s.nb = 0;
    s.coff = 0;
    if (r < m.cols) {
      int nv = m.cols - r;
      s.nb = (nv >= 4 ? 4 : nv) * 4;
      s.coff = m.col_off(r);
    } else if (s.ones) {
      s.nb = 16;
    }
  }
  template <int T>
  __device__ __forceinline__ const float* src(const State<T>& s, int k, int& nb) const {
    if (k >= m.rows || s.nb == 0) {
      nb = 0;
      return m.p;
    }
    nb = s.nb;
    if (s.ones) return g_one4;
    return m.p + (long long)k * m.ld + s.coff;
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
  const float* x;
  ConvGeom g;
  template <int T>
  struct State {
    const float* base[T / 16];  // x at (n, oh*st - p, ow*st - p, 0) (may point outside x)
    int h0[T / 16], w0[T / 16];
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    const int Mtot = g.N * g.Ho * g.Wo;
#pragma unroll
    for (int i = 0; i < T / 16; ++i) {
      int m = row0 + (tid >> 3) + 16 * i;
      if (m < Mtot) {
        int n = g.fHoWo.div(m), rem = m - n * g.Ho * g.Wo;
        int oh = g.fWo.div(rem), ow = rem - oh * g.Wo;
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
  // per-stage tap of this thread's k chunk
  struct Tap {
    int r, s;
    long long off;
    bool ok;
  };
  __device__ __forceinline__ Tap tap(int k) const {
    Tap t;
    t.ok = k < g.R * g.S * g.C;
    int rs = g.fC.div(k), c = k - rs * g.C;
    t.r = g.fS.div(rs);
    t.s = rs - t.r * g.S;
    t.off = ((long long)t.r * g.W + t.s) * g.C + c;
    return t;
  }
  template <int T>
  __device__ __forceinline__ const float* src(const State<T>& s, int i, const Tap& t, int& nb) const {
    int h = s.h0[i] + t.r, w = s.w0[i] + t.s;
    if (t.ok && (unsigned)h < (unsigned)g.H && (unsigned)w < (unsigned)g.W) {
      nb = 16;
      return s.base[i] + t.off;
    }
    nb = 0;
    return x;
  }
};

// Convolution data gradient, A(m, k): m = (n, h, w) over the input,
// k = (r, s, co); value dy[n][(h+p-r)/st][(w+p-s)/st][co] when integral & in range.
struct LdConvDgradA {
  static constexpr int kMN = 0;
  const float* dy;
  ConvGeom g;
  template <int T>
  struct State {
    const float* base[T / 16];  // stride 1: dy at (n, h+p, w+p, 0)
    int hp[T / 16], wp[T / 16], n[T / 16];
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    const int Mtot = g.N * g.H * g.W;
#pragma unroll
    for (int i = 0; i < T / 16; ++i) {
      int m = row0 + (tid >> 3) + 16 * i;
      if (m < Mtot) {
        int n = g.fHW.div(m), rem = m - n * g.H * g.W;
        int h = g.fW.div(rem), w = rem - h * g.W;
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
  struct Tap {
    int r, s, co;
    long long off;
    bool ok;
  };
  __device__ __forceinline__ Tap tap(int k) const {
    Tap t;
    t.ok = k < g.R * g.S * g.Co;
    int rs = g.fCo.div(k);
    t.co = k - rs * g.Co;
    t.r = g.fS.div(rs);
    t.s = rs - t.r * g.S;
    t.off = -((long long)t.r * g.Wo + t.s) * g.Co + t.co;
    return t;
  }
  template <int T>
  __device__ __forceinline__ const float* src(const State<T>& s, int i, const Tap& t, int& nb) const {
    nb = 0;
    if (!t.ok) return dy;
    int oh = s.hp[i] - t.r, ow = s.wp[i] - t.s;
    if (g.st == 1) {
      if ((unsigned)oh < (unsigned)g.Ho && (unsigned)ow < (unsigned)g.Wo) {
        nb = 16;
        return s.base[i] + t.off;
      }
      return dy;
    }
    if (oh < 0 || ow < 0 || oh % g.st || ow % g.st) return dy;
    oh /= g.st;
    ow /= g.st;
    if (oh >= g.Ho || ow >= g.Wo) return dy;
    nb = 16;
    return dy + (((long long)s.n[i] * g.Ho + oh) * g.Wo + ow) * g.Co + t.co;
  }
};

// Convolution data gradient, B(c, k) = W[co][r][s][c] with k = (r, s, co); MN-major (c contiguous).
struct LdConvDgradB {
  static constexpr int kMN = 1;
  const float* Wt;
  ConvGeom g;
  template <int T>
  struct State {
    int c;
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    s.c = row0 + MNMap<T>::mn(tid);
  }
  template <int T>
  __device__ __forceinline__ const float* src(const State<T>& s, int k, int& nb) const {
    nb = 0;
    if (s.c >= g.C || k >= g.R * g.S * g.Co) return Wt;
    int rs = g.fCo.div(k), co = k - rs * g.Co;
    nb = 16;
    return Wt + ((long long)co * g.R * g.S + rs) * g.C + s.c;
  }
};

// Convolution weight gradient, A(kg, m) = x[n][oh*st-p+r][ow*st-p+s][c] with
// kg = (r, s, c) the GEMM row and m = (n, oh, ow) the reduction index; MN-major.
// Row ones_row (= R*S*C) is the ones row of the fused bias gradient.
struct LdConvWgradA {
  static constexpr int kMN = 1;
  const float* x;
  ConvGeom g;
  int ones_row;
  template <int T>
  struct State {
    int r, s;
    long long off;  // (r*W + s)*C + c
    int mode;       // 0 outside, 1 data, 2 ones
  };
  template <int T>
  __device__ __forceinline__ void init(State<T>& s, int row0, int tid) const {
    int kg = row0 + MNMap<T>::mn(tid);
    s.mode = 0;
    s.r = s.s = 0;
    s.off = 0;
    if (kg < g.R * g.S * g.C) {
      int rs = g.fC.div(kg), c = kg - rs * g.C;
      s.r = g.fS.div(rs);
      s.s = rs - s.r * g.S;
      s.off = ((long long)s.r * g.W + s.s) * g.C + c;
      s.mode = 1;
    } else if (kg == ones_row) {
      s.mode = 2;
    }
  }
  template <int T>
  __device__ __forceinline__ const float* src(const State<T>& s, int m, int& nb) const {
    nb = 0;
    if (s.mode == 0 || m >= g.N * g.Ho * g.Wo) return x;
    if (s.mode == 2) {
      nb = 16;
      return g_one4;
    }
    int n = g.fHoWo.div(m), rem = m - n * g.Ho * g.Wo;
    int oh = g.fWo.div(rem), ow = rem - oh * g.Wo;
    int h0 = oh * g.st - g.pad, w0 = ow * g.st - g.pad;
    int h = h0 + s.r, w = w0 + s.s;
    if ((unsigned)h >= (unsigned)g.H || (unsigned)w >= (unsigned)g.W) return x;
    nb = 16;
    return x + (((long long)n * g.H + h0) * g.W + w0) * g.C + s.off;
  }
};

// Loaders whose K-major chunk address depends on a per-stage "tap" (filter offset).
template <class L>
struct requires_tap {
  static constexpr bool value = false;
};
template <>
struct requires_tap<LdConvFwdA> {
  static constexpr bool value = true;
};
template <>
struct requires_tap<LdConvDgradA> {
  static constexpr bool value = true;
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
  int mvalid, xrow;
  float* xout;
  float* ws;
  long long ws_ld, ws_split_stride;
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
  int kb_per_split;  // k-blocks handled by one CTA (blockIdx.z = split)
  EpiArgs epi;
};

// ---------------------------------------------------------------------------
// Producer: one stage of an operand tile (T rows x BK) into shared memory.
template <int T, class LD>
__device__ __forceinline__ void load_stage(const LD& ld, const typename LD::template State<T>& st, uint32_t sm,
                                           int k0, int tid) {
  if constexpr (LD::kMN == 0) {
    // K-major SWIZZLE_128B: row r at (r >> 3) * 1024 + (r & 7) * 128, chunk c at c ^ (r & 7).
    const int kc = tid & 7, r7 = (tid >> 3) & 7;
    const uint32_t d0 = sm + ((tid >> 6) << 10) + (r7 << 7) + ((kc ^ r7) << 4);
    const int k = k0 + kc * 4;
    if constexpr (requires_tap<LD>::value) {
      const auto t = ld.tap(k);
#pragma unroll
      for (int i = 0; i < T / 16; ++i) {
        int nb;
        const float* g = ld.src(st, i, t, nb);
        cp_async16(d0 + i * 2048, g, nb);
      }
    } else {
#pragma unroll
      for (int i = 0; i < T / 16; ++i) {
        int nb;
        const float* g = ld.template src<T>(st, i, k, nb);
        cp_async16(d0 + i * 2048, g, nb);
      }
    }
  } else {
    // MN-major SWIZZLE_128B_BASE32B: k-line kr of MN-atom a at a*(BK*128) + kr*128;
    // within the line the 32-byte granule g sits at g ^ (kr & 3).  LBO = BK*128, SBO = 512.
    const int mn = MNMap<T>::mn(tid);
    const uint32_t dmn = sm + (mn >> 5) * (GEMM_BK * 128) + ((mn & 4) << 2);
    const int g32 = (mn & 31) >> 3;
#pragma unroll
    for (int i = 0; i < T / 16; ++i) {
      const int kr = MNMap<T>::kr(tid, i);
      int nb;
      const float* g = ld.template src<T>(st, k0 + kr, nb);
      cp_async16(dmn + kr * 128 + ((g32 ^ (kr & 3)) << 5), g, nb);
    }
  }
}

template <int T, int MN>
__device__ __forceinline__ uint64_t tile_desc(uint32_t sm, int kk) {
  if constexpr (MN == 0) {
    return umma_desc_sw128(sm + kk * 32, 16, 1024);
  } else {
    return umma_desc_mn_sw128_32b(sm + kk * 8 * 128, GEMM_BK * 128, 512);
  }
}

template <int BN, int STAGES>
constexpr int gemm_smem_bytes() {
  return STAGES * (GEMM_BM * GEMM_BK * 4 + BN * GEMM_BK * 4) + 1024 /*align*/ + 256 /*barriers*/;
}

template <int BN, int STAGES, class LA, class LB>
__global__ void __launch_bounds__(GEMM_THREADS, 1) gemm_tc_kernel(const __grid_constant__ GemmArgs<LA, LB> args) {
  constexpr int A_BYTES = GEMM_BM * GEMM_BK * 4;
  constexpr int B_BYTES = BN * GEMM_BK * 4;
  constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
  constexpr int LAG = STAGES > 2 ? STAGES - 2 : 1;
  static_assert(BN % 32 == 0 && BN <= 256, "BN");

  extern __shared__ uint8_t smem_raw[];
  const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bar_base = sbase + STAGES * STAGE_BYTES;
  // full[s] at bar_base + 8s, empty[s] at +8(STAGES+s), accum at +16 STAGES, tmem slot after.
  const uint32_t accum_bar = bar_base + 16 * STAGES;
  const uint32_t tmem_slot = accum_bar + 8;
  uint32_t* tmem_slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (tmem_slot - smem_u32(smem_raw)));

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int m0 = blockIdx.x * GEMM_BM;
  const int n0 = blockIdx.y * BN;
  const int nkb_total = (args.K + GEMM_BK - 1) / GEMM_BK;
  const int kb_begin = blockIdx.z * args.kb_per_split;
  int kb_end = kb_begin + args.kb_per_split;
  if (kb_end > nkb_total) kb_end = nkb_total;
  const int nkb = kb_end - kb_begin;

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(bar_base + 8 * s, 128);                // one arrive per producer thread
      mbar_init(bar_base + 8 * (STAGES + s), 1);       // tcgen05.commit
    }
    mbar_init(accum_bar, 1);
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc<TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot_ptr;

  if (warp < 4) {
    // ------------------------------ producers ------------------------------
    typename LA::template State<GEMM_BM> sa_st;
    typename LB::template State<BN> sb_st;
    args.a.template init<GEMM_BM>(sa_st, m0, tid);
    args.b.template init<BN>(sb_st, n0, tid);
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const int round = it / STAGES;
      if (round > 0) mbar_wait(bar_base + 8 * (STAGES + s), (round - 1) & 1);
      const uint32_t sa = sbase + s * STAGE_BYTES;
      const int k0 = (kb_begin + it) * GEMM_BK;
      load_stage<GEMM_BM>(args.a, sa_st, sa, k0, tid);
      load_stage<BN>(args.b, sb_st, sa + A_BYTES, k0, tid);
      cp_async_commit();
      if (it >= LAG) {
        // this thread's copies for k-block it-LAG have landed: make them visible
        // to the tensor-core (async) proxy, then release the stage.
        cp_async_wait<LAG>();
        fence_proxy_async_smem();
        mbar_arrive(bar_base + 8 * ((it - LAG) % STAGES));
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int j = (nkb > LAG ? nkb - LAG : 0); j < nkb; ++j) mbar_arrive(bar_base + 8 * (j % STAGES));
  } else if (tid == 128) {
    // ------------------------------ MMA issuer -----------------------------
    constexpr uint32_t idesc = idesc_tf32(GEMM_BM, BN, LA::kMN, LB::kMN);
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      mbar_wait(bar_base + 8 * s, (it / STAGES) & 1);
      tc_fence_after();
      const uint32_t sa = sbase + s * STAGE_BYTES;
#pragma unroll
      for (int kk = 0; kk < GEMM_BK / 8; ++kk) {
        uint64_t ad = tile_desc<GEMM_BM, LA::kMN>(sa, kk);
        uint64_t bd = tile_desc<BN, LB::kMN>(sa + A_BYTES, kk);
        mma_tf32(tmem, ad, bd, idesc, (it | kk) ? 1u : 0u);
      }
      mma_commit(bar_base + 8 * (STAGES + s));
    }
    mma_commit(accum_bar);
  }

  // -------------------------------- epilogue --------------------------------
  if (warp < 4) {
    if (nkb > 0) mbar_wait(accum_bar, 0);
    tc_fence_after();
    const int row = m0 + warp * 32 + (tid & 31);
    const EpiArgs& e = args.epi;
    const uint32_t tbase = tmem + ((uint32_t)(warp * 32) << 16);
    const bool plain_vec = !e.trans && e.cb >= args.N && (e.ld & 3) == 0 && !e.bias_on_m;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      if (n0 + c0 >= args.N) break;
      float v[16];
      if (nkb > 0) {
        tmem_ld16(tbase + c0, v);
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0.f;
      }
      if (row >= args.M) continue;
      if (e.ws) {
        float* dst = e.ws + blockIdx.z * e.ws_split_stride + (long long)row * e.ws_ld + n0 + c0;
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
      if (row >= e.mvalid) {
        if (row == e.xrow) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (n0 + c0 + i < args.N) e.xout[n0 + c0 + i] = v[i];
        }
        continue;
      }
      if (plain_vec && n0 + c0 + 15 < args.N) {
        float* dst = e.p + (long long)row * e.ld + n0 + c0;
#pragma unroll
        for (int i = 0; i < 16; i += 4) {
          float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          if (e.bias) {
            o.x += e.bias[n0 + c0 + i];
            o.y += e.bias[n0 + c0 + i + 1];
            o.z += e.bias[n0 + c0 + i + 2];
            o.w += e.bias[n0 + c0 + i + 3];
          }
          if (e.relu) {
            o.x = fmaxf(o.x, 0.f);
            o.y = fmaxf(o.y, 0.f);
            o.z = fmaxf(o.z, 0.f);
            o.w = fmaxf(o.w, 0.f);
          }
          *reinterpret_cast<float4*>(dst + i) = o;
        }
        continue;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int col = n0 + c0 + i;
        if (col >= args.N) break;
        float o = v[i];
        if (e.bias) o += e.bias_on_m ? e.bias[row] : e.bias[col];
        if (e.relu) o = fmaxf(o, 0.f);
        if (e.trans)
          *out_at(e, col, row, e.mvalid) = o;
        else
          *out_at(e, row, col, args.N) = o;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<TMEM_COLS>(tmem);
  }
}

}  // namespace sg
