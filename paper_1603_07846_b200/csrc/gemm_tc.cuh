// tcgen05 (kind::tf32) implicit-GEMM engine shared by the convolution and
// inner-product layers ("rotates (multiply W)"
// convolution).
//
//   D[m][n] = sum_k A(m, k) * B(n, k)      fp32 storage, TF32 operands, fp32 accumulate
//
// One CTA computes a 128 x BN output tile (optionally one K-split of it):
//   warps 0-3 : producers — gather 16-byte chunks with cp.async (zero-filled
//               outside the operand) straight into the UMMA SWIZZLE_128B
//               canonical layout, one stage of BK = 32 fp32 (128 B) per step;
//               then the epilogue (TMEM -> registers -> global).
//   warp 4    : TMEM allocation and the single MMA-issuing thread.
// Operands are "loaders": each maps a (row, k) of the GEMM onto the layer's
// native tensor (NHWC activations, KRSC / [d_v][d_h] weights), so the im2col
// of the convolution is never materialised.  A loader is K-major (4
// consecutive k contiguous in memory) or MN-major (4 consecutive rows
// contiguous); tcgen05 kind::tf32 accepts both from shared memory
// (instruction-descriptor bits 15/16); MN-major tf32 must use the
// SWIZZLE_128B_BASE32B layout (32-byte swizzle granules, 4-line atoms).
#pragma once
#include "sg_common.cuh"

namespace sg {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 32;  // fp32 elements = 128 bytes = one swizzle row
constexpr int GEMM_THREADS = 160;

// ---------------------------------------------------------------------------
// Blocked row-major matrix view: element (i, j) at p[(j / cb) * bs + i * ld + j % cb].
// cb >= cols means a plain row-major matrix.  Column blocking is how a tensor
// gathered along the feature dimension by NCCL is laid out ([K][rows][cols/K]).
struct MatView {
  const float* p;
  long long ld, bs;
  int cb, rows, cols;
  __device__ __forceinline__ const float* at(int i, int j) const {
    if (cb >= cols) return p + (long long)i * ld + j;
    int blk = j / cb;
    return p + (long long)blk * bs + (long long)i * ld + (j - blk * cb);
  }
};

// K-major dense operand: op(r, k) = M(r, k).
struct LdDenseK {
  static constexpr int kMN = 0;
  MatView m;
  __device__ __forceinline__ const float* src(int r, int k, int& nbytes) const {
    if (r < m.rows && k < m.cols) {
      int nv = m.cols - k;
      nbytes = (nv >= 4 ? 4 : nv) * 4;
      return m.at(r, k);
    }
    nbytes = 0;
    return m.p;
  }
};

// MN-major dense operand: op(r, k) = M(k, r)  (4 consecutive r contiguous).
struct LdDenseMN {
  static constexpr int kMN = 1;
  MatView m;
  __device__ __forceinline__ const float* src(int r, int k, int& nbytes) const {
    if (k < m.rows && r < m.cols) {
      int nv = m.cols - r;
      nbytes = (nv >= 4 ? 4 : nv) * 4;
      return m.at(k, r);
    }
    nbytes = 0;
    return m.p;
  }
};

struct ConvGeom {
  int N, H, W, C;       // input (C multiple of 4)
  int Co, R, S;         // filter
  int Ho, Wo, st, pad;  // output
};

// Convolution forward, A(m, k): m = (n, oh, ow), k = (r, s, c) ; x NHWC.
struct LdConvFwdA {
  static constexpr int kMN = 0;
  const float* x;
  ConvGeom g;
  __device__ __forceinline__ const float* src(int m, int k, int& nbytes) const {
    nbytes = 0;
    int HoWo = g.Ho * g.Wo;
    if (m >= g.N * HoWo || k >= g.R * g.S * g.C) return x;
    int n = m / HoWo, rem = m - n * HoWo;
    int oh = rem / g.Wo, ow = rem - oh * g.Wo;
    int rs = k / g.C, c = k - rs * g.C;
    int r = rs / g.S, s = rs - r * g.S;
    int h = oh * g.st - g.pad + r, w = ow * g.st - g.pad + s;
    if ((unsigned)h >= (unsigned)g.H || (unsigned)w >= (unsigned)g.W) return x;
    nbytes = 16;
    return x + (((long long)n * g.H + h) * g.W + w) * g.C + c;
  }
};

// Convolution data gradient, A(m, k): m = (n, h, w) over the input,
// k = (r, s, co);  value dy[n][(h+p-r)/st][(w+p-s)/st][co] when integral & in range.
struct LdConvDgradA {
  static constexpr int kMN = 0;
  const float* dy;
  ConvGeom g;
  __device__ __forceinline__ const float* src(int m, int k, int& nbytes) const {
    nbytes = 0;
    int HW = g.H * g.W;
    if (m >= g.N * HW || k >= g.R * g.S * g.Co) return dy;
    int n = m / HW, rem = m - n * HW;
    int h = rem / g.W, w = rem - h * g.W;
    int rs = k / g.Co, co = k - rs * g.Co;
    int r = rs / g.S, s = rs - r * g.S;
    int oh = h + g.pad - r, ow = w + g.pad - s;
    if (oh < 0 || ow < 0) return dy;
    if (g.st > 1) {
      if (oh % g.st || ow % g.st) return dy;
      oh /= g.st;
      ow /= g.st;
    }
    if (oh >= g.Ho || ow >= g.Wo) return dy;
    nbytes = 16;
    return dy + (((long long)n * g.Ho + oh) * g.Wo + ow) * g.Co + co;
  }
};

// Convolution data gradient, B(c, k) = W[co][r][s][c] with k = (r, s, co); MN-major (c contiguous).
struct LdConvDgradB {
  static constexpr int kMN = 1;
  const float* Wt;
  ConvGeom g;
  __device__ __forceinline__ const float* src(int c, int k, int& nbytes) const {
    nbytes = 0;
    if (c >= g.C || k >= g.R * g.S * g.Co) return Wt;
    int rs = k / g.Co, co = k - rs * g.Co;
    nbytes = 16;
    return Wt + ((long long)co * g.R * g.S + rs) * g.C + c;
  }
};

// Convolution weight gradient, A(kg, m) = x[n][oh*st-p+r][ow*st-p+s][c] with
// kg = (r, s, c) the GEMM row and m = (n, oh, ow) the reduction index; MN-major.
struct LdConvWgradA {
  static constexpr int kMN = 1;
  const float* x;
  ConvGeom g;
  __device__ __forceinline__ const float* src(int kg, int m, int& nbytes) const {
    nbytes = 0;
    int HoWo = g.Ho * g.Wo;
    if (kg >= g.R * g.S * g.C || m >= g.N * HoWo) return x;
    int n = m / HoWo, rem = m - n * HoWo;
    int oh = rem / g.Wo, ow = rem - oh * g.Wo;
    int rs = kg / g.C, c = kg - rs * g.C;
    int r = rs / g.S, s = rs - r * g.S;
    int h = oh * g.st - g.pad + r, w = ow * g.st - g.pad + s;
    if ((unsigned)h >= (unsigned)g.H || (unsigned)w >= (unsigned)g.W) return x;
    nbytes = 16;
    return x + (((long long)n * g.H + h) * g.W + w) * g.C + c;
  }
};

// ---------------------------------------------------------------------------
// Epilogue parameters.  Output element (m, n) goes to out(m, n) (trans = 0) or
// out(n, m) (trans = 1) of a blocked row-major view; with ws != nullptr the
// CTA writes its raw K-split partial to ws[split][m][n] (ld = ws_ld) instead.
struct EpiArgs {
  float* p;
  long long ld, bs;
  int cb, trans;
  const float* bias;  // indexed by n (bias_on_m = 0) or by m
  int bias_on_m;
  int relu;
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
// Producer: write one operand tile (T rows x BK) of one stage.
template <int T, class LD>
__device__ __forceinline__ void load_tile(const LD& ld, uint32_t sm, int row0, int k0, int tid) {
  if constexpr (LD::kMN == 0) {
    // K-major: row r at r*128 B (8-row groups of 1024 B), 16-byte chunk c stored at c ^ (r & 7).
#pragma unroll
    for (int i = 0; i < T / 16; ++i) {
      int q = tid + 128 * i;
      int r = q >> 3, kc = q & 7;
      int nb;
      const float* g = ld.src(row0 + r, k0 + kc * 4, nb);
      cp_async16(sm + (r >> 3) * 1024 + (r & 7) * 128 + ((kc ^ (r & 7)) << 4), g, nb);
    }
  } else {
    // MN-major (tf32 requires SWIZZLE_128B_BASE32B): 32 consecutive rows (128 B) per
    // k-line; k-line kr of MN-atom a at a*(BK*128) + kr*128; within the line the
    // 32-byte granule g sits at g ^ (kr & 3).  LBO = BK*128 (atom stride), SBO = 512
    // (4 k-lines).
    constexpr int CPR = T / 4;
#pragma unroll
    for (int i = 0; i < T / 16; ++i) {
      int q = tid + 128 * i;
      int kr = q / CPR, mn = (q % CPR) * 4;
      int nb;
      const float* g = ld.src(row0 + mn, k0 + kr, nb);
      cp_async16(sm + (mn >> 5) * (GEMM_BK * 128) + kr * 128 + ((((mn & 31) >> 3) ^ (kr & 3)) << 5) + ((mn & 4) << 2),
                 g, nb);
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
    for (int it = 0; it < nkb; ++it) {
      const int s = it % STAGES;
      const int round = it / STAGES;
      if (round > 0) mbar_wait(bar_base + 8 * (STAGES + s), (round - 1) & 1);
      const uint32_t sa = sbase + s * STAGE_BYTES;
      const int k0 = (kb_begin + it) * GEMM_BK;
      load_tile<GEMM_BM>(args.a, sa, m0, k0, tid);
      load_tile<BN>(args.b, sa + A_BYTES, n0, k0, tid);
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
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int col = n0 + c0 + i;
        if (col >= args.N) break;
        float o = v[i];
        if (e.bias) o += e.bias_on_m ? e.bias[row] : e.bias[col];
        if (e.relu) o = fmaxf(o, 0.f);
        if (e.trans)
          *out_at(e, col, row, args.M) = o;
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
