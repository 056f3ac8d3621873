// Launchers for the tcgen05 implicit-GEMM engine: convolution forward / data
// gradient / weight gradient (+ fused bias gradient) and inner-product forward /
// data gradient / weight gradient (§4.1.2, §5.4.1; SURVEY
// §8(a) a3, a8, a10, a15), deterministic split-K reduction and column sums.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "gemm_tc.cuh"
#include "ops.h"

namespace sg {

long long g_kernel_launches = 0;

// cp.async producers release a stage with cp.async.mbarrier.arrive (default) or
// with the older wait_group-LAG scheme (SG_ASYNC_ARRIVE=0, for A/B).
bool async_arrive() {
  static int on = -1;
  if (on < 0) {
    const char* env = getenv("SG_ASYNC_ARRIVE");
    on = env ? atoi(env) != 0 : 1;
  }
  return on != 0;
}


bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* env = getenv("SG_PDL");
    on = env ? atoi(env) != 0 : 1;
  }
  return on != 0;
}


namespace {

constexpr int kNumSMs = 148;
constexpr int kMinKbPerSplit = 8;
constexpr int kSplitCounters = 512;  // ints at the head of the workspace: 2 x 256 tile counters

// Split-K reduction by a separate fixed-order kernel (default) or inside the GEMM
// by the splits themselves (SG_SPLITK_FIXUP=1: every split of a tile is a
// resident CTA and reduces a row slice once the tile counter is full).  The
// in-GEMM variant measured slower on every config (CIFAR-10 467K -> 424K img/s,
// MLP ip1 forward 16 -> 29 us): the cross-CTA wait costs more than the launch.
bool splitk_fixup() {
  static int on = -1;
  if (on < 0) {
    const char* env = getenv("SG_SPLITK_FIXUP");
    on = env ? atoi(env) != 0 : 0;
  }
  return on != 0;
}

struct Plan {
  int bn, mt, nt, splits, kb_per_split;
  int mt2 = 0;  // 256-row work items (mt counts 128-row tiles; see tile256())
};

inline long long pad4(int n) { return (n + 3) & ~3; }

Plan plan_gemm(int M, int N, int K, size_t ws_floats_avail, bool wide192 = true) {
  Plan p;
  static const int big_bn = getenv("SG_BN_BIG") ? atoi(getenv("SG_BN_BIG")) : 1;
  static const int bn192 = getenv("SG_BN192") ? atoi(getenv("SG_BN192")) : 1;
  p.bn = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  // N a multiple of 192 (AlexNet conv2 192, conv3 384 channels): 192-wide tiles
  // waste no accumulator columns (256-wide: 75% used); not for the TMA weight
  // gradient, whose long-K split plan measured slower with them (AlexNet conv2 325 -> 343 us)
  if (bn192 && wide192 && N > 128 && N % 192 == 0) p.bn = 192;
  p.mt = (M + GEMM_BM - 1) / GEMM_BM;
  const int nkb0 = (K + GEMM_BK - 1) / GEMM_BK;
  // wide tiles halve the operand bytes per MMA; keep them when split-K can fill the machine
  const bool can_split = nkb0 >= 2 * kMinKbPerSplit * ((kNumSMs + p.mt - 1) / p.mt);
  if (p.bn >= 192 && p.mt * ((N + p.bn - 1) / p.bn) < kNumSMs && !(big_bn && can_split)) p.bn = 128;
  p.nt = (N + p.bn - 1) / p.bn;
  const int nkb = (K + GEMM_BK - 1) / GEMM_BK;
  const int tiles = p.mt * p.nt;
  int splits = 1;
  if (tiles < kNumSMs && nkb >= 2 * kMinKbPerSplit) {
    // persistent grid of kNumSMs CTAs: tiles x splits must not spill into a second round
    splits = std::min(kNumSMs / tiles, nkb / kMinKbPerSplit);
    while (splits > 1 && (size_t)splits * M * pad4(N) > ws_floats_avail) --splits;
    if (splits < 1) splits = 1;
  }
  p.kb_per_split = (nkb + splits - 1) / splits;
  if (p.kb_per_split < 1) p.kb_per_split = 1;
  p.splits = (nkb + p.kb_per_split - 1) / p.kb_per_split;
  if (p.splits < 1) p.splits = 1;
  return p;
}

// Fixed-order split-K reduction.  A block of G warps owns 128 consecutive
// entries of the padded workspace row space (m * pad4(N) + n, one float4 per
// lane); warp g sums the splits g, g+G, g+2G, ... in ascending order, then warp 0
// adds the G partial sums in ascending g.  G = min(32, splits) depends on the
// shape only, so the result is deterministic.
__device__ __forceinline__ void reduce_store(const EpiArgs& e, int m, int n, int N, float t) {
  if (m >= e.mvalid) {
    if (m == e.xrow) e.xout[n] = t;
    return;
  }
  if (e.bias) t += e.bias_on_m ? e.bias[m] : e.bias[n];
  if (e.relu) t = fmaxf(t, 0.f);
  if (e.rn) t = tf32_rna(t);
  if (e.trans)
    *out_at(e, n, m, e.mvalid) = t;
  else
    *out_at(e, m, n, N) = t;
}

__global__ void __launch_bounds__(1024) splitk_reduce_kernel(const float* __restrict__ ws, int splits,
                                                            long long split_stride, int M, int N, EpiArgs e) {
  pdl_entry();
  __shared__ float4 part[32][32];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5, G = blockDim.x >> 5;
  const int ldw = (N + 3) & ~3;
  const long long q = ((long long)blockIdx.x * 32 + lane) * 4;  // first padded entry of this lane
  const bool in = q < (long long)M * ldw;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (in) {
    const float* p = ws + q;
#pragma unroll 4
    for (int s = g; s < splits; s += G) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p + s * split_stride));
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
  }
  if (G > 1) {
    part[g][lane] = acc;
    __syncthreads();
    if (g != 0) return;
    acc = part[0][lane];
    for (int j = 1; j < G; ++j) {
      const float4 v = part[j][lane];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
  }
  if (!in) return;
  const int m = (int)(q / ldw), n = (int)(q - (long long)m * ldw);
  const float r[4] = {acc.x, acc.y, acc.z, acc.w};
  if (!e.trans && e.cb >= N && !e.bias_on_m && m < e.mvalid && n + 3 < N && (e.ld & 3) == 0) {
    float4 o = acc;
    if (e.bias) {
      o.x += e.bias[n];
      o.y += e.bias[n + 1];
      o.z += e.bias[n + 2];
      o.w += e.bias[n + 3];
    }
    if (e.relu) {
      o.x = fmaxf(o.x, 0.f);
      o.y = fmaxf(o.y, 0.f);
      o.z = fmaxf(o.z, 0.f);
      o.w = fmaxf(o.w, 0.f);
    }
    *reinterpret_cast<float4*>(e.p + (long long)m * e.ld + n) = tf32_rna4_if(o, e.rn);
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (n + i < N) reduce_store(e, m, n + i, N, r[i]);
}

template <int BN, class LA, class LB, int MT = 1>
cudaError_t launch_bn(const GemmArgs<LA, LB>& args, const Plan& p, cudaStream_t st) {
  constexpr int STAGES = gemm_stages<BN, ScratchOf<LA>::value, MT>();
  constexpr int SMEM = gemm_smem_bytes<BN, STAGES, ScratchOf<LA>::value, MT>();
  auto kern = gemm_tc_kernel<BN, STAGES, LA, LB, MT>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int nwork = (MT == 1 ? p.mt : (p.mt + 1) / 2) * p.nt * p.splits;
  return launch_k(kern, std::min(nwork, kNumSMs), GEMM_ALL_THREADS, SMEM, st, args);
}

// 256-row work items (two accumulators sharing each B stage) for narrow N:
// TMA A operands whose box can be encoded 256 rows tall (TmaIm2col), no split-K,
// and at least one full wave of 256-row items.
inline bool tile256(const Plan& p) {
  static const int on = getenv("SG_TILE256") ? atoi(getenv("SG_TILE256")) : 1;
  return on && p.bn <= 64 && p.splits == 1 && ((p.mt + 1) / 2) * p.nt >= kNumSMs;
}

template <class LA, class LB>
cudaError_t run_gemm_planned(const LA& a, const LB& b, const Plan& p, int M, int N, int K, EpiArgs epi, Workspace ws,
                             cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  GemmArgs<LA, LB> args{a, b, M, N, K, p.kb_per_split, epi, async_arrive() ? 1 : 0};
  // workspace: kSplitCounters tile counters (kept zero between GEMMs), then the
  // split partials [split][M][pad4(N)]
  float* part = ws.ptr + kSplitCounters;
  // cooperative reduction needs one resident CTA per work item
  const bool fixup = splitk_fixup() && p.mt * p.nt * p.splits <= kNumSMs && p.mt * p.nt <= kSplitDone;
  args.epi.cnt = nullptr;
  if (p.splits > 1) {
    args.epi.ws = part;
    args.epi.ws_ld = pad4(N);
    args.epi.ws_split_stride = (long long)M * pad4(N);
    if (fixup) args.epi.cnt = reinterpret_cast<int*>(ws.ptr);
  } else {
    args.epi.ws = nullptr;
  }
  cudaError_t e;
  if constexpr (LA::kTMA && ScratchOf<LA>::value == 0) {
    if (p.mt2) {
      switch (p.bn) {
        case 32: return launch_bn<32, LA, LB, 2>(args, p, st);
        case 64: return launch_bn<64, LA, LB, 2>(args, p, st);
        default: return cudaErrorInvalidValue;
      }
    }
  }
  if (p.mt2) return cudaErrorInvalidValue;
  switch (p.bn) {
    case 32: e = launch_bn<32>(args, p, st); break;
    case 64: e = launch_bn<64>(args, p, st); break;
    case 128: e = launch_bn<128>(args, p, st); break;
    case 192: e = launch_bn<192>(args, p, st); break;
    default: e = launch_bn<256>(args, p, st); break;
  }
  if (e != cudaSuccess || p.splits == 1 || fixup) return e;
  const long long total4 = (long long)M * pad4(N) / 4;
  const int G = std::min(32, p.splits);  // 32 measured ~1% faster than 16 on CIFAR-10 (148-split conv1 wgrad)
  return launch_k(splitk_reduce_kernel, (unsigned)((total4 + 31) / 32), 32 * G, 0, st, (const float*)part, p.splits,
                  (long long)M * pad4(N), M, N, epi);
}

template <class LA, class LB>
cudaError_t run_gemm(const LA& a, const LB& b, int M, int N, int K, EpiArgs epi, Workspace ws, cudaStream_t st) {
  // 192-wide tiles only for TMA operands (the cp.async loaders' thread maps assume power-of-two widths)
  return run_gemm_planned(a, b, plan_gemm(M, N, K, ws.floats, LA::kTMA), M, N, K, epi, ws, st);
}

// TMA operands: the tensor maps' boxes depend on the tile chosen by the plan.
template <class MA, class MB>
cudaError_t run_gemm_mk(MA mkA, MB mkB, int M, int N, int K, EpiArgs epi, Workspace ws, cudaStream_t st) {
  const Plan p = plan_gemm(M, N, K, ws.floats);
  return run_gemm_planned(mkA(GEMM_BM), mkB(p.bn), p, M, N, K, epi, ws, st);
}

// ------------------------------------------------------- tensor-map encode --
PFN_cuTensorMapEncodeTiled_v12000 g_enc_tiled = nullptr;
PFN_cuTensorMapEncodeIm2col_v12000 g_enc_im2col = nullptr;

// TMA operand paths per operation (default all; an operation falls back to the
// cp.async gather when its shapes do not fit TMA, e.g. 4-channel first layers;
// SG_TMA_OPS overrides for A/B measurements):
// bit 0 conv fwd, 1 conv dgrad, 2 conv wgrad, 3 inner product, 4 plain GEMM.
int tma_ops() {
  static int ops = -1;
  if (ops < 0) {
    const char* env = getenv("SG_TMA_OPS");
    ops = env ? atoi(env) : 0x1f;
  }
  return ops;
}
bool tma_on_impl();
bool tma_on(int op_bit) { return (tma_ops() >> op_bit & 1) && tma_on_impl(); }

bool tma_on_impl() {
  static int state = -1;
  if (state < 0) {
    const char* env = getenv("SG_TMA");
    state = 0;
    if (!(env && env[0] == '0')) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&g_enc_tiled, cudaEnableDefault, &q) ==
              cudaSuccess &&
          cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", (void**)&g_enc_im2col, cudaEnableDefault, &q) ==
              cudaSuccess &&
          g_enc_tiled && g_enc_im2col)
        state = 1;
    }
  }
  return state == 1;
}

bool aligned16p(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// rank-2/3 tiled fp32 map; dims innermost first, strides in bytes for dims 1..
CUtensorMap enc_tiled(const void* p, int rank, const cuuint64_t* dims, const cuuint64_t* strides_b,
                      const cuuint32_t* box, CUtensorMapSwizzle sw, bool* ok) {
  CUtensorMap m;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};  // element strides, one per dimension (rank <= 5)
  CUresult r = g_enc_tiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(p), dims, strides_b, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  *ok = *ok && r == CUDA_SUCCESS;
  return m;
}

CUtensorMap enc_im2col(const void* x, int N, int H, int W, int C, int lo_w, int lo_h, int up_w, int up_h,
                       int channels, int pixels, int st, CUtensorMapSwizzle sw, bool* ok) {
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
  int lower[2] = {lo_w, lo_h}, upper[2] = {up_w, up_h};
  cuuint32_t es[4] = {1, (cuuint32_t)st, (cuuint32_t)st, 1};
  CUresult r = g_enc_im2col(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(x), dims, strides, lower, upper,
                            channels, pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  // driver <= 13.1 quirk for small tensors (as in CUTLASS's im2col descriptor builder)
  if ((size_t)N * H * W * C * 4 < 131072) reinterpret_cast<uint64_t*>(&m)[1] &= ~(1llu << 21);
  *ok = *ok && r == CUDA_SUCCESS && lo_w >= -128 && lo_w <= 127 && lo_h >= -128 && lo_h <= 127 && up_w >= -128 &&
        up_w <= 127 && up_h >= -128 && up_h <= 127;
  return m;
}

// K-major tile of a row-major [rows][cols] matrix (ld elements), optionally column-blocked.
TmaK tma_k(const View2D& v, int box_rows, bool* ok) {
  TmaK t{};
  const bool blocked = v.cb > 0 && v.cb < v.cols;
  t.blocked = blocked;
  t.cb = blocked ? v.cb : v.cols;
  if (blocked) {
    *ok = *ok && v.cb % 32 == 0 && (v.bs * 4) % 16 == 0;
    cuuint64_t dims[3] = {(cuuint64_t)v.cb, (cuuint64_t)v.rows, (cuuint64_t)((v.cols + v.cb - 1) / v.cb)};
    cuuint64_t strides[2] = {(cuuint64_t)v.ld * 4, (cuuint64_t)v.bs * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
    t.map = enc_tiled(v.p, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, ok);
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)v.cols, (cuuint64_t)v.rows};
    cuuint64_t strides[1] = {(cuuint64_t)v.ld * 4};
    cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
    t.map = enc_tiled(v.p, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B, ok);
  }
  *ok = *ok && aligned16p(v.p) && (v.ld * 4) % 16 == 0 && box_rows <= 256;
  return t;
}

// MN-major tile of M(k, mn) = v(row = k, col = mn); valid / ones_row as TmaMN.
// A plain matrix with 32 | cols and no constant atoms is loaded as ONE box per
// stage through the 3-D view {32, rows, cols/32} (atom stride 128 B).
TmaMN tma_mn(const View2D& v, int valid, int ones_row, int box_rows, bool* ok) {
  TmaMN t{};
  const bool blocked = v.cb > 0 && v.cb < v.cols;
  t.blocked = blocked;
  t.cb = blocked ? v.cb : v.cols;
  t.valid = valid;
  t.ones_row = ones_row;
  t.atoms = !blocked && ones_row < 0 && v.cols % 32 == 0 && valid == v.cols;
  if (t.atoms) {
    cuuint64_t dims[3] = {32, (cuuint64_t)v.rows, (cuuint64_t)(v.cols / 32)};
    cuuint64_t strides[2] = {(cuuint64_t)v.ld * 4, 128};
    cuuint32_t box[3] = {32, 32, (cuuint32_t)(box_rows / 32)};
    t.map = enc_tiled(v.p, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, ok);
  } else if (blocked) {
    *ok = *ok && v.cb % 32 == 0 && (v.bs * 4) % 16 == 0;
    cuuint64_t dims[3] = {(cuuint64_t)v.cb, (cuuint64_t)v.rows, (cuuint64_t)((v.cols + v.cb - 1) / v.cb)};
    cuuint64_t strides[2] = {(cuuint64_t)v.ld * 4, (cuuint64_t)v.bs * 4};
    cuuint32_t box[3] = {32, 32, 1};
    t.map = enc_tiled(v.p, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, ok);
  } else {
    cuuint64_t dims[2] = {(cuuint64_t)v.cols, (cuuint64_t)v.rows};
    cuuint64_t strides[1] = {(cuuint64_t)v.ld * 4};
    cuuint32_t box[2] = {32, 32};
    t.map = enc_tiled(v.p, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, ok);
  }
  *ok = *ok && aligned16p(v.p) && (v.ld * 4) % 16 == 0;
  return t;
}

View2D vplain(const float* p, int rows, int cols, long long ld) {
  return View2D{const_cast<float*>(p), ld, 0, cols, rows, cols};
}

MatView mv(const float* p, int rows, int cols, long long ld, long long bs = 0, int cb = 0) {
  MatView v;
  v.p = p;
  v.rows = rows;
  v.cols = cols;
  v.ld = ld;
  v.bs = bs;
  v.cb = cb > 0 ? cb : cols;
  v.fcb = make_fastdiv(v.cb);
  return v;
}
MatView mv(const View2D& d) { return mv(d.p, d.rows, d.cols, d.ld, d.bs, d.cb); }

// `flags`: EPI_RELU | EPI_RN (ops.h).
EpiArgs epi_plain(float* p, long long ld, int trans, const float* bias, int bias_on_m, int flags, int mvalid) {
  EpiArgs e{};
  e.p = p;
  e.ld = ld;
  e.bs = 0;
  e.cb = 1 << 30;
  e.trans = trans;
  e.bias = bias;
  e.bias_on_m = bias_on_m;
  e.relu = (flags & EPI_RELU) ? 1 : 0;
  e.rn = (flags & EPI_RN) ? 1 : 0;
  e.mvalid = mvalid;
  e.xrow = -1;
  e.xout = nullptr;
  return e;
}
EpiArgs epi_view(const View2D& d, const float* bias, int flags) {
  EpiArgs e = epi_plain(d.p, d.ld, 0, bias, 0, flags, d.rows);
  e.bs = d.bs;
  e.cb = d.cb > 0 ? d.cb : d.cols;
  if (e.cb >= d.cols) e.cb = 1 << 30;
  return e;
}

ConvGeom geom(const ConvShape& s) {
  ConvGeom g;
  g.N = s.N;
  g.H = s.H;
  g.W = s.W;
  g.C = s.C;
  g.Co = s.Co;
  g.R = s.R;
  g.S = s.S;
  g.Ho = s.Ho;
  g.Wo = s.Wo;
  g.st = s.st;
  g.pad = s.pad;
  g.fC = make_fastdiv(s.C);
  g.fS = make_fastdiv(s.S);
  g.fCo = make_fastdiv(s.Co);
  g.fHoWo = make_fastdiv(s.Ho * s.Wo);
  g.fWo = make_fastdiv(s.Wo);
  g.fHW = make_fastdiv(s.H * s.W);
  g.fW = make_fastdiv(s.W);
  return g;
}

// Shared-memory im2col (4-channel first layers): every `unit` consecutive
// output pixels (GEMM tile rows or k-block) lie in one image and the padded
// image fits the loader scratch.  SG_SMEM_IM2COL=0 disables it (A/B).
bool smem_im2col_ok(const ConvShape& s, int unit, SmemImage* im) {
  static int on = -1;
  if (on < 0) {
    const char* env = getenv("SG_SMEM_IM2COL");
    on = env ? atoi(env) : 1;
  }
  // 1: 4-channel layers only; 2: every layer whose padded image fits
  if (!on || s.C % 4 != 0 || (on == 1 && s.C != 4) || (s.Ho * s.Wo) % unit != 0) return false;
  const int Hp = (s.Ho - 1) * s.st + s.R, Wp = (s.Wo - 1) * s.st + s.S, C4 = s.C / 4;
  if ((long long)Hp * Wp * C4 * 16 > kIm2colScratch) return false;
  *im = SmemImage{nullptr, geom(s), Hp, Wp, C4, make_fastdiv(Wp * C4), make_fastdiv(C4)};
  return true;
}

// ---------------------------------------------------------- column sums ----
constexpr int CS_ROWS_PER_BLOCK = 1024;

__global__ void colsum_partial_kernel(const float* __restrict__ X, int M, int N, long long ld,
                                      float* __restrict__ part) {
  pdl_entry();
  __shared__ float red[8][33];
  const int col = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * CS_ROWS_PER_BLOCK;
  int r1 = r0 + CS_ROWS_PER_BLOCK;
  if (r1 > M) r1 = M;
  float acc = 0.f;
  if (col < N)
    for (int r = r0 + threadIdx.y; r < r1; r += 8) acc += X[(long long)r * ld + col];
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && col < N) {
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += red[i][threadIdx.x];
    part[(long long)blockIdx.y * N + col] = s;
  }
}

__global__ void colsum_final_kernel(const float* __restrict__ part, int nparts, int N, float* __restrict__ out) {
  pdl_entry();
  int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= N) return;
  float s = 0.f;
  for (int i = 0; i < nparts; ++i) s += part[(long long)i * N + col];
  out[col] = s;
}

}  // namespace

// Tiled fp32 tensor map for kernels outside this file (conv_img.cu).
bool encode_tiled_f32(CUtensorMap* m, const void* p, int rank, const cuuint64_t* dims, const cuuint64_t* strides_b,
                      const cuuint32_t* box, CUtensorMapSwizzle sw) {
  bool ok = tma_on_impl();
  if (!ok) return false;
  *m = enc_tiled(p, rank, dims, strides_b, box, sw, &ok);
  return ok;
}

size_t gemm_ws_floats(int M, int N, int K) {
  Plan p = plan_gemm(M, N, K, (size_t)1 << 62);
  // the weight-gradient GEMMs may add one ones-row (fused bias gradient)
  return p.splits > 1 ? kSplitCounters + (size_t)p.splits * (M + 4) * pad4(N) : 0;
}

cudaError_t colsum(const float* X, int M, int N, long long ld, float* out, Workspace ws, cudaStream_t st) {
  int nparts = (M + CS_ROWS_PER_BLOCK - 1) / CS_ROWS_PER_BLOCK;
  if ((size_t)nparts * N > ws.floats) return cudaErrorInvalidValue;
  dim3 grid((N + 31) / 32, nparts);
  cudaError_t e = launch_k(colsum_partial_kernel, grid, dim3(32, 8), 0, st, X, M, N, ld, ws.ptr);
  if (e != cudaSuccess) return e;
  return launch_k(colsum_final_kernel, (N + 127) / 128, 128, 0, st, ws.ptr, nparts, N, out);
}

size_t colsum_ws_floats(int M, int N) { return (size_t)((M + CS_ROWS_PER_BLOCK - 1) / CS_ROWS_PER_BLOCK) * N; }

// ------------------------------------------------------------ small GEMMs ----
// Contractions too small to fill the tensor cores (M*N*K <= kSmallMacs, e.g. the
// CIFAR-10 / MLP output layers: 128x12x1024) are dominated by the GEMM engine's
// fixed cost (prologue, pipeline fill, split-K reduction).  Their forward and
// data gradient run on CUDA cores in fp32: op(A)(m, k) = A(m, k) or A(k, m),
// op(B)(k, n) = B(k, n) or B(n, k), row `ones_row` of op(A) = 1; fixed summation
// order per output (a warp per output: lanes stride K in ascending order, then
// an xor butterfly; K-contiguous A with K >= 128) or a thread per output
// (ascending k).
constexpr long long kSmallMacs = 4ll << 20;

__device__ __forceinline__ float mat_at(const MatView& v, int i, int j) { return v.p[(long long)i * v.ld + v.col_off(j)]; }

__device__ __forceinline__ void epi_store1(const EpiArgs& e, int row, int col, float o, int N) {
  if (row >= e.mvalid) {
    if (row == e.xrow) e.xout[col] = o;
    return;
  }
  if (e.bias) o += e.bias_on_m ? e.bias[row] : e.bias[col];
  if (e.relu) o = fmaxf(o, 0.f);
  if (e.rn) o = tf32_rna(o);
  if (e.trans)
    *out_at(e, col, row, e.mvalid) = o;
  else
    *out_at(e, row, col, N) = o;
}

struct SmallArgs {
  MatView a, b;
  int ta, tb, ones_row, M, N, K;
  EpiArgs e;
};

__device__ __forceinline__ float small_a(const SmallArgs& g, int m, int k) {
  if (m == g.ones_row) return 1.f;
  return g.ta ? mat_at(g.a, k, m) : mat_at(g.a, m, k);
}
__device__ __forceinline__ float small_b(const SmallArgs& g, int k, int n) {
  return g.tb ? mat_at(g.b, n, k) : mat_at(g.b, k, n);
}

// warp per output (op(A) rows contiguous along k)
__global__ void small_gemm_warp_kernel(const __grid_constant__ SmallArgs g) {
  pdl_entry();
  const int lane = threadIdx.x & 31;
  const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (w >= (long long)g.M * g.N) return;
  const int m = (int)(w / g.N), n = (int)(w - (long long)m * g.N);
  float acc = 0.f;
#pragma unroll 8
  for (int k = lane; k < g.K; k += 32) acc = fmaf(small_a(g, m, k), small_b(g, k, n), acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) epi_store1(g.e, m, n, acc, g.N);
}

// thread per output; consecutive threads along n (coalesced output rows and
// op(B) rows), or along m when op(A) = A^T (coalesced A columns)
__global__ void small_gemm_thread_kernel(const __grid_constant__ SmallArgs g) {
  pdl_entry();
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)g.M * g.N) return;
  int m, n;
  if (g.ta) {
    n = (int)(t / g.M);
    m = (int)(t - (long long)n * g.M);
  } else {
    m = (int)(t / g.N);
    n = (int)(t - (long long)m * g.N);
  }
  float acc = 0.f;
#pragma unroll 16  // loads of later k issue while earlier FMAs wait (loop-carried acc only)
  for (int k = 0; k < g.K; ++k) acc = fmaf(small_a(g, m, k), small_b(g, k, n), acc);
  epi_store1(g.e, m, n, acc, g.N);
}

bool small_gemm_on() {
  static int on = -1;
  if (on < 0) {
    const char* env = getenv("SG_SMALL_GEMM");
    on = env ? atoi(env) != 0 : 1;
  }
  return on != 0;
}

bool small_ok(int M, int N, int K) { return small_gemm_on() && (long long)M * N * K <= kSmallMacs; }

cudaError_t run_small(const MatView& a, int ta, const MatView& b, int tb, int ones_row, int M, int N, int K,
                      const EpiArgs& e, cudaStream_t st) {
  SmallArgs g{a, b, ta, tb, ones_row, M, N, K, e};
  const long long outs = (long long)M * N;
  if (!ta && K >= 128)  // long contiguous rows of op(A): split K over a warp
    return launch_k(small_gemm_warp_kernel, (unsigned)((outs * 32 + 255) / 256), 256, 0, st, g);
  return launch_k(small_gemm_thread_kernel, (unsigned)((outs + 255) / 256), 256, 0, st, g);
}

// ------------------------------------------------------------ convolution ----
cudaError_t conv_fwd(const ConvShape& s, const float* x, const float* W, const float* b, float* y, int flags,
                     Workspace ws, cudaStream_t st) {
  const int M = s.N * s.Ho * s.Wo, N = s.Co, K = s.R * s.S * s.C;
  if (conv_img_fwd_ok(s) && aligned16p(x) && aligned16p(W) && aligned16p(y)) return conv_img_fwd(s, x, W, b, y, flags, st);
  const EpiArgs e = epi_plain(y, s.Co, 0, b, 0, flags, M);
  if (tma_on(0) && s.C % 32 == 0 && aligned16p(x)) {
    bool ok = true;
    TmaIm2col a{};
    Plan p = plan_gemm(M, N, K, ws.floats);
    p.mt2 = tile256(p);
    a.map = enc_im2col(x, s.N, s.H, s.W, s.C, -s.pad, -s.pad, s.pad - (s.S - 1), s.pad - (s.R - 1), 32,
                       GEMM_BM * (p.mt2 ? 2 : 1), s.st, CU_TENSOR_MAP_SWIZZLE_128B, &ok);
    a.C = s.C;
    a.R = s.R;
    a.S = s.S;
    a.gH = s.Ho;
    a.gW = s.Wo;
    a.st = s.st;
    a.lo = -s.pad;
    a.flip = 0;
    a.fC = make_fastdiv(s.C);
    a.fS = make_fastdiv(s.S);
    a.fHW = make_fastdiv(s.Ho * s.Wo);
    a.fW = make_fastdiv(s.Wo);
    TmaK bw = tma_k(vplain(W, s.Co, K, K), p.bn, &ok);
    if (ok) return run_gemm_planned(a, bw, p, M, N, K, e, ws, st);
  }
  LdDenseK bw{mv(W, s.Co, K, K)};
  SmemImage im;
  if (smem_im2col_ok(s, GEMM_BM, &im)) {
    im.x = x;
    return run_gemm(LdConvFwdSmemA{im}, bw, M, N, K, e, ws, st);
  }
  LdConvFwdA a{x, geom(s)};
  return run_gemm(a, bw, M, N, K, e, ws, st);
}

cudaError_t conv_dgrad(const ConvShape& s, const float* dy, const float* W, float* dx, Workspace ws,
                       cudaStream_t st, int flags) {
  const int M = s.N * s.H * s.W, N = s.C, K = s.R * s.S * s.Co;
  if (conv_img_dgrad_ok(s) && aligned16p(dy) && aligned16p(W) && aligned16p(dx))
    return conv_img_dgrad(s, dy, W, dx, st, flags);
  const EpiArgs e = epi_plain(dx, s.C, 0, nullptr, 0, flags, M);
  if (tma_on(1) && s.st == 1 && s.Co % 32 == 0 && s.C % 32 == 0 && aligned16p(dy) && aligned16p(W)) {
    bool ok = true;
    const int lo = s.pad - (s.R - 1);
    TmaIm2col a{};
    Plan p = plan_gemm(M, N, K, ws.floats);
    p.mt2 = tile256(p);
    a.map = enc_im2col(dy, s.N, s.Ho, s.Wo, s.Co, lo, lo, lo + (s.W - s.Wo), lo + (s.H - s.Ho), 32,
                       GEMM_BM * (p.mt2 ? 2 : 1), 1, CU_TENSOR_MAP_SWIZZLE_128B, &ok);
    a.C = s.Co;
    a.R = s.R;
    a.S = s.S;
    a.gH = s.H;
    a.gW = s.W;
    a.st = 1;
    a.lo = lo;
    a.flip = 1;
    a.fC = make_fastdiv(s.Co);
    a.fS = make_fastdiv(s.S);
    a.fHW = make_fastdiv(s.H * s.W);
    a.fW = make_fastdiv(s.W);
    TmaDgradB bw{};
    // whole B tile in one 4-D box (atoms of 32 channels consecutive)
    cuuint64_t dims[4] = {32, (cuuint64_t)(s.R * s.S), (cuuint64_t)s.Co, (cuuint64_t)(s.C / 32)};
    cuuint64_t strides[3] = {(cuuint64_t)s.C * 4, (cuuint64_t)s.R * s.S * s.C * 4, 128};
    cuuint32_t box[4] = {32, 1, 32, (cuuint32_t)(p.bn / 32)};
    bw.map = enc_tiled(W, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, &ok);
    bw.atoms4 = 1;
    bw.C = s.C;
    bw.Co = s.Co;
    bw.fCo = make_fastdiv(s.Co);
    if (ok) return run_gemm_planned(a, bw, p, M, N, K, e, ws, st);
  }
  LdConvDgradA a{dy, geom(s)};
  LdConvDgradB bw{W, geom(s)};
  return run_gemm(a, bw, M, N, K, e, ws, st);
}

cudaError_t conv_wgrad(const ConvShape& s, const float* x, const float* dy, float* dW, float* db, Workspace ws,
                       cudaStream_t st) {
  const int Kg = s.R * s.S * s.C, Mtot = s.N * s.Ho * s.Wo;
  if (conv_img_wgrad_ok(s) && ws.floats >= conv_img_wgrad_ws_floats(s) && aligned16p(x) && aligned16p(dy))
    return conv_img_wgrad(s, x, dy, dW, db, ws, st);
  if (conv_img4_wgrad_ok(s) && ws.floats >= conv_img4_wgrad_ws_floats(s) && aligned16p(x) && aligned16p(dy))
    return conv_img4_wgrad(s, x, dy, dW, db, ws, st);
  // D[kg][co] stored transposed into dW[co][kg]; row Kg (ones) = db
  EpiArgs e = epi_plain(dW, Kg, 1, nullptr, 0, 0, Kg);
  if (db) {
    e.xrow = Kg;
    e.xout = db;
  }
  const int M = db ? Kg + 1 : Kg;
  // TMA im2col issues one 32-pixel box per 32 channels of every tap; with a single
  // channel block (C = 32) the TMA unit, not the tensor core, sets the pace and the
  // 256-thread cp.async gather is faster (measured: CIFAR conv2 wgrad 48.6 -> 36.3 us,
  // AlexNet conv2 (C = 64) 376 -> 416 us the other way).
  if (tma_on(2) && s.C % 32 == 0 && s.C >= 64 && aligned16p(x) && aligned16p(dy)) {
    bool ok = true;
    TmaWgradA a{};
    a.map = enc_im2col(x, s.N, s.H, s.W, s.C, -s.pad, -s.pad, s.pad - (s.S - 1), s.pad - (s.R - 1), 32, GEMM_BK, s.st,
                       CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, &ok);
    a.C = s.C;
    a.S = s.S;
    a.Ho = s.Ho;
    a.Wo = s.Wo;
    a.st = s.st;
    a.pad = s.pad;
    a.valid = Kg;
    a.ones_row = db ? Kg : -1;
    a.fC = make_fastdiv(s.C);
    a.fS = make_fastdiv(s.S);
    a.fHoWo = make_fastdiv(s.Ho * s.Wo);
    a.fWo = make_fastdiv(s.Wo);
    const Plan p = plan_gemm(M, s.Co, Mtot, ws.floats, false);
    TmaMN bd = tma_mn(vplain(dy, Mtot, s.Co, s.Co), s.Co, -1, p.bn, &ok);
    if (ok) return run_gemm_planned(a, bd, p, M, s.Co, Mtot, e, ws, st);
  }
  LdDenseMN bd{mv(dy, Mtot, s.Co, s.Co), -1};
  SmemImage im;
  if (smem_im2col_ok(s, GEMM_BK, &im)) {
    im.x = x;
    return run_gemm(LdConvWgradSmemA{im, db ? Kg : -1}, bd, M, s.Co, Mtot, e, ws, st);
  }
  LdConvWgradA a{x, geom(s), db ? Kg : -1};
  return run_gemm(a, bd, M, s.Co, Mtot, e, ws, st);
}

// ---------------------------------------------------------- inner product ----
cudaError_t ip_fwd(View2D x, const float* W, int dv, int dh, const float* b, View2D y, int flags, Workspace ws,
                   cudaStream_t st) {
  const EpiArgs e = epi_view(y, b, flags);
  if (small_ok(x.rows, dh, dv)) return run_small(mv(x), 0, mv(W, dv, dh, dh), 0, -1, x.rows, dh, dv, e, st);
  if (tma_on(3)) {
    bool ok = true;
    const Plan p = plan_gemm(x.rows, dh, dv, ws.floats);
    TmaK a = tma_k(x, GEMM_BM, &ok);
    TmaMN bw = tma_mn(vplain(W, dv, dh, dh), dh, -1, p.bn, &ok);  // op(n, k) = W(k, n)
    if (ok) return run_gemm_planned(a, bw, p, x.rows, dh, dv, e, ws, st);
  }
  LdDenseK a{mv(x)};
  LdDenseMN bw{mv(W, dv, dh, dh), -1};
  return run_gemm(a, bw, x.rows, dh, dv, e, ws, st);
}

cudaError_t ip_dgrad(View2D dy, const float* W, int dv, int dh, View2D dx, Workspace ws, cudaStream_t st,
                     int flags) {
  const EpiArgs e = epi_view(dx, nullptr, flags);
  // op(B)(k = h, n = v) = W(v, h)
  if (small_ok(dy.rows, dv, dh)) return run_small(mv(dy), 0, mv(W, dv, dh, dh), 1, -1, dy.rows, dv, dh, e, st);
  if (tma_on(3)) {
    bool ok = true;
    TmaK a = tma_k(dy, GEMM_BM, &ok);
    const Plan p = plan_gemm(dy.rows, dv, dh, ws.floats);
    TmaK bw = tma_k(vplain(W, dv, dh, dh), p.bn, &ok);  // op(n = v, k = h) = W(v, h)
    if (ok) return run_gemm_planned(a, bw, p, dy.rows, dv, dh, e, ws, st);
  }
  LdDenseK a{mv(dy)};
  LdDenseK bw{mv(W, dv, dh, dh)};
  return run_gemm(a, bw, dy.rows, dv, dh, e, ws, st);
}

cudaError_t ip_wgrad(View2D x, View2D dy, int dv, int dh, float* dW, float* db, Workspace ws, cudaStream_t st) {
  // (no CUDA-core path here: it measured no faster for the weight gradients,
  // CIFAR ip1 14 -> 18 us, MLP ip2 13.7 -> 13.6 us)
  if (tma_on(3)) {
    bool ok = true;
    const int dv32 = (dv + 31) & ~31;  // the ones row starts its own (prefilled) MN atom
    const Plan p = plan_gemm(db ? dv32 + 1 : dv, dh, x.rows, ws.floats);
    TmaMN a = tma_mn(x, dv, db ? dv32 : -1, GEMM_BM, &ok);
    TmaMN bd = tma_mn(dy, dh, -1, p.bn, &ok);
    EpiArgs e = epi_plain(dW, dh, 0, nullptr, 0, 0, dv);
    if (db) {
      e.xrow = dv32;
      e.xout = db;
    }
    if (ok) return run_gemm_planned(a, bd, p, db ? dv32 + 1 : dv, dh, x.rows, e, ws, st);
  }
  const int dv4 = (dv + 3) & ~3;
  LdDenseMN a{mv(x), db ? dv4 : -1};   // op(m = v, k = row) = x(row, v); row dv4 = ones
  LdDenseMN bd{mv(dy), -1};            // op(n = h, k = row) = dy(row, h)
  EpiArgs e = epi_plain(dW, dh, 0, nullptr, 0, 0, dv);
  if (db) {
    e.xrow = dv4;
    e.xout = db;
  }
  return run_gemm(a, bd, db ? dv4 + 1 : dv, dh, x.rows, e, ws, st);
}

cudaError_t gemm_plain(const float* A, int ta, const float* B, int tb, float* C, int M, int N, int K, Workspace ws,
                       cudaStream_t st) {
  EpiArgs e = epi_plain(C, N, 0, nullptr, 0, 0, M);
  if (tma_on(4)) {
    bool ok = true;
    const Plan p = plan_gemm(M, N, K, ws.floats);
    if (!ta && !tb) {
      TmaK a = tma_k(vplain(A, M, K, K), GEMM_BM, &ok);
      TmaMN b = tma_mn(vplain(B, K, N, N), N, -1, p.bn, &ok);
      if (ok) return run_gemm_planned(a, b, p, M, N, K, e, ws, st);
    } else if (!ta && tb) {
      TmaK a = tma_k(vplain(A, M, K, K), GEMM_BM, &ok);
      TmaK b = tma_k(vplain(B, N, K, K), p.bn, &ok);
      if (ok) return run_gemm_planned(a, b, p, M, N, K, e, ws, st);
    } else if (ta && !tb) {
      TmaMN a = tma_mn(vplain(A, K, M, M), M, -1, GEMM_BM, &ok);
      TmaMN b = tma_mn(vplain(B, K, N, N), N, -1, p.bn, &ok);
      if (ok) return run_gemm_planned(a, b, p, M, N, K, e, ws, st);
    } else {
      TmaMN a = tma_mn(vplain(A, K, M, M), M, -1, GEMM_BM, &ok);
      TmaK b = tma_k(vplain(B, N, K, K), p.bn, &ok);
      if (ok) return run_gemm_planned(a, b, p, M, N, K, e, ws, st);
    }
  }
  if (!ta && !tb) return run_gemm(LdDenseK{mv(A, M, K, K)}, LdDenseMN{mv(B, K, N, N), -1}, M, N, K, e, ws, st);
  if (!ta && tb) return run_gemm(LdDenseK{mv(A, M, K, K)}, LdDenseK{mv(B, N, K, K)}, M, N, K, e, ws, st);
  if (ta && !tb)
    return run_gemm(LdDenseMN{mv(A, K, M, M), -1}, LdDenseMN{mv(B, K, N, N), -1}, M, N, K, e, ws, st);
  return run_gemm(LdDenseMN{mv(A, K, M, M), -1}, LdDenseK{mv(B, N, K, K)}, M, N, K, e, ws, st);
}

}  // namespace sg

#ifdef SG_GEMM_TRACE
// Debug-variant export of the CTA-0 GEMM timeline (7 x 256 clock64 values).
extern "C" __attribute__((visibility("default"))) int sg_debug_gemm_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, sg::g_gemm_trace, sizeof(sg::g_gemm_trace));
}
#endif
