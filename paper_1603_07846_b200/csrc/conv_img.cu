// Resident-image convolution on tcgen05 (PAPER.md
// §5.4.1): forward and data gradient of stride-1 convolutions whose
// zero-padded input image fits in shared memory (the CIFAR-10 conv2 / conv3
// shapes).
//
// The implicit GEMM re-reads every input element R*S times; here one CTA
// stages its sample's padded image ONCE, in the UMMA K-major SWIZZLE_128B layout
// (pixel rows of 32 channels, 128 B, one plane per 32-channel block), and every
// filter tap (r, s) is a tcgen05.mma whose A descriptor simply starts
// (r*Wp + s) rows further into the image: output pixel q = oh*Wp + ow
// ("padded-width" numbering, columns ow >= Wo are discarded) reads input row
// q + r*Wp + s.  The swizzle is address-based, so any 128-byte row start is a
// valid operand (probed by tools/desc_shift.cu).  The image and the whole
// filter bank are staged by a handful of TMA boxes (zero padding = TMA
// out-of-bounds fill); after that the CTA issues MMAs only.
//
//   forward  y[q][co]  = b[co] + sum_{t, c} img_x[q + off_t][c] * W[co][t][c]
//            B = W tap tile K-major (row co, 32 channels per block)
//   dgrad    dx[q][c]  = sum_{t', co} img_dy[q + off_t'][co] * W[co][R-1-r'][S-1-s'][c]
//            (dy padded by R-1-p: a forward convolution with the flipped kernel)
//            B = W tap tile MN-major (k-line co, 32 output channels per atom)
//
// Roles (160 threads): thread 0 issues the TMA staging; warp 4 allocates TMEM
// and issues the MMAs (one lane); warps 0-3 run the epilogue (TMEM lane group =
// warp).  All accumulators of the sample (tiles x N columns) stay in TMEM.
#include <cudaTypedefs.h>

#include <algorithm>

#include "elt_common.cuh"
#include "ops.h"
#include "sg_common.cuh"

namespace sg {

bool encode_tiled_f32(CUtensorMap* m, const void* p, int rank, const cuuint64_t* dims, const cuuint64_t* strides_b,
                      const cuuint32_t* box, CUtensorMapSwizzle sw);

namespace {

constexpr int kImgThreads = 160;

#ifdef SG_GEMM_TRACE
__device__ long long g_img_trace[6][64];  // CTA 0: tap produced / tap ready / tap issued, image ready, done, start
#define IMG_TRACE(row, idx)                                                          \
  do {                                                                               \
    if (blockIdx.x == 0 && (idx) < 64) g_img_trace[row][idx] = (long long)clock64(); \
  } while (0)
#else
#define IMG_TRACE(row, idx) \
  do {                      \
  } while (0)
#endif

struct ImgConvArgs {
  CUtensorMap img_map;  // source NHWC viewed {C, W, H, N}, box {32, Wp, Hrows, 1}, SWIZZLE_128B
  CUtensorMap w_map;    // filter viewed {C, Co, T} (fwd) / {C, 32-co block rows, T} (dgrad), box {32, rows, T}
  const float* src;    // NHWC [nimg][H][W][C] (x, or dy for dgrad)
  const float* wt;     // KRSC [Co][R][S][C] of the layer
  const float* bias;   // [N] or null
  float* out;          // NHWC [nimg][Ho][Wo][N]
  int H, W, C;         // source image
  int pad, R, S;       // zero padding of the source, filter
  int Hp, Wp, Ho, Wo;  // padded source, output
  int N;               // output channels (multiple of 32)
  int layer_c, layer_co;  // the layer's C / Co (weight tensor strides)
  int ntiles, img_rows, relu, dgrad;  // relu: epilogue flags EPI_RELU | EPI_RN (ops.h)
  int split;  // CTAs per sample (strong scaling: few samples per rank), NT tiles each
  int Hrows;  // padded image rows staged (img_rows = Hrows * Wp rounded up to 8)
  int wsplit;  // filter bank staged one K block at a time
};

__device__ __forceinline__ uint32_t ksw(int row, int chunk) {  // K-major SW128 offset of a 16-B chunk
  return row * 128 + ((chunk ^ (row & 7)) << 4);
}

// Epilogue of the resident-image kernels: warp w (TMEM lane group) drains the
// NT tiles' NB accumulator columns for its 32 output rows; all tcgen05.ld of a
// tile are issued before one wait, the bias is read once.
template <int NB>
__device__ __forceinline__ void img_epilogue(uint32_t tmem, int ntiles, int warp, int lane, int Wp, int Ho, int Wo,
                                             float* outn, const float* bias, int flags, int t0 = 0) {
  float bv[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) bv[c] = bias ? __ldg(bias + c) : 0.f;
#pragma unroll 1
  for (int i = 0; i < ntiles; ++i) {
    uint32_t r[NB / 16][16];
#pragma unroll
    for (int c = 0; c < NB / 16; ++c) tmem_ld16_nowait(tmem + ((uint32_t)(warp * 32) << 16) + i * NB + c * 16, r[c]);
    tmem_wait_ld();
    const int q = (t0 + i) * 128 + warp * 32 + lane;  // tile t0 + i of the sample
    const int oh = q / Wp, ow = q - oh * Wp;
    if (oh >= Ho || ow >= Wo) continue;
    float4* dst = reinterpret_cast<float4*>(outn + ((size_t)oh * Wo + ow) * NB);
#pragma unroll
    for (int j = 0; j < NB; j += 4) {
      float4 o = make_float4(__uint_as_float(r[j / 16][j % 16]) + bv[j], __uint_as_float(r[j / 16][j % 16 + 1]) + bv[j + 1],
                             __uint_as_float(r[j / 16][j % 16 + 2]) + bv[j + 2],
                             __uint_as_float(r[j / 16][j % 16 + 3]) + bv[j + 3]);
      if (flags & EPI_RELU) o = make_float4(fmaxf(o.x, 0.f), fmaxf(o.y, 0.f), fmaxf(o.z, 0.f), fmaxf(o.w, 0.f));
      dst[j / 4] = tf32_rna4_if(o, flags & EPI_RN);
    }
  }
}

// NT output tiles of 128 padded-width rows, CB 32-channel K blocks of the
// source (compile time, so the MMA issue of a tap is straight-line code).
// Shared memory: image planes [CB][img_rows][128 B], then the filter bank
//   forward: [CB][T][Co][128 B]  (K-major SW128, row co of tap t, block cb)
//   dgrad:   [KB][NA][T][32][128 B]  (MN-major BASE32B, k-line co_in of tap t,
//            K block kb of the layer's Co, atom a of the layer's C; taps in the
//            layer's order, the flip is applied when the MMA picks the tap).
template <int NB, bool DGRAD, int NT, int CB, bool WSPLIT>
__global__ void __launch_bounds__(kImgThreads, 1) conv_img_kernel(const __grid_constant__ ImgConvArgs a) {
  constexpr int TCOLS = NT * NB <= 32 ? 32 : NT * NB <= 64 ? 64 : NT * NB <= 128 ? 128 : NT * NB <= 256 ? 256 : 512;
  constexpr int NA = NB / 32;  // dgrad: MN atoms of the output channels
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t img = base;
  const uint32_t img_plane = a.img_rows * 128;
  const uint32_t wbase = img + CB * img_plane;
  const int T = a.R * a.S;
  // WSPLIT: one K block of the filter bank resident at a time (restaged per block)
  const uint32_t wblk = (uint32_t)T * NB * 128, wbytes = (WSPLIT ? 1 : CB) * wblk;
  const uint32_t bar = wbase + wbytes, done_bar = bar + 8, wbar = done_bar + 8, wfree = wbar + 8, slot = wfree + 8;
  uint32_t* slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (slot - smem_u32(smem_raw)));
  // warp index made warp-uniform (the MMA warp's loops then stay in uniform registers)
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  // sample n, tiles [t0, t0 + nvalid) of it (a sample's tiles may be split over `split` CTAs)
  const int n = blockIdx.x / a.split, t0 = (blockIdx.x % a.split) * NT;
  const int nvalid = min(NT, a.ntiles - t0);

  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(done_bar, 1);
    mbar_init(wbar, 1);
    mbar_init(wfree, 1);
    fence_barrier_init();
    prefetch_tmap(&a.img_map);
    prefetch_tmap(&a.w_map);
  }
  if (warp == 4) tmem_alloc<TCOLS>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot_ptr;
  pdl_entry();
  if (tid == 0) {
    IMG_TRACE(5, 0);
    // one box per 32-channel plane (zero padding by out-of-bounds fill) + the filter bank
    const uint32_t img_tx = (uint32_t)a.Hrows * a.Wp * 128;
    mbar_arrive_expect_tx(bar, CB * img_tx + wbytes);
    for (int cb = 0; cb < CB; ++cb)
      tma_load_4d(img + cb * img_plane, &a.img_map, cb * 32, -a.pad, -a.pad, n, bar);
    auto load_w = [&](int kb, uint32_t dst, uint32_t b) {  // K block kb of the filter bank
      if (!DGRAD)
        tma_load_3d(dst, &a.w_map, kb * 32, 0, 0, b);
      else
        for (int at = 0; at < NA; ++at) tma_load_3d(dst + at * T * 4096, &a.w_map, at * 32, kb * 32, 0, b);
    };
    if (!WSPLIT) {
      for (int kb = 0; kb < CB; ++kb) load_w(kb, wbase + kb * wblk, bar);
    } else {
      load_w(0, wbase, bar);
      for (int kb = 1; kb < CB; ++kb) {  // restage once the MMAs of block kb-1 are done
        mbar_wait(wfree, (kb - 1) & 1);
        mbar_arrive_expect_tx(wbar, wblk);
        load_w(kb, wbase, wbar);
      }
    }
  }
  if (warp == 4) {
    // ---- MMA issue: the whole warp, elected lane issues; straight-line MMAs per tap ----
    constexpr uint32_t idesc = idesc_tf32(128, NB, 0, DGRAD ? 1 : 0);
    const uint64_t ad0 = umma_desc_sw128(img, 16, 1024);
    const uint64_t bd0 =
        DGRAD ? umma_desc_mn_sw128_32b(wbase, (uint32_t)T * 4096, 512) : umma_desc_sw128(wbase, 16, 1024);
    const uint32_t a_lo0 = (uint32_t)ad0, a_hi = (uint32_t)(ad0 >> 32);
    const uint32_t b_lo0 = (uint32_t)bd0, b_hi = (uint32_t)(bd0 >> 32);
    const uint32_t plane16 = img_plane >> 4;
    mbar_wait(bar, 0);
    if (lane == 0) IMG_TRACE(3, 0);
    tc_fence_after();
    if (WSPLIT) {
      for (int kb = 0; kb < CB; ++kb) {
        if (kb > 0) {
          mbar_wait(wbar, (kb - 1) & 1);
          tc_fence_after();
        }
        {
          int r = 0, sc = 0;
          for (int t = 0; t < T; ++t) {
            const uint32_t a_t = a_lo0 + (uint32_t)(r * a.Wp + sc) * 8 + kb * plane16;
            const uint32_t b_c = DGRAD ? b_lo0 + ((uint32_t)(T - 1 - t) * 4096 >> 4) : b_lo0 + ((uint32_t)t * NB * 128 >> 4);
#pragma unroll
            for (int i = 0; i < NT; ++i)
              if (i < nvalid)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_tf32_lh_warp(tmem + i * NB, a_t + (t0 + i) * 1024 + kk * 2, a_hi, b_c + kk * (DGRAD ? 64 : 2), b_hi,
                              idesc, (t | kb | kk) ? 1u : 0u);
            if (++sc == a.S) {
              sc = 0;
              ++r;
            }
          }
          mma_commit_warp(kb + 1 < CB ? wfree : done_bar);
        }
        __syncwarp();
      }
    }
    if (!WSPLIT) {
      int r = 0, sc = 0;
      for (int t = 0; t < T; ++t) {
        const uint32_t a_t = a_lo0 + (uint32_t)(r * a.Wp + sc) * 8;
#pragma unroll
        for (int i = 0; i < NT; ++i)
          if (i < nvalid)
#pragma unroll
          for (int cb = 0; cb < CB; ++cb) {
            // forward: tap t of block cb; dgrad: flipped tap of K block cb (atom 0; LBO = T*4096)
            const uint32_t b_c = DGRAD ? b_lo0 + ((uint32_t)(cb * NA * T + (T - 1 - t)) * 4096 >> 4)
                                       : b_lo0 + ((uint32_t)(cb * T + t) * NB * 128 >> 4);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_tf32_lh_warp(tmem + i * NB, a_t + (t0 + i) * 1024 + cb * plane16 + kk * 2, a_hi,
                          b_c + kk * (DGRAD ? 64 : 2), b_hi, idesc, (t | cb | kk) ? 1u : 0u);
          }
        if (++sc == a.S) {
          sc = 0;
          ++r;
        }
      }
      if (lane == 0) IMG_TRACE(2, 0);
      mma_commit_warp(done_bar);
    }
    __syncwarp();
  } else {
    // ---- epilogue: TMEM lane = output row q of the tile ----
    mbar_wait_sleep(done_bar, 0);
    if (tid == 0) IMG_TRACE(4, 0);
    tc_fence_after();
    img_epilogue<NB>(tmem, nvalid, warp, lane, a.Wp, a.Ho, a.Wo, a.out + (size_t)n * a.Ho * a.Wo * NB, a.bias, a.relu,
                     t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<TCOLS>(tmem);
  }
}

// On by default (SG_IMG_CONV=0 falls back to the implicit GEMM).  Staging by
// TMA matters: with per-thread cp.async staging the MMA issue ran at ~100 cycles
// per 128x32x8 MMA instead of the ~48 measured here and in tools/mma_rate.cu.
bool img_conv_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* env = getenv("SG_IMG_CONV");
    on = env ? atoi(env) != 0 : 1;
  }
  return on != 0;
}

// Geometry of one direction; false if the shape does not qualify.
bool plan_img(const ConvShape& s, bool dgrad, ImgConvArgs* a, size_t* smem) {
  if (!img_conv_enabled() || s.st != 1 || s.C % 32 || s.Co % 32) return false;
  ImgConvArgs g{};
  g.R = s.R;
  g.S = s.S;
  g.layer_c = s.C;
  g.layer_co = s.Co;
  if (!dgrad) {
    g.H = s.H, g.W = s.W, g.C = s.C, g.pad = s.pad, g.N = s.Co;
  } else {
    g.H = s.Ho, g.W = s.Wo, g.C = s.Co, g.pad = s.R - 1 - s.pad, g.N = s.C;
    if (g.pad < 0 || s.R != s.S) return false;
  }
  g.Hp = g.H + 2 * g.pad;
  g.Wp = g.W + 2 * g.pad;
  g.Ho = g.Hp - s.R + 1;
  g.Wo = g.Wp - s.S + 1;
  if (g.N != 32 && g.N != 64) return false;
  g.ntiles = (g.Ho * g.Wp + 127) / 128;
  if (g.ntiles > 4 || g.C / 32 > 2) return false;
  g.img_rows = ((g.ntiles * 128 + (s.R - 1) * g.Wp + s.S - 1) + 7) / 8 * 8;
  g.dgrad = dgrad;
  const size_t CB = g.C / 32, T = (size_t)s.R * s.S;
  g.Hrows = (g.img_rows + g.Wp - 1) / g.Wp;  // whole padded rows (TMA box), extra rows OOB-zero
  if (g.Hrows > 256 || g.Wp > 256 || T > 256) return false;
  g.img_rows = (g.Hrows * g.Wp + 7) / 8 * 8;
  const size_t img_bytes = CB * g.img_rows * 128, w_bytes = CB * T * g.N * 128;
  *smem = 1024 + img_bytes + w_bytes + 64;
  g.wsplit = 0;
  if (*smem > 227 * 1024 && CB > 1) {  // one K block of the filter bank at a time
    g.wsplit = 1;
    *smem = 1024 + img_bytes + w_bytes / CB + 64;
  }
  if (*smem > 227 * 1024) return false;
  *a = g;
  return true;
}

template <int NB, bool DG, int NT, int CB>
cudaError_t launch_img(const ImgConvArgs& a, size_t smem, int nimg, cudaStream_t st) {
  const bool split = CB > 1 && a.wsplit;
  auto k = split ? conv_img_kernel<NB, DG, NT, CB, true> : conv_img_kernel<NB, DG, NT, CB, false>;
  static size_t set[2] = {0, 0};  // per kernel variant
  if (smem > set[split]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set[split] = smem;
  }
  return launch_k(k, nimg * a.split, kImgThreads, smem, st, a);
}

// CTAs per sample: with fewer samples than SMs (strong scaling, small b/K) a
// sample's output tiles are spread over several CTAs, each staging the whole
// sample; returns the tiles per CTA.
int img_split(int ntiles, int nimg, int* split) {
  static const int maxs = getenv("SG_IMG_SPLIT") ? atoi(getenv("SG_IMG_SPLIT")) : 1 << 20;
  int s = std::max(1, std::min({ntiles, 148 / std::max(nimg, 1), maxs}));
  const int per = (ntiles + s - 1) / s;
  *split = (ntiles + per - 1) / per;
  return per;
}

template <int NB, bool DG, int NT>
cudaError_t run_img_cb(const ImgConvArgs& a, size_t smem, int nimg, cudaStream_t st) {
  return a.C / 32 == 1 ? launch_img<NB, DG, NT, 1>(a, smem, nimg, st) : launch_img<NB, DG, NT, 2>(a, smem, nimg, st);
}
template <int NB, bool DG>
cudaError_t run_img_nt(ImgConvArgs a, size_t smem, int nimg, cudaStream_t st) {
  switch (img_split(a.ntiles, nimg, &a.split)) {
    case 1: return run_img_cb<NB, DG, 1>(a, smem, nimg, st);
    case 2: return run_img_cb<NB, DG, 2>(a, smem, nimg, st);
    case 3: return run_img_cb<NB, DG, 3>(a, smem, nimg, st);
    default: return run_img_cb<NB, DG, 4>(a, smem, nimg, st);
  }
}
cudaError_t run_img(ImgConvArgs a, size_t smem, int nimg, cudaStream_t st) {
  if (a.dgrad) return a.N == 32 ? run_img_nt<32, true>(a, smem, nimg, st) : run_img_nt<64, true>(a, smem, nimg, st);
  return a.N == 32 ? run_img_nt<32, false>(a, smem, nimg, st) : run_img_nt<64, false>(a, smem, nimg, st);
}

// --------------------------------------------- 4-channel first layer forward --
// Same idea for C = 4 (CIFAR conv1), with TWO filter taps per K = 8 MMA: the
// image is staged unpadded (16 B per pixel, no swizzle) and the A operand is a
// SWIZZLE_NONE K-major descriptor with 8-row stride SBO = 128 B and K-chunk
// stride LBO = 16 B, i.e. overlapping core matrices:
//   A[m][k] = img[q0 + off + m + k/4][k % 4]   (taps (r, s) and (r, s+1))
// (probed exactly by tools/desc_overlap.cu).  The filter bank is staged tap-major
// with each filter row padded to an even number of taps (zero weights), so the
// B operand of a tap pair is W[(r*SP + s) .. +1][co][4] with LBO = Co*16 B.
struct Img4Args {
  CUtensorMap y_map;    // staged epilogue: y {Co, Ho*Wo, N}, box {32, kI4Box, 1}, SWIZZLE_128B
  const float* x;       // [N][H][W][4]
  const float* w;       // [Co][R][S][4]
  int H, W;
  const float* bias;
  float* out;
  int pad, R, S, SP, Wp, Ho, Wo, Hrows, img_rows, ntiles, relu;  // relu: epilogue flags
  int split, tpc;  // CTAs per sample, tiles per CTA
  int staged;      // 1: output tile staged in shared memory and written by TMA stores
  uint32_t y_off;  // staged output: byte offset of the staging area from the aligned base
  int y_rows;      // staged output rows per channel atom (Ho*Wo rounded up to kI4Box)
};
constexpr int kI4Box = 256;    // output pixels per TMA store box
constexpr int kI4MaxTiles = 16;
constexpr int kI4Group = 3;     // tiles per MMA commit group

// The sample's output pixels p = oh*Wo + ow, staged as [atom][p][32 ch] rows of
// 128 B in the TMA SWIZZLE_128B layout (16-B chunk c of row p at c ^ (p & 7)),
// so a warp's 32 rows hit 8 distinct bank groups.
template <int NB>
__device__ __forceinline__ void img4_stage_tile(uint32_t tmem, int i, int t0, int warp, int lane, const Img4Args& a,
                                                const float* bv, uint32_t ys) {
  uint32_t r[NB / 16][16];
#pragma unroll
  for (int c = 0; c < NB / 16; ++c) tmem_ld16_nowait(tmem + ((uint32_t)(warp * 32) << 16) + i * NB + c * 16, r[c]);
  tmem_wait_ld();
  const int q = (t0 + i) * 128 + warp * 32 + lane;
  const int oh = q / a.Wp, ow = q - oh * a.Wp;
  if (oh >= a.Ho || ow >= a.Wo) return;
  const uint32_t p = (uint32_t)(oh * a.Wo + ow);
#pragma unroll
  for (int j = 0; j < NB; j += 4) {
    float4 o = make_float4(__uint_as_float(r[j / 16][j % 16]) + bv[j], __uint_as_float(r[j / 16][j % 16 + 1]) + bv[j + 1],
                           __uint_as_float(r[j / 16][j % 16 + 2]) + bv[j + 2],
                           __uint_as_float(r[j / 16][j % 16 + 3]) + bv[j + 3]);
    if (a.relu & EPI_RELU) o = make_float4(fmaxf(o.x, 0.f), fmaxf(o.y, 0.f), fmaxf(o.z, 0.f), fmaxf(o.w, 0.f));
    o = tf32_rna4_if(o, a.relu & EPI_RN);
    const uint32_t at = (uint32_t)(j / 32), c = (uint32_t)((j % 32) / 4);
    const uint32_t addr = ys + at * (uint32_t)a.y_rows * 128 + p * 128 + ((c ^ (p & 7)) << 4);
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(o.x), "f"(o.y), "f"(o.z), "f"(o.w)
                 : "memory");
  }
}

template <int NB>
__global__ void __launch_bounds__(kImgThreads, 1) conv_img4_fwd_kernel(const __grid_constant__ Img4Args a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t img = base;
  const uint32_t wbase = img + ((a.img_rows * 16 + 1023) & ~1023);
  const uint32_t wbytes = (uint32_t)a.R * a.SP * NB * 16;
  // barriers: image+filter, then one per tile (its MMAs are done)
  const uint32_t bar = wbase + ((wbytes + 1023) & ~1023u), tbar0 = bar + 8, slot = tbar0 + 8 * kI4MaxTiles;
  const uint32_t ys = base + a.y_off;
  uint32_t* slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (slot - smem_u32(smem_raw)));
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int n = blockIdx.x / a.split, t0 = (blockIdx.x % a.split) * a.tpc;  // sample, first tile
  const int t1 = min(a.ntiles, t0 + a.tpc);

  // zero the padded image (the interior rows are then overwritten by bulk copies)
  // and the weights of the padding taps s in [S, SP); both before the predecessor ends
  for (int i = tid; i < a.img_rows; i += kImgThreads)
    asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(img + i * 16), "f"(0.f) : "memory");
  for (int i = tid; i < a.R * (a.SP - a.S) * NB; i += kImgThreads) {
    const int r = i / ((a.SP - a.S) * NB), rem = i - r * (a.SP - a.S) * NB;
    const int sc = a.S + rem / NB, co = rem % NB;
    asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(wbase + ((r * a.SP + sc) * NB + co) * 16), "f"(0.f)
                 : "memory");
  }
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(bar, 1);
    for (int i = 0; i < kI4MaxTiles; ++i) mbar_init(tbar0 + 8 * i, 1);
    fence_barrier_init();
    if (a.staged) prefetch_tmap(&a.y_map);
  }
  if (warp == 4) tmem_alloc<512>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot_ptr;
  pdl_entry();
  if (tid == 0) {
    // image rows: one contiguous bulk copy of W pixels x 16 B per row
    IMG_TRACE(5, 0);
    mbar_arrive_expect_tx(bar, (uint32_t)a.H * a.W * 16);
    const float* xn = a.x + (size_t)n * a.H * a.W * 4;
    for (int h = 0; h < a.H; ++h)
      bulk_g2s(img + (uint32_t)((h + a.pad) * a.Wp + a.pad) * 16, xn + (size_t)h * a.W * 4, (uint32_t)a.W * 16, bar);
  }
  // filter bank [co][r][s][4] -> shared [r][SP][co] 16-B rows (SIMT; all loads of a
  // thread in flight before its stores)
  for (int i0 = tid; i0 < NB * a.R * a.S; i0 += 8 * kImgThreads) {
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k * kImgThreads;
      if (i < NB * a.R * a.S) v[k] = __ldg(reinterpret_cast<const float4*>(a.w) + i);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = i0 + k * kImgThreads;
      if (i >= NB * a.R * a.S) break;
      const int co = i / (a.R * a.S), t = i - co * (a.R * a.S), r = t / a.S, sc = t - r * a.S;
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(wbase + ((r * a.SP + sc) * NB + co) * 16),
                   "f"(v[k].x), "f"(v[k].y), "f"(v[k].z), "f"(v[k].w)
                   : "memory");
    }
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (warp == 4) {
    constexpr uint32_t idesc = idesc_tf32(128, NB, 0, 0);
    const uint64_t ad0 = umma_desc_noswz(img, 16, 128), bd0 = umma_desc_noswz(wbase, NB * 16, 128);
    const uint32_t a_lo0 = (uint32_t)ad0, a_hi = (uint32_t)(ad0 >> 32);
    const uint32_t b_lo0 = (uint32_t)bd0, b_hi = (uint32_t)(bd0 >> 32);
    mbar_wait(bar, 0);
    tc_fence_after();
    // whole warp, elected lane issues (uniform-register descriptors); groups of
    // kI4Group tiles, taps outer inside a group (consecutive MMAs go to
    // independent accumulators), one commit per group, so the epilogue of a
    // group overlaps the MMAs of the next
    if (lane == 0) IMG_TRACE(3, 0);
    for (int g0 = t0; g0 < t1; g0 += kI4Group) {
      const int g1 = min(t1, g0 + kI4Group);
      for (int r = 0; r < a.R; ++r)
        for (int sc = 0; sc < a.S; sc += 2) {
          const uint32_t a_t = a_lo0 + (uint32_t)(r * a.Wp + sc);  // 16-B pixel rows: start field += 1
          const uint32_t b_t = b_lo0 + (uint32_t)(r * a.SP + sc) * NB;
          for (int i = g0; i < g1; ++i)
            mma_tf32_lh_warp(tmem + (i - t0) * NB, a_t + i * 128, a_hi, b_t, b_hi, idesc, (r | sc) ? 1u : 0u);
        }
      mma_commit_warp(tbar0 + 8 * (g1 - 1 - t0));
    }
    if (lane == 0) IMG_TRACE(2, 0);
    __syncwarp();
  } else {
    float bv[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) bv[c] = a.bias ? __ldg(a.bias + c) : 0.f;
    if (a.staged) {
      // TMEM -> swizzled shared staging -> TMA stores of whole 256-pixel boxes as soon as
      // every tile covering them is staged (the last tile flushes the rest)
      const int P = a.Ho * a.Wo;
      int next_box = 0;
      for (int i = 0; i < t1 - t0; ++i) {
        mbar_wait_sleep(tbar0 + 8 * (min(t1 - t0, (i / kI4Group + 1) * kI4Group) - 1), 0);  // i's group
        tc_fence_after();
        if (i == 0 && tid == 0) IMG_TRACE(4, 0);
        img4_stage_tile<NB>(tmem, i, t0, warp, lane, a, bv, ys);
        fence_proxy_async_smem();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (tid == 0) {
          // pixels staged so far: every q < (t0 + i + 1) * 128
          const int qd = (t0 + i + 1) * 128;
          const int pd = i + 1 == t1 - t0 ? P : min(P, (qd / a.Wp) * a.Wo + min(qd % a.Wp, a.Wo));
          bool issued = false;
          while (next_box * kI4Box < P && ((next_box + 1) * kI4Box <= pd || pd == P)) {
            for (int at = 0; at < NB / 32; ++at)
              tma_store_3d(&a.y_map, at * 32, next_box * kI4Box, n,
                           ys + (uint32_t)at * a.y_rows * 128 + (uint32_t)next_box * kI4Box * 128);
            ++next_box;
            issued = true;
          }
          if (issued) bulk_commit();
        }
      }
      if (tid == 0) bulk_wait_read0();  // the staging area is read; the writes complete with the grid
    } else {
      mbar_wait_sleep(tbar0 + 8 * (t1 - t0 - 1), 0);
      if (tid == 0) IMG_TRACE(4, 0);
      tc_fence_after();
      img_epilogue<NB>(tmem, t1 - t0, warp, lane, a.Wp, a.Ho, a.Wo, a.out + (size_t)n * a.Ho * a.Wo * NB, a.bias,
                       a.relu, t0);
    }
  }
  if (tid == 0) IMG_TRACE(0, 0);
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

bool plan_img4(const ConvShape& s, Img4Args* a, size_t* smem) {
  if (!img_conv_enabled() || s.C != 4 || s.st != 1 || (s.Co != 32 && s.Co != 64)) return false;
  Img4Args g{};
  g.pad = s.pad, g.R = s.R, g.S = s.S, g.SP = s.S + (s.S & 1);
  g.Wp = s.W + 2 * s.pad, g.Ho = s.Ho, g.Wo = s.Wo;
  g.ntiles = (g.Ho * g.Wp + 127) / 128;
  if (g.ntiles * s.Co > 512 || g.ntiles > kI4MaxTiles) return false;
  // rows read: tiles x 128 + the largest tap shift + the pair's second pixel
  const int need = g.ntiles * 128 + (s.R - 1) * g.Wp + g.SP - 1;
  g.Hrows = (need + g.Wp - 1) / g.Wp;
  g.img_rows = g.Hrows * g.Wp;
  if (g.Hrows > 256 || g.Wp > 256 || s.S > 256) return false;
  const size_t core = (((size_t)g.img_rows * 16 + 1023) & ~(size_t)1023) +
                      (((size_t)s.R * g.SP * s.Co * 16 + 1023) & ~(size_t)1023) + 1024;  // + barriers / slot
  *smem = 1024 + core;
  if (*smem > 227 * 1024) return false;
  // staged epilogue when the sample's whole output fits next to the operands
  g.y_rows = (g.Ho * g.Wo + kI4Box - 1) / kI4Box * kI4Box;
  const size_t ybytes = (size_t)(s.Co / 32) * g.y_rows * 128;
  static const int stage_env = getenv("SG_IMG4_STAGED") ? atoi(getenv("SG_IMG4_STAGED")) : 1;
  if (stage_env && 1024 + core + ybytes <= 227 * 1024 && g.Ho * g.Wo <= 256 * kI4Box) {
    g.staged = 1;
    g.y_off = (uint32_t)core;
    *smem = 1024 + core + ybytes;
  }
  *a = g;
  return true;
}

// ------------------------------------------------------------ weight gradient --
// dW[co][(r,s,c)] = sum_n sum_q img_x[q + r*Wp + s][c] * dy_pad[q][co]  (stride 1, C = 32)
// One CTA per sample n: the padded image (MN-major, k-line = padded pixel, 32
// channels) and dy in padded-width numbering (k-line q = oh*Wp + ow, zero for
// ow >= Wo: TMA out-of-bounds fill) are staged by TMA.  An M tile is four
// 32-channel atoms = four taps whose image shifts form an arithmetic sequence
// (start off, stride delta rows: the descriptor's atom stride LBO = delta*128 B,
// probed by tools/desc_shift_mn.cu); the host groups the R*S taps into such
// tiles.  A CTA takes spc consecutive samples (double-buffered TMA staging) and
// accumulates all of them in TMEM; the epilogue writes the CTA's partial dW (and
// db = sum dy, by SIMT); conv_wgrad_sum_kernel adds the partials in ascending
// CTA order (deterministic: the partition depends on the shape only).
constexpr int kMaxWTiles = 8;

struct ImgWgradArgs {
  CUtensorMap img_map;  // x NHWC {C, W, H, N}, box {32, Wp, Hrows_i, 1}, SWIZZLE_128B_ATOM_32B
  CUtensorMap dy_map;   // dy NHWC {Co, Wo, Ho, N}, box {32, Wp, Hrows_d, 1}, SWIZZLE_128B_ATOM_32B
  const float* dy;
  float* part;          // [CTA][Co*Kg + Co]
  int C, Co, R, S, pad, Wp, Ho, Wo;
  int Hrows_i, Hrows_d, rows_i, rows_d, ksteps;
  int nimg, spc;  // staged units (samples, or bands of samples), units per CTA (accumulated in TMEM)
  int split, kpc;  // CTAs per sample group (strong scaling), K steps per CTA
  int ntile;
  int t_off[kMaxWTiles], t_delta[kMaxWTiles], t_tap[kMaxWTiles][4];
  int t_cb[kMaxWTiles];  // 32-channel block of the tile's atoms (t_off includes its plane)
  int cpl;               // channel planes C / 32 of the staged image
  int nb, BR;            // bands per sample (1: whole image) and output rows per band
  int dyrows;            // dy rows per TMA box (Hrows_d; BR for bands: the k-lines past BR*Wp are zeroed once)
};

template <int NB>
__global__ void __launch_bounds__(kImgThreads, 1) conv_img_wgrad_kernel(const __grid_constant__ ImgWgradArgs a) {
  constexpr int NA = NB / 32;  // co atoms
  constexpr int TCOLS = kMaxWTiles * NB <= 256 ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t dy_plane = a.rows_d * 128;
  const uint32_t buf_bytes = a.cpl * a.rows_i * 128 + NA * dy_plane;  // one unit: image planes, then dy atoms
  const uint32_t bars = base + 2 * buf_bytes;                // full[2], empty[2], done
  const uint32_t done_bar = bars + 32, slot = done_bar + 8;
  uint32_t* slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (slot - smem_u32(smem_raw)));
  __shared__ float red[128];
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  // sample group blockIdx.x / split; K steps (pixel rows of 8) [k0, k1) of it
  const int part = blockIdx.x % a.split;
  const int n0 = (blockIdx.x / a.split) * a.spc, n1 = min(a.nimg, n0 + a.spc), ns = n1 - n0;
  const int k0 = part * a.kpc, k1 = min(a.ksteps, k0 + a.kpc);
  const int Kg = a.R * a.S * a.C, per = a.Co * Kg + a.Co;
  // unit q = band q % nb of sample q / nb: output rows [b*BR, b*BR + BR)

  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(bars + 8 * b, 1);        // TMA transaction barrier
      mbar_init(bars + 16 + 8 * b, 1);   // tcgen05.commit: buffer free
    }
    mbar_init(done_bar, 1);
    fence_barrier_init();
    prefetch_tmap(&a.img_map);
    prefetch_tmap(&a.dy_map);
  }
  {
    // band units: the dy k-lines [dyrows*Wp, ksteps*8) belong to no box (the next
    // band's rows must not enter): zero them once in both buffers
    const int z0 = a.dyrows * a.Wp, z1 = a.ksteps * 8;
    for (int i = tid; i < 2 * NA * (z1 - z0) * 8; i += kImgThreads) {
      const int c16 = i & 7, r = i >> 3, line = z0 + r % (z1 - z0), pl = r / (z1 - z0);
      const uint32_t addr = base + (pl / NA) * buf_bytes + a.cpl * a.rows_i * 128 + (pl % NA) * dy_plane + line * 128 +
                            c16 * 16;
      asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "f"(0.f) : "memory");
    }
    fence_proxy_async_smem();
  }
  if (warp == 4) tmem_alloc<TCOLS>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot_ptr;
  pdl_entry();
  const uint32_t tx = (uint32_t)(a.cpl * a.Hrows_i * a.Wp + NA * a.dyrows * a.Wp) * 128;
  auto stage = [&](int k) {  // TMA staging of unit n0 + k into buffer k & 1
    const int b = k & 1, q = n0 + k, sn = q / a.nb, y0 = (q % a.nb) * a.BR;
    const uint32_t img = base + b * buf_bytes, dyb = img + a.cpl * a.rows_i * 128;
    mbar_arrive_expect_tx(bars + 8 * b, tx);
    for (int cb = 0; cb < a.cpl; ++cb)
      tma_load_4d(img + cb * a.rows_i * 128, &a.img_map, cb * 32, -a.pad, y0 - a.pad, sn, bars + 8 * b);
    for (int at = 0; at < NA; ++at) tma_load_4d(dyb + at * dy_plane, &a.dy_map, at * 32, 0, y0, sn, bars + 8 * b);
  };
  if (warp == 4) {
    {
      // ---- MMA issue over the CTA's samples, accumulating in TMEM (whole warp, elected lane) ----
      constexpr uint32_t idesc = idesc_tf32(128, NB, 1, 1);
      for (int k = 0; k < ns; ++k) {
        const int b = k & 1;
        mbar_wait(bars + 8 * b, (k >> 1) & 1);
        tc_fence_after();
        const uint32_t img = base + b * buf_bytes, dyb = img + a.cpl * a.rows_i * 128;
        const uint64_t bd0 = umma_desc_mn_sw128_32b(dyb, dy_plane, 512);
        const uint32_t b_lo0 = (uint32_t)bd0, b_hi = (uint32_t)(bd0 >> 32);
        for (int g = 0; g < a.ntile; ++g) {
          const uint64_t ad0 = umma_desc_mn_sw128_32b(img + a.t_off[g] * 128, a.t_delta[g] * 128, 512);
          const uint32_t a_lo0 = (uint32_t)ad0, a_hi = (uint32_t)(ad0 >> 32);
          for (int ks = k0; ks < k1; ++ks)
            mma_tf32_lh_warp(tmem + g * NB, a_lo0 + ks * 64, a_hi, b_lo0 + ks * 64, b_hi, idesc,
                        (k | (ks - k0)) ? 1u : 0u);
        }
        if (k + 2 < ns) mma_commit_warp(bars + 16 + 8 * b);  // buffer b is restaged once these complete
      }
      mma_commit_warp(done_bar);
    }
    __syncwarp();
  } else {
    // ---- TMA staging, double-buffered over the CTA's units; db = the sum of the
    // staged dy tiles (thread per output channel, k-lines of this CTA's K range in
    // order, units in order), read from shared memory before a buffer is restaged ----
    if (tid == 0) {
      stage(0);
      if (ns > 1) stage(1);
    }
    float sacc = 0.f;
    const int kl0 = k0 * 8, kl1 = min(k1 * 8, a.dyrows * a.Wp);
    for (int k = 0; k < ns; ++k) {
      const int b = k & 1;
      mbar_wait(bars + 8 * b, (k >> 1) & 1);
      if (tid < a.Co) {
        const uint32_t dyb = base + b * buf_bytes + a.cpl * a.rows_i * 128 + (tid >> 5) * dy_plane;
        const uint32_t co = tid & 31;
        for (int q = kl0; q < kl1; ++q) {
          float v;
          asm volatile("ld.shared.f32 %0, [%1];"
                       : "=f"(v)
                       : "r"(dyb + q * 128 + (((co >> 3) ^ ((uint32_t)q & 3)) << 5) + (co & 7) * 4));
          sacc += v;
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // every dy read of buffer b done
      if (tid == 0 && k + 2 < ns) {
        mbar_wait(bars + 16 + 8 * b, (k >> 1) & 1);  // its MMAs done
        stage(k + 2);
      }
    }
    const int groups = 1;
    red[tid] = sacc;
    mbar_wait_sleep(done_bar, 0);
    tc_fence_after();
    // partial dW: TMEM lane = (atom = warp, channel = lane) of tile g, columns = co
    float* out = a.part + (size_t)blockIdx.x * per;
    for (int g = 0; g < a.ntile; ++g) {
      const int tap = a.t_tap[g][warp];
      const int kg = tap * a.C + a.t_cb[g] * 32 + lane;
#pragma unroll 1
      for (int c0 = 0; c0 < NB; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + g * NB + c0, v);
        if (tap < 0) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j) out[(size_t)(c0 + j) * Kg + kg] = v[j];
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");  // red[] complete (epilogue warps only)
    if (tid < a.Co) {
      float t = 0.f;
      for (int gi = 0; gi < groups; ++gi) t += red[gi * a.Co + tid];
      out[(size_t)a.Co * Kg + tid] = t;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<TCOLS>(tmem);
  }
}

// dW / db = sum over the samples' partials in ascending n: block = 32 outputs x
// 16 warps; warp w sums partials w, w+16, ...; warp 0 adds the 16 in order.
// With has_fu (first layer, K = 1) the summed element is also run through the
// Updater (fused_update1: the same arithmetic as the Updater kernels).
__global__ void __launch_bounds__(512) conv_wgrad_sum_kernel(const float* __restrict__ part, int nparts, int per,
                                                             int nw, float* __restrict__ dW, float* __restrict__ db,
                                                             FusedUpdate fu, int has_fu) {
  __shared__ float red[16][32];
  pdl_entry();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  float v = 0.f;
  if (i < per)
    for (int k = w; k < nparts; k += 16) v += __ldg(part + (size_t)k * per + i);
  red[w][lane] = v;
  __syncthreads();
  if (w != 0 || i >= per) return;
  float t = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) t += red[k][lane];
  if (i < nw) {
    dW[i] = t;
    if (has_fu) fused_update1(fu, fu.w, fu.v, fu.wk, i, t, true);
  } else if (db) {
    db[i - nw] = t;
    if (has_fu) fused_update1(fu, fu.wb, fu.vb, fu.wkb, i - nw, t, false);
  }
}

// Tap grouping: per filter row r, runs of 4 consecutive s (stride 1 row); the
// leftover columns s of all rows in runs of 4 (stride Wp rows); at most
// kMaxWTiles tiles, unused atoms marked -1.
bool plan_wgrad(const ConvShape& s, ImgWgradArgs* a, size_t* smem) {
  if (!img_conv_enabled() || s.st != 1 || (s.C != 32 && s.C != 64) || (s.Co != 32 && s.Co != 64)) return false;
  ImgWgradArgs g{};
  g.C = s.C, g.Co = s.Co, g.R = s.R, g.S = s.S, g.pad = s.pad;
  g.Wp = s.W + 2 * s.pad, g.Ho = s.Ho, g.Wo = s.Wo;
  g.cpl = s.C / 32;
  // tap tiles per 32-channel plane (t_off in k-lines of the plane; the plane
  // offset is added once the plane height is known)
  int off_in[kMaxWTiles], used[kMaxWTiles];
  g.ntile = 0;
  auto add = [&](int cb, int off, int delta, const int* taps, int cnt) {
    if (g.ntile >= kMaxWTiles) return false;
    off_in[g.ntile] = off;
    used[g.ntile] = cnt;
    g.t_cb[g.ntile] = cb;
    g.t_delta[g.ntile] = delta;
    for (int k = 0; k < 4; ++k) g.t_tap[g.ntile][k] = k < cnt ? taps[k] : -1;
    ++g.ntile;
    return true;
  };
  const int full = s.S / 4;
  for (int cb = 0; cb < g.cpl; ++cb) {
    for (int r = 0; r < s.R; ++r)
      for (int b = 0; b < full; ++b) {
        int taps[4];
        for (int k = 0; k < 4; ++k) taps[k] = r * s.S + b * 4 + k;
        if (!add(cb, r * g.Wp + b * 4, 1, taps, 4)) return false;
      }
    for (int sc = full * 4; sc < s.S; ++sc)
      for (int r0 = 0; r0 < s.R; r0 += 4) {
        int taps[4], cnt = 0;
        for (int k = 0; k < 4 && r0 + k < s.R; ++k) taps[cnt++] = (r0 + k) * s.S + sc;
        if (!add(cb, r0 * g.Wp + sc, g.Wp, taps, cnt)) return false;
      }
  }
  if (g.ntile * s.Co > 512) return false;
  // staging unit: the whole sample, or (image too large for two buffers) a band
  // of BR output rows with its R - 1 halo rows (TMA boxes at row offsets, zero
  // fill past the image)
  auto size_for = [&](int BR, size_t* sm) {
    g.BR = BR;
    g.nb = (g.Ho + BR - 1) / BR;
    const int K = BR * g.Wp;
    g.ksteps = (K + 7) / 8;
    // image rows the used atoms read; an unused 4th atom of a 3-tap tile reads
    // past them (discarded accumulator rows) but must stay inside the unit's buffer
    int need_rows = 0;
    for (int t = 0; t < g.ntile; ++t)
      need_rows = std::max(need_rows, off_in[t] + (used[t] - 1) * g.t_delta[t] + g.ksteps * 8);
    g.Hrows_i = (need_rows + g.Wp - 1) / g.Wp;
    g.Hrows_d = (g.ksteps * 8 + g.Wp - 1) / g.Wp;
    if (g.Hrows_i > 256 || g.Hrows_d > 256 || g.Wp > 256) return false;
    g.rows_i = (g.Hrows_i * g.Wp + 7) / 8 * 8;
    // a band's dy box is BR rows and the rest of its k-lines is zeroed: no halo rows
    g.rows_d = BR < g.Ho ? (g.ksteps * 8 + 7) / 8 * 8 : (g.Hrows_d * g.Wp + 7) / 8 * 8;
    const int unit_lines = g.cpl * g.rows_i + (s.Co / 32) * g.rows_d;
    for (int t = 0; t < g.ntile; ++t)
      if (off_in[t] + g.t_cb[t] * g.rows_i + 3 * g.t_delta[t] + g.ksteps * 8 > unit_lines) return false;
    *sm = 1024 + 2 * ((size_t)g.cpl * g.rows_i * 128 + (size_t)(s.Co / 32) * g.rows_d * 128) + 64;
    return *sm <= 227 * 1024;
  };
  if (!size_for(g.Ho, smem)) {
    static const int band_env = getenv("SG_WGRAD_BANDS") ? atoi(getenv("SG_WGRAD_BANDS")) : 1;
    if (!band_env) return false;
    int BR = g.Ho - 1;
    while (BR >= 1 && !size_for(BR, smem)) --BR;
    if (BR < 1) return false;
  }
  for (int t = 0; t < g.ntile; ++t) g.t_off[t] = g.t_cb[t] * g.rows_i + off_in[t];
  g.nimg = s.N * g.nb;
  g.dyrows = g.nb == 1 ? g.Hrows_d : g.BR;
  if (g.nb == 1) {
    // Samples per CTA (SG_WGRAD_SPC, default 1): accumulating several samples per
    // CTA measured slower (CIFAR conv2: 26 -> 36 us at 2, 87 us at 3).  A sample's
    // partial (Co*Kg floats, written and re-read by the reduction) must be
    // amortised by its MMAs: below ~200 MMAs per sample the implicit GEMM wins
    // (CIFAR conv3: 24 vs 20 us), so such shapes are declined.
    static const int spc_env = getenv("SG_WGRAD_SPC") ? atoi(getenv("SG_WGRAD_SPC")) : 1;
    g.spc = std::max(1, std::min(s.N, spc_env));
    if (g.ntile * g.ksteps < 200) return false;
    // strong scaling: spread a sample's K steps over several CTAs when the
    // samples alone cannot fill the machine (partials summed by the reduction)
    static const int maxs = getenv("SG_IMG_SPLIT") ? atoi(getenv("SG_IMG_SPLIT")) : 1 << 20;
    const int groups = (s.N + g.spc - 1) / g.spc;
    int sp = std::max(1, std::min({148 / std::max(groups, 1), maxs, g.ksteps / 8}));
    g.kpc = (g.ksteps + sp - 1) / sp;
    g.split = (g.ksteps + g.kpc - 1) / g.kpc;
  } else {
    // bands: one wave of CTAs, each accumulating a contiguous run of bands in TMEM
    g.spc = (g.nimg + 147) / 148;
    g.kpc = g.ksteps;
    g.split = 1;
  }
  *a = g;
  return true;
}

}  // namespace

bool conv_img_wgrad_ok(const ConvShape& s) {
  ImgWgradArgs a;
  size_t smem;
  return plan_wgrad(s, &a, &smem);
}

size_t conv_img_wgrad_ws_floats(const ConvShape& s) {
  // partials after the 1024-float head the GEMM engine keeps its split-K counters in
  ImgWgradArgs a;
  size_t smem;
  if (!plan_wgrad(s, &a, &smem)) return 0;
  const size_t ctas = (size_t)((a.nimg + a.spc - 1) / a.spc) * a.split;
  return 1024 + ctas * (size_t)(s.Co * s.R * s.S * s.C + s.Co);
}

cudaError_t conv_img_wgrad(const ConvShape& s, const float* x, const float* dy, float* dW, float* db, Workspace ws,
                           cudaStream_t st) {
  ImgWgradArgs a;
  size_t smem;
  if (!plan_wgrad(s, &a, &smem) || ws.floats < conv_img_wgrad_ws_floats(s)) return cudaErrorInvalidValue;
  a.dy = dy;
  a.part = ws.ptr + 1024;
  const cuuint64_t xd[4] = {(cuuint64_t)s.C, (cuuint64_t)s.W, (cuuint64_t)s.H, (cuuint64_t)s.N};
  const cuuint64_t xs[3] = {(cuuint64_t)s.C * 4, (cuuint64_t)s.W * s.C * 4, (cuuint64_t)s.H * s.W * s.C * 4};
  const cuuint32_t xb[4] = {32, (cuuint32_t)a.Wp, (cuuint32_t)a.Hrows_i, 1};
  const cuuint64_t dd[4] = {(cuuint64_t)s.Co, (cuuint64_t)s.Wo, (cuuint64_t)s.Ho, (cuuint64_t)s.N};
  const cuuint64_t ds[3] = {(cuuint64_t)s.Co * 4, (cuuint64_t)s.Wo * s.Co * 4, (cuuint64_t)s.Ho * s.Wo * s.Co * 4};
  const cuuint32_t db4[4] = {32, (cuuint32_t)a.Wp, (cuuint32_t)a.dyrows, 1};
  if (!encode_tiled_f32(&a.img_map, x, 4, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
      !encode_tiled_f32(&a.dy_map, dy, 4, dd, ds, db4, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
    return cudaErrorInvalidValue;
  auto k = s.Co == 32 ? conv_img_wgrad_kernel<32> : conv_img_wgrad_kernel<64>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int ctas = ((a.nimg + a.spc - 1) / a.spc) * a.split;
  e = launch_k(k, ctas, kImgThreads, smem, st, a);
  if (e != cudaSuccess) return e;
  const int nw = s.Co * s.R * s.S * s.C, per = nw + s.Co;
  return launch_k(conv_wgrad_sum_kernel, (per + 31) / 32, 512, 0, st, (const float*)a.part, ctas, per, nw, dW, db,
                  FusedUpdate{}, 0);
}

bool conv_img_fwd_ok(const ConvShape& s) {
  ImgConvArgs a;
  Img4Args a4;
  size_t smem;
  return plan_img(s, false, &a, &smem) || plan_img4(s, &a4, &smem);
}
bool conv_img_dgrad_ok(const ConvShape& s) {
  ImgConvArgs a;
  size_t smem;
  return plan_img(s, true, &a, &smem);
}

bool encode_maps(const ConvShape& s, ImgConvArgs* a) {
  // source image NHWC {C, W, H, N}; box {32, Wp, Hrows, 1} from (cb*32, -pad, -pad, n)
  const cuuint64_t idims[4] = {(cuuint64_t)a->C, (cuuint64_t)a->W, (cuuint64_t)a->H, (cuuint64_t)s.N};
  const cuuint64_t istr[3] = {(cuuint64_t)a->C * 4, (cuuint64_t)a->W * a->C * 4, (cuuint64_t)a->H * a->W * a->C * 4};
  const cuuint32_t ibox[4] = {32, (cuuint32_t)a->Wp, (cuuint32_t)a->Hrows, 1};
  if (!encode_tiled_f32(&a->img_map, a->src, 4, idims, istr, ibox, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  // filter KRSC [Co][T][C]: view {c, co, t} with strides (T*C*4, C*4)
  const int T = s.R * s.S;
  const cuuint64_t wdims[3] = {(cuuint64_t)s.C, (cuuint64_t)s.Co, (cuuint64_t)T};
  const cuuint64_t wstr[2] = {(cuuint64_t)T * s.C * 4, (cuuint64_t)s.C * 4};
  if (!a->dgrad) {
    const cuuint32_t wbox[3] = {32, (cuuint32_t)s.Co, (cuuint32_t)T};
    return encode_tiled_f32(&a->w_map, a->wt, 3, wdims, wstr, wbox, CU_TENSOR_MAP_SWIZZLE_128B);
  }
  const cuuint32_t wbox[3] = {32, 32, (cuuint32_t)T};
  return encode_tiled_f32(&a->w_map, a->wt, 3, wdims, wstr, wbox, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
}

cudaError_t conv_img_fwd(const ConvShape& s, const float* x, const float* W, const float* b, float* y, int relu,
                         cudaStream_t st) {
  ImgConvArgs a;
  size_t smem;
  Img4Args a4;
  if (plan_img4(s, &a4, &smem)) {
    a4.bias = b;
    a4.out = y;
    a4.relu = relu;
    a4.x = x;
    a4.w = W;
    a4.H = s.H, a4.W = s.W;
    a4.tpc = img_split(a4.ntiles, s.N, &a4.split);
    if (a4.staged && a4.split > 1) {  // a split sample's CTAs own partial image rows: direct stores
      a4.staged = 0;
      smem = 1024 + a4.y_off;
    }
    if (a4.staged) {
      const cuuint64_t yd[3] = {(cuuint64_t)s.Co, (cuuint64_t)s.Ho * s.Wo, (cuuint64_t)s.N};
      const cuuint64_t ys[2] = {(cuuint64_t)s.Co * 4, (cuuint64_t)s.Ho * s.Wo * s.Co * 4};
      const cuuint32_t yb[3] = {32, (cuuint32_t)kI4Box, 1};
      if (!encode_tiled_f32(&a4.y_map, y, 3, yd, ys, yb, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
    }
    auto k = s.Co == 32 ? conv_img4_fwd_kernel<32> : conv_img4_fwd_kernel<64>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    return launch_k(k, s.N * a4.split, kImgThreads, smem, st, a4);
  }
  if (!plan_img(s, false, &a, &smem)) return cudaErrorInvalidValue;
  a.src = x;
  a.wt = W;
  a.bias = b;
  a.out = y;
  a.relu = relu;
  if (!encode_maps(s, &a)) return cudaErrorInvalidValue;
  return run_img(a, smem, s.N, st);
}

cudaError_t conv_img_dgrad(const ConvShape& s, const float* dy, const float* W, float* dx, cudaStream_t st,
                           int flags) {
  ImgConvArgs a;
  size_t smem;
  if (!plan_img(s, true, &a, &smem)) return cudaErrorInvalidValue;
  a.src = dy;
  a.wt = W;
  a.bias = nullptr;
  a.out = dx;
  a.relu = flags & EPI_RN;
  if (!encode_maps(s, &a)) return cudaErrorInvalidValue;
  return run_img(a, smem, s.N, st);
}

namespace {

// ------------------------------------ 4-channel first layer: weight gradient --
// CIFAR conv1 (C = 4 padded channels, stride 1, Co = 32), optionally fused with
// the backward of the max-pooling layer that consumes it (SURVEY §8(a)
// a13 + a15):
//
//   dy[q][co]          = sum of the pool's output gradient over the windows whose
//                        argmax is q (ascending window order, = maxpool_bwd_kernel;
//                        written out: the pool's dx blob stays materialised)
//   dW[co][(r,s,c)]    = sum_n sum_q img[q + r*Wp + s][c] * dy[q][co]
//   db[co]             = sum_n sum_q dy[q][co]       (ones row of the GEMM)
//
// One CTA per sample (persistent over samples, accumulating in TMEM).  The
// sample's dy (all pixels x 32 channels, 128 KB) is built ONCE in shared memory
// in the UMMA MN-major SWIZZLE_128B_BASE32B layout (k-line = pixel) and serves as
// the B operand of every MMA; the padded image is staged by one TMA box (zero
// padding = out-of-bounds fill) and the A operand (MN-major, row kg = (tap, c),
// k-line = pixel) is an im2col built from it in shared memory, 32 pixels per
// stage, 4-stage pipeline.  Rows kg >= R*S*4 are constant (the ones row of the
// bias gradient, zeros) and written once per stage buffer.
//   warps 0-15: dy (pool backward), im2col producers; warps 0-3 the epilogue
//   warp 16   : TMEM allocation, the MMA issuer (one lane)
// The per-CTA partial is reduced by conv_wgrad_sum_kernel (fixed order).
#ifndef SG_I4W_FENCE
#define SG_I4W_FENCE 0
#endif
constexpr int kI4WProd = 512;  // producer threads (16 warps)
constexpr int kI4WThreads = kI4WProd + 32;
constexpr int kI4WStages = 4;
constexpr int kI4WKB = 32;  // pixels per stage

struct Img4WgradArgs {
  CUtensorMap img_map;  // x {4, W, H, N}, box {4, Wp, Hp, 1}, no swizzle
  CUtensorMap dyo_map;  // POOL: dy_out viewed {32, N*Ho*Wo}, box {32, 256}, SWIZZLE_128B_ATOM_32B (= dyS layout)
  const float* dy;      // !POOL: the layer's output gradient [N][Ho][Wo][32]
  float* dy_out;        // POOL: the pool's dx (= the layer's dy) [N][Ho][Wo][32]
  const float* gpool;   // POOL: pool output gradient [N][Hq][Wq][32]
  const uint8_t* mask;  // POOL: argmax window offsets [N][Hq][Wq][32]
  float* part;          // [gridDim][32 * Kg + 32]
  int nimg, Ho, Wo, Wp, Hp, R, S, T, pad, kblocks;
  int pk, ps, Hq, Wq;  // pooling window, stride, output size (pad 0)
  int rn;              // round dy to TF32 (reading A19: it is a GEMM operand)
  FastDiv fWo, fS, fps, fpk;
};

template <bool POOL>
__global__ void __launch_bounds__(kI4WThreads, 1) conv_img4_wgrad_kernel(const __grid_constant__ Img4WgradArgs a) {
  constexpr int NB = 32;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t img = base;
  const uint32_t img_bytes = ((uint32_t)a.Hp * a.Wp * 16 + 1023u) & ~1023u;
  const uint32_t dyS = img + img_bytes;
  const uint32_t dy_bytes = (uint32_t)a.kblocks * kI4WKB * 128;
  const uint32_t stage_bytes = 4 * kI4WKB * 128;  // 4 MN atoms (kg 0..127) x 32 k-lines
  const uint32_t abuf = dyS + dy_bytes;
  const uint32_t bars = abuf + kI4WStages * stage_bytes;
  // img_bar, dy_ready, img_done, full[S], empty[S], slot
  const uint32_t img_bar = bars, dy_ready = bars + 8, img_done = bars + 16;
  const uint32_t full0 = bars + 24, empty0 = full0 + 8 * kI4WStages, pool_bar = empty0 + 8 * kI4WStages;
  const uint32_t slot = pool_bar + 8;
  // POOL: the pool's output gradient and argmax of the sample are staged in the A stage buffers
  const uint32_t gps = abuf, mks = abuf + (uint32_t)a.Hq * a.Wq * NB * 4;
  uint32_t* slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (slot - smem_u32(smem_raw)));
  // warp index broadcast from lane 0: the compiler then treats role branches as
  // warp-uniform and keeps the MMA issuer's descriptors in uniform registers
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int HoWo = a.Ho * a.Wo, Kg = a.T * 4;
  const int nmine = a.nimg > (int)blockIdx.x ? (a.nimg - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  // constant A rows (tap >= T): the ones row (tap T, channel 0) and zeros, in every
  // stage buffer (rewritten per sample: the buffers also stage the pool's inputs)
  auto prefill = [&](int t0, int nt) {
    for (int i = t0; i < kI4WStages * kI4WKB * (32 - a.T); i += nt) {
      const int st = i / (kI4WKB * (32 - a.T)), rem = i - st * kI4WKB * (32 - a.T);
      const int px = rem / (32 - a.T), t = a.T + rem % (32 - a.T);
      const int at = t >> 3, lt = t & 7;
      const uint32_t dst = abuf + st * stage_bytes + at * (kI4WKB * 128) + px * 128 + (((lt >> 1) ^ (px & 3)) << 5) +
                           ((lt & 1) << 4);
      const float one = t == a.T ? 1.f : 0.f;
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %2, %2};" ::"r"(dst), "f"(one), "f"(0.f) : "memory");
    }
  };
  if (!POOL) prefill(tid, kI4WThreads);
  fence_proxy_async_smem();
  if (tid == 0) {
    mbar_init(img_bar, 1);
    mbar_init(dy_ready, kI4WProd);
    mbar_init(img_done, 1);
    mbar_init(pool_bar, 1);
    for (int st = 0; st < kI4WStages; ++st) {
      mbar_init(full0 + 8 * st, SG_I4W_FENCE == 1 ? 1 : kI4WProd / kI4WStages);  // one producer group per stage
      mbar_init(empty0 + 8 * st, 1);
    }
    fence_barrier_init();
    prefetch_tmap(&a.img_map);
  }
  constexpr int MMA_WARP = kI4WProd / 32;
  if (warp == MMA_WARP) tmem_alloc<32>(slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot_ptr;
  pdl_entry();
  if (tid == 0) IMG_TRACE(5, 0);

  if (warp == MMA_WARP) {
    // ---------------- MMA issuer (whole warp, elected lane issues) ----------------
    constexpr uint32_t idesc = idesc_tf32(128, NB, 1, 1);
    int it = 0;
    for (int i = 0; i < nmine; ++i) {
      mbar_wait(dy_ready, i & 1);
      tc_fence_after();
      for (int j = 0; j < a.kblocks; ++j, ++it) {
        const int st = it % kI4WStages;
        mbar_wait(full0 + 8 * st, (it / kI4WStages) & 1);
        tc_fence_after();
        const uint32_t as = abuf + st * stage_bytes, bs = dyS + j * kI4WKB * 128;
#pragma unroll
        for (int kk = 0; kk < kI4WKB / 8; ++kk) {
          const uint64_t ad = umma_desc_mn_sw128_32b(as + kk * 8 * 128, kI4WKB * 128, 512);
          const uint64_t bd = umma_desc_mn_sw128_32b(bs + kk * 8 * 128, kI4WKB * 128, 512);
          mma_tf32_warp(tmem, ad, bd, idesc, (i | j | kk) ? 1u : 0u);
        }
        mma_commit_warp(empty0 + 8 * st);
        if (lane == 0) IMG_TRACE(2, j);
      }
      mma_commit_warp(img_done);  // this sample's MMAs done: dyS may be rebuilt
    }
    __syncwarp();
  } else {
    // ---------------- producers (kI4WProd threads) ----------------
    // im2col work: the producer warps form 4 groups of 4 warps, group g builds the
    // stages of iterations it = g (mod 4) (its own stage buffer), so the
    // proxy fence + barrier arrive of one group overlaps the others' copies.
    // A warp task = (atom a, 4 consecutive pixels) x 8 taps t = 8a + (lane & 7):
    // its 4 k-lines of 128 B are written conflict-free; tap t >= T lanes idle.
    const int grp = warp >> 2, gw = warp & 3;
    constexpr int kMaxTask = 8;  // ceil(32 taps / 8) atoms x 8 pixel quads / 4 warps
    // (task u of this warp: k = gw + 4u; all arrays indexed by unrolled constants -> registers)
    int toff[kMaxTask], tdst[kMaxTask], tpx[kMaxTask];
    const int natom = (a.T + 7) / 8;
#pragma unroll
    for (int u = 0; u < kMaxTask; ++u) {
      const int k = gw + 4 * u;
      const int at = k / (kI4WKB / 4), px = (k % (kI4WKB / 4)) * 4 + (lane >> 3), lt = lane & 7;
      const int t = at * 8 + lt;
      const int r = a.fS.div(t), sc = t - r * a.S;
      toff[u] = (at < natom && t < a.T) ? r * a.Wp + sc : -1;
      tdst[u] = at * (kI4WKB * 128) + px * 128 + (((lt >> 1) ^ (px & 3)) << 5) + ((lt & 1) << 4);
      tpx[u] = px;
    }
    int it = 0;
    for (int i = 0; i < nmine; ++i) {
      const int n = blockIdx.x + i * gridDim.x;
      asm volatile("bar.sync 2, %0;" ::"n"(kI4WProd) : "memory");  // producers done with the previous sample's image
      if (tid == 0) {
        mbar_arrive_expect_tx(img_bar, (uint32_t)a.Hp * a.Wp * 16);
        tma_load_4d(img, &a.img_map, 0, -a.pad, -a.pad, n, img_bar);
      }
      if (i > 0) mbar_wait(img_done, (i - 1) & 1);  // the previous sample's MMAs no longer read dyS / A
      if (POOL && tid == 0) {
        const uint32_t gb = (uint32_t)a.Hq * a.Wq * NB * 4, mb = (uint32_t)a.Hq * a.Wq * NB;
        mbar_arrive_expect_tx(pool_bar, gb + mb);
        bulk_g2s(gps, a.gpool + (size_t)n * a.Hq * a.Wq * NB, gb, pool_bar);
        bulk_g2s(mks, a.mask + (size_t)n * a.Hq * a.Wq * NB, mb, pool_bar);
      }
      if (POOL) {
        if (i > 0 && tid == 0) bulk_wait_read0();  // the previous sample's dy_out store has read dyS
        asm volatile("bar.sync 2, %0;" ::"n"(kI4WProd) : "memory");
      }
      if (tid == 0) IMG_TRACE(0, 0);
      // ---- dy of this sample into dyS (and, fused, the pool's dx blob) ----
      const int nchunk = a.kblocks * kI4WKB * 8;  // (pixel, 4 channels) chunks incl. the zero tail
      auto dys_addr = [&](int q, int co) {        // MN-major SWIZZLE_128B_BASE32B, k-line = pixel
        return dyS + q * 128 + ((((uint32_t)co >> 3) ^ (q & 3)) << 5) + (co & 7) * 4;
      };
      if (POOL) {
        // max-pool backward (a13) as 4 scatter passes over the windows of one
        // (oh mod 2, ow mod 2) class: with k <= 2s windows of a class never
        // overlap, so every pass is race-free, and a pixel receives its windows'
        // gradients in the class order (= maxpool_bwd_kernel's summation order)
        for (int e = tid; e < nchunk; e += kI4WProd)
          asm volatile("st.shared.v4.f32 [%0], {%1, %1, %1, %1};" ::"r"(dys_addr(e >> 3, (e & 7) * 4)), "f"(0.f)
                       : "memory");
        mbar_wait(pool_bar, i & 1);
        for (int pass = 0; pass < 4; ++pass) {
          asm volatile("bar.sync 2, %0;" ::"n"(kI4WProd) : "memory");
          if (tid == 0) IMG_TRACE(0, 3 + pass);
          const int po = pass >> 1, pw = pass & 1;
          const int noh = (a.Hq - po + 1) >> 1, now_ = (a.Wq - pw + 1) >> 1;
          for (int e = tid; e < noh * now_ * 8; e += kI4WProd) {
            const int c4 = e & 7, wi = e >> 3;
            const int ohi = wi / now_, owi = wi - ohi * now_;
            const int oh = 2 * ohi + po, ow = 2 * owi + pw;
            const uint32_t o = (uint32_t)(oh * a.Wq + ow) * NB + c4 * 4;
            uint32_t mw;
            float g[4];
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(mw) : "r"(mks + o));
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(g[0]), "=f"(g[1]), "=f"(g[2]), "=f"(g[3])
                         : "r"(gps + o * 4));
            uint32_t ad[4];
            float v[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // 4 distinct channels: distinct addresses, loads first
              const int off = (mw >> (8 * c)) & 255;
              const int r = a.fpk.div(off), cc = off - r * a.pk;
              const int q = (oh * a.ps + r) * a.Wo + ow * a.ps + cc;
              ad[c] = dys_addr(q, c4 * 4 + c);
              asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[c]) : "r"(ad[c]));
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) asm volatile("st.shared.f32 [%0], %1;" ::"r"(ad[c]), "f"(v[c] + g[c]) : "memory");
          }
        }
        asm volatile("bar.sync 2, %0;" ::"n"(kI4WProd) : "memory");
        if (tid == 0) IMG_TRACE(0, 7);
        // TF32 rounding (the conv's dy is a GEMM operand); the materialised blob
        // (the pool's dx) is written from dyS by a TMA store once dy is complete
        if (a.rn)
          for (int e = tid; e < HoWo * 8; e += kI4WProd) {
            const uint32_t ad = dys_addr(e >> 3, (e & 7) * 4);
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(ad)
                         : "memory");
            v = tf32_rna4(v);
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(ad), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                         : "memory");
          }
      } else {
        for (int e = tid; e < nchunk; e += kI4WProd) {
          const int q = e >> 3, c4 = e & 7;
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (q < HoWo) v = __ldg(reinterpret_cast<const float4*>(a.dy) + ((size_t)n * HoWo + q) * 8 + c4);
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(dys_addr(q, c4 * 4)), "f"(v.x), "f"(v.y),
                       "f"(v.z), "f"(v.w)
                       : "memory");
        }
      }
      if (POOL) {
        if (tid == 0) IMG_TRACE(0, 8);
        asm volatile("bar.sync 2, %0;" ::"n"(kI4WProd) : "memory");  // the staged pool inputs are consumed
        if (tid == 0) IMG_TRACE(0, 9);
        prefill(tid, kI4WProd);
      }
      fence_proxy_async_smem();
      mbar_arrive(dy_ready);
      if (POOL && tid == 0) {  // dy_out <- dyS (TMA store un-swizzles; overlaps the MMA phase)
        mbar_wait(dy_ready, i & 1);
        for (int r0 = 0; r0 < HoWo; r0 += 256) tma_store_2d(&a.dyo_map, 0, n * HoWo + r0, dyS + r0 * 128);
        bulk_commit();
      }
      if (tid == 0) IMG_TRACE(0, 1);
      mbar_wait(img_bar, i & 1);
      if (tid == 0) IMG_TRACE(0, 2);
      // ---- im2col A stages (group grp: iterations it = grp mod 4) ----
      const int it0 = it;
      it += a.kblocks;
      for (int j = (grp - it0 % kI4WStages + kI4WStages) % kI4WStages; j < a.kblocks; j += kI4WStages) {
        const int itj = it0 + j, st = grp;
        if (itj >= kI4WStages) mbar_wait(empty0 + 8 * st, ((itj / kI4WStages) - 1) & 1);
        const uint32_t as = abuf + st * stage_bytes;
#pragma unroll
        for (int u = 0; u < kMaxTask; ++u) {
          if (toff[u] < 0) continue;
          const int q = j * kI4WKB + tpx[u];
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (q < HoWo) {
            const int oh = a.fWo.div(q), ow = q - oh * a.Wo;
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"(img + (uint32_t)(oh * a.Wp + ow + toff[u]) * 16));
          }
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(as + tdst[u]), "f"(v.x), "f"(v.y), "f"(v.z),
                       "f"(v.w)
                       : "memory");
        }
#ifndef SG_I4W_FENCE
#define SG_I4W_FENCE 0
#endif
#if SG_I4W_FENCE == 0
        fence_proxy_async_smem();
        mbar_arrive(full0 + 8 * st);
#elif SG_I4W_FENCE == 1
        asm volatile("bar.sync %0, 128;" ::"r"(4 + grp) : "memory");
        if ((tid & 127) == 0) {
          fence_proxy_async_smem();
          mbar_arrive(full0 + 8 * st);
        }
#else
        mbar_arrive(full0 + 8 * st);
#endif
        if (tid == 0) IMG_TRACE(1, j);
      }
    }
    // ---------------- epilogue: the CTA's partial dW / db ----------------
    if (warp < 4) {
      if (nmine > 0) mbar_wait_sleep(img_done, (nmine - 1) & 1);
      if (tid == 0) IMG_TRACE(3, 0);
      tc_fence_after();
      const int kg = warp * 32 + lane;
      float* out = a.part + (size_t)blockIdx.x * (NB * Kg + NB);
#pragma unroll 1
      for (int c0 = 0; c0 < NB; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
        if (nmine == 0) {
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = 0.f;
        }
        if (kg < Kg) {
#pragma unroll
          for (int k = 0; k < 16; ++k) out[(size_t)(c0 + k) * Kg + kg] = v[k];
        } else if (kg == Kg) {
#pragma unroll
          for (int k = 0; k < 16; ++k) out[(size_t)NB * Kg + c0 + k] = v[k];
        }
      }
    }
  }
  if (POOL && tid == 0) bulk_wait0();  // dy_out fully written before the CTA exits
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc<32>(tmem);
  }
}

bool plan_img4_wgrad(const ConvShape& s, Img4WgradArgs* a, size_t* smem) {
  if (!img_conv_enabled() || s.C != 4 || s.st != 1 || s.Co != 32) return false;
  Img4WgradArgs g{};
  g.R = s.R, g.S = s.S, g.T = s.R * s.S, g.pad = s.pad;
  g.Ho = s.Ho, g.Wo = s.Wo;
  g.Wp = s.W + 2 * s.pad, g.Hp = s.H + 2 * s.pad;
  if (g.T > 31 || g.Wp > 256 || g.Hp > 256) return false;
  if (g.Wo + s.S - 1 != g.Wp || g.Ho + s.R - 1 != g.Hp) return false;  // "same"-geometry stride-1 layer
  g.kblocks = (g.Ho * g.Wo + kI4WKB - 1) / kI4WKB;
  g.nimg = s.N;
  g.fWo = make_fastdiv(g.Wo);
  g.fS = make_fastdiv(g.S);
  const size_t img_bytes = ((size_t)g.Hp * g.Wp * 16 + 1023) & ~(size_t)1023;
  *smem = 1024 + img_bytes + (size_t)g.kblocks * kI4WKB * 128 + (size_t)kI4WStages * 4 * kI4WKB * 128 + 256;
  if (*smem > 227 * 1024) return false;
  *a = g;
  return true;
}

int img4_wgrad_ctas(int nimg) { return std::min(nimg, 148); }

cudaError_t launch_img4_wgrad(Img4WgradArgs& a, size_t smem, const float* x, const ConvShape& s, bool pool,
                              float* dW, float* db, cudaStream_t st, const FusedUpdate* fu = nullptr) {
  const cuuint64_t xd[4] = {4, (cuuint64_t)s.W, (cuuint64_t)s.H, (cuuint64_t)s.N};
  const cuuint64_t xs[3] = {16, (cuuint64_t)s.W * 16, (cuuint64_t)s.H * s.W * 16};
  const cuuint32_t xb[4] = {4, (cuuint32_t)a.Wp, (cuuint32_t)a.Hp, 1};
  if (!encode_tiled_f32(&a.img_map, x, 4, xd, xs, xb, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
  auto k = pool ? conv_img4_wgrad_kernel<true> : conv_img4_wgrad_kernel<false>;
  static size_t set[2] = {0, 0};
  if (smem > set[pool]) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set[pool] = smem;
  }
  const int ctas = img4_wgrad_ctas(s.N);
  cudaError_t e = launch_k(k, ctas, kI4WThreads, smem, st, a);
  if (e != cudaSuccess) return e;
  const int nw = s.Co * a.T * 4, per = nw + s.Co;
  return launch_k(conv_wgrad_sum_kernel, (per + 31) / 32, 512, 0, st, (const float*)a.part, ctas, per, nw, dW, db,
                  fu ? *fu : FusedUpdate{}, fu ? 1 : 0);
}

}  // namespace

bool conv_img4_wgrad_ok(const ConvShape& s) {
  Img4WgradArgs a;
  size_t smem;
  return plan_img4_wgrad(s, &a, &smem);
}

size_t conv_img4_wgrad_ws_floats(const ConvShape& s) {
  Img4WgradArgs a;
  size_t smem;
  if (!plan_img4_wgrad(s, &a, &smem)) return 0;
  return 1024 + (size_t)img4_wgrad_ctas(s.N) * (size_t)(s.Co * a.T * 4 + s.Co);
}

cudaError_t conv_img4_wgrad(const ConvShape& s, const float* x, const float* dy, float* dW, float* db, Workspace ws,
                            cudaStream_t st) {
  Img4WgradArgs a;
  size_t smem;
  if (!plan_img4_wgrad(s, &a, &smem) || ws.floats < conv_img4_wgrad_ws_floats(s)) return cudaErrorInvalidValue;
  a.dy = dy;
  a.part = ws.ptr + 1024;
  return launch_img4_wgrad(a, smem, x, s, false, dW, db, st);
}

bool conv_img4_pool_bwd_ok(const ConvShape& s, const PoolShape& p) {
  return conv_img4_wgrad_ok(s) && p.p == 0 && p.N == s.N && p.H == s.Ho && p.W == s.Wo && p.C == s.Co &&
         p.k * p.k <= 256 && p.k <= 2 * p.s && (size_t)p.Ho * p.Wo * s.Co * 5 <= (size_t)kI4WStages * 4 * kI4WKB * 128 &&
         (s.Ho * s.Wo) % 256 == 0;  // whole 256-pixel TMA store boxes per sample
}

cudaError_t conv_img4_pool_bwd(const ConvShape& s, const PoolShape& p, const float* x, const float* gpool,
                               const uint8_t* mask, float* dy_out, int rn, float* dW, float* db, Workspace ws,
                               cudaStream_t st, const FusedUpdate* fu) {
  Img4WgradArgs a;
  size_t smem;
  if (!conv_img4_pool_bwd_ok(s, p) || !plan_img4_wgrad(s, &a, &smem) || ws.floats < conv_img4_wgrad_ws_floats(s))
    return cudaErrorInvalidValue;
  a.gpool = gpool;
  a.mask = mask;
  a.dy_out = dy_out;
  {
    const cuuint64_t dd[2] = {32, (cuuint64_t)s.N * s.Ho * s.Wo};
    const cuuint64_t ds[1] = {32 * 4};
    const cuuint32_t db[2] = {32, 256};
    if (!encode_tiled_f32(&a.dyo_map, dy_out, 2, dd, ds, db, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return cudaErrorInvalidValue;
  }
  a.rn = rn;
  a.pk = p.k, a.ps = p.s, a.Hq = p.Ho, a.Wq = p.Wo;
  a.fps = make_fastdiv(p.s);
  a.fpk = make_fastdiv(p.k);
  a.part = ws.ptr + 1024;
  return launch_img4_wgrad(a, smem, x, s, true, dW, db, st, fu);
}

}  // namespace sg

#ifdef SG_GEMM_TRACE
extern "C" __attribute__((visibility("default"))) int sg_debug_img_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, sg::g_img_trace, sizeof(sg::g_img_trace));
}
#endif
