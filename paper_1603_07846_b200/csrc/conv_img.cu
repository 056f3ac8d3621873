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
// valid operand (probed by tools/desc_shift.cu).  No per-tile operand traffic
// remains except the filter taps, streamed through a cp.async ring.
//
//   forward  y[q][co]  = b[co] + sum_{t, c} img_x[q + off_t][c] * W[co][t][c]
//            B = W tap tile K-major (row co, 32 channels per block)
//   dgrad    dx[q][c]  = sum_{t', co} img_dy[q + off_t'][co] * W[co][R-1-r'][S-1-s'][c]
//            (dy padded by R-1-p: a forward convolution with the flipped kernel)
//            B = W tap tile MN-major (k-line co, 32 output channels per atom)
//
// Roles (192 threads): warps 0-3 stage the image (cp.async, mbarrier
// completion) and run the epilogue (TMEM lane group = warp); warp 4 streams the
// taps; warp 5 allocates TMEM and issues the MMAs (one elected lane).  All
// accumulators of the sample (tiles x N columns) stay in TMEM until the end.
#include <algorithm>

#include "ops.h"
#include "sg_common.cuh"

namespace sg {
namespace {

constexpr int kImgThreads = 192;

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
constexpr int kMaxStages = 8;

struct ImgConvArgs {
  const float* src;    // NHWC [nimg][H][W][C] (x, or dy for dgrad)
  const float* wt;     // KRSC [Co][R][S][C] of the layer
  const float* bias;   // [N] or null
  float* out;          // NHWC [nimg][Ho][Wo][N]
  int H, W, C;         // source image
  int pad, R, S;       // zero padding of the source, filter
  int Hp, Wp, Ho, Wo;  // padded source, output
  int N;               // output channels (multiple of 32)
  int layer_c, layer_co;  // the layer's C / Co (weight tensor strides)
  int ntiles, img_rows, relu, dgrad;
  int G, NS;  // filter taps per ring stage, ring stages (G = R*S, NS = 1: filter bank resident)
};

__device__ __forceinline__ uint32_t ksw(int row, int chunk) {  // K-major SW128 offset of a 16-B chunk
  return row * 128 + ((chunk ^ (row & 7)) << 4);
}

template <int NB, bool DGRAD>
__global__ void __launch_bounds__(kImgThreads, 1) conv_img_kernel(const __grid_constant__ ImgConvArgs a) {
  constexpr int TAP_BYTES_PER_CB = NB * 128;  // one 32-wide K block of a tap tile
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const int CB = a.C / 32;
  const uint32_t img = base;
  const uint32_t img_plane = a.img_rows * 128;
  const uint32_t wstage0 = img + CB * img_plane;
  const uint32_t tap_bytes = CB * TAP_BYTES_PER_CB;
  const uint32_t stage_bytes = a.G * tap_bytes;
  const int T = a.R * a.S, NS = a.NS, chunks = (T + a.G - 1) / a.G;
  const uint32_t bars = wstage0 + NS * stage_bytes;  // full[NS], empty[NS], img, done
  const uint32_t img_bar = bars + 16 * kMaxStages, done_bar = img_bar + 8, slot = done_bar + 8;
  uint32_t* slot_ptr = reinterpret_cast<uint32_t*>(smem_raw + (slot - smem_u32(smem_raw)));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = blockIdx.x;
  int tcols = 32;
  while (tcols < a.ntiles * NB) tcols <<= 1;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bars + 8 * s, 32);                // producer lanes (cp.async arrive)
      mbar_init(bars + 8 * (kMaxStages + s), 1);  // tcgen05.commit
    }
    mbar_init(img_bar, 128);
    mbar_init(done_bar, 1);
    fence_barrier_init();
  }
  if (warp == 5) {
    if (tcols <= 32) tmem_alloc<32>(slot);
    else if (tcols <= 64) tmem_alloc<64>(slot);
    else if (tcols <= 128) tmem_alloc<128>(slot);
    else if (tcols <= 256) tmem_alloc<256>(slot);
    else tmem_alloc<512>(slot);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot_ptr;
  pdl_entry();
  if (tid == 0) IMG_TRACE(5, 0);

  if (warp < 4) {
    // ---- stage the zero-padded image: plane cb, row rho = ph*Wp + pw ----
    const float4* src = reinterpret_cast<const float4*>(a.src) + (size_t)n * a.H * a.W * (a.C / 4);
    const int chunks = CB * a.img_rows * 8;
    for (int i = tid; i < chunks; i += 128) {
      const int cb = i / (a.img_rows * 8), rem = i - cb * a.img_rows * 8;
      const int rho = rem >> 3, c16 = rem & 7;
      const int ph = rho / a.Wp, pw = rho - ph * a.Wp;
      const int ih = ph - a.pad, iw = pw - a.pad;
      const bool in = rho < a.Hp * a.Wp && (unsigned)ih < (unsigned)a.H && (unsigned)iw < (unsigned)a.W;
      cp_async16(img + cb * img_plane + ksw(rho, c16), in ? src + ((ih * a.W + iw) * (a.C / 4) + cb * 8 + c16) : src,
                 in ? 16 : 0);
    }
    cp_async_mbar_arrive_noinc(img_bar);
  } else if (warp == 4) {
    // ---- stream the filter taps through the ring, G taps per stage ----
    for (int ch = 0; ch < chunks; ++ch) {
      const int s = ch % NS, round = ch / NS;
      if (round > 0) mbar_wait(bars + 8 * (kMaxStages + s), (round - 1) & 1);
      const int t_end = min(T, (ch + 1) * a.G);
      for (int t = ch * a.G; t < t_end; ++t) {
        const uint32_t st = wstage0 + s * stage_bytes + (t - ch * a.G) * tap_bytes;
        const int r = t / a.S, sc = t - r * a.S;
        if (!DGRAD) {
          // B[n = co][k = c] K-major: chunk (cb, co, c16) <- W[co][r][s][cb*32 + 4*c16 ..]
          for (int i = lane; i < CB * NB * 8; i += 32) {
            const int cb = i / (NB * 8), rem = i - cb * NB * 8, co = rem >> 3, c16 = rem & 7;
            const float* g = a.wt + ((size_t)(co * T + t) * a.layer_c + cb * 32 + c16 * 4);
            cp_async16(st + cb * TAP_BYTES_PER_CB + ksw(co, c16), g, 16);
          }
        } else {
          // B[n = c][k = co] MN-major, flipped tap: k-line co (K block kb), atom c/32,
          // 16-B chunk of 4 c <- W[co][R-1-r][S-1-s][c ..]
          const int tsrc = (a.R - 1 - r) * a.S + (a.S - 1 - sc);
          for (int i = lane; i < CB * NB * 8; i += 32) {
            const int kb = i / (NB * 8), rem = i - kb * NB * 8;
            const int co_in = rem / (NB / 4), cq = rem - co_in * (NB / 4);  // cq: 4-channel chunk of c
            const int c = cq * 4, atom = c >> 5, cin = c & 31;
            const float* g = a.wt + ((size_t)((kb * 32 + co_in) * T + tsrc) * a.layer_c + c);
            const uint32_t dst = st + kb * TAP_BYTES_PER_CB + atom * 4096 + co_in * 128 +
                                 ((((cin >> 3) ^ (co_in & 3))) << 5) + ((cin >> 2) & 1) * 16;
            cp_async16(dst, g, 16);
          }
        }
      }
      cp_async_mbar_arrive_noinc(bars + 8 * s);
      if (lane == 0) IMG_TRACE(0, ch);
    }
    cp_async_wait_all();
  } else {
    // ---- MMA issue ----
    constexpr uint32_t idesc = idesc_tf32(128, NB, 0, DGRAD ? 1 : 0);
    const uint64_t ad0 = umma_desc_sw128(img, 16, 1024);
    const uint64_t bd0 = DGRAD ? umma_desc_mn_sw128_32b(wstage0, 4096, 512) : umma_desc_sw128(wstage0, 16, 1024);
    const uint32_t a_lo0 = (uint32_t)ad0, a_hi = (uint32_t)(ad0 >> 32);
    const uint32_t b_lo0 = (uint32_t)bd0, b_hi = (uint32_t)(bd0 >> 32);
    mbar_wait(img_bar, 0);
    if (lane == 0) IMG_TRACE(3, 0);
    fence_proxy_async_smem();
    for (int ch = 0; ch < chunks; ++ch) {
      const int s = ch % NS;
      mbar_wait(bars + 8 * s, (ch / NS) & 1);
      if (lane == 0) IMG_TRACE(1, ch);
      fence_proxy_async_smem();
      tc_fence_after();
      if (lane == 0) {
        // descriptor start fields advance by (bytes >> 4): tap shift off*128 B,
        // tile 128 rows, channel plane, kk slice 32 B (K-major) / 1024 B (MN-major)
        const int t_end = min(T, (ch + 1) * a.G);
        for (int t = ch * a.G; t < t_end; ++t) {
          const int r = t / a.S, sc = t - r * a.S;
          const uint32_t a_t = a_lo0 + (uint32_t)(r * a.Wp + sc) * 8;
          const uint32_t b_t = b_lo0 + (uint32_t)(s * stage_bytes + (t - ch * a.G) * tap_bytes) / 16;
          for (int i = 0; i < a.ntiles; ++i) {
            const uint32_t acc = tmem + i * NB;
            for (int cb = 0; cb < CB; ++cb) {
              const uint32_t a_c = a_t + (uint32_t)i * 1024 + (uint32_t)cb * (img_plane >> 4);
              const uint32_t b_c = b_t + (uint32_t)cb * (TAP_BYTES_PER_CB >> 4);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_tf32_lh(acc, a_c + kk * 2, a_hi, b_c + kk * (DGRAD ? 64 : 2), b_hi, idesc, (t | cb | kk) ? 1u : 0u);
            }
          }
        }
        // release the stage only if the ring wraps onto it (a commit drains the pipe)
        if (ch + NS < chunks) mma_commit(bars + 8 * (kMaxStages + s));
        IMG_TRACE(2, ch);
      }
      __syncwarp();
    }
    if (lane == 0) mma_commit(done_bar);
    __syncwarp();
  }

  if (warp < 4) {
    // ---- epilogue: TMEM lane = output row q of the tile ----
    mbar_wait_sleep(done_bar, 0);
    if (tid == 0) IMG_TRACE(4, 0);
    tc_fence_after();
    float* outn = a.out + (size_t)n * a.Ho * a.Wo * NB;
    for (int i = 0; i < a.ntiles; ++i) {
      const int q = i * 128 + warp * 32 + lane;
      const int oh = q / a.Wp, ow = q - oh * a.Wp;
      const bool valid = oh < a.Ho && ow < a.Wo;
      float* dst = outn + ((size_t)oh * a.Wo + ow) * NB;
#pragma unroll 1
      for (int c0 = 0; c0 < NB; c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + i * NB + c0, v);
        if (!valid) continue;
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          if (a.bias) {
            o.x += __ldg(a.bias + c0 + j);
            o.y += __ldg(a.bias + c0 + j + 1);
            o.z += __ldg(a.bias + c0 + j + 2);
            o.w += __ldg(a.bias + c0 + j + 3);
          }
          if (a.relu) {
            o.x = fmaxf(o.x, 0.f);
            o.y = fmaxf(o.y, 0.f);
            o.z = fmaxf(o.z, 0.f);
            o.w = fmaxf(o.w, 0.f);
          }
          *reinterpret_cast<float4*>(dst + c0 + j) = o;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    if (tcols <= 32) tmem_dealloc<32>(tmem);
    else if (tcols <= 64) tmem_dealloc<64>(tmem);
    else if (tcols <= 128) tmem_dealloc<128>(tmem);
    else if (tcols <= 256) tmem_dealloc<256>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

// Off by default (SG_IMG_CONV=1 enables it): on B200 the MMA issue of this
// kernel runs at ~100 cycles per 128x32x8 TF32 MMA, twice the rate the same
// instruction sequence reaches in tools/mma_rate.cu, and the CIFAR-10 conv2 / conv3
// layers measured slower than the implicit GEMM (33 vs 25 us forward).
bool img_conv_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* env = getenv("SG_IMG_CONV");
    on = env ? atoi(env) != 0 : 0;
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
  if (g.ntiles * g.N > 512) return false;
  g.img_rows = ((g.ntiles * 128 + (s.R - 1) * g.Wp + s.S - 1) + 7) / 8 * 8;
  g.dgrad = dgrad;
  const size_t CB = g.C / 32, T = (size_t)s.R * s.S;
  const size_t tap_bytes = CB * g.N * 128, img_bytes = CB * g.img_rows * 128;
  const size_t budget = 227 * 1024 - 1024 - 256;
  if (img_bytes + 2 * tap_bytes > budget) return false;
  const size_t wbudget = budget - img_bytes;
  if (T * tap_bytes <= wbudget) {  // whole filter bank resident: one stage, no ring
    g.G = (int)T;
    g.NS = 1;
  } else {  // ring of 2..8 stages of G taps
    g.G = (int)std::max<size_t>(1, wbudget / (4 * tap_bytes));
    const size_t chunks = (T + g.G - 1) / g.G;
    g.NS = (int)std::min<size_t>({chunks, (size_t)kMaxStages, wbudget / (g.G * tap_bytes)});
    if (g.NS < 2) return false;
  }
  *smem = 1024 + img_bytes + (size_t)g.NS * g.G * tap_bytes + 256;
  if (*smem > 227 * 1024) return false;
  *a = g;
  return true;
}

template <int NB, bool DG>
cudaError_t launch_img(const ImgConvArgs& a, size_t smem, int nimg, cudaStream_t st) {
  auto k = conv_img_kernel<NB, DG>;
  static size_t set = 0;
  if (smem > set) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set = smem;
  }
  return launch_k(k, nimg, kImgThreads, smem, st, a);
}

cudaError_t run_img(ImgConvArgs a, size_t smem, int nimg, cudaStream_t st) {
  if (a.dgrad) return a.N == 32 ? launch_img<32, true>(a, smem, nimg, st) : launch_img<64, true>(a, smem, nimg, st);
  return a.N == 32 ? launch_img<32, false>(a, smem, nimg, st) : launch_img<64, false>(a, smem, nimg, st);
}

}  // namespace

bool conv_img_fwd_ok(const ConvShape& s) {
  ImgConvArgs a;
  size_t smem;
  return plan_img(s, false, &a, &smem);
}
bool conv_img_dgrad_ok(const ConvShape& s) {
  ImgConvArgs a;
  size_t smem;
  return plan_img(s, true, &a, &smem);
}

cudaError_t conv_img_fwd(const ConvShape& s, const float* x, const float* W, const float* b, float* y, int relu,
                         cudaStream_t st) {
  ImgConvArgs a;
  size_t smem;
  if (!plan_img(s, false, &a, &smem)) return cudaErrorInvalidValue;
  a.src = x;
  a.wt = W;
  a.bias = b;
  a.out = y;
  a.relu = relu;
  return run_img(a, smem, s.N, st);
}

cudaError_t conv_img_dgrad(const ConvShape& s, const float* dy, const float* W, float* dx, cudaStream_t st) {
  ImgConvArgs a;
  size_t smem;
  if (!plan_img(s, true, &a, &smem)) return cudaErrorInvalidValue;
  a.src = dy;
  a.wt = W;
  a.bias = nullptr;
  a.out = dx;
  a.relu = 0;
  return run_img(a, smem, s.N, st);
}

}  // namespace sg

#ifdef SG_GEMM_TRACE
extern "C" __attribute__((visibility("default"))) int sg_debug_img_trace(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, sg::g_img_trace, sizeof(sg::g_img_trace));
}
#endif
