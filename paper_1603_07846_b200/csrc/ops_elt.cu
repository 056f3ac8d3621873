// HBM-bound layer kernels: ReLU / sigmoid (P:241 logistic), pooling (P:553,
// Caffe geometry P:658-659), LRN across channels, softmax
// cross-entropy and Euclidean losses, the fused
// SGD-momentum Updater and the input layer's channel padding.
// Readings A5-A8 of DESIGN.md fix the definitions left open by the paper.
// All reductions run in a fixed order (bit-reproducible).
#include <cstdint>
#include <initializer_list>

#include "elt_common.cuh"
#include "ops.h"
#include "sg_common.cuh"

namespace sg {

namespace {

inline unsigned blocks_for(long long n, int per_block) {
  long long b = (n + per_block - 1) / per_block;
  if (b > 148LL * 64) b = 148LL * 64;
  return (unsigned)(b < 1 ? 1 : b);
}

// ------------------------------------------------------------ elementwise --
template <class F>
__global__ void map1_kernel(const float* __restrict__ x, float* __restrict__ y, long long n, F f, int rn) {
  pdl_entry();
  long long n4 = n >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4* y4 = reinterpret_cast<float4*>(y);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 v = x4[i];
    y4[i] = tf32_rna4_if(make_float4(f(v.x), f(v.y), f(v.z), f(v.w)), rn);
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = rn ? tf32_rna(f(x[i])) : f(x[i]);
}

template <class F>
__global__ void map2_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ y,
                            long long n, F f, int rn) {
  pdl_entry();
  long long n4 = n >> 2;
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* y4 = reinterpret_cast<float4*>(y);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 u = a4[i], v = b4[i];
    y4[i] = tf32_rna4_if(make_float4(f(u.x, v.x), f(u.y, v.y), f(u.z, v.z), f(u.w, v.w)), rn);
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = rn ? tf32_rna(f(a[i], b[i])) : f(a[i], b[i]);
}

struct ReluF {
  __device__ float operator()(float x) const { return fmaxf(x, 0.f); }
};
struct ReluB {  // dx = dy * [y > 0]
  __device__ float operator()(float y, float dy) const { return y > 0.f ? dy : 0.f; }
};
struct SigF {  // stable branch for x < 0
  __device__ float operator()(float x) const {
    if (x >= 0.f) return 1.f / (1.f + expf(-x));
    float e = expf(x);
    return e / (1.f + e);
  }
};
struct SigB {
  __device__ float operator()(float y, float dy) const { return dy * y * (1.f - y); }
};

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <class F>
cudaError_t launch_map1(const float* x, float* y, long long n, F f, cudaStream_t st, int rn) {
  if (n <= 0) return cudaSuccess;
  if (!aligned16(x) || !aligned16(y)) return cudaErrorMisalignedAddress;
  return launch_k(map1_kernel<F>, blocks_for(n / 4 + 1, 256), 256, 0, st, x, y, n, f, rn);
}
template <class F>
cudaError_t launch_map2(const float* a, const float* b, float* y, long long n, F f, cudaStream_t st, int rn) {
  if (n <= 0) return cudaSuccess;
  if (!aligned16(a) || !aligned16(b) || !aligned16(y)) return cudaErrorMisalignedAddress;
  return launch_k(map2_kernel<F>, blocks_for(n / 4 + 1, 256), 256, 0, st, a, b, y, n, f, rn);
}

// ---------------------------------------------------------------- pooling --
// Index math is 32-bit with multiply-high division by the shape constants
// (element counts < 2^31 are checked by the launchers).
struct PoolK {
  PoolShape s;
  FastDiv fC4, fWo, fHo, fW, fH, fS;
};
PoolK pool_k(const PoolShape& s) {
  return PoolK{s, make_fastdiv(s.C >> 2), make_fastdiv(s.Wo), make_fastdiv(s.Ho), make_fastdiv(s.W),
               make_fastdiv(s.H), make_fastdiv(s.s)};
}

// Window scans of the pooling forward.  KS > 0: the k x k window is a compile-time
// size, its loads are all issued before the compares (out-of-range taps
// predicated off); KS == 0: runtime k.  Same (h, w) scan order either way, so
// the same bits and argmax (first maximum, strict >; reading A5).
template <int KS>
__device__ __forceinline__ float4 maxpool_at(const PoolK& P, const float* __restrict__ x, int i, uchar4& arg) {
  const PoolShape& s = P.s;
  const int C4 = s.C >> 2;
  const int t = P.fC4.div(i), c4 = i - t * C4;
  const int t2 = P.fWo.div(t), ow = t - t2 * s.Wo;
  const int n = P.fHo.div(t2), oh = t2 - n * s.Ho;
  const int h0 = oh * s.s - s.p, w0 = ow * s.s - s.p;
  const int hs = max(h0, 0), he = min(h0 + s.k, s.H), ws = max(w0, 0), we = min(w0 + s.k, s.W);
  float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  int a[4] = {0, 0, 0, 0};
  const float* xn = x + (size_t)n * s.H * s.W * s.C + c4 * 4;
  auto take = [&](const float4& v, int off) {
    if (v.x > m[0]) { m[0] = v.x; a[0] = off; }
    if (v.y > m[1]) { m[1] = v.y; a[1] = off; }
    if (v.z > m[2]) { m[2] = v.z; a[2] = off; }
    if (v.w > m[3]) { m[3] = v.w; a[3] = off; }
  };
  if constexpr (KS > 0) {
    float4 v[KS * KS];
#pragma unroll
    for (int dh = 0; dh < KS; ++dh)
#pragma unroll
      for (int dw = 0; dw < KS; ++dw) {
        const int h = h0 + dh, w = w0 + dw;
        const bool ok = h >= hs && h < he && w >= ws && w < we;
        v[dh * KS + dw] = ok ? __ldg(reinterpret_cast<const float4*>(xn + (h * s.W + w) * s.C))
                             : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      }
#pragma unroll
    for (int j = 0; j < KS * KS; ++j) take(v[j], j);  // -inf never beats the running maximum
  } else {
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w)
        take(__ldg(reinterpret_cast<const float4*>(xn + (h * s.W + w) * s.C)), (h - h0) * s.k + (w - w0));
  }
  arg = make_uchar4(a[0], a[1], a[2], a[3]);
  return make_float4(m[0], m[1], m[2], m[3]);
}
template <int KS>
__device__ __forceinline__ float4 avgpool_at(const PoolK& P, const float* __restrict__ x, int i) {
  const PoolShape& s = P.s;
  const int C4 = s.C >> 2;
  const int t = P.fC4.div(i), c4 = i - t * C4;
  const int t2 = P.fWo.div(t), ow = t - t2 * s.Wo;
  const int n = P.fHo.div(t2), oh = t2 - n * s.Ho;
  const int h0 = oh * s.s - s.p, w0 = ow * s.s - s.p;
  const int he_u = min(h0 + s.k, s.H + s.p), we_u = min(w0 + s.k, s.W + s.p);
  const float inv = 1.f / (float)((he_u - h0) * (we_u - w0));
  const int hs = max(h0, 0), he = min(he_u, s.H), ws = max(w0, 0), we = min(we_u, s.W);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const float* xn = x + (size_t)n * s.H * s.W * s.C + c4 * 4;
  if constexpr (KS > 0) {
    float4 v[KS * KS];
    bool ok[KS * KS];
#pragma unroll
    for (int dh = 0; dh < KS; ++dh)
#pragma unroll
      for (int dw = 0; dw < KS; ++dw) {
        const int h = h0 + dh, w = w0 + dw;
        ok[dh * KS + dw] = h >= hs && h < he && w >= ws && w < we;
        v[dh * KS + dw] = ok[dh * KS + dw] ? __ldg(reinterpret_cast<const float4*>(xn + (h * s.W + w) * s.C))
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
    for (int j = 0; j < KS * KS; ++j)
      if (ok[j]) {  // the in-range taps in scan order, as the runtime loop adds them
        acc.x += v[j].x; acc.y += v[j].y; acc.z += v[j].z; acc.w += v[j].w;
      }
  } else {
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(xn + (h * s.W + w) * s.C));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
  }
  return make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
}

// Thread per (n, oh, ow, 4 channels).  Window origin (oh*s - p, ow*s - p);
// the argmax is stored as the uint8 offset (h - h0)*k + (w - w0); first maximum
// in (h, w) scan order (strict >), reading A5.
template <int KS>
__global__ void maxpool_fwd_kernel(PoolK P, const float* __restrict__ x, float* __restrict__ y,
                                   uint8_t* __restrict__ arg, float* __restrict__ relu_out, int rn) {
  pdl_entry();
  const PoolShape& s = P.s;
  const int total = s.N * s.Ho * s.Wo * (s.C >> 2);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uchar4 a4;
    const float4 o = maxpool_at<KS>(P, x, i, a4);
    *reinterpret_cast<float4*>(y + (size_t)i * 4) = tf32_rna4_if(o, rn & RN_OUT);
    *reinterpret_cast<uchar4*>(arg + (size_t)i * 4) = a4;
    if (relu_out) *reinterpret_cast<float4*>(relu_out + (size_t)i * 4) = tf32_rna4_if(relu4(o), rn & RN_AUX);
  }
}

// Windows containing input coordinate h (padded hp = h + p): oh*s <= hp < oh*s + k.
__device__ __forceinline__ void pool_windows(int hp, int k, int Ho, const FastDiv& fS, int& o0, int& o1) {
  o0 = hp >= k ? fS.div(hp - k) + 1 : 0;
  o1 = min(fS.div(hp), Ho - 1);
}

// Gather form of the backward: thread per input (n, h, w, 4 channels) sums dy
// of every window whose argmax is this element.  Fixed summation order: with
// k <= 2s (at most 2 x 2 windows per element) the windows are taken in order of
// (oh mod 2, ow mod 2) -- even rows first, even columns first -- which is the
// order of the scatter passes of the fused first-layer backward
// (conv_img.cu), so both give the same bits; otherwise ascending (oh, ow).
__global__ void maxpool_bwd_kernel(PoolK P, const float* __restrict__ dy, const uint8_t* __restrict__ arg,
                                   float* __restrict__ dx, const float* __restrict__ relu_y,
                                   float* __restrict__ dx_relu, int rn) {
  pdl_entry();
  const PoolShape& s = P.s;
  const int C4 = s.C >> 2;
  const int total = s.N * s.H * s.W * C4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int t = P.fC4.div(i), c4 = i - t * C4;
    const int t2 = P.fW.div(t), w = t - t2 * s.W;
    const int n = P.fH.div(t2), h = t2 - n * s.H;
    const int hp = h + s.p, wp = w + s.p;
    int oh0, oh1, ow0, ow1;
    pool_windows(hp, s.k, s.Ho, P.fS, oh0, oh1);
    pool_windows(wp, s.k, s.Wo, P.fS, ow0, ow1);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const size_t nb = (size_t)n * s.Ho * s.Wo * s.C + c4 * 4;
    auto add = [&](int oh, int ow, uchar4 a, float4 g) {
      const int off = (hp - oh * s.s) * s.k + (wp - ow * s.s);
      if (a.x == off) acc.x += g.x;
      if (a.y == off) acc.y += g.y;
      if (a.z == off) acc.z += g.z;
      if (a.w == off) acc.w += g.w;
    };
    if (s.k <= 2 * s.s) {
      // at most 2 x 2 windows: issue all loads first, add in (oh mod 2, ow mod 2) order
      uchar4 a[4];
      float4 g[4];
      int whs[4], wws[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int oh = oh0 + ((w >> 1) ^ (oh0 & 1)), ow = ow0 + ((w & 1) ^ (ow0 & 1));
        const bool ok = oh <= oh1 && ow <= ow1;
        whs[w] = ok ? oh : -1;
        wws[w] = ow;
        const size_t o = nb + (size_t)(ok ? oh * s.Wo + ow : 0) * s.C;
        a[w] = ok ? __ldg(reinterpret_cast<const uchar4*>(arg + o)) : make_uchar4(255, 255, 255, 255);
        g[w] = ok ? __ldg(reinterpret_cast<const float4*>(dy + o)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int w = 0; w < 4; ++w)
        if (whs[w] >= 0) add(whs[w], wws[w], a[w], g[w]);
    } else {
      for (int oh = oh0; oh <= oh1; ++oh)
        for (int ow = ow0; ow <= ow1; ++ow) {
          const size_t o = nb + (size_t)(oh * s.Wo + ow) * s.C;
          add(oh, ow, __ldg(reinterpret_cast<const uchar4*>(arg + o)), __ldg(reinterpret_cast<const float4*>(dy + o)));
        }
    }
    *reinterpret_cast<float4*>(dx + (size_t)i * 4) = tf32_rna4_if(acc, rn & RN_OUT);
    if (dx_relu)
      *reinterpret_cast<float4*>(dx_relu + (size_t)i * 4) =
          tf32_rna4_if(mask4(acc, __ldg(reinterpret_cast<const float4*>(relu_y) + i)), rn & RN_AUX);
  }
}

template <int KS>
__global__ void avgpool_fwd_kernel(PoolK P, const float* __restrict__ x, float* __restrict__ y,
                                   float* __restrict__ relu_out, int rn) {
  pdl_entry();
  const PoolShape& s = P.s;
  const int total = s.N * s.Ho * s.Wo * (s.C >> 2);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const float4 o = avgpool_at<KS>(P, x, i);
    *reinterpret_cast<float4*>(y + (size_t)i * 4) = tf32_rna4_if(o, rn & RN_OUT);
    if (relu_out) *reinterpret_cast<float4*>(relu_out + (size_t)i * 4) = tf32_rna4_if(relu4(o), rn & RN_AUX);
  }
}

__global__ void avgpool_bwd_kernel(PoolK P, const float* __restrict__ dy, float* __restrict__ dx,
                                   const float* __restrict__ relu_y, float* __restrict__ dx_relu, int rn) {
  pdl_entry();
  const PoolShape& s = P.s;
  const int C4 = s.C >> 2;
  const int total = s.N * s.H * s.W * C4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const int t = P.fC4.div(i), c4 = i - t * C4;
    const int t2 = P.fW.div(t), w = t - t2 * s.W;
    const int n = P.fH.div(t2), h = t2 - n * s.H;
    const int hp = h + s.p, wp = w + s.p;
    int oh0, oh1, ow0, ow1;
    pool_windows(hp, s.k, s.Ho, P.fS, oh0, oh1);
    pool_windows(wp, s.k, s.Wo, P.fS, ow0, ow1);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* dyn = dy + (size_t)n * s.Ho * s.Wo * s.C + c4 * 4;
    auto add = [&](int oh, int ow, float4 g) {
      const int h0 = oh * s.s - s.p, w0 = ow * s.s - s.p;
      const int hsz = min(h0 + s.k, s.H + s.p) - h0, wsz = min(w0 + s.k, s.W + s.p) - w0;
      const float inv = 1.f / (float)(hsz * wsz);
      acc.x += g.x * inv; acc.y += g.y * inv; acc.z += g.z * inv; acc.w += g.w * inv;
    };
    if (oh1 - oh0 <= 1 && ow1 - ow0 <= 1) {
      // at most 2 x 2 windows: issue all loads first, add in (oh, ow) order
      float4 g[4];
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const int oh = oh0 + (w >> 1), ow = ow0 + (w & 1);
        const bool ok = oh <= oh1 && ow <= ow1;
        g[w] = ok ? __ldg(reinterpret_cast<const float4*>(dyn + (oh * s.Wo + ow) * s.C)) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int w = 0; w < 4; ++w)
        if (oh0 + (w >> 1) <= oh1 && ow0 + (w & 1) <= ow1) add(oh0 + (w >> 1), ow0 + (w & 1), g[w]);
    } else {
      for (int oh = oh0; oh <= oh1; ++oh)
        for (int ow = ow0; ow <= ow1; ++ow)
          add(oh, ow, __ldg(reinterpret_cast<const float4*>(dyn + (oh * s.Wo + ow) * s.C)));
    }
    *reinterpret_cast<float4*>(dx + (size_t)i * 4) = tf32_rna4_if(acc, rn & RN_OUT);
    if (dx_relu)
      *reinterpret_cast<float4*>(dx_relu + (size_t)i * 4) =
          tf32_rna4_if(mask4(acc, __ldg(reinterpret_cast<const float4*>(relu_y) + i)), rn & RN_AUX);
  }
}

__global__ void argmax_expand_kernel(PoolShape s, const uint8_t* __restrict__ arg, int32_t* __restrict__ out) {
  pdl_entry();
  long long total = (long long)s.N * s.Ho * s.Wo * s.C;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    long long t = i / s.C;
    int ow = (int)(t % s.Wo);
    int oh = (int)((t / s.Wo) % s.Ho);
    int off = arg[i];
    int h = oh * s.s - s.p + off / s.k, w = ow * s.s - s.p + off % s.k;
    out[i] = h * s.W + w;
  }
}

// -------------------------------------------------------------------- LRN --
__global__ void lrn_fwd_kernel(LrnK K, const float* __restrict__ x, float* __restrict__ y, float* __restrict__ scale,
                               int rn) {
  pdl_entry();
  const int valid = (int)(K.s.pixels * K.C4);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K.total; i += gridDim.x * blockDim.x) {
    const bool in = i < valid;
    const int c4 = i % K.C4;  // C4 is a power of two
    const float4 v = in ? __ldg(reinterpret_cast<const float4*>(x) + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    float4 sc4, o4;
    lrn_apply(K.s, K.C4, v, c4, sc4, o4);
    if (in) {
      reinterpret_cast<float4*>(scale)[i] = sc4;
      reinterpret_cast<float4*>(y)[i] = tf32_rna4_if(o4, rn);
    }
  }
}

// Pooling -> (ReLU) -> LRN in one pass (layer fusion): thread per (output pixel,
// 4 channels), the LRN channel window by warp shuffles; writes the pooling
// output (+ argmax), the ReLU output and the LRN output + scale, each computed
// exactly as by the separate kernels.
template <bool MAX, int KS>
__global__ void pool_lrn_fwd_kernel(PoolK P, LrnK K, const float* __restrict__ x, float* __restrict__ py,
                                    uint8_t* __restrict__ arg, float* __restrict__ relu_out, float* __restrict__ ly,
                                    float* __restrict__ scale, int rn) {
  pdl_entry();
  const int valid = (int)(K.s.pixels * K.C4);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K.total; i += gridDim.x * blockDim.x) {
    const bool in = i < valid;
    const int c4 = i % K.C4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (in) {
      uchar4 a4;
      v = MAX ? maxpool_at<KS>(P, x, i, a4) : avgpool_at<KS>(P, x, i);
      reinterpret_cast<float4*>(py)[i] = v;
      if (MAX) reinterpret_cast<uchar4*>(arg)[i] = a4;
      if (relu_out) {
        v = relu4(v);
        reinterpret_cast<float4*>(relu_out)[i] = v;
      }
    }
    float4 sc4, o4;
    lrn_apply(K.s, K.C4, v, c4, sc4, o4);
    if (in) {
      reinterpret_cast<float4*>(scale)[i] = sc4;
      reinterpret_cast<float4*>(ly)[i] = tf32_rna4_if(o4, rn);
    }
  }
}

__global__ void lrn_bwd_kernel(LrnK K, const float* __restrict__ x, const float* __restrict__ y,
                               const float* __restrict__ scale, const float* __restrict__ dy, float* __restrict__ dx,
                               const float* __restrict__ relu_y, float* __restrict__ dx_relu, int rn) {
  pdl_entry();
  const LrnShape& s = K.s;
  const int half = s.n / 2;
  const float coef = 2.f * s.alpha * s.beta / (float)s.n;
  const int valid = (int)(s.pixels * K.C4);
  const float4 z = make_float4(0.f, 0.f, 0.f, 1.f);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < K.total; i += gridDim.x * blockDim.x) {
    const bool in = i < valid;
    const int c4 = i % K.C4;
    const float4 g = in ? __ldg(reinterpret_cast<const float4*>(dy) + i) : z;
    const float4 yv = in ? __ldg(reinterpret_cast<const float4*>(y) + i) : z;
    const float4 sv = in ? __ldg(reinterpret_cast<const float4*>(scale) + i) : make_float4(1.f, 1.f, 1.f, 1.f);
    const float4 xv = in ? __ldg(reinterpret_cast<const float4*>(x) + i) : z;
    float e[12];
    lrn_neighbours(make_float4(lrn_bwd_t(g.x, yv.x, sv.x), lrn_bwd_t(g.y, yv.y, sv.y), lrn_bwd_t(g.z, yv.z, sv.z),
                               lrn_bwd_t(g.w, yv.w, sv.w)),
                   c4, K.C4, e);
    const float gs[4] = {g.x, g.y, g.z, g.w}, ss[4] = {sv.x, sv.y, sv.z, sv.w}, xs[4] = {xv.x, xv.y, xv.z, xv.w};
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float acc = 0.f;
      // ascending d over the window (half <= 4): compile-time indices keep e[] in registers
#pragma unroll
      for (int d = -4; d <= 4; ++d)
        if (d >= -half && d <= half) acc = __fadd_rn(acc, e[4 + j + d]);
      o[j] = lrn_bwd_out(gs[j], ss[j], xs[j], acc, s.beta, coef);
    }
    if (in) {
      const float4 d = make_float4(o[0], o[1], o[2], o[3]);
      reinterpret_cast<float4*>(dx)[i] = tf32_rna4_if(d, rn & RN_OUT);
      if (dx_relu)
        reinterpret_cast<float4*>(dx_relu)[i] =
            tf32_rna4_if(mask4(d, __ldg(reinterpret_cast<const float4*>(relu_y) + i)), rn & RN_AUX);
    }
  }
}

// Generic channel counts: thread per element.
__global__ void lrn_fwd_generic_kernel(LrnShape s, const float* __restrict__ x, float* __restrict__ y,
                                       float* __restrict__ scale, int rn) {
  pdl_entry();
  long long total = s.pixels * s.C;
  const int half = s.n / 2;
  const float an = s.alpha / (float)s.n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % s.C);
    const float* px = x + (i - c);
    int lo = max(c - half, 0), hi = min(c + half, s.C - 1);
    float acc = 0.f;
    for (int cc = lo; cc <= hi; ++cc) acc += px[cc] * px[cc];
    float sc = s.k + an * acc;
    scale[i] = sc;
    const float o = x[i] * pow_neg(sc, s.beta);
    y[i] = rn ? tf32_rna(o) : o;
  }
}

__global__ void lrn_bwd_generic_kernel(LrnShape s, const float* __restrict__ x, const float* __restrict__ y,
                                       const float* __restrict__ scale, const float* __restrict__ dy,
                                       float* __restrict__ dx, const float* __restrict__ relu_y,
                                       float* __restrict__ dx_relu, int rn) {
  pdl_entry();
  long long total = s.pixels * s.C;
  const int half = s.n / 2;
  const float coef = 2.f * s.alpha * s.beta / (float)s.n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c = (int)(i % s.C);
    long long base = i - c;
    int lo = max(c - half, 0), hi = min(c + half, s.C - 1);
    float acc = 0.f;
    for (int cc = lo; cc <= hi; ++cc) acc += dy[base + cc] * y[base + cc] / scale[base + cc];
    const float d = dy[i] * pow_neg(scale[i], s.beta) - coef * x[i] * acc;
    dx[i] = (rn & RN_OUT) ? tf32_rna(d) : d;
    if (dx_relu) {
      const float dr = relu_y[i] > 0.f ? d : 0.f;
      dx_relu[i] = (rn & RN_AUX) ? tf32_rna(dr) : dr;
    }
  }
}

// ------------------------------------------------------------------ losses --
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ const float* vat(const View2D& v, int i, int j) {
  if (v.cb >= v.cols || v.cb <= 0) return v.p + (long long)i * v.ld + j;
  int b = j / v.cb;
  return v.p + (long long)b * v.bs + (long long)i * v.ld + (j - b * v.cb);
}
__device__ __forceinline__ float* vat_w(const View2D& v, int i, int j) { return const_cast<float*>(vat(v, i, j)); }

// Warp per row: max, sum of exp, loss, dz.  Lane-strided sums then a fixed
// xor-butterfly: deterministic.
__global__ void softmax_ce_kernel(View2D z, const int32_t* __restrict__ labels, float* __restrict__ row_loss,
                                  View2D dz, float inv_nloc, int* err, int rn) {
  pdl_entry();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < z.rows; r += gridDim.x * warps) {
    float m = -INFINITY;
    for (int j = lane; j < z.cols; j += 32) m = fmaxf(m, *vat(z, r, j));
    m = warp_max(m);
    float sum = 0.f;
    for (int j = lane; j < z.cols; j += 32) sum += expf(*vat(z, r, j) - m);
    sum = warp_sum(sum);
    int y = labels[r];
    bool bad = (y < 0 || y >= z.cols);
    if (bad) {
      if (lane == 0 && err) atomicOr(err, 1);
      y = 0;
    }
    float inv = 1.f / sum;
    for (int j = lane; j < z.cols; j += 32) {
      float p = expf(*vat(z, r, j) - m) * inv;
      const float d = (p - (j == y ? 1.f : 0.f)) * inv_nloc;
      *vat_w(dz, r, j) = rn ? tf32_rna(d) : d;
    }
    if (lane == 0) row_loss[r] = bad ? 0.f : (m + logf(sum)) - *vat(z, r, y);
  }
}

__global__ void euclidean_kernel(View2D u, View2D v, float* __restrict__ row_loss, View2D du, float inv_nloc, int rn) {
  pdl_entry();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < u.rows; r += gridDim.x * warps) {
    float acc = 0.f;
    for (int j = lane; j < u.cols; j += 32) {
      float d = *vat(u, r, j) - *vat(v, r, j);
      acc += d * d;
      *vat_w(du, r, j) = rn ? tf32_rna(d * inv_nloc) : d * inv_nloc;
    }
    acc = warp_sum(acc);
    if (lane == 0) row_loss[r] = 0.5f * acc;
  }
}

__global__ void sum_scaled_kernel(const float* __restrict__ v, int n, float scale, float* out, int* err) {
  pdl_entry();
  __shared__ float red[32];
  float acc = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += v[i];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) {
      float r = t * scale;
      out[0] = r;
      if (err && !isfinite(r)) atomicOr(err, 2);
    }
  }
}

// ----------------------------------------------------------------- Updater --
// Master copy w and history v updated in place; when wk != nullptr the
// working copy the GEMMs read is written too: wk[i] = TF32-RN(w[i]) for
// i < rn_end (weights, tensor-core operands, reading A19), wk[i] = w[i] beyond
// (biases, added in fp32 by the epilogues).
__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ v,
                           float* __restrict__ wk, long long rn_end, long long n, const float* lr_dev, float lr_scale,
                           float lr_val, float mu, float wd, float s) {
  pdl_entry();
  const float lr = lr_dev ? lr_dev[0] * lr_scale : lr_val;
  long long n4 = n >> 2;
  float4* w4 = reinterpret_cast<float4*>(w);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* v4 = reinterpret_cast<float4*>(v);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 ww = w4[i], gg = g4[i], vv = v4[i];
    sgd1(ww.x, gg.x, vv.x, lr, mu, wd, s);
    sgd1(ww.y, gg.y, vv.y, lr, mu, wd, s);
    sgd1(ww.z, gg.z, vv.z, lr, mu, wd, s);
    sgd1(ww.w, gg.w, vv.w, lr, mu, wd, s);
    w4[i] = ww;
    v4[i] = vv;
    if (wk) {
      const long long e = 4 * i;
      float4 k = ww;
      if (e < rn_end) k.x = tf32_rna(k.x);
      if (e + 1 < rn_end) k.y = tf32_rna(k.y);
      if (e + 2 < rn_end) k.z = tf32_rna(k.z);
      if (e + 3 < rn_end) k.w = tf32_rna(k.w);
      reinterpret_cast<float4*>(wk)[i] = k;
    }
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float ww = w[i], vv = v[i];
    sgd1(ww, g[i], vv, lr, mu, wd, s);
    w[i] = ww;
    v[i] = vv;
    if (wk) wk[i] = i < rn_end ? tf32_rna(ww) : ww;
  }
}

// AdaGrad (reading A26), same working-copy convention as sgd_kernel.
__global__ void adagrad_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ h,
                               float* __restrict__ wk, long long rn_end, long long n, const float* lr_dev,
                               float lr_scale, float lr_val, float wd, float s, float eps) {
  pdl_entry();
  const float lr = lr_dev ? lr_dev[0] * lr_scale : lr_val;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    float ww = w[i], hh = h[i];
    adagrad1(ww, g[i], hh, lr, wd, s, eps);
    w[i] = ww;
    h[i] = hh;
    if (wk) wk[i] = i < rn_end ? tf32_rna(ww) : ww;
  }
}

// ------------------------------------------------------------- input layer --
__global__ void pad_channels_kernel(const float* __restrict__ x, float* __restrict__ y, long long pixels, int cin,
                                    int cout, int rn) {
  pdl_entry();
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pixels; p += (long long)gridDim.x * blockDim.x) {
    const float* src = x + p * cin;
    float* dst = y + p * cout;
    if (cout == 4 && cin == 3) {
      *reinterpret_cast<float4*>(dst) = tf32_rna4_if(make_float4(src[0], src[1], src[2], 0.f), rn);
    } else {
      for (int c = 0; c < cout; ++c) dst[c] = c < cin ? (rn ? tf32_rna(src[c]) : src[c]) : 0.f;
    }
  }
}

__global__ void copy2d_kernel(const float* __restrict__ src, long long sld, float* __restrict__ dst, long long dld,
                              int rows, int cols, int rn) {
  pdl_entry();
  long long total = (long long)rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int r = (int)(i / cols), c = (int)(i % cols);
    const float v = src[(long long)r * sld + c];
    dst[(long long)r * dld + c] = rn ? tf32_rna(v) : v;
  }
}

// In-place TF32 rounding of a GEMM operand that arrived by a reduction
// collective (sum of rounded partials, reading A19).
__global__ void round_tf32_kernel(float* __restrict__ p, long long n) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = tf32_rna(p[i]);
}

__global__ void relu2d_kernel(const float* __restrict__ x, float* __restrict__ y, int rows, int cols, long long ld) {
  pdl_entry();
  long long total = (long long)rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int r = (int)(i / cols), c = (int)(i % cols);
    y[(long long)r * ld + c] = fmaxf(x[(long long)r * ld + c], 0.f);
  }
}

}  // namespace

cudaError_t relu_fwd(const float* x, float* y, long long n, cudaStream_t st, int rn) {
  return launch_map1(x, y, n, ReluF{}, st, rn);
}
cudaError_t relu_bwd(const float* y, const float* dy, float* dx, long long n, cudaStream_t st, int rn) {
  return launch_map2(y, dy, dx, n, ReluB{}, st, rn);
}
cudaError_t sigmoid_fwd(const float* x, float* y, long long n, cudaStream_t st, int rn) {
  return launch_map1(x, y, n, SigF{}, st, rn);
}
cudaError_t sigmoid_bwd(const float* y, const float* dy, float* dx, long long n, cudaStream_t st, int rn) {
  return launch_map2(y, dy, dx, n, SigB{}, st, rn);
}
cudaError_t relu_fwd2d(const float* x, float* y, int rows, int cols, long long ld, cudaStream_t st) {
  return launch_k(relu2d_kernel, blocks_for((long long)rows * cols, 256), 256, 0, st, x, y, rows, cols, ld);
}

static bool fits32(long long n) { return n < (1LL << 31); }

cudaError_t maxpool_fwd(const PoolShape& s, const float* x, float* y, uint8_t* arg, cudaStream_t st, float* relu_out,
                        int rn) {
  const long long n = (long long)s.N * s.Ho * s.Wo * s.C / 4;
  if (s.C % 4 || s.k * s.k > 256 || !fits32(n * 4) || !fits32((long long)s.N * s.H * s.W * s.C))
    return cudaErrorInvalidValue;
  return launch_k(s.k == 3 ? maxpool_fwd_kernel<3> : maxpool_fwd_kernel<0>, blocks_for(n, 256), 256, 0, st, pool_k(s), x,
                  y, arg, relu_out, rn);
}
cudaError_t maxpool_bwd(const PoolShape& s, const float* dy, const uint8_t* arg, float* dx, cudaStream_t st,
                        const float* relu_y, float* dx_relu, int rn) {
  const long long n = (long long)s.N * s.H * s.W * s.C / 4;
  if (s.C % 4 || !fits32(n * 4)) return cudaErrorInvalidValue;
  return launch_k(maxpool_bwd_kernel, blocks_for(n, 256), 256, 0, st, pool_k(s), dy, arg, dx, relu_y, dx_relu, rn);
}
cudaError_t avgpool_fwd(const PoolShape& s, const float* x, float* y, cudaStream_t st, float* relu_out, int rn) {
  const long long n = (long long)s.N * s.Ho * s.Wo * s.C / 4;
  if (s.C % 4 || !fits32(n * 4) || !fits32((long long)s.N * s.H * s.W * s.C)) return cudaErrorInvalidValue;
  return launch_k(s.k == 3 ? avgpool_fwd_kernel<3> : avgpool_fwd_kernel<0>, blocks_for(n, 256), 256, 0, st, pool_k(s), x,
                  y, relu_out, rn);
}
cudaError_t avgpool_bwd(const PoolShape& s, const float* dy, float* dx, cudaStream_t st, const float* relu_y,
                        float* dx_relu, int rn) {
  const long long n = (long long)s.N * s.H * s.W * s.C / 4;
  if (s.C % 4 || !fits32(n * 4)) return cudaErrorInvalidValue;
  return launch_k(avgpool_bwd_kernel, blocks_for(n, 256), 256, 0, st, pool_k(s), dy, dx, relu_y, dx_relu, rn);
}
cudaError_t pool_argmax_expand(const PoolShape& s, const uint8_t* arg, int32_t* out, cudaStream_t st) {
  return launch_k(argmax_expand_kernel, blocks_for((long long)s.N * s.Ho * s.Wo * s.C, 256), 256, 0, st, s, arg, out);
}

// float4 + warp-shuffle path when a pixel's channels fit one warp (C/4 a power of
// two <= 32), the window reaches at most one neighbouring float4 (n <= 9) and the
// blobs are 16-byte aligned; else the element-wise kernel.
static bool lrn_fast(const LrnShape& s, std::initializer_list<const void*> ptrs, LrnK* k) {
  const int C4 = s.C / 4;
  if (s.C % 4 || C4 > 32 || (C4 & (C4 - 1)) || s.n / 2 > 4 || !fits32(s.pixels * C4 + 32)) return false;
  for (const void* p : ptrs)
    if (!aligned16(p)) return false;
  k->s = s;
  k->C4 = C4;
  k->total = (int)((s.pixels * C4 + 31) / 32 * 32);
  return true;
}
cudaError_t lrn_fwd(const LrnShape& s, const float* x, float* y, float* scale, cudaStream_t st, int rn) {
  LrnK k;
  if (lrn_fast(s, {x, y, scale}, &k))
    return launch_k(lrn_fwd_kernel, blocks_for(k.total, 256), 256, 0, st, k, x, y, scale, rn);
  return launch_k(lrn_fwd_generic_kernel, blocks_for(s.pixels * s.C, 256), 256, 0, st, s, x, y, scale, rn);
}
cudaError_t lrn_bwd(const LrnShape& s, const float* x, const float* y, const float* scale, const float* dy, float* dx,
                    cudaStream_t st, const float* relu_y, float* dx_relu, int rn) {
  LrnK k;
  if (lrn_fast(s, {x, y, scale, dy, dx, dx_relu ? relu_y : x, dx_relu ? dx_relu : dx}, &k))
    return launch_k(lrn_bwd_kernel, blocks_for(k.total, 256), 256, 0, st, k, x, y, scale, dy, dx, relu_y, dx_relu, rn);
  return launch_k(lrn_bwd_generic_kernel, blocks_for(s.pixels * s.C, 256), 256, 0, st, s, x, y, scale, dy, dx, relu_y,
                  dx_relu, rn);
}

cudaError_t pool_lrn_fwd(const PoolShape& ps, bool max_pool, const float* x, float* py, uint8_t* arg, float* relu_out,
                         const LrnShape& ls, float* ly, float* scale, cudaStream_t st, int rn) {
  LrnK k;
  const long long n4 = (long long)ps.N * ps.Ho * ps.Wo * ps.C / 4;
  if (ps.C % 4 || ls.C != ps.C || ls.pixels != (long long)ps.N * ps.Ho * ps.Wo || !fits32(n4 * 4) ||
      !fits32((long long)ps.N * ps.H * ps.W * ps.C) || (max_pool && ps.k * ps.k > 256) ||
      !lrn_fast(ls, {py, ly, scale, relu_out ? relu_out : py}, &k))
    return cudaErrorInvalidValue;
  auto kern = max_pool ? (ps.k == 3 ? pool_lrn_fwd_kernel<true, 3> : pool_lrn_fwd_kernel<true, 0>)
                      : (ps.k == 3 ? pool_lrn_fwd_kernel<false, 3> : pool_lrn_fwd_kernel<false, 0>);
  return launch_k(kern, blocks_for(k.total, 256), 256, 0, st, pool_k(ps), k, x, py, arg, relu_out, ly, scale, rn);
}
bool pool_lrn_fusable(const PoolShape& ps, const LrnShape& ls) {
  LrnK k;
  float dummy[4] __attribute__((aligned(16)));
  return ps.C % 4 == 0 && ls.C == ps.C && ls.pixels == (long long)ps.N * ps.Ho * ps.Wo && ps.k * ps.k <= 256 &&
         fits32((long long)ps.N * ps.H * ps.W * ps.C) && lrn_fast(ls, {dummy}, &k);
}

cudaError_t softmax_ce(View2D z, const int32_t* labels, float* row_loss, View2D dz, float inv_nloc, int* err,
                       cudaStream_t st, int rn) {
  if (z.rows <= 0) return cudaSuccess;
  return launch_k(softmax_ce_kernel, (z.rows + 7) / 8, 256, 0, st, z, labels, row_loss, dz, inv_nloc, err, rn);
}
cudaError_t euclidean(View2D u, View2D v, float* row_loss, View2D du, float inv_nloc, cudaStream_t st, int rn) {
  if (u.rows <= 0) return cudaSuccess;
  return launch_k(euclidean_kernel, (u.rows + 7) / 8, 256, 0, st, u, v, row_loss, du, inv_nloc, rn);
}
cudaError_t sum_scaled(const float* v, int n, float scale, float* out, int* err, cudaStream_t st) {
  return launch_k(sum_scaled_kernel, 1, 1024, 0, st, v, n, scale, out, err);
}

cudaError_t sgd_momentum(float* w, const float* g, float* v, long long n, float lr, float mu, float wd, float s,
                         cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (!aligned16(w) || !aligned16(g) || !aligned16(v)) return cudaErrorMisalignedAddress;
  return launch_k(sgd_kernel, blocks_for(n / 4 + 1, 256), 256, 0, st, w, g, v, (float*)nullptr, 0LL, n,
                  (const float*)nullptr, 1.f, lr, mu, wd, s);
}
cudaError_t sgd_momentum_dev(float* w, const float* g, float* v, long long n, const float* lr_dev, float lr_scale,
                             float mu, float wd, float s, cudaStream_t st, float* wk, long long rn_end) {
  if (n <= 0) return cudaSuccess;
  if (!aligned16(w) || !aligned16(g) || !aligned16(v) || (wk && !aligned16(wk))) return cudaErrorMisalignedAddress;
  return launch_k(sgd_kernel, blocks_for(n / 4 + 1, 256), 256, 0, st, w, g, v, wk, rn_end, n, lr_dev, lr_scale, 0.f,
                  mu, wd, s);
}

cudaError_t adagrad(float* w, const float* g, float* h, long long n, float lr, float wd, float s, float eps,
                    cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_k(adagrad_kernel, blocks_for(n, 256), 256, 0, st, w, g, h, (float*)nullptr, 0LL, n,
                  (const float*)nullptr, 1.f, lr, wd, s, eps);
}
cudaError_t adagrad_dev(float* w, const float* g, float* h, long long n, const float* lr_dev, float lr_scale, float wd,
                        float s, float eps, cudaStream_t st, float* wk, long long rn_end) {
  if (n <= 0) return cudaSuccess;
  return launch_k(adagrad_kernel, blocks_for(n, 256), 256, 0, st, w, g, h, wk, rn_end, n, lr_dev, lr_scale, 0.f, wd,
                  s, eps);
}

cudaError_t pad_channels(const float* x, float* y, long long pixels, int cin, int cout, cudaStream_t st, int rn) {
  if (cout == 4 && !aligned16(y)) return cudaErrorMisalignedAddress;
  return launch_k(pad_channels_kernel, blocks_for(pixels, 256), 256, 0, st, x, y, pixels, cin, cout, rn);
}
cudaError_t copy2d(const float* src, long long sld, float* dst, long long dld, int rows, int cols, cudaStream_t st,
                   int rn) {
  return launch_k(copy2d_kernel, blocks_for((long long)rows * cols, 256), 256, 0, st, src, sld, dst, dld, rows, cols,
                  rn);
}
cudaError_t round_tf32(float* p, long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  return launch_k(round_tf32_kernel, blocks_for(n, 256), 256, 0, st, p, n);
}

}  // namespace sg

namespace sg {
namespace {
__global__ void fill_scalar_kernel(float* p, float v) { pdl_entry(); *p = v; }
}  // namespace
cudaError_t fill_scalar(float* p, float v, cudaStream_t st) {
  return launch_k(fill_scalar_kernel, 1, 1, 0, st, p, v);
}
}  // namespace sg
