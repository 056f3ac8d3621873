// HBM-bound layer kernels: ReLU / sigmoid (P:241 logistic), pooling (P:553,
// Caffe geometry P:658-659), LRN across channels, softmax
// cross-entropy and Euclidean losses, the fused
// SGD-momentum Updater and the input layer's channel padding.
// Readings A5-A8 of DESIGN.md fix the definitions left open by the paper.
// All reductions run in a fixed order (bit-reproducible).
#include <cstdint>

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
__global__ void map1_kernel(const float* __restrict__ x, float* __restrict__ y, long long n, F f) {
  pdl_entry();
  long long n4 = n >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  float4* y4 = reinterpret_cast<float4*>(y);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 v = x4[i];
    y4[i] = make_float4(f(v.x), f(v.y), f(v.z), f(v.w));
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = f(x[i]);
}

template <class F>
__global__ void map2_kernel(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ y,
                            long long n, F f) {
  pdl_entry();
  long long n4 = n >> 2;
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* y4 = reinterpret_cast<float4*>(y);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 u = a4[i], v = b4[i];
    y4[i] = make_float4(f(u.x, v.x), f(u.y, v.y), f(u.z, v.z), f(u.w, v.w));
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    y[i] = f(a[i], b[i]);
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
cudaError_t launch_map1(const float* x, float* y, long long n, F f, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (!aligned16(x) || !aligned16(y)) return cudaErrorMisalignedAddress;
  return launch_k(map1_kernel<F>, blocks_for(n / 4 + 1, 256), 256, 0, st, x, y, n, f);
}
template <class F>
cudaError_t launch_map2(const float* a, const float* b, float* y, long long n, F f, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (!aligned16(a) || !aligned16(b) || !aligned16(y)) return cudaErrorMisalignedAddress;
  return launch_k(map2_kernel<F>, blocks_for(n / 4 + 1, 256), 256, 0, st, a, b, y, n, f);
}

// ---------------------------------------------------------------- pooling --
// Thread per (n, oh, ow, 4 channels).  Window origin (oh*s - p, ow*s - p);
// the argmax is stored as the uint8 offset (h - h0)*k + (w - w0).
__global__ void maxpool_fwd_kernel(PoolShape s, const float* __restrict__ x, float* __restrict__ y,
                                   uint8_t* __restrict__ arg) {
  pdl_entry();
  const int C4 = s.C >> 2;
  long long total = (long long)s.N * s.Ho * s.Wo * C4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c4 = (int)(i % C4);
    long long t = i / C4;
    int ow = (int)(t % s.Wo);
    t /= s.Wo;
    int oh = (int)(t % s.Ho);
    int n = (int)(t / s.Ho);
    int h0 = oh * s.s - s.p, w0 = ow * s.s - s.p;
    int hs = max(h0, 0), he = min(h0 + s.k, s.H), ws = max(w0, 0), we = min(w0 + s.k, s.W);
    float m[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int a[4] = {0, 0, 0, 0};
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w) {
        float4 v = *reinterpret_cast<const float4*>(x + (((long long)n * s.H + h) * s.W + w) * s.C + c4 * 4);
        int off = (h - h0) * s.k + (w - w0);
        if (v.x > m[0]) { m[0] = v.x; a[0] = off; }
        if (v.y > m[1]) { m[1] = v.y; a[1] = off; }
        if (v.z > m[2]) { m[2] = v.z; a[2] = off; }
        if (v.w > m[3]) { m[3] = v.w; a[3] = off; }
      }
    long long o = i * 4;
    *reinterpret_cast<float4*>(y + o) = make_float4(m[0], m[1], m[2], m[3]);
    *reinterpret_cast<uchar4*>(arg + o) = make_uchar4(a[0], a[1], a[2], a[3]);
  }
}

// Gather form of the backward: thread per input (n, h, w, 4 channels) sums dy
// of every window whose argmax is this element, windows in ascending (oh, ow).
__global__ void maxpool_bwd_kernel(PoolShape s, const float* __restrict__ dy, const uint8_t* __restrict__ arg,
                                   float* __restrict__ dx) {
  pdl_entry();
  const int C4 = s.C >> 2;
  long long total = (long long)s.N * s.H * s.W * C4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c4 = (int)(i % C4);
    long long t = i / C4;
    int w = (int)(t % s.W);
    t /= s.W;
    int h = (int)(t % s.H);
    int n = (int)(t / s.H);
    // windows containing h: oh*s - p <= h < oh*s - p + k
    int hp = h + s.p, wp = w + s.p;
    int oh0 = hp >= s.k ? (hp - s.k) / s.s + 1 : 0, oh1 = min(hp / s.s, s.Ho - 1);
    int ow0 = wp >= s.k ? (wp - s.k) / s.s + 1 : 0, ow1 = min(wp / s.s, s.Wo - 1);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int oh = oh0; oh <= oh1; ++oh)
      for (int ow = ow0; ow <= ow1; ++ow) {
        int off = (hp - oh * s.s) * s.k + (wp - ow * s.s);
        long long o = (((long long)n * s.Ho + oh) * s.Wo + ow) * s.C + c4 * 4;
        uchar4 a = *reinterpret_cast<const uchar4*>(arg + o);
        float4 g = *reinterpret_cast<const float4*>(dy + o);
        if (a.x == off) acc[0] += g.x;
        if (a.y == off) acc[1] += g.y;
        if (a.z == off) acc[2] += g.z;
        if (a.w == off) acc[3] += g.w;
      }
    *reinterpret_cast<float4*>(dx + i * 4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
  }
}

__global__ void avgpool_fwd_kernel(PoolShape s, const float* __restrict__ x, float* __restrict__ y) {
  pdl_entry();
  const int C4 = s.C >> 2;
  long long total = (long long)s.N * s.Ho * s.Wo * C4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c4 = (int)(i % C4);
    long long t = i / C4;
    int ow = (int)(t % s.Wo);
    t /= s.Wo;
    int oh = (int)(t % s.Ho);
    int n = (int)(t / s.Ho);
    int h0 = oh * s.s - s.p, w0 = ow * s.s - s.p;
    int he_u = min(h0 + s.k, s.H + s.p), we_u = min(w0 + s.k, s.W + s.p);
    float inv = 1.f / (float)((he_u - h0) * (we_u - w0));
    int hs = max(h0, 0), he = min(he_u, s.H), ws = max(w0, 0), we = min(we_u, s.W);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int h = hs; h < he; ++h)
      for (int w = ws; w < we; ++w) {
        float4 v = *reinterpret_cast<const float4*>(x + (((long long)n * s.H + h) * s.W + w) * s.C + c4 * 4);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    *reinterpret_cast<float4*>(y + i * 4) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  }
}

__global__ void avgpool_bwd_kernel(PoolShape s, const float* __restrict__ dy, float* __restrict__ dx) {
  pdl_entry();
  const int C4 = s.C >> 2;
  long long total = (long long)s.N * s.H * s.W * C4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int c4 = (int)(i % C4);
    long long t = i / C4;
    int w = (int)(t % s.W);
    t /= s.W;
    int h = (int)(t % s.H);
    int n = (int)(t / s.H);
    int hp = h + s.p, wp = w + s.p;
    int oh0 = hp >= s.k ? (hp - s.k) / s.s + 1 : 0, oh1 = min(hp / s.s, s.Ho - 1);
    int ow0 = wp >= s.k ? (wp - s.k) / s.s + 1 : 0, ow1 = min(wp / s.s, s.Wo - 1);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int oh = oh0; oh <= oh1; ++oh) {
      int h0 = oh * s.s - s.p;
      int hsz = min(h0 + s.k, s.H + s.p) - h0;
      for (int ow = ow0; ow <= ow1; ++ow) {
        int w0 = ow * s.s - s.p;
        int wsz = min(w0 + s.k, s.W + s.p) - w0;
        float inv = 1.f / (float)(hsz * wsz);
        float4 g = *reinterpret_cast<const float4*>(dy + (((long long)n * s.Ho + oh) * s.Wo + ow) * s.C + c4 * 4);
        acc.x += g.x * inv; acc.y += g.y * inv; acc.z += g.z * inv; acc.w += g.w * inv;
      }
    }
    *reinterpret_cast<float4*>(dx + i * 4) = acc;
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
__device__ __forceinline__ float pow_neg(float base, float beta) { return exp2f(-beta * log2f(base)); }

__global__ void lrn_fwd_kernel(LrnShape s, const float* __restrict__ x, float* __restrict__ y,
                               float* __restrict__ scale) {
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
    y[i] = x[i] * pow_neg(sc, s.beta);
  }
}

__global__ void lrn_bwd_kernel(LrnShape s, const float* __restrict__ x, const float* __restrict__ y,
                               const float* __restrict__ scale, const float* __restrict__ dy, float* __restrict__ dx) {
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
    dx[i] = dy[i] * pow_neg(scale[i], s.beta) - coef * x[i] * acc;
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
                                  View2D dz, float inv_nloc, int* err) {
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
      *vat_w(dz, r, j) = (p - (j == y ? 1.f : 0.f)) * inv_nloc;
    }
    if (lane == 0) row_loss[r] = bad ? 0.f : (m + logf(sum)) - *vat(z, r, y);
  }
}

__global__ void euclidean_kernel(View2D u, View2D v, float* __restrict__ row_loss, View2D du, float inv_nloc) {
  pdl_entry();
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * warps + (threadIdx.x >> 5); r < u.rows; r += gridDim.x * warps) {
    float acc = 0.f;
    for (int j = lane; j < u.cols; j += 32) {
      float d = *vat(u, r, j) - *vat(v, r, j);
      acc += d * d;
      *vat_w(du, r, j) = d * inv_nloc;
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
// g' = s g + wd w ; v = mu v - lr g' ; w = w + v ; fixed FMA order.
__device__ __forceinline__ void sgd1(float& w, float g, float& v, float lr, float mu, float wd, float s) {
  float gp = __fmaf_rn(wd, w, __fmul_rn(s, g));
  v = __fmaf_rn(mu, v, -__fmul_rn(lr, gp));
  w = __fadd_rn(w, v);
}

__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ v, long long n,
                           const float* lr_dev, float lr_scale, float lr_val, float mu, float wd, float s) {
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
  }
  for (long long i = (n4 << 2) + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float ww = w[i], vv = v[i];
    sgd1(ww, g[i], vv, lr, mu, wd, s);
    w[i] = ww;
    v[i] = vv;
  }
}

// ------------------------------------------------------------- input layer --
__global__ void pad_channels_kernel(const float* __restrict__ x, float* __restrict__ y, long long pixels, int cin,
                                    int cout) {
  pdl_entry();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < pixels * cout;
       i += (long long)gridDim.x * blockDim.x) {
    long long p = i / cout;
    int c = (int)(i - p * cout);
    y[i] = c < cin ? x[p * cin + c] : 0.f;
  }
}

__global__ void copy2d_kernel(const float* __restrict__ src, long long sld, float* __restrict__ dst, long long dld,
                              int rows, int cols) {
  pdl_entry();
  long long total = (long long)rows * cols;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int r = (int)(i / cols), c = (int)(i % cols);
    dst[(long long)r * dld + c] = src[(long long)r * sld + c];
  }
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

cudaError_t relu_fwd(const float* x, float* y, long long n, cudaStream_t st) { return launch_map1(x, y, n, ReluF{}, st); }
cudaError_t relu_bwd(const float* y, const float* dy, float* dx, long long n, cudaStream_t st) {
  return launch_map2(y, dy, dx, n, ReluB{}, st);
}
cudaError_t sigmoid_fwd(const float* x, float* y, long long n, cudaStream_t st) { return launch_map1(x, y, n, SigF{}, st); }
cudaError_t sigmoid_bwd(const float* y, const float* dy, float* dx, long long n, cudaStream_t st) {
  return launch_map2(y, dy, dx, n, SigB{}, st);
}
cudaError_t relu_fwd2d(const float* x, float* y, int rows, int cols, long long ld, cudaStream_t st) {
  return launch_k(relu2d_kernel, blocks_for((long long)rows * cols, 256), 256, 0, st, x, y, rows, cols, ld);
}

cudaError_t maxpool_fwd(const PoolShape& s, const float* x, float* y, uint8_t* arg, cudaStream_t st) {
  if (s.C % 4 || s.k * s.k > 256) return cudaErrorInvalidValue;
  return launch_k(maxpool_fwd_kernel, blocks_for((long long)s.N * s.Ho * s.Wo * s.C / 4, 256), 256, 0, st, s, x, y, arg);
}
cudaError_t maxpool_bwd(const PoolShape& s, const float* dy, const uint8_t* arg, float* dx, cudaStream_t st) {
  if (s.C % 4) return cudaErrorInvalidValue;
  return launch_k(maxpool_bwd_kernel, blocks_for((long long)s.N * s.H * s.W * s.C / 4, 256), 256, 0, st, s, dy, arg, dx);
}
cudaError_t avgpool_fwd(const PoolShape& s, const float* x, float* y, cudaStream_t st) {
  if (s.C % 4) return cudaErrorInvalidValue;
  return launch_k(avgpool_fwd_kernel, blocks_for((long long)s.N * s.Ho * s.Wo * s.C / 4, 256), 256, 0, st, s, x, y);
}
cudaError_t avgpool_bwd(const PoolShape& s, const float* dy, float* dx, cudaStream_t st) {
  if (s.C % 4) return cudaErrorInvalidValue;
  return launch_k(avgpool_bwd_kernel, blocks_for((long long)s.N * s.H * s.W * s.C / 4, 256), 256, 0, st, s, dy, dx);
}
cudaError_t pool_argmax_expand(const PoolShape& s, const uint8_t* arg, int32_t* out, cudaStream_t st) {
  return launch_k(argmax_expand_kernel, blocks_for((long long)s.N * s.Ho * s.Wo * s.C, 256), 256, 0, st, s, arg, out);
}

cudaError_t lrn_fwd(const LrnShape& s, const float* x, float* y, float* scale, cudaStream_t st) {
  return launch_k(lrn_fwd_kernel, blocks_for(s.pixels * s.C, 256), 256, 0, st, s, x, y, scale);
}
cudaError_t lrn_bwd(const LrnShape& s, const float* x, const float* y, const float* scale, const float* dy, float* dx,
                    cudaStream_t st) {
  return launch_k(lrn_bwd_kernel, blocks_for(s.pixels * s.C, 256), 256, 0, st, s, x, y, scale, dy, dx);
}

cudaError_t softmax_ce(View2D z, const int32_t* labels, float* row_loss, View2D dz, float inv_nloc, int* err,
                       cudaStream_t st) {
  if (z.rows <= 0) return cudaSuccess;
  return launch_k(softmax_ce_kernel, (z.rows + 7) / 8, 256, 0, st, z, labels, row_loss, dz, inv_nloc, err);
}
cudaError_t euclidean(View2D u, View2D v, float* row_loss, View2D du, float inv_nloc, cudaStream_t st) {
  if (u.rows <= 0) return cudaSuccess;
  return launch_k(euclidean_kernel, (u.rows + 7) / 8, 256, 0, st, u, v, row_loss, du, inv_nloc);
}
cudaError_t sum_scaled(const float* v, int n, float scale, float* out, int* err, cudaStream_t st) {
  return launch_k(sum_scaled_kernel, 1, 1024, 0, st, v, n, scale, out, err);
}

cudaError_t sgd_momentum(float* w, const float* g, float* v, long long n, float lr, float mu, float wd, float s,
                         cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (!aligned16(w) || !aligned16(g) || !aligned16(v)) return cudaErrorMisalignedAddress;
  return launch_k(sgd_kernel, blocks_for(n / 4 + 1, 256), 256, 0, st, w, g, v, n, nullptr, 1.f, lr, mu, wd, s);
}
cudaError_t sgd_momentum_dev(float* w, const float* g, float* v, long long n, const float* lr_dev, float lr_scale,
                             float mu, float wd, float s, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (!aligned16(w) || !aligned16(g) || !aligned16(v)) return cudaErrorMisalignedAddress;
  return launch_k(sgd_kernel, blocks_for(n / 4 + 1, 256), 256, 0, st, w, g, v, n, lr_dev, lr_scale, 0.f, mu, wd, s);
}

cudaError_t pad_channels(const float* x, float* y, long long pixels, int cin, int cout, cudaStream_t st) {
  return launch_k(pad_channels_kernel, blocks_for(pixels * cout, 256), 256, 0, st, x, y, pixels, cin, cout);
}
cudaError_t copy2d(const float* src, long long sld, float* dst, long long dld, int rows, int cols, cudaStream_t st) {
  return launch_k(copy2d_kernel, blocks_for((long long)rows * cols, 256), 256, 0, st, src, sld, dst, dld, rows, cols);
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
