// Strided first-layer convolution by space-to-depth (AlexNet conv1: 11x11,
// stride 4, 4 padded channels; PAPER.md P:752-753 workload, conv a3 / a15 of
// SURVEY §8(a)).
//
// With R' = ceil(R / st), the convolution
//   y[n][oh][ow][co] = sum_{r,s,c} W[co][r][s][c] x[n][st*oh + r - p][st*ow + s - p][c]
// equals a STRIDE-1, unpadded convolution with R' x S' taps over the
// space-to-depth image
//   xs[n][i][j][(dy*st + dx)*C + c] = x[n][st*i + dy - p][st*j + dx - p][c]   (0 outside)
// and the rearranged filter
//   Ws[co][r'][s'][(dy*st + dx)*C + c] = W[co][st*r' + dy][st*s' + dx][c]    (0 for taps >= R, S)
// (substitute r = st*r' + dy).  The extra taps multiply zeros, so the sum is
// the same up to the order of the fp32 additions.  The stride-1 form has
// st*st*C = 64 channels per pixel: TMA im2col boxes of 128 pixels x 32 channels
// instead of 16-byte gathers of the 4-channel image.  The weight gradient is
// formed on the same image (dWs) and folded back: dW[co][r][s][c] =
// dWs[co][r/st][s/st][((r%st)*st + s%st)*C + c].
#include "ops.h"
#include "sg_common.cuh"

namespace sg {

namespace {

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15) == 0; }
inline unsigned blocks_of(long long n, int per) {
  long long b = (n + per - 1) / per;
  if (b > 148LL * 32) b = 148LL * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

// thread per float4 of xs (4 channels of one sub-pixel (dy, dx))
__global__ void s2d_x_kernel(ConvShape s, int Hs, int Ws, const float* __restrict__ x, float* __restrict__ xs) {
  pdl_entry();
  const int C4 = s.C >> 2, sub = s.st * s.st * C4;
  const long long total = (long long)s.N * Hs * Ws * sub;
  for (long long o = blockIdx.x * (long long)blockDim.x + threadIdx.x; o < total;
       o += (long long)gridDim.x * blockDim.x) {
    const int q = (int)(o % sub);
    const long long pix = o / sub;
    const int j = (int)(pix % Ws);
    const long long t = pix / Ws;
    const int i = (int)(t % Hs), n = (int)(t / Hs);
    const int d = q / C4, c4 = q - d * C4;
    const int dy = d / s.st, dx = d - dy * s.st;
    const int h = s.st * i + dy - s.pad, w = s.st * j + dx - s.pad;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (h >= 0 && h < s.H && w >= 0 && w < s.W)
      v = __ldg(reinterpret_cast<const float4*>(x) + (((long long)n * s.H + h) * s.W + w) * C4 + c4);
    reinterpret_cast<float4*>(xs)[o] = v;
  }
}

// thread per element of Ws [Co][R'][S'][st*st*C]
__global__ void s2d_w_kernel(ConvShape s, int Rs, int Ss, const float* __restrict__ W, float* __restrict__ Wt) {
  pdl_entry();
  const int Cs = s.st * s.st * s.C;
  const int total = s.Co * Rs * Ss * Cs;
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
    const int cc = o % Cs, t = o / Cs;
    const int ss = t % Ss, t2 = t / Ss;
    const int rs = t2 % Rs, co = t2 / Rs;
    const int c = cc % s.C, d = cc / s.C, dy = d / s.st, dx = d - dy * s.st;
    const int r = s.st * rs + dy, sc = s.st * ss + dx;
    Wt[o] = (r < s.R && sc < s.S) ? __ldg(W + (((size_t)co * s.R + r) * s.S + sc) * s.C + c) : 0.f;
  }
}

// thread per element of dW [Co][R][S][C]
__global__ void s2d_dw_kernel(ConvShape s, int Rs, int Ss, const float* __restrict__ dWt, float* __restrict__ dW) {
  pdl_entry();
  const int Cs = s.st * s.st * s.C;
  const int total = s.Co * s.R * s.S * s.C;
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < total; o += gridDim.x * blockDim.x) {
    const int c = o % s.C, t = o / s.C;
    const int sc = t % s.S, t2 = t / s.S;
    const int r = t2 % s.R, co = t2 / s.R;
    const int cc = ((r % s.st) * s.st + sc % s.st) * s.C + c;
    dW[o] = __ldg(dWt + (((size_t)co * Rs + r / s.st) * Ss + sc / s.st) * Cs + cc);
  }
}

// The input layer's channel padding (3 -> 4, TF32-rounded when rn) writing the
// padded blob AND the space-to-depth image of the first convolution in one pass
// (thread per pixel; every pixel lands in exactly one sub-pixel slot of xs; the
// slots outside the image stay zero from the allocation).
__global__ void pad_s2d_kernel(ConvShape s, int Hs, int Ws, const float* __restrict__ x, int cin,
                               float* __restrict__ y, float* __restrict__ xs, int rn) {
  pdl_entry();
  const long long pixels = (long long)s.N * s.H * s.W;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < pixels;
       p += (long long)gridDim.x * blockDim.x) {
    const float* src = x + p * cin;
    float4 v = make_float4(src[0], cin > 1 ? src[1] : 0.f, cin > 2 ? src[2] : 0.f, cin > 3 ? src[3] : 0.f);
    v = tf32_rna4_if(v, rn);
    reinterpret_cast<float4*>(y)[p] = v;
    const int w = (int)(p % s.W);
    const long long t = p / s.W;
    const int h = (int)(t % s.H), n = (int)(t / s.H);
    const int hp = h + s.pad, wp = w + s.pad;
    const int i = hp / s.st, dy = hp - i * s.st, j = wp / s.st, dx = wp - j * s.st;
    if (i < Hs && j < Ws)
      reinterpret_cast<float4*>(xs)[(((long long)n * Hs + i) * Ws + j) * (s.st * s.st) + dy * s.st + dx] = v;
  }
}

}  // namespace

cudaError_t pad_channels_s2d(const float* x, int cin, float* y, float* xs, const ConvShape& s, cudaStream_t st,
                             int rn) {
  if (s.C != 4 || cin > 4 || !aligned16(y) || !aligned16(xs)) return cudaErrorInvalidValue;
  const ConvShape t = conv_s2d_shape(s);
  const long long pixels = (long long)s.N * s.H * s.W;
  return launch_k(pad_s2d_kernel, blocks_of(pixels, 256), 256, 0, st, s, t.H, t.W, x, cin, y, xs, rn);
}

bool conv_s2d_ok(const ConvShape& s) {
  static const int on = getenv("SG_S2D") ? atoi(getenv("SG_S2D")) : 1;
  return on && s.st > 1 && s.C % 4 == 0 && (s.st * s.st * s.C) % 32 == 0 && s.R >= s.st && s.S >= s.st;
}

ConvShape conv_s2d_shape(const ConvShape& s) {
  ConvShape t = s;
  const int Rs = (s.R + s.st - 1) / s.st, Ss = (s.S + s.st - 1) / s.st;
  t.H = s.Ho + Rs - 1;
  t.W = s.Wo + Ss - 1;
  t.C = s.st * s.st * s.C;
  t.R = Rs;
  t.S = Ss;
  t.st = 1;
  t.pad = 0;
  return t;
}

size_t conv_s2d_x_floats(const ConvShape& s) {
  const ConvShape t = conv_s2d_shape(s);
  return (size_t)t.N * t.H * t.W * t.C;
}
size_t conv_s2d_w_floats(const ConvShape& s) {
  const ConvShape t = conv_s2d_shape(s);
  return (size_t)t.Co * t.R * t.S * t.C;
}

cudaError_t conv_s2d_input(const ConvShape& s, const float* x, float* xs, cudaStream_t st) {
  const ConvShape t = conv_s2d_shape(s);
  const long long n4 = (long long)t.N * t.H * t.W * (t.C >> 2);
  return launch_k(s2d_x_kernel, blocks_of(n4, 256), 256, 0, st, s, t.H, t.W, x, xs);
}

cudaError_t conv_fwd_s2d(const ConvShape& s, const float* xs, const float* W, float* Wt, const float* b, float* y,
                         int flags, Workspace ws, cudaStream_t st) {
  const ConvShape t = conv_s2d_shape(s);
  const int nw = (int)conv_s2d_w_floats(s);
  cudaError_t e = launch_k(s2d_w_kernel, blocks_of(nw, 256), 256, 0, st, s, t.R, t.S, W, Wt);
  if (e != cudaSuccess) return e;
  return conv_fwd(t, xs, Wt, b, y, flags, ws, st);
}

cudaError_t conv_wgrad_s2d(const ConvShape& s, const float* xs, const float* dy, float* dWt, float* dW, float* db,
                           Workspace ws, cudaStream_t st) {
  const ConvShape t = conv_s2d_shape(s);
  cudaError_t e = conv_wgrad(t, xs, dy, dWt, db, ws, st);
  if (e != cudaSuccess) return e;
  const int n = s.Co * s.R * s.S * s.C;
  return launch_k(s2d_dw_kernel, blocks_of(n, 256), 256, 0, st, s, t.R, t.S, dWt, dW);
}

}  // namespace sg
