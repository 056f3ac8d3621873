// Device helpers shared by the layer kernels (ops_elt.cu) and the convolution
// kernels that fuse a following pooling / ReLU / LRN layer (conv_img.cu): ONE
// definition, so the fused and the separate kernels compute identical bits.
#pragma once
#include "ops.h"
#include "sg_common.cuh"

namespace sg {

// Optional ReLU fusion helpers (bit-identical to ReluF / ReluB).
__device__ __forceinline__ float4 relu4(float4 v) {
  return make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
}
__device__ __forceinline__ float4 mask4(float4 d, float4 y) {
  return make_float4(y.x > 0.f ? d.x : 0.f, y.y > 0.f ? d.y : 0.f, y.z > 0.f ? d.z : 0.f, y.w > 0.f ? d.w : 0.f);
}


// -------------------------------------------------------------------- LRN --
__device__ __forceinline__ float pow_neg(float base, float beta) { return exp2f(-beta * log2f(base)); }

// Thread per (pixel, 4 channels); the channel window reaches at most 4 channels
// into the neighbouring lanes' float4s (n <= 9), fetched with warp shuffles.
// Requires C % 4 == 0 and (C / 4) | 32, so a pixel's channels sit in one warp.
// Window sums run over ascending channels c' = c - n/2 ... c + n/2 (in range).
struct LrnK {
  LrnShape s;
  int C4, total;  // total = pixels * C4 rounded up to a multiple of 32
};

__device__ __forceinline__ void lrn_neighbours(float4 me, int c4, int C4, float (&e)[12]) {
  const float4 l = make_float4(__shfl_up_sync(0xffffffffu, me.x, 1), __shfl_up_sync(0xffffffffu, me.y, 1),
                               __shfl_up_sync(0xffffffffu, me.z, 1), __shfl_up_sync(0xffffffffu, me.w, 1));
  const float4 r = make_float4(__shfl_down_sync(0xffffffffu, me.x, 1), __shfl_down_sync(0xffffffffu, me.y, 1),
                               __shfl_down_sync(0xffffffffu, me.z, 1), __shfl_down_sync(0xffffffffu, me.w, 1));
  const bool hl = c4 > 0, hr = c4 < C4 - 1;
  e[0] = hl ? l.x : 0.f; e[1] = hl ? l.y : 0.f; e[2] = hl ? l.z : 0.f; e[3] = hl ? l.w : 0.f;
  e[4] = me.x; e[5] = me.y; e[6] = me.z; e[7] = me.w;
  e[8] = hr ? r.x : 0.f; e[9] = hr ? r.y : 0.f; e[10] = hr ? r.z : 0.f; e[11] = hr ? r.w : 0.f;
}

// LRN of the float4 v (channels 4*c4 .. 4*c4+3 of a pixel); every lane of the
// warp must call it (shuffles).
__device__ __forceinline__ void lrn_apply(const LrnShape& s, int C4, float4 v, int c4, float4& sc4, float4& o4) {
  const int half = s.n / 2;
  const float an = s.alpha / (float)s.n;
  float e[12];
  lrn_neighbours(make_float4(v.x * v.x, v.y * v.y, v.z * v.z, v.w * v.w), c4, C4, e);
  float sc[4], o[4];
  const float xv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float acc = 0.f;
    // ascending d over the window (half <= 4): compile-time indices keep e[] in registers
#pragma unroll
    for (int d = -4; d <= 4; ++d)
      if (d >= -half && d <= half) acc += e[4 + j + d];
    sc[j] = s.k + an * acc;
    o[j] = xv[j] * pow_neg(sc[j], s.beta);
  }
  sc4 = make_float4(sc[0], sc[1], sc[2], sc[3]);
  o4 = make_float4(o[0], o[1], o[2], o[3]);
}


// LRN backward of one channel (reading A6; a12): t = g*y/s of the window's
// channels, o = g*s^-beta - coef*x*sum(t), coef = 2*alpha*beta/n.  Explicit
// round-to-nearest intrinsics (no FMA contraction), so the separate kernel and
// the convolution epilogue that fuses it produce identical bits.
__device__ __forceinline__ float lrn_bwd_t(float g, float y, float s) { return __fdiv_rn(__fmul_rn(g, y), s); }
__device__ __forceinline__ float lrn_bwd_out(float g, float s, float x, float acc, float beta, float coef) {
  return __fsub_rn(__fmul_rn(g, pow_neg(s, beta)), __fmul_rn(__fmul_rn(coef, x), acc));
}

// ---------------------------------------------------------------- Updater --
// g' = s g + wd w ; v = mu v - lr g' ; w = w + v ; fixed FMA order.
__device__ __forceinline__ void sgd1(float& w, float g, float& v, float lr, float mu, float wd, float s) {
  float gp = __fmaf_rn(wd, w, __fmul_rn(s, g));
  v = __fmaf_rn(mu, v, -__fmul_rn(lr, gp));
  w = __fadd_rn(w, v);
}

// AdaGrad (reading A26), same working-copy convention as the SGD update.
__device__ __forceinline__ void adagrad1(float& w, float g, float& h, float lr, float wd, float s, float eps) {
  const float gp = __fmaf_rn(wd, w, __fmul_rn(s, g));
  h = __fmaf_rn(gp, gp, h);
  w = __fsub_rn(w, __fdiv_rn(__fmul_rn(lr, gp), __fadd_rn(__fsqrt_rn(h), eps)));
}


// A weight-gradient reduction that also applies the Updater to the elements it
// produced (first layer at K = 1: its Update is the step's last operation).
struct FusedUpdate {
  float* w;    // fp32 master of dW's elements (then the bias part: wb)
  float* v;    // history
  float* wk;   // TF32-RN working copy (weights), exact copy (bias)
  float* wb;
  float* vb;
  float* wkb;
  const float* lr_dev;
  float lr_scale, mu, wd, s, eps;
  int type;    // 0 SGD momentum, 1 AdaGrad
};
__device__ __forceinline__ void fused_update1(const FusedUpdate& u, float* w, float* v, float* wk, long long i, float g,
                                              bool rn) {
  const float lr = u.lr_dev[0] * u.lr_scale;
  float ww = w[i], vv = v[i];
  if (u.type == 0)
    sgd1(ww, g, vv, lr, u.mu, u.wd, u.s);
  else
    adagrad1(ww, g, vv, lr, u.wd, u.s, u.eps);
  w[i] = ww;
  v[i] = vv;
  wk[i] = rn ? tf32_rna(ww) : ww;
}

}  // namespace sg
