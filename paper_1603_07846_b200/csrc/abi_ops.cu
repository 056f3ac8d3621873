// extern "C" entry points: errors, partition map and the layer-isolated
// operations of include/singa_b200.h (argument checking + launch only).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "abi_common.h"
#include "ops.h"

namespace sg {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}
const char* get_error() { return g_err.c_str(); }

// Per-device scratch for the op-level API (grown on demand; never shrinks).
static std::mutex g_ws_mu;
static std::vector<Workspace> g_ws;

static sg_status op_workspace(size_t floats, Workspace* out) {
  int dev = 0;
  SG_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_ws_mu);
  if ((int)g_ws.size() <= dev) g_ws.resize(dev + 1);
  Workspace& w = g_ws[dev];
  if (w.floats < floats) {
    if (w.ptr) {
      SG_CUDA(cudaDeviceSynchronize());
      SG_CUDA(cudaFree(w.ptr));
      w.ptr = nullptr;
      w.floats = 0;
    }
    size_t n = floats < ((size_t)1 << 20) ? ((size_t)1 << 20) : floats;
    cudaError_t e = cudaMalloc(&w.ptr, n * sizeof(float));
    if (e != cudaSuccess) SG_FAIL(SG_ERR_OOM, "workspace allocation of %zu floats failed", n);
    SG_CUDA(cudaMemset(w.ptr, 0, 4096));  // split-K tile counters live at the head
    w.floats = n;
  }
  *out = w;
  return SG_OK;
}

size_t colsum_ws_floats(int M, int N);

}  // namespace sg

using namespace sg;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define SG_LAUNCH(expr)                                                                                   \
  do {                                                                                                    \
    cudaError_t _e = (expr);                                                                              \
    if (_e != cudaSuccess) SG_FAIL(SG_ERR_CUDA, "%s: launch failed: %s", __func__, cudaGetErrorString(_e)); \
  } while (0)

extern "C" {

SG_API const char* sg_last_error(void) { return get_error(); }
SG_API int32_t sg_abi_version(void) { return SG_ABI_VERSION; }

SG_API sg_status sg_partition_range(int64_t extent, int32_t parts, int32_t idx, int64_t* off, int64_t* len) {
  SG_CHECK(off && len, SG_ERR_INVALID_ARG, "sg_partition_range: null output");
  SG_CHECK(parts >= 1 && idx >= 0 && idx < parts, SG_ERR_INVALID_ARG, "sg_partition_range: parts=%d idx=%d", parts,
           idx);
  SG_CHECK(extent >= parts, SG_ERR_PARTITION, "partition error: %d parts > extent %lld", parts, (long long)extent);
  const int64_t base = extent / parts, rem = extent % parts;
  *len = base + (idx < rem ? 1 : 0);
  *off = (int64_t)idx * base + (idx < rem ? idx : rem);
  return SG_OK;
}

SG_API sg_status sg_op_gemm(const float* A, int32_t ta, const float* B, int32_t tb, float* C, int32_t M, int32_t N,
                            int32_t K, void* stream) {
  SG_CHECK(A && B && C, SG_ERR_INVALID_ARG, "sg_op_gemm: null pointer");
  SG_CHECK(M > 0 && N > 0 && K > 0, SG_ERR_DIMENSION, "sg_op_gemm: M=%d N=%d K=%d", M, N, K);
  SG_CHECK(((ta ? M : K) % 4 == 0) && ((tb ? K : N) % 4 == 0), SG_ERR_DIMENSION,
           "sg_op_gemm: leading dimensions must be multiples of 4 (M=%d N=%d K=%d ta=%d tb=%d)", M, N, K, ta, tb);
  Workspace ws;
  SG_TRY(op_workspace(gemm_ws_floats(M, N, K), &ws));
  SG_LAUNCH(gemm_plain(A, ta, B, tb, C, M, N, K, ws, S(stream)));
  return SG_OK;
}

static sg_status conv_shape(const sg_conv_desc* d, ConvShape* s) {
  SG_CHECK(d, SG_ERR_INVALID_ARG, "null conv desc");
  SG_CHECK(d->N > 0 && d->H > 0 && d->W > 0 && d->C > 0 && d->Co > 0 && d->R > 0 && d->S > 0 && d->stride > 0 &&
               d->pad >= 0,
           SG_ERR_DIMENSION, "conv: bad shape N=%d H=%d W=%d C=%d Co=%d R=%d S=%d stride=%d pad=%d", d->N, d->H,
           d->W, d->C, d->Co, d->R, d->S, d->stride, d->pad);
  SG_CHECK(d->C % 4 == 0 && d->Co % 4 == 0, SG_ERR_DIMENSION,
           "conv: Cin (%d) and Cout (%d) must be multiples of 4 (pad the input channels)", d->C, d->Co);
  int Ho = (d->H + 2 * d->pad - d->R) / d->stride + 1, Wo = (d->W + 2 * d->pad - d->S) / d->stride + 1;
  SG_CHECK(Ho > 0 && Wo > 0, SG_ERR_DIMENSION, "conv: empty output (%dx%d)", Ho, Wo);
  *s = ConvShape{d->N, d->H, d->W, d->C, d->Co, d->R, d->S, d->stride, d->pad, Ho, Wo};
  return SG_OK;
}

SG_API sg_status sg_conv_out_shape(const sg_conv_desc* d, int32_t* Ho, int32_t* Wo) {
  ConvShape s;
  SG_TRY(conv_shape(d, &s));
  SG_CHECK(Ho && Wo, SG_ERR_INVALID_ARG, "null output");
  *Ho = s.Ho;
  *Wo = s.Wo;
  return SG_OK;
}

SG_API sg_status sg_op_conv_forward(const sg_conv_desc* d, const float* x, const float* W, const float* b, float* y,
                                    void* stream) {
  ConvShape s;
  SG_TRY(conv_shape(d, &s));
  SG_CHECK(x && W && y, SG_ERR_INVALID_ARG, "conv forward: null pointer");
  Workspace ws;
  SG_TRY(op_workspace(gemm_ws_floats(s.N * s.Ho * s.Wo, s.Co, s.R * s.S * s.C), &ws));
  SG_LAUNCH(conv_fwd(s, x, W, b, y, 0, ws, S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_conv_backward(const sg_conv_desc* d, const float* x, const float* W, const float* dy,
                                     float* dx, float* dW, float* db, void* stream) {
  ConvShape s;
  SG_TRY(conv_shape(d, &s));
  SG_CHECK(x && W && dy && dW, SG_ERR_INVALID_ARG, "conv backward: null pointer");
  const int Mtot = s.N * s.Ho * s.Wo;
  size_t need = gemm_ws_floats(s.R * s.S * s.C, s.Co, Mtot);
  size_t cs = colsum_ws_floats(Mtot, s.Co);
  if (cs > need) need = cs;
  need = std::max(need, conv_img_wgrad_ws_floats(s));
  if (dx) {
    size_t dn = gemm_ws_floats(s.N * s.H * s.W, s.C, s.R * s.S * s.Co);
    if (dn > need) need = dn;
  }
  Workspace ws;
  SG_TRY(op_workspace(need, &ws));
  SG_LAUNCH(conv_wgrad(s, x, dy, dW, db, ws, S(stream)));
  if (dx) SG_LAUNCH(conv_dgrad(s, dy, W, dx, ws, S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_ip_forward(const float* x, const float* W, const float* b, float* y, int32_t rows, int32_t dv,
                                  int32_t dh, void* stream) {
  SG_CHECK(x && W && y, SG_ERR_INVALID_ARG, "ip forward: null pointer");
  SG_CHECK(rows > 0 && dv > 0 && dh > 0, SG_ERR_DIMENSION, "ip forward: rows=%d dv=%d dh=%d", rows, dv, dh);
  SG_CHECK(dv % 4 == 0 && dh % 4 == 0, SG_ERR_DIMENSION, "ip: d_v (%d) and d_h (%d) must be multiples of 4", dv, dh);
  Workspace ws;
  SG_TRY(op_workspace(gemm_ws_floats(rows, dh, dv), &ws));
  SG_LAUNCH(ip_fwd(plain(const_cast<float*>(x), rows, dv), W, dv, dh, b, plain(y, rows, dh), 0, ws, S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_ip_backward(const float* x, const float* W, const float* dy, float* dx, float* dW, float* db,
                                   int32_t rows, int32_t dv, int32_t dh, void* stream) {
  SG_CHECK(x && W && dy && dW, SG_ERR_INVALID_ARG, "ip backward: null pointer");
  SG_CHECK(rows > 0 && dv > 0 && dh > 0, SG_ERR_DIMENSION, "ip backward: rows=%d dv=%d dh=%d", rows, dv, dh);
  SG_CHECK(dv % 4 == 0 && dh % 4 == 0 && rows % 4 == 0, SG_ERR_DIMENSION,
           "ip backward: rows (%d), d_v (%d), d_h (%d) must be multiples of 4", rows, dv, dh);
  size_t need = gemm_ws_floats(dv, dh, rows);
  size_t a = gemm_ws_floats(rows, dv, dh), c = colsum_ws_floats(rows, dh);
  if (a > need) need = a;
  if (c > need) need = c;
  Workspace ws;
  SG_TRY(op_workspace(need, &ws));
  View2D xv = plain(const_cast<float*>(x), rows, dv), dyv = plain(const_cast<float*>(dy), rows, dh);
  SG_LAUNCH(ip_wgrad(xv, dyv, dv, dh, dW, db, ws, S(stream)));
  if (dx) SG_LAUNCH(ip_dgrad(dyv, W, dv, dh, plain(dx, rows, dv), ws, S(stream)));
  return SG_OK;
}

static sg_status pool_shape(const sg_pool_desc* d, PoolShape* s) {
  SG_CHECK(d, SG_ERR_INVALID_ARG, "null pool desc");
  SG_CHECK(d->N > 0 && d->H > 0 && d->W > 0 && d->C > 0 && d->kernel > 0 && d->stride > 0 && d->pad >= 0 &&
               d->pad < d->kernel && (d->mode == 0 || d->mode == 1),
           SG_ERR_DIMENSION, "pool: bad shape N=%d H=%d W=%d C=%d k=%d s=%d p=%d mode=%d", d->N, d->H, d->W, d->C,
           d->kernel, d->stride, d->pad, d->mode);
  SG_CHECK(d->C % 4 == 0, SG_ERR_DIMENSION, "pool: C (%d) must be a multiple of 4", d->C);
  SG_CHECK(d->kernel <= 16, SG_ERR_DIMENSION, "pool: kernel %d > 16", d->kernel);
  auto osz = [&](int h) {
    int ho = (h + 2 * d->pad - d->kernel + d->stride - 1) / d->stride + 1;  // ceil
    if (d->pad > 0 && (ho - 1) * d->stride >= h + d->pad) --ho;
    return ho;
  };
  SG_CHECK(d->H + 2 * d->pad >= d->kernel && d->W + 2 * d->pad >= d->kernel, SG_ERR_DIMENSION,
           "pool: window %d larger than padded input %dx%d", d->kernel, d->H, d->W);
  *s = PoolShape{d->N, d->H, d->W, d->C, d->kernel, d->stride, d->pad, osz(d->H), osz(d->W)};
  return SG_OK;
}

SG_API sg_status sg_pool_out_shape(const sg_pool_desc* d, int32_t* Ho, int32_t* Wo) {
  PoolShape s;
  SG_TRY(pool_shape(d, &s));
  SG_CHECK(Ho && Wo, SG_ERR_INVALID_ARG, "null output");
  *Ho = s.Ho;
  *Wo = s.Wo;
  return SG_OK;
}

SG_API sg_status sg_op_pool_forward(const sg_pool_desc* d, const float* x, float* y, uint8_t* mask, void* stream) {
  PoolShape s;
  SG_TRY(pool_shape(d, &s));
  SG_CHECK(x && y && (d->mode == 1 || mask), SG_ERR_INVALID_ARG, "pool forward: null pointer");
  if (d->mode == 0)
    SG_LAUNCH(maxpool_fwd(s, x, y, mask, S(stream)));
  else
    SG_LAUNCH(avgpool_fwd(s, x, y, S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_pool_backward(const sg_pool_desc* d, const float* dy, const uint8_t* mask, float* dx,
                                     void* stream) {
  PoolShape s;
  SG_TRY(pool_shape(d, &s));
  SG_CHECK(dy && dx && (d->mode == 1 || mask), SG_ERR_INVALID_ARG, "pool backward: null pointer");
  if (d->mode == 0)
    SG_LAUNCH(maxpool_bwd(s, dy, mask, dx, S(stream)));
  else
    SG_LAUNCH(avgpool_bwd(s, dy, dx, S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_pool_argmax(const sg_pool_desc* d, const uint8_t* mask, int32_t* argmax, void* stream) {
  PoolShape s;
  SG_TRY(pool_shape(d, &s));
  SG_CHECK(mask && argmax && d->mode == 0, SG_ERR_INVALID_ARG, "pool argmax: null pointer or avg pool");
  SG_LAUNCH(pool_argmax_expand(s, mask, argmax, S(stream)));
  return SG_OK;
}

static sg_status lrn_shape(const sg_lrn_desc* d, LrnShape* s) {
  SG_CHECK(d, SG_ERR_INVALID_ARG, "null lrn desc");
  SG_CHECK(d->pixels > 0 && d->C > 0 && d->size > 0 && d->size % 2 == 1 && d->k > 0.f, SG_ERR_DIMENSION,
           "lrn: pixels=%lld C=%d size=%d k=%g (size must be odd, k > 0)", (long long)d->pixels, d->C, d->size,
           (double)d->k);
  *s = LrnShape{d->pixels, d->C, d->size, d->alpha, d->beta, d->k};
  return SG_OK;
}

SG_API sg_status sg_op_lrn_forward(const sg_lrn_desc* d, const float* x, float* y, float* scale, void* stream) {
  LrnShape s;
  SG_TRY(lrn_shape(d, &s));
  SG_CHECK(x && y && scale, SG_ERR_INVALID_ARG, "lrn forward: null pointer");
  SG_LAUNCH(lrn_fwd(s, x, y, scale, S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_lrn_backward(const sg_lrn_desc* d, const float* x, const float* y, const float* scale,
                                    const float* dy, float* dx, void* stream) {
  LrnShape s;
  SG_TRY(lrn_shape(d, &s));
  SG_CHECK(x && y && scale && dy && dx, SG_ERR_INVALID_ARG, "lrn backward: null pointer");
  SG_LAUNCH(lrn_bwd(s, x, y, scale, dy, dx, S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_neuron_forward(int32_t kind, const float* x, float* y, int64_t n, void* stream) {
  SG_CHECK(x && y && n >= 0, SG_ERR_INVALID_ARG, "neuron forward: bad argument");
  if (kind == SG_RELU)
    SG_LAUNCH(relu_fwd(x, y, n, S(stream)));
  else if (kind == SG_SIGMOID)
    SG_LAUNCH(sigmoid_fwd(x, y, n, S(stream)));
  else
    SG_FAIL(SG_ERR_INVALID_ARG, "neuron forward: kind %d is not SG_RELU / SG_SIGMOID", kind);
  return SG_OK;
}

SG_API sg_status sg_op_neuron_backward(int32_t kind, const float* y, const float* dy, float* dx, int64_t n,
                                       void* stream) {
  SG_CHECK(y && dy && dx && n >= 0, SG_ERR_INVALID_ARG, "neuron backward: bad argument");
  if (kind == SG_RELU)
    SG_LAUNCH(relu_bwd(y, dy, dx, n, S(stream)));
  else if (kind == SG_SIGMOID)
    SG_LAUNCH(sigmoid_bwd(y, dy, dx, n, S(stream)));
  else
    SG_FAIL(SG_ERR_INVALID_ARG, "neuron backward: kind %d is not SG_RELU / SG_SIGMOID", kind);
  return SG_OK;
}

SG_API sg_status sg_op_softmax_ce(const float* z, const int32_t* labels, int32_t rows, int32_t C, int32_t n_loc,
                                  float* row_loss, float* dz, int32_t* err, void* stream) {
  SG_CHECK(z && labels && row_loss && dz, SG_ERR_INVALID_ARG, "softmax_ce: null pointer");
  SG_CHECK(rows > 0 && C > 0 && n_loc > 0, SG_ERR_DIMENSION, "softmax_ce: rows=%d C=%d n_loc=%d", rows, C, n_loc);
  SG_LAUNCH(softmax_ce(plain(const_cast<float*>(z), rows, C), labels, row_loss, plain(dz, rows, C), 1.f / n_loc,
                       reinterpret_cast<int*>(err), S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_euclidean(const float* u, const float* v, int32_t rows, int32_t d, int32_t n_loc,
                                 float* row_loss, float* du, void* stream) {
  SG_CHECK(u && v && row_loss && du, SG_ERR_INVALID_ARG, "euclidean: null pointer");
  SG_CHECK(rows > 0 && d > 0 && n_loc > 0, SG_ERR_DIMENSION, "euclidean: rows=%d d=%d n_loc=%d", rows, d, n_loc);
  SG_LAUNCH(euclidean(plain(const_cast<float*>(u), rows, d), plain(const_cast<float*>(v), rows, d), row_loss,
                      plain(du, rows, d), 1.f / n_loc, S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_sgd_momentum(float* w, const float* g, float* v, int64_t n, float lr, float mu, float wd,
                                    float s, void* stream) {
  SG_CHECK(w && g && v && n >= 0, SG_ERR_INVALID_ARG, "sgd_momentum: bad argument");
  SG_LAUNCH(sgd_momentum(w, g, v, n, lr, mu, wd, s, S(stream)));
  return SG_OK;
}

SG_API sg_status sg_op_adagrad(float* w, const float* g, float* h, int64_t n, float lr, float wd, float s, float eps,
                               void* stream) {
  SG_CHECK(w && g && h && n >= 0 && eps > 0.f, SG_ERR_INVALID_ARG, "adagrad: bad argument");
  SG_LAUNCH(adagrad(w, g, h, n, lr, wd, s, eps, S(stream)));
  return SG_OK;
}

}  // extern "C"
