// Internal kernel launchers (host side).  Every function enqueues work on
// `st` and returns cudaError_t from the launch; shapes are validated by the
// callers (runtime / ABI layer).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <utility>

namespace sg {

// Number of kernels launched by this library (all launchers bump it).
extern long long g_kernel_launches;
inline cudaError_t launched() {
  ++g_kernel_launches;
  return cudaGetLastError();
}

// Programmatic dependent launch on/off (SG_PDL, default on).
bool pdl_enabled();

// Launch `k` on `st` with programmatic stream serialisation, so its prologue
// overlaps the tail of the previous kernel (every kernel of this library starts
// with pdl_wait(); see sg_common.cuh).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
  ++g_kernel_launches;
  return e != cudaSuccess ? e : cudaGetLastError();
}

// GEMM / convolution epilogue flags: ReLU of the output (layer fusion) and
// TF32 round-to-nearest of the stored values (reading A19: the output is read
// as a tensor-core operand by the next GEMM).
enum { EPI_RELU = 1, EPI_RN = 2 };

// Scratch for deterministic split-K partials (owned by the caller).
struct Workspace {
  float* ptr = nullptr;
  size_t floats = 0;
};

// Blocked row-major 2-D view description for FC operands / outputs:
// element (i, j) at p[(j / cb) * bs + i * ld + j % cb]; cb = cols for a plain matrix.
struct View2D {
  float* p;
  long long ld, bs;
  int cb, rows, cols;
};
inline View2D plain(float* p, int rows, int cols, long long ld = -1) {
  return View2D{p, ld < 0 ? cols : ld, 0, cols, rows, cols};
}

struct ConvShape {
  int N, H, W, C;  // C multiple of 4 (padded)
  int Co, R, S, st, pad;
  int Ho, Wo;
};

// Number of floats of split-K workspace a GEMM of this shape may use.
size_t gemm_ws_floats(int M, int N, int K);

// Resident-image tcgen05 convolution (conv_img.cu): stride 1, C and Co
// multiples of 32, padded image in shared memory.  conv_fwd / conv_dgrad use
// it whenever the *_ok predicate holds (SG_IMG_CONV=0 disables it).
bool conv_img_fwd_ok(const ConvShape& s);
bool conv_img_dgrad_ok(const ConvShape& s);
cudaError_t conv_img_fwd(const ConvShape& s, const float* x, const float* W, const float* b, float* y, int flags,
                         cudaStream_t st);
cudaError_t conv_img_dgrad(const ConvShape& s, const float* dy, const float* W, float* dx, cudaStream_t st,
                           int flags = 0);
bool conv_img_wgrad_ok(const ConvShape& s);
size_t conv_img_wgrad_ws_floats(const ConvShape& s);  // per-sample partials
cudaError_t conv_img_wgrad(const ConvShape& s, const float* x, const float* dy, float* dW, float* db, Workspace ws,
                           cudaStream_t st);


// 4-channel stride-1 first layer (CIFAR conv1) weight / bias gradient on the
// resident image (conv_img.cu): from dy, or fused with the backward of the
// max-pooling layer that consumes the convolution (dy = the pool's dx is built
// in shared memory and written to dy_out, TF32-rounded when rn).
bool conv_img4_wgrad_ok(const ConvShape& s);
size_t conv_img4_wgrad_ws_floats(const ConvShape& s);
cudaError_t conv_img4_wgrad(const ConvShape& s, const float* x, const float* dy, float* dW, float* db, Workspace ws,
                            cudaStream_t st);
struct PoolShape;
struct FusedUpdate;  // elt_common.cuh
bool conv_img4_pool_bwd_ok(const ConvShape& s, const PoolShape& p);
// fu (optional, K = 1): the reduction of dW / db also applies the Updater
cudaError_t conv_img4_pool_bwd(const ConvShape& s, const PoolShape& p, const float* x, const float* gpool,
                               const uint8_t* mask, float* dy_out, int rn, float* dW, float* db, Workspace ws,
                               cudaStream_t st, const FusedUpdate* fu = nullptr);

// ---- convolution (implicit GEMM, tcgen05 kind::tf32) ----
// flags: EPI_RELU | EPI_RN
cudaError_t conv_fwd(const ConvShape& s, const float* x, const float* W, const float* b, float* y, int flags,
                     Workspace ws, cudaStream_t st);
cudaError_t conv_dgrad(const ConvShape& s, const float* dy, const float* W, float* dx, Workspace ws,
                       cudaStream_t st, int flags = 0);
// dW [Co][R][S][C]; db [Co] (db may be null)
cudaError_t conv_wgrad(const ConvShape& s, const float* x, const float* dy, float* dW, float* db, Workspace ws,
                       cudaStream_t st);

// ---- strided convolution by space-to-depth (conv_s2d.cu) ----
// A stride-st convolution equals a stride-1, unpadded one with ceil(R/st) x
// ceil(S/st) taps over the st x st space-to-depth image (st*st*C channels).
bool conv_s2d_ok(const ConvShape& s);
ConvShape conv_s2d_shape(const ConvShape& s);
size_t conv_s2d_x_floats(const ConvShape& s);
size_t conv_s2d_w_floats(const ConvShape& s);
cudaError_t conv_s2d_input(const ConvShape& s, const float* x, float* xs, cudaStream_t st);
// input layer: channel padding cin -> 4 into y and the space-to-depth image xs of
// the first convolution (shape s, C = 4) in one pass; xs borders must be zero
cudaError_t pad_channels_s2d(const float* x, int cin, float* y, float* xs, const ConvShape& s, cudaStream_t st,
                             int rn);
// Wt: scratch for the rearranged filter (conv_s2d_w_floats)
cudaError_t conv_fwd_s2d(const ConvShape& s, const float* xs, const float* W, float* Wt, const float* b, float* y,
                         int flags, Workspace ws, cudaStream_t st);
// dWt: scratch for the space-to-depth filter gradient (conv_s2d_w_floats)
cudaError_t conv_wgrad_s2d(const ConvShape& s, const float* xs, const float* dy, float* dWt, float* dW, float* db,
                           Workspace ws, cudaStream_t st);

// ---- inner product:  y = x W + b ; W [d_v][d_h] ----
cudaError_t ip_fwd(View2D x, const float* W, int dv, int dh, const float* b, View2D y, int flags, Workspace ws,
                   cudaStream_t st);
cudaError_t ip_dgrad(View2D dy, const float* W, int dv, int dh, View2D dx, Workspace ws, cudaStream_t st,
                     int flags = 0);
cudaError_t ip_wgrad(View2D x, View2D dy, int dv, int dh, float* dW, float* db, Workspace ws, cudaStream_t st);

// Generic TF32 GEMM on plain row-major matrices (test entry):
// C[M][N] = op(A) op(B) with A [M][K] (ta=0) or [K][M] (ta=1), B [K][N] (tb=0) or [N][K] (tb=1).
cudaError_t gemm_plain(const float* A, int ta, const float* B, int tb, float* C, int M, int N, int K, Workspace ws,
                       cudaStream_t st);

// ---- column sums (bias gradient): out[n] = sum_m X[m][n] ----
cudaError_t colsum(const float* X, int M, int N, long long ld, float* out, Workspace ws, cudaStream_t st);

// ---- elementwise / pooling / LRN / loss ----
// `rn` (every launcher below): TF32 round-to-nearest of the stored output
// (reading A19).  Kernels with two outputs take a mask: RN_OUT rounds the
// primary output (y / dx), RN_AUX the fused ReLU output (relu_out / dx_relu).
enum { RN_OUT = 1, RN_AUX = 2 };
cudaError_t relu_fwd(const float* x, float* y, long long n, cudaStream_t st, int rn = 0);
cudaError_t relu_bwd(const float* y, const float* dy, float* dx, long long n, cudaStream_t st, int rn = 0);
cudaError_t sigmoid_fwd(const float* x, float* y, long long n, cudaStream_t st, int rn = 0);
cudaError_t sigmoid_bwd(const float* y, const float* dy, float* dx, long long n, cudaStream_t st, int rn = 0);
// 2-D variants for column-sliced FC features (rows x cols with leading dim ld)
cudaError_t relu_fwd2d(const float* x, float* y, int rows, int cols, long long ld, cudaStream_t st);

struct PoolShape {
  int N, H, W, C, k, s, p, Ho, Wo;
};
// Optional ReLU fusion (runtime layer fusion, bit-identical to the separate ReLU
// kernels): forward `relu_out` = max(y, 0) besides y; backward `dx_relu` =
// dx * [relu_y > 0] besides dx (the gradient through the ReLU feeding this layer).
cudaError_t maxpool_fwd(const PoolShape& s, const float* x, float* y, uint8_t* arg, cudaStream_t st,
                        float* relu_out = nullptr, int rn = 0);
cudaError_t maxpool_bwd(const PoolShape& s, const float* dy, const uint8_t* arg, float* dx, cudaStream_t st,
                        const float* relu_y = nullptr, float* dx_relu = nullptr, int rn = 0);
cudaError_t avgpool_fwd(const PoolShape& s, const float* x, float* y, cudaStream_t st, float* relu_out = nullptr,
                        int rn = 0);
cudaError_t avgpool_bwd(const PoolShape& s, const float* dy, float* dx, cudaStream_t st, const float* relu_y = nullptr,
                        float* dx_relu = nullptr, int rn = 0);
// argmax window offset -> int32 flat h*W+w in the input plane (ABI export format)
cudaError_t pool_argmax_expand(const PoolShape& s, const uint8_t* arg, int32_t* out, cudaStream_t st);

struct LrnShape {
  long long pixels;
  int C, n;
  float alpha, beta, k;
};
cudaError_t lrn_fwd(const LrnShape& s, const float* x, float* y, float* scale, cudaStream_t st, int rn = 0);
// Pooling (+ the ReLU after it) + LRN in one pass (runtime layer fusion).
bool pool_lrn_fusable(const PoolShape& ps, const LrnShape& ls);
cudaError_t pool_lrn_fwd(const PoolShape& ps, bool max_pool, const float* x, float* py, uint8_t* arg, float* relu_out,
                         const LrnShape& ls, float* ly, float* scale, cudaStream_t st, int rn = 0);
cudaError_t lrn_bwd(const LrnShape& s, const float* x, const float* y, const float* scale, const float* dy, float* dx,
                    cudaStream_t st, const float* relu_y = nullptr, float* dx_relu = nullptr, int rn = 0);

// Softmax cross-entropy over rows of a (blocked) logits view; per-row loss and
// dz = (softmax - onehot) / n_loc written with the same blocking. Labels out of
// [0, C) set *err = 1.
cudaError_t softmax_ce(View2D z, const int32_t* labels, float* row_loss, View2D dz, float inv_nloc, int* err,
                       cudaStream_t st, int rn = 0);
// Euclidean: per-row 0.5 ||u - v||^2 and du = (u - v) / n_loc.
cudaError_t euclidean(View2D u, View2D v, float* row_loss, View2D du, float inv_nloc, cudaStream_t st, int rn = 0);
// out[0] = scale * sum(v[0..n)) (fixed-order, single block); also flags non-finite in *err (bit 2)
cudaError_t sum_scaled(const float* v, int n, float scale, float* out, int* err, cudaStream_t st);

// ---- Updater: g' = s g + wd w ; v = mu v - lr g' ; w += v ----
cudaError_t sgd_momentum(float* w, const float* g, float* v, long long n, float lr, float mu, float wd, float s,
                         cudaStream_t st);
// Same with lr read from device memory (graph-capturable): lr = lr_dev[0] * lr_scale.
// wk (optional): working copy written alongside, TF32-RN for elements < rn_end.
cudaError_t sgd_momentum_dev(float* w, const float* g, float* v, long long n, const float* lr_dev, float lr_scale,
                             float mu, float wd, float s, cudaStream_t st, float* wk = nullptr, long long rn_end = 0);

// ---- AdaGrad: g' = s g + wd w ; h += g'^2 ; w -= lr g' / (sqrt(h) + eps) ----
cudaError_t adagrad(float* w, const float* g, float* h, long long n, float lr, float wd, float s, float eps,
                    cudaStream_t st);
cudaError_t adagrad_dev(float* w, const float* g, float* h, long long n, const float* lr_dev, float lr_scale, float wd,
                        float s, float eps, cudaStream_t st, float* wk = nullptr, long long rn_end = 0);

// ---- input layer: NHWC with C=3 (user layout) -> padded C=4 ----
cudaError_t pad_channels(const float* x, float* y, long long pixels, int cin, int cout, cudaStream_t st, int rn = 0);
// copy rows x cols fp32 (strided) — used for feature-blocked gathers on the host side of tests
cudaError_t copy2d(const float* src, long long sld, float* dst, long long dld, int rows, int cols, cudaStream_t st,
                   int rn = 0);
// in-place TF32 round-to-nearest of n floats
cudaError_t round_tf32(float* p, long long n, cudaStream_t st);

}  // namespace sg

namespace sg {
// p[0] = v (stream-ordered; used to feed per-step scalars to captured graphs)
cudaError_t fill_scalar(float* p, float v, cudaStream_t st);
}  // namespace sg
