// Launchers for the tcgen05 implicit-GEMM engine: convolution forward / data
// gradient / weight gradient (+ fused bias gradient) and inner-product forward /
// data gradient / weight gradient (§4.1.2, §5.4.1; SURVEY
// §8(a) a3, a8, a10, a15), deterministic split-K reduction and column sums.
#include <algorithm>

#include "gemm_tc.cuh"
#include "ops.h"

namespace sg {

long long g_kernel_launches = 0;

namespace {

constexpr int kNumSMs = 148;
constexpr int kMinKbPerSplit = 8;

struct Plan {
  int bn, mt, nt, splits, kb_per_split;
};

inline long long pad4(int n) { return (n + 3) & ~3; }

Plan plan_gemm(int M, int N, int K, size_t ws_floats_avail) {
  Plan p;
  p.bn = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  p.mt = (M + GEMM_BM - 1) / GEMM_BM;
  if (p.bn == 256 && p.mt * ((N + 255) / 256) < kNumSMs) p.bn = 128;
  p.nt = (N + p.bn - 1) / p.bn;
  const int nkb = (K + GEMM_BK - 1) / GEMM_BK;
  const int tiles = p.mt * p.nt;
  int splits = 1;
  if (tiles < kNumSMs && nkb >= 2 * kMinKbPerSplit) {
    splits = std::min((kNumSMs + tiles - 1) / tiles, nkb / kMinKbPerSplit);
    while (splits > 1 && (size_t)splits * M * pad4(N) > ws_floats_avail) --splits;
    if (splits < 1) splits = 1;
  }
  p.kb_per_split = (nkb + splits - 1) / splits;
  if (p.kb_per_split < 1) p.kb_per_split = 1;
  p.splits = (nkb + p.kb_per_split - 1) / p.kb_per_split;
  if (p.splits < 1) p.splits = 1;
  return p;
}

__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, long long split_stride, int M, int N,
                                     EpiArgs e) {
  long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)M * N) return;
  int m, n;
  if (e.trans) {  // consecutive threads -> consecutive m (coalesced store)
    n = (int)(idx / M);
    m = (int)(idx - (long long)n * M);
  } else {
    m = (int)(idx / N);
    n = (int)(idx - (long long)m * N);
  }
  if (m >= e.mvalid && m != e.xrow) return;
  float acc = 0.f;
  const float* p = ws + (long long)m * ((N + 3) & ~3) + n;
  for (int s = 0; s < splits; ++s) acc += p[s * split_stride];
  if (m == e.xrow) {
    e.xout[n] = acc;
    return;
  }
  if (e.bias) acc += e.bias_on_m ? e.bias[m] : e.bias[n];
  if (e.relu) acc = fmaxf(acc, 0.f);
  if (e.trans)
    *out_at(e, n, m, e.mvalid) = acc;
  else
    *out_at(e, m, n, N) = acc;
}

template <int BN, class LA, class LB>
cudaError_t launch_bn(const GemmArgs<LA, LB>& args, const Plan& p, cudaStream_t st) {
  constexpr int STAGES = BN >= 256 ? 3 : 4;
  constexpr int SMEM = gemm_smem_bytes<BN, STAGES>();
  auto kern = gemm_tc_kernel<BN, STAGES, LA, LB>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(p.mt, p.nt, p.splits);
  kern<<<grid, GEMM_THREADS, SMEM, st>>>(args);
  return launched();
}

template <class LA, class LB>
cudaError_t run_gemm(const LA& a, const LB& b, int M, int N, int K, EpiArgs epi, Workspace ws, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  Plan p = plan_gemm(M, N, K, ws.floats);
  GemmArgs<LA, LB> args{a, b, M, N, K, p.kb_per_split, epi};
  if (p.splits > 1) {
    args.epi.ws = ws.ptr;
    args.epi.ws_ld = pad4(N);
    args.epi.ws_split_stride = (long long)M * pad4(N);
  } else {
    args.epi.ws = nullptr;
  }
  cudaError_t e;
  switch (p.bn) {
    case 32: e = launch_bn<32>(args, p, st); break;
    case 64: e = launch_bn<64>(args, p, st); break;
    case 128: e = launch_bn<128>(args, p, st); break;
    default: e = launch_bn<256>(args, p, st); break;
  }
  if (e != cudaSuccess || p.splits == 1) return e;
  long long total = (long long)M * N;
  splitk_reduce_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(ws.ptr, p.splits, (long long)M * pad4(N), M,
                                                                         N, epi);
  return launched();
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

EpiArgs epi_plain(float* p, long long ld, int trans, const float* bias, int bias_on_m, int relu, int mvalid) {
  EpiArgs e{};
  e.p = p;
  e.ld = ld;
  e.bs = 0;
  e.cb = 1 << 30;
  e.trans = trans;
  e.bias = bias;
  e.bias_on_m = bias_on_m;
  e.relu = relu;
  e.mvalid = mvalid;
  e.xrow = -1;
  e.xout = nullptr;
  return e;
}
EpiArgs epi_view(const View2D& d, const float* bias, int relu) {
  EpiArgs e = epi_plain(d.p, d.ld, 0, bias, 0, relu, d.rows);
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

// ---------------------------------------------------------- column sums ----
constexpr int CS_ROWS_PER_BLOCK = 1024;

__global__ void colsum_partial_kernel(const float* __restrict__ X, int M, int N, long long ld,
                                      float* __restrict__ part) {
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
  int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= N) return;
  float s = 0.f;
  for (int i = 0; i < nparts; ++i) s += part[(long long)i * N + col];
  out[col] = s;
}

}  // namespace

size_t gemm_ws_floats(int M, int N, int K) {
  Plan p = plan_gemm(M, N, K, (size_t)1 << 62);
  // the weight-gradient GEMMs may add one ones-row (fused bias gradient)
  return p.splits > 1 ? (size_t)p.splits * (M + 4) * pad4(N) : 0;
}

cudaError_t colsum(const float* X, int M, int N, long long ld, float* out, Workspace ws, cudaStream_t st) {
  int nparts = (M + CS_ROWS_PER_BLOCK - 1) / CS_ROWS_PER_BLOCK;
  if ((size_t)nparts * N > ws.floats) return cudaErrorInvalidValue;
  dim3 grid((N + 31) / 32, nparts);
  colsum_partial_kernel<<<grid, dim3(32, 8), 0, st>>>(X, M, N, ld, ws.ptr);
  cudaError_t e = launched();
  if (e != cudaSuccess) return e;
  colsum_final_kernel<<<(N + 127) / 128, 128, 0, st>>>(ws.ptr, nparts, N, out);
  return launched();
}

size_t colsum_ws_floats(int M, int N) { return (size_t)((M + CS_ROWS_PER_BLOCK - 1) / CS_ROWS_PER_BLOCK) * N; }

// ------------------------------------------------------------ convolution ----
cudaError_t conv_fwd(const ConvShape& s, const float* x, const float* W, const float* b, float* y, int relu,
                     Workspace ws, cudaStream_t st) {
  const int M = s.N * s.Ho * s.Wo, N = s.Co, K = s.R * s.S * s.C;
  LdConvFwdA a{x, geom(s)};
  LdDenseK bw{mv(W, s.Co, K, K)};
  return run_gemm(a, bw, M, N, K, epi_plain(y, s.Co, 0, b, 0, relu, M), ws, st);
}

cudaError_t conv_dgrad(const ConvShape& s, const float* dy, const float* W, float* dx, Workspace ws,
                       cudaStream_t st) {
  const int M = s.N * s.H * s.W, N = s.C, K = s.R * s.S * s.Co;
  LdConvDgradA a{dy, geom(s)};
  LdConvDgradB bw{W, geom(s)};
  return run_gemm(a, bw, M, N, K, epi_plain(dx, s.C, 0, nullptr, 0, 0, M), ws, st);
}

cudaError_t conv_wgrad(const ConvShape& s, const float* x, const float* dy, float* dW, float* db, Workspace ws,
                       cudaStream_t st) {
  const int Kg = s.R * s.S * s.C, Mtot = s.N * s.Ho * s.Wo;
  LdConvWgradA a{x, geom(s), db ? Kg : -1};
  LdDenseMN bd{mv(dy, Mtot, s.Co, s.Co), -1};
  // D[kg][co] stored transposed into dW[co][kg]; row Kg (ones) = db
  EpiArgs e = epi_plain(dW, Kg, 1, nullptr, 0, 0, Kg);
  if (db) {
    e.xrow = Kg;
    e.xout = db;
  }
  return run_gemm(a, bd, db ? Kg + 1 : Kg, s.Co, Mtot, e, ws, st);
}

// ---------------------------------------------------------- inner product ----
cudaError_t ip_fwd(View2D x, const float* W, int dv, int dh, const float* b, View2D y, int relu, Workspace ws,
                   cudaStream_t st) {
  LdDenseK a{mv(x)};
  LdDenseMN bw{mv(W, dv, dh, dh), -1};  // op(n, k) = W(k, n)
  return run_gemm(a, bw, x.rows, dh, dv, epi_view(y, b, relu), ws, st);
}

cudaError_t ip_dgrad(View2D dy, const float* W, int dv, int dh, View2D dx, Workspace ws, cudaStream_t st) {
  LdDenseK a{mv(dy)};
  LdDenseK bw{mv(W, dv, dh, dh)};   // op(n = v, k = h) = W(v, h)
  return run_gemm(a, bw, dy.rows, dv, dh, epi_view(dx, nullptr, 0), ws, st);
}

cudaError_t ip_wgrad(View2D x, View2D dy, int dv, int dh, float* dW, float* db, Workspace ws, cudaStream_t st) {
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
  if (!ta && !tb) return run_gemm(LdDenseK{mv(A, M, K, K)}, LdDenseMN{mv(B, K, N, N), -1}, M, N, K, e, ws, st);
  if (!ta && tb) return run_gemm(LdDenseK{mv(A, M, K, K)}, LdDenseK{mv(B, N, K, K)}, M, N, K, e, ws, st);
  if (ta && !tb)
    return run_gemm(LdDenseMN{mv(A, K, M, M), -1}, LdDenseMN{mv(B, K, N, N), -1}, M, N, K, e, ws, st);
  return run_gemm(LdDenseMN{mv(A, K, M, M), -1}, LdDenseK{mv(B, N, K, K)}, M, N, K, e, ws, st);
}

}  // namespace sg
