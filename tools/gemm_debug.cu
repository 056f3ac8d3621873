// Standalone debug driver for the tcgen05 GEMM engine (not part of the library).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1603_07846_b200/csrc/ops.h"
int main(int argc, char** argv) {
  int shapes[][3] = {{128, 32, 32}, {128, 64, 64}, {256, 128, 96}};
  for (auto& sh : shapes) {
    int M = sh[0], N = sh[1], K = sh[2];
    std::vector<float> A(M * K), B(K * N), Cm(M * N);
    srand(1);
    for (auto& v : A) v = (rand() % 17) - 8;
    for (auto& v : B) v = (rand() % 13) - 6;
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, Cm.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int ta = 0; ta < 2; ++ta)
      for (int tb = 0; tb < 2; ++tb)
        for (int mode = 0; mode < 1; ++mode) {
          cudaMemset(dC, 0xff, Cm.size() * 4);
          sg::Workspace ws{nullptr, 0};
          cudaError_t e = sg::gemm_plain(dA, ta, dB, tb, dC, M, N, K, ws, 0);
          cudaError_t e2 = cudaDeviceSynchronize();
          cudaMemcpy(Cm.data(), dC, Cm.size() * 4, cudaMemcpyDeviceToHost);
          // A stored [M][K] (ta=0) or [K][M]; B stored [K][N] (tb=0) or [N][K]; same logical values reused
          double err = 0, ref2 = 0; int nz = 0;
          for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
              double acc = 0;
              for (int k = 0; k < K; ++k) {
                double a = ta ? A[k * M + m] : A[m * K + k];
                double b = tb ? B[n * K + k] : B[k * N + n];
                acc += a * b;
              }
              double d = Cm[m * N + n] - acc;
              err += d * d; ref2 += acc * acc; nz += Cm[m * N + n] != 0;
            }
          printf("M=%d N=%d K=%d ta=%d tb=%d mode=%2d: %s/%s relerr=%.3e nonzero=%d C00=%g\n", M, N, K, ta, tb, mode,
                 cudaGetErrorString(e), cudaGetErrorString(e2), sqrt(err / ref2), nz, Cm[0]);
          if (e2 != cudaSuccess) return 1;
        }
  }
  return 0;
}
