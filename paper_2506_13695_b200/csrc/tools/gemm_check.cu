// Standalone correctness + speed check of gemm_bf16 (tcgen05) against a
// straightforward fp32 reference kernel on the same bf16 inputs.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../gemm.cuh"

using namespace orx;

__global__ void ref_kernel(const __nv_bfloat16* A, int lda, const __nv_bfloat16* B, int ldb, int M, int N, int K,
                           const float* bias, float* C) {
  int n = blockIdx.x * blockDim.x + threadIdx.x, m = blockIdx.y;
  if (n >= N || m >= M) return;
  float s = 0;
  for (int k = 0; k < K; ++k) s += __bfloat162float(A[(size_t)m * lda + k]) * __bfloat162float(B[(size_t)n * ldb + k]);
  if (bias) s += bias[n];
  C[(size_t)m * N + n] = s;
}

__global__ void fill(__nv_bfloat16* p, size_t n, uint32_t seed) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t h = (uint32_t)i * 2654435761u ^ seed;
  h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
  p[i] = __float2bfloat16((float)(h & 0xFFFF) / 65536.f - 0.5f);
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

int check(int M, int N, int K, bool bias_on, bool bf16_out, int iters) {
  int lda = K, ldb = K;
  __nv_bfloat16 *A, *B;
  float *C, *R, *bias = nullptr;
  CK(cudaMalloc(&A, (size_t)M * lda * 2));
  CK(cudaMalloc(&B, (size_t)N * ldb * 2));
  CK(cudaMalloc(&C, (size_t)M * N * 4));
  CK(cudaMalloc(&R, (size_t)M * N * 4));
  fill<<<((size_t)M * lda + 255) / 256, 256>>>(A, (size_t)M * lda, 1);
  fill<<<((size_t)N * ldb + 255) / 256, 256>>>(B, (size_t)N * ldb, 2);
  if (bias_on) {
    CK(cudaMalloc(&bias, N * 4));
    std::vector<float> hb(N);
    for (int i = 0; i < N; ++i) hb[i] = 0.01f * (i % 17);
    CK(cudaMemcpy(bias, hb.data(), N * 4, cudaMemcpyHostToDevice));
  }
  void* out = C;
  __nv_bfloat16* Cb = nullptr;
  if (bf16_out) { CK(cudaMalloc(&Cb, (size_t)M * N * 2)); out = Cb; }
  Epi e;
  e.bias = bias; e.out = out; e.ldo = N; e.out_bf16 = bf16_out; e.n_out = N; e.m_valid = M;
  gemm_bf16(A, lda, B, ldb, M, N, K, e, nullptr, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  ref_kernel<<<dim3((N + 127) / 128, M), 128>>>(A, lda, B, ldb, M, N, K, bias, R);
  CK(cudaDeviceSynchronize());
  std::vector<float> hc((size_t)M * N), hr((size_t)M * N);
  if (bf16_out) {
    std::vector<__nv_bfloat16> t((size_t)M * N);
    CK(cudaMemcpy(t.data(), Cb, t.size() * 2, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < t.size(); ++i) hc[i] = __bfloat162float(t[i]);
  } else {
    CK(cudaMemcpy(hc.data(), C, hc.size() * 4, cudaMemcpyDeviceToHost));
  }
  CK(cudaMemcpy(hr.data(), R, hr.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  size_t bad = 0;
  for (size_t i = 0; i < hc.size(); ++i) {
    double d = fabs(hc[i] - hr[i]);
    maxerr = fmax(maxerr, d);
    maxref = fmax(maxref, fabs(hr[i]));
    if (d > 1e-2 * (1 + fabs(hr[i])) || std::isnan(hc[i])) {
      if (bad < 5) printf("  mismatch at (%zu,%zu): got %f want %f\n", i / N, i % N, hc[i], hr[i]);
      ++bad;
    }
  }
  float ms = 0;
  if (iters > 0) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) gemm_bf16(A, lda, B, ldb, M, N, K, e, nullptr, 0);
    cudaEventRecord(a);
    for (int i = 0; i < iters; ++i) gemm_bf16(A, lda, B, ldb, M, N, K, e, nullptr, 0);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    cudaEventElapsedTime(&ms, a, b);
    ms /= iters;
  }
  printf("M=%d N=%d K=%d bias=%d bf16out=%d: maxerr=%.3e maxref=%.3e bad=%zu %s  %.3f ms  %.1f TFLOP/s\n", M, N, K,
         bias_on, bf16_out, maxerr, maxref, bad, bad ? "FAIL" : "OK", ms,
         ms > 0 ? 2.0 * M * N * K / (ms * 1e-3) / 1e12 : 0.0);
  cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(R);
  if (bias) cudaFree(bias);
  if (Cb) cudaFree(Cb);
  return bad ? 1 : 0;
}

int main() {
  int fails = 0;
  fails += check(128, 256, 64, false, false, 0);
  fails += check(128, 128, 64, false, false, 0);
  fails += check(256, 512, 128, true, false, 0);
  fails += check(300, 1000, 200, true, true, 0);
  fails += check(1000, 1024, 2176, true, true, 0);
  fails += check(16384, 1024, 1024, false, true, 10);
  fails += check(16384, 8192, 1024, false, false, 5);
  fails += check(8192, 8192, 8192, false, true, 5);
  printf(fails ? "GEMM CHECK FAILED\n" : "GEMM CHECK PASSED\n");
  return fails;
}
