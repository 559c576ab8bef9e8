// dense_cta.cuh — small CTA-wide dense kernels on shared memory (setup only).
#pragma once
#include "internal.h"

// ------------------------------------------------------------------ CTA-wide dense helpers (smem)
// Cholesky in place (lower, row-major, leading dim ld); returns 1 if a pivot was <= 0.
__device__ inline int cta_chol(double* M, int n, int ld) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      double s = M[j * ld + j];
      for (int k = 0; k < j; ++k) s -= M[j * ld + k] * M[j * ld + k];
      if (!(s > 0)) { bad = 1; s = 1.0; }
      M[j * ld + j] = sqrt(s);
    }
    __syncthreads();
    double d = M[j * ld + j];
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      double t = M[i * ld + j];
      for (int k = 0; k < j; ++k) t -= M[i * ld + k] * M[j * ld + k];
      M[i * ld + j] = t / d;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int i = e / n, k = e % n;
    if (k > i) M[i * ld + k] = 0.0;
  }
  __syncthreads();
  int r = bad;
  __syncthreads();
  return r;
}

// X = L^{-1} (lower triangular), thread per column
__device__ inline void cta_trinv(const double* L, double* X, int n, int ld) {
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    for (int i = 0; i < c; ++i) X[i * ld + c] = 0.0;
    for (int i = c; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int k = c; k < i; ++k) s -= L[i * ld + k] * X[k * ld + c];
      X[i * ld + c] = s / L[i * ld + i];
    }
  }
  __syncthreads();
}

// Orthonormalise the raw basis whose Gram matrix is in M (n x n, smem): C = (chol of M)^-1, then one
// more CholQR pass on C M C^T (CholQR2). Writes C to out (global). Returns pivot failure.
__device__ inline int cta_cholqr2(double* M, double* T1, double* T2, int n, double* out) {
  int ld = n;
  // T1 = copy of M (Gram)
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) T1[e] = M[e];
  __syncthreads();
  int bad = cta_chol(M, n, ld);       // M = L1
  cta_trinv(M, T2, n, ld);            // T2 = C1 = L1^-1
  // M = C1 Gram C1^T   (reuse M as output; T1 = Gram)
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int a = e / n, b = e % n;
    double s = 0;
    for (int k = 0; k <= a; ++k) {
      double t = 0;
      for (int l = 0; l <= b; ++l) t += T1[k * n + l] * T2[b * n + l];
      s += T2[a * n + k] * t;
    }
    M[e] = s;
  }
  __syncthreads();
  bad |= cta_chol(M, n, ld);          // M = L2
  cta_trinv(M, T1, n, ld);            // T1 = L2^-1
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    int a = e / n, b = e % n;
    double s = 0;
    for (int k = b; k <= a; ++k) s += T1[a * n + k] * T2[k * n + b];
    out[e] = s;  // lower triangular
  }
  __syncthreads();
  return bad;
}

