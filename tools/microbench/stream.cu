// Streaming-bandwidth microbenchmark: cp.async.bulk ring vs vectorised loads (B200 sm_100a).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1903_11357_b200/csrc/tma.cuh"

__global__ void k_bulk(const double* __restrict__ src, size_t n_per_cta, int S, uint32_t B, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = (uint64_t*)sm;
  unsigned char* ring = sm + 256;
  const char* base = (const char*)(src + (size_t)blockIdx.x * n_per_cta);
  const size_t bytes = n_per_cta * 8;
  const int nunits = (int)(bytes / B);
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) for (int u = 0; u < S && u < nunits; ++u) bulk_load(ring + (size_t)u * B, base + (size_t)u * B, B, &bars[u]);
  uint32_t ph = 0;
  double acc = 0;
  for (int u = 0; u < nunits; ++u) {
    int s = u % S;
    mbar_wait(&bars[s], (ph >> s) & 1); ph ^= 1u << s;
    const double* d = (const double*)(ring + (size_t)s * B);
    for (int i = threadIdx.x; i < (int)(B / 8); i += blockDim.x) acc += d[i];
    __syncthreads();
    if (threadIdx.x == 0 && u + S < nunits) bulk_load(ring + (size_t)s * B, base + (size_t)(u + S) * B, B, &bars[s]);
  }
  if (acc == 12345.678) out[0] = acc;
}

// same ring, but each unit is split into `parts` bulk copies
__global__ void k_bulk_split(const double* __restrict__ src, size_t n_per_cta, int S, uint32_t B, int parts, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bars = (uint64_t*)sm;
  unsigned char* ring = sm + 256;
  const char* base = (const char*)(src + (size_t)blockIdx.x * n_per_cta);
  const size_t bytes = n_per_cta * 8;
  const int nunits = (int)(bytes / B);
  if (threadIdx.x == 0) { for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1); fence_mbar_init(); }
  __syncthreads();
  auto issue = [&](int u) {
    int s = u % S;
    mbar_expect_tx(&bars[s], B);
    uint32_t pb = B / parts;
    for (int p = 0; p < parts; ++p) bulk_g2s(ring + (size_t)s * B + p * pb, base + (size_t)u * B + p * pb, pb, &bars[s]);
  };
  if (threadIdx.x == 0) for (int u = 0; u < S && u < nunits; ++u) issue(u);
  uint32_t ph = 0;
  double acc = 0;
  for (int u = 0; u < nunits; ++u) {
    int s = u % S;
    mbar_wait(&bars[s], (ph >> s) & 1); ph ^= 1u << s;
    const double* d = (const double*)(ring + (size_t)s * B);
    for (int i = threadIdx.x; i < (int)(B / 8); i += blockDim.x) acc += d[i];
    __syncthreads();
    if (threadIdx.x == 0 && u + S < nunits) issue(u + S);
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void k_ldg(const double2* __restrict__ src, size_t n2, double* out) {
  double acc = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, stride = (size_t)gridDim.x * blockDim.x;
#pragma unroll 8
  for (; i < n2; i += stride) { double2 v = __ldcs(src + i); acc += v.x + v.y; }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  size_t N = (size_t)1 << 28;  // 2 GiB of doubles
  double *src, *out;
  cudaMalloc(&src, N * 8); cudaMalloc(&out, 64); cudaMemset(src, 0, N * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_bulk_split, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k_ldg<<<nsm * 8, 256>>>((const double2*)src, N / 2, out); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); if (rep) printf("ldg.128 grid=%d: %.0f GB/s\n", nsm * 8, N * 8 / ms / 1e6);
  }
  int ctas_per_sm[] = {1, 2, 4};
  uint32_t Bs[] = {4096, 16384, 32768, 65536};
  int Ss[] = {2, 3, 6, 12};
  for (int cps : ctas_per_sm)
    for (uint32_t B : Bs)
      for (int S : Ss) {
        size_t smem = 256 + (size_t)S * B;
        if (smem * cps > 225 * 1024) continue;
        int grid = nsm * cps;
        size_t npc = N / grid / (B / 8) * (B / 8);
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(a); k_bulk<<<grid, 256, smem>>>(src, npc, S, B, out); cudaEventRecord(b); cudaEventSynchronize(b);
          cudaEventElapsedTime(&ms, a, b);
        }
        printf("bulk cta/sm=%d B=%6u S=%2d inflight/SM=%4zu KB: %.0f GB/s\n", cps, B, S, (size_t)cps * S * B / 1024, npc * grid * 8 / ms / 1e6);
      }
  for (int parts : {2, 4, 8, 16})
    for (int cps : {1, 2}) {
      uint32_t B = 65536; int S = cps == 1 ? 3 : 1;
      if (cps == 2) { B = 32768; S = 3; }
      size_t smem = 256 + (size_t)S * B; int grid = nsm * cps;
      size_t npc = N / grid / (B / 8) * (B / 8);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a); k_bulk_split<<<grid, 256, smem>>>(src, npc, S, B, parts, out); cudaEventRecord(b); cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
      }
      printf("split parts=%2d cta/sm=%d B=%u S=%d: %.0f GB/s\n", parts, cps, B, S, npc * grid * 8 / ms / 1e6);
    }
  cudaError_t e = cudaGetLastError(); printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
