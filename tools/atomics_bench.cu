// Shared / global atomics throughput on sm_100a (the symmetric-PI feasibility check).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_atoms(float* out, int iters, int stride) {
  __shared__ float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0.f;
  __syncthreads();
  unsigned a = (threadIdx.x * stride) & 4095;
  float v = 1.0f + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    atomicAdd(&s[a], v);
    atomicAdd(&s[(a + 1024) & 4095], v);
    atomicAdd(&s[(a + 2048) & 4095], v);
    atomicAdd(&s[(a + 3072) & 4095], v);
    a = (a + 97) & 4095;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0] + s[4095];
}
__global__ void k_ffma(float* out, int iters) {
  float a = threadIdx.x, b = 1.0001f, c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
  for (int it = 0; it < iters; ++it) { c0 = fmaf(a, b, c0); c1 = fmaf(a, b, c1); c2 = fmaf(a, b, c2); c3 = fmaf(a, b, c3); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c0 + c1 + c2 + c3;
}
int main_a() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  for (int stride : {1, 33, 0}) {
    k_atoms<<<148 * 4, 256>>>(out, iters, stride);
    cudaEventRecord(e0);
    k_atoms<<<148 * 4, 256>>>(out, iters, stride);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = 148.0 * 4 * 256 * iters * 4;
    printf("ATOMS.F32 stride %d: %.3f ms, %.1f G atomics/s, %.2f per SM per clk (1.965 GHz)\n", stride, ms, n / ms / 1e6, n / (ms * 1e-3) / 148 / 1.965e9);
  }
  k_ffma<<<148 * 4, 256>>>(out, iters);
  cudaEventRecord(e0);
  k_ffma<<<148 * 4, 256>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = 148.0 * 4 * 256 * iters * 4;
  printf("FFMA: %.3f ms, %.2f per SM per clk\n", ms, n / (ms * 1e-3) / 148 / 1.965e9);
  return 0;
}
__global__ void k_atoms64(unsigned long long* out, int iters, int stride) {
  __shared__ unsigned long long s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned a = (threadIdx.x * stride) & 4095;
  unsigned long long v = 1 + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    atomicAdd(&s[a], v); atomicAdd(&s[(a + 1024) & 4095], v);
    atomicAdd(&s[(a + 2048) & 4095], v); atomicAdd(&s[(a + 3072) & 4095], v);
    a = (a + 97) & 4095;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0] + s[4095];
}
__global__ void k_atoms32(unsigned* out, int iters, int stride) {
  __shared__ unsigned s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
  __syncthreads();
  unsigned a = (threadIdx.x * stride) & 4095;
  unsigned v = 1 + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    atomicAdd(&s[a], v); atomicAdd(&s[(a + 1024) & 4095], v);
    atomicAdd(&s[(a + 2048) & 4095], v); atomicAdd(&s[(a + 3072) & 4095], v);
    a = (a + 97) & 4095;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0] + s[4095];
}
__global__ void k_red64(unsigned long long* g, long long n, int iters) {
  unsigned long long x = (blockIdx.x * 1024ull + threadIdx.x) * 2654435761ull;
  for (int it = 0; it < iters; ++it) {
    x = x * 6364136223846793005ull + 1442695040888963407ull;
    atomicAdd(&g[(x >> 20) % n], 1ull);
  }
}
__global__ void k_red64_seq(unsigned long long* g, long long n, int iters) {
  long long base = (long long)blockIdx.x * 256 * iters;
  for (int it = 0; it < iters; ++it) atomicAdd(&g[(base + it * 256 + threadIdx.x) % n], 1ull);
}
int main_b() {
  unsigned long long* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096; float ms;
  for (int w = 0; w < 2; ++w) {
    k_atoms64<<<148 * 4, 256>>>(out, iters, 1); cudaEventRecord(e0);
    k_atoms64<<<148 * 4, 256>>>(out, iters, 1); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double n = 148.0 * 4 * 256 * iters * 4;
    if (w) printf("ATOMS u64: %.2f per SM per clk\n", n / (ms * 1e-3) / 148 / 1.965e9);
    k_atoms32<<<148 * 4, 256>>>((unsigned*)out, iters, 1); cudaEventRecord(e0);
    k_atoms32<<<148 * 4, 256>>>((unsigned*)out, iters, 1); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (w) printf("ATOMS u32: %.2f per SM per clk\n", n / (ms * 1e-3) / 148 / 1.965e9);
  }
  long long n = 40ll << 20;  // 40M u64 = 320 MB
  unsigned long long* g; cudaMalloc(&g, n * 8); cudaMemset(g, 0, n * 8);
  int it2 = 256;
  for (int w = 0; w < 2; ++w) {
    k_red64<<<148 * 16, 1024>>>(g, n, it2); cudaEventRecord(e0);
    k_red64<<<148 * 16, 1024>>>(g, n, it2); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double na = 148.0 * 16 * 1024 * it2;
    if (w) printf("global RED u64 random over 320 MB: %.1f G/s\n", na / ms / 1e6);
    k_red64_seq<<<148 * 64, 256>>>(g, n, it2); cudaEventRecord(e0);
    k_red64_seq<<<148 * 64, 256>>>(g, n, it2); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    na = 148.0 * 64 * 256 * it2;
    if (w) printf("global RED u64 coalesced: %.1f G/s\n", na / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

int main() { main_a(); main_b(); return 0; }
