// Throughput of the atomics a symmetric interaction kernel (K5s) would use on sm_100a:
//   * ATOMS.CAS.128: a float4 (ax, ay, az, drho) reaction added to a staged row in shared
//     memory by a 128-bit compare-and-swap loop (shared float atomics are CAS loops anyway);
//   * ATOMS.CAS.64 x2: the same with two 64-bit CAS loops;
//   * REDG.E.ADD.F32x4: the per-block flush of staged-row accumulators to global memory
//     (coalesced rows), and the same scattered;
//   * RED.MAX.U32 (global, coalesced): the viscous-dt maximum.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/atomics128 tools/atomics128_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void cas128_add(uint32_t addr, float4 c) {
  float4 old;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(old.x), "=f"(old.y), "=f"(old.z), "=f"(old.w) : "r"(addr) : "memory");
  while (true) {
    unsigned long long o0 = ((unsigned long long)__float_as_uint(old.y) << 32) | __float_as_uint(old.x);
    unsigned long long o1 = ((unsigned long long)__float_as_uint(old.w) << 32) | __float_as_uint(old.z);
    unsigned long long n0 = ((unsigned long long)__float_as_uint(old.y + c.y) << 32) | __float_as_uint(old.x + c.x);
    unsigned long long n1 = ((unsigned long long)__float_as_uint(old.w + c.w) << 32) | __float_as_uint(old.z + c.z);
    unsigned long long r0, r1;
    asm volatile("{ .reg .b128 d, cmp, val; mov.b128 cmp, {%2, %3}; mov.b128 val, {%4, %5};"
                 " atom.shared.cas.b128 d, [%6], cmp, val; mov.b128 {%0, %1}, d; }"
                 : "=l"(r0), "=l"(r1) : "l"(o0), "l"(o1), "l"(n0), "l"(n1), "r"(addr) : "memory");
    if (r0 == o0 && r1 == o1) break;
    old = make_float4(__uint_as_float((unsigned)r0), __uint_as_float((unsigned)(r0 >> 32)),
                      __uint_as_float((unsigned)r1), __uint_as_float((unsigned)(r1 >> 32)));
  }
}

__device__ __forceinline__ void cas64_add(uint32_t addr, float a, float b) {
  unsigned long long old;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(old) : "r"(addr) : "memory");
  while (true) {
    float x = __uint_as_float((unsigned)old) + a, y = __uint_as_float((unsigned)(old >> 32)) + b;
    unsigned long long nw = ((unsigned long long)__float_as_uint(y) << 32) | __float_as_uint(x);
    unsigned long long r;
    asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(r) : "r"(addr), "l"(old), "l"(nw) : "memory");
    if (r == old) break;
    old = r;
  }
}

template <int MODE>
__global__ void k_smem(float* out, int iters, int spread) {
  __shared__ __align__(16) float4 s[3072];
  for (int i = threadIdx.x; i < 3072; i += blockDim.x) s[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  uint32_t x = threadIdx.x * 2654435761u + blockIdx.x;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(s);
  const float4 c = make_float4(1.f, 2.f, 3.f, 4.f);
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    const uint32_t row = spread ? (x >> 20) % 3072u : (threadIdx.x & 31);
    const uint32_t a = base + 16u * row;
    if (MODE == 0) cas128_add(a, c);
    else { cas64_add(a, c.x, c.y); cas64_add(a + 8, c.z, c.w); }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[7].x + s[3000].w;
}

__global__ void k_red4(float4* g, long long nrows, int iters, int scattered) {
  for (int it = 0; it < iters; ++it) {
    long long r;
    if (scattered) {
      unsigned long long x = ((blockIdx.x * 1024ull + threadIdx.x) * 2654435761ull) ^ (it * 0x9E3779B97F4A7C15ull);
      x = x * 6364136223846793005ull + 1442695040888963407ull;
      r = (long long)((x >> 20) % nrows);
    } else {
      r = ((long long)blockIdx.x * iters + it) * blockDim.x + threadIdx.x;
      r %= nrows;
    }
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(g + r), "f"(1.f), "f"(2.f),
                 "f"(3.f), "f"(4.f) : "memory");
  }
}

__global__ void k_redmax(unsigned* g, long long n, int iters) {
  for (int it = 0; it < iters; ++it) {
    long long r = (((long long)blockIdx.x * iters + it) * blockDim.x + threadIdx.x) % n;
    asm volatile("red.global.max.u32 [%0], %1;" ::"l"(g + r), "r"(threadIdx.x) : "memory");
  }
}

int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  float* out;
  cudaMalloc(&out, 1 << 20);
  const double clk = 1.965e9;
  const int iters = 2048;
  for (int spread = 1; spread >= 0; --spread) {
    for (int w = 0; w < 2; ++w) {
      k_smem<0><<<148, 384>>>(out, iters, spread);
      cudaEventRecord(e0);
      k_smem<0><<<148, 384>>>(out, iters, spread);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double n = 148.0 * 384 * iters;
      if (w) printf("ATOMS.CAS.128 float4 add (%s): %.2f per SM per clk\n",
                    spread ? "random rows of 3072" : "32 rows, every warp on the same 32",
                    n / (ms * 1e-3) / 148 / clk);
      k_smem<1><<<148, 384>>>(out, iters, spread);
      cudaEventRecord(e0);
      k_smem<1><<<148, 384>>>(out, iters, spread);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (w) printf("2x ATOMS.CAS.64 float4 add (%s): %.2f float4 per SM per clk\n",
                    spread ? "random rows" : "32 rows", n / (ms * 1e-3) / 148 / clk);
    }
  }
  long long nrows = 12ll << 20;  // 12M float4 rows = 192 MB (> L2)
  float4* g;
  cudaMalloc(&g, nrows * 16);
  cudaMemset(g, 0, nrows * 16);
  for (int sc = 0; sc < 2; ++sc)
    for (int w = 0; w < 2; ++w) {
      int it2 = 64;
      k_red4<<<148 * 16, 512>>>(g, nrows, it2, sc);
      cudaEventRecord(e0);
      k_red4<<<148 * 16, 512>>>(g, nrows, it2, sc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double n = 148.0 * 16 * 512 * it2;
      if (w) printf("REDG.F32x4 %s over 192 MB: %.1f G rows/s (%.0f GB/s of payload)\n",
                    sc ? "scattered" : "coalesced", n / ms / 1e6, n * 16 / ms / 1e6);
    }
  for (int w = 0; w < 2; ++w) {
    int it2 = 64;
    k_redmax<<<148 * 16, 512>>>((unsigned*)g, nrows * 4, it2);
    cudaEventRecord(e0);
    k_redmax<<<148 * 16, 512>>>((unsigned*)g, nrows * 4, it2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double n = 148.0 * 16 * 512 * it2;
    if (w) printf("RED.MAX.U32 coalesced: %.1f G/s\n", n / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
