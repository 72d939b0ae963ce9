// Pipe-peak microbenchmark for the roofline denominators that MEASURED_PEAKS.json
// does not carry: FP32 FFMA, FP64 DFMA, MUFU (rsqrt/rcp) throughput on one B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float v[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) v[k] = threadIdx.x * 1e-3f + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = fmaf(v[k], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += v[k];
  if (s == 123.456f) out[0] = s;
}

template <int ILP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double v[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) v[k] = threadIdx.x * 1e-3 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = fma(v[k], a, b);
  }
  double s = 0.;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += v[k];
  if (s == 123.456) out[0] = s;
}

// packed FP32x2 (sm_100a FFMA2): two FMAs per thread per instruction
template <int ILP>
__global__ void ffma2_kernel(float* out, int iters, float a, float b) {
  unsigned long long v[ILP], av, bv;
  {
    float2 t = make_float2(a, a), u = make_float2(b, b);
    av = *reinterpret_cast<unsigned long long*>(&t);
    bv = *reinterpret_cast<unsigned long long*>(&u);
  }
#pragma unroll
  for (int k = 0; k < ILP; ++k) {
    float2 t = make_float2(threadIdx.x * 1e-3f + k, k + 0.5f);
    v[k] = *reinterpret_cast<unsigned long long*>(&t);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[k]) : "l"(av), "l"(bv));
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < ILP; ++k) {
    float2 t = *reinterpret_cast<float2*>(&v[k]);
    s += t.x + t.y;
  }
  if (s == 123.456f) out[0] = s;
}

template <int ILP>
__global__ void mufu_kernel(float* out, int iters) {
  float v[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) v[k] = 1.0f + threadIdx.x * 1e-6f + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) v[k] = rsqrtf(v[k]);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += v[k];
  if (s == 123.456f) out[0] = s;
}

int main() {
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* fo; double* dfo;
  cudaMalloc(&fo, 16); cudaMalloc(&dfo, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = nsm * 8, threads = 256;
  const int iters = 4096;
  float ms;
  // FP32
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    ffma_kernel<8><<<blocks, threads>>>(fo, iters, 0.9999f, 1e-7f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double f32 = 2.0 * 8 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    ffma2_kernel<8><<<blocks, threads>>>(fo, iters, 0.9999f, 1e-7f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double f32x2 = 4.0 * 8 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
  // low occupancy (2 warps per scheduler, 2-way ILP): the k_interact regime
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    ffma_kernel<2><<<nsm * 2, 128>>>(fo, iters * 4, 0.9999f, 1e-7f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double f32_lo = 2.0 * 2 * (double)iters * 4 * nsm * 2 * 128 / (ms * 1e-3) / 1e12;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    ffma2_kernel<2><<<nsm * 2, 128>>>(fo, iters * 4, 0.9999f, 1e-7f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double f32x2_lo = 4.0 * 2 * (double)iters * 4 * nsm * 2 * 128 / (ms * 1e-3) / 1e12;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, threads>>>(dfo, iters / 4, 0.9999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double f64 = 2.0 * 8 * (double)(iters / 4) * blocks * threads / (ms * 1e-3) / 1e12;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    mufu_kernel<8><<<blocks, threads>>>(fo, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double mufu = 8.0 * (double)(iters / 4) * blocks * threads / (ms * 1e-3) / 1e12;
  printf("{\"sms\": %d, \"clock_mhz\": %d, \"fp32_tflops\": %.2f, \"fp64_tflops\": %.2f, \"mufu_rsqrt_tops\": %.3f, \"fp32x2_tflops\": %.2f, "
         "\"fp32_8warps_ilp2_tflops\": %.2f, \"fp32x2_8warps_ilp2_tflops\": %.2f}\n",
         nsm, clk / 1000, f32, f64, mufu, f32x2, f32_lo, f32x2_lo);
  return 0;
}
