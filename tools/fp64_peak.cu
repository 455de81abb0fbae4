// Microbenchmark: fp64 DFMA and DMMA (mma.sync m8n8k4 f64) peak on this GPU.
// Used once to fix the P64 roofline denominator, not part of the product.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main(int argc, char** argv) {
  // "sustained": DMMA kernels back to back for ~4 s, average rate
  if (argc > 1 && argv[1][0] == 's') {
    cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
    double* out; cudaMalloc(&out, 1 << 24);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = prop.multiProcessorCount * 4, threads = 256, iters = 2000, reps = 480;
    dmma_kernel<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * (blocks * threads / 32) * (double)iters * 16 * 4 * reps;
    printf("{\"dmma_tflops_sustained\": %.2f, \"ms\": %.1f}\n", flops / ms / 1e9, ms);
    return 0;
  }
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  printf("{\"name\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"clock_khz\": %d, \"mem_clock_khz\": %d, \"bus_bits\": %d, \"regs_per_sm\": %d}\n",
         prop.name, prop.multiProcessorCount, prop.l2CacheSize, prop.sharedMemPerBlockOptin, prop.clockRate,
         prop.memoryClockRate, prop.memoryBusWidth, prop.regsPerMultiprocessor);
  double* out; cudaMalloc(&out, 1 << 24);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = prop.multiProcessorCount;
  for (int rep = 0; rep < 3; ++rep) {
    int blocks = sms * 4, threads = 256, iters = 4000;
    dfma_kernel<<<blocks, threads>>>(out, 10, 0.999, 1e-3);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
    printf("{\"dfma_tflops\": %.2f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  for (int rep = 0; rep < 3; ++rep) {
    int blocks = sms * 4, threads = 256, iters = 2000;
    dmma_kernel<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * (blocks * threads / 32) * (double)iters * 16 * 4;
    printf("{\"dmma_tflops\": %.2f, \"ms\": %.3f}\n", flops / ms / 1e9, ms);
  }
  size_t n = (size_t)1 << 28;  // 4 GiB per buffer of double2? no: 2^28 * 16 B = 4 GiB
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"copy_gbs\": %.1f}\n", 2.0 * n * 16 / ms / 1e6);
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
