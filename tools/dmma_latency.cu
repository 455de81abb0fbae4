// Microbenchmark: DMMA m8n8k4 f64 dependent-chain latency and per-SM issue
// throughput on sm_100a (development aid; informs the apply3d schedule).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void chain(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double d[CHAINS][2];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) d[c][0] = d[c][1] = c;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) dmma(d[c][0], d[c][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void dfma_chain(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4, d = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) d = fma(a, d, b);
  long long t1 = clock64();
  out[threadIdx.x] = d;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lds_chain(double* out, long long* cyc, int iters) {
  __shared__ double sm[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  int idx = threadIdx.x & 31;
  long long t0 = clock64();
  double v = 0;
  for (int i = 0; i < iters; ++i) {
    v += sm[idx];
    idx = (idx + (int)v) & 31;
  }
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void shfl_chain(double* out, long long* cyc, int iters) {
  double v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_down_sync(0xffffffffu, v, 1, 4);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 8);
  long long h;
  const int it = 4096;
  chain<1><<<1, 32>>>(out, cyc, it);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dmma dependent latency: %.1f cycles\n", (double)h / it);
  for (int w : {1, 2, 4, 8, 16}) {
    chain<4><<<1, 32 * w>>>(out, cyc, it);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dmma 4 chains, %2d warps/SM: %.2f cycles per dmma per SM\n", w, (double)h / (it * 4.0 * w));
  }
  for (int w : {4, 8, 16}) {
    chain<8><<<1, 32 * w>>>(out, cyc, it);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dmma 8 chains, %2d warps/SM: %.2f cycles per dmma per SM\n", w, (double)h / (it * 8.0 * w));
  }
  dfma_chain<<<1, 32>>>(out, cyc, it);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dfma dependent latency: %.1f cycles\n", (double)h / it);
  lds_chain<<<1, 32>>>(out, cyc, it);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("lds.64 + dadd dependent latency: %.1f cycles\n", (double)h / it);
  shfl_chain<<<1, 32>>>(out, cyc, it);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("shfl.64 (2x shfl) dependent latency: %.1f cycles\n", (double)h / it);
  return 0;
}
