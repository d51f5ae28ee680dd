// dmma_probe.cu -- microbenchmark (not product code): FP64 throughput of the
// vector pipe (DFMA) vs the FP64 MMA instruction (mma.sync m8n8k4 f64) on the
// GPU at hand, to size the next round's kernel design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe tools/dmma_probe.cu
//   ./dmma_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
  const double b = 1.0000001, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

// 4 independent accumulators per warp: D(8x8) += A(8x4) B(4x8), f64
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double d[4][2];
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k][0] = d[k][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
          : "+d"(d[k][0]), "+d"(d[k][1])
          : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1];
  if (s == 1.2345) out[0] = s;
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int block = 256, grid = sms * 8, iters = 4096;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fma = double(grid) * block * iters * 16;
    if (rep) printf("{\"dfma_per_s\": %.4g, \"fp64_tflops_vector\": %.2f}\n", fma / (ms * 1e-3),
                    2 * fma / (ms * 1e-3) / 1e12);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dmma_kernel<<<grid, block>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // one m8n8k4 = 8*8*4 FMA per warp
    const double fma = double(grid) * (block / 32) * iters * 4 * 256;
    if (rep) printf("{\"dmma_fma_per_s\": %.4g, \"fp64_tflops_mma\": %.2f, \"err\": \"%s\"}\n",
                    fma / (ms * 1e-3), 2 * fma / (ms * 1e-3) / 1e12,
                    cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
