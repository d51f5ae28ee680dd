// fp64_probe.cu -- microbenchmark (not product code): FP64 DFMA pipe rate on
// the GPU at hand vs resident warps per SM and operand source, plus DFMA and
// DMMA issued concurrently by different warps (is the FP64 MMA a separate
// pipe?). Sizes the compiled-pass design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

struct Consts { double k[64]; };

// MODE 0: b, c in registers; 1: 16 distinct literal constants per sweep
// (immediates: two UMOVs each); 2: constants from a kernel-parameter block
template <int MODE>
__global__ void dfma_kernel(double* out, int iters, Consts cs) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
  const double b = 1.0000001 + threadIdx.x * 1e-15, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) a[i] = fma(a[i], b, c);
      else if (MODE == 1) a[i] = fma(a[i], 1.0000001 + i * 0x1.123456789abcdp-40, 0x1.3456789abcdefp-30 * (i + 1));
      else a[i] = fma(a[i], cs.k[i], cs.k[i + 16]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

__device__ __forceinline__ void dmma4(double (&d)[4][2], double a, double b) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
}

// even warps DFMA, odd warps DMMA (or all DFMA / all DMMA)
__global__ void mixed_kernel(double* out, int iters, int mode) {
  const int w = threadIdx.x >> 5;
  const bool mma = mode == 2 || (mode == 1 && (w & 1));
  double s = 0;
  if (!mma) {
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-9 + i;
    const double b = 1.0000001, c = 1e-7;
    for (int it = 0; it < 4 * iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
  } else {
    double d[4][2] = {};
    const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
    for (int it = 0; it < iters; ++it) dmma4(d, a, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1];
  }
  if (s == 1.2345) out[0] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  f();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  Consts cs;
  for (int i = 0; i < 64; ++i) cs.k[i] = 1.0 + i * 1e-9;
  const int iters = 2048;
  printf("{\"sms\": %d, \"dfma\": [", sms);
  bool first = true;
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {4, 8, 16, 32, 64}) {
      const int block = 128;  // 4 warps per CTA, warps/4 CTAs per SM
      const int grid = sms * warps / 4;
      float ms = 0;
      if (mode == 0) ms = timeit([&] { dfma_kernel<0><<<grid, block>>>(out, iters, cs); });
      if (mode == 1) ms = timeit([&] { dfma_kernel<1><<<grid, block>>>(out, iters, cs); });
      if (mode == 2) ms = timeit([&] { dfma_kernel<2><<<grid, block>>>(out, iters, cs); });
      const double fma = double(grid) * block * iters * 16;
      printf("%s{\"operands\": \"%s\", \"warps_per_sm\": %d, \"dfma_per_s\": %.4g, \"per_sm_clk_at_1.9GHz\": %.1f}",
             first ? "" : ", ", mode == 0 ? "registers" : mode == 1 ? "literals" : "param_bank", warps,
             fma / (ms * 1e-3), fma / (ms * 1e-3) / sms / 1.9e9);
      first = false;
    }
  }
  printf("], \"mixed\": [");
  for (int mode = 0; mode < 3; ++mode) {
    const int block = 256, grid = sms * 2;  // 16 warps per SM
    const float ms = timeit([&] { mixed_kernel<<<grid, block>>>(out, iters, mode); });
    // DFMA warps: 4*iters*16 FMA per thread; DMMA warps: iters*4*256 FMA per warp
    const double nw = double(grid) * (block / 32);
    const double dfma_w = mode == 0 ? nw : mode == 1 ? nw / 2 : 0;
    const double dmma_w = nw - dfma_w;
    const double f = dfma_w * 32 * 4.0 * iters * 16 + dmma_w * iters * 4.0 * 256;
    printf("%s{\"mode\": \"%s\", \"ms\": %.3f, \"fma_per_s\": %.4g}", mode ? ", " : "",
           mode == 0 ? "all_dfma" : mode == 1 ? "half_dfma_half_dmma" : "all_dmma", ms, f / (ms * 1e-3));
  }
  printf("], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
