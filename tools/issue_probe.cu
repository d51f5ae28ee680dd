// issue_probe.cu -- microbenchmark (not product code): do non-FP64
// instructions issue for free between DFMAs? Each loop iteration runs 16
// independent DFMAs plus X * 16 independent integer (LOP3) or uniform-move
// style instructions; the time per iteration vs X tells whether a DFMA holds
// the issue port for one cycle (time flat until X = 1) or two (time ~ 2 + X).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_probe tools/issue_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int XI>  // integer instructions per 16 DFMAs
__global__ void __launch_bounds__(512, 1) probe(double* out, unsigned* iout, int iters) {
  double a[16];
  unsigned z[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    a[i] = threadIdx.x * 1e-9 + i;
    z[i] = threadIdx.x * 2654435761u + i;
  }
  const double b = 1.0000001 + threadIdx.x * 1e-15, c = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[i]) : "d"(b), "d"(c));
      if (i * XI / 16 != (i + 1) * XI / 16 || XI >= 16) {
#pragma unroll
        for (int r = 0; r < (XI + 15) / 16; ++r)
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(z[(i + r) & 15]) : "r"(z[(i + 5 + r) & 15]), "r"(0x9e3779b9u + i));
      }
    }
  }
  double s = 0;
  unsigned q = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) { s += a[i]; q ^= z[i]; }
  if (s == 1.2345) out[0] = s;
  if (q == 0x12345u) iout[0] = q;
}

template <int XI>
void run(double* d, unsigned* di, int sms, const char* name) {
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int threads : {256, 512}) {
    probe<XI><<<sms, threads>>>(d, di, 1000);
    cudaEventRecord(e0);
    probe<XI><<<sms, threads>>>(d, di, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dfma = double(sms) * threads * 16.0 * iters;
    printf("%s threads %d: %.3f ms, %.3e DFMA/s, ns per 16-DFMA iteration per warp-slot %.2f\n", name, threads, ms,
           dfma / (ms * 1e-3), ms * 1e6 / iters);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  unsigned* di;
  cudaMalloc(&d, 8);
  cudaMalloc(&di, 8);
  run<0>(d, di, sms, "X=0   ");
  run<4>(d, di, sms, "X=0.25");
  run<8>(d, di, sms, "X=0.5 ");
  run<12>(d, di, sms, "X=0.75");
  run<16>(d, di, sms, "X=1   ");
  run<32>(d, di, sms, "X=2   ");
  run<48>(d, di, sms, "X=3   ");
  return 0;
}
