// FP64 throughput microbenchmark for the roofline denominator (B200, sm_100a).
// DFMA: independent FMA chains per thread; DMMA: mma.sync.m16n8k4 f64 (and m8n8k4).
// Prints JSON with TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_kernel(double *out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 123.456) out[threadIdx.x] = s;
}

__global__ void dmma_k4_kernel(double *out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-6, a1 = 0.5, b0 = 0.25;
  double c[4][4];
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 123.456) out[threadIdx.x] = s;
}

__global__ void dmma_k16_kernel(double *out, int iters) {
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-6 + i;
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i;
  double c[2][4];
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 123.456) out[threadIdx.x] = s;
}

int main() {
  double *d;
  cudaMalloc(&d, 1 << 20);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // DFMA: 8 chains, 256 threads, 4 CTAs/SM
  int iters = 20000;
  dim3 grid(sms * 8), blk(256);
  dfma_kernel<8><<<grid, blk>>>(d, 100, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  dfma_kernel<8><<<grid, blk>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double dfma = 2.0 * 8 * iters * (double)grid.x * blk.x / (ms * 1e-3) / 1e12;
  // DMMA m16n8k4: 512 FMA per warp-instr, 4 independent accumulators
  int it2 = 20000;
  dmma_k4_kernel<<<grid, blk>>>(d, 100);
  cudaEventRecord(e0);
  dmma_k4_kernel<<<grid, blk>>>(d, it2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double dmma4 = 2.0 * 512 * 4 * it2 * (double)grid.x * (blk.x / 32) / (ms * 1e-3) / 1e12;
  dmma_k16_kernel<<<grid, blk>>>(d, 100);
  cudaEventRecord(e0);
  dmma_k16_kernel<<<grid, blk>>>(d, it2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double dmma16 = 2.0 * 2048 * 2 * it2 * (double)grid.x * (blk.x / 32) / (ms * 1e-3) / 1e12;
  cudaError_t err = cudaGetLastError();
  printf("{\"dfma_tflops\": %.3f, \"dmma_m16n8k4_tflops\": %.3f, \"dmma_m16n8k16_tflops\": %.3f, \"sms\": %d, \"err\": \"%s\"}\n",
         dfma, dmma4, dmma16, sms, cudaGetErrorString(err));
  return 0;
}
