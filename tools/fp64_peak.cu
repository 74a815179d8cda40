// FP64 throughput microbenchmark for the roofline denominator (B200, sm_100a).
// DFMA: independent FMA chains per thread; DMMA: mma.sync.m16n8k4 f64 (and m8n8k4).
// Prints JSON with TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cstdlib>
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

// time `launch` once (burst) and back to back for `secs` seconds (sustained);
// returns {burst ms, sustained ms per launch}
template <class F>
static void time_it(F launch, double secs, float &burst, float &sustained) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();  // warm-up
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&burst, e0, e1);
  const int reps = secs > 0 ? (int)(secs * 1e3 / burst) + 1 : 1;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float tot = 0;
  cudaEventElapsedTime(&tot, e0, e1);
  sustained = tot / reps;
}

int main(int argc, char **argv) {
  const double secs = argc > 1 ? atof(argv[1]) : 0.0;  // sustained window per kernel
  double *d;
  cudaMalloc(&d, 1 << 20);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  const int iters = 20000;
  dim3 grid(sms * 8), blk(256);
  float b1, s1, b2, s2, b3, s3;
  // DFMA: 8 chains, 256 threads, 8 CTAs/SM
  time_it([&] { dfma_kernel<8><<<grid, blk>>>(d, iters, 1.0000001, 1e-9); }, secs, b1, s1);
  const double fl_dfma = 2.0 * 8 * iters * (double)grid.x * blk.x;
  // DMMA m16n8k4: 512 FMA per warp-instruction, 4 independent accumulators
  time_it([&] { dmma_k4_kernel<<<grid, blk>>>(d, iters); }, secs, b2, s2);
  const double fl_k4 = 2.0 * 512 * 4 * iters * (double)grid.x * (blk.x / 32);
  time_it([&] { dmma_k16_kernel<<<grid, blk>>>(d, iters); }, secs, b3, s3);
  const double fl_k16 = 2.0 * 2048 * 2 * iters * (double)grid.x * (blk.x / 32);
  cudaError_t err = cudaGetLastError();
  printf("{\"dfma_tflops\": %.3f, \"dmma_m16n8k4_tflops\": %.3f, \"dmma_m16n8k16_tflops\": %.3f, "
         "\"dfma_tflops_sustained\": %.3f, \"dmma_m16n8k4_tflops_sustained\": %.3f, "
         "\"dmma_m16n8k16_tflops_sustained\": %.3f, \"sustained_seconds_per_kernel\": %.1f, \"sms\": %d, \"err\": \"%s\"}\n",
         fl_dfma / (b1 * 1e-3) / 1e12, fl_k4 / (b2 * 1e-3) / 1e12, fl_k16 / (b3 * 1e-3) / 1e12,
         fl_dfma / (s1 * 1e-3) / 1e12, fl_k4 / (s2 * 1e-3) / 1e12, fl_k16 / (s3 * 1e-3) / 1e12, secs, sms,
         cudaGetErrorString(err));
  return 0;
}
