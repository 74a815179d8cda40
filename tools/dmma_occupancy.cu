// DMMA (mma.sync m16n8k4 f64) throughput vs resident warps per SM on the B200:
// does a kernel with 3 warps per SM sub-partition saturate the FP64 tensor pipe?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_occupancy tools/dmma_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void __launch_bounds__(128) k(double *out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-6, a1 = 0.5, b0 = 0.25;
  double c[ACC][4];
#pragma unroll
  for (int j = 0; j < ACC; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < ACC; ++j)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < ACC; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[j][i];
  if (s == 123.456) out[threadIdx.x] = s;
}

template <int ACC>
void run(double *d, int sms, int nb) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4000;
  k<ACC><<<sms * nb, 128>>>(d, 10);
  cudaEventRecord(e0);
  k<ACC><<<sms * nb, 128>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double tf = 2.0 * 512 * ACC * (double)iters * sms * nb * 4 / (ms * 1e-3) / 1e12;
  printf("{\"acc\": %d, \"ctas_per_sm\": %d, \"warps_per_sm\": %d, \"tflops\": %.2f}\n", ACC, nb, 4 * nb, tf);
}

int main() {
  double *d;
  cudaMalloc(&d, 1 << 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int nb : {1, 2, 3, 4, 6, 8, 16}) run<12>(d, sms, nb);
  for (int nb : {1, 2, 3, 4}) run<4>(d, sms, nb);
  for (int nb : {1, 2, 3, 4}) run<24>(d, sms, nb);
  return 0;
}
