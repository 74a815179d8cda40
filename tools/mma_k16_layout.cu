// Determines the operand fragment layout of mma.sync.m16n8k16.f64 on the B200
// by testing candidate layouts against a host product (exact small integers).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/mma_k16_layout tools/mma_k16_layout.cu
#include <cstdio>
#include <cuda_runtime.h>

// candidate A layouts: slot i of lane (gid, tig) holds A[row][k]
__host__ __device__ inline void a_pos(int cand, int gid, int tig, int i, int &row, int &k) {
  if (cand == 0) {  // k8-style pairs: row gid + 8 (i & 1), k = tig + 4 (i >> 1)
    row = gid + 8 * (i & 1);
    k = tig + 4 * (i >> 1);
  } else {  // row gid + 8 (i >> 2), k = tig + 4 (i & 3)
    row = gid + 8 * (i >> 2);
    k = tig + 4 * (i & 3);
  }
}
__host__ __device__ inline void b_pos(int cand, int gid, int tig, int i, int &k, int &n) {
  if (cand == 0) {
    k = tig + 4 * i;
    n = gid;
  } else {
    k = 4 * tig + i;
    n = gid;
  }
}

__global__ void probe(const double *A, const double *B, double *C, int ca, int cb) {
  const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
  double a[8], b[4], c[4] = {0, 0, 0, 0};
  for (int i = 0; i < 8; ++i) {
    int r, k;
    a_pos(ca, gid, tig, i, r, k);
    a[i] = A[r * 16 + k];
  }
  for (int i = 0; i < 4; ++i) {
    int k, n;
    b_pos(cb, gid, tig, i, k, n);
    b[i] = B[k * 8 + n];
  }
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]), "d"(b[1]),
        "d"(b[2]), "d"(b[3]));
  // C fragment as for m16n8k4: c0,c1 row gid, cols 2 tig, 2 tig + 1; c2,c3 row gid + 8
  for (int v = 0; v < 4; ++v) C[(gid + 8 * (v >> 1)) * 8 + 2 * tig + (v & 1)] = c[v];
}

int main() {
  double hA[256], hB[128], hC[128], ref[128];
  for (int i = 0; i < 256; ++i) hA[i] = (i * 7 + 3) % 11 - 5;
  for (int i = 0; i < 128; ++i) hB[i] = (i * 5 + 1) % 9 - 4;
  for (int r = 0; r < 16; ++r)
    for (int n = 0; n < 8; ++n) {
      double s = 0;
      for (int k = 0; k < 16; ++k) s += hA[r * 16 + k] * hB[k * 8 + n];
      ref[r * 8 + n] = s;
    }
  double *dA, *dB, *dC;
  cudaMalloc(&dA, sizeof hA);
  cudaMalloc(&dB, sizeof hB);
  cudaMalloc(&dC, sizeof hC);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  for (int ca = 0; ca < 2; ++ca)
    for (int cb = 0; cb < 2; ++cb) {
      probe<<<1, 32>>>(dA, dB, dC, ca, cb);
      cudaMemcpy(hC, dC, sizeof hC, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int i = 0; i < 128; ++i) bad += hC[i] != ref[i];
      printf("{\"a_layout\": %d, \"b_layout\": %d, \"mismatches\": %d, \"err\": \"%s\"}\n", ca, cb, bad,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
