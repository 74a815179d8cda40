// Streaming-rate microbenchmark for the dataflow kernel's load path: one
// producer warp per CTA fills a ring of NS shared-memory slots of SLOT bytes
// from HBM; four consumer warps wait on each slot, read it (a sum over the
// slot, so the data is used) and release it.  Variants:
//   mode 0: 1-D TMA bulk copies (cp.async.bulk) of CB bytes each, issued by the
//           producer's 32 lanes;
//   mode 1: cp.async 16-byte copies issued by the producer's 32 lanes
//           (completion through cp.async.mbarrier.arrive.noinc);
//   mode 2: as mode 1, but a slot is SLOT / cb column segments of cb bytes of
//           a column-major factor block (column stride `stride` bytes): the
//           dataflow kernel's forward tile shape.  Unit u = row block
//           (u % nrb) of block (u / nrb), NCOL columns, dealt round robin.
//   mode 3: as mode 2, but a CTA walks whole units (all NCOL columns of its
//           row block, slot after slot) and takes units from a global
//           counter in (block, row block) order: the flow kernel's schedule;
//   direct: no ring — 128-thread CTAs (7 per SM) take the same units from a
//           counter and read them with ld.global.nc 16-byte loads, a warp
//           walking columns w, w + 4, ... 8 columns (16 loads per lane) ahead:
//           the per-stage nrhs = 1 kernel's access pattern.
// Reports GB/s over a 4 GiB buffer (far larger than L2), CUDA events, best of 5.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_stream tools/tma_stream.cu
//   tools/tma_stream > profiles/r02_tma_stream.txt
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_cp_async_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *smem, const void *gmem, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

template <int NS, int SLOT, int MODE>
__global__ void __launch_bounds__(160) stream_kernel(const char *src, int64_t nslots_total, unsigned cb,
                                                     double *sink, int64_t stride = 0, int nrb = 1, int ncol = 0) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + NS * SLOT);
  uint64_t *empty = full + NS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(full + i, MODE == 0 ? 1 : 64);
      mbar_init(empty + i, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // slots of this CTA: blockIdx.x, blockIdx.x + gridDim.x, ...
  int64_t mine = (nslots_total - blockIdx.x + gridDim.x - 1) / gridDim.x;
  __shared__ int64_t s_units;
  if (MODE == 3) {
    // the units this CTA takes are decided by the producer; the consumer learns
    // the slot count from a sentinel (a slot whose first word is -1)
    mine = INT64_MAX;
  }
  if (MODE == 3 && warp == 4) {
    const int spu = ncol / (SLOT / cb);
    const int64_t nunits = nslots_total / spu;
    int64_t it = 0;
    for (;;) {
      int64_t u = 0;
      if (lane == 0) u = atomicAdd(reinterpret_cast<unsigned long long *>(sink + 512), 1ull);
      u = __shfl_sync(0xffffffffu, u, 0);
      const bool stop = u >= nunits;
      for (int c = 0; c < (stop ? 1 : spu); ++c, ++it) {
        const int slot = it % NS;
        mbar_wait(empty + slot, ((it / NS) & 1) ^ 1);
        unsigned char *d = smem + slot * SLOT;
        if (stop) {
          if (lane == 0) *reinterpret_cast<long long *>(d) = -1;
        } else {
          const int64_t blk = u / nrb, rb = u % nrb;
          const char *base = src + blk * stride * ncol + rb * cb + (int64_t)c * (SLOT / cb) * stride;
          for (int j = 0; j < SLOT / (int)cb; ++j)
            for (int o = lane * 16; o < (int)cb; o += 512) {
              const unsigned s = (unsigned)__cvta_generic_to_shared(d + j * cb + o);
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(base + j * stride + o));
            }
        }
        mbar_cp_async_arrive(full + slot);
        mbar_arrive(full + slot);
      }
      if (stop) break;
    }
    return;
  }
  if (warp == 4) {
    for (int64_t it = 0; it < mine; ++it) {
      const int slot = it % NS;
      mbar_wait(empty + slot, ((it / NS) & 1) ^ 1);
      const char *g = src + (blockIdx.x + it * gridDim.x) * (int64_t)SLOT;
      unsigned char *d = smem + slot * SLOT;
      if (MODE == 0) {
        if (lane == 0) mbar_arrive_expect_tx(full + slot, SLOT);
        __syncwarp();
        for (int o = lane * cb; o < SLOT; o += 32 * cb) bulk_g2s(d + o, g + o, cb, full + slot);
      } else if (MODE == 3) {
        // handled by the unit loop below
      } else if (MODE == 2) {
        // slot index q of this CTA -> unit (block, row block) and column group
        const int64_t q = blockIdx.x + it * gridDim.x;
        const int spu = ncol / (SLOT / cb);            // slots per unit
        const int64_t unit = q / spu, cg = q % spu;
        const int64_t blk = unit / nrb, rb = unit % nrb;
        const char *base = src + blk * stride * ncol + rb * cb + cg * (SLOT / cb) * stride;
        for (int j = 0; j < SLOT / (int)cb; ++j)
          for (int o = lane * 16; o < (int)cb; o += 512) {
            const unsigned s = (unsigned)__cvta_generic_to_shared(d + j * cb + o);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(base + j * stride + o));
          }
        mbar_cp_async_arrive(full + slot);
        mbar_arrive(full + slot);
      } else {
        for (int o = lane * 16; o < SLOT; o += 512) {
          const unsigned s = (unsigned)__cvta_generic_to_shared(d + o);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g + o));
        }
        mbar_cp_async_arrive(full + slot);
        mbar_arrive(full + slot);
      }
    }
    return;
  }
  double acc = 0.0;
  for (int64_t it = 0; it < mine; ++it) {
    const int slot = it % NS;
    mbar_wait(full + slot, (it / NS) & 1);
    const double2 *p = reinterpret_cast<const double2 *>(smem + slot * SLOT);
    if (MODE == 3 && *reinterpret_cast<const long long *>(p) == -1) break;
    for (int i = threadIdx.x; i < SLOT / 16; i += 128) acc += p[i].x + p[i].y;
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + slot);
  }
  if (acc == 12345.678) sink[threadIdx.x] = acc;
}

__global__ void __launch_bounds__(128) direct_kernel(const char *src, int64_t nunits, int nrb, int ncol,
                                                     int64_t stride, double *sink, unsigned long long *ctr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __shared__ long long s_u;
  double acc = 0.0;
  for (;;) {
    if (threadIdx.x == 0) s_u = (long long)atomicAdd(ctr, 1ull);
    __syncthreads();
    const long long u = s_u;
    __syncthreads();
    if (u >= nunits) break;
    const int64_t blk = u / nrb, rb = u % nrb;
    const char *base = src + blk * stride * ncol + rb * 1024;
    for (int j0 = warp * 8; j0 < ncol; j0 += 32) {
      double2 t[16];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const char *col = base + (int64_t)(j0 + j) * stride;
        asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(t[2 * j].x), "=d"(t[2 * j].y) : "l"(col + lane * 16));
        asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(t[2 * j + 1].x), "=d"(t[2 * j + 1].y) : "l"(col + 512 + lane * 16));
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) acc += t[j].x + t[j].y;
    }
  }
  if (acc == 12345.678) sink[threadIdx.x] = acc;
}

void run_direct(const char *buf, int64_t bytes, double *sink) {
  const int64_t stride = 14400, ncol = 704, nrb = 14;
  const int64_t nunits = (bytes / (stride * ncol)) * nrb;
  int sms = 0, per = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, direct_kernel, 128, 0);
  per = per > 7 ? 7 : per;
  unsigned long long *ctr = reinterpret_cast<unsigned long long *>(sink + 512);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaMemset(ctr, 0, 8);
    cudaEventRecord(a);
    direct_kernel<<<sms * per, 128>>>(buf, nunits, nrb, ncol, stride, sink, ctr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
  printf("direct ld.global.nc  1024 B segments, %d CTAs/SM x 4 warps x 16 loads/lane: %7.1f GB/s\n", per,
         (double)nunits * 1024 * ncol / (best * 1e-3) / 1e9);
}

template <int NS, int SLOT, int MODE>
void run(const char *buf, int64_t bytes, unsigned cb, int ctas_per_sm, double *sink, int64_t stride = 0,
         int nrb = 1, int ncol = 0) {
  const int smem = NS * SLOT + 2 * NS * 8;
  cudaFuncSetAttribute(stream_kernel<NS, SLOT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, stream_kernel<NS, SLOT, MODE>, 160, smem);
  if (per < ctas_per_sm) {
    printf("mode %d NS %d SLOT %d cb %u: only %d CTAs/SM fit\n", MODE, NS, SLOT, cb, per);
    return;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * ctas_per_sm;
  int64_t nslots = bytes / SLOT;
  if (MODE >= 2) {  // whole blocks only
    const int64_t blk_bytes = stride * ncol;
    nslots = (bytes / blk_bytes) * nrb * (ncol / (SLOT / cb));
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaMemset(sink + 512, 0, 8);
    cudaEventRecord(a);
    stream_kernel<NS, SLOT, MODE><<<grid, 160, smem>>>(buf, nslots, cb, sink, stride, nrb, ncol);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (r > 0 && ms < best) best = ms;
  }
  cudaError_t e = cudaGetLastError();
  printf("mode %s  NS %2d  SLOT %6d  %s %6u B  CTAs/SM %d  in flight/SM %4d KB:  %7.1f GB/s %s\n",
         MODE == 0 ? "bulk   " : (MODE == 1 ? "cpasync" : (MODE == 2 ? "strided" : "units  ")), NS, SLOT, MODE >= 2 ? "segment" : "copy   ",
         MODE == 0 || MODE >= 2 ? cb : 16u, ctas_per_sm, NS * SLOT * ctas_per_sm / 1024,
         (double)nslots * SLOT / (best * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  const int64_t bytes = int64_t(4) << 30;
  char *buf = nullptr;
  double *sink = nullptr;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  cudaMalloc(&sink, 8192);
  run<6, 32768, 0>(buf, bytes, 512, 1, sink);
  run<6, 32768, 0>(buf, bytes, 1024, 1, sink);
  run<6, 32768, 0>(buf, bytes, 2048, 1, sink);
  run<6, 32768, 0>(buf, bytes, 4096, 1, sink);
  run<6, 32768, 0>(buf, bytes, 32768 / 32, 1, sink);
  run<3, 32768, 0>(buf, bytes, 1024, 2, sink);
  run<5, 16384, 0>(buf, bytes, 512, 2, sink);
  run<5, 16384, 0>(buf, bytes, 1024, 2, sink);
  run<12, 16384, 0>(buf, bytes, 1024, 1, sink);
  run<12, 16384, 0>(buf, bytes, 512, 1, sink);
  run<6, 32768, 1>(buf, bytes, 16, 1, sink);
  run<3, 32768, 1>(buf, bytes, 16, 2, sink);
  run<5, 16384, 1>(buf, bytes, 16, 2, sink);
  // strided column segments: column stride 14,400 B (a 900-row complex column), 700 columns per block
  for (int seg : {1024, 2048, 4096}) {
    const int nrb = 14400 / seg;
    run<3, 32768, 2>(buf, bytes, seg, 2, sink, 14400, nrb, 704);
    run<6, 32768, 2>(buf, bytes, seg, 1, sink, 14400, nrb, 704);
    run<3, 32768, 3>(buf, bytes, seg, 2, sink, 14400, nrb, 704);
  }
  run_direct(buf, bytes, sink);
  return 0;
}
