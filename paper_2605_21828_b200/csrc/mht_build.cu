// libmht plan-construction kernels (include/mht_build.h).
//
// The precompute of the butterfly factorization (§2; cost
// P:316-336) evaluates the selected submatrices Phi(tau, J) and takes their
// column interpolative decompositions (reading A5).  Three kernels run those
// steps on batches of blocks:
//   flat_blocks_kernel   Phi(rows, cols) = exp(i k.x) in-kernel
//   sphere_table_kernel  real orthonormal Y_lm by the normalised Legendre
//                        recurrence (reading A11)
//   cpqr_kernel          Householder QR with column pivoting, one CTA per
//                        block, exact norms after every reflector, rank rule
//                        |R_jj| <= tol |R_00| (reading A5)
// Outside the timed apply path; the host builder (precompute/gpu_builder.py)
// arranges the batches and writes the plan file.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "../../include/mht_build.h"

namespace mht {
mht_status set_error(mht_status s, const char *msg);  // mht_plan.cu (thread-local mht_last_error)
}

namespace {

using mht::set_error;

// ------------------------------------------------------------ flat blocks
// At[b][c][r] = exp(i (k[cols[b][c]] . x[rows[b][r]])), 0 on padding.  One
// thread per entry, r fastest (coalesced 16-byte stores).
__global__ void flat_blocks_kernel(const double *__restrict__ x, const double *__restrict__ k,
                                   const int64_t *__restrict__ rows, const int64_t *__restrict__ cols, int R, int C,
                                   int64_t total, double2 *__restrict__ At) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e % R;
    const int64_t bc = e / R;  // b * C + c
    const int64_t b = bc / C;
    const int64_t ri = rows[b * R + r], ci = cols[bc];
    double2 v = make_double2(0.0, 0.0);
    if (ri >= 0 && ci >= 0) {
      const double ph = k[2 * ci] * x[2 * ri] + k[2 * ci + 1] * x[2 * ri + 1];
      double s, c;
      sincos(ph, &s, &c);
      v = make_double2(c, s);
    }
    At[e] = v;
  }
}

// ------------------------------------------------------------ sphere table
// One CTA per point, thread mm = order |m| (0..lmax).  Thread mm forms
// P_mm^mm = sqrt((2m+1)/(2m)) sin(theta) P_{m-1}^{m-1} (P_0^0 = 1/sqrt(4 pi)),
// then P_{m+1}^m = sqrt(2m+3) cos(theta) P_m^m and
// P_l^m = a_lm (cos(theta) P_{l-1}^m - b_lm P_{l-2}^m),
// a_lm = sqrt((4l^2-1)/(l^2-m^2)), b_lm = sqrt(((l-1)^2-m^2)/(4(l-1)^2-1)),
// and writes Y_l,+-m.  At step l the active threads (mm <= l) write the
// contiguous runs l^2+l+mm and l^2+l-mm of the point's row.
__global__ void sphere_table_kernel(const double *__restrict__ theta, const double *__restrict__ phi, int lmax,
                                    double *__restrict__ Y) {
  const int64_t j = blockIdx.x;
  const int64_t M = (int64_t)(lmax + 1) * (lmax + 1);
  double *row = Y + j * M;
  const double ct = cos(theta[j]), st = sin(theta[j]);
  for (int mm = threadIdx.x; mm <= lmax; mm += blockDim.x) {
    double pmm = 1.0 / sqrt(4.0 * M_PI);
    for (int q = 1; q <= mm; ++q) pmm = sqrt((2.0 * q + 1.0) / (2.0 * q)) * st * pmm;
    double cm = 1.0, sm = 0.0;
    if (mm > 0) sincos(mm * phi[j], &sm, &cm);
    const double sc = mm == 0 ? 1.0 : sqrt(2.0);
    double p2 = 0.0, p1 = pmm;  // P_{l-2}^m, P_{l-1}^m
    for (int l = mm; l <= lmax; ++l) {
      double p;
      if (l == mm) {
        p = pmm;
      } else if (l == mm + 1) {
        p = sqrt(2.0 * mm + 3.0) * ct * pmm;
      } else {
        const double L2 = (double)l * l, m2 = (double)mm * mm, lm1 = l - 1.0;
        const double a = sqrt((4.0 * L2 - 1.0) / (L2 - m2));
        const double b = sqrt((lm1 * lm1 - m2) / (4.0 * lm1 * lm1 - 1.0));
        p = a * (ct * p1 - b * p2);
      }
      if (l > mm) {
        p2 = p1;
        p1 = p;
      }
      const int64_t base = (int64_t)l * l + l;
      if (mm == 0) {
        row[base] = p;
      } else {
        row[base + mm] = sc * p * cm;
        row[base - mm] = sc * p * sm;
      }
    }
  }
}

// ------------------------------------------------------------ CPQR
template <class S>
struct Q;
template <>
struct Q<double> {
  static __device__ __forceinline__ double zero() { return 0.0; }
  static __device__ __forceinline__ double abs2(double a) { return a * a; }
  static __device__ __forceinline__ double cdot(double v, double a) { return v * a; }  // conj(v) a
  static __device__ __forceinline__ double add(double a, double b) { return a + b; }
  static __device__ __forceinline__ double sub_mul(double a, double w, double v) { return a - w * v; }
  static __device__ __forceinline__ double scale(double a, double s) { return a * s; }
  static __device__ __forceinline__ double shfl_down(double a, int o) { return __shfl_down_sync(0xffffffffu, a, o); }
  // alpha = -phase(x0) * rjj (phase = sign, +1 at 0)
  static __device__ __forceinline__ double alpha(double x0, double rjj) { return x0 < 0 ? rjj : -rjj; }
};
template <>
struct Q<double2> {
  static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ double abs2(double2 a) { return a.x * a.x + a.y * a.y; }
  static __device__ __forceinline__ double2 cdot(double2 v, double2 a) {
    return make_double2(v.x * a.x + v.y * a.y, v.x * a.y - v.y * a.x);
  }
  static __device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
  static __device__ __forceinline__ double2 sub_mul(double2 a, double2 w, double2 v) {
    return make_double2(a.x - (w.x * v.x - w.y * v.y), a.y - (w.x * v.y + w.y * v.x));
  }
  static __device__ __forceinline__ double2 scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
  static __device__ __forceinline__ double2 shfl_down(double2 a, int o) {
    return make_double2(__shfl_down_sync(0xffffffffu, a.x, o), __shfl_down_sync(0xffffffffu, a.y, o));
  }
  // alpha = -(x0 / |x0|) rjj (phase 1 at x0 = 0)
  static __device__ __forceinline__ double2 alpha(double2 x0, double rjj) {
    const double ax = hypot(x0.x, x0.y);
    if (ax > 0) return make_double2(-x0.x / ax * rjj, -x0.y / ax * rjj);
    return make_double2(-rjj, 0.0);
  }
};

constexpr int QR_THREADS = 1024;
constexpr int QR_WARPS = QR_THREADS / 32;

template <class S>
__device__ __forceinline__ S warp_sum(S v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = Q<S>::add(v, Q<S>::shfl_down(v, o));
  return v;
}

// Block-wide sum of one double per thread (result valid in every thread).
__device__ __forceinline__ double block_sum(double v, double *scr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();  // scr free
  if (lane == 0) scr[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < QR_WARPS; ++w) s += scr[w];  // fixed order: deterministic
  return s;
}

// Dynamic shared memory: nrm[C] (squared column norms of the trailing rows),
// pv[C] (column permutation), then v[R] (the Householder vector) unless the
// block is too tall for it, in which case v lives in the global scratch
// vglob (R scalars per block; written and read by this CTA only, ordered by
// its barriers).
template <class S>
__global__ void __launch_bounds__(QR_THREADS, 1)
    cpqr_kernel(S *__restrict__ At, int C, int R, double tol, int64_t *__restrict__ ranks, int64_t *__restrict__ perm,
                S *vglob) {
  using X = Q<S>;
  extern __shared__ __align__(16) unsigned char qsm[];
  double *nrm = reinterpret_cast<double *>(qsm);
  int *pv = reinterpret_cast<int *>(nrm + C);
  S *v = vglob ? vglob + (int64_t)blockIdx.x * R
               : reinterpret_cast<S *>(qsm + (((size_t)C * (sizeof(double) + sizeof(int)) + 15) & ~(size_t)15));
  __shared__ double scr[QR_WARPS];
  __shared__ int scr_i[QR_WARPS];
  __shared__ int s_piv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  S *A = At + (int64_t)blockIdx.x * C * R;

  // squared column norms (one warp per column), identity permutation
  for (int c = warp; c < C; c += QR_WARPS) {
    const S *col = A + (int64_t)c * R;
    double s = 0.0;
    for (int r = lane; r < R; r += 32) s += X::abs2(col[r]);
    s = warp_sum(s);
    if (lane == 0) nrm[c] = s;
  }
  for (int c = tid; c < C; c += QR_THREADS) pv[c] = c;
  __syncthreads();
  double mx = 0.0;
  for (int c = tid; c < C; c += QR_THREADS) mx = fmax(mx, nrm[c]);
  // block max
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if (lane == 0) scr[warp] = mx;
  __syncthreads();
  double r00sq = 0.0;
  for (int w = 0; w < QR_WARPS; ++w) r00sq = fmax(r00sq, scr[w]);
  const double thr = tol * sqrt(r00sq);
  const int kmax = min(R, C);
  int rank = kmax;

  for (int j = 0; j < kmax; ++j) {
    // pivot: first column of largest remaining norm among positions j..C-1
    double best = -1.0;
    int bi = C;
    for (int c = j + tid; c < C; c += QR_THREADS)
      if (nrm[c] > best) best = nrm[c], bi = c;  // c increasing: keeps the first of ties
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_down_sync(0xffffffffu, best, o);
      const int oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) best = ob, bi = oi;
    }
    __syncthreads();  // scr / scr_i free (previous readers done)
    if (lane == 0) scr[warp] = best, scr_i[warp] = bi;
    __syncthreads();
    if (tid == 0) {
      double bb = scr[0];
      int ii = scr_i[0];
      for (int w = 1; w < QR_WARPS; ++w)
        if (scr[w] > bb || (scr[w] == bb && scr_i[w] < ii)) bb = scr[w], ii = scr_i[w];
      s_piv = ii;
    }
    __syncthreads();
    const int p = s_piv;
    if (p != j) {
      S *cj = A + (int64_t)j * R, *cp = A + (int64_t)p * R;
      for (int r = tid; r < R; r += QR_THREADS) {
        const S t = cj[r];
        cj[r] = cp[r];
        cp[r] = t;
      }
      if (tid == 0) {
        const double tn = nrm[j];
        nrm[j] = nrm[p];
        nrm[p] = tn;
        const int tp = pv[j];
        pv[j] = pv[p];
        pv[p] = tp;
      }
    }
    __syncthreads();
    const double rjj = sqrt(fmax(nrm[j], 0.0));
    if (rjj <= thr) {  // same smem value in every thread: uniform exit
      rank = j;
      break;
    }
    // Householder vector of x = A[j:, j]: v = (x - alpha e_0) / |x - alpha e_0|
    S *cj = A + (int64_t)j * R;
    const S alpha = X::alpha(cj[j], rjj);
    double s = 0.0;
    for (int r = j + tid; r < R; r += QR_THREADS) {
      S t = cj[r];
      if (r == j) t = X::add(t, X::scale(alpha, -1.0));
      v[r - j] = t;
      s += X::abs2(t);
    }
    const double vn = sqrt(block_sum(s, scr));
    const double inv = vn > 0 ? 1.0 / vn : 1.0;
    for (int r = j + tid; r < R; r += QR_THREADS) v[r - j] = X::scale(v[r - j], inv);
    __syncthreads();
    // trailing columns: a <- a - 2 (v^H a) v, then the norm of rows j+1..
    for (int c = j + 1 + warp; c < C; c += QR_WARPS) {
      S *col = A + (int64_t)c * R;
      S w = X::zero();
      for (int r = j + lane; r < R; r += 32) w = X::add(w, X::cdot(v[r - j], col[r]));
      w = warp_sum(w);  // lane 0 holds the total: broadcast it
      if constexpr (sizeof(S) == 16) {
        w.x = __shfl_sync(0xffffffffu, w.x, 0);
        w.y = __shfl_sync(0xffffffffu, w.y, 0);
      } else {
        w = __shfl_sync(0xffffffffu, w, 0);
      }
      w = X::scale(w, 2.0);
      double ns = 0.0;
      for (int r = j + lane; r < R; r += 32) {
        const S a = X::sub_mul(col[r], w, v[r - j]);
        col[r] = a;
        if (r > j) ns += X::abs2(a);
      }
      ns = warp_sum(ns);
      if (lane == 0) nrm[c] = ns;
    }
    for (int r = j + tid; r < R; r += QR_THREADS) cj[r] = r == j ? alpha : X::zero();
    __syncthreads();
  }
  if (tid == 0) ranks[blockIdx.x] = rank;
  for (int c = tid; c < C; c += QR_THREADS) perm[(int64_t)blockIdx.x * C + c] = pv[c];
}

inline cudaStream_t as_stream(void *s) { return static_cast<cudaStream_t>(s); }

mht_status cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return MHT_OK;
  static thread_local char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return set_error(e == cudaErrorMemoryAllocation ? MHT_ERR_OOM : MHT_ERR_CUDA, buf);
}

int grid_for(int64_t total, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (total + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * 16));
}

template <class S>
mht_status cpqr_launch(void *At, int B, int C, int R, double tol, int64_t *ranks, int64_t *perm, cudaStream_t st) {
  constexpr size_t kMaxSmem = 220u * 1024u;
  const size_t head = ((size_t)C * (sizeof(double) + sizeof(int)) + 15) & ~(size_t)15;
  if (head > kMaxSmem) return set_error(MHT_ERR_UNSUPPORTED, "mhtb_cpqr: too many columns for one CTA's shared memory");
  const bool v_smem = head + (size_t)R * sizeof(S) <= kMaxSmem;
  const size_t smem = v_smem ? head + (size_t)R * sizeof(S) : head;
  S *vglob = nullptr;
  if (!v_smem) {
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&vglob), (size_t)B * R * sizeof(S), st);
    if (e != cudaSuccess) return cuda_status(e, "mhtb_cpqr: scratch for the Householder vectors");
  }
  if (smem > 48u * 1024u) {
    // per call: the attribute applies to the device current when it is set
    const cudaError_t e = cudaFuncSetAttribute(cpqr_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(cpqr_kernel)");
  }
  cpqr_kernel<S><<<B, QR_THREADS, smem, st>>>(static_cast<S *>(At), C, R, tol, ranks, perm, vglob);
  const mht_status r = cuda_status(cudaGetLastError(), "cpqr_kernel launch");
  if (vglob) cudaFreeAsync(vglob, st);
  return r;
}

}  // namespace

extern "C" {

mht_status mhtb_flat_blocks(const double *x, const double *k, const int64_t *rows, const int64_t *cols, int B, int R,
                            int C, void *At, void *stream) {
  if (B < 0 || R < 0 || C < 0) return set_error(MHT_ERR_INVALID_ARG, "mhtb_flat_blocks: negative size");
  const int64_t total = (int64_t)B * C * R;
  if (total == 0) return MHT_OK;
  if (!x || !k || !rows || !cols || !At) return set_error(MHT_ERR_INVALID_ARG, "mhtb_flat_blocks: null pointer");
  flat_blocks_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(x, k, rows, cols, R, C, total,
                                                                          static_cast<double2 *>(At));
  return cuda_status(cudaGetLastError(), "flat_blocks_kernel launch");
}

mht_status mhtb_sphere_table(const double *theta, const double *phi, int64_t n, int lmax, double *Y, void *stream) {
  if (n < 0 || lmax < 0 || lmax > 2047) return set_error(MHT_ERR_INVALID_ARG, "mhtb_sphere_table: bad n or lmax");
  if (n == 0) return MHT_OK;
  if (!theta || !phi || !Y) return set_error(MHT_ERR_INVALID_ARG, "mhtb_sphere_table: null pointer");
  if (n > 0x7fffffff) return set_error(MHT_ERR_INVALID_ARG, "mhtb_sphere_table: n too large");
  const int threads = std::min(1024, ((lmax + 1 + 31) / 32) * 32);
  sphere_table_kernel<<<(unsigned)n, threads, 0, as_stream(stream)>>>(theta, phi, lmax, Y);
  return cuda_status(cudaGetLastError(), "sphere_table_kernel launch");
}

mht_status mhtb_cpqr(void *At, int B, int C, int R, int dtype, double tol, int64_t *ranks, int64_t *perm,
                     void *stream) {
  if (B < 0 || R < 0 || C < 0) return set_error(MHT_ERR_INVALID_ARG, "mhtb_cpqr: negative size");
  if (dtype != MHT_DTYPE_F64 && dtype != MHT_DTYPE_C128) return set_error(MHT_ERR_INVALID_ARG, "mhtb_cpqr: bad dtype");
  if (B == 0) return MHT_OK;
  if (!ranks || !perm || (!At && (int64_t)C * R > 0)) return set_error(MHT_ERR_INVALID_ARG, "mhtb_cpqr: null pointer");
  return dtype == MHT_DTYPE_C128 ? cpqr_launch<double2>(At, B, C, R, tol, ranks, perm, as_stream(stream))
                                 : cpqr_launch<double>(At, B, C, R, tol, ranks, perm, as_stream(stream));
}

}  // extern "C"
