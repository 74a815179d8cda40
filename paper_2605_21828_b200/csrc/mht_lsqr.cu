// LSQR vector kernels for the inverse MHT (§7.1, Eq. inverse-MHT,
// "we use the BF-MHT within the LSQR iterative least squares
// algorithm").  The transforms of each iteration are the plan's own apply /
// adjoint; everything else of an iteration runs in the three kernels below,
// on the plan's stream, with every per-column scalar (alpha, beta, the Givens
// rotation, the norm estimates) kept on the device: the host only launches,
// and reads the scalars back at the convergence checks.
//
// Vectors use the ABI layout: column r of an n x k block is x[r * n + i].
// Norm reductions are two-pass (fixed per-block partials, then one block per
// column sums them in order): deterministic, no atomics.
#include <cuda_runtime.h>

#include "mht_internal.cuh"

namespace mht {
namespace {

constexpr int LT = 256;       // threads per block
constexpr int LPER = 8;       // elements per thread per block-pass

__device__ __forceinline__ double sq(double v) { return v * v; }
__device__ __forceinline__ double sq(double2 v) { return v.x * v.x + v.y * v.y; }
__device__ __forceinline__ double axpy_(double y, double s, double u) { return y - s * u; }
__device__ __forceinline__ double2 axpy_(double2 y, double s, double2 u) { return make_double2(y.x - s * u.x, y.y - s * u.y); }
__device__ __forceinline__ double scl(double v, double s) { return v * s; }
__device__ __forceinline__ double2 scl(double2 v, double s) { return make_double2(v.x * s, v.y * s); }
__device__ __forceinline__ double add_(double a, double b) { return a + b; }
__device__ __forceinline__ double2 add_(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }

__device__ double block_sum(double v) {
  __shared__ double red[LT / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < LT / 32; ++w) s += red[w];
  __syncthreads();
  return s;  // valid in thread 0
}

// u <- y - coef[r] * u (coef == nullptr: u <- y); partial ||u||^2 per block.
// grid (nblk, k)
template <class S>
__global__ void __launch_bounds__(LT) axpy_norm_kernel(const S *__restrict__ y, S *__restrict__ u, int64_t len,
                                                        const LsqrCol *__restrict__ col, int which,
                                                        double *__restrict__ partial) {
  const int r = blockIdx.y;
  const double s = col ? (which == 0 ? col[r].alpha : col[r].beta) : 0.0;
  const int64_t base = (int64_t)r * len;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * LT * LPER + threadIdx.x; i < len && i < (int64_t)(blockIdx.x + 1) * LT * LPER;
       i += LT) {
    const S v = col ? axpy_(y[base + i], s, u[base + i]) : y[base + i];  // col == nullptr: u <- y
    u[base + i] = v;
    acc += sq(v);
  }
  const double t = block_sum(acc);
  if (threadIdx.x == 0) partial[(int64_t)r * gridDim.x + blockIdx.x] = t;
}

// per column: norm = sqrt(sum of partials, in block order); stage 0 -> beta,
// stage 1 -> alpha and the plane rotation of the iteration; stage 2 / 3: the
// initial beta / alpha.  One block per column.
__global__ void __launch_bounds__(LT) scalars_kernel(const double *__restrict__ partial, int nblk, LsqrCol *col,
                                                     int stage) {
  const int r = blockIdx.x;
  double acc = 0.0;
  // fixed order: thread t sums blocks t, t + LT, ...; then the block reduction
  for (int b = threadIdx.x; b < nblk; b += LT) acc += partial[(int64_t)r * nblk + b];
  const double tot = block_sum(acc);
  if (threadIdx.x != 0) return;
  LsqrCol c = col[r];
  const double nrm = sqrt(tot);
  if (stage == 2) {  // beta_1 u_1 = b
    c.beta = nrm;
    c.bnorm = nrm;
    c.phibar = nrm;
    c.anorm2 = 0.0;
    c.cs = 1.0;
  } else if (stage == 3) {  // alpha_1 v_1 = A^* u_1
    c.alpha = nrm;
    c.rhobar = nrm;
  } else if (stage == 0) {  // beta_{i+1}
    c.beta = nrm;
    c.anorm2 += c.alpha * c.alpha + c.beta * c.beta;
  } else {  // alpha_{i+1}, then the rotation eliminating beta_{i+1}
    c.alpha = nrm;
    const double rho = hypot(c.rhobar, c.beta);
    const double cs = rho > 0 ? c.rhobar / rho : 1.0;
    const double sn = rho > 0 ? c.beta / rho : 0.0;
    const double theta = sn * c.alpha;
    c.rhobar = -cs * c.alpha;
    const double phi = cs * c.phibar;
    c.phibar = sn * c.phibar;
    c.cs = cs;
    c.step_x = rho > 0 ? phi / rho : 0.0;      // x += (phi / rho) w
    c.step_w = rho > 0 ? theta / rho : 0.0;    // w = v - (theta / rho) w
    c.rnorm = c.phibar;
    c.arnorm = c.phibar * c.alpha * fabs(cs);
  }
  col[r] = c;
}

// u <- u / (beta or alpha)  (norm 0: left as is); grid (nblk, k)
template <class S>
__global__ void __launch_bounds__(LT) scale_kernel(S *__restrict__ u, int64_t len, const LsqrCol *__restrict__ col,
                                                   int which) {
  const int r = blockIdx.y;
  const double nrm = which == 0 ? col[r].beta : col[r].alpha;
  const double s = nrm > 0 ? 1.0 / nrm : 1.0;
  const int64_t base = (int64_t)r * len;
  for (int64_t i = (int64_t)blockIdx.x * LT * LPER + threadIdx.x; i < len && i < (int64_t)(blockIdx.x + 1) * LT * LPER;
       i += LT)
    u[base + i] = scl(u[base + i], s);
}

// v <- v / alpha;  x <- x + step_x w;  w <- v - step_w w   (first == 1: w <- v, x <- 0)
template <class S>
__global__ void __launch_bounds__(LT) update_kernel(S *__restrict__ v, S *__restrict__ w, S *__restrict__ x,
                                                    int64_t len, const LsqrCol *__restrict__ col, int first) {
  const int r = blockIdx.y;
  const LsqrCol c = col[r];
  const double s = c.alpha > 0 ? 1.0 / c.alpha : 1.0;
  const int64_t base = (int64_t)r * len;
  for (int64_t i = (int64_t)blockIdx.x * LT * LPER + threadIdx.x; i < len && i < (int64_t)(blockIdx.x + 1) * LT * LPER;
       i += LT) {
    const S vv = scl(v[base + i], s);
    v[base + i] = vv;
    if (first) {
      w[base + i] = vv;
      x[base + i] = scl(vv, 0.0);
    } else {
      const S ww = w[base + i];
      x[base + i] = add_(x[base + i], scl(ww, c.step_x));
      w[base + i] = axpy_(vv, c.step_w, ww);
    }
  }
}

// ||x||^2 partials (convergence test 1)
template <class S>
__global__ void __launch_bounds__(LT) norm_kernel(const S *__restrict__ x, int64_t len, double *__restrict__ partial) {
  const int r = blockIdx.y;
  const int64_t base = (int64_t)r * len;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * LT * LPER + threadIdx.x; i < len && i < (int64_t)(blockIdx.x + 1) * LT * LPER;
       i += LT)
    acc += sq(x[base + i]);
  const double t = block_sum(acc);
  if (threadIdx.x == 0) partial[(int64_t)r * gridDim.x + blockIdx.x] = t;
}

__global__ void __launch_bounds__(LT) xnorm_kernel(const double *__restrict__ partial, int nblk, LsqrCol *col) {
  const int r = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < nblk; b += LT) acc += partial[(int64_t)r * nblk + b];
  const double tot = block_sum(acc);
  if (threadIdx.x == 0) col[r].xnorm = sqrt(tot);
}

inline int nblk_for(int64_t len) { return (int)((len + LT * LPER - 1) / (LT * LPER)); }

}  // namespace

int lsqr_partials(int64_t len) { return nblk_for(len); }

void lsqr_axpy_norm(bool cplx, const void *y, void *u, int64_t len, int k, const LsqrCol *col, int which,
                    double *partial, void *stream) {
  const dim3 g(nblk_for(len), k);
  cudaStream_t st = (cudaStream_t)stream;
  if (cplx)
    axpy_norm_kernel<double2><<<g, LT, 0, st>>>((const double2 *)y, (double2 *)u, len, col, which, partial);
  else
    axpy_norm_kernel<double><<<g, LT, 0, st>>>((const double *)y, (double *)u, len, col, which, partial);
}

void lsqr_scalars(const double *partial, int nblk, int k, LsqrCol *col, int stage, void *stream) {
  scalars_kernel<<<k, LT, 0, (cudaStream_t)stream>>>(partial, nblk, col, stage);
}

void lsqr_scale(bool cplx, void *u, int64_t len, int k, const LsqrCol *col, int which, void *stream) {
  const dim3 g(nblk_for(len), k);
  cudaStream_t st = (cudaStream_t)stream;
  if (cplx)
    scale_kernel<double2><<<g, LT, 0, st>>>((double2 *)u, len, col, which);
  else
    scale_kernel<double><<<g, LT, 0, st>>>((double *)u, len, col, which);
}

void lsqr_update(bool cplx, void *v, void *w, void *x, int64_t len, int k, const LsqrCol *col, int first,
                 void *stream) {
  const dim3 g(nblk_for(len), k);
  cudaStream_t st = (cudaStream_t)stream;
  if (cplx)
    update_kernel<double2><<<g, LT, 0, st>>>((double2 *)v, (double2 *)w, (double2 *)x, len, col, first);
  else
    update_kernel<double><<<g, LT, 0, st>>>((double *)v, (double *)w, (double *)x, len, col, first);
}

void lsqr_xnorm(bool cplx, const void *x, int64_t len, int k, double *partial, LsqrCol *col, void *stream) {
  const dim3 g(nblk_for(len), k);
  cudaStream_t st = (cudaStream_t)stream;
  if (cplx)
    norm_kernel<double2><<<g, LT, 0, st>>>((const double2 *)x, len, partial);
  else
    norm_kernel<double><<<g, LT, 0, st>>>((const double *)x, len, partial);
  xnorm_kernel<<<k, LT, 0, st>>>(partial, g.x, col);
}

}  // namespace mht
