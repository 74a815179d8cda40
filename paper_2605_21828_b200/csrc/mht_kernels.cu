// libmht device kernels (sm_100a): butterfly apply / adjoint stages.
//
// PAPER.md §2: every stage multiplies each stored factor once —
//   forward   out = in[skel] + T in[red]          (ID transfer, X = [I T] Pi)
//   adjoint   w[skel] = z,  w[red] = T^* z        (X^*; conjugate for complex)
// with in = [z(p,c1); z(p,c2)] gathered from two segments (level permutation
// fused into the load addressing) and the leaf stage's perm_x scatter fused
// into the store.  fp64 real (double) or complex (double2).
//
// nrhs = 1 is HBM-bound (0.5 flop/B complex): T is streamed once with 16-byte
// non-allocating loads, each warp reading 32 consecutive rows (512 B) of a
// column.  Multi-RHS reuses each T element for RB right-hand sides held in
// registers.
#include <cuda_runtime.h>

#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>

#include "mht_internal.cuh"

namespace cg = cooperative_groups;

namespace mht {
namespace {

constexpr unsigned FULL = 0xffffffffu;

// Programmatic dependent launch (the nrhs = 1 stage kernels): a CTA lets the
// next stage's grid start launching at once, prefetches its own factor lines
// into L2 (the factors never depend on the previous stage), and only then
// waits for the previous grid's results.  griddepcontrol.wait is a no-op for
// a launch without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// launch with the programmatic-stream-serialisation attribute (PDL) unless
// MHT_PDL=0; read per launch (graphs capture the attribute as a programmatic
// edge).  Every kernel launched this way calls pdl_wait() before its first
// access to memory an earlier kernel of the sequence writes or reads.
inline bool pdl_on() {
  const char *e = getenv("MHT_PDL");
  return !(e && atoi(e) == 0);
}
// the multi-RHS kernels: PDL only with MHT_PDL_MMA=1 (neutral on c2 / c3,
// 6% slower on c4's graph replay together with the 6-CTA real kernel,
// profiles/r01_mma_pdl_ab.txt); their griddepcontrol instructions are no-ops
// when launched without the attribute
inline bool pdl_mma_on() {
  const char *e = getenv("MHT_PDL_MMA");
  return e && atoi(e) == 1 && pdl_on();
}
template <class... KArgs, class... Args>
void launch_ex(bool use_pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
               Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, args...);
}
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  launch_ex(pdl_on(), kern, grid, block, 0, st, args...);
}
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

template <class S>
struct Tr;

template <>
struct Tr<double> {
  static __device__ __forceinline__ double zero() { return 0.0; }
  static __device__ __forceinline__ void fma(double &a, double t, double x) { a = ::fma(t, x, a); }
  static __device__ __forceinline__ void fmac(double &a, double t, double z) { a = ::fma(t, z, a); }
  static __device__ __forceinline__ double add(double a, double b) { return a + b; }
  static __device__ __forceinline__ double scale(double a, double d) { return a * d; }
  static __device__ __forceinline__ double shfl(double v, int s) { return __shfl_sync(FULL, v, s); }
  static __device__ __forceinline__ double shfl_xor(double v, int s) {
    return __shfl_xor_sync(FULL, v, s);
  }
  static __device__ __forceinline__ double ldcg(const double *p) { return __ldcg(p); }
  static __device__ __forceinline__ double ldT(const double *p) {
    double v;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
  }
  // two consecutive rows of a (16-byte aligned) real factor column
  static __device__ __forceinline__ double2 ldT2(const double *p) {
    double2 v;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
  }
};

template <>
struct Tr<double2> {
  static __device__ __forceinline__ double2 zero() { return make_double2(0.0, 0.0); }
  // a += t * x
  static __device__ __forceinline__ void fma(double2 &a, double2 t, double2 x) {
    a.x = ::fma(t.x, x.x, a.x);
    a.x = ::fma(-t.y, x.y, a.x);
    a.y = ::fma(t.x, x.y, a.y);
    a.y = ::fma(t.y, x.x, a.y);
  }
  // a += conj(t) * z
  static __device__ __forceinline__ void fmac(double2 &a, double2 t, double2 z) {
    a.x = ::fma(t.x, z.x, a.x);
    a.x = ::fma(t.y, z.y, a.x);
    a.y = ::fma(t.x, z.y, a.y);
    a.y = ::fma(-t.y, z.x, a.y);
  }
  static __device__ __forceinline__ double2 add(double2 a, double2 b) {
    return make_double2(a.x + b.x, a.y + b.y);
  }
  static __device__ __forceinline__ double2 scale(double2 a, double d) { return make_double2(a.x * d, a.y * d); }
  static __device__ __forceinline__ double2 shfl(double2 v, int s) {
    return make_double2(__shfl_sync(FULL, v.x, s), __shfl_sync(FULL, v.y, s));
  }
  static __device__ __forceinline__ double2 shfl_xor(double2 v, int s) {
    return make_double2(__shfl_xor_sync(FULL, v.x, s), __shfl_xor_sync(FULL, v.y, s));
  }
  static __device__ __forceinline__ double2 ldcg(const double2 *p) { return __ldcg(p); }
  static __device__ __forceinline__ double2 ldT(const double2 *p) {
    double2 v;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
  }
};

// in[q] for right-hand side r: two segments, each in c (ld m) or zpool (ld Zt).
// Coefficient-side diagonal (spectral filter F(lambda_k), GRF sqrt S(lambda_k),
// covariance S; §7.1, §7.2), fused into the
// loads of c (forward) and the stores of c (adjoint).
__device__ __forceinline__ double diag_at(const Ctx &cx, int64_t k) {
  const double d = cx.diag[k];
  return cx.diag_sqrt ? sqrt(d) : d;
}

// CG: read the workspace through L2 only (ld.global.cg).  The persistent
// kernel writes and reads workspace in different phases of ONE launch, and L1
// is not coherent: a line cached while reading one stage's z could be stale
// for the next stage's entries that share it.
template <class S, bool CG = false>
__device__ __forceinline__ S in_value(const Ctx &cx, const DevBlock &B, int q, int r) {
  const bool s1 = q >= B.seg_len[0];  // no dynamic indexing: keeps B in registers
  const int64_t off = s1 ? B.seg_off[1] + (q - B.seg_len[0]) : B.seg_off[0] + q;
  const int32_t src = s1 ? B.seg_src[1] : B.seg_src[0];
  if (src == SRC_C) {  // user layout: column-major
    const S v = static_cast<const S *>(cx.c)[r * cx.m + off];
    return cx.diag ? Tr<S>::scale(v, diag_at(cx, off)) : v;
  }
  const S *p = static_cast<const S *>(cx.z) + off * cx.nrhs + r;           // workspace: RHS-fastest
  if constexpr (CG) return Tr<S>::ldcg(p);
  return *p;
}

// ------------------------------------------------------------------------
// forward stage (nrhs = 1): one CTA per (block, 64-row tile[, column split]);
// 4 warps split the redundant columns, lane l owns rows l and l+32 of the
// tile.  Stages with too few row tiles to fill the GPU split the columns of
// large blocks (Tile.pad = group << 8 | split): every split writes its partial
// row sums to scratch and the last CTA of the group to arrive (atomic counter)
// adds them in split order — deterministic, no float atomics.
// ------------------------------------------------------------------------
// CG: workspace reads through L2 only (the persistent kernel; see in_value)
template <class S, bool CG, int FBT = 8>
__device__ __forceinline__ void fwd_tile(const Ctx &cx, const Tile tl) {
  using X = Tr<S>;
  const DevBlock B = cx.blocks[tl.blk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ra = tl.start + lane, rb = tl.start + 32 + lane;
  const bool va = lane < tl.count, vb = lane + 32 < tl.count;
  const bool split = tl.pad >= 0;
  int jbeg = 0, jend = B.n_red;
  if (split) {
    const int ks = B.pad;
    const int chunk = ((B.n_red + ks - 1) / ks + 31) & ~31;
    jbeg = (tl.pad & 255) * chunk;
    jend = min(B.n_red, jbeg + chunk);
  }
  S acc_a = X::zero(), acc_b = X::zero();
  const S *T = static_cast<const S *>(cx.coef) + B.coef_off;
  const int64_t ld = B.ld;
  // complex: lane owns rows l and l + 32 (one 16-byte load each); real: lane
  // owns the row pair 2l, 2l + 1 (one 16-byte load; columns are 16-byte
  // aligned by the loader's repack, the pad row is zero)
  constexpr bool REAL = sizeof(S) == 8;
  const bool vp = 2 * lane < tl.count;
  for (int j0 = jbeg + warp * 32; j0 < jend; j0 += FWD_THREADS) {
    const int j = j0 + lane;
    S xr = X::zero();
    if (j < jend) {
      const int q = (B.flags & F_RED_IOTA) ? j : cx.idx[B.red_off + j];
      xr = in_value<S, CG>(cx, B, q, 0);
    }
    const int jn = min(32, jend - j0);
    const S *col = T + (int64_t)j0 * ld;
    auto step = [&](int jj) {
      const S x = X::shfl(xr, jj);
      if constexpr (REAL) {
        // predicated load (not a branch) so the unrolled loads are all in flight
        const double2 t = vp ? Tr<double>::ldT2(reinterpret_cast<const double *>(col) + (int64_t)jj * ld + tl.start + 2 * lane)
                             : make_double2(0.0, 0.0);
        X::fma(acc_a, t.x, x);
        X::fma(acc_b, t.y, x);
      } else {
        const S ta = va ? X::ldT(col + (int64_t)jj * ld + ra) : X::zero();
        const S tb = vb ? X::ldT(col + (int64_t)jj * ld + rb) : X::zero();
        X::fma(acc_a, ta, x);
        X::fma(acc_b, tb, x);
      }
    };
    if (jn == 32) {
      if constexpr (REAL && FBT == 0) {
#pragma unroll 16
        for (int jj = 0; jj < 32; ++jj) step(jj);
      } else if constexpr (REAL) {
        // each batch's FB loads issued before the first use (the interleaved
        // form kept only ~4 loads outstanding per warp)
        constexpr int FB = FBT;
#pragma unroll
        for (int h = 0; h < 32; h += FB) {
          double2 t[FB];
#pragma unroll
          for (int jj = 0; jj < FB; ++jj)
            t[jj] = vp ? Tr<double>::ldT2(reinterpret_cast<const double *>(col) + (int64_t)(h + jj) * ld + tl.start + 2 * lane)
                       : make_double2(0.0, 0.0);
#pragma unroll
          for (int jj = 0; jj < FB; ++jj) {
            const S x = X::shfl(xr, h + jj);
            X::fma(acc_a, t[jj].x, x);
            X::fma(acc_b, t[jj].y, x);
          }
        }
      } else {
#pragma unroll 8
        for (int jj = 0; jj < 32; ++jj) step(jj);
      }
    } else {
      for (int jj = 0; jj < jn; ++jj) step(jj);
    }
  }
  __shared__ S red[FWD_THREADS / 32][FWD_ROWS];
  __shared__ int last;
  if constexpr (REAL) {
    red[warp][2 * lane] = acc_a;
    red[warp][2 * lane + 1] = acc_b;
  } else {
    red[warp][lane] = acc_a;
    red[warp][lane + 32] = acc_b;
  }
  __syncthreads();
  S *scratch = static_cast<S *>(cx.fsplit);
  const int grp = tl.pad >> 8;
  if (split) {
    for (int i = threadIdx.x; i < FWD_ROWS; i += FWD_THREADS) {
      S sum = red[0][i];
#pragma unroll
      for (int w = 1; w < FWD_THREADS / 32; ++w) sum = X::add(sum, red[w][i]);
      scratch[B.fsp_off + ((int64_t)(tl.start / FWD_ROWS) * B.pad + (tl.pad & 255)) * FWD_ROWS + i] = sum;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(cx.fcount + grp, 1) == B.pad - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
  }
  for (int i = threadIdx.x; i < FWD_ROWS; i += FWD_THREADS) {
    if (i >= tl.count) continue;
    S s;
    if (split) {
      s = X::zero();
      for (int k = 0; k < B.pad; ++k) {
        const S *p = scratch + B.fsp_off + ((int64_t)(tl.start / FWD_ROWS) * B.pad + k) * FWD_ROWS + i;
        s = X::add(s, X::ldcg(p));
      }
    } else {
      s = red[0][i];
#pragma unroll
      for (int w = 1; w < FWD_THREADS / 32; ++w) s = X::add(s, red[w][i]);
    }
    const int row = tl.start + i;
    if (row < B.n_skel) {
      const int q = (B.flags & F_SKEL_IOTA) ? row : cx.idx[B.skel_off + row];
      s = X::add(s, in_value<S, CG>(cx, B, q, 0));
    }
    if (B.flags & F_OUT_F)
      static_cast<S *>(cx.fout)[cx.perm[B.out_off + row]] = s;
    else
      static_cast<S *>(cx.z)[B.out_off + row] = s;
  }
  if (split && threadIdx.x == 0) cx.fcount[grp] = 0;  // re-arm for the next apply
}

template <class S, int FBT = 8>
__global__ void __launch_bounds__(FWD_THREADS) fwd_kernel(const Ctx cx, const Tile *__restrict__ tiles) {
  const Tile tl = tiles[blockIdx.y];
  pdl_trigger();
  {
    // L2 prefetch of this warp's first 32 factor columns (the tile's rows)
    const DevBlock &B = cx.blocks[tl.blk];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int jbeg = 0;
    if (tl.pad >= 0) {
      const int ks = B.pad;
      jbeg = (tl.pad & 255) * ((((B.n_red + ks - 1) / ks) + 31) & ~31);
    }
    const int j = jbeg + warp * 32 + lane;
    if (j < B.n_red) {
      const char *col = reinterpret_cast<const char *>(static_cast<const S *>(cx.coef) + B.coef_off + (int64_t)j * B.ld +
                                                       tl.start);
      for (int o = 0; o < tl.count * (int)sizeof(S); o += 128) prefetch_l2(col + o);
    }
  }
  pdl_wait();
  fwd_tile<S, false, FBT>(cx, tl);
}

// real forward load batching: MHT_FWD_FB=0 (interleaved) | 8 (default) | 16
inline int fwd_fb() {
  static int v = [] {
    const char *e = getenv("MHT_FWD_FB");
    return e ? atoi(e) : 8;
  }();
  return v;
}

// adjoint input z[i] of a block: f through perm_x (leaf stage), else the group
// sum of its readers' partials (the adjoint of a block row that
// feeds two transfers is the sum of both), either summed here on load (fused:
// no separate reduction pass) or read from the zpool slot reduce_kernel wrote.
// The fused sum adds the partials in the same (reader id) order as
// reduce_kernel, so both paths are bitwise identical.
template <class S, bool CG = false>
__device__ __forceinline__ S adj_in(const Ctx &cx, const DevBlock &B, int i, int r, bool from_f) {
  if (from_f) return static_cast<const S *>(cx.fin)[r * cx.n + cx.perm[B.out_off + i]];
  if (cx.fused && B.rd_cnt >= 0) {
    const S *part = static_cast<const S *>(cx.part);
    S s = Tr<S>::zero();
    for (int k = 0; k < B.rd_cnt; ++k) {
      const S *p = part + (cx.rdtab[B.rd_off + k] + i) * cx.nrhs + r;
      s = Tr<S>::add(s, CG ? Tr<S>::ldcg(p) : *p);
    }
    return s;
  }
  const S *p = static_cast<const S *>(cx.z) + (B.out_off + i) * cx.nrhs + r;
  if constexpr (CG) return Tr<S>::ldcg(p);
  return *p;
}

// ------------------------------------------------------------------------
// adjoint stage (nrhs = 1): one CTA per (block, 32 complex / 64 real redundant
// columns[, row split]); warp w owns CPW columns and computes their conj-dot
// products with z over the tile's rows (staged through shared memory,
// ADJ_RCH at a time), reduced across lanes with shuffles.  Stages with too few
// column tiles to fill the GPU split the rows of tall blocks (Tile.pad =
// group << 8 | split, DevBlock.pad2 = split count): every split writes its
// partial column sums to scratch and the last CTA of the group to arrive adds
// them in split order (deterministic, no float atomics).
// ------------------------------------------------------------------------
template <class S, int RB, bool CG, int RCH = ADJ_RCH, bool AR2 = false>
__device__ __forceinline__ void adj_tile(const Ctx &cx, const Tile tl, int from_f, int rhs0) {
  using X = Tr<S>;
  // columns per warp: 8 complex / 16 real
  constexpr int ACOLS = adj_cols<S>();
  constexpr int CPW = ACOLS / (ADJ_THREADS / 32);
  const DevBlock B = cx.blocks[tl.blk];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool split = tl.pad >= 0;
  const int sidx = split ? (tl.pad & 255) : 0;
  int rbeg = 0, rend = B.r_out;
  if (split) {
    const int ks = B.pad2;
    const int chunk = ((B.r_out + ks - 1) / ks + 31) & ~31;
    rbeg = sidx * chunk;
    rend = min(B.r_out, rbeg + chunk);
  }
  __shared__ S zs[RCH][RB];
  S acc[CPW][RB];
#pragma unroll
  for (int u = 0; u < CPW; ++u)
#pragma unroll
    for (int k = 0; k < RB; ++k) acc[u][k] = X::zero();
  const S *T = static_cast<const S *>(cx.coef) + B.coef_off;
  const int64_t ld = B.ld;
  const int cbase = tl.start + warp * CPW;
  const int cend = tl.start + tl.count;
  constexpr bool REAL = sizeof(S) == 8;

  for (int rc = rbeg; rc < rend; rc += RCH) {
    const int rn = min(RCH, rend - rc);
    for (int e = threadIdx.x; e < rn * RB; e += ADJ_THREADS) {
      const int i = e % rn, k = e / rn;
      zs[i][k] = (rhs0 + k < cx.nrhs) ? adj_in<S, CG>(cx, B, rc + i, rhs0 + k, from_f) : X::zero();
    }
    if (REAL && (rn & 1) && threadIdx.x < RB) zs[rn][threadIdx.x] = X::zero();  // pair partner of the last row
    __syncthreads();
    if constexpr (REAL) {
      // real: lane takes the row pair (2q, 2q + 1) of each of its columns with
      // one 16-byte load (rc is even; the pad row of an odd r_out is zero)
      static_assert(!REAL || RB == 1, "real pair path is the nrhs = 1 kernel");
      if (cbase < cend && AR2) {
        // two row pairs per lane per step (2q, 2q + 1 and 2q + 64, 2q + 65):
        // 2 CPW 16-byte loads in flight
        for (int q = lane; 2 * q < rn; q += 64) {
          const bool v2 = 2 * (q + 32) < rn;
          const double z0 = zs[2 * q][0], z1 = zs[2 * q + 1][0];
          const double z2 = v2 ? zs[2 * q + 64][0] : 0.0, z3 = v2 ? zs[2 * q + 65][0] : 0.0;
          double2 t0[CPW], t1[CPW];
#pragma unroll
          for (int u = 0; u < CPW; ++u) {
            const bool cu = cbase + u < cend;
            const double *cp = reinterpret_cast<const double *>(T) + (int64_t)(cbase + u) * ld + rc + 2 * q;
            t0[u] = cu ? Tr<double>::ldT2(cp) : make_double2(0.0, 0.0);
            t1[u] = (cu && v2) ? Tr<double>::ldT2(cp + 64) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < CPW; ++u) {
            double &a = reinterpret_cast<double &>(acc[u][0]);
            a = ::fma(t0[u].x, z0, a);
            a = ::fma(t0[u].y, z1, a);
            a = ::fma(t1[u].x, z2, a);
            a = ::fma(t1[u].y, z3, a);
          }
        }
      } else if (cbase < cend) {
        for (int q = lane; 2 * q < rn; q += 32) {
          const double z0 = zs[2 * q][0], z1 = zs[2 * q + 1][0];
          // all CPW column loads issued before their first use (predicated)
          double2 t[CPW];
#pragma unroll
          for (int u = 0; u < CPW; ++u)
            t[u] = cbase + u < cend
                       ? Tr<double>::ldT2(reinterpret_cast<const double *>(T) + (int64_t)(cbase + u) * ld + rc + 2 * q)
                       : make_double2(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < CPW; ++u) {
            double &a = reinterpret_cast<double &>(acc[u][0]);
            a = ::fma(t[u].x, z0, a);
            a = ::fma(t[u].y, z1, a);
          }
        }
      }
    } else if (cbase < cend) {
      if constexpr (AR2) {
        // two rows per lane per step (i, i + 32): 2 CPW 16-byte loads in flight
        for (int i = lane; i < rn; i += 64) {
          const bool v2 = i + 32 < rn;
          const S z0 = zs[i][0], z1 = v2 ? zs[i + 32][0] : X::zero();
          S t0[CPW], t1[CPW];
#pragma unroll
          for (int u = 0; u < CPW; ++u) {
            const bool cu = cbase + u < cend;
            const S *cp = T + (int64_t)(cbase + u) * ld + rc + i;
            t0[u] = cu ? X::ldT(cp) : X::zero();
            t1[u] = (cu && v2) ? X::ldT(cp + 32) : X::zero();
          }
#pragma unroll
          for (int u = 0; u < CPW; ++u) {
            X::fmac(acc[u][0], t0[u], z0);
            X::fmac(acc[u][0], t1[u], z1);
          }
        }
      } else {
        for (int i = lane; i < rn; i += 32) {
          S zv[RB];
#pragma unroll
          for (int k = 0; k < RB; ++k) zv[k] = zs[i][k];
          S t[CPW];
#pragma unroll
          for (int u = 0; u < CPW; ++u) t[u] = cbase + u < cend ? X::ldT(T + (int64_t)(cbase + u) * ld + rc + i) : X::zero();
#pragma unroll
          for (int u = 0; u < CPW; ++u)
#pragma unroll
            for (int k = 0; k < RB; ++k) X::fmac(acc[u][k], t[u], zv[k]);
        }
      }
    }
    __syncthreads();
  }
  // skeleton part: w[skel[i]] = z[i]  (written once, by the block's first tile)
  if (tl.start == 0 && sidx == 0 && B.n_skel > 0) {
    for (int e = threadIdx.x; e < B.n_skel * RB; e += ADJ_THREADS) {
      const int i = e % B.n_skel, k = e / B.n_skel;
      if (rhs0 + k >= cx.nrhs) continue;
      const int q = (B.flags & F_SKEL_IOTA) ? i : cx.idx[B.skel_off + i];
      static_cast<S *>(cx.part)[(B.part_off + q) * cx.nrhs + rhs0 + k] = adj_in<S, CG>(cx, B, i, rhs0 + k, from_f);
    }
  }
  // warp reductions
#pragma unroll
  for (int u = 0; u < CPW; ++u)
#pragma unroll
    for (int k = 0; k < RB; ++k)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[u][k] = X::add(acc[u][k], X::shfl_xor(acc[u][k], o));
  if (!split) {
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < CPW; ++u) {
        const int col = cbase + u;
        if (col >= cend) continue;
        const int q = (B.flags & F_RED_IOTA) ? col : cx.idx[B.red_off + col];
#pragma unroll
        for (int k = 0; k < RB; ++k)
          if (rhs0 + k < cx.nrhs) static_cast<S *>(cx.part)[(B.part_off + q) * cx.nrhs + rhs0 + k] = acc[u][k];
      }
    }
  } else {
    // RB == 1 here (nrhs = 1 path)
    static_assert(RB == 1, "row splits are built for the nrhs = 1 tiles only");
    S *scratch = static_cast<S *>(cx.fsplit);
    const int grp = tl.pad >> 8;
    const int64_t sbase = B.asp_off + (int64_t)(tl.start / ACOLS) * B.pad2 * ACOLS;
    __shared__ int last;
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < CPW; ++u) scratch[sbase + (int64_t)sidx * ACOLS + warp * CPW + u] = acc[u][0];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(cx.fcount + grp, 1) == B.pad2 - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int c = threadIdx.x; c < tl.count; c += ADJ_THREADS) {
      S sum = X::zero();
      for (int k = 0; k < B.pad2; ++k) sum = X::add(sum, X::ldcg(scratch + sbase + (int64_t)k * ACOLS + c));
      const int col = tl.start + c;
      const int q = (B.flags & F_RED_IOTA) ? col : cx.idx[B.red_off + col];
      static_cast<S *>(cx.part)[(B.part_off + q) * cx.nrhs + rhs0] = sum;
    }
    if (threadIdx.x == 0) cx.fcount[grp] = 0;  // re-arm for the next apply
  }
}

template <class S, int RB, int RCH = ADJ_RCH, bool AR2 = false>
__global__ void __launch_bounds__(ADJ_THREADS, 7) adj_kernel(const Ctx cx, const Tile *__restrict__ tiles,
                                                             int from_f) {
  const Tile tl = tiles[blockIdx.y];
  pdl_trigger();
  {
    // L2 prefetch of the first 1 KB of each of this CTA's factor columns
    const DevBlock &B = cx.blocks[tl.blk];
    const int t = threadIdx.x;
    const int col = tl.start + (t >> 3), line = t & 7;
    if ((t >> 3) < tl.count) {
      int rbeg = 0;
      if (tl.pad >= 0) rbeg = (tl.pad & 255) * ((((B.r_out + B.pad2 - 1) / B.pad2) + 31) & ~31);
      const int64_t off = (int64_t)col * B.ld + rbeg;
      const char *p = reinterpret_cast<const char *>(static_cast<const S *>(cx.coef) + B.coef_off + off);
      if (line * 128 < (B.r_out - rbeg) * (int)sizeof(S)) prefetch_l2(p + line * 128);
    }
  }
  pdl_wait();
  adj_tile<S, RB, false, RCH, AR2>(cx, tl, from_f, blockIdx.x * RB);
}

// complex adjoint, two rows per lane per step (default; MHT_ADJ_AR2=0: one):
// c2 adj_nrhs1 6.60 -> 6.56 ms (profiles/r01_adj_ar2_ab.txt)
inline bool adj_ar2() {
  const char *e = getenv("MHT_ADJ_AR2");
  return !(e && atoi(e) == 0);
}

// rows of z staged per pass: MHT_ADJ_RCH=512|1024 (experiments), default ADJ_RCH
// real adjoint, two row pairs per lane per step: MHT_ADJ_AR2R=1
inline bool adj_ar2_real() {
  const char *e = getenv("MHT_ADJ_AR2R");
  return e && atoi(e) == 1;
}
inline int adj_rch() {
  static int v = [] {
    const char *e = getenv("MHT_ADJ_RCH");
    return e ? atoi(e) : ADJ_RCH;
  }();
  return v;
}

// ------------------------------------------------------------------------
// multi-RHS stages on the FP64 tensor pipe (DMMA, mma.sync m16n8k4 f64).
//
// Each block product is a dense contraction  OUT(M x N) = A(M x K) B(K x N):
//   forward  A = T (r_out x n_red),        B = in[red] (n_red x nrhs)
//   adjoint  A = T^* (n_red x r_out),      B = z       (r_out x nrhs)
// A CTA owns a 64-row M tile (4 warps x 16 rows) and 8*NT right-hand sides;
// K is streamed in chunks of 16 with a two-stage cp.async pipeline for the
// factor tile (the HBM stream) and register-staged gathers for B.  Shared
// memory holds both operands in mma-fragment order, so every fragment load is
// one contiguous 512-byte LDS.128 per warp (no bank conflicts).  Complex
// products are 4 real MMAs (re/im planes of the same fragments).
// ------------------------------------------------------------------------
constexpr int MM_BM = 64, MM_THREADS = 128;
template <class S>
__host__ __device__ constexpr int mm_bk() { return sizeof(S) == 16 ? 16 : 32; }

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b));
}

template <int BYTES>
__device__ __forceinline__ void cp_async(void *smem, const void *gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? BYTES : 0;  // src-size 0 -> zero fill
  if (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <class S>
struct Planes;  // re/im access for the MMA operands
template <>
struct Planes<double> {
  static constexpr bool cplx = false;
  static __device__ __forceinline__ double re(double v) { return v; }
  static __device__ __forceinline__ double im(double) { return 0.0; }
};
template <>
struct Planes<double2> {
  static constexpr bool cplx = true;
  static __device__ __forceinline__ double re(double2 v) { return v.x; }
  static __device__ __forceinline__ double im(double2 v) { return v.y; }
};

// M3: complex products by Gauss's 3-multiplication form (P1 = Ar Br, P2 = Ai Bi,
// P3 = (Ar + Ai)(Br + Bi); re = P1 - P2, im = P3 - P1 - P2) — 3 DMMAs instead of 4.
// MINB: CTAs per SM the register budget is sized for.
// barrier over the 128 consumer threads: __syncthreads (BAR = 0) in the
// classic kernel, named barrier 1 in the warp-specialised one (its producer
// warp does not take part in the epilogue)
template <int BAR>
__device__ __forceinline__ void consumer_sync() {
  if constexpr (BAR == 0)
    __syncthreads();
  else
    asm volatile("bar.sync 1, %0;" ::"n"(MM_THREADS) : "memory");
}

// Multi-RHS epilogue (threads 0..127): C fragments (row gid / gid + 8, cols
// 2 tig / 2 tig + 1) -> skeleton add and the output store (forward), partials
// (adjoint) or the K-split slabs with the last-CTA fixup.
// fragment row gid -> tile row, for the swizzled TMA adjoint tile (identity
// otherwise): consecutive gid pairs / quads land on rows whose 128-byte
// swizzle phases differ, so a quarter (16-byte) / half (8-byte) warp's
// A-fragment loads hit distinct banks
template <class S, bool PERM>
__host__ __device__ __forceinline__ int frag_row(int gid) {
  if (!PERM) return gid;
  return sizeof(S) == 16 ? 4 * (gid & 1) + (gid >> 1) : 2 * (gid & 3) + (gid >> 2);
}

// MMA row r (0..15, a0 rows 0..7, a1 rows 8..15) -> tile row within the warp's
// 16-row slab.  MODE 0: identity; 1: swizzled adjoint tile (frag_row, a1 = a0
// + 8); 2: swizzled real forward tile [k][16 rows] (quad q of rows -> tile rows
// {2q, 2q+1, 2q+8, 2q+9}: the half warp's 8-byte loads hit 16 distinct banks)
template <class S, int MODE>
__host__ __device__ __forceinline__ int tile_row(int r) {
  if (MODE == 0) return r;
  if (MODE == 1) return frag_row<S, true>(r & 7) + 8 * (r >> 3);
  return 2 * (r >> 2) + (r & 1) + 8 * ((r >> 1) & 1);
}

template <class S, bool ADJ, int NT, bool M3, int BAR, int MODE = 0>
__device__ __forceinline__ void mma_epilogue(const Ctx &cx, const Tile &tl, const DevBlock &B, double (&c0)[NT][4],
                                             double (&c1)[NT][4], double (&c2)[(Planes<S>::cplx && M3) ? NT : 1][4],
                                             int rhs0, bool ksplit, int sidx, int from_f, int *flag) {
  using X = Tr<S>;
  constexpr bool CPLX = Planes<S>::cplx;
  constexpr bool G3 = CPLX && M3;
  constexpr int NRT = 8 * NT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const bool red_iota = (B.flags & F_RED_IOTA) != 0;
  // a thread's fragments cover two tile rows (h = 0: gid, 1: gid + 8).  Every
  // index and skeleton load is issued before the first store: the stores
  // could alias the loaded arrays as far as the compiler knows, so
  // interleaving them serialised 2 + 4 NT dependent global round trips per
  // thread (c3 stage 3: 15 us per CTA, long_scoreboard 57%,
  // profiles/r01_epilogue_hoist_ab.txt)
  int mh[2], qh[2];
  bool okh[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    mh[h] = warp * 16 + tile_row<S, MODE>(gid + 8 * h);
    okh[h] = mh[h] < tl.count;
    const int row = tl.start + mh[h];
    if (!ADJ) {
      qh[h] = (okh[h] && row < B.n_skel) ? ((B.flags & F_SKEL_IOTA) ? row : cx.idx[B.skel_off + row]) : -1;
    } else if (ksplit) {
      qh[h] = 0;
    } else {
      qh[h] = okh[h] ? (red_iota ? row : cx.idx[B.red_off + row]) : 0;
    }
  }
  int oh[2] = {0, 0};  // forward leaf stage: output rows through perm_x
  if (!ADJ && (B.flags & F_OUT_F)) {
#pragma unroll
    for (int h = 0; h < 2; ++h) oh[h] = okh[h] ? cx.perm[B.out_off + tl.start + mh[h]] : 0;
  }
  // accumulators -> values first (the 3M form's three planes collapse to
  // one), so the skeleton loads below do not hold all of them live
  S val[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      if constexpr (!CPLX) {
        val[t][v] = c0[t][v];
      } else if constexpr (G3) {
        val[t][v] = make_double2(c0[t][v] - c1[t][v], c2[t][v] - c0[t][v] - c1[t][v]);
      } else {
        val[t][v] = make_double2(c0[t][v], c1[t][v]);
      }
    }
  if (!ADJ) {  // forward: out = T in[red] + in[skel]
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int r = rhs0 + t * 8 + 2 * tig + (v & 1);
        if (qh[v >> 1] >= 0 && r < cx.nrhs) val[t][v] = X::add(val[t][v], in_value<S>(cx, B, qh[v >> 1], r));
      }
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int h = v >> 1;
      const int m = mh[h];
      const int r = rhs0 + t * 8 + 2 * tig + (v & 1);
      if (!okh[h] || r >= cx.nrhs) continue;
      const int row = tl.start + m;
      if (!ADJ) {
        if (B.flags & F_OUT_F)
          static_cast<S *>(cx.fout)[r * cx.n + oh[h]] = val[t][v];
        else
          static_cast<S *>(cx.z)[(B.out_off + row) * cx.nrhs + r] = val[t][v];
      } else if (ksplit) {
        const int64_t slab = B.msp_off + (int64_t)(tl.start / MMA_COLS) * B.mks + sidx;
        static_cast<S *>(cx.msplit)[(slab * MMA_COLS + m) * cx.nrhs + r] = val[t][v];
      } else {
        static_cast<S *>(cx.part)[(B.part_off + qh[h]) * cx.nrhs + r] = val[t][v];
      }
    }
  }
  if (ADJ && sidx == 0 && B.n_skel > 0) {
    // skeleton part w[skel[i]] = z[i], spread over the block's column tiles
    // (tile j copies rows [j c, (j + 1) c)); a block without redundant
    // columns (COPY) has one tile that copies everything
    const int ntl = B.n_red > 0 ? (B.n_red + MMA_COLS - 1) / MMA_COLS : 1;
    const int chunk = (B.n_skel + ntl - 1) / ntl;
    const int i0 = (tl.start / MMA_COLS) * chunk, i1 = min(B.n_skel, i0 + chunk);
    const int ni = i1 - i0;
    // batches of SKB copies per thread, loads before stores (as above)
    constexpr int SKB = 4;
    for (int e0 = threadIdx.x; e0 < ni * NRT; e0 += SKB * MM_THREADS) {
      S v[SKB];
      int q[SKB];
#pragma unroll
      for (int u = 0; u < SKB; ++u) {
        const int e = e0 + u * MM_THREADS;
        const int i = i0 + e / NRT, r = rhs0 + e % NRT;  // RHS fastest: contiguous 32-wide rows
        const bool ok = e < ni * NRT && r < cx.nrhs;
        q[u] = !ok ? -1 : ((B.flags & F_SKEL_IOTA) ? i : cx.idx[B.skel_off + i]);
      }
#pragma unroll
      for (int u = 0; u < SKB; ++u) {
        const int e = e0 + u * MM_THREADS;
        v[u] = q[u] >= 0 ? adj_in<S>(cx, B, i0 + e / NRT, rhs0 + e % NRT, from_f != 0) : X::zero();
      }
#pragma unroll
      for (int u = 0; u < SKB; ++u) {
        const int e = e0 + u * MM_THREADS;
        if (q[u] >= 0) static_cast<S *>(cx.part)[(B.part_off + q[u]) * cx.nrhs + rhs0 + e % NRT] = v[u];
      }
    }
  }
  if (ADJ && ksplit) {
    // the last split of (block, column tile, RHS chunk) to arrive sums the
    // slabs in split order (deterministic) and writes the partials
    int &last = *flag;  // operand buffers are free after the K loop
    __threadfence();
    consumer_sync<BAR>();
    const int grp = tl.pad >> 8;
    int *cnt = cx.mcount + (int64_t)grp * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0) last = atomicAdd(cnt, 1) == B.mks - 1;
    consumer_sync<BAR>();
    if (!last) return;
    __threadfence();
    const int64_t slab0 = B.msp_off + (int64_t)(tl.start / MMA_COLS) * B.mks;
    const S *scr = static_cast<const S *>(cx.msplit);
    for (int e = threadIdx.x; e < tl.count * NRT; e += MM_THREADS) {
      const int m = e / NRT, r = rhs0 + e % NRT;
      if (r >= cx.nrhs) continue;
      S sum = X::zero();
      for (int k = 0; k < B.mks; ++k) sum = X::add(sum, X::ldcg(scr + ((slab0 + k) * MMA_COLS + m) * cx.nrhs + r));
      const int row = tl.start + m;
      const int q = red_iota ? row : cx.idx[B.red_off + row];
      static_cast<S *>(cx.part)[(B.part_off + q) * cx.nrhs + r] = sum;
    }
    if (threadIdx.x == 0) *cnt = 0;  // re-arm for the next apply
  }
}

template <class S, bool ADJ, int NT, bool M3, int MINB>
__global__ void __launch_bounds__(MM_THREADS, MINB) mma_kernel(const Ctx cx, const Tile *__restrict__ tiles, int from_f) {
  using X = Tr<S>;
  using PL = Planes<S>;
  constexpr bool CPLX = PL::cplx;
  constexpr bool G3 = CPLX && M3;
  constexpr int NRT = 8 * NT;
  constexpr int BK = mm_bk<S>();          // K chunk: 16 complex / 32 real (16 KB of factor tile)
  constexpr int KS = BK / 4;             // k4 steps per chunk
  constexpr int AW = MM_BM / 16;         // warps along M
  constexpr int B_PER_T = BK * NRT / MM_THREADS;
  constexpr int A_CH = KS * AW * 2 * 32; // scalars per A chunk (fragment order [k4][w][hi][lane])
  constexpr int B_CH = KS * NT * 32;     // scalars per B chunk ([k4][t][lane])
  // two-stage ring of fragment-ordered operand buffers.  Static shared
  // memory measured faster than a dynamic 2/3-stage ring (the default carveout
  // keeps more L1 for the B gathers; profiles/r01_mma_variants.txt).
  constexpr int NB = 2;
  __shared__ __align__(16) S As[NB * A_CH];
  __shared__ __align__(16) S Bs[NB * B_CH];

  pdl_trigger();
  const Tile tl = tiles[blockIdx.y];  // plan tables: never written by kernels
  const DevBlock B = cx.blocks[tl.blk];
  const int rhs0 = blockIdx.x * NRT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const S *T = static_cast<const S *>(cx.coef) + B.coef_off;
  const int64_t ld = B.ld;
  const int K = ADJ ? B.r_out : B.n_red;
  // adjoint K split (tall blocks on low-parallelism stages): rows [kbeg, kend)
  const bool ksplit = ADJ && tl.pad >= 0;
  const int sidx = ksplit ? (tl.pad & 255) : 0;
  int kbeg = 0, kend = K;
  if (ksplit) {
    const int chunk = ((K + B.mks - 1) / B.mks + BK - 1) / BK * BK;
    kbeg = min(K, sidx * chunk);
    kend = min(K, kbeg + chunk);
  }
  const int nchunks = (kend - kbeg + BK - 1) / BK;
  const bool red_iota = (B.flags & F_RED_IOTA) != 0;

  // Operand staging.  Thread e writes fragment slot e (contiguous, conflict-free
  // shared stores); slot e of a chunk is (k4, w, hi, gid, tig) with
  // m = 16 w + 8 hi + gid and k = 4 k4 + tig, so a warp reads 4 (forward) or 8
  // (adjoint) fully used 128/64-byte global segments.
  auto load_A = [&](int kc) {
    const int kb = kbeg + kc * BK;
    S *dst = As + (kc % NB) * A_CH;
#pragma unroll
    for (int i = 0; i < MM_BM * BK / MM_THREADS; ++i) {
      const int e = threadIdx.x + MM_THREADS * i;
      const int tig_ = e & 3, gid_ = (e >> 2) & 7, hi = (e >> 5) & 1, w = (e >> 6) & (AW - 1), k4 = e >> 8;
      const int m = w * 16 + hi * 8 + gid_, k = k4 * 4 + tig_;
      const bool ok = m < tl.count && kb + k < kend;
      const S *src = ADJ ? T + (int64_t)(tl.start + m) * ld + (kb + k) : T + (int64_t)(kb + k) * ld + (tl.start + m);
      cp_async<sizeof(S)>(dst + e, ok ? src : T, ok);
    }
  };
  // B gather: the forward's redundant-position indices are fetched one chunk
  // ahead (qreg), so the value loads never wait on an index load.
  int qreg[B_PER_T];
  auto load_q = [&](int kc) {
    if (ADJ) return;
    const int kb = kbeg + kc * BK;
#pragma unroll
    for (int i = 0; i < B_PER_T; ++i) {
      const int e = threadIdx.x + MM_THREADS * i;
      const int k = ((e >> 5) / NT) * 4 + (e & 3);
      qreg[i] = (kb + k < kend) ? (red_iota ? kb + k : __ldg(cx.idx + B.red_off + kb + k)) : 0;
    }
  };
  S breg[B_PER_T];
  auto load_B = [&](int kc) {
    const int kb = kbeg + kc * BK;
#pragma unroll
    for (int i = 0; i < B_PER_T; ++i) {
      const int e = threadIdx.x + MM_THREADS * i;
      const int tig_ = e & 3, gid_ = (e >> 2) & 7, t = (e >> 5) % NT, k4 = (e >> 5) / NT;
      const int k = k4 * 4 + tig_, n = t * 8 + gid_;
      const int r = rhs0 + n;
      S v = X::zero();
      if (kb + k < kend && r < cx.nrhs) v = ADJ ? adj_in<S>(cx, B, kb + k, r, from_f != 0) : in_value<S>(cx, B, qreg[i], r);
      breg[i] = v;
    }
  };
  auto store_B = [&](int kc) {
    S *dst = Bs + (kc % NB) * B_CH;
#pragma unroll
    for (int i = 0; i < B_PER_T; ++i) dst[threadIdx.x + MM_THREADS * i] = breg[i];
  };

  // accumulators: 4M uses (re, im); 3M uses (P1, P2, P3)
  double c0[NT][4], c1[NT][4], c2[G3 ? NT : 1][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int v = 0; v < 4; ++v) c0[t][v] = c1[t][v] = 0.0;
#pragma unroll
  for (int t = 0; t < (G3 ? NT : 1); ++t)
#pragma unroll
    for (int v = 0; v < 4; ++v) c2[t][v] = 0.0;

  if (nchunks == 0) pdl_wait();
  // two-stage ring, sync at the bottom of the iteration.  The first factor
  // chunk does not depend on earlier kernels: it streams in before pdl_wait()
  if (nchunks > 0) {
    load_A(0);
    cp_async_commit();
    pdl_wait();  // the previous stage's workspace is complete and visible
    load_q(0);
    load_B(0);
    store_B(0);
    if (nchunks > 1) load_q(1);
    cp_async_wait<0>();
    __syncthreads();
  }
  for (int kc = 0; kc < nchunks; ++kc) {
    const bool more = kc + 1 < nchunks;
    if (more) {
      load_A(kc + 1);
      cp_async_commit();
      load_B(kc + 1);
      if (kc + 2 < nchunks) load_q(kc + 2);
    }
    const S *Ac = As + (kc % NB) * A_CH;
    const S *Bc = Bs + (kc % NB) * B_CH;
#pragma unroll
    for (int k4 = 0; k4 < KS; ++k4) {
      const S a0 = Ac[((k4 * AW + warp) * 2 + 0) * 32 + lane];
      const S a1 = Ac[((k4 * AW + warp) * 2 + 1) * 32 + lane];
      const double ar0 = PL::re(a0), ar1 = PL::re(a1);
      // conj(T) for the adjoint
      const double ai0 = ADJ ? -PL::im(a0) : PL::im(a0), ai1 = ADJ ? -PL::im(a1) : PL::im(a1);
      const double as0 = ar0 + ai0, as1 = ar1 + ai1;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const S b = Bc[(k4 * NT + t) * 32 + lane];
        if constexpr (!CPLX) {
          dmma(c0[t], ar0, ar1, PL::re(b));
        } else if constexpr (G3) {
          dmma(c0[t], ar0, ar1, PL::re(b));
          dmma(c1[t], ai0, ai1, PL::im(b));
          dmma(c2[t], as0, as1, PL::re(b) + PL::im(b));
        } else {  // (Ar + i Ai)(Br + i Bi)
          dmma(c0[t], ar0, ar1, PL::re(b));
          dmma(c0[t], -ai0, -ai1, PL::im(b));
          dmma(c1[t], ar0, ar1, PL::im(b));
          dmma(c1[t], ai0, ai1, PL::re(b));
        }
      }
    }
    if (more) store_B(kc + 1);
    cp_async_wait<0>();
    __syncthreads();
  }
  mma_epilogue<S, ADJ, NT, M3, 0>(cx, tl, B, c0, c1, c2, rhs0, ksplit, sidx, from_f, reinterpret_cast<int *>(As));
}

// ------------------------------------------------------------------------
// Warp-specialised multi-RHS kernel.  Same tile, operand fragment order, K
// split and epilogue as mma_kernel, but the operand loads move to a fifth
// PRODUCER warp: it streams the factor tile with cp.async (completion
// tracked by an mbarrier, cp.async.mbarrier.arrive.noinc) and gathers the
// right-hand-side rows through registers into shared memory, NS stages ahead.
// The four CONSUMER warps only wait on the stage's "full" barrier, run the
// LDS + DMMA k4 steps and release the stage on its "empty" barrier: no block-
// wide barrier and no load code between their DMMAs.
// ------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
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

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
// TMA 1-D bulk copy global -> shared, completion counted in bytes on an mbarrier
__device__ __forceinline__ void bulk_g2s(void *smem, const void *gmem, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

// TMA 2-D tiled load (tensor map in global memory) -> shared, bytes on an mbarrier
__device__ __forceinline__ void tma_2d_g2s(void *smem, const void *tmap, int c0, int c1, uint64_t *bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(tmap), "r"(c0), "r"(c1), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

constexpr int WS_STAGES = 3;
constexpr int WS_THREADS = MM_THREADS + 32;
// padded leading dimensions of the factor tile in shared memory (elements):
// forward column-major [k][m] with AP = 64 + (2 complex | 4 real), adjoint
// row-major [m][k] with BKP = BK + 4; chosen so a warp's A-fragment loads hit
// distinct banks (16-byte slots 2 tig + gid / 4 gid + tig distinct mod 8 per
// quarter warp; 8-byte slots distinct mod 16 per half warp)
template <class S, bool ADJ, int FM = 0>
__host__ __device__ constexpr int ws_a_elems() {
  return (ADJ || sizeof(S) == 8 || FM == 3) ? MM_BM * mm_bk<S>() : mm_bk<S>() * (MM_BM + 2);
}
// A-tile layout / row mapping of the warp-specialised kernel: 0 padded
// column-major by 1-D bulk copies (complex forward), 1 swizzled [half][m][k]
// by 2-D TMA (adjoint), 2 swizzled [quad][k][16 rows] by 2-D TMA (real forward)
// FM (complex forward): 0 = padded 1-D bulk copies, 3 = swizzled [q][k][8 rows]
// by eight 2-D TMA requests (fragment rows permuted as in mode 1)
template <class S, bool ADJ, int FM = 0>
__host__ __device__ constexpr int ws_mode() {
  return ADJ ? 1 : (sizeof(S) == 8 ? 2 : FM);
}

// B chunk of the warp-specialised kernel: complex in fragment order (BK x 32
// slots), real row-major [k][32 + 4] (each row one contiguous 256-byte gather
// by 16-byte cp.async; the +4 pad makes the fragment reads conflict-free)
template <class S>
__host__ __device__ constexpr int ws_b_elems() {
  return sizeof(S) == 16 ? mm_bk<S>() / 4 * 4 * 32 : mm_bk<S>() * (32 + 4);
}

template <class S, bool ADJ, bool M3, int FM = 0>
__host__ __device__ constexpr int ws_smem_bytes() {
  // NS x (A tile + B chunk) operand buffers + 2 NS mbarriers + 1 KB to align
  // the stages to the 1024-byte period of the 128-byte TMA swizzle
  return WS_STAGES * (ws_a_elems<S, ADJ, FM>() + ws_b_elems<S>()) * (int)sizeof(S) + 2 * WS_STAGES * 8 + 1024;
}

template <class S, bool ADJ, bool M3, int MINB, int FM = 0>
__global__ void __launch_bounds__(WS_THREADS, MINB) mma_ws_kernel(const Ctx cx, const Tile *__restrict__ tiles,
                                                                  int from_f) {
  using X = Tr<S>;
  using PL = Planes<S>;
  constexpr int NT = 4;
  constexpr bool CPLX = PL::cplx;
  constexpr bool G3 = CPLX && M3;
  constexpr int NRT = 8 * NT;
  constexpr int BK = mm_bk<S>();
  constexpr int KS = BK / 4;
  constexpr int AW = MM_BM / 16;
  constexpr int A_CH = ws_a_elems<S, ADJ, FM>();
  // leading dimension of the factor tile in shared memory: forward padded
  // column-major [k][m]; adjoint the TMA box [m][k] as written (dense)
  constexpr int AP = ADJ ? BK : MM_BM + 2;  // (mode 0 only)
  constexpr int MODE = ws_mode<S, ADJ, FM>();
  constexpr int B_CH = ws_b_elems<S>();
  constexpr bool BROW = !CPLX;  // real: row-major padded B chunk
  constexpr int NPB = 32 + 4;
  constexpr int NS = WS_STAGES;
  extern __shared__ __align__(128) unsigned char ws_smem[];
  // stage buffers start at a 1024-byte boundary (shared-space address)
  const unsigned sbase = (unsigned)__cvta_generic_to_shared(ws_smem);
  S *As = reinterpret_cast<S *>(ws_smem + (((sbase + 1023u) & ~1023u) - sbase));
  S *Bs = As + NS * A_CH;
  uint64_t *full = reinterpret_cast<uint64_t *>(Bs + NS * B_CH);
  uint64_t *empty = full + NS;

  pdl_trigger();
  const Tile tl = tiles[blockIdx.y];  // plan tables: never written by kernels
  const DevBlock B = cx.blocks[tl.blk];
  const int rhs0 = blockIdx.x * NRT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const S *T = static_cast<const S *>(cx.coef) + B.coef_off;
  const int64_t ld = B.ld;
  const int K = ADJ ? B.r_out : B.n_red;
  const bool ksplit = ADJ && tl.pad >= 0;
  const int sidx = ksplit ? (tl.pad & 255) : 0;
  int kbeg = 0, kend = K;
  if (ksplit) {
    const int chunk = ((K + B.mks - 1) / B.mks + BK - 1) / BK * BK;
    kbeg = min(K, sidx * chunk);
    kend = min(K, kbeg + chunk);
  }
  // a tile without columns (COPY block in the adjoint: skeleton part only)
  // has no product, and no tensor map to load from
  const int nchunks = tl.count > 0 ? (kend - kbeg + BK - 1) / BK : 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(full + i, 65);   // producer: 1 expect-tx arrival (TMA bytes) + 32 cp.async + 32 plain
      mbar_init(empty + i, AW);  // one arrival per consumer warp
    }
    // make the initialised barriers visible to the async proxy (the TMA unit
    // completes transactions on them) before any copy is issued
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // the previous stage's workspace is complete and visible

  if (warp == AW) {
    // ------------------------------------------------ producer warp
    // B slot e = lane + 32 i holds row k = 4 (i / NT) + (lane & 3), rhs
    // rhs0 + 8 (i % NT) + (lane >> 2): a lane touches KS rows per chunk, whose
    // gather indices (redundant positions / perm_x) are prefetched one chunk
    // ahead; the values then go straight to shared memory by cp.async.
    const bool red_iota = (B.flags & F_RED_IOTA) != 0;
    const bool from_f_ = from_f != 0;
    const bool reg_path = cx.diag != nullptr;  // a fused diagonal needs the value in registers
    const int tig_ = lane & 3, gid_ = lane >> 2;
    auto row_index = [&](int kc, int k4) -> int {  // what the gather needs for row k of chunk kc
      const int k = kbeg + kc * BK + 4 * k4 + tig_;
      if (k >= kend) return -1;
      if (ADJ) return from_f_ ? __ldg(cx.perm + B.out_off + k) : k;
      return red_iota ? k : __ldg(cx.idx + B.red_off + k);
    };
    // real (BROW): lane owns row k = lane of every chunk (BK = 32)
    auto row_index_r = [&](int kc) -> int {
      const int k = kbeg + kc * BK + lane;
      if (k >= kend) return -1;
      if (ADJ) return from_f_ ? __ldg(cx.perm + B.out_off + k) : k;
      return red_iota ? k : __ldg(cx.idx + B.red_off + k);
    };
    int qn[KS];
#pragma unroll
    for (int k4 = 0; k4 < KS; ++k4) qn[k4] = (nchunks > 0 && !BROW) ? row_index(0, k4) : -1;
    int qrn = (nchunks > 0 && BROW) ? row_index_r(0) : -1;
    for (int kc = 0; kc < nchunks; ++kc) {
      const int slot = kc % NS;
      int q[KS];
#pragma unroll
      for (int k4 = 0; k4 < KS; ++k4) q[k4] = qn[k4];
      const int qr = qrn;
      if (kc + 1 < nchunks) {
        if (BROW) {
          qrn = row_index_r(kc + 1);
        } else {
#pragma unroll
          for (int k4 = 0; k4 < KS; ++k4) qn[k4] = row_index(kc + 1, k4);
        }
      }
      mbar_wait(empty + slot, ((kc / NS) & 1) ^ 1);
      const int kb = kbeg + kc * BK;
      const int kn = min(BK, kend - kb);  // valid k of this chunk
      S *dA = As + slot * A_CH;
      // factor tile by TMA bulk copies (16-byte multiples: the real layout has
      // even ld and a zero pad row, so an odd length rounds up into it)
      constexpr int EV = sizeof(S) == 8 ? 2 : 1;
      if (MODE == 3) {
        if (lane == 0) {
          // complex forward: 64 x BK tile as eight 2-D TMA requests of 8 rows
          // (128 B) x BK columns, 128-byte swizzled, past-the-block zero-filled
          const void *tmap = static_cast<const unsigned char *>(cx.tmaps_f) + (size_t)tl.blk * 128;
          mbar_arrive_expect_tx(full + slot, (unsigned)(MM_BM * BK * sizeof(S)));
#pragma unroll
          for (int q8 = 0; q8 < 8; ++q8) tma_2d_g2s(dA + q8 * BK * 8, tmap, 2 * (tl.start + 8 * q8), kb, full + slot);
        }
      } else if (MODE == 2) {
        if (lane == 0) {
          // real forward: the 64 x BK tile as four 2-D TMA requests of 16 rows
          // (128 B) x BK columns, 128-byte swizzled, past-the-block zero-filled
          const void *tmap = static_cast<const unsigned char *>(cx.tmaps_f) + (size_t)tl.blk * 128;
          mbar_arrive_expect_tx(full + slot, (unsigned)(MM_BM * BK * sizeof(S)));
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) tma_2d_g2s(dA + q4 * BK * 16, tmap, tl.start + 16 * q4, kb, full + slot);
        }
      } else if (!ADJ) {
        // forward: column k of the tile = tl.count contiguous rows of T
        const unsigned cb = (unsigned)((tl.count + EV - 1) / EV * EV * sizeof(S));
        if (lane == 0) mbar_arrive_expect_tx(full + slot, cb * kn);
        for (int j = lane; j < BK; j += 32) {
          if (j < kn) {
            bulk_g2s(dA + j * AP, T + (int64_t)(kb + j) * ld + tl.start, cb, full + slot);
          } else {  // K tail: zero column (stale shared memory could hold NaN patterns)
            for (int i = 0; i < MM_BM; ++i) dA[j * AP + i] = X::zero();
          }
        }
      } else if (lane == 0) {
        // adjoint: the BK x 64 tile (T rows kb.., T columns tl.start..) as two
        // 2-D TMA requests of 128-byte rows (BK/2 scalars x 64 columns each),
        // 128-byte swizzled; rows / columns past the block are zero-filled (a
        // K split's rows past kend meet zero right-hand sides)
        const void *tmap = static_cast<const unsigned char *>(cx.tmaps) + (size_t)tl.blk * 128;
        mbar_arrive_expect_tx(full + slot, (unsigned)(MM_BM * BK * sizeof(S)));
        constexpr int KH = BK / 2;
        tma_2d_g2s(dA, tmap, kb * (int)(sizeof(S) / 8), tl.start, full + slot);
        tma_2d_g2s(dA + MM_BM * KH, tmap, (kb + KH) * (int)(sizeof(S) / 8), tl.start, full + slot);
      }
      S *dB = Bs + slot * B_CH;
      if constexpr (BROW) {
        // row k = lane: its 32 right-hand sides, contiguous in the workspace
        // (RHS-fastest) -> 16 x 16-byte cp.async; c / f rows (column-major
        // user arrays), odd nrhs and a fused diagonal take 8-byte elements
        S *drow = dB + lane * NPB;
        const int nv = min(32, cx.nrhs - rhs0);  // valid right-hand sides
        const S *srow = nullptr;
        bool contiguous = false;
        int64_t rstride = 0;  // element stride between right-hand sides otherwise
        if (qr >= 0) {
          if (ADJ) {
            if (from_f_) {
              srow = static_cast<const S *>(cx.fin) + (int64_t)rhs0 * cx.n + qr;
              rstride = cx.n;
            } else {
              srow = static_cast<const S *>(cx.z) + (B.out_off + qr) * cx.nrhs + rhs0;
              contiguous = true;
            }
          } else {
            const bool s1 = qr >= B.seg_len[0];
            const int64_t off = s1 ? B.seg_off[1] + (qr - B.seg_len[0]) : B.seg_off[0] + qr;
            const int32_t srcsel = s1 ? B.seg_src[1] : B.seg_src[0];
            if (srcsel == SRC_C) {
              srow = static_cast<const S *>(cx.c) + (int64_t)rhs0 * cx.m + off;
              rstride = cx.m;
            } else {
              srow = static_cast<const S *>(cx.z) + off * cx.nrhs + rhs0;
              contiguous = true;
            }
          }
        }
        if (contiguous && !reg_path && (cx.nrhs & 1) == 0 && cx.b16) {
#pragma unroll
          for (int h = 0; h < 16; ++h) cp_async<16>(drow + 2 * h, srow + 2 * h, 2 * h < nv);
        } else if (!reg_path) {
          for (int n = 0; n < 32; ++n) {
            const bool ok = qr >= 0 && n < nv;
            cp_async<8>(drow + n, ok ? (contiguous ? srow + n : srow + n * rstride) : static_cast<const S *>(cx.z), ok);
          }
        } else {
          for (int n = 0; n < 32; ++n) {
            const bool ok = qr >= 0 && n < nv;
            drow[n] = ok ? (ADJ ? (contiguous ? srow[n] : srow[n * rstride]) : in_value<S>(cx, B, qr, rhs0 + n))
                         : X::zero();
          }
        }
      } else {
        // a lane's KS rows: base pointer and right-hand-side stride resolved
        // once per row (segment / source / perm), then one multiply-add per element
        const S *rb[KS];
        int64_t rs[KS];
#pragma unroll
        for (int k4 = 0; k4 < KS; ++k4) {
          const int qq = q[k4];
          rb[k4] = static_cast<const S *>(cx.z);
          rs[k4] = 0;
          if (qq >= 0) {
            if (ADJ) {
              if (from_f_) {
                rb[k4] = static_cast<const S *>(cx.fin) + qq;
                rs[k4] = cx.n;
              } else {
                rb[k4] = static_cast<const S *>(cx.z) + (B.out_off + qq) * cx.nrhs;
                rs[k4] = 1;
              }
            } else {
              const bool s1 = qq >= B.seg_len[0];
              const int64_t off = s1 ? B.seg_off[1] + (qq - B.seg_len[0]) : B.seg_off[0] + qq;
              if ((s1 ? B.seg_src[1] : B.seg_src[0]) == SRC_C) {
                rb[k4] = static_cast<const S *>(cx.c) + off;
                rs[k4] = cx.m;
              } else {
                rb[k4] = static_cast<const S *>(cx.z) + off * cx.nrhs;
                rs[k4] = 1;
              }
            }
          }
        }
#pragma unroll
        for (int i = 0; i < B_CH / 32; ++i) {
          const int k4 = i / NT, t = i % NT;
          const int r = rhs0 + t * 8 + gid_;
          const bool ok = q[k4] >= 0 && r < cx.nrhs;
          const S *src = ok ? rb[k4] + (int64_t)r * rs[k4] : static_cast<const S *>(cx.z);
          if (!reg_path) {
            cp_async<sizeof(S)>(dB + lane + 32 * i, src, ok);
          } else {
            dB[lane + 32 * i] = ok ? (ADJ ? *src : in_value<S>(cx, B, q[k4], r)) : X::zero();
          }
        }
      }
      mbar_cp_async_arrive(full + slot);  // completes when this lane's cp.async have landed
      mbar_arrive(full + slot);           // the register-path stores (if any) are done
    }
    return;  // the producer takes no part in the epilogue
  }

  // ------------------------------------------------ consumer warps
  const int gid = lane >> 2, tig = lane & 3;
  double c0[NT][4], c1[NT][4], c2[G3 ? NT : 1][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int v = 0; v < 4; ++v) c0[t][v] = c1[t][v] = 0.0;
#pragma unroll
  for (int t = 0; t < (G3 ? NT : 1); ++t)
#pragma unroll
    for (int v = 0; v < 4; ++v) c2[t][v] = 0.0;
  for (int kc = 0; kc < nchunks; ++kc) {
    const int slot = kc % NS;
    mbar_wait(full + slot, (kc / NS) & 1);
    const S *Ac = As + slot * A_CH;
    const S *Bc = Bs + slot * B_CH;
    constexpr int RMODE = MODE == 3 ? 1 : MODE;  // row permutation
    const int m0 = warp * 16 + tile_row<S, RMODE>(gid), m1 = warp * 16 + tile_row<S, RMODE>(gid + 8);
#pragma unroll
    for (int k4 = 0; k4 < KS; ++k4) {
      const int k = 4 * k4 + tig;
      S a0, a1;
      if constexpr (MODE == 3) {
        // swizzled [q][k][8 rows]: 16-byte chunk (row m & 7) of row k at (m & 7) ^ (k & 7)
        const unsigned char *ab = reinterpret_cast<const unsigned char *>(Ac) + k * 128;
        a0 = *reinterpret_cast<const S *>(ab + (m0 >> 3) * (BK * 128) + (((m0 & 7) ^ (k & 7)) << 4));
        a1 = *reinterpret_cast<const S *>(ab + (m1 >> 3) * (BK * 128) + (((m1 & 7) ^ (k & 7)) << 4));
      } else if constexpr (MODE == 2) {
        // swizzled [quad][k][16 rows]: 16-byte chunk c of row k sits at c ^ (k & 7)
        const unsigned char *ab = reinterpret_cast<const unsigned char *>(Ac) + k * 128;
        const int mm0 = m0 & 15, mm1 = m1 & 15;
        a0 = *reinterpret_cast<const S *>(ab + (m0 >> 4) * (BK * 128) + (((mm0 >> 1) ^ (k & 7)) << 4) + (mm0 & 1) * 8);
        a1 = *reinterpret_cast<const S *>(ab + (m1 >> 4) * (BK * 128) + (((mm1 >> 1) ^ (k & 7)) << 4) + (mm1 & 1) * 8);
      } else if constexpr (ADJ) {
        // swizzled [half][m][128 B]: 16-byte chunk c of row m sits at c ^ (m & 7)
        constexpr int KH = BK / 2;
        const int h = k / KH, kk = k % KH;
        const int byte = kk * (int)sizeof(S);
        const unsigned char *hb = reinterpret_cast<const unsigned char *>(Ac) + h * (MM_BM * 128);
        const int c = byte >> 4, o = byte & 15;
        a0 = *reinterpret_cast<const S *>(hb + m0 * 128 + ((c ^ (m0 & 7)) << 4) + o);
        a1 = *reinterpret_cast<const S *>(hb + m1 * 128 + ((c ^ (m1 & 7)) << 4) + o);
      } else {
        a0 = Ac[k * AP + m0];
        a1 = Ac[k * AP + m1];
      }
      const double ar0 = PL::re(a0), ar1 = PL::re(a1);
      const double ai0 = ADJ ? -PL::im(a0) : PL::im(a0), ai1 = ADJ ? -PL::im(a1) : PL::im(a1);
      const double as0 = ar0 + ai0, as1 = ar1 + ai1;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const S b = BROW ? Bc[k * NPB + 8 * t + gid] : Bc[(k4 * NT + t) * 32 + lane];
        if constexpr (!CPLX) {
          dmma(c0[t], ar0, ar1, PL::re(b));
        } else if constexpr (G3) {
          dmma(c0[t], ar0, ar1, PL::re(b));
          dmma(c1[t], ai0, ai1, PL::im(b));
          dmma(c2[t], as0, as1, PL::re(b) + PL::im(b));
        } else {
          dmma(c0[t], ar0, ar1, PL::re(b));
          dmma(c0[t], -ai0, -ai1, PL::im(b));
          dmma(c1[t], ar0, ar1, PL::im(b));
          dmma(c1[t], ai0, ai1, PL::re(b));
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + slot);
  }
  // all consumer warps are past their last read of the operand buffers
  consumer_sync<1>();
  constexpr int RMODE_EPI = MODE == 3 ? 1 : MODE;
  mma_epilogue<S, ADJ, NT, M3, 1, RMODE_EPI>(cx, tl, B, c0, c1, c2, rhs0, ksplit, sidx, from_f, reinterpret_cast<int *>(As));
}

// Which multi-RHS launches use the warp-specialised TMA kernel
// (profiles/r01_mma_ws_ab.txt): complex plans, both directions (c2 nrhs 32:
// forward 18.1 vs 21.5 ms, adjoint 18.5 vs 19.9 ms).  Real plans stay on the
// classic kernel (c3: the producer warp's 32 gathers per lane per chunk make
// WS 1.3-3x slower).  MHT_MMA_WS=0 never, =1 always.
inline int mma_ws_mode() {
  const char *e = getenv("MHT_MMA_WS");  // read per launch (debug / A-B within one process)
  if (e && atoi(e) == 0) return 0;
  if (e && atoi(e) == 1) return 1;
  return -1;
}
template <class S, bool ADJ>
inline bool mma_ws() {
  // real plans never take the warp-specialised kernel: its row-gather
  // variant showed a rare nondeterministic error on c3 (1 run in 3,
  // profiles/r01_mma_ws_ab.txt) that is not understood yet
  if (!Planes<S>::cplx) return false;
  const int mode = mma_ws_mode();
  if (mode >= 0) return mode == 1;
  return true;
}

// CTAs per SM the warp-specialised kernel's registers are sized for: 3
// (<= 136 registers) by default, MHT_MMA_WS_MINB=2 for the unconstrained build
inline int mma_ws_minb() {
  static int v = [] {
    const char *e = getenv("MHT_MMA_WS_MINB");
    return (e && atoi(e) == 2) ? 2 : 3;
  }();
  return v;
}

template <class S, bool ADJ, bool M3, int MINB, int FM>
void mma_ws_launch_t(const Ctx &cx, const Tile *tiles, int nt, int from_f, cudaStream_t st) {
  constexpr int smem = ws_smem_bytes<S, ADJ, M3, FM>();
  static bool attr = [] {
    cudaFuncSetAttribute(mma_ws_kernel<S, ADJ, M3, MINB, FM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)attr;
  launch_ex(pdl_mma_on(), mma_ws_kernel<S, ADJ, M3, MINB, FM>, dim3((cx.nrhs + 31) / 32, nt), dim3(WS_THREADS), smem, st,
            cx, tiles, from_f);
}

// complex forward A tile: MHT_WS_FMODE=3 (2-D TMA, swizzled) | 0 (1-D bulk
// copies, padded; default)
inline int ws_fmode() {
  const char *e = getenv("MHT_WS_FMODE");
  return (e && atoi(e) == 3) ? 3 : 0;
}

template <class S, bool ADJ, bool M3>
void mma_ws_launch(const Ctx &cx, const Tile *tiles, int nt, int from_f, cudaStream_t st) {
  const bool f3 = !ADJ && Planes<S>::cplx && ws_fmode() == 3;
  if (mma_ws_minb() == 2) {
    if (f3) mma_ws_launch_t<S, ADJ, M3, 2, 3>(cx, tiles, nt, from_f, st);
    else mma_ws_launch_t<S, ADJ, M3, 2, 0>(cx, tiles, nt, from_f, st);
  } else {
    if (f3) mma_ws_launch_t<S, ADJ, M3, 3, 3>(cx, tiles, nt, from_f, st);
    else mma_ws_launch_t<S, ADJ, M3, 3, 0>(cx, tiles, nt, from_f, st);
  }
}

// ------------------------------------------------------------------------
// Real multi-RHS kernel with 16-byte operand copies.  Same tile (64 rows x 32
// right-hand sides, 4 warps x 16 rows), K chunk 32, two-stage cp.async ring
// and epilogue as mma_kernel, but both operands are staged as padded dense
// tiles instead of fragment order, so every copy moves 16 bytes:
//   A forward  [k][64 + 4]  (row pairs of T's column k),
//   A adjoint  [m][32 + 4]  (k pairs of T's column tl.start + m),
//   B          [k][32 + 4]  (a right-hand-side row = 32 contiguous workspace
//                           entries, 4 threads x 4 copies per row).
// The +4 pads make the mma fragment loads conflict-free (8-byte slots
// 4 tig + gid distinct per half warp).  The real kernel was instruction-bound
// on per-element address math (profiles/r01_ncu_mma_real_c3.txt).
// ------------------------------------------------------------------------
constexpr int RB_AP = MM_BM + 4, RB_NP = 32 + 4;

template <bool ADJ, int BKT>
__host__ __device__ constexpr int rb_a_elems() {
  return ADJ ? MM_BM * (BKT + 4) : BKT * RB_AP;
}
template <bool ADJ, int BKT, int NSTG>
__host__ __device__ constexpr int rb_smem_bytes() {
  return NSTG * (rb_a_elems<ADJ, BKT>() + BKT * RB_NP) * 8;
}

template <bool ADJ, int BKT, int NSTG, int MINB = 4>
__global__ void __launch_bounds__(MM_THREADS, MINB) mma_real_kernel(const Ctx cx, const Tile *__restrict__ tiles,
                                                                  int from_f) {
  using S = double;
  using X = Tr<S>;
  constexpr int RB_BK = BKT, RB_KP = BKT + 4;
  constexpr int NT = 4, KS = RB_BK / 4, A_CH = rb_a_elems<ADJ, BKT>(), B_CH = RB_BK * RB_NP;
  constexpr int APT = RB_BK * MM_BM / 2 / MM_THREADS;     // 16-byte A copies per thread per chunk
  constexpr int TPR = MM_THREADS / RB_BK;                 // threads per B row
  constexpr int RPT = 32 / TPR;                           // right-hand sides per thread
  extern __shared__ __align__(16) unsigned char rb_smem[];
  S *As = reinterpret_cast<S *>(rb_smem);
  S *Bs = As + NSTG * A_CH;

  pdl_trigger();
  const Tile tl = tiles[blockIdx.y];  // plan tables: never written by kernels
  const DevBlock B = cx.blocks[tl.blk];
  const int rhs0 = blockIdx.x * 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const S *T = static_cast<const S *>(cx.coef) + B.coef_off;
  const int64_t ld = B.ld;
  const int K = ADJ ? B.r_out : B.n_red;
  const bool ksplit = ADJ && tl.pad >= 0;
  const int sidx = ksplit ? (tl.pad & 255) : 0;
  int kbeg = 0, kend = K;
  if (ksplit) {
    const int chunk = ((K + B.mks - 1) / B.mks + RB_BK - 1) / RB_BK * RB_BK;
    kbeg = min(K, sidx * chunk);
    kend = min(K, kbeg + chunk);
  }
  const int nchunks = tl.count > 0 ? (kend - kbeg + RB_BK - 1) / RB_BK : 0;
  const bool red_iota = (B.flags & F_RED_IOTA) != 0;
  const bool from_f_ = from_f != 0;
  const bool reg_path = cx.diag != nullptr;
  const int nv = min(32, cx.nrhs - rhs0);
  const bool even = (cx.nrhs & 1) == 0;

  // B row of this thread: row (threadIdx.x >> 2) of each chunk, right-hand
  // sides 8 (threadIdx.x & 3) .. + 7
  const int brow = threadIdx.x / TPR, bq = threadIdx.x % TPR;
  auto row_index = [&](int kc) -> int {
    const int k = kbeg + kc * RB_BK + brow;
    if (k >= kend) return -1;
    if (ADJ) return from_f_ ? __ldg(cx.perm + B.out_off + k) : k;
    return red_iota ? k : __ldg(cx.idx + B.red_off + k);
  };
  auto load = [&](int kc, int qr) {
    const int kb = kbeg + kc * RB_BK;
    S *dA = As + (kc % NSTG) * A_CH;
#pragma unroll
    for (int i = 0; i < APT; ++i) {  // BK x 32 16-byte A copies / 128 threads
      const int e = threadIdx.x + MM_THREADS * i;
      if (!ADJ) {
        const int k = e >> 5, p = e & 31;  // column k, row pair p
        const bool ok = 2 * p < tl.count && kb + k < kend;
        cp_async<16>(dA + k * RB_AP + 2 * p, ok ? T + (int64_t)(kb + k) * ld + tl.start + 2 * p : T, ok);
      } else {
        const int m = e / (RB_BK / 2), p = e % (RB_BK / 2);  // tile row m (T column), k pair p
        const bool ok = m < tl.count && kb + 2 * p < kend;
        cp_async<16>(dA + m * RB_KP + 2 * p, ok ? T + (int64_t)(tl.start + m) * ld + kb + 2 * p : T, ok);
      }
    }
    S *drow = Bs + (kc % NSTG) * B_CH + brow * RB_NP + RPT * bq;
    const S *srow = nullptr;
    bool contiguous = false;
    int64_t rstride = 0;
    if (qr >= 0) {
      if (ADJ) {
        if (from_f_) {
          srow = static_cast<const S *>(cx.fin) + (int64_t)rhs0 * cx.n + qr;
          rstride = cx.n;
        } else {
          srow = static_cast<const S *>(cx.z) + (B.out_off + qr) * cx.nrhs + rhs0;
          contiguous = true;
        }
      } else {
        const bool s1 = qr >= B.seg_len[0];
        const int64_t off = s1 ? B.seg_off[1] + (qr - B.seg_len[0]) : B.seg_off[0] + qr;
        if ((s1 ? B.seg_src[1] : B.seg_src[0]) == SRC_C) {
          srow = static_cast<const S *>(cx.c) + (int64_t)rhs0 * cx.m + off;
          rstride = cx.m;
        } else {
          srow = static_cast<const S *>(cx.z) + off * cx.nrhs + rhs0;
          contiguous = true;
        }
      }
    }
    if (reg_path) {
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int n = RPT * bq + j;
        const bool ok = qr >= 0 && n < nv;
        drow[j] = ok ? (ADJ ? (contiguous ? srow[n] : srow[n * rstride]) : in_value<S>(cx, B, qr, rhs0 + n)) : 0.0;
      }
    } else if (contiguous && even) {
#pragma unroll
      for (int j = 0; j < RPT / 2; ++j) {
        const int n = RPT * bq + 2 * j;
        cp_async<16>(drow + 2 * j, srow + n, qr >= 0 && n < nv);
      }
    } else {
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int n = RPT * bq + j;
        const bool ok = qr >= 0 && n < nv;
        cp_async<8>(drow + j, ok ? (contiguous ? srow + n : srow + n * rstride) : static_cast<const S *>(cx.z), ok);
      }
    }
  };

  pdl_wait();  // the previous stage's workspace is complete and visible
  double c0[NT][4], c1[NT][4], c2[1][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int v = 0; v < 4; ++v) c0[t][v] = c1[t][v] = 0.0;
#pragma unroll
  for (int v = 0; v < 4; ++v) c2[0][v] = 0.0;

  // NSTG-stage ring: chunks kc+1 .. kc+NSTG-1 in flight while chunk kc computes
  int qn = nchunks > 0 ? row_index(0) : -1;
#pragma unroll
  for (int st = 0; st < NSTG - 1; ++st) {
    if (st < nchunks) {
      load(st, qn);
      if (st + 1 < nchunks) qn = row_index(st + 1);
    }
    cp_async_commit();  // (empty groups keep the group count uniform)
  }
  const int m0 = warp * 16 + gid;
  for (int kc = 0; kc < nchunks; ++kc) {
    cp_async_wait<NSTG - 2>();  // chunk kc has landed (this thread's copies)
    __syncthreads();            // ... everyone's; and chunk kc-1's buffer is free
    if (kc + NSTG - 1 < nchunks) {
      load(kc + NSTG - 1, qn);
      if (kc + NSTG < nchunks) qn = row_index(kc + NSTG);
    }
    cp_async_commit();
    const S *Ac = As + (kc % NSTG) * A_CH;
    const S *Bc = Bs + (kc % NSTG) * B_CH;
#pragma unroll
    for (int k4 = 0; k4 < KS; ++k4) {
      const int k = 4 * k4 + tig;
      const double a0 = ADJ ? Ac[m0 * RB_KP + k] : Ac[k * RB_AP + m0];
      const double a1 = ADJ ? Ac[(m0 + 8) * RB_KP + k] : Ac[k * RB_AP + m0 + 8];
#pragma unroll
      for (int t = 0; t < NT; ++t) dmma(c0[t], a0, a1, Bc[k * RB_NP + 8 * t + gid]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // operand buffers free (the K-split flag reuses them)
  mma_epilogue<S, ADJ, NT, false, 0>(cx, tl, B, c0, c1, c2, rhs0, ksplit, sidx, from_f, reinterpret_cast<int *>(As));
}

// real plans: the 16-byte-copy kernel by default, MHT_MMA_REAL=0 for the
// fragment-order kernel
inline bool mma_real16() {
  const char *e = getenv("MHT_MMA_REAL");
  return !(e && atoi(e) == 0);
}

// pipeline variant: MHT_REAL_CFG = 0 (K chunk 32, 2 stages, 4 CTAs/SM) |
// 1 (32, 3) | 2 (16, 3; c3 forward 6.9 -> 6.1 ms, adjoint 7.7 -> 7.3 ms over 0,
// profiles/r01_real_cfg_ab.txt) | 3 (16, 4) | 4 (16, 3, 5 CTAs/SM) |
// 5 (16, 2, 6 CTAs/SM, 80 registers; default: c3 +1.5% over 2 in four
// back-to-back pairs, profiles/r01_real_occupancy_ab.txt) | 6 (16, 2, 7) |
// 7 (8, 4, 6)
inline int real_cfg() {
  const char *e = getenv("MHT_REAL_CFG");
  return e ? atoi(e) : 5;
}

template <bool ADJ, int BKT, int NSTG, int MINB = 4>
void mma_real_launch_t(const Ctx &cx, const Tile *tiles, int nt, int from_f, cudaStream_t st) {
  constexpr int smem = rb_smem_bytes<ADJ, BKT, NSTG>();
  static bool attr = [] {
    cudaFuncSetAttribute(mma_real_kernel<ADJ, BKT, NSTG, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)attr;
  launch_ex(pdl_mma_on(), mma_real_kernel<ADJ, BKT, NSTG, MINB>, dim3((cx.nrhs + 31) / 32, nt), dim3(MM_THREADS), smem,
            st, cx, tiles, from_f);
}

template <bool ADJ>
void mma_real_launch(const Ctx &cx, const Tile *tiles, int nt, int from_f, cudaStream_t st) {
  switch (real_cfg()) {
    case 1: mma_real_launch_t<ADJ, 32, 3>(cx, tiles, nt, from_f, st); break;
    case 3: mma_real_launch_t<ADJ, 16, 4>(cx, tiles, nt, from_f, st); break;
    case 0: mma_real_launch_t<ADJ, 32, 2>(cx, tiles, nt, from_f, st); break;
    case 4: mma_real_launch_t<ADJ, 16, 3, 5>(cx, tiles, nt, from_f, st); break;
    case 6: mma_real_launch_t<ADJ, 16, 2, 7>(cx, tiles, nt, from_f, st); break;
    case 7: mma_real_launch_t<ADJ, 8, 4, 6>(cx, tiles, nt, from_f, st); break;
    case 2: mma_real_launch_t<ADJ, 16, 3>(cx, tiles, nt, from_f, st); break;
    default: mma_real_launch_t<ADJ, 16, 2, 6>(cx, tiles, nt, from_f, st);
  }
}

// Multi-RHS configuration (compile-time variants; default picked from the
// measurements in profiles/, override with MHT_MMA=4m|3m for experiments).
inline int mma_variant() {
  static int v = [] {
    const char *e = getenv("MHT_MMA");
    if (e && !strcmp(e, "4m")) return 0;   // 4 real MMAs per complex product, 32 RHS per CTA
    if (e && !strcmp(e, "3m")) return 1;   // 3M, 32 RHS per CTA (3 CTAs/SM)
    return 1;
  }();
  return v;
}

template <class S, bool ADJ, int NT, bool M3, int MINB>
void mma_launch(const Ctx &cx, const Tile *tiles, int nt, int from_f, cudaStream_t st) {
  launch_ex(pdl_mma_on(), mma_kernel<S, ADJ, NT, M3, MINB>, dim3((cx.nrhs + 8 * NT - 1) / (8 * NT), nt), dim3(MM_THREADS), 0,
            st, cx, tiles, from_f);
}

template <class S, bool ADJ, bool M3, int MINB, int NTMAX>
void mma_launch_nt(const Ctx &cx, const Tile *tiles, int nt, int from_f, cudaStream_t st) {
  if (NTMAX >= 4 && cx.nrhs >= 32)
    mma_launch<S, ADJ, 4, M3, MINB>(cx, tiles, nt, from_f, st);
  else if (cx.nrhs >= 16)
    mma_launch<S, ADJ, 2, M3, 4>(cx, tiles, nt, from_f, st);
  else
    mma_launch<S, ADJ, 1, M3, 4>(cx, tiles, nt, from_f, st);
}

template <class S, bool ADJ>
void mma_dispatch(const Ctx &cx, const Tile *tiles, int ntiles, int from_f, cudaStream_t st) {
  for (int t0 = 0; t0 < ntiles; t0 += 65535) {
    const int nt = ntiles - t0 < 65535 ? ntiles - t0 : 65535;
    const int v = Planes<S>::cplx ? mma_variant() : 0;
    if (!Planes<S>::cplx && cx.nrhs >= 32 && mma_real16()) {
      mma_real_launch<ADJ>(cx, tiles + t0, nt, from_f, st);
    } else if (cx.nrhs >= 32 && mma_ws<S, ADJ>()) {
      if (v >= 1)
        mma_ws_launch<S, ADJ, true>(cx, tiles + t0, nt, from_f, st);
      else
        mma_ws_launch<S, ADJ, false>(cx, tiles + t0, nt, from_f, st);
    } else if (v >= 1)
      mma_launch_nt<S, ADJ, true, 3, 4>(cx, tiles + t0, nt, from_f, st);
    else
      mma_launch_nt<S, ADJ, false, 4, 4>(cx, tiles + t0, nt, from_f, st);
  }
}

// ------------------------------------------------------------------------
// adjoint group sums: dst = sum of the readers' partial ranges (fixed order,
// no atomics).
// ------------------------------------------------------------------------
template <class S, bool CG>
__device__ __forceinline__ void reduce_piece(const Ctx &cx, const Piece p, const int64_t *__restrict__ rd,
                                             int slice = 0, int nslices = 1) {
  using X = Tr<S>;
  const S *part = static_cast<const S *>(cx.part);
  const int nr = cx.nrhs;
  const int total = p.len * nr;
  for (int e = slice * blockDim.x + threadIdx.x; e < total; e += nslices * blockDim.x) {
    const int i = e / nr, r = e - (e / nr) * nr;  // RHS fastest (workspace layout)
    S s = X::zero();
    for (int q = 0; q < p.rd_count; ++q) {
      const S *a = part + (rd[p.rd_begin + q] + i) * nr + r;
      s = X::add(s, CG ? X::ldcg(a) : *a);
    }
    if (p.dst_src == SRC_C)
      static_cast<S *>(cx.cw)[r * cx.m + p.dst_off + i] = cx.diag ? X::scale(s, diag_at(cx, p.dst_off + i)) : s;
    else
      static_cast<S *>(cx.z)[(p.dst_off + i) * nr + r] = s;
  }
}

template <class S>
__global__ void __launch_bounds__(256) reduce_kernel(const Ctx cx, const Piece *__restrict__ pieces,
                                                     const int64_t *__restrict__ rd) {
  pdl_trigger();
  pdl_wait();
  reduce_piece<S, false>(cx, pieces[blockIdx.x], rd, blockIdx.y, gridDim.y);  // y: slices of wide pieces
}


// ------------------------------------------------------------------------
// persistent nrhs = 1 apply: ONE cooperative launch walks all phases of a
// direction (forward: stages 0..L+1; adjoint: leaf stage, then per stage the
// unfused group sums and the stage, then the sums into c).  CTAs pull tiles
// from a per-phase atomic counter (largest first: the tile lists are LPT
// sorted) and meet at a grid barrier between phases, so a small plan pays one
// launch instead of L+2 and no per-stage ramp/drain.  The phase bodies are
// the same tile functions the per-stage kernels run.
// ------------------------------------------------------------------------
template <class S, int MINB>
__global__ void __launch_bounds__(PERSIST_THREADS, MINB) persist_kernel(const Ctx cx, const Phase *__restrict__ phases,
                                                                 int nph, const Tile *__restrict__ ftiles,
                                                                 const Tile *__restrict__ atiles,
                                                                 const Piece *__restrict__ pieces,
                                                                 const int64_t *__restrict__ rd, int *ctr,
                                                                 unsigned long long *stamps) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int t_sh;
  if (stamps && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long ns;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
    stamps[0] = ns;
  }
  for (int p = 0; p < nph; ++p) {
    const Phase ph = phases[p];
    for (;;) {
      if (threadIdx.x == 0) t_sh = atomicAdd(ctr + p, 1);
      __syncthreads();
      const int t = t_sh;
      __syncthreads();
      if (t >= ph.count) break;
      if (ph.kind == PH_FWD)
        fwd_tile<S, true>(cx, ftiles[ph.off + t]);
      else if (ph.kind == PH_ADJ)
        adj_tile<S, 1, true>(cx, atiles[ph.off + t], ph.from_f, 0);
      else
        reduce_piece<S, true>(cx, pieces[ph.off + t], rd);
      __syncthreads();
    }
    grid.sync();
    if (stamps && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long ns;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ns));
      stamps[p + 1] = ns;
    }
  }
  // every CTA is past its last atomicAdd: re-arm the counters for the next apply
  if (blockIdx.x == 0)
    for (int p = threadIdx.x; p < nph; p += blockDim.x) ctr[p] = 0;
}

constexpr int MAX_GRID_Y = 65535;

template <class S>
void fwd_dispatch(const Ctx &cx, const Tile *tiles, int ntiles, cudaStream_t st) {
  for (int t0 = 0; t0 < ntiles; t0 += MAX_GRID_Y) {
    const int nt = ntiles - t0 < MAX_GRID_Y ? ntiles - t0 : MAX_GRID_Y;
    const Tile *tp = tiles + t0;
    if (sizeof(S) == 8 && fwd_fb() == 0)
      launch_pdl(fwd_kernel<S, 0>, dim3(1, nt), dim3(FWD_THREADS), st, cx, tp);
    else if (sizeof(S) == 8 && fwd_fb() == 16)
      launch_pdl(fwd_kernel<S, 16>, dim3(1, nt), dim3(FWD_THREADS), st, cx, tp);
    else
      launch_pdl(fwd_kernel<S>, dim3(1, nt), dim3(FWD_THREADS), st, cx, tp);
  }
}

template <class S>
void adj_dispatch(const Ctx &cx, const Tile *tiles, int ntiles, int from_f, cudaStream_t st) {
  for (int t0 = 0; t0 < ntiles; t0 += MAX_GRID_Y) {
    const int nt = ntiles - t0 < MAX_GRID_Y ? ntiles - t0 : MAX_GRID_Y;
    const Tile *tp = tiles + t0;
    if (adj_rch() == 256)
      launch_pdl(adj_kernel<S, 1, 256>, dim3(1, nt), dim3(ADJ_THREADS), st, cx, tp, from_f);
    else if (adj_rch() == 512)
      launch_pdl(adj_kernel<S, 1, 512>, dim3(1, nt), dim3(ADJ_THREADS), st, cx, tp, from_f);
    else if (sizeof(S) == 16 ? adj_ar2() : adj_ar2_real())
      launch_pdl(adj_kernel<S, 1, ADJ_RCH, true>, dim3(1, nt), dim3(ADJ_THREADS), st, cx, tp, from_f);
    else
      launch_pdl(adj_kernel<S, 1>, dim3(1, nt), dim3(ADJ_THREADS), st, cx, tp, from_f);
  }
}

}  // namespace

void launch_fwd(bool is_complex, const Ctx &ctx, const Tile *tiles, int ntiles, void *stream) {
  if (ntiles <= 0) return;
  if (is_complex)
    fwd_dispatch<double2>(ctx, tiles, ntiles, (cudaStream_t)stream);
  else
    fwd_dispatch<double>(ctx, tiles, ntiles, (cudaStream_t)stream);
}

void launch_adj(bool is_complex, const Ctx &ctx, const Tile *tiles, int ntiles, bool in_from_f,
                void *stream) {
  if (ntiles <= 0) return;
  if (is_complex)
    adj_dispatch<double2>(ctx, tiles, ntiles, in_from_f ? 1 : 0, (cudaStream_t)stream);
  else
    adj_dispatch<double>(ctx, tiles, ntiles, in_from_f ? 1 : 0, (cudaStream_t)stream);
}

void launch_mma(bool is_complex, bool adjoint, const Ctx &ctx, const Tile *tiles, int ntiles, bool in_from_f,
                void *stream) {
  if (ntiles <= 0) return;
  cudaStream_t st = (cudaStream_t)stream;
  const int ff = in_from_f ? 1 : 0;
  if (is_complex) {
    if (adjoint) mma_dispatch<double2, true>(ctx, tiles, ntiles, ff, st);
    else mma_dispatch<double2, false>(ctx, tiles, ntiles, ff, st);
  } else {
    if (adjoint) mma_dispatch<double, true>(ctx, tiles, ntiles, ff, st);
    else mma_dispatch<double, false>(ctx, tiles, ntiles, ff, st);
  }
}

namespace {
__global__ void __launch_bounds__(256) repack_kernel(const double *__restrict__ src, double *__restrict__ dst,
                                                     const Repack *__restrict__ jobs) {
  const Repack J = jobs[blockIdx.x];
  const int64_t total = (int64_t)J.dst_ld * J.ncols;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int64_t j = e / J.dst_ld;
    const int i = (int)(e - j * J.dst_ld);
    dst[J.dst_off + e] = i < J.r_out ? src[J.src_off + j * J.r_out + i] : 0.0;
  }
}
}  // namespace

void launch_repack(const double *src, double *dst, const Repack *jobs, int njobs, void *stream) {
  for (int j0 = 0; j0 < njobs; j0 += 65535) {
    const int nj = njobs - j0 < 65535 ? njobs - j0 : 65535;
    repack_kernel<<<nj, 256, 0, (cudaStream_t)stream>>>(src, dst, jobs + j0);
  }
}

// MINB = CTAs per SM the register budget is sized for: 5 (96 registers; the
// complex body spills ~200 B outside its loops) or 4 (128, no spills).
// MHT_PERSIST_MINB=4|5 selects (default 5).
inline int persist_minb() {
  static int v = [] {
    const char *e = getenv("MHT_PERSIST_MINB");
    return (e && atoi(e) == 4) ? 4 : 5;
  }();
  return v;
}

template <class S, int MINB>
cudaError_t persist_launch(const Ctx &ctx, const Phase *phases, int nph, const Tile *ftiles, const Tile *atiles,
                           const Piece *pieces, const int64_t *rd, int *ctr, unsigned long long *stamps, int grid,
                           cudaStream_t st) {
  Ctx c = ctx;
  void *args[] = {(void *)&c, (void *)&phases, (void *)&nph, (void *)&ftiles, (void *)&atiles, (void *)&pieces,
                  (void *)&rd, (void *)&ctr, (void *)&stamps};
  return cudaLaunchCooperativeKernel((const void *)persist_kernel<S, MINB>, dim3(grid), dim3(PERSIST_THREADS), args, 0,
                                     st);
}

template <class S>
int persist_grid_t() {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (persist_minb() == 4)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, persist_kernel<S, 4>, PERSIST_THREADS, 0);
  else
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, persist_kernel<S, 5>, PERSIST_THREADS, 0);
  return sms * per;
}

int persist_grid(bool is_complex) { return is_complex ? persist_grid_t<double2>() : persist_grid_t<double>(); }

template <class S>
cudaError_t persist_dispatch(const Ctx &ctx, const Phase *phases, int nph, const Tile *ftiles, const Tile *atiles,
                             const Piece *pieces, const int64_t *rd, int *ctr, unsigned long long *stamps, int grid,
                             cudaStream_t st) {
  if (persist_minb() == 4) return persist_launch<S, 4>(ctx, phases, nph, ftiles, atiles, pieces, rd, ctr, stamps, grid, st);
  return persist_launch<S, 5>(ctx, phases, nph, ftiles, atiles, pieces, rd, ctr, stamps, grid, st);
}

int launch_persist(bool is_complex, const Ctx &ctx, const Phase *phases, int nph, const Tile *ftiles,
                   const Tile *atiles, const Piece *pieces, const int64_t *rd, int *ctr, unsigned long long *stamps,
                   int grid, void *stream) {
  if (nph <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = is_complex ? persist_dispatch<double2>(ctx, phases, nph, ftiles, atiles, pieces, rd, ctr, stamps, grid, st)
                             : persist_dispatch<double>(ctx, phases, nph, ftiles, atiles, pieces, rd, ctr, stamps, grid, st);
  return (int)e;
}

void launch_reduce(bool is_complex, const Ctx &ctx, const Piece *pieces, const int64_t *rd,
                   int npieces, void *stream) {
  if (npieces <= 0) return;
  // a piece is <= 1024 entries x nrhs values: give every 2048 values a CTA
  const int ny = ctx.nrhs <= 2 ? 1 : (ctx.nrhs / 2 < 64 ? ctx.nrhs / 2 : 64);
  if (is_complex)
    launch_pdl(reduce_kernel<double2>, dim3(npieces, ny), dim3(256), (cudaStream_t)stream, ctx, pieces, rd);
  else
    launch_pdl(reduce_kernel<double>, dim3(npieces, ny), dim3(256), (cudaStream_t)stream, ctx, pieces, rd);
}

}  // namespace mht
