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

#include <cstdlib>
#include <cstring>

#include "mht_internal.cuh"

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
// The nrhs = 1 stage kernels and the group sums launch with the programmatic-
// stream-serialisation attribute (graphs capture it as a programmatic edge);
// every kernel launched this way calls pdl_wait() before its first access to
// memory an earlier kernel of the sequence writes or reads.  The multi-RHS
// kernels launch without it (neutral on c2 / c3, 6% slower on c4's graph
// replay, profiles/r01_mma_pdl_ab.txt); their griddepcontrol instructions are
// no-ops then.
constexpr bool PDL_NRHS1 = true, PDL_MMA = false;
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
  launch_ex(PDL_NRHS1, kern, grid, block, 0, st, args...);
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
// c is read and written in the user's order: the plan's frequency position q
// is the user's coefficient perm_k[q] (plan v2, quadtree-frequency plans,
// reading A18); without perm_k the orders agree
__device__ __forceinline__ int64_t user_c_index(const Ctx &cx, int64_t q) { return cx.permk ? cx.permk[q] : q; }
// (the diagonal is indexed like c: user order)
__device__ __forceinline__ double diag_at(const Ctx &cx, int64_t k) {
  const double d = cx.diag[k];
  return cx.diag_sqrt ? sqrt(d) : d;
}

template <class S>
__device__ __forceinline__ S in_value(const Ctx &cx, const DevBlock &B, int q, int r) {
  const bool s1 = q >= B.seg_len[0];  // no dynamic indexing: keeps B in registers
  const int64_t off = s1 ? B.seg_off[1] + (q - B.seg_len[0]) : B.seg_off[0] + q;
  const int32_t src = s1 ? B.seg_src[1] : B.seg_src[0];
  if (src == SRC_C) {  // user layout: column-major, user order (plan position -> user index by perm_k)
    const int64_t ci = user_c_index(cx, off);
    const S v = static_cast<const S *>(cx.c)[r * cx.m + ci];
    return cx.diag ? Tr<S>::scale(v, diag_at(cx, ci)) : v;
  }
  return static_cast<const S *>(cx.z)[off * cx.nrhs + r];  // workspace: RHS-fastest
}

// Where a block's outputs go: the workspace, or — a switch-stage block of a
// sharded plan with the fused exchange on — the destination rank's receive
// buffer over peer memory (the all-to-all folded into the stores; the entry
// offset is shifted by zdel so out_off + row lands in that rank's layout)
template <class S>
__device__ __forceinline__ S *z_out(const Ctx &cx, const DevBlock &B, int64_t &off) {
  if ((B.flags & F_REMOTE) && cx.zrem) {
    const int h = B.flags >> 16;
    off += cx.zdel[h];
    return static_cast<S *>(cx.zrem[h]);
  }
  return static_cast<S *>(cx.z);
}

// ------------------------------------------------------------------------
// forward stage (nrhs = 1): one CTA per (block, 64-row tile[, column split]);
// 4 warps split the redundant columns, lane l owns rows l and l+32 of the
// tile.  Stages with too few row tiles to fill the GPU split the columns of
// large blocks (Tile.pad = group << 8 | split): every split writes its partial
// row sums to scratch and the last CTA of the group to arrive (atomic counter)
// adds them in split order — deterministic, no float atomics.
// ------------------------------------------------------------------------
// PFD: the L2 prefetch runs this many batch rounds ahead (8: c1 107.6 -> 105.0 us,
// c4 81.4 -> 79.9 us against 2; profiles/r02_fwd_variants_ab.txt)
template <class S, int PFD = 8>
__device__ __forceinline__ void fwd_tile_lat(const Ctx &cx, const Tile tl) {
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
  // x = in[red[j]] for a chunk of up to XCH columns is staged in shared memory
  // first (one gather round trip for the whole chunk, all threads), so the
  // factor loads never wait behind an index -> value chain; the warps then
  // take batches of FB columns in turn (w, w + 4, ...: a tile's tail costs at
  // most one batch), all of a batch's loads issued before their first use,
  // with an L2 prefetch of the warp's batch PFD rounds ahead
  constexpr int XCH = REAL ? 2048 : 1024;  // 16 KB
  constexpr int FB = REAL ? 8 : 4;
  __shared__ S xs[XCH];
  const bool red_iota = (B.flags & F_RED_IOTA) != 0;
  const int seg_bytes = tl.count * (int)sizeof(S);  // the tile's rows of one column
  for (int jc = jbeg; jc < jend; jc += XCH) {
    const int jn = min(XCH, jend - jc);
    if (jc > jbeg) __syncthreads();  // every warp is past its reads of the previous chunk
    for (int j = threadIdx.x; j < jn; j += FWD_THREADS) {
      const int q = red_iota ? jc + j : cx.idx[B.red_off + jc + j];
      xs[j] = in_value<S>(cx, B, q, 0);
    }
    __syncthreads();
    const int wb = warp * FB, we = jn;
    constexpr int JS = 4 * FB;
    const S *colc = T + (int64_t)jc * ld;
    for (int j = wb; j < we; j += JS) {
      {  // L2 prefetch of the batch PFD rounds ahead: column (lane >> 2), 128-byte lines (lane & 3) (+ 4)
        const int jp = j + PFD * JS + (lane >> 2);
        if (jp < we) {
          const char *pc = reinterpret_cast<const char *>(colc + (int64_t)jp * ld + tl.start);
          const int o = (lane & 3) * 128;
          if (o < seg_bytes) prefetch_l2(pc + o);
          if (o + 512 < seg_bytes) prefetch_l2(pc + o + 512);
        }
      }
      if constexpr (REAL) {
        double2 t[FB];
#pragma unroll
        for (int jj = 0; jj < FB; ++jj)
          t[jj] = (vp && j + jj < we)
                      ? Tr<double>::ldT2(reinterpret_cast<const double *>(colc) + (int64_t)(j + jj) * ld + tl.start + 2 * lane)
                      : make_double2(0.0, 0.0);
#pragma unroll
        for (int jj = 0; jj < FB; ++jj) {
          if (j + jj < we) {
            const S x = xs[j + jj];
            X::fma(acc_a, t[jj].x, x);
            X::fma(acc_b, t[jj].y, x);
          }
        }
      } else {
        S ta[FB], tb[FB];
#pragma unroll
        for (int jj = 0; jj < FB; ++jj) {
          const bool vj = j + jj < we;
          const S *cp = colc + (int64_t)(j + jj) * ld;
          ta[jj] = (va && vj) ? X::ldT(cp + ra) : X::zero();
          tb[jj] = (vb && vj) ? X::ldT(cp + rb) : X::zero();
        }
#pragma unroll
        for (int jj = 0; jj < FB; ++jj) {
          if (j + jj < we) {
            const S x = xs[j + jj];
            X::fma(acc_a, ta[jj], x);
            X::fma(acc_b, tb[jj], x);
          }
        }
      }
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
      s = X::add(s, in_value<S>(cx, B, q, 0));
    }
    if (B.flags & F_OUT_F) {
      static_cast<S *>(cx.fout)[cx.perm[B.out_off + row]] = s;
    } else {
      int64_t o = B.out_off + row;
      z_out<S>(cx, B, o)[o] = s;
    }
  }
  if (split && threadIdx.x == 0) cx.fcount[grp] = 0;  // re-arm for the next apply
}

// nrhs = 1 forward, latency variant (stages with few tiles: c1, c4, the small
// stages of c2 / c3): x staged per chunk, balanced 4-column batches, L2
// prefetch two batches ahead, 7 CTAs per SM.  c1 forward 126 -> 108 us, c4 95
// -> 80 us; on stages of many waves the streaming variant below is faster (c2
// 6.49 vs 7.52 ms, c3 3.06 vs 3.23 ms; profiles/r02_fwd_variants_ab.txt), so
// the loader picks per stage by tile count.
template <class S>
__global__ void __launch_bounds__(FWD_THREADS, 7) fwd_lat_kernel(const Ctx cx, const Tile *__restrict__ tiles) {
  const Tile tl = tiles[blockIdx.y];
  pdl_trigger();
  {
    // L2 prefetch of the tile's rows of its first 128 columns (every warp's
    // first batches)
    const DevBlock &B = cx.blocks[tl.blk];
    int jbeg = 0, jend = B.n_red;
    if (tl.pad >= 0) {
      const int ks = B.pad;
      const int chunk = (((B.n_red + ks - 1) / ks) + 31) & ~31;
      jbeg = (tl.pad & 255) * chunk;
      jend = min(B.n_red, jbeg + chunk);
    }
    const int j = jbeg + threadIdx.x;
    if (j < jend) {
      const char *col = reinterpret_cast<const char *>(static_cast<const S *>(cx.coef) + B.coef_off + (int64_t)j * B.ld +
                                                       tl.start);
      for (int o = 0; o < tl.count * (int)sizeof(S); o += 128) prefetch_l2(col + o);
    }
  }
  pdl_wait();
  fwd_tile_lat<S>(cx, tl);
}

// nrhs = 1 forward, streaming variant (stages of many waves): lane j of a
// warp gathers x for its 32-column group, broadcast by shuffle, 8 columns'
// loads in flight per step, 72 registers (7 CTAs per SM without the x buffer).
template <class S>
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
      xr = in_value<S>(cx, B, q, 0);
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
      if constexpr (REAL) {
        // each batch's FB loads issued before the first use (the interleaved
        // form kept only ~4 loads outstanding per warp; c3 3.35 -> 3.07 ms)
        constexpr int FB = 8;
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
      s = X::add(s, in_value<S>(cx, B, q, 0));
    }
    if (B.flags & F_OUT_F) {
      static_cast<S *>(cx.fout)[cx.perm[B.out_off + row]] = s;
    } else {
      int64_t o = B.out_off + row;
      z_out<S>(cx, B, o)[o] = s;
    }
  }
  if (split && threadIdx.x == 0) cx.fcount[grp] = 0;  // re-arm for the next apply
}

template <class S>
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
  fwd_tile<S>(cx, tl);
}

// adjoint input z[i] of a block: f through perm_x (leaf stage), else the group
// sum of its readers' partials (the adjoint of a block row that
// feeds two transfers is the sum of both), either summed here on load (fused:
// no separate reduction pass) or read from the zpool slot reduce_kernel wrote.
// The fused sum adds the partials in the same (reader id) order as
// reduce_kernel, so both paths are bitwise identical.
template <class S>
__device__ __forceinline__ S adj_in(const Ctx &cx, const DevBlock &B, int i, int r, bool from_f) {
  if (from_f) return static_cast<const S *>(cx.fin)[r * cx.n + cx.perm[B.out_off + i]];
  if (cx.fused && B.rd_cnt >= 0) {
    const S *part = static_cast<const S *>(cx.part);
    S s = Tr<S>::zero();
    for (int k = 0; k < B.rd_cnt; ++k) s = Tr<S>::add(s, part[(cx.rdtab[B.rd_off + k] + i) * cx.nrhs + r]);
    return s;
  }
  return static_cast<const S *>(cx.z)[(B.out_off + i) * cx.nrhs + r];
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
template <class S>
__device__ __forceinline__ void adj_tile(const Ctx &cx, const Tile tl, int from_f) {
  using X = Tr<S>;
  // columns per warp: 8 complex / 16 real
  constexpr int ACOLS = adj_cols<S>();
  constexpr int CPW = ACOLS / (ADJ_THREADS / 32);
  constexpr int RCH = ADJ_RCH;
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
  __shared__ S zs[RCH];
  S acc[CPW];
#pragma unroll
  for (int u = 0; u < CPW; ++u) acc[u] = X::zero();
  const S *T = static_cast<const S *>(cx.coef) + B.coef_off;
  const int64_t ld = B.ld;
  const int cbase = tl.start + warp * CPW;
  const int cend = tl.start + tl.count;
  constexpr bool REAL = sizeof(S) == 8;

  for (int rc = rbeg; rc < rend; rc += RCH) {
    const int rn = min(RCH, rend - rc);
    for (int i = threadIdx.x; i < rn; i += ADJ_THREADS) zs[i] = adj_in<S>(cx, B, rc + i, 0, from_f);
    if (REAL && (rn & 1) && threadIdx.x == 0) zs[rn] = X::zero();  // pair partner of the last row
    __syncthreads();
    if (cbase < cend) {
      if constexpr (REAL) {
        // real: lane takes the row pair (2q, 2q + 1) of each of its columns with
        // one 16-byte load (rc is even; the pad row of an odd r_out is zero);
        // all CPW column loads issued before their first use (predicated)
        for (int q = lane; 2 * q < rn; q += 32) {
          const double z0 = zs[2 * q], z1 = zs[2 * q + 1];
          double2 t[CPW];
#pragma unroll
          for (int u = 0; u < CPW; ++u)
            t[u] = cbase + u < cend
                       ? Tr<double>::ldT2(reinterpret_cast<const double *>(T) + (int64_t)(cbase + u) * ld + rc + 2 * q)
                       : make_double2(0.0, 0.0);
#pragma unroll
          for (int u = 0; u < CPW; ++u) {
            double &a = reinterpret_cast<double &>(acc[u]);
            a = ::fma(t[u].x, z0, a);
            a = ::fma(t[u].y, z1, a);
          }
        }
      } else {
        // complex: two rows per lane per step (i, i + 32), 2 CPW 16-byte loads
        // in flight (c2 adj_nrhs1 6.60 -> 6.56 ms, profiles/r01_adj_ar2_ab.txt);
        // a lane still accumulates its rows in ascending order
        for (int i = lane; i < rn; i += 64) {
          const bool v2 = i + 32 < rn;
          const S z0 = zs[i], z1 = v2 ? zs[i + 32] : X::zero();
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
            X::fmac(acc[u], t0[u], z0);
            X::fmac(acc[u], t1[u], z1);
          }
        }
      }
    }
    __syncthreads();
  }
  // skeleton part: w[skel[i]] = z[i]  (written once, by the block's first tile)
  if (tl.start == 0 && sidx == 0 && B.n_skel > 0) {
    for (int i = threadIdx.x; i < B.n_skel; i += ADJ_THREADS) {
      const int q = (B.flags & F_SKEL_IOTA) ? i : cx.idx[B.skel_off + i];
      static_cast<S *>(cx.part)[B.part_off + q] = adj_in<S>(cx, B, i, 0, from_f);
    }
  }
  // warp reductions
#pragma unroll
  for (int u = 0; u < CPW; ++u)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[u] = X::add(acc[u], X::shfl_xor(acc[u], o));
  if (!split) {
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < CPW; ++u) {
        const int col = cbase + u;
        if (col >= cend) continue;
        const int q = (B.flags & F_RED_IOTA) ? col : cx.idx[B.red_off + col];
        static_cast<S *>(cx.part)[B.part_off + q] = acc[u];
      }
    }
  } else {
    S *scratch = static_cast<S *>(cx.fsplit);
    const int grp = tl.pad >> 8;
    const int64_t sbase = B.asp_off + (int64_t)(tl.start / ACOLS) * B.pad2 * ACOLS;
    __shared__ int last;
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < CPW; ++u) scratch[sbase + (int64_t)sidx * ACOLS + warp * CPW + u] = acc[u];
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
      static_cast<S *>(cx.part)[B.part_off + q] = sum;
    }
    if (threadIdx.x == 0) cx.fcount[grp] = 0;  // re-arm for the next apply
  }
}

template <class S>
__global__ void __launch_bounds__(ADJ_THREADS, 7) adj_kernel(const Ctx cx, const Tile *__restrict__ tiles,
                                                             int from_f) {
  const Tile tl = tiles[blockIdx.y];
  pdl_trigger();
  {
    // L2 prefetch of the first 1 KB of each of this CTA's factor columns (a
    // whole-tile prefetch on few-tile stages measured neutral on c1 / c4,
    // profiles/r02_fwd_variants_ab.txt)
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
  adj_tile<S>(cx, tl, from_f);
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
// + 8)
template <class S, int MODE>
__host__ __device__ __forceinline__ int tile_row(int r) {
  if (MODE == 0) return r;
  return frag_row<S, true>(r & 7) + 8 * (r >> 3);
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
          {
            int64_t o = B.out_off + row;
            S *zb = z_out<S>(cx, B, o);
            zb[o * cx.nrhs + r] = val[t][v];
          }
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
constexpr int WS_MINB = 3;  // CTAs per SM the registers are sized for (<= 136 registers)
// Factor tile in shared memory (complex, BK = 16): forward padded column-major
// [k][64 + 2] filled by 1-D bulk copies (one per column of T); adjoint the two
// 128-byte-swizzled 2-D TMA boxes [half][m][128 B].  The +2 pad makes a
// quarter warp's 16-byte A-fragment loads (slots 2 tig + gid) hit distinct banks.
template <bool ADJ>
__host__ __device__ constexpr int ws_a_elems() {
  return ADJ ? MM_BM * 16 : 16 * (MM_BM + 2);
}
// B chunk: fragment order (BK x 8 NT slots)
template <int NT>
__host__ __device__ constexpr int ws_b_elems() {
  return 16 * 8 * NT;
}

template <bool ADJ, int NT>
__host__ __device__ constexpr int ws_smem_bytes() {
  // NS x (A tile + B chunk) operand buffers + 2 NS mbarriers + 1 KB to align
  // the stages to the 1024-byte period of the 128-byte TMA swizzle
  return WS_STAGES * (ws_a_elems<ADJ>() + ws_b_elems<NT>()) * 16 + 2 * WS_STAGES * 8 + 1024;
}

// Complex plans, nrhs >= 16: 8 NT right-hand sides per CTA (NT = 4 for nrhs >=
// 32, NT = 2 for 16..31) (profiles/r01_mma_ws_ab.txt: c2 nrhs 32 forward 18.1
// vs 21.5 ms, adjoint 18.5 vs 19.9 ms against the classic structure; the
// classic kernel's per-element forward gather ran the c5 stand-in's nrhs = 16
// forward at 20 TF).  Complex products by Gauss's 3-multiplication form.
template <bool ADJ, int NT>
__global__ void __launch_bounds__(WS_THREADS, WS_MINB) mma_ws_kernel(const Ctx cx, const Tile *__restrict__ tiles,
                                                                     int from_f) {
  using S = double2;
  using X = Tr<S>;
  using PL = Planes<S>;
  constexpr bool M3 = true;
  constexpr int BK = mm_bk<S>();
  constexpr int KS = BK / 4;
  constexpr int AW = MM_BM / 16;
  constexpr int A_CH = ws_a_elems<ADJ>();
  constexpr int AP = MM_BM + 2;  // forward tile leading dimension
  constexpr int MODE = ADJ ? 1 : 0;
  constexpr int B_CH = ws_b_elems<NT>();
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
  const int rhs0 = blockIdx.x * 8 * NT;
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
    int qn[KS];
#pragma unroll
    for (int k4 = 0; k4 < KS; ++k4) qn[k4] = nchunks > 0 ? row_index(0, k4) : -1;
    for (int kc = 0; kc < nchunks; ++kc) {
      const int slot = kc % NS;
      int q[KS];
#pragma unroll
      for (int k4 = 0; k4 < KS; ++k4) q[k4] = qn[k4];
      if (kc + 1 < nchunks) {
#pragma unroll
        for (int k4 = 0; k4 < KS; ++k4) qn[k4] = row_index(kc + 1, k4);
      }
      mbar_wait(empty + slot, ((kc / NS) & 1) ^ 1);
      const int kb = kbeg + kc * BK;
      const int kn = min(BK, kend - kb);  // valid k of this chunk
      S *dA = As + slot * A_CH;
      if (!ADJ) {
        // forward: column k of the tile = tl.count contiguous rows of T (TMA bulk copies)
        const unsigned cb = (unsigned)(tl.count * sizeof(S));
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
        tma_2d_g2s(dA, tmap, kb * 2, tl.start, full + slot);
        tma_2d_g2s(dA + MM_BM * KH, tmap, (kb + KH) * 2, tl.start, full + slot);
      }
      S *dB = Bs + slot * B_CH;
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
              rb[k4] = static_cast<const S *>(cx.c) + user_c_index(cx, off);
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
      mbar_cp_async_arrive(full + slot);  // completes when this lane's cp.async have landed
      mbar_arrive(full + slot);           // the register-path stores (if any) are done
    }
    return;  // the producer takes no part in the epilogue
  }

  // ------------------------------------------------ consumer warps
  const int gid = lane >> 2, tig = lane & 3;
  double c0[NT][4], c1[NT][4], c2[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int v = 0; v < 4; ++v) c0[t][v] = c1[t][v] = c2[t][v] = 0.0;
  const int m0 = warp * 16 + tile_row<S, MODE>(gid), m1 = warp * 16 + tile_row<S, MODE>(gid + 8);
  for (int kc = 0; kc < nchunks; ++kc) {
    const int slot = kc % NS;
    mbar_wait(full + slot, (kc / NS) & 1);
    const S *Ac = As + slot * A_CH;
    const S *Bc = Bs + slot * B_CH;
#pragma unroll
    for (int k4 = 0; k4 < KS; ++k4) {
      const int k = 4 * k4 + tig;
      S a0, a1;
      if constexpr (ADJ) {
        // swizzled [half][m][128 B]: 16-byte chunk c of row m sits at c ^ (m & 7)
        constexpr int KH = BK / 2;
        const int h = k / KH, c = k % KH;
        const unsigned char *hb = reinterpret_cast<const unsigned char *>(Ac) + h * (MM_BM * 128);
        a0 = *reinterpret_cast<const S *>(hb + m0 * 128 + ((c ^ (m0 & 7)) << 4));
        a1 = *reinterpret_cast<const S *>(hb + m1 * 128 + ((c ^ (m1 & 7)) << 4));
      } else {
        a0 = Ac[k * AP + m0];
        a1 = Ac[k * AP + m1];
      }
      const double ar0 = PL::re(a0), ar1 = PL::re(a1);
      // conj(T) for the adjoint
      const double ai0 = ADJ ? -PL::im(a0) : PL::im(a0), ai1 = ADJ ? -PL::im(a1) : PL::im(a1);
      const double as0 = ar0 + ai0, as1 = ar1 + ai1;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const S b = Bc[(k4 * NT + t) * 32 + lane];
        dmma(c0[t], ar0, ar1, PL::re(b));
        dmma(c1[t], ai0, ai1, PL::im(b));
        dmma(c2[t], as0, as1, PL::re(b) + PL::im(b));
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + slot);
  }
  // all consumer warps are past their last read of the operand buffers
  consumer_sync<1>();
  mma_epilogue<S, ADJ, NT, M3, 1, MODE>(cx, tl, B, c0, c1, c2, rhs0, ksplit, sidx, from_f, reinterpret_cast<int *>(As));
}

// dynamic shared memory above 48 KB is opted into per kernel and per device
// (the attribute applies to the device current when it is set): one device
// bitmask per kernel (the template argument is the kernel itself)
template <auto KERN>
void smem_optin(int bytes) {
  static unsigned long long done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && (done >> dev & 1ull)) return;
  cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (dev < 64) done |= 1ull << dev;
}

template <bool ADJ, int NT>
void mma_ws_launch(const Ctx &cx, const Tile *tiles, int nt, int from_f, cudaStream_t st) {
  constexpr int smem = ws_smem_bytes<ADJ, NT>();
  smem_optin<mma_ws_kernel<ADJ, NT>>(smem);
  launch_ex(PDL_MMA, mma_ws_kernel<ADJ, NT>, dim3((cx.nrhs + 8 * NT - 1) / (8 * NT), nt), dim3(WS_THREADS), smem, st, cx,
            tiles, from_f);
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
          srow = static_cast<const S *>(cx.c) + (int64_t)rhs0 * cx.m + user_c_index(cx, off);
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

// Real multi-RHS pipeline: K chunk 16 in a 2-stage cp.async ring at 6 CTAs/SM
// (80 registers): c3 +1.5% over a 3-stage ring at 4 CTAs/SM, and 16 > 32 for
// the chunk (c3 forward 6.9 -> 6.1 ms; profiles/r01_real_cfg_ab.txt,
// r01_real_occupancy_ab.txt)
constexpr int REAL_BK = 16, REAL_NSTG = 2, REAL_MINB = 6;

template <bool ADJ>
void mma_real_launch(const Ctx &cx, const Tile *tiles, int nt, int from_f, cudaStream_t st) {
  constexpr int smem = rb_smem_bytes<ADJ, REAL_BK, REAL_NSTG>();
  constexpr auto kern = mma_real_kernel<ADJ, REAL_BK, REAL_NSTG, REAL_MINB>;
  smem_optin<kern>(smem);
  launch_ex(PDL_MMA, kern, dim3((cx.nrhs + 31) / 32, nt), dim3(MM_THREADS), smem, st, cx, tiles, from_f);
}

// Multi-RHS dispatch: real plans at nrhs >= 32 -> mma_real_kernel; complex
// plans at nrhs >= 16 -> mma_ws_kernel (32 or 16 right-hand sides per CTA);
// narrower widths -> mma_kernel with 8 or 16 right-hand sides per CTA (complex
// products in Gauss's 3-product form).
template <class S, bool ADJ, int NT>
void mma_launch(const Ctx &cx, const Tile *tiles, int nt, int from_f, cudaStream_t st) {
  launch_ex(PDL_MMA, mma_kernel<S, ADJ, NT, true, 4>, dim3((cx.nrhs + 8 * NT - 1) / (8 * NT), nt), dim3(MM_THREADS), 0,
            st, cx, tiles, from_f);
}

template <class S, bool ADJ>
void mma_dispatch(const Ctx &cx, const Tile *tiles, int ntiles, int from_f, cudaStream_t st) {
  for (int t0 = 0; t0 < ntiles; t0 += 65535) {
    const int nt = ntiles - t0 < 65535 ? ntiles - t0 : 65535;
    if (cx.nrhs >= 32) {
      if constexpr (Planes<S>::cplx)
        mma_ws_launch<ADJ, 4>(cx, tiles + t0, nt, from_f, st);
      else
        mma_real_launch<ADJ>(cx, tiles + t0, nt, from_f, st);
    } else if (cx.nrhs >= 16) {
      if constexpr (Planes<S>::cplx)
        mma_ws_launch<ADJ, 2>(cx, tiles + t0, nt, from_f, st);
      else
        mma_launch<S, ADJ, 2>(cx, tiles + t0, nt, from_f, st);
    } else {
      mma_launch<S, ADJ, 1>(cx, tiles + t0, nt, from_f, st);
    }
  }
}

// ------------------------------------------------------------------------
// adjoint group sums: dst = sum of the readers' partial ranges (fixed order,
// no atomics).
// ------------------------------------------------------------------------
template <class S>
__device__ __forceinline__ void reduce_piece(const Ctx &cx, const Piece p, const int64_t *__restrict__ rd, int slice,
                                             int nslices, int tid, int nthr) {
  using X = Tr<S>;
  const S *part = static_cast<const S *>(cx.part);
  const int nr = cx.nrhs;
  const int total = p.len * nr;
  for (int e = slice * nthr + tid; e < total; e += nslices * nthr) {
    const int i = e / nr, r = e - (e / nr) * nr;  // RHS fastest (workspace layout)
    S s = X::zero();
    for (int q = 0; q < p.rd_count; ++q) {
      const S *a = part + (rd[p.rd_begin + q] + i) * nr + r;
      s = X::add(s, *a);
    }
    if (p.dst_src == SRC_C) {
      const int64_t ci = user_c_index(cx, p.dst_off + i);
      static_cast<S *>(cx.cw)[r * cx.m + ci] = cx.diag ? X::scale(s, diag_at(cx, ci)) : s;
    }
    else if (p.remote > 0 && cx.zrem)  // fused reverse exchange: into the owner's send buffer
      static_cast<S *>(cx.zrem[cx.zG + p.remote - 1])[(p.dst_off + cx.zdel[cx.zG + p.remote - 1] + i) * nr + r] = s;
    else
      static_cast<S *>(cx.z)[(p.dst_off + i) * nr + r] = s;
  }
}

template <class S>
__global__ void __launch_bounds__(256) reduce_kernel(const Ctx cx, const Piece *__restrict__ pieces,
                                                     const int64_t *__restrict__ rd) {
  pdl_trigger();
  pdl_wait();
  reduce_piece<S>(cx, pieces[blockIdx.x], rd, blockIdx.y, gridDim.y, threadIdx.x, blockDim.x);  // y: slices
}


constexpr int MAX_GRID_Y = 65535;

template <class S>
void fwd_dispatch(const Ctx &cx, const Tile *tiles, int ntiles, bool latency, cudaStream_t st) {
  for (int t0 = 0; t0 < ntiles; t0 += MAX_GRID_Y) {
    const int nt = ntiles - t0 < MAX_GRID_Y ? ntiles - t0 : MAX_GRID_Y;
    if (latency)
      launch_pdl(fwd_lat_kernel<S>, dim3(1, nt), dim3(FWD_THREADS), st, cx, tiles + t0);
    else
      launch_pdl(fwd_kernel<S>, dim3(1, nt), dim3(FWD_THREADS), st, cx, tiles + t0);
  }
}

template <class S>
void adj_dispatch(const Ctx &cx, const Tile *tiles, int ntiles, int from_f, cudaStream_t st) {
  for (int t0 = 0; t0 < ntiles; t0 += MAX_GRID_Y) {
    const int nt = ntiles - t0 < MAX_GRID_Y ? ntiles - t0 : MAX_GRID_Y;
    launch_pdl(adj_kernel<S>, dim3(1, nt), dim3(ADJ_THREADS), st, cx, tiles + t0, from_f);
  }
}

}  // namespace

void launch_fwd(bool is_complex, const Ctx &ctx, const Tile *tiles, int ntiles, bool latency, void *stream) {
  if (ntiles <= 0) return;
  if (is_complex)
    fwd_dispatch<double2>(ctx, tiles, ntiles, latency, (cudaStream_t)stream);
  else
    fwd_dispatch<double>(ctx, tiles, ntiles, latency, (cudaStream_t)stream);
}

void launch_adj(bool is_complex, const Ctx &ctx, const Tile *tiles, int ntiles, bool in_from_f, void *stream) {
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

namespace {
// Fused exchange signalling.  The kernel boundary before xsignal orders every
// earlier store of the stream (the remote stores into the peers' buffers
// included) before it; the system-scope fence then makes them visible to the
// peers before the release store of the flag.
__global__ void xsignal_kernel(unsigned long long *own_sync, unsigned long long *const *peer_sync, int dir, int g,
                               int G) {
  __shared__ unsigned long long e;
  unsigned long long *epoch = own_sync + 2 * G;
  if (threadIdx.x == 0) e = ++epoch[dir];  // this rank's counter: single writer
  __syncthreads();
  if (threadIdx.x < G) {
    unsigned long long *f = peer_sync[threadIdx.x] + dir * G + g;
    asm volatile("fence.sc.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(e) : "memory");
  }
}
__global__ void xwait_kernel(const unsigned long long *own_sync, int dir, int G) {
  const unsigned long long e = own_sync[2 * G + dir];  // incremented by this rank's own xsignal
  if (threadIdx.x < G) {
    const unsigned long long *f = own_sync + dir * G + threadIdx.x;
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(f) : "memory");
      if (v >= e) break;
      __nanosleep(256);
    }
  }
  __syncthreads();
}
}  // namespace

void launch_xsignal(unsigned long long *own_sync, unsigned long long *const *peer_sync, int dir, int g, int G,
                    void *stream) {
  xsignal_kernel<<<1, 32 * ((G + 31) / 32), 0, (cudaStream_t)stream>>>(own_sync, peer_sync, dir, g, G);
}
void launch_xwait(const unsigned long long *own_sync, int dir, int G, void *stream) {
  xwait_kernel<<<1, 32 * ((G + 31) / 32), 0, (cudaStream_t)stream>>>(own_sync, dir, G);
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
