// Internal device-side layout of a loaded butterfly plan (libmht).
//
// The plan file's per-stage block tables are resolved on the
// host into a flat list of *materialised* blocks — the ones that do work —
// plus per-stage tile lists.  IDENTITY blocks whose two input segments are
// adjacent in memory become aliases and cost nothing (SURVEY.md §8(a) a2:
// "the level permutation lives in these offsets").
#pragma once
#include <cstdint>

namespace mht {

enum : int32_t {
  SRC_C = 0,     // user coefficient vector c (ld = m)
  SRC_Z = 1,     // plan workspace zpool (ld = Zt)
};

enum : int32_t {
  F_SKEL_IOTA = 1,  // skeleton positions are 0..n_skel-1 (COPY blocks)
  F_RED_IOTA = 2,   // redundant positions are 0..n_red-1 (DENSE blocks)
  F_OUT_F = 4,      // output rows go to f through perm_x (leaf stage)
  F_REMOTE = 8,     // sharded switch stage: outputs bound for rank (flags >> 16); with the
                    // fused exchange on they are stored straight into that rank's receive buffer
};

// One materialised block: out[i] = in[skel[i]] (i < n_skel) + sum_j T[i,j] in[red[j]]
// with in = concat(seg0, seg1), T column-major r_out x n_red (ld = r_out).
struct DevBlock {
  int64_t coef_off;    // element offset of T in the coefficient pool
  int64_t skel_off;    // offset into the index pool (ID blocks)
  int64_t red_off;     // offset into the index pool (ID blocks)
  int64_t seg_off[2];  // element offset of each input segment in its source
  int64_t out_off;     // zpool offset (stages 0..L) or sp_off row (leaf stage)
  int64_t part_off;    // adjoint partial slot (r_in entries)
  int32_t seg_len[2];
  int32_t seg_src[2];  // SRC_C | SRC_Z
  int32_t r_out, r_in, n_skel, n_red;
  int32_t flags;
  int32_t pad;  // forward column splits (nrhs = 1), 0 = none
  // adjoint input fused into the load: z[i] = sum_k part[rdtab[rd_off + k] + i]
  // over the rd_cnt readers of this block's output (-1: not fusable, read z).
  int64_t rd_off;
  int32_t rd_cnt;
  int32_t pad2;     // adjoint row splits (nrhs = 1), 0 = none
  int64_t fsp_off;  // split scratch base of this block's forward row tiles (scalars)
  int64_t asp_off;  // split scratch base of this block's adjoint column tiles (scalars)
  int32_t ld;       // leading dimension of T in the device pool (r_out, rounded up to
                    // even for float64 so every column starts 16-byte aligned)
  int32_t mks;      // multi-RHS adjoint K (row) splits, 0 = none
  int64_t msp_off;  // first split slab of this block's multi-RHS adjoint tiles
};
static_assert(sizeof(DevBlock) == 144, "DevBlock layout");

// Device repack of one block's factor (real plans): column-major r_out x ncols
// with ld = r_out  ->  ld = dst_ld (>= r_out), padding rows zero.
struct Repack {
  int64_t src_off, dst_off;
  int32_t r_out, ncols, dst_ld, pad;
};

// A unit of work: rows [start, start+count) (forward) or redundant columns
// [start, start+count) (adjoint) of block `blk`.
struct Tile {
  int32_t blk, start, count;
  int32_t pad;  // forward split tiles: (group << 8) | split; -1 otherwise
};

// Adjoint group-sum piece: dst[dst_off + i] = sum_r part[rd[rd_begin + r] + i].
struct Piece {
  int64_t dst_off;
  int64_t rd_begin;
  int32_t dst_src;  // SRC_C | SRC_Z
  int32_t len;
  int32_t rd_count;
  int32_t remote;   // sharded: 1 + the rank whose send buffer this receive-buffer sum belongs to, else 0
};

struct Ctx {  // per-launch pointers
  const void *coef;
  const int32_t *idx;
  const int32_t *perm;
  const int32_t *permk;  // plan frequency position -> user c index (plan v2), nullptr = identity
  const DevBlock *blocks;
  const void *c;   // SRC_C base
  void *cw;        // writable c (adjoint output)
  void *z;         // zpool
  void *part;      // partial pool
  const void *fin; // f input (adjoint)
  void *fout;      // f output (forward)
  void *fsplit;    // forward split-K partial rows
  void *msplit;    // multi-RHS adjoint split slabs: [slab][64 columns][nrhs]
  int *mcount;     // multi-RHS adjoint split arrival counters [group][rhs chunk]
  int *fcount;     // forward split-K arrival counters (zero between applies)
  const double *diag;    // optional real diagonal on the coefficient side (m entries):
                         // forward reads c_k * g(d_k), adjoint writes g(d_k) * c_k
  int diag_sqrt;         // g(d) = sqrt(d) (GRF sampling) instead of d
  const int64_t *rdtab;  // fused adjoint sums: reader partial offsets
  const void *tmaps;     // per-block 2-D TMA descriptors of T (CUtensorMap, 128 B each; complex adjoint tiles)
  int fused;             // 1: adjoint inputs are summed from the partials on load
  int64_t m, n, Zt, Pt;  // Zt/Pt: workspace entries per RHS (layout [entry][rhs])
  int nrhs;
  // fused exchange of a sharded plan (nullptr: off): zrem[h] / zdel[h] (h < G)
  // the base and entry delta of rank h's receive buffer for this rank's
  // switch-stage outputs, zrem[G + g] / zdel[G + g] those of rank g's send
  // buffer for the adjoint sums formed here
  void *const *zrem;
  const int64_t *zdel;
  int zG;
};

constexpr int FWD_ROWS = 64;     // rows per forward tile (2 per lane)
constexpr int FWD_THREADS = 128; // 4 warps split the columns
constexpr int ADJ_COLS = 32;     // redundant columns per adjoint tile, complex (8 per warp)
constexpr int ADJ_COLS_REAL = 64;  // ... real (16 per warp)
template <class S>
__host__ __device__ constexpr int adj_cols() { return sizeof(S) == 16 ? ADJ_COLS : ADJ_COLS_REAL; }
constexpr int ADJ_THREADS = 128;
constexpr int ADJ_RCH = 1024;    // adjoint rows staged in smem per pass (most blocks: one pass;
                                 // 256 / 512 measured 8% slower on c2, profiles/r01_adj_rch_ab.txt)
constexpr int MMA_COLS = 64;     // redundant columns per multi-RHS adjoint tile

// LSQR per-column state (device resident; mht_lsqr.cu)
struct LsqrCol {
  double alpha, beta, rhobar, phibar, cs;
  double step_x, step_w;        // x += step_x w;  w = v - step_w w
  double rnorm, arnorm, anorm2, bnorm, xnorm;
};

// LSQR vector kernels (mht_lsqr.cu).  stage: 0 beta / 1 alpha + rotation /
// 2 initial beta / 3 initial alpha.  which: 0 alpha, 1 beta (axpy); 0 beta,
// 1 alpha (scale).
int lsqr_partials(int64_t len);
void lsqr_axpy_norm(bool cplx, const void *y, void *u, int64_t len, int k, const LsqrCol *col, int which,
                    double *partial, void *stream);
void lsqr_scalars(const double *partial, int nblk, int k, LsqrCol *col, int stage, void *stream);
void lsqr_scale(bool cplx, void *u, int64_t len, int k, const LsqrCol *col, int which, void *stream);
void lsqr_update(bool cplx, void *v, void *w, void *x, int64_t len, int k, const LsqrCol *col, int first,
                 void *stream);
void lsqr_xnorm(bool cplx, const void *x, int64_t len, int k, double *partial, LsqrCol *col, void *stream);

// Launchers (mht_kernels.cu).  is_complex selects double2 vs double.
// latency: the few-tile variant (x staged per chunk, balanced batches, L2
// prefetch) instead of the streaming one; the loader picks per stage.
void launch_fwd(bool is_complex, const Ctx &ctx, const Tile *tiles, int ntiles, bool latency, void *stream);
void launch_adj(bool is_complex, const Ctx &ctx, const Tile *tiles, int ntiles, bool in_from_f, void *stream);
// multi-RHS (nrhs >= 2): DMMA kernels; forward uses the 64-row tiles, the
// adjoint uses 64-column tiles (adjm lists).
void launch_mma(bool is_complex, bool adjoint, const Ctx &ctx, const Tile *tiles, int ntiles, bool in_from_f,
                void *stream);
void launch_repack(const double *src, double *dst, const Repack *jobs, int njobs, void *stream);
void launch_reduce(bool is_complex, const Ctx &ctx, const Piece *pieces, const int64_t *rd,
                   int npieces, void *stream);
// fused exchange signalling (sharded plans): own_sync = this rank's
// [2][G] arrival flags then its 2 epoch counters; peer_sync[h] = rank h's.
// signal: epoch[dir] += 1, then flag[dir][g] = epoch on every rank (system
// scope, after a system fence); wait: until every flag[dir][*] >= epoch[dir].
void launch_xsignal(unsigned long long *own_sync, unsigned long long *const *peer_sync, int dir, int g, int G,
                    void *stream);
void launch_xwait(const unsigned long long *own_sync, int dir, int G, void *stream);

}  // namespace mht
