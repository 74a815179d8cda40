/*
 * libmht — B200 (sm_100a) butterfly manifold-harmonic-transform apply.
 *
 * The C ABI of the hot path of arxiv/paper_2605_21828 ("butterfly-accelerated
 * manifold harmonic transform", BF-MHT).  The library applies a precomputed
 * row-wise butterfly factorization of the MHT matrix
 *
 *     Phi in C^{n x m},  Phi_jk = phi_k(x_j)     (§1 Eq. MHT-sum)
 *
 * to coefficient vectors (synthesis f = Phi c) and applies its adjoint
 * (analysis c = Phi^* f; "fast adjoint transform", §1).  The
 * factorization {V_nu, R_{tau nu}, U_tau} is the one of §2:
 * leaf projection, L transfer levels, leaf interpolation, applied "one
 * multiply per stored factor" (§6.2).  Multi-RHS
 * (§7.1; §7.2) applies the same operator to nrhs
 * columns.  Factor construction is a host precompute that writes a plan file
 * (format: DESIGN.md §4); this library only loads and applies it.
 *
 * Conventions for every entry point
 *  - Element type is fixed by the plan: MHT_DTYPE_C128 = interleaved complex
 *    double (re, im) (flat square), MHT_DTYPE_F64 = double (sphere, meshes).
 *  - Vectors are column-major blocks: c is m x nrhs with leading dimension m
 *    (a contiguous (nrhs, m) array), f is n x nrhs with leading dimension n.
 *  - c is in the user's frequency order (eigenvalue order); f is in the user's
 *    point order.  The plan's perm_x maps its space-tree order back to the
 *    points; a version-2 plan's perm_k maps its frequency-tree order back to
 *    the coefficients (the quadtree-frequency plans, reading A18),
 *    fused into the loads / stores of c like perm_x into those of f.
 *  - Device-pointer calls (mht_apply, mht_apply_adjoint) enqueue on the plan's
 *    stream and return without synchronising; a device fault surfaces as
 *    MHT_ERR_CUDA on a later call or on mht_sync.
 *  - A plan owns all device memory for factors and workspace; the caller owns
 *    c and f.  Destinations are fully overwritten (c = 0 gives f = 0 exactly).
 *  - A plan is NOT safe for concurrent applies (shared workspace).  Different
 *    plans may be used from different threads.
 *  - No C++ exception crosses this boundary.  Every function returns a status;
 *    mht_last_error() gives a thread-local detail string for the last failure.
 */
#ifndef MHT_H_
#define MHT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mht_plan mht_plan; /* opaque */

typedef enum {
  MHT_OK = 0,
  MHT_ERR_INVALID_ARG = 1, /* null pointer, nrhs < 1, bad device id        */
  MHT_ERR_FORMAT = 2,      /* bad magic/version/checksum, chain invariant  */
  MHT_ERR_SHAPE = 3,       /* inconsistent sizes inside the plan           */
  MHT_ERR_OOM = 4,         /* host or device allocation failed             */
  MHT_ERR_CUDA = 5,        /* CUDA runtime error (incl. earlier async faults) */
  MHT_ERR_UNSUPPORTED = 6, /* no sm_100 device / feature not built          */
  MHT_ERR_IO = 7           /* file open/read failure                        */
} mht_status;

enum { MHT_DTYPE_F64 = 1, MHT_DTYPE_C128 = 2 };

typedef struct {
  int64_t n, m;          /* rows (points) and columns (eigenfunctions) of Phi */
  int32_t L;             /* tree depth: 2^L leaves on both trees             */
  int32_t dtype;         /* MHT_DTYPE_F64 | MHT_DTYPE_C128                   */
  double tol;            /* ID tolerance the plan was built with             */
  int64_t plan_bytes;    /* bytes of the plan file                           */
  int64_t factor_entries;/* stored non-identity coefficients (T and U)       */
  int64_t device_bytes;  /* device memory held by factors + index tables     */
  int64_t index_entries; /* int32 skeleton/redundant indices on the device   */
  int32_t n_materialized;/* blocks that run (ID, DENSE, COPY)                */
  int32_t n_alias;       /* identity blocks resolved to an alias (no work)   */
  int32_t fwd_launches;  /* kernel launches per forward apply                */
  int32_t adj_launches;  /* kernel launches per adjoint apply                */
} mht_plan_info;

/* Parse + validate a plan file, pack it into the level-contiguous device
 * layout and upload it to `device` (a CUDA ordinal).  The plan holds the
 * factorization of PAPER.md §2: space tree (perm_x, leaf
 * offsets), frequency tree (leaf offsets), per-level ID transfer blocks
 * X = [I T] Pi and the leaf interpolation blocks U_tau.  Reads the whole file
 * once; the checksum is verified on the fly.  *out is set only on MHT_OK.
 * Errors: MHT_ERR_IO (open/read), MHT_ERR_FORMAT (magic, version, checksum,
 * chain invariant r_in = r_out(p,c1) + r_out(p,c2)),
 * MHT_ERR_SHAPE, MHT_ERR_OOM, MHT_ERR_CUDA, MHT_ERR_UNSUPPORTED. */
mht_status mht_plan_load(const char *path, int device, mht_plan **out);

/* Sizes of the loaded plan (SPEC S:293-300 memory report: stored entries,
 * bytes).  Never fails on a valid plan. */
mht_status mht_plan_info_get(const mht_plan *plan, mht_plan_info *info);

/* Stream for subsequent calls (a cudaStream_t passed as void*; NULL = the
 * legacy default stream).  Callers using PyTorch pass
 * torch.cuda.current_stream().cuda_stream.  The caller keeps ownership of
 * `stream`; the plan's own loader stream stays owned by the plan.  Work
 * queued on the previous stream is synchronised first. */
mht_status mht_plan_set_stream(mht_plan *plan, void *stream);

/* Pre-size the workspace for up to `nrhs` right-hand sides (otherwise grown
 * on demand by the first apply with a larger nrhs, which synchronises). */
mht_status mht_reserve(mht_plan *plan, int nrhs);

/* Synthesis f = Phi_BF c (Eq. MHT-sum, f_j = sum_k c_k
 * phi_k(x_j); evaluated through the factorization of §2, one
 * multiply per stored factor).  c: device, m x nrhs (ld m), in
 * the user's frequency order (perm_k, if any, applied on load); f: device, n x nrhs (ld n), user point order,
 * fully overwritten.  Runs the leaf projection, the L transfer stages and the
 * leaf interpolation (perm_x scatter fused into the store).  nrhs >= 1;
 * c and f must not overlap.  Errors: MHT_ERR_INVALID_ARG (null, nrhs < 1,
 * sharded plan), MHT_ERR_OOM (workspace growth), MHT_ERR_CUDA. */
mht_status mht_apply(mht_plan *plan, const void *c, void *f, int nrhs);

/* Analysis c = Phi_BF^* f (the "fast adjoint transform", PAPER.md P:153-155,
 * §1; used by the inverse MHT, and covariance products,
 * P:1196-1198).  f: device n x nrhs (ld n, user point order); c: device
 * m x nrhs (ld m), fully overwritten.  Exact reverse of mht_apply with
 * conjugate transposes; the sum over the two transfers that read a block row
 * is formed from per-block partials in a fixed order (no atomics, bitwise
 * deterministic).  Errors as mht_apply. */
mht_status mht_apply_adjoint(mht_plan *plan, const void *f, void *c, int nrhs);

/* Same operations as mht_apply / mht_apply_adjoint from
 * and to HOST memory: copies c (or f) host->device on the plan stream,
 * applies, copies the result device->host and synchronises.  The output host
 * buffer must hold n*nrhs (or m*nrhs) scalars of the plan's dtype (the C side
 * cannot check this).  Host
 * buffers should be pinned for full copy bandwidth.  Used for the end-to-end
 * measurement. */
mht_status mht_apply_host(mht_plan *plan, const void *c_host, void *f_host, int nrhs);
mht_status mht_apply_adjoint_host(mht_plan *plan, const void *f_host, void *c_host, int nrhs);

/* A batch of independent host-buffer transforms, pipelined (the serving
 * loop's end-to-end path): job i is a synthesis (dir 0: in = c, m x nrhs;
 * out = f, n x nrhs) or an analysis (dir 1: in = f, out = c;
 * P:153-155), both host pointers in the ABI layout (pinned for full copy
 * bandwidth).  Job i's host-to-device copy and job i-1's device-to-host copy
 * run on the plan's copy streams while job i-1 / job i transform, through two
 * device staging slots ordered by events, so copies overlap the transforms.
 * Returns when every output is in host memory.  Results are bitwise those of
 * mht_apply_host / mht_apply_adjoint_host.  Inputs and outputs must not
 * overlap each other.  Errors: MHT_ERR_INVALID_ARG (null plan or job pointer,
 * dir not 0/1, nrhs < 1, sharded plan), MHT_ERR_OOM, MHT_ERR_CUDA. */
typedef struct {
  int32_t dir;  /* 0 synthesis, 1 analysis */
  int32_t nrhs;
  const void *in;
  void *out;
} mht_host_job;
mht_status mht_apply_host_batch(mht_plan *plan, const mht_host_job *jobs, int njobs);

/* ---- sharded plans: one plan across G GPUs -----------
 * The factorization is split at a switch level ls (log2 G <= ls <= L - log2 G;
 * switch_level < 0 picks max(log2 G, L/2)).  Rank g holds, for stages 0..ls,
 * the blocks of the g-th frequency subtree at height L - log2 G (a frequency
 * block (tau, nu) only reads its children nu's, §2) and,
 * for stages ls+1..L+1, the blocks of the g-th space subtree at depth log2 G
 * (only reads its parent tau's).  The one exchange step is an all-to-all of
 * z_ls: rank g sends rank h the z_ls(tau, nu) with tau in h's space subtree
 * and nu in g's frequency subtree.  Each rank loads and stores only its own
 * blocks' coefficients (~1/G of the plan; the whole-file checksum is not
 * verified by a shard).  nshards = 1 loads the whole plan (= mht_plan_load).
 * G must be a power of two. */
mht_status mht_plan_load_shard(const char *path, int device, int nshards, int shard, int switch_level,
                               mht_plan **out);
/* Exchange layout, in workspace entries (each entry = nrhs scalars, the
 * workspace is [entry][rhs]): arrays of nshards.  send_off/len[h]: the block
 * this rank sends to rank h (contiguous, ascending h); recv_off/len[g]: where
 * the block from rank g lands (contiguous, ascending g).  Any pointer may be
 * NULL.  nshards/shard/switch_level report the plan's sharding. */
mht_status mht_shard_info(const mht_plan *plan, int32_t *nshards, int32_t *shard, int32_t *switch_level,
                          int64_t *send_off, int64_t *send_len, int64_t *recv_off, int64_t *recv_len);
/* Ensure the workspace for nrhs columns and return its device base pointer
 * (the buffer the exchange reads and writes).  May synchronise (growth). */
mht_status mht_shard_workspace(mht_plan *plan, int nrhs, void **zpool);
/* Sharded synthesis: begin runs stages 0..ls on this rank's slice of c (c is
 * the full m x nrhs array; only this rank's frequency range is read) and
 * leaves the send blocks in the workspace; after the caller's all-to-all
 * (send -> recv), end runs stages ls+1..L+1 and writes this rank's rows of f
 * (full n x nrhs array; other rows untouched). */
mht_status mht_apply_shard_begin(mht_plan *plan, const void *c, int nrhs);
mht_status mht_apply_shard_end(mht_plan *plan, void *f, int nrhs);
/* Sharded analysis: begin reads this rank's rows of f and leaves the adjoint
 * of z_ls in the RECEIVE blocks; after the reverse all-to-all (recv -> send),
 * end finishes and writes this rank's frequency range of c (other entries
 * untouched). */
mht_status mht_apply_adjoint_shard_begin(mht_plan *plan, const void *f, int nrhs);
mht_status mht_apply_adjoint_shard_end(mht_plan *plan, void *c, int nrhs);

/* Fused exchange (one process per GPU on one node, NVLink /
 * NVSwitch peer memory): instead of an all-to-all between _begin and _end,
 * the switch stage's kernels store every z_ls block bound for rank h straight
 * into rank h's receive buffer (remote stores, so the transfer overlaps the
 * stage's math tile by tile), and in the analysis the sums of z_ls's adjoint
 * formed for rank g are stored straight into rank g's send buffer; _begin then
 * signals every rank (system-scope release of a per-rank arrival flag after a
 * system fence) and _end waits for every rank's flag before reading.  No
 * collective library call is left on the data path.  All ranks must run the
 * same sequence of sharded applies at the same nrhs (<= the set-up nrhs).
 *   mht_shard_export:  sizes the workspace for `nrhs` right-hand sides and
 *     writes this rank's IPC handle of it (cudaIpcMemHandle_t, 64 bytes; NULL
 *     to skip) and its layout: layout[0..G) = receive offsets per source,
 *     layout[G..2G) = send offsets per destination (workspace entries),
 *     layout[2G] = the byte offset of its sync area (2 G + 2 u64, zeroed).
 *   mht_shard_open_peers:  opens the other ranks' handles (ipc_handles: G x 64
 *     bytes in rank order; this rank's entry is ignored) and sets them up.
 *   mht_shard_set_peers:  the same from device pointers already mapped in this
 *     process (bases[h] = rank h's workspace; bases[shard] must be this plan's
 *     own) — the one-process emulation of G ranks on one GPU.
 *   layouts: G x (2 G + 1) int64, rank h's export at h (2 G + 1).
 *   mht_shard_close_peers: back to the all-to-all path, IPC mappings released.
 * Errors: MHT_ERR_INVALID_ARG (not sharded, bad pointers, nrhs above the
 * set-up width), MHT_ERR_OOM, MHT_ERR_CUDA (IPC failures included). */
mht_status mht_shard_export(mht_plan *plan, int nrhs, void *ipc_handle, int64_t *layout);
mht_status mht_shard_open_peers(mht_plan *plan, int nrhs, const void *ipc_handles, const int64_t *layouts);
mht_status mht_shard_set_peers(mht_plan *plan, int nrhs, void *const *bases, const int64_t *layouts);
mht_status mht_shard_close_peers(mht_plan *plan);

/* ---- applications on top of the transform (§7) ----------------
 * A real diagonal on the coefficient side is fused into the transform's own
 * loads of c (synthesis) or its final stores of c (analysis): no extra pass
 * over c.  d / S: device float64 arrays of m entries in the order of c; the
 * same diagonal for every right-hand side.
 *
 * Spectral filtering (§7.1):  f = Phi diag(F(lambda)) c. */
mht_status mht_apply_diag(mht_plan *plan, const void *c, const double *d, void *f, int nrhs);
/* Filtered analysis:  c = diag(d) Phi^* f. */
mht_status mht_apply_adjoint_diag(mht_plan *plan, const void *f, const double *d, void *c, int nrhs);
/* Gaussian random field samples (§7.2, Eq. KL-expansion):
 * y = Phi sqrt(S) z with z ~ N(0, I) supplied by the caller (m x nrhs; for a
 * complex plan, complex z); sqrt(S_k) is taken inside the fused load. */
mht_status mht_grf_sample(mht_plan *plan, const void *z, const double *S, void *y, int nrhs);
/* Covariance matrix-vector product (§7.2):  out = Phi S Phi^* v
 * (v, out: n x nrhs).  Analysis with S fused into its final sums into a plan-
 * owned m x nrhs buffer, then synthesis. */
mht_status mht_covariance_apply(mht_plan *plan, const void *v, const double *S, void *out, int nrhs);

/* Inverse MHT by LSQR (§7.1, Eq. inverse-MHT):
 *   x = argmin_c ||Phi c - b||_2  for each of the nrhs columns of b.
 * b: device n x nrhs; x: device m x nrhs (output; the iterate).  Paige &
 * Saunders' LSQR from x_0 = 0; each iteration is one synthesis and one
 * analysis of the plan plus fused vector kernels; all per-column scalars stay
 * on the device.  Stops after max_iters, or earlier (checked every 10
 * iterations) when every column satisfies Paige & Saunders' test 1
 * ||r|| <= btol ||b|| + atol ||A|| ||x|| or test 2 ||A^* r|| <= atol ||A|| ||r||
 * (atol = btol = 0: exactly max_iters iterations).  Optional host outputs:
 * *iters_done, and per column rnorm[r] ~ ||b - Phi x||, arnorm[r] ~ ||Phi^*(b - Phi x)||
 * (the recurrences' estimates).  Synchronises.  Work vectors (5 vectors of
 * n or m x nrhs) are owned by the plan and grown with nrhs. */
mht_status mht_lsqr(mht_plan *plan, const void *b, void *x, int nrhs, int max_iters, double atol, double btol,
                    int *iters_done, double *rnorm, double *arnorm);

/* Execution option (no paper passage): capture each
 * (direction, nrhs, c, f) apply sequence in a CUDA graph and replay it on later
 * calls with the same arguments (on = 1, default on). */
mht_status mht_set_graphs(mht_plan *plan, int on);

/* Adjoint group sums (a block row read by two transfers receives
 * the sum of both adjoint contributions).  on = 1 (default): each consumer
 * sums its producers' per-block partials while loading its input, so no
 * separate reduction pass runs except the final one into c (used at nrhs = 1;
 * multi-RHS applies always reduce first, which measured faster).  on = 0: one
 * reduce pass per stage writes the sums to the workspace first.  Both orders
 * add the same partials in the same order (results are bitwise identical).
 * Synchronises the plan's stream and drops captured graphs. */
mht_status mht_set_fused_sums(mht_plan *plan, int on);

/* Block until the plan's stream is idle; returns MHT_ERR_CUDA on a fault
 * (the asynchronous error surface of the calls above). */
mht_status mht_sync(mht_plan *plan);

/* Per-stage statistics of the packed plan (bytes per level, the paper's
 * storage-as-runtime proxy).  stage in [0, L+1].
 *   coef_bytes: factor bytes read by the stage per apply (per RHS column);
 *   n_tiles_fwd / n_tiles_adj: work tiles; n_mat: materialised blocks. */
mht_status mht_stage_stats(const mht_plan *plan, int stage, int64_t *coef_bytes,
                           int32_t *n_mat, int32_t *n_tiles_fwd, int32_t *n_tiles_adj);

/* Kernel-level profiling on the launching stream (measurement).  When on, every kernel
 * launch of an apply is bracketed by CUDA events (kind 0 = forward stage,
 * 1 = adjoint stage, 2 = adjoint group-sum).  mht_profile_get synchronises and
 * returns the summed device time (ms) and launch count over all recorded
 * launches of (kind, stage, nrhs); stage = -1 or nrhs = 0 match any.
 * mht_profile_reset drops the records (keeps profiling on/off as is). */
mht_status mht_set_profiling(mht_plan *plan, int on);
mht_status mht_profile_get(mht_plan *plan, int kind, int stage, int nrhs, double *ms, int64_t *launches);
mht_status mht_profile_reset(mht_plan *plan);

/* Destroy the plan and every device buffer it owns (synchronises its
 * streams first).  NULL is a no-op. */
void mht_plan_destroy(mht_plan *plan);

const char *mht_status_string(mht_status s);
const char *mht_last_error(void);

/* Status name / thread-local detail of the last failure; build id ("sm_100a ..."). */
const char *mht_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* MHT_H_ */
