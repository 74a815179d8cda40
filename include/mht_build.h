/*
 * libmht — device kernels of the plan construction.
 *
 * The butterfly factorization is a precompute outside the timed apply path
 * (§2: "the precomputation ... is dominated by level 0",
 * O(r^2 n m)).  Its inner steps are evaluating the selected submatrices of
 * Phi (P:231-239 level 0, P:241-271 transfers: the blocks Phi(tau, J) of the
 * skeleton columns J) and their column interpolative decompositions (
 * reading A5: column-pivoted QR, rank k = first j with |R_jj| <= tol |R_00|,
 * T = R11^{-1} R12).  These entry points run those steps as hand-written
 * sm_100a kernels on batches of blocks; the host builder
 * (paper_2605_21828_b200/precompute/gpu_builder.py) only arranges the batches,
 * draws the Gaussian sketches (library GEMM) and writes the plan file.
 *
 * Conventions (as include/mht.h): device pointers unless stated, enqueued on
 * `stream` (a cudaStream_t as void*, NULL = legacy default stream), no
 * synchronisation; errors as mht_status with mht_last_error() detail; no
 * C++ exception crosses the boundary.  Batched blocks are stored
 * "column-contiguous": At[b][c][r] = A_b(r, c), i.e. B consecutive C x R
 * row-major arrays, each the transpose of the R x C block A_b, so column c of
 * A_b is R consecutive scalars.
 */
#ifndef MHT_BUILD_H_
#define MHT_BUILD_H_

#include <stdint.h>

#include "mht.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Flat-square basis blocks evaluated in-kernel (PAPER.md P:53-56 and P:84-90:
 * phi_k(x) = exp(i k.x), unnormalised, reading A11):
 *   At[b][c][r] = exp(i (k[cols[b][c]] . x[rows[b][r]]))     (complex128)
 * and 0 where rows[b][r] < 0 or cols[b][c] < 0 (batch padding).
 *   x:    n x 2 doubles (point coordinates), k: m x 2 doubles (wave vectors);
 *   rows: B x R int64 point indices (-1 = padding); cols: B x C int64 mode
 *         indices (-1 = padding); At: B x C x R complex128, fully written.
 * Indices are not range-checked against n / m (caller contract).
 * Errors: MHT_ERR_INVALID_ARG (null pointer, B, R or C < 0), MHT_ERR_CUDA. */
mht_status mhtb_flat_blocks(const double *x, const double *k, const int64_t *rows, const int64_t *cols, int B,
                            int R, int C, void *At, void *stream);

/* Real orthonormal spherical harmonics at n points (§6.2 sphere
 * basis; reading A11: Y_l0 = N_l0 P_l, Y_lm = sqrt2 N_lm P_l^m cos(m phi),
 * Y_l,-m = sqrt2 N_lm P_l^m sin(m phi), no Condon-Shortley phase), by the
 * fully-normalised associated-Legendre recurrence in theta:
 *   Y[j * (lmax+1)^2 + l^2 + l + m] = Y_lm(theta_j, phi_j),  l <= lmax, |m| <= l.
 *   theta, phi: n doubles (colatitude, longitude); Y: n x (lmax+1)^2 doubles.
 * Errors: MHT_ERR_INVALID_ARG (null, n < 0, lmax < 0 or > 2047), MHT_ERR_CUDA. */
mht_status mhtb_sphere_table(const double *theta, const double *phi, int64_t n, int lmax, double *Y, void *stream);

/* Batched Householder QR with column pivoting (Businger-Golub; the pivot is
 * the first column of largest remaining norm, the norms recomputed exactly
 * after every reflector) of the B blocks A_b = At_b^T, in place, with the
 * rank rule of reading A5: ranks[b] = the first j with
 * |R_jj| <= tol * |R_00| (min(R, C) if none); the factorization of block b
 * stops at that step.  On return, for j < ranks[b] and r <= j:
 *   At[b][j'][r] = R_b(r, j') for every column position j' (R's first
 *   ranks[b] rows; entries below the diagonal of the first ranks[b] columns
 *   are zero), and perm[b][j'] = the original column at position j'.
 *   At:    B x C x R scalars (dtype MHT_DTYPE_F64 double or MHT_DTYPE_C128
 *          interleaved complex double), overwritten;
 *   ranks: B int64 (device); perm: B x C int64 (device).
 * Limits: one CTA (1,024 threads) per block; the column norms and the
 * permutation live in shared memory (12 C bytes <= 220 KB, else
 * MHT_ERR_UNSUPPORTED), the Householder vector too when it fits, otherwise in
 * a stream-ordered scratch allocation (B R scalars, freed on the stream).
 * Errors: MHT_ERR_INVALID_ARG (null, B/R/C < 0, bad dtype), MHT_ERR_UNSUPPORTED,
 * MHT_ERR_OOM, MHT_ERR_CUDA. */
mht_status mhtb_cpqr(void *At, int B, int C, int R, int dtype, double tol, int64_t *ranks, int64_t *perm,
                     void *stream);

#ifdef __cplusplus
}
#endif

#endif /* MHT_BUILD_H_ */
