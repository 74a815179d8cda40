/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the butterfly MHT hot path
 * (arxiv/paper_2605_21828).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with the CUDA path (paper_2605_21828_b200/);
 * it has its own plan-file reader written from the format description in
 * DESIGN.md §4.
 *
 * O1 — dense direct sums (the result the method approximates):
 *   f_j  = sum_k c_k phi_k(x_j)                (§1 Eq. MHT-sum)
 *   c'_k = sum_j conj(phi_k(x_j)) f_j          (adjoint, "fast adjoint transform",
 *                                               P:153-155, §1)
 *   flat:   phi_k(x) = exp(i (k1 x1 + k2 x2))  (§1 Eq. 2D-DFT; §5)
 *   sphere: real orthonormal spherical harmonics, Condon–Shortley phase excluded
 *           (SURVEY.md reading A11), evaluated by the fully-normalised associated
 *           Legendre three-term recurrence.
 *   dense:  f = Phi c with Phi stored (meshes; §6.2).
 *
 * O2 — independent CPU butterfly apply / adjoint, following the row-wise
 *   butterfly recursion of §2 step by step:
 *     level 0:   z_0(nu)      = X_nu c(nu)
 *     level l:   z_l(tau,nu)  = X_{tau nu} [z_{l-1}(p,c1); z_{l-1}(p,c2)]
 *                (tau at depth l with parent p, nu at height l with children
 *                 c1, c2, reading A2)
 *     leaves:    f(tau)       = U_tau z_L(tau)
 *   and the adjoint as the exact reverse with conjugate transposes (A1).
 *   X is IDENTITY, ID  (out = in[skel] + T in[red], T = R11^{-1} R12 of a
 *   column ID) or DENSE.  Multi-RHS = the same per column.
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py
 * (FFT on a uniform grid, addition theorem, Gauss–Legendre orthonormality,
 * scipy sph_harm_y, brute force at n = m = 64, full-rank plan == dense,
 * adjoint identity).  See DESIGN.md §3.
 */
#define _GNU_SOURCE
#include <errno.h>
#include <fcntl.h>
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

/* ------------------------------------------------------------------------ */
/* O1: flat periodic square                                                  */
/* ------------------------------------------------------------------------ */

/* f[r*n + j] = sum_k c[r*m + k] exp(i k.x_j); x (n,2), k (m,2), complex
 * interleaved (re, im), column-major (each RHS contiguous). */
int orc_flat_synth(int64_t n, int64_t m, const double *x, const int64_t *k,
                   const double *c, int64_t nrhs, double *f) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t r = 0; r < nrhs; ++r) {
      double sr = 0.0, si = 0.0;
      const double *cr = c + 2 * r * m;
      for (int64_t q = 0; q < m; ++q) {
        double ph = (double)k[2 * q] * x[2 * j] + (double)k[2 * q + 1] * x[2 * j + 1];
        double cs = cos(ph), sn = sin(ph);
        double a = cr[2 * q], b = cr[2 * q + 1];
        sr += a * cs - b * sn;
        si += a * sn + b * cs;
      }
      f[2 * (r * n + j)] = sr;
      f[2 * (r * n + j) + 1] = si;
    }
  }
  return 0;
}

/* c[r*m + q] = sum_j exp(-i k_q.x_j) f[r*n + j] */
int orc_flat_analysis(int64_t n, int64_t m, const double *x, const int64_t *k,
                      const double *f, int64_t nrhs, double *c) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < m; ++q) {
    for (int64_t r = 0; r < nrhs; ++r) {
      double sr = 0.0, si = 0.0;
      const double *fr = f + 2 * r * n;
      for (int64_t j = 0; j < n; ++j) {
        double ph = (double)k[2 * q] * x[2 * j] + (double)k[2 * q + 1] * x[2 * j + 1];
        double cs = cos(ph), sn = -sin(ph);
        double a = fr[2 * j], b = fr[2 * j + 1];
        sr += a * cs - b * sn;
        si += a * sn + b * cs;
      }
      c[2 * (r * m + q)] = sr;
      c[2 * (r * m + q) + 1] = si;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O1: sphere — real orthonormal spherical harmonics                         */
/* ------------------------------------------------------------------------ */

/* Fully normalised associated Legendre functions without the Condon–Shortley
 * phase: p[l(l+1)/2 + m] = N_lm P_l^m(cos theta), N_lm^2 = (2l+1)/(4 pi) (l-m)!/(l+m)!,
 * for 0 <= m <= l <= lmax.  Standard recurrences:
 *   p_00 = 1/sqrt(4 pi)
 *   p_mm = sqrt((2m+1)/(2m)) sin(theta) p_{m-1,m-1}
 *   p_{m+1,m} = sqrt(2m+3) cos(theta) p_mm
 *   p_lm = a_lm (cos(theta) p_{l-1,m} - b_lm p_{l-2,m}),
 *     a_lm = sqrt((4l^2-1)/(l^2-m^2)), b_lm = sqrt(((l-1)^2-m^2)/(4(l-1)^2-1)). */
static void orc_legendre(int lmax, double theta, double *p) {
  const double x = cos(theta), s = sin(theta);
  p[0] = 1.0 / sqrt(4.0 * M_PI);
  for (int mm = 1; mm <= lmax; ++mm) {
    int i = mm * (mm + 1) / 2 + mm, im = (mm - 1) * mm / 2 + (mm - 1);
    p[i] = sqrt((2.0 * mm + 1.0) / (2.0 * mm)) * s * p[im];
  }
  for (int mm = 0; mm < lmax; ++mm) {
    int l = mm + 1;
    p[l * (l + 1) / 2 + mm] = sqrt(2.0 * mm + 3.0) * x * p[mm * (mm + 1) / 2 + mm];
  }
  for (int mm = 0; mm <= lmax; ++mm) {
    for (int l = mm + 2; l <= lmax; ++l) {
      double a = sqrt((4.0 * l * l - 1.0) / ((double)l * l - (double)mm * mm));
      double b = sqrt((((double)l - 1) * (l - 1) - (double)mm * mm) / (4.0 * (l - 1) * (l - 1) - 1.0));
      p[l * (l + 1) / 2 + mm] =
          a * (x * p[(l - 1) * l / 2 + mm] - b * p[(l - 2) * (l - 1) / 2 + mm]);
    }
  }
}

/* All real harmonics at one point, index l^2 + l + m (m = -l..l):
 *   Y_l0 = p_l0;  Y_lm = sqrt2 p_lm cos(m phi);  Y_l,-m = sqrt2 p_lm sin(m phi). */
static void orc_ylm_all(int lmax, double theta, double phi, double *p, double *y) {
  orc_legendre(lmax, theta, p);
  for (int l = 0; l <= lmax; ++l) {
    y[l * l + l] = p[l * (l + 1) / 2];
    for (int mm = 1; mm <= l; ++mm) {
      double v = sqrt(2.0) * p[l * (l + 1) / 2 + mm];
      y[l * l + l + mm] = v * cos(mm * phi);
      y[l * l + l - mm] = v * sin(mm * phi);
    }
  }
}

/* Evaluate Y (n x M, row-major) at points — used by tests to build Phi. */
int orc_sphere_matrix(int64_t n, const double *theta, const double *phi, int lmax, double *Y) {
  int64_t M = (int64_t)(lmax + 1) * (lmax + 1);
#pragma omp parallel
  {
    double *p = malloc(sizeof(double) * (size_t)((lmax + 1) * (lmax + 2) / 2));
#pragma omp for schedule(static)
    for (int64_t j = 0; j < n; ++j) orc_ylm_all(lmax, theta[j], phi[j], p, Y + j * M);
    free(p);
  }
  return 0;
}

/* f[r*n + j] = sum_q c[r*M + q] Y_q(x_j), M = (lmax+1)^2, real. */
int orc_sphere_synth(int64_t n, const double *theta, const double *phi, int lmax,
                     const double *c, int64_t nrhs, double *f) {
  int64_t M = (int64_t)(lmax + 1) * (lmax + 1);
#pragma omp parallel
  {
    double *p = malloc(sizeof(double) * (size_t)((lmax + 1) * (lmax + 2) / 2));
    double *y = malloc(sizeof(double) * (size_t)M);
#pragma omp for schedule(dynamic, 8)
    for (int64_t j = 0; j < n; ++j) {
      orc_ylm_all(lmax, theta[j], phi[j], p, y);
      for (int64_t r = 0; r < nrhs; ++r) {
        double s = 0.0;
        for (int64_t q = 0; q < M; ++q) s += c[r * M + q] * y[q];
        f[r * n + j] = s;
      }
    }
    free(p);
    free(y);
  }
  return 0;
}

/* c[r*M + q] = sum_j Y_q(x_j) f[r*n + j]. */
int orc_sphere_analysis(int64_t n, const double *theta, const double *phi, int lmax,
                        const double *f, int64_t nrhs, double *c) {
  int64_t M = (int64_t)(lmax + 1) * (lmax + 1);
  memset(c, 0, sizeof(double) * (size_t)(M * nrhs));
#pragma omp parallel
  {
    double *p = malloc(sizeof(double) * (size_t)((lmax + 1) * (lmax + 2) / 2));
    double *y = malloc(sizeof(double) * (size_t)M);
    double *acc = calloc((size_t)(M * nrhs), sizeof(double));
#pragma omp for schedule(dynamic, 8)
    for (int64_t j = 0; j < n; ++j) {
      orc_ylm_all(lmax, theta[j], phi[j], p, y);
      for (int64_t r = 0; r < nrhs; ++r) {
        double fj = f[r * n + j];
        for (int64_t q = 0; q < M; ++q) acc[r * M + q] += y[q] * fj;
      }
    }
#pragma omp critical
    for (int64_t i = 0; i < M * nrhs; ++i) c[i] += acc[i];
    free(p);
    free(y);
    free(acc);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O1: stored Phi (meshes).  Phi column-major n x m (column k = phi_k).      */
/* is_complex: interleaved complex128 for Phi, c, f.                         */
/* ------------------------------------------------------------------------ */
int orc_dense_synth(int64_t n, int64_t m, const double *Phi, int is_complex,
                    const double *c, int64_t nrhs, double *f) {
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t j = 0; j < n; ++j) {
    for (int64_t r = 0; r < nrhs; ++r) {
      if (!is_complex) {
        double s = 0.0;
        for (int64_t q = 0; q < m; ++q) s += Phi[q * n + j] * c[r * m + q];
        f[r * n + j] = s;
      } else {
        double sr = 0.0, si = 0.0;
        for (int64_t q = 0; q < m; ++q) {
          double a = Phi[2 * (q * n + j)], b = Phi[2 * (q * n + j) + 1];
          double u = c[2 * (r * m + q)], v = c[2 * (r * m + q) + 1];
          sr += a * u - b * v;
          si += a * v + b * u;
        }
        f[2 * (r * n + j)] = sr;
        f[2 * (r * n + j) + 1] = si;
      }
    }
  }
  return 0;
}

int orc_dense_analysis(int64_t n, int64_t m, const double *Phi, int is_complex,
                       const double *f, int64_t nrhs, double *c) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t q = 0; q < m; ++q) {
    for (int64_t r = 0; r < nrhs; ++r) {
      if (!is_complex) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += Phi[q * n + j] * f[r * n + j];
        c[r * m + q] = s;
      } else {
        double sr = 0.0, si = 0.0;
        for (int64_t j = 0; j < n; ++j) {
          double a = Phi[2 * (q * n + j)], b = -Phi[2 * (q * n + j) + 1];
          double u = f[2 * (r * n + j)], v = f[2 * (r * n + j) + 1];
          sr += a * u - b * v;
          si += a * v + b * u;
        }
        c[2 * (r * m + q)] = sr;
        c[2 * (r * m + q) + 1] = si;
      }
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* O2: independent CPU butterfly apply from a plan file                      */
/* ------------------------------------------------------------------------ */
/* Plan file v1, little-endian:
 *   header (256 B): "BFMHTPLN", u32 version=1, u32 dtype (1 f64 | 2 c128),
 *     i64 n, i64 m, i32 L, i32 0, f64 tol, i64 n_stages (= L+2),
 *     u64 checksum (wrapping sum of the body's u64 words), i64 body_bytes.
 *   body: i32 perm_x[n] (padded to 8 B); i64 sp_off[2^L+1]; i64 fr_off[2^L+1];
 *     version 2 only: i32 perm_k[m] (padded to 8 B), plan frequency position ->
 *     user coefficient index (reading A18: quadtree-frequency plans keep the
 *     user's c order; c[perm_k[q]] is the plan's column q);
 *     then per stage s = 0..L+1: i64 s, i64 nblk, i64 nidx, i64 ncoef,
 *     scalar coef[ncoef] (8 or 16 B each),
 *     nblk x {i32 kind, i32 r_out, i32 r_in, i32 0, i64 idx_off, i64 coef_off},
 *     i32 idx[nidx] (padded to 8 B). */
enum { ORC_IDENTITY = 0, ORC_ID = 1, ORC_DENSE = 2 };

typedef struct {
  int32_t kind, r_out, r_in, pad;
  int64_t idx_off, coef_off;
} orc_blk;

typedef struct {
  int64_t nblk, nidx, ncoef;
  const orc_blk *blk;
  const int32_t *idx;
  const double *coef; /* interleaved if complex */
} orc_stage;

typedef struct {
  void *map;
  size_t map_bytes;
  int dtype; /* 1 real, 2 complex */
  int64_t n, m;
  int L;
  double tol;
  const int32_t *perm;
  const int64_t *sp_off, *fr_off;
  const int32_t *perm_k; /* NULL: the plan's frequency order is the user's */
  orc_stage *st; /* L + 2 */
} orc_plan;

static char orc_err[512];
const char *orc_last_error(void) { return orc_err; }

void orc_plan_close(orc_plan *p) {
  if (!p) return;
  if (p->map) munmap(p->map, p->map_bytes);
  free(p->st);
  free(p);
}

orc_plan *orc_plan_open(const char *path, int verify_checksum) {
  int fd = open(path, O_RDONLY);
  if (fd < 0) {
    snprintf(orc_err, sizeof orc_err, "open %s: %s", path, strerror(errno));
    return NULL;
  }
  struct stat sb;
  fstat(fd, &sb);
  size_t bytes = (size_t)sb.st_size;
  if (bytes < 256) {
    close(fd);
    snprintf(orc_err, sizeof orc_err, "file too small");
    return NULL;
  }
  void *map = mmap(NULL, bytes, PROT_READ, MAP_SHARED, fd, 0);
  close(fd);
  if (map == MAP_FAILED) {
    snprintf(orc_err, sizeof orc_err, "mmap failed");
    return NULL;
  }
  const char *h = (const char *)map;
  orc_plan *p = calloc(1, sizeof *p);
  p->map = map;
  p->map_bytes = bytes;
  const uint32_t version = *(const uint32_t *)(h + 8);
  if (memcmp(h, "BFMHTPLN", 8) != 0 || (version != 1u && version != 2u)) {
    snprintf(orc_err, sizeof orc_err, "bad magic/version");
    orc_plan_close(p);
    return NULL;
  }
  p->dtype = (int)*(const uint32_t *)(h + 12);
  p->n = *(const int64_t *)(h + 16);
  p->m = *(const int64_t *)(h + 24);
  p->L = *(const int32_t *)(h + 32);
  p->tol = *(const double *)(h + 40);
  int64_t nst = *(const int64_t *)(h + 48);
  uint64_t csum = *(const uint64_t *)(h + 56);
  int64_t body = *(const int64_t *)(h + 64);
  if ((p->dtype != 1 && p->dtype != 2) || nst != p->L + 2 || body < 0 ||
      (size_t)body + 256 != bytes || p->L < 0 || p->L > 30) {
    snprintf(orc_err, sizeof orc_err, "bad header");
    orc_plan_close(p);
    return NULL;
  }
  if (verify_checksum) {
    const uint64_t *w = (const uint64_t *)(h + 256);
    uint64_t s = 0;
    for (int64_t i = 0; i < body / 8; ++i) s += w[i];
    if (s != csum) {
      snprintf(orc_err, sizeof orc_err, "checksum mismatch");
      orc_plan_close(p);
      return NULL;
    }
  }
  const char *q = h + 256;
  int64_t nl = (int64_t)1 << p->L;
  p->perm = (const int32_t *)q;
  q += ((p->n * 4 + 7) / 8) * 8;
  p->sp_off = (const int64_t *)q;
  q += 8 * (nl + 1);
  p->fr_off = (const int64_t *)q;
  q += 8 * (nl + 1);
  p->perm_k = NULL;
  if (version == 2u) {
    p->perm_k = (const int32_t *)q;
    q += ((p->m * 4 + 7) / 8) * 8;
  }
  p->st = calloc((size_t)nst, sizeof(orc_stage));
  size_t sc = p->dtype == 2 ? 16 : 8;
  for (int s = 0; s < nst; ++s) {
    const int64_t *sh = (const int64_t *)q;
    if (sh[0] != s) {
      snprintf(orc_err, sizeof orc_err, "stage %d header mismatch", s);
      orc_plan_close(p);
      return NULL;
    }
    orc_stage *S = &p->st[s];
    S->nblk = sh[1];
    S->nidx = sh[2];
    S->ncoef = sh[3];
    q += 32;
    S->coef = (const double *)q;
    q += sc * S->ncoef;
    S->blk = (const orc_blk *)q;
    q += 32 * S->nblk;
    S->idx = (const int32_t *)q;
    q += ((S->nidx * 4 + 7) / 8) * 8;
    if (S->nblk != nl || q > h + bytes) {
      snprintf(orc_err, sizeof orc_err, "stage %d truncated or wrong block count", s);
      orc_plan_close(p);
      return NULL;
    }
  }
  return p;
}

int64_t orc_plan_n(const orc_plan *p) { return p->n; }
int64_t orc_plan_m(const orc_plan *p) { return p->m; }
int orc_plan_L(const orc_plan *p) { return p->L; }
int orc_plan_dtype(const orc_plan *p) { return p->dtype; }

/* y = X x for one block; x has r_in entries, y has r_out (scalars of size cw
 * doubles, cw = 1 real / 2 complex). */
static void orc_block_apply(const orc_plan *P, const orc_stage *S, const orc_blk *b,
                            const double *x, double *y) {
  const int cw = P->dtype == 2 ? 2 : 1;
  const int ro = b->r_out, ri = b->r_in;
  if (b->kind == ORC_IDENTITY) {
    memcpy(y, x, sizeof(double) * cw * (size_t)ri);
    return;
  }
  const double *T = S->coef + (size_t)cw * (size_t)b->coef_off;
  if (b->kind == ORC_ID) {
    const int32_t *skel = S->idx + b->idx_off, *red = skel + ro;
    const int nr = ri - ro;
    for (int i = 0; i < ro; ++i) {
      double sr = x[cw * skel[i]], si = cw == 2 ? x[2 * skel[i] + 1] : 0.0;
      for (int j = 0; j < nr; ++j) {
        if (cw == 1) {
          sr += T[(size_t)j * ro + i] * x[red[j]];
        } else {
          double a = T[2 * ((size_t)j * ro + i)], bb = T[2 * ((size_t)j * ro + i) + 1];
          double u = x[2 * red[j]], v = x[2 * red[j] + 1];
          sr += a * u - bb * v;
          si += a * v + bb * u;
        }
      }
      y[cw * i] = sr;
      if (cw == 2) y[2 * i + 1] = si;
    }
    return;
  }
  /* DENSE */
  for (int i = 0; i < ro; ++i) {
    double sr = 0.0, si = 0.0;
    for (int j = 0; j < ri; ++j) {
      if (cw == 1) {
        sr += T[(size_t)j * ro + i] * x[j];
      } else {
        double a = T[2 * ((size_t)j * ro + i)], bb = T[2 * ((size_t)j * ro + i) + 1];
        double u = x[2 * j], v = x[2 * j + 1];
        sr += a * u - bb * v;
        si += a * v + bb * u;
      }
    }
    y[cw * i] = sr;
    if (cw == 2) y[2 * i + 1] = si;
  }
}

/* w += X^* z for one block; z has r_out entries, w has r_in. */
static void orc_block_adjoint_add(const orc_plan *P, const orc_stage *S, const orc_blk *b,
                                  const double *z, double *w) {
  const int cw = P->dtype == 2 ? 2 : 1;
  const int ro = b->r_out, ri = b->r_in;
  if (b->kind == ORC_IDENTITY) {
    for (int i = 0; i < cw * ri; ++i) w[i] += z[i];
    return;
  }
  const double *T = S->coef + (size_t)cw * (size_t)b->coef_off;
  if (b->kind == ORC_ID) {
    const int32_t *skel = S->idx + b->idx_off, *red = skel + ro;
    const int nr = ri - ro;
    for (int i = 0; i < ro; ++i) {
      w[cw * skel[i]] += z[cw * i];
      if (cw == 2) w[2 * skel[i] + 1] += z[2 * i + 1];
    }
    for (int j = 0; j < nr; ++j) {
      double sr = 0.0, si = 0.0;
      for (int i = 0; i < ro; ++i) {
        if (cw == 1) {
          sr += T[(size_t)j * ro + i] * z[i];
        } else { /* conj(T) z */
          double a = T[2 * ((size_t)j * ro + i)], bb = -T[2 * ((size_t)j * ro + i) + 1];
          double u = z[2 * i], v = z[2 * i + 1];
          sr += a * u - bb * v;
          si += a * v + bb * u;
        }
      }
      w[cw * red[j]] += sr;
      if (cw == 2) w[2 * red[j] + 1] += si;
    }
    return;
  }
  for (int j = 0; j < ri; ++j) {
    double sr = 0.0, si = 0.0;
    for (int i = 0; i < ro; ++i) {
      if (cw == 1) {
        sr += T[(size_t)j * ro + i] * z[i];
      } else {
        double a = T[2 * ((size_t)j * ro + i)], bb = -T[2 * ((size_t)j * ro + i) + 1];
        double u = z[2 * i], v = z[2 * i + 1];
        sr += a * u - bb * v;
        si += a * v + bb * u;
      }
    }
    w[cw * j] += sr;
    if (cw == 2) w[cw * j + 1] += si;
  }
}

/* Validate the chain invariant r_in(l, (t,v)) = r_out(l-1,(p,2v)) + r_out(l-1,(p,2v+1)). */
int orc_plan_validate(const orc_plan *P) {
  int64_t nl = (int64_t)1 << P->L;
  for (int64_t v = 0; v < nl; ++v)
    if (P->st[0].blk[v].r_in != P->fr_off[v + 1] - P->fr_off[v]) return -1;
  for (int l = 1; l <= P->L; ++l) {
    int64_t nf = nl >> l, nfp = nl >> (l - 1);
    for (int64_t t = 0; t < ((int64_t)1 << l); ++t)
      for (int64_t v = 0; v < nf; ++v) {
        const orc_blk *b = &P->st[l].blk[t * nf + v];
        int64_t p = t >> 1;
        int64_t r = P->st[l - 1].blk[p * nfp + 2 * v].r_out + P->st[l - 1].blk[p * nfp + 2 * v + 1].r_out;
        if (b->r_in != r) return -(100 + l);
      }
  }
  for (int64_t t = 0; t < nl; ++t) {
    const orc_blk *b = &P->st[P->L + 1].blk[t];
    if (b->r_in != P->st[P->L].blk[t].r_out) return -2;
    if (b->r_out != P->sp_off[t + 1] - P->sp_off[t]) return -3;
  }
  return 0;
}

/* f = BF c  (c: m x nrhs column-major; f: n x nrhs).  OpenMP over the blocks
 * of a level (SURVEY.md §8(d) CPU baseline protocol). */
int orc_bf_apply(const orc_plan *P, const double *c, double *f, int64_t nrhs) {
  const int cw = P->dtype == 2 ? 2 : 1;
  const int L = P->L;
  const int64_t nl = (int64_t)1 << L;
  int64_t *zoff_prev = malloc(sizeof(int64_t) * (size_t)(nl + 1));
  int64_t *zoff = malloc(sizeof(int64_t) * (size_t)(nl + 1));
  double *cperm = P->perm_k ? malloc(sizeof(double) * cw * (size_t)P->m) : NULL;
  for (int64_t r = 0; r < nrhs; ++r) {
    const double *cr = c + (size_t)cw * (size_t)(r * P->m);
    double *fr = f + (size_t)cw * (size_t)(r * P->n);
    if (P->perm_k) { /* the plan's column q is the user's coefficient perm_k[q] */
      for (int64_t q = 0; q < P->m; ++q)
        for (int k = 0; k < cw; ++k) cperm[cw * q + k] = cr[cw * (int64_t)P->perm_k[q] + k];
      cr = cperm;
    }
    /* level 0 */
    zoff_prev[0] = 0;
    for (int64_t v = 0; v < nl; ++v) zoff_prev[v + 1] = zoff_prev[v] + P->st[0].blk[v].r_out;
    double *zp = malloc(sizeof(double) * cw * (size_t)(zoff_prev[nl] > 0 ? zoff_prev[nl] : 1));
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t v = 0; v < nl; ++v)
      orc_block_apply(P, &P->st[0], &P->st[0].blk[v], cr + cw * P->fr_off[v], zp + cw * zoff_prev[v]);
    /* levels 1..L */
    for (int l = 1; l <= L; ++l) {
      const int64_t nf = nl >> l, nfp = nl >> (l - 1);
      zoff[0] = 0;
      for (int64_t b = 0; b < nl; ++b) zoff[b + 1] = zoff[b] + P->st[l].blk[b].r_out;
      double *zn = malloc(sizeof(double) * cw * (size_t)(zoff[nl] > 0 ? zoff[nl] : 1));
#pragma omp parallel
      {
        double *in = NULL;
        size_t cap = 0;
#pragma omp for schedule(dynamic, 1)
        for (int64_t b = 0; b < nl; ++b) {
          int64_t t = b / nf, v = b % nf, p = t >> 1;
          int64_t b1 = p * nfp + 2 * v, b2 = b1 + 1;
          int64_t n1 = zoff_prev[b1 + 1] - zoff_prev[b1], n2 = zoff_prev[b2 + 1] - zoff_prev[b2];
          size_t need = (size_t)cw * (size_t)(n1 + n2 + 1);
          if (need > cap) {
            free(in);
            in = malloc(sizeof(double) * need);
            cap = need;
          }
          /* in = [z_{l-1}(p,c1); z_{l-1}(p,c2)] */
          memcpy(in, zp + cw * zoff_prev[b1], sizeof(double) * cw * (size_t)n1);
          memcpy(in + cw * n1, zp + cw * zoff_prev[b2], sizeof(double) * cw * (size_t)n2);
          orc_block_apply(P, &P->st[l], &P->st[l].blk[b], in, zn + cw * zoff[b]);
        }
        free(in);
      }
      free(zp);
      zp = zn;
      int64_t *tmp = zoff_prev;
      zoff_prev = zoff;
      zoff = tmp;
    }
    /* leaf interpolation f(tau) = U_tau z_L(tau), scattered through perm_x */
    const orc_stage *SU = &P->st[L + 1];
#pragma omp parallel
    {
      double *y = NULL;
      size_t cap = 0;
#pragma omp for schedule(dynamic, 1)
      for (int64_t t = 0; t < nl; ++t) {
        int64_t rows = P->sp_off[t + 1] - P->sp_off[t];
        size_t need = (size_t)cw * (size_t)(rows + 1);
        if (need > cap) {
          free(y);
          y = malloc(sizeof(double) * need);
          cap = need;
        }
        orc_block_apply(P, SU, &SU->blk[t], zp + cw * zoff_prev[t], y);
        for (int64_t i = 0; i < rows; ++i) {
          int64_t j = P->perm[P->sp_off[t] + i];
          fr[cw * j] = y[cw * i];
          if (cw == 2) fr[cw * j + 1] = y[cw * i + 1];
        }
      }
      free(y);
    }
    free(zp);
  }
  free(cperm);
  free(zoff_prev);
  free(zoff);
  return 0;
}

/* c = BF^* f, the exact reverse with conjugate transposes. */
int orc_bf_adjoint(const orc_plan *P, const double *f, double *c, int64_t nrhs) {
  const int cw = P->dtype == 2 ? 2 : 1;
  const int L = P->L;
  const int64_t nl = (int64_t)1 << L;
  int64_t *zoff = malloc(sizeof(int64_t) * (size_t)(nl + 1));
  int64_t *zoff_lo = malloc(sizeof(int64_t) * (size_t)(nl + 1));
  double *cperm = P->perm_k ? malloc(sizeof(double) * cw * (size_t)P->m) : NULL;
  for (int64_t r = 0; r < nrhs; ++r) {
    const double *fr = f + (size_t)cw * (size_t)(r * P->n);
    double *cuser = c + (size_t)cw * (size_t)(r * P->m);
    double *cr = P->perm_k ? cperm : cuser; /* the plan's frequency order; scattered below */
    /* z_L(tau) = U_tau^* f(tau) */
    const orc_stage *SU = &P->st[L + 1];
    zoff[0] = 0;
    for (int64_t t = 0; t < nl; ++t) zoff[t + 1] = zoff[t] + SU->blk[t].r_in;
    double *z = calloc((size_t)cw * (size_t)(zoff[nl] + 1), sizeof(double));
#pragma omp parallel
    {
      double *x = NULL;
      size_t cap = 0;
#pragma omp for schedule(dynamic, 1)
      for (int64_t t = 0; t < nl; ++t) {
        int64_t rows = P->sp_off[t + 1] - P->sp_off[t];
        size_t need = (size_t)cw * (size_t)(rows + 1);
        if (need > cap) {
          free(x);
          x = malloc(sizeof(double) * need);
          cap = need;
        }
        for (int64_t i = 0; i < rows; ++i) {
          int64_t j = P->perm[P->sp_off[t] + i];
          x[cw * i] = fr[cw * j];
          if (cw == 2) x[cw * i + 1] = fr[cw * j + 1];
        }
        orc_block_adjoint_add(P, SU, &SU->blk[t], x, z + cw * zoff[t]);
      }
      free(x);
    }
    /* levels L..1: [z(p,c1); z(p,c2)] = X_{tau1 nu}^* z(tau1,nu) + X_{tau2 nu}^* z(tau2,nu) */
    for (int l = L; l >= 1; --l) {
      const int64_t nf = nl >> l, nfp = nl >> (l - 1);
      const orc_stage *Sl = &P->st[l];
      zoff_lo[0] = 0;
      for (int64_t b = 0; b < nl; ++b) zoff_lo[b + 1] = zoff_lo[b] + P->st[l - 1].blk[b].r_out;
      double *zl = calloc((size_t)cw * (size_t)(zoff_lo[nl] + 1), sizeof(double));
      /* group (p, v): children tau = 2p, 2p+1 of p; writes z_{l-1}(p, 2v), z_{l-1}(p, 2v+1) */
#pragma omp parallel for schedule(dynamic, 1)
      for (int64_t g = 0; g < nl / 2; ++g) {
        int64_t p = g / nf, v = g % nf;
        int64_t b1 = p * nfp + 2 * v; /* z_{l-1}(p, 2v); (p, 2v+1) follows contiguously */
        for (int64_t ch = 0; ch < 2; ++ch) {
          int64_t t = 2 * p + ch, b = t * nf + v;
          orc_block_adjoint_add(P, Sl, &Sl->blk[b], z + cw * zoff[b], zl + cw * zoff_lo[b1]);
        }
      }
      free(z);
      z = zl;
      int64_t *tmp = zoff;
      zoff = zoff_lo;
      zoff_lo = tmp;
    }
    /* c(nu) = X_nu^* z_0(nu) */
    for (int64_t i = 0; i < cw * P->m; ++i) cr[i] = 0.0;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t v = 0; v < nl; ++v)
      orc_block_adjoint_add(P, &P->st[0], &P->st[0].blk[v], z + cw * zoff[v], cr + cw * P->fr_off[v]);
    free(z);
    if (P->perm_k) /* the plan's column q is the user's coefficient perm_k[q] */
      for (int64_t q = 0; q < P->m; ++q)
        for (int k = 0; k < cw; ++k) cuser[cw * (int64_t)P->perm_k[q] + k] = cperm[cw * q + k];
  }
  free(cperm);
  free(zoff);
  free(zoff_lo);
  return 0;
}

/* Count stored non-identity coefficient entries (E in SURVEY.md §8(d)). */
int64_t orc_plan_entries(const orc_plan *P) {
  int64_t e = 0;
  for (int s = 0; s < P->L + 2; ++s) e += P->st[s].ncoef;
  return e;
}

int orc_num_threads(void) { return omp_get_max_threads(); }
void orc_set_threads(int t) { omp_set_num_threads(t); }
