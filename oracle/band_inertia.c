/* Sylvester inertia count for a real symmetric band pencil — TEST INFRASTRUCTURE ONLY.
 *
 * count(sigma) = number of eigenvalues of A x = lambda B x below sigma, from the
 * signs of D in the unpivoted band LDL^T of (A - sigma B).  This is the
 * independent eigenvalue-count oracle SURVEY.md §8(c) asks for on config 4
 * (N = 1e6, kd = 16), where a dense eigensolver is out of reach.
 *
 * Storage: 'L' band layout as LAPACK dsbev uses and feastlib's feast_sb accepts
 * (banded.py:21-47, uplo='L'): ab[d*n + j] = A[j+d, j], d = 0..kd.
 */
#include <stdlib.h>
#include <string.h>

/* Returns the number of negative pivots, or -1 on allocation failure. */
long band_inertia_count(const double *ab, int kda, const double *bb, int kdb,
                        long n, double sigma) {
  int kd = kda > kdb ? kda : kdb;
  /* w holds the active (kd+1) x (kd+1) lower window, row-major by lag:
   * col[c][d] = M[j+c+d, j+c] for the next kd+1 columns, rolling. */
  int w = kd + 1;
  double *col = (double *)malloc(sizeof(double) * (size_t)w * w);
  if (!col) return -1;
  long neg = 0;
  /* load column j of (A - sigma B) lower part into slot c */
#define LOADCOL(slot, jj)                                               \
  do {                                                                  \
    double *cc = col + (size_t)(slot) * w;                              \
    for (int d = 0; d < w; ++d) {                                       \
      long r = (jj) + d;                                                \
      double v = 0.0;                                                   \
      if (r < n) {                                                      \
        if (d <= kda) v += ab[(size_t)d * n + (jj)];                    \
        if (bb && d <= kdb) v -= sigma * bb[(size_t)d * n + (jj)];      \
        else if (!bb && d == 0) v -= sigma;                             \
      }                                                                 \
      cc[d] = v;                                                        \
    }                                                                   \
  } while (0)
  for (int c = 0; c < w && c < n; ++c) LOADCOL(c, (long)c);
  int head = 0; /* slot holding column j */
  for (long j = 0; j < n; ++j) {
    double *cj = col + (size_t)head * w;
    double dj = cj[0];
    if (dj < 0) ++neg;
    if (dj == 0.0) dj = 1e-300;
    /* l[d] = M[j+d, j] / dj; update columns j+c (c=1..kd): M[j+c+e, j+c] -= l[c+e] * dj * l[c] */
    for (int c = 1; c < w && j + c < n; ++c) {
      double *cc = col + (size_t)((head + c) % w) * w;
      double lc = cj[c];
      if (lc == 0.0) continue;
      double f = lc / dj;
      for (int e = 0; c + e < w; ++e) cc[e] -= f * cj[c + e];
    }
    /* slot head is free: load column j+w */
    if (j + w < n) LOADCOL(head, j + w);
    head = (head + 1) % w;
  }
#undef LOADCOL
  free(col);
  return neg;
}
