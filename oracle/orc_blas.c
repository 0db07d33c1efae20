/*
 * orc_blas.c — cache-blocked, vectorised restatements of the reference's three
 * dense contractions (TEST INFRASTRUCTURE, part of the oracle; see pcal_oracle.h).
 *
 *   matmul      (kernels.cpp:105-122)  c(i,j) = Σ_k b(k,j)·a(i,k), k ascending
 *   matmul_at_b (kernels.cpp:124-137)  c(i,j) = Σ_r a(r,i)·b(r,j), r ascending
 *   gram        (kernels.cpp:139-153)  upper triangle of matmul_at_b(x, x), mirrored
 *
 * Every output element is still ONE sequential sum in the reference's order,
 * started from 0.0, one IEEE multiply then one IEEE add per term (the file is
 * compiled with -ffp-contract=off, no FMA).  Blocking only changes WHICH
 * elements are in flight together and where a partial sum waits between
 * blocks (a register or memory round trip is exact), so the results are bit
 * for bit the reference's — tests/test_oracle_golden.py pins that against
 * outputs of the unmodified reference.  What changes is speed: the reference's
 * loops are a latency-bound dot per element (matmul_at_b, gram) and one pass
 * over the whole operand per output column (matmul); here many independent
 * sums advance per instruction and each operand block is reused from cache,
 * so the long parity windows (config 2's 500 iterations and its ulp
 * ensemble, configs 3–5's shapes) run in minutes instead of hours.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef double v8 __attribute__((vector_size(64), aligned(8)));

#if defined(__x86_64__) && !defined(ORC_NO_CLONES)
#define ORC_CLONES __attribute__((target_clones("avx512f", "avx2", "default")))
#else
#define ORC_CLONES
#endif

static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* ---------------------------------------------------------------- matmul */
enum { MM_MR = 16, MM_NR = 8, MM_KB = 128, MM_MB = 256 };

/* One MM_MR x MM_NR tile of c over kb terms.  a: rows i.. of column k0 (lda),
 * bp: packed b rows k0.. of one 8-column group ([k][8]), c: tile origin (ldc).
 * rows < MM_MR / cols < MM_NR are tails (zero-padded b columns are computed
 * and discarded). */
ORC_CLONES
static void mm_tile(const double* a, int64_t lda, const double* bp, int64_t kb, double* c,
                    int64_t ldc, int rows, int cols) {
  if (rows == MM_MR) {
    v8 acc0[MM_NR], acc1[MM_NR];
    for (int jj = 0; jj < MM_NR; ++jj) {
      if (jj < cols) {
        acc0[jj] = *(const v8*)(c + jj * ldc);
        acc1[jj] = *(const v8*)(c + jj * ldc + 8);
      } else {
        acc0[jj] = (v8){0};
        acc1[jj] = (v8){0};
      }
    }
    for (int64_t k = 0; k < kb; ++k) {
      const v8 a0 = *(const v8*)(a + k * lda);
      const v8 a1 = *(const v8*)(a + k * lda + 8);
      const double* bk = bp + k * MM_NR;
#pragma GCC unroll 8
      for (int jj = 0; jj < MM_NR; ++jj) {
        const double s = bk[jj];
        acc0[jj] += s * a0;
        acc1[jj] += s * a1;
      }
    }
    for (int jj = 0; jj < cols; ++jj) {
      *(v8*)(c + jj * ldc) = acc0[jj];
      *(v8*)(c + jj * ldc + 8) = acc1[jj];
    }
    return;
  }
  for (int jj = 0; jj < cols; ++jj)
    for (int ii = 0; ii < rows; ++ii) {
      double s = c[ii + jj * ldc];
      for (int64_t k = 0; k < kb; ++k) s += bp[k * MM_NR + jj] * a[ii + k * lda];
      c[ii + jj * ldc] = s;
    }
}

void orc_blas_matmul(const double* a, int64_t m, int64_t kdim, const double* b, int64_t ncols,
                     double* c, int threads) {
  memset(c, 0, sizeof(double) * (size_t)(m * ncols));
  if (m == 0 || ncols == 0 || kdim == 0) return;
  const int64_t njg = (ncols + MM_NR - 1) / MM_NR;
  /* b packed per 8-column group: bp[(g*kdim + k)*8 + jj] = b(k, 8g+jj) or 0 */
  double* bp = (double*)malloc(sizeof(double) * (size_t)(njg * kdim * MM_NR));
  for (int64_t g = 0; g < njg; ++g)
    for (int64_t k = 0; k < kdim; ++k)
      for (int jj = 0; jj < MM_NR; ++jj) {
        const int64_t j = g * MM_NR + jj;
        bp[(g * kdim + k) * MM_NR + jj] = j < ncols ? b[k + j * kdim] : 0.0;
      }
  const int64_t nmt = (m + MM_MB - 1) / MM_MB;
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(dynamic, 1)
  for (int64_t t = 0; t < nmt; ++t) {
    const int64_t i0 = t * MM_MB, i1 = min64(m, i0 + MM_MB);
    for (int64_t k0 = 0; k0 < kdim; k0 += MM_KB) {  /* k blocks in ascending order */
      const int64_t kb = min64(MM_KB, kdim - k0);
      for (int64_t g = 0; g < njg; ++g) {
        const int cols = (int)min64(MM_NR, ncols - g * MM_NR);
        for (int64_t i = i0; i < i1; i += MM_MR)
          mm_tile(a + i + k0 * m, m, bp + (g * kdim + k0) * MM_NR, kb, c + i + g * MM_NR * m, m,
                  (int)min64(MM_MR, i1 - i), cols);
      }
    }
  }
  free(bp);
}

/* ---------------------------------------------------- matmul_at_b / gram */
enum { AT_IR = 6, AT_JR = 16, AT_RB = 256, AT_IRANGE = 24, AT_JRANGE = 64 };

/* AT_IR x AT_JR accumulators over rb terms: acc(ii, jj) += a_ii[r]·bp[r][jj].
 * cl: accumulator tile, row-major with leading dimension ldl. */
ORC_CLONES
static void atb_tile(const double* const* acols, const double* bp, int64_t rb, double* cl,
                     int64_t ldl) {
  v8 acc[AT_IR][2];
  for (int ii = 0; ii < AT_IR; ++ii) {
    acc[ii][0] = *(const v8*)(cl + ii * ldl);
    acc[ii][1] = *(const v8*)(cl + ii * ldl + 8);
  }
  const double* a0 = acols[0];
  const double* a1 = acols[1];
  const double* a2 = acols[2];
  const double* a3 = acols[3];
  const double* a4 = acols[4];
  const double* a5 = acols[5];
  for (int64_t r = 0; r < rb; ++r) {
    const v8 b0 = *(const v8*)(bp + r * AT_JR);
    const v8 b1 = *(const v8*)(bp + r * AT_JR + 8);
    double s;
    s = a0[r]; acc[0][0] += s * b0; acc[0][1] += s * b1;
    s = a1[r]; acc[1][0] += s * b0; acc[1][1] += s * b1;
    s = a2[r]; acc[2][0] += s * b0; acc[2][1] += s * b1;
    s = a3[r]; acc[3][0] += s * b0; acc[3][1] += s * b1;
    s = a4[r]; acc[4][0] += s * b0; acc[4][1] += s * b1;
    s = a5[r]; acc[5][0] += s * b0; acc[5][1] += s * b1;
  }
  for (int ii = 0; ii < AT_IR; ++ii) {
    *(v8*)(cl + ii * ldl) = acc[ii][0];
    *(v8*)(cl + ii * ldl + 8) = acc[ii][1];
  }
}

/* c(i,j) = Σ_r a(r,i)·b(r,j) for i < m, j < ncols (a: n×m, b: n×ncols, both
 * column-major with leading dimension n).  upper != 0: only i ≤ j is needed;
 * those entries are written to c(i,j) and mirrored to c(j,i) (gram). */
static void atb_driver(const double* a, int64_t n, int64_t m, const double* b, int64_t ncols,
                       double* c, int threads, int upper) {
  if (m == 0 || ncols == 0) return;
  const int64_t nib = (m + AT_IRANGE - 1) / AT_IRANGE;
  const int64_t njb = (ncols + AT_JRANGE - 1) / AT_JRANGE;
  double* zeros = (double*)calloc((size_t)AT_RB, sizeof(double));
#pragma omp parallel num_threads(threads > 0 ? threads : 1)
  {
    double* bp = (double*)malloc(sizeof(double) * (size_t)(AT_RB * AT_JRANGE));
    double* cl = (double*)malloc(sizeof(double) * (size_t)(AT_IRANGE * AT_JRANGE));
#pragma omp for schedule(dynamic, 1) collapse(2)
    for (int64_t jb = 0; jb < njb; ++jb)
      for (int64_t ib = 0; ib < nib; ++ib) {
        const int64_t i0 = ib * AT_IRANGE, j0 = jb * AT_JRANGE;
        const int64_t jn = min64(AT_JRANGE, ncols - j0);
        const int64_t in = min64(AT_IRANGE, m - i0);
        if (upper && i0 > j0 + jn - 1) continue; /* entirely below the diagonal */
        memset(cl, 0, sizeof(double) * (size_t)(AT_IRANGE * AT_JRANGE));
        for (int64_t r0 = 0; r0 < n; r0 += AT_RB) { /* r blocks in ascending order */
          const int64_t rb = min64(AT_RB, n - r0);
          for (int64_t js = 0; js < AT_JRANGE / AT_JR; ++js)
            for (int64_t r = 0; r < rb; ++r)
              for (int jj = 0; jj < AT_JR; ++jj) {
                const int64_t j = j0 + js * AT_JR + jj;
                bp[(js * rb + r) * AT_JR + jj] = j < ncols ? b[r0 + r + j * n] : 0.0;
              }
          for (int64_t js = 0; js < AT_JRANGE / AT_JR; ++js) {
            if (js * AT_JR >= jn) break;
            for (int64_t is = 0; is < AT_IRANGE / AT_IR; ++is) {
              const int64_t ia = i0 + is * AT_IR;
              if (is * AT_IR >= in) break;
              if (upper && ia > j0 + js * AT_JR + AT_JR - 1) continue;
              const double* cols[AT_IR];
              for (int ii = 0; ii < AT_IR; ++ii)
                cols[ii] = (ia + ii < m) ? a + r0 + (ia + ii) * n : zeros;
              atb_tile(cols, bp + js * rb * AT_JR, rb, cl + is * AT_IR * AT_JRANGE + js * AT_JR,
                       AT_JRANGE);
            }
          }
        }
        for (int64_t ii = 0; ii < in; ++ii)
          for (int64_t jj = 0; jj < jn; ++jj) {
            const int64_t i = i0 + ii, j = j0 + jj;
            const double v = cl[ii * AT_JRANGE + jj];
            if (!upper) {
              c[i + j * m] = v;
            } else if (i <= j) {
              c[i + j * m] = v;
              c[j + i * m] = v;
            }
          }
      }
    free(bp);
    free(cl);
  }
  free(zeros);
}

void orc_blas_at_b(const double* a, int64_t n, int64_t m, const double* b, int64_t ncols,
                   double* c, int threads) {
  atb_driver(a, n, m, b, ncols, c, threads, 0);
}

void orc_blas_gram(const double* x, int64_t n, int64_t p, double* g, int threads) {
  atb_driver(x, n, p, x, p, g, threads, 1);
}
