/*
 * pcal_oracle.c — CPU restatement of the reference PCAL path.
 *
 * TEST INFRASTRUCTURE ONLY (see pcal_oracle.h).  Compile with
 * -O2 -ffp-contract=off: the reference is built that way
 * (/root/reference/proj/CMakeLists.txt:12-14) and every loop below keeps the
 * reference's accumulation order, so dense-model runs are bitwise identical
 * to the reference (tests/golden pins this).
 */
#include "pcal_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------ */
/* RNG — rng.hpp:13-55 (xoshiro256++ / splitmix64), kernels.cpp:65-78 (normal) */

static uint64_t splitmix64(uint64_t* x) {
  *x += 0x9e3779b97f4a7c15ULL;
  uint64_t z = *x;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

void orc_rng_init(orc_rng* r, uint64_t seed) {
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&s);
  r->spare = 0.0;
  r->has_spare = 0;
}

uint64_t orc_rng_next(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t result = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return result;
}

double orc_rng_uniform(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* Box–Muller pair from two uniform draws, u1 in (0,1], u2 in [0,1). */
static void box_muller(orc_rng* r, double* c, double* s) {
  const double u1 = 1.0 - orc_rng_uniform(r);
  const double u2 = orc_rng_uniform(r);
  const double rr = sqrt(-2.0 * log(u1));
  const double t = 6.283185307179586476925286766559 * u2;
  *s = rr * sin(t);
  *c = rr * cos(t);
}

double orc_rng_normal(orc_rng* r) {
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  double c, s;
  box_muller(r, &c, &s);
  r->spare = s;
  r->has_spare = 1;
  return c;
}

/* random_normal (kernels.cpp:49-55).  Pair m produces values 2m (cos) and
 * 2m+1 (sin, the cached spare); chunks of pairs restart from checkpointed
 * generator states so threads reproduce the sequential fill bit for bit. */
void orc_random_normal(int64_t count, uint64_t seed, double* out, int threads) {
  orc_rng r;
  orc_rng_init(&r, seed);
  const int64_t npairs = (count + 1) / 2;
  if (threads <= 1 || npairs < (1 << 16)) {
    for (int64_t k = 0; k < count; ++k) out[k] = orc_rng_normal(&r);
    return;
  }
  const int64_t chunk = 1 << 16; /* pairs per checkpoint */
  const int64_t nchunks = (npairs + chunk - 1) / chunk;
  orc_rng* cps = (orc_rng*)malloc(sizeof(orc_rng) * (size_t)nchunks);
  for (int64_t c = 0; c < nchunks; ++c) {
    cps[c] = r;
    const int64_t pairs = (c + 1 < nchunks) ? chunk : npairs - c * chunk;
    for (int64_t q = 0; q < 2 * pairs; ++q) (void)orc_rng_next(&r);
  }
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4)
  for (int64_t c = 0; c < nchunks; ++c) {
    orc_rng g = cps[c];
    const int64_t p0 = c * chunk;
    const int64_t p1 = (c + 1 < nchunks) ? p0 + chunk : npairs;
    for (int64_t m = p0; m < p1; ++m) {
      double cv, sv;
      box_muller(&g, &cv, &sv);
      out[2 * m] = cv;
      if (2 * m + 1 < count) out[2 * m + 1] = sv;
    }
  }
  free(cps);
}

void orc_random_uniform(int64_t count, uint64_t seed, double* out) {
  orc_rng r;
  orc_rng_init(&r, seed);
  for (int64_t k = 0; k < count; ++k) out[k] = orc_rng_uniform(&r);
}

/* ------------------------------------------------------------------------ */
/* Dense kernels — kernels.cpp                                                */

double orc_dot(const double* a, const double* b, int64_t n) { /* kernels.cpp:20-24 */
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

double orc_frobenius_norm(const double* a, int64_t count) { /* kernels.cpp:305-313 */
  return sqrt(orc_dot(a, a, count));
}

void orc_sym_part(const double* m, int64_t n, double* out) { /* kernels.cpp:28-36 */
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i <= j; ++i) {
      const double v = 0.5 * (m[i + j * n] + m[j + i * n]);
      out[i + j * n] = v;
      out[j + i * n] = v;
    }
}

/* matmul (kernels.cpp:105-122), matmul_at_b (:124-137), gram (:139-153):
 * the blocked restatements in orc_blas.c (same per-element operation order,
 * bitwise equal to the reference). */
void orc_matmul(const double* a, int64_t m, int64_t kdim, const double* b, int64_t ncols,
                double* c, int threads) {
  orc_blas_matmul(a, m, kdim, b, ncols, c, threads);
}

void orc_matmul_at_b(const double* a, int64_t n, int64_t m, const double* b, int64_t ncols,
                     double* c, int threads) {
  orc_blas_at_b(a, n, m, b, ncols, c, threads);
}

void orc_gram(const double* x, int64_t n, int64_t p, double* g, int threads) {
  orc_blas_gram(x, n, p, g, threads);
}

/* cholesky_lower (kernels.cpp:159-175). */
static int cholesky_lower(const double* a, int64_t p, double floor_, double* l) {
  memset(l, 0, sizeof(double) * (size_t)(p * p));
  for (int64_t j = 0; j < p; ++j) {
    double d = a[j + j * p];
    for (int64_t k = 0; k < j; ++k) d -= l[j + k * p] * l[j + k * p];
    if (!(d > floor_)) return 0;
    const double ljj = sqrt(d);
    l[j + j * p] = ljj;
    for (int64_t i = j + 1; i < p; ++i) {
      double s = a[i + j * p];
      for (int64_t k = 0; k < j; ++k) s -= l[i + k * p] * l[j + k * p];
      l[i + j * p] = s / ljj;
    }
  }
  return 1;
}

/* solve_right_lt (kernels.cpp:178-195): Q·Lᵀ = X, column by column.  Each
 * element q(i,j) = (x(i,j) − Σ_{k<j} l(j,k)·q(i,k), k ascending)·(1/l(j,j)) only
 * depends on its own row, so row blocks run in parallel, bitwise neutral. */
static void solve_right_lt(const double* x, int64_t n, int64_t p, const double* l, double* q,
                           int threads) {
  const int64_t rb = 512, nrb = (n + rb - 1) / rb;
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) schedule(dynamic, 1)
  for (int64_t b = 0; b < nrb; ++b) {
    const int64_t i0 = b * rb, i1 = (i0 + rb < n) ? i0 + rb : n;
    for (int64_t j = 0; j < p; ++j) {
      double* qj = q + j * n;
      memcpy(qj + i0, x + j * n + i0, sizeof(double) * (size_t)(i1 - i0));
      for (int64_t k = 0; k < j; ++k) {
        const double s = l[j + k * p];
        const double* qk = q + k * n;
        for (int64_t i = i0; i < i1; ++i) qj[i] -= s * qk[i];
      }
      const double inv = 1.0 / l[j + j * p];
      for (int64_t i = i0; i < i1; ++i) qj[i] *= inv;
    }
  }
}

/* mgs2 (kernels.cpp:212-246); only Q is needed by the solver. */
static int mgs2(const double* x, int64_t n, int64_t p, double floor_, double* q) {
  memcpy(q, x, sizeof(double) * (size_t)(n * p));
  for (int pass = 0; pass < 2; ++pass)
    for (int64_t j = 0; j < p; ++j) {
      double* qj = q + j * n;
      for (int64_t k = 0; k < j; ++k) {
        const double* qk = q + k * n;
        const double s = orc_dot(qk, qj, n);
        for (int64_t i = 0; i < n; ++i) qj[i] -= s * qk[i];
      }
      const double nrm2 = orc_dot(qj, qj, n);
      if (!(nrm2 > floor_)) return ORC_E_RANK;
      const double inv = 1.0 / sqrt(nrm2);
      for (int64_t i = 0; i < n; ++i) qj[i] *= inv;
    }
  return ORC_OK;
}

int orc_mgs2(const double* x, int64_t n, int64_t p, double floor_, double* q) {
  return mgs2(x, n, p, floor_, q);
}

/* orthonormalize_with_r (kernels.cpp:250-261). */
int orc_orthonormalize(const double* x, int64_t n, int64_t p, double* q) {
  return orc_orthonormalize_t(x, n, p, q, 1);
}

int orc_orthonormalize_t(const double* x, int64_t n, int64_t p, double* q, int threads) {
  double* b = (double*)malloc(sizeof(double) * (size_t)(p * p));
  double* l = (double*)malloc(sizeof(double) * (size_t)(p * p));
  double* q1 = (double*)malloc(sizeof(double) * (size_t)(n * p));
  int rc = ORC_OK;
  orc_gram(x, n, p, b, threads);
  const double floor_ = 1e-14 * orc_frobenius_norm(b, p * p);
  if (!cholesky_lower(b, p, floor_, l)) {
    rc = mgs2(x, n, p, floor_, q);
  } else {
    solve_right_lt(x, n, p, l, q1, threads);
    orc_gram(q1, n, p, b, threads);
    if (!cholesky_lower(b, p, floor_, l)) rc = mgs2(x, n, p, floor_, q);
    else solve_right_lt(q1, n, p, l, q, threads);
  }
  free(b);
  free(l);
  free(q1);
  return rc;
}

/* spectral_norm_estimate (kernels.cpp:267-293). */
double orc_spectral_norm_estimate(const double* a, int64_t n, uint64_t seed, int threads) {
  const double fro = orc_frobenius_norm(a, n * n);
  if (fro == 0.0) return 0.0;
  double* v = (double*)malloc(sizeof(double) * (size_t)n);
  double* w = (double*)malloc(sizeof(double) * (size_t)n);
  double* t = (double*)malloc(sizeof(double) * (size_t)n);
  orc_random_normal(n, seed, v, 1);
  {
    const double nv = sqrt(orc_dot(v, v, n));
    if (nv == 0.0) v[0] = 1.0;
    else for (int64_t i = 0; i < n; ++i) v[i] /= nv;
  }
  double prev = -1.0, est = 0.0;
  for (int it = 0; it < 500; ++it) {
    orc_matmul(a, n, n, v, 1, w, threads);
    est = sqrt(orc_dot(w, w, n));
    orc_matmul(a, n, n, w, 1, t, threads);
    const double nt = sqrt(orc_dot(t, t, n));
    if (nt == 0.0) break;
    for (int64_t i = 0; i < n; ++i) t[i] /= nt;
    double* sw = v; v = t; t = sw;
    if (prev >= 0.0 && fabs(est - prev) <= 1e-6 * (est > 1e-300 ? est : 1e-300)) break;
    prev = est;
  }
  free(v);
  free(w);
  free(t);
  return est < fro ? est : fro;
}

/* ------------------------------------------------------------------------ */
/* Grid operators.  L = −Δ_h, h = 1:
 * (Lx)_i = 6 x_i − x_{i−ex} − x_{i+ex} − x_{i−ey} − x_{i+ey} − x_{i−ez} − x_{i+ez}
 * on the periodic grid, evaluated left to right in exactly that order. */

void orc_laplacian_apply(const double* x, int64_t nx, int64_t ny, int64_t nz, int64_t p,
                         double* lx) {
  const int64_t n = nx * ny * nz;
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < p; ++j) {
    const double* xj = x + j * n;
    double* oj = lx + j * n;
    for (int64_t z = 0; z < nz; ++z)
      for (int64_t y = 0; y < ny; ++y)
        for (int64_t xx = 0; xx < nx; ++xx) {
          const int64_t i = xx + nx * (y + ny * z);
          const int64_t xm = (xx == 0 ? nx - 1 : xx - 1) + nx * (y + ny * z);
          const int64_t xp = (xx == nx - 1 ? 0 : xx + 1) + nx * (y + ny * z);
          const int64_t ym = xx + nx * ((y == 0 ? ny - 1 : y - 1) + ny * z);
          const int64_t yp = xx + nx * ((y == ny - 1 ? 0 : y + 1) + ny * z);
          const int64_t zm = xx + nx * (y + ny * (z == 0 ? nz - 1 : z - 1));
          const int64_t zp = xx + nx * (y + ny * (z == nz - 1 ? 0 : z + 1));
          oj[i] = 6.0 * xj[i] - xj[xm] - xj[xp] - xj[ym] - xj[yp] - xj[zm] - xj[zp];
        }
  }
}

/* Real orthonormal eigenbasis of the periodic N-point second difference
 * (2 on the diagonal, −1 to both periodic neighbours).  Mode order:
 * m=0 constant; m=2k−1 cos(2πki/N), m=2k sin(2πki/N) for 1 ≤ k < N/2;
 * m=N−1 the alternating mode when N is even.  lam[m] = 2 − 2cos(2πk/N). */
void orc_fourier_basis(int64_t N, double* q, double* lam) {
  const double two_pi = 6.283185307179586476925286766559;
  const double c0 = 1.0 / sqrt((double)N);
  const double c1 = sqrt(2.0 / (double)N);
  for (int64_t i = 0; i < N; ++i) q[i] = c0;
  lam[0] = 0.0;
  int64_t m = 1;
  for (int64_t k = 1; 2 * k < N; ++k) {
    const double th = two_pi * (double)k / (double)N;
    for (int64_t i = 0; i < N; ++i) {
      const double ang = two_pi * (double)((k * i) % N) / (double)N;
      q[i + N * m] = c1 * cos(ang);
      q[i + N * (m + 1)] = c1 * sin(ang);
    }
    lam[m] = 2.0 - 2.0 * cos(th);
    lam[m + 1] = lam[m];
    m += 2;
  }
  if (N % 2 == 0) {
    for (int64_t i = 0; i < N; ++i) q[i + N * m] = (i % 2 == 0) ? c0 : -c0;
    lam[m] = 4.0;
  }
}

typedef struct {
  double *qx, *qy, *qz, *lx, *ly, *lz;
  double* tmp;
} ks_tables;

int orc_model_prepare(orc_model* m) {
  if (m->kind != ORC_MODEL_KOHN_SHAM) return ORC_OK;
  if (m->nx * m->ny * m->nz != m->n) return ORC_E_DIM;
  ks_tables* t = (ks_tables*)calloc(1, sizeof(ks_tables));
  t->qx = (double*)malloc(sizeof(double) * (size_t)(m->nx * m->nx));
  t->qy = (double*)malloc(sizeof(double) * (size_t)(m->ny * m->ny));
  t->qz = (double*)malloc(sizeof(double) * (size_t)(m->nz * m->nz));
  t->lx = (double*)malloc(sizeof(double) * (size_t)m->nx);
  t->ly = (double*)malloc(sizeof(double) * (size_t)m->ny);
  t->lz = (double*)malloc(sizeof(double) * (size_t)m->nz);
  t->tmp = (double*)malloc(sizeof(double) * (size_t)m->n * 2);
  orc_fourier_basis(m->nx, t->qx, t->lx);
  orc_fourier_basis(m->ny, t->qy, t->ly);
  orc_fourier_basis(m->nz, t->qz, t->lz);
  m->work = t;
  return ORC_OK;
}

void orc_model_release(orc_model* m) {
  ks_tables* t = (ks_tables*)m->work;
  if (!t) return;
  free(t->qx); free(t->qy); free(t->qz); free(t->lx); free(t->ly); free(t->lz); free(t->tmp);
  free(t);
  m->work = NULL;
}

/* One axis of a separable transform: out[.., m, ..] = Σ_i Q[i, m]·in[.., i, ..]
 * (forward, transpose=1) or Σ_m Q[i, m]·in[.., m, ..] (inverse, transpose=0),
 * accumulated in index order.  stride = distance between consecutive axis
 * entries, lines enumerate the other two axes. */
static void axis_transform(const double* in, double* out, const double* q, int64_t N,
                           int64_t nx, int64_t ny, int64_t nz, int axis, int forward) {
  const int64_t n = nx * ny * nz;
  const int64_t stride = axis == 0 ? 1 : (axis == 1 ? nx : nx * ny);
  for (int64_t base = 0; base < n; ++base) {
    /* base enumerates line starts: entries whose axis coordinate is 0 */
    const int64_t coord = (base / stride) % N;
    if (coord != 0) continue;
    for (int64_t o = 0; o < N; ++o) {
      double s = 0.0;
      for (int64_t i = 0; i < N; ++i) {
        const double qv = forward ? q[i + N * o] : q[o + N * i];
        s += qv * in[base + i * stride];
      }
      out[base + o * stride] = s;
    }
  }
  (void)nz;
}

/* L†ρ: forward real Fourier transform along x, y, z; divide mode (mx,my,mz)
 * by λx+λy+λz, zero the constant mode; inverse along z, y, x. */
int orc_pseudo_inverse_laplacian(const orc_model* m, const double* rho, double* out) {
  const ks_tables* t = (const ks_tables*)m->work;
  if (!t) return ORC_E_PARAM;
  const int64_t nx = m->nx, ny = m->ny, nz = m->nz, n = m->n;
  double* a = t->tmp;
  double* b = t->tmp + n;
  axis_transform(rho, a, t->qx, nx, nx, ny, nz, 0, 1);
  axis_transform(a, b, t->qy, ny, nx, ny, nz, 1, 1);
  axis_transform(b, a, t->qz, nz, nx, ny, nz, 2, 1);
  for (int64_t z = 0; z < nz; ++z)
    for (int64_t y = 0; y < ny; ++y)
      for (int64_t x = 0; x < nx; ++x) {
        const int64_t i = x + nx * (y + ny * z);
        const double lam = t->lx[x] + t->ly[y] + t->lz[z];
        a[i] = (i == 0) ? 0.0 : a[i] / lam;
      }
  axis_transform(a, b, t->qz, nz, nx, ny, nz, 2, 0);
  axis_transform(b, a, t->qy, ny, nx, ny, nz, 1, 0);
  axis_transform(a, out, t->qx, nx, nx, ny, nz, 0, 0);
  return ORC_OK;
}

static int all_finite(const double* a, int64_t count) { /* kernels.cpp:353-357 */
  for (int64_t k = 0; k < count; ++k)
    if (!isfinite(a[k])) return 0;
  return 1;
}

/* ObjectiveModel::evaluate.
 *  dense   — QuadraticModel::evaluate (problems.cpp:130-141)
 *  stencil — f = ½⟨X, LX + V∘X⟩, G = LX + V∘X
 *  KS      — E = ¼⟨X,LX⟩ + ½Σ V_i ρ_i + ¼ ρᵀL†ρ + ½ Σ ρ_i ε(ρ_i),
 *            G = ½LX + (V + L†ρ − c ρ^{1/3})∘X, c = (3/π)^{1/3} */
int orc_evaluate(const orc_model* m, const double* x, double* f, double* g, int threads) {
  const int64_t n = m->n, p = m->p, np = n * p;
  if (m->kind == ORC_MODEL_DENSE) {
    orc_matmul(m->a, n, n, x, p, g, threads);
    const double quad = 0.5 * orc_dot(x, g, np);
    double lin = 0.0;
    if (m->g0) {
      lin = orc_dot(m->g0, x, np);
      for (int64_t k = 0; k < np; ++k) g[k] += 1.0 * m->g0[k];
    }
    *f = quad + lin;
  } else if (m->kind == ORC_MODEL_STENCIL) {
    orc_laplacian_apply(x, m->nx, m->ny, m->nz, p, g);
    for (int64_t j = 0; j < p; ++j)
      for (int64_t i = 0; i < n; ++i) g[i + j * n] = g[i + j * n] + m->v[i] * x[i + j * n];
    *f = 0.5 * orc_dot(x, g, np);
  } else if (m->kind == ORC_MODEL_KOHN_SHAM) {
    const double c = cbrt(3.0 / 3.14159265358979323846);
    double* rho = (double*)malloc(sizeof(double) * (size_t)n);
    double* h = (double*)malloc(sizeof(double) * (size_t)n);
    double* u = (double*)malloc(sizeof(double) * (size_t)n);
    /* ρ = row_sq_norms(X) (kernels.cpp:295-303 order: column-outer) */
    for (int64_t i = 0; i < n; ++i) rho[i] = 0.0;
    for (int64_t j = 0; j < p; ++j)
      for (int64_t i = 0; i < n; ++i) rho[i] += x[i + j * n] * x[i + j * n];
    orc_pseudo_inverse_laplacian(m, rho, h);
    orc_laplacian_apply(x, m->nx, m->ny, m->nz, p, g);
    const double lap = orc_dot(x, g, np); /* ⟨X, LX⟩ */
    double vr = 0.0, rh = 0.0, ex = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double cr = cbrt(rho[i]);
      vr += m->v[i] * rho[i];
      rh += rho[i] * h[i];
      ex += rho[i] * cr;
      u[i] = m->v[i] + h[i] - c * cr;
    }
    *f = 0.25 * lap + 0.5 * vr + 0.25 * rh - 0.375 * c * ex;
    for (int64_t j = 0; j < p; ++j)
      for (int64_t i = 0; i < n; ++i)
        g[i + j * n] = 0.5 * g[i + j * n] + u[i] * x[i + j * n];
    free(rho);
    free(h);
    free(u);
  } else {
    return ORC_E_PARAM;
  }
  if (!isfinite(*f) || !all_finite(g, np)) return ORC_E_EVAL; /* problems.cpp:27-30 */
  return ORC_OK;
}

/* fd_gradient_check (problems.cpp:296-325); the coordinate sample is drawn
 * from Rng(seed) exactly as the reference does (std::set ⇒ ascending order). */
static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}
double orc_fd_gradient_check(const orc_model* m, const double* x, double h, uint64_t seed) {
  const int64_t n = m->n, np = m->n * m->p;
  double* g = (double*)malloc(sizeof(double) * (size_t)np);
  double* gs = (double*)malloc(sizeof(double) * (size_t)np);
  double* probe = (double*)malloc(sizeof(double) * (size_t)np);
  double f0;
  orc_evaluate(m, x, &f0, g, 1);
  const int64_t want = np < 50 ? np : 50;
  int64_t* coords = (int64_t*)malloc(sizeof(int64_t) * (size_t)want);
  int64_t have = 0;
  orc_rng r;
  orc_rng_init(&r, seed);
  while (have < want) {
    const int64_t c = (int64_t)(orc_rng_next(&r) % (uint64_t)np);
    int dup = 0;
    for (int64_t q = 0; q < have; ++q) dup |= coords[q] == c;
    if (!dup) coords[have++] = c;
  }
  qsort(coords, (size_t)want, sizeof(int64_t), cmp_i64);
  memcpy(probe, x, sizeof(double) * (size_t)np);
  double worst = 0.0;
  for (int64_t q = 0; q < want; ++q) {
    const int64_t c = coords[q];
    const int64_t i = c % n, j = c / n;
    const double x0 = x[i + j * n];
    const double hh = h * (1.0 + fabs(x0));
    double fp, fm;
    probe[i + j * n] = x0 + hh;
    orc_evaluate(m, probe, &fp, gs, 1);
    probe[i + j * n] = x0 - hh;
    orc_evaluate(m, probe, &fm, gs, 1);
    probe[i + j * n] = x0;
    const double fd = (fp - fm) / (2.0 * hh);
    const double gv = g[i + j * n];
    const double e = fabs(fd - gv) / (1.0 + fabs(gv));
    if (e > worst) worst = e;
  }
  free(g); free(gs); free(probe); free(coords);
  return worst;
}

/* ------------------------------------------------------------------------ */
/* Solver — solver.cpp                                                        */

void orc_config_default(orc_config* c) {
  c->beta = -1.0;
  c->eta_kind = ORC_ETA_ABB;
  c->gamma = 1.0;
  c->eta_min = 1e-10;
  c->eta_max = 1e10;
  c->eta0 = 0.0;
  c->multiplier_rule = ORC_MULT_PCAL;
  c->tol_rel_kkt = 1e-8;
  c->max_iter = 3000;
  c->threads = 1;
  c->final_orth = 1;
  c->algorithm = ORC_ALG_PCAL;
}

static double clamp_eta(const orc_config* c, double v) { /* solver.cpp:95-97 */
  double r = v > c->eta_min ? v : c->eta_min;
  return r < c->eta_max ? r : c->eta_max;
}

double orc_flops_estimate_pcal(int64_t n, int64_t p) { /* diagnostics.cpp:100-114 */
  return 7.0 * ((double)n * (double)p * (double)p);
}

/* Per-iterate data, eval_iterate (solver.cpp:52-88). */
typedef struct {
  double f, kkt_abs, feas;
  double *grad_f, *gtx, *w, *kkt_mat, *xtx, *c;
} iterate_data;

static void idata_alloc(iterate_data* d, int64_t n, int64_t p) {
  d->grad_f = (double*)malloc(sizeof(double) * (size_t)(n * p));
  d->kkt_mat = (double*)malloc(sizeof(double) * (size_t)(n * p));
  d->gtx = (double*)malloc(sizeof(double) * (size_t)(p * p));
  d->w = (double*)malloc(sizeof(double) * (size_t)(p * p));
  d->xtx = (double*)malloc(sizeof(double) * (size_t)(p * p));
  d->c = (double*)malloc(sizeof(double) * (size_t)(p * p));
}
static void idata_free(iterate_data* d) {
  free(d->grad_f); free(d->kkt_mat); free(d->gtx); free(d->w); free(d->xtx); free(d->c);
}

static int eval_iterate(const orc_model* m, const double* x, iterate_data* d, double* tmp_np,
                        int threads) {
  const int64_t n = m->n, p = m->p, np = n * p;
  int rc = orc_evaluate(m, x, &d->f, d->grad_f, threads);
  if (rc) return rc;
  orc_matmul_at_b(d->grad_f, n, p, x, p, d->gtx, threads);       /* :78 */
  orc_sym_part(d->gtx, p, d->w);                                 /* :79 */
  orc_matmul(x, n, p, d->w, p, tmp_np, threads);                 /* :80 */
  for (int64_t k = 0; k < np; ++k) d->kkt_mat[k] = d->grad_f[k] + -1.0 * tmp_np[k];
  orc_gram(x, n, p, d->xtx, threads);                            /* :81 */
  memcpy(d->c, d->xtx, sizeof(double) * (size_t)(p * p));        /* :83-84 */
  for (int64_t i = 0; i < p; ++i) d->c[i + i * p] += -1.0;
  d->kkt_abs = orc_frobenius_norm(d->kkt_mat, np);               /* :85 */
  d->feas = orc_frobenius_norm(d->c, p * p);                     /* :86 */
  return ORC_OK;
}

/* PCAL multiplier/gradient branch (solver.cpp:385-409). */
static void pcal_grad_l(const iterate_data* d, const double* x, int64_t n, int64_t p,
                        double beta, int mult_rule, double* gl, double* tmp_np, int threads) {
  const int64_t np = n * p;
  orc_matmul(x, n, p, d->c, p, tmp_np, threads);                               /* :390 */
  for (int64_t k = 0; k < np; ++k) gl[k] = d->kkt_mat[k] + beta * tmp_np[k];
  if (mult_rule == ORC_MULT_PCAL) {                                            /* :392-405 */
    for (int64_t j = 0; j < p; ++j) {
      const double* xj = x + j * n;
      double* oj = gl + j * n;
      double dj = 0.0;
      for (int64_t i = 0; i < n; ++i) dj += xj[i] * oj[i];
      for (int64_t i = 0; i < n; ++i) oj[i] -= dj * xj[i];
    }
  }
}

int orc_pcal_grad_l(const orc_model* m, const double* x, double beta, int mult_rule,
                    double* grad_l, double* f, double* kkt_abs, double* feas, int threads) {
  iterate_data d;
  idata_alloc(&d, m->n, m->p);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)(m->n * m->p));
  int rc = eval_iterate(m, x, &d, tmp, threads);
  if (!rc) {
    pcal_grad_l(&d, x, m->n, m->p, beta < 0 ? 1.0 : beta, mult_rule, grad_l, tmp, threads);
    *f = d.f;
    *kkt_abs = d.kkt_abs;
    *feas = d.feas;
  }
  free(tmp);
  idata_free(&d);
  return rc;
}

/* stepsize_select (solver.cpp:212-251).  xp == NULL means "no memory". */
double orc_stepsize_select(const orc_config* c, int64_t iter, double eta_prev, double eta0,
                           const double* x, const double* xp, const double* gl,
                           const double* glp, int64_t count) {
  if (c->eta_kind == ORC_ETA_CONSTANT) return clamp_eta(c, c->gamma);
  const double fallback = eta_prev > 0.0 ? eta_prev : eta0;
  if (!xp || !glp || iter == 0) return clamp_eta(c, eta0 > 0.0 ? eta0 : fallback);
  double ss = 0.0, sy = 0.0, yy = 0.0;
  for (int64_t k = 0; k < count; ++k) { /* :218-222, storage-order sums */
    const double s = x[k] + -1.0 * xp[k];
    ss += s * s;
  }
  for (int64_t k = 0; k < count; ++k) {
    const double s = x[k] + -1.0 * xp[k];
    const double y = gl[k] + -1.0 * glp[k];
    sy += s * y;
  }
  for (int64_t k = 0; k < count; ++k) {
    const double y = gl[k] + -1.0 * glp[k];
    yy += y * y;
  }
  double bb1 = (ss == 0.0 || sy == 0.0) ? fallback : fabs(sy) / ss;
  double bb2 = (sy == 0.0) ? fallback : yy / fabs(sy);
  double eta = fallback;
  switch (c->eta_kind) {
    case ORC_ETA_BB1: eta = bb1; break;
    case ORC_ETA_BB2: eta = bb2; break;
    case ORC_ETA_ABB: eta = (iter % 2 == 1) ? bb1 : bb2; break;
    case ORC_ETA_DIFFERENTIAL: eta = (ss == 0.0) ? fallback : sqrt(yy) / sqrt(ss); break;
    default: break;
  }
  return clamp_eta(c, eta);
}

/* pcal_step (solver.cpp:264-307). */
int orc_pcal_step(const double* x, const double* gl, int64_t n, int64_t p, double eta,
                  double* out, int64_t* degenerate, int threads) {
  if (!(eta > 0.0)) return ORC_E_PARAM;
  const double inv_eta = 1.0 / eta;
  int64_t deg = 0;
#pragma omp parallel for num_threads(threads > 0 ? threads : 1) reduction(+ : deg)
  for (int64_t j = 0; j < p; ++j) {
    double* zj = out + j * n;
    const double* xj = x + j * n;
    const double* gj = gl + j * n;
    double nrm2 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const double v = xj[i] - inv_eta * gj[i];
      zj[i] = v;
      nrm2 += v * v;
    }
    const double nrm = sqrt(nrm2);
    if (nrm < 1e-14) {
      deg += 1;
      double pn = 0.0;
      for (int64_t i = 0; i < n; ++i) pn += xj[i] * xj[i];
      pn = sqrt(pn);
      if (pn > 0.0) {
        const double inv = 1.0 / pn;
        for (int64_t i = 0; i < n; ++i) zj[i] = xj[i] * inv;
      } else {
        for (int64_t i = 0; i < n; ++i) zj[i] = 0.0;
        zj[j % n] = 1.0;
      }
      continue;
    }
    const double inv = 1.0 / nrm;
    for (int64_t i = 0; i < n; ++i) zj[i] *= inv;
  }
  if (degenerate) *degenerate = deg;
  if (!all_finite(out, n * p)) return ORC_E_DIVERGE;
  return ORC_OK;
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static double relative_kkt(double kkt_abs, double den) { /* solver.cpp:90-93 */
  if (den > 0.0) return kkt_abs / den;
  return kkt_abs == 0.0 ? 0.0 : INFINITY;
}

static int validate(const orc_config* c) { /* solver.cpp:106-118 */
  if (c->beta >= 0.0 && !isfinite(c->beta)) return ORC_E_PARAM;
  if (!(c->tol_rel_kkt > 0.0)) return ORC_E_PARAM;
  if (c->max_iter < 1) return ORC_E_PARAM;
  if (c->threads < 1) return ORC_E_PARAM;
  if (!(c->eta_min < c->eta_max)) return ORC_E_PARAM;
  if (c->eta_kind == ORC_ETA_CONSTANT && !(c->gamma > 0.0)) return ORC_E_PARAM;
  return ORC_OK;
}

static void snap(orc_report* r, int64_t k, const double* x, double eta, int64_t np) {
  for (int q = 0; q < r->nsnap; ++q)
    if (r->snap_iters[q] == k) {
      memcpy(r->snaps + (int64_t)q * np, x, sizeof(double) * (size_t)np);
      if (r->snap_eta) r->snap_eta[q] = eta;
    }
}

/* iterate_main (solver.cpp:320-474) and solve (:626-633). */
int orc_solve_pcal(const orc_model* m, const orc_config* c, const double* x0, orc_report* r) {
  return orc_solve(m, c, x0, r);
}

int orc_solve(const orc_model* m, const orc_config* c, const double* x0, orc_report* r) {
  const double t0 = now_s();
  int rc = validate(c);
  if (rc) return rc;
  const int alg = c->algorithm;
  if (alg == ORC_ALG_ALM || alg < 0 || alg > ORC_ALG_PCALDA) return ORC_E_PARAM;
  const int64_t n = m->n, p = m->p, np = n * p;
  const int threads = c->threads;
  const int da = alg == ORC_ALG_PLAMDA || alg == ORC_ALG_PCALDA;                /* :326-330 */
  const int normalized = alg == ORC_ALG_PCAL || alg == ORC_ALG_PCALDA;
  const int retraction = alg == ORC_ALG_MOPTQR;
  const int mult = (alg == ORC_ALG_PCAL) ? c->multiplier_rule : ORC_MULT_PLAM;
  double beta;                                                                  /* :120-134 */
  if (c->beta >= 0.0) beta = c->beta;
  else if (alg == ORC_ALG_PCAL || alg == ORC_ALG_PCALDA) beta = 1.0;
  else if (alg == ORC_ALG_MOPTQR) beta = 0.0;
  else beta = m->s + 0.1;
  const double eta0 = c->eta0 > 0.0 ? clamp_eta(c, c->eta0)                /* :99-102 */
                                    : clamp_eta(c, m->s + 2.0 * beta);
  r->beta_used = beta;
  r->eta0_used = eta0;
  r->trace_len = 0;
  r->has_post = 0;
  r->has_x = 0;
  r->iterations = 0;
  r->degenerate_steps = 0;
  for (int q = 0; q < 4; ++q) r->final_pre[q] = r->final_post[q] = 0.0;

  double* x = (double*)malloc(sizeof(double) * (size_t)np);
  double* xp = (double*)malloc(sizeof(double) * (size_t)np);
  double* gl = (double*)malloc(sizeof(double) * (size_t)np);
  double* glp = (double*)malloc(sizeof(double) * (size_t)np);
  double* xn = (double*)malloc(sizeof(double) * (size_t)np);
  double* tmp = (double*)malloc(sizeof(double) * (size_t)np);
  double* lam = (double*)calloc((size_t)(p * p), sizeof(double));
  double* mm = (double*)malloc(sizeof(double) * (size_t)(p * p));
  iterate_data d;
  idata_alloc(&d, n, p);
  memcpy(x, x0, sizeof(double) * (size_t)np);
  int have_prev = 0;
  double eta_state = 0.0;
  int status = ORC_MAXITER;
  double rel = 0.0, kkt_den = 0.0;

#define RECORD(iter_, eta_)                                            \
  do {                                                                 \
    double* row = r->trace + r->trace_len * ORC_TRACE_COLS;            \
    row[0] = (double)(iter_);                                          \
    row[1] = d.f;                                                      \
    row[2] = d.kkt_abs;                                                \
    row[3] = relative_kkt(d.kkt_abs, kkt_den);                         \
    row[4] = d.feas;                                                   \
    row[5] = (eta_);                                                   \
    row[6] = now_s() - t0;                                             \
    r->trace_len++;                                                    \
    rel = row[3];                                                      \
  } while (0)

  snap(r, 0, x, 0.0, np);
  rc = eval_iterate(m, x, &d, tmp, threads);
  if (rc) {
    status = ORC_DIVERGED;
  } else {
    kkt_den = d.kkt_abs;
    RECORD(0, eta0);
    if (rel < c->tol_rel_kkt) {
      status = ORC_CONVERGED;
    } else {
      for (int64_t k = 0; k < c->max_iter; ++k) {
        if (retraction) {                                   /* :371-374 */
          orc_matmul(x, n, p, d.gtx, p, tmp, threads);
          for (int64_t q = 0; q < np; ++q) gl[q] = d.grad_f[q] + -1.0 * tmp[q];
        } else if (da) {                                    /* :375-384 */
          if (k == 0) {
            memcpy(lam, d.w, sizeof(double) * (size_t)(p * p));
          } else {
            /* lambda.add_scaled(-beta, xtx.add_scaled(-1, I)): upper triangle, mirrored */
            for (int64_t jj = 0; jj < p; ++jj)
              for (int64_t ii = 0; ii <= jj; ++ii) {
                const double cij = d.xtx[ii + jj * p] + -1.0 * (ii == jj ? 1.0 : 0.0);
                const double v = lam[ii + jj * p] + -beta * cij;
                lam[ii + jj * p] = v;
                lam[jj + ii * p] = v;
              }
          }
          for (int64_t q = 0; q < p * p; ++q) mm[q] = beta * d.c[q] - lam[q];
          orc_matmul(x, n, p, mm, p, tmp, threads);
          for (int64_t q = 0; q < np; ++q) gl[q] = d.grad_f[q] + 1.0 * tmp[q];
        } else {                                            /* :385-409 */
          pcal_grad_l(&d, x, n, p, beta, mult, gl, tmp, threads);
        }
        const double eta = orc_stepsize_select(c, k, eta_state, eta0, x, have_prev ? xp : NULL,
                                               gl, have_prev ? glp : NULL, np);
        int64_t deg = 0;
        if (retraction) {                                   /* :415-418 */
          if (!(eta > 0.0)) { rc = ORC_E_PARAM; goto done_error; }
          const double sc = -1.0 / eta;
          for (int64_t q = 0; q < np; ++q) tmp[q] = x[q] + sc * gl[q];
          if (orc_orthonormalize_t(tmp, n, p, xn, threads) != ORC_OK) { status = ORC_DIVERGED; rc = ORC_OK; break; }
        } else if (normalized) {                            /* :419-422 */
          rc = orc_pcal_step(x, gl, n, p, eta, xn, &deg, threads);
          if (rc == ORC_E_PARAM) goto done_error;
          if (rc == ORC_E_DIVERGE) { status = ORC_DIVERGED; rc = ORC_OK; break; }
        } else {                                            /* plam_step :253-262 */
          if (!(eta > 0.0)) { rc = ORC_E_PARAM; goto done_error; }
          const double sc = -1.0 / eta;
          for (int64_t q = 0; q < np; ++q) xn[q] = x[q] + sc * gl[q];
          if (!all_finite(xn, np)) { status = ORC_DIVERGED; rc = ORC_OK; break; }
        }
        r->degenerate_steps += deg;
        /* rotate: prev ← current, current ← next (:427-430) */
        { double* t = xp; xp = x; x = xn; xn = t; }
        { double* t = glp; glp = gl; gl = t; }
        have_prev = 1;
        eta_state = eta;
        snap(r, k + 1, x, eta, np);
        rc = eval_iterate(m, x, &d, tmp, threads);
        if (rc) { status = ORC_DIVERGED; rc = ORC_OK; break; }
        r->iterations = k + 1;
        RECORD(k + 1, eta);
        if (rel < c->tol_rel_kkt) { status = ORC_CONVERGED; break; }
      }
    }
    if (status != ORC_DIVERGED) {
      r->final_pre[0] = d.f;
      r->final_pre[1] = d.kkt_abs;
      r->final_pre[2] = rel;
      r->final_pre[3] = d.feas;
      if (r->stop_x) memcpy(r->stop_x, x, sizeof(double) * (size_t)np);
      if (r->final_x) memcpy(r->final_x, x, sizeof(double) * (size_t)np);
      r->has_x = 1;
      if (c->final_orth) {                                                 /* :445-459 */
        if (orc_orthonormalize_t(x, n, p, xn, threads) == ORC_OK) {
          int erc = eval_iterate(m, xn, &d, tmp, threads);
          if (erc) {
            status = ORC_DIVERGED;
          } else {
            r->final_post[0] = d.f;
            r->final_post[1] = d.kkt_abs;
            r->final_post[2] = relative_kkt(d.kkt_abs, kkt_den);
            r->final_post[3] = d.feas;
            r->has_post = 1;
            if (r->final_x) memcpy(r->final_x, xn, sizeof(double) * (size_t)np);
          }
        }
      }
    }
  }
  if (status == ORC_DIVERGED && r->trace_len > 0) {                        /* :467-471 */
    const double* last = r->trace + (r->trace_len - 1) * ORC_TRACE_COLS;
    r->final_pre[0] = last[1];
    r->final_pre[1] = last[2];
    r->final_pre[2] = last[3];
    r->final_pre[3] = last[4];
    r->has_post = 0;
  }
  r->status = status;
  rc = ORC_OK;
done_error:
  r->wall_time = now_s() - t0;
  free(x); free(xp); free(gl); free(glp); free(xn); free(tmp); free(lam); free(mm);
  idata_free(&d);
#undef RECORD
  return rc;
}
