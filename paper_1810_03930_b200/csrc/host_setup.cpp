// host_setup.cpp — problem setup on the host: the reference's documented
// random stream (rng.hpp:13-55, kernels.cpp:65-78: xoshiro256++ seeded by
// splitmix64, uniforms from the top 53 bits, Box–Muller normals with a cached
// spare) and the periodic Fourier basis of the Kohn–Sham model.  The stream is
// part of the reference's data contract (same seed ⇒ same instance), so the
// draws here are bitwise identical to the reference; the Box–Muller work is
// spread over threads from checkpointed generator states.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <set>
#include <thread>
#include <vector>

#include "../../include/pcal_b200.h"
#include "host_setup.h"

namespace {

struct Rng {
  uint64_t s[4];
  explicit Rng(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s) w = splitmix64(x);
  }
  static uint64_t splitmix64(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ULL;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t next() {
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
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  // One Box–Muller pair: the first value is returned by normal(), the second
  // is the cached spare (kernels.cpp:65-78).
  void pair(double& c, double& sn) {
    const double u1 = 1.0 - uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 6.283185307179586476925286766559 * u2;
    sn = r * std::sin(t);
    c = r * std::cos(t);
  }
};

}  // namespace

namespace pcal {

void host_fd_coordinates(int64_t total, uint64_t seed, int64_t want, int64_t* out) {
  Rng rng(seed);
  std::set<int64_t> coords;
  while ((int64_t)coords.size() < want) coords.insert((int64_t)(rng.next() % (uint64_t)total));
  int64_t k = 0;
  for (int64_t c : coords) out[k++] = c;
}

void host_random_normal(int64_t count, uint64_t seed, double* out, int threads) {
  Rng r(seed);
  const int64_t npairs = (count + 1) / 2;
  const int64_t chunk = int64_t(1) << 16;
  const int64_t nchunks = (npairs + chunk - 1) / chunk;
  if (threads <= 1 || nchunks < 2) {
    for (int64_t m = 0; m < npairs; ++m) {
      double c, s;
      r.pair(c, s);
      out[2 * m] = c;
      if (2 * m + 1 < count) out[2 * m + 1] = s;
    }
    return;
  }
  std::vector<Rng> cps;
  cps.reserve(static_cast<size_t>(nchunks));
  for (int64_t c = 0; c < nchunks; ++c) {
    cps.push_back(r);
    const int64_t pairs = (c + 1 < nchunks) ? chunk : npairs - c * chunk;
    for (int64_t q = 0; q < 2 * pairs; ++q) (void)r.next();
  }
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (int64_t c = t; c < nchunks; c += threads) {
        Rng g = cps[static_cast<size_t>(c)];
        const int64_t p0 = c * chunk, p1 = (c + 1 < nchunks) ? p0 + chunk : npairs;
        for (int64_t m = p0; m < p1; ++m) {
          double cv, sv;
          g.pair(cv, sv);
          out[2 * m] = cv;
          if (2 * m + 1 < count) out[2 * m + 1] = sv;
        }
      }
    });
  for (auto& th : pool) th.join();
}

// Rows [row0, row0 + nrows) of random_normal(n, p, Rng(seed)) (column-major
// fill, kernels.cpp:49-55): value (i, j) is draw k = i + j·n of the normal
// stream, i.e. the cos (k even) or sin (k odd) half of Box–Muller pair ⌊k/2⌋.
// One sequential pass of raw draws checkpoints the generator at each column's
// first pair; the columns' Box–Muller work then runs on `threads` threads.
// Bitwise the same values as the full fill, for any slab.
void host_random_normal_rows(int64_t n, int64_t p, uint64_t seed, int64_t row0, int64_t nrows,
                             double* out, int threads) {
  if (nrows <= 0 || p <= 0) return;
  Rng r(seed);
  std::vector<Rng> cps;
  cps.reserve(static_cast<size_t>(p));
  int64_t pos = 0;  // Box–Muller pairs consumed so far
  for (int64_t j = 0; j < p; ++j) {
    const int64_t m0 = (j * n + row0) / 2;
    for (int64_t q = 0; q < 2 * (m0 - pos); ++q) (void)r.next();
    pos = m0;
    cps.push_back(r);
  }
  auto column = [&](int64_t j) {
    Rng g = cps[static_cast<size_t>(j)];
    double* o = out + j * nrows;
    int64_t i = 0;
    double c, sn;
    if ((j * n + row0) % 2 == 1) {  // the slab starts on a pair's sin half
      g.pair(c, sn);
      o[i++] = sn;
    }
    while (i < nrows) {
      g.pair(c, sn);
      o[i++] = c;
      if (i < nrows) o[i++] = sn;
    }
  };
  threads = std::max(1, threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      for (int64_t j = t; j < p; j += threads) column(j);
    });
  for (auto& th : pool) th.join();
}

void host_uniform_after_normals(int64_t nnormals, uint64_t seed, int64_t count, double* out) {
  Rng r(seed);
  const int64_t skip = 2 * ((nnormals + 1) / 2);
  for (int64_t q = 0; q < skip; ++q) (void)r.next();
  for (int64_t k = 0; k < count; ++k) out[k] = r.uniform();
}

void host_random_uniform(int64_t count, uint64_t seed, double* out) {
  Rng r(seed);
  for (int64_t k = 0; k < count; ++k) out[k] = r.uniform();
}

}  // namespace pcal

// Real orthonormal eigenbasis of the periodic N-point second difference
// (DESIGN.md §3): column m of q (q[i + N·m]) is mode m; lam[m] its eigenvalue.
void pcal_fourier_basis(int64_t N, double* q, double* lam) {
  const double two_pi = 6.283185307179586476925286766559;
  const double c0 = 1.0 / std::sqrt(static_cast<double>(N));
  const double c1 = std::sqrt(2.0 / static_cast<double>(N));
  for (int64_t i = 0; i < N; ++i) q[i] = c0;
  lam[0] = 0.0;
  int64_t m = 1;
  for (int64_t k = 1; 2 * k < N; ++k) {
    const double th = two_pi * static_cast<double>(k) / static_cast<double>(N);
    for (int64_t i = 0; i < N; ++i) {
      const double ang = two_pi * static_cast<double>((k * i) % N) / static_cast<double>(N);
      q[i + N * m] = c1 * std::cos(ang);
      q[i + N * (m + 1)] = c1 * std::sin(ang);
    }
    lam[m] = 2.0 - 2.0 * std::cos(th);
    lam[m + 1] = lam[m];
    m += 2;
  }
  if (N % 2 == 0) {
    for (int64_t i = 0; i < N; ++i) q[i + N * m] = (i % 2 == 0) ? c0 : -c0;
    lam[m] = 4.0;
  }
}

extern "C" {

int pcal_random_normal(int64_t rows, int64_t cols, uint64_t seed, double* out, int32_t threads) {
  if (!out || rows < 1 || cols < 1) return PCAL_E_PARAMETER;
  pcal::host_random_normal(rows * cols, seed, out, threads);
  return PCAL_OK;
}

int pcal_random_uniform(int64_t count, uint64_t seed, double* out) {
  if (!out || count < 0) return PCAL_E_PARAMETER;
  pcal::host_random_uniform(count, seed, out);
  return PCAL_OK;
}

// sym_part(random_normal(n,n,Rng(seed))) (problems.cpp:45-48, kernels.cpp:28-36).
int pcal_gen_dense_operator(int64_t n, uint64_t seed, double* a, int32_t threads) {
  if (!a || n < 1) return PCAL_E_PARAMETER;
  pcal::host_random_normal(n * n, seed, a, threads);
  // in place: a(i,j) = a(j,i) = 0.5·(b(i,j) + b(j,i)) for i ≤ j (same value both sides)
  const int nt = threads > 1 ? threads : 1;
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([=] {
      for (int64_t j = t; j < n; j += nt)
        for (int64_t i = 0; i <= j; ++i) {
          const double v = 0.5 * (a[i + j * n] + a[j + i * n]);
          a[i + j * n] = v;
          a[j + i * n] = v;
        }
    });
  for (auto& th : pool) th.join();
  return PCAL_OK;
}

// spectral_norm_estimate (kernels.cpp:267-293) on the host, bitwise: power
// iteration on A² from a Box–Muller start vector; the column-axpy products of
// matmul (kernels.cpp:105-122) are split over row blocks, which keeps every
// element's k-order; norms and the Frobenius bound are sequential sums.
int pcal_spectral_norm_estimate_host(const double* a, int64_t n, uint64_t seed, int32_t threads,
                                     double* out) {
  if (!a || !out || n < 1) return PCAL_E_PARAMETER;
  auto seq_dot = [](const double* x, const double* y, int64_t m) {
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += x[i] * y[i];
    return s;
  };
  const double fro = std::sqrt(seq_dot(a, a, n * n));
  if (fro == 0.0) {
    *out = 0.0;
    return PCAL_OK;
  }
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(threads > 0 ? threads : 1, n / 64 + 1));
  auto matvec = [&](const double* v, double* w) {  // w = A·v, column axpy order
    std::vector<std::thread> pool;
    const int64_t blk = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([=] {
        const int64_t i0 = t * blk, i1 = std::min(n, i0 + blk);
        for (int64_t i = i0; i < i1; ++i) w[i] = 0.0;
        for (int64_t k = 0; k < n; ++k) {
          const double s = v[k];
          const double* ak = a + k * n;
          for (int64_t i = i0; i < i1; ++i) w[i] += s * ak[i];
        }
      });
    for (auto& th : pool) th.join();
  };
  std::vector<double> v((size_t)n), w((size_t)n), t((size_t)n);
  pcal::host_random_normal(n, seed, v.data(), 1);
  {
    const double nv = std::sqrt(seq_dot(v.data(), v.data(), n));
    if (nv == 0.0) v[0] = 1.0;
    else
      for (auto& e : v) e /= nv;
  }
  double prev = -1.0, est = 0.0;
  for (int it = 0; it < 500; ++it) {
    matvec(v.data(), w.data());
    est = std::sqrt(seq_dot(w.data(), w.data(), n));
    matvec(w.data(), t.data());
    const double ntn = std::sqrt(seq_dot(t.data(), t.data(), n));
    if (ntn == 0.0) break;
    for (auto& e : t) e /= ntn;
    std::swap(v, t);
    if (prev >= 0.0 && std::abs(est - prev) <= 1e-6 * std::max(est, 1e-300)) break;
    prev = est;
  }
  *out = std::min(est, fro);
  return PCAL_OK;
}

}  // extern "C"

// L⁻¹ for the density models: the reference's LinearSolver (linsolve.cpp:10-102)
// — Cholesky when every pivot is positive and finite, else LU with partial
// pivoting and a 1e-14·max|L| singularity floor — solved against e_j for each
// column j with the same forward / back substitution loops.  Columns are
// independent, so they are spread over `threads`.
int pcal_density_inverse(const double* l, int64_t n, double* linv, int32_t threads) {
  if (!l || !linv || n < 1) return PCAL_E_PARAMETER;
  const size_t N = (size_t)n;
  // factors stored row-major (F(i,j) at i·n + j): the factorisation's inner
  // loops and the substitutions' row loops then run along memory; the
  // arithmetic and its order are the reference's.
  std::vector<double> f(N * N);
  auto F = [&](int64_t i, int64_t j) -> double& { return f[(size_t)j + (size_t)i * N]; };
  bool spd = true;
  for (int64_t j = 0; j < n && spd; ++j) {  // try_cholesky (linsolve.cpp:10-26)
    double d = l[j + j * n];
    for (int64_t k = 0; k < j; ++k) d -= F(j, k) * F(j, k);
    if (!(d > 0.0) || !std::isfinite(d)) {
      spd = false;
      break;
    }
    const double ljj = std::sqrt(d);
    F(j, j) = ljj;
    for (int64_t i = j + 1; i < n; ++i) {
      double s = l[i + j * n];
      for (int64_t k = 0; k < j; ++k) s -= F(i, k) * F(j, k);
      F(i, j) = s / ljj;
    }
  }
  std::vector<int64_t> perm;
  if (!spd) {  // LU with partial pivoting on a dense copy (linsolve.cpp:36-67)
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) F(i, j) = l[i + j * n];
    perm.resize(N);
    for (int64_t i = 0; i < n; ++i) perm[(size_t)i] = i;
    double scale = 0.0;
    for (double v : f) scale = std::max(scale, std::abs(v));
    const double floor = 1e-14 * std::max(scale, 1e-300);
    for (int64_t k = 0; k < n; ++k) {
      int64_t piv = k;
      double best = std::abs(F(k, k));
      for (int64_t i = k + 1; i < n; ++i)
        if (std::abs(F(i, k)) > best) {
          best = std::abs(F(i, k));
          piv = i;
        }
      if (!(best > floor)) return PCAL_E_PARAMETER;  // generation_error: numerically singular
      if (piv != k) {
        for (int64_t j = 0; j < n; ++j) std::swap(F(k, j), F(piv, j));
        std::swap(perm[(size_t)k], perm[(size_t)piv]);
      }
      const double inv = 1.0 / F(k, k);
      for (int64_t i = k + 1; i < n; ++i) {
        const double m = F(i, k) * inv;
        F(i, k) = m;
        if (m != 0.0)
          for (int64_t j = k + 1; j < n; ++j) F(i, j) -= m * F(k, j);
      }
    }
  }
  // column-major copy for the Cholesky back substitution's column loop
  std::vector<double> fc;
  if (spd) {
    fc.resize(N * N);
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) fc[(size_t)i + (size_t)j * N] = F(i, j);
  }
  // LinearSolver::solve(e_c) for every column c (linsolve.cpp:70-102)
  auto solve_col = [&](int64_t c, std::vector<double>& y) {
    for (int64_t i = 0; i < n; ++i) y[(size_t)i] = (spd ? i : perm[(size_t)i]) == c ? 1.0 : 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double s = y[(size_t)i];
      for (int64_t k = 0; k < i; ++k) s -= F(i, k) * y[(size_t)k];
      y[(size_t)i] = spd ? s / F(i, i) : s;
    }
    for (int64_t i = n - 1; i >= 0; --i) {
      double s = y[(size_t)i];
      if (spd)
        for (int64_t k = i + 1; k < n; ++k) s -= fc[(size_t)k + (size_t)i * N] * y[(size_t)k];
      else
        for (int64_t k = i + 1; k < n; ++k) s -= F(i, k) * y[(size_t)k];
      y[(size_t)i] = s / F(i, i);
    }
    std::memcpy(linv + c * n, y.data(), sizeof(double) * N);
  };
  const int nt = std::max(1, std::min<int>(threads, (int)n));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&, t] {
      std::vector<double> y(N);
      for (int64_t c = t; c < n; c += nt) solve_col(c, y);
    });
  for (auto& th : pool) th.join();
  return PCAL_OK;
}
