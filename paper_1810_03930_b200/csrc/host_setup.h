// host_setup.h — host-side setup helpers (reference RNG stream, Fourier basis).
#pragma once
#include <cstdint>

namespace pcal {
void host_random_normal(int64_t count, uint64_t seed, double* out, int threads);
// rows [row0, row0+nrows) of random_normal(n, p, Rng(seed)), nrows × p column-major
void host_random_normal_rows(int64_t n, int64_t p, uint64_t seed, int64_t row0, int64_t nrows,
                             double* out, int threads);
void host_random_uniform(int64_t count, uint64_t seed, double* out);
// `count` uniforms of Rng(seed) drawn after `nnormals` normal() calls (each
// Box–Muller pair consumes two raw draws; a cached spare does not).
void host_uniform_after_normals(int64_t nnormals, uint64_t seed, int64_t count, double* out);
// fd_gradient_check's coordinate sample (problems.cpp:301-305): distinct
// Rng(seed).next_u64() % total until `want` are drawn, in ascending order.
void host_fd_coordinates(int64_t total, uint64_t seed, int64_t want, int64_t* out);
}  // namespace pcal

void pcal_fourier_basis(int64_t N, double* q, double* lam);
