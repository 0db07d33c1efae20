// host_setup.h — host-side setup helpers (reference RNG stream, Fourier basis).
#pragma once
#include <cstdint>

namespace pcal {
void host_random_normal(int64_t count, uint64_t seed, double* out, int threads);
void host_random_uniform(int64_t count, uint64_t seed, double* out);
}  // namespace pcal

void pcal_fourier_basis(int64_t N, double* q, double* lam);
