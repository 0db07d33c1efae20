// session.cu — native runtime of the B200 PCAL solver and its C ABI.
//
// One host thread drives one CUDA stream.  A PCAL iteration (solver.cpp:369-439)
// is a fixed sequence of kernels with every scalar (η, flags, trace row) kept
// in device memory, captured once per buffer parity into a CUDA graph; the
// host enqueues graphs ahead of the stopping decision and polls the device
// `done` flag asynchronously, so the iteration never waits on the host.
//
// Memory layout (HBM): every n×p matrix is column-major with leading dimension
// ld = round_up(n,32) and pp = round_up(p,32) columns, zero padded.  The
// iterate X_k and the PCAL gradient buffer P_k (∇f(X_k), then overwritten in
// place by g_plam = ∇f − XW + βXC) are stored side by side as a pair
// [P_k | X_k] so the Gram GEMM reads [P|X]ᵀX as ONE operand; two pairs
// ping-pong (k even / odd).  GL = P − d∘X is never stored: it is recomputed in
// registers by the two streaming kernels that need it.
#include <cuda_runtime.h>

#include <algorithm>
#include <functional>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/pcal_b200.h"
#include "comm.h"
#include "common.cuh"
#include "gemm_types.h"
#include "host_setup.h"
#include "operators.cuh"
#include "pcal_kernels.cuh"
#include "stencil_tma.cuh"

namespace pcal {

thread_local int64_t* g_launch_counter = nullptr;
thread_local KernelProfiler* g_kprof = nullptr;
thread_local std::string g_last_error;
// which branch of orthonormalize (kernels.cpp:250-261) the calling thread's last
// device orthonormalisation took: 0 CholeskyQR2, 1 / 2 MGS2 after the first /
// second Cholesky pass hit the pivot floor, -1 rank-deficient (MGS2 failed too)
thread_local int32_t g_orth_path = 0;

// ------------------------------------------------------------------------------
// small dense kernels of the final orthonormalization (kernels.cpp:159-195)
// ------------------------------------------------------------------------------

// ‖B‖_F² over the full (mirrored) p×p Gram; b: pp×pp, upper triangle valid.
__global__ void k_sym_fro2(const double* __restrict__ b, int64_t ldb, int64_t p, double* out) {
  __shared__ double sm[32];
  double acc = 0.0;
  for (int64_t e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int64_t i = e % p, j = e / p;
    const double v = b[min(i, j) + max(i, j) * ldb];
    acc += v * v;
  }
  const double s = block_sum<1024>(acc, sm);
  if (threadIdx.x == 0) *out = s;
}

// cholesky_lower (kernels.cpp:159-175): left-looking, column j after column j.
// floor = 1e-14·sqrt(fro2[0]) of the FIRST Gram (kernels.cpp:252); status[0]=0 on failure.
__global__ void k_cholesky(const double* __restrict__ b, int64_t ldb, int64_t p,
                           const double* fro2_first, double* __restrict__ l, int64_t ldl,
                           int32_t* status, const int32_t* prev_ok = nullptr,
                           const Ctl* ctl = nullptr) {
  __shared__ double s_ljj;
  __shared__ int s_ok;
  if (ctl && ctl->done) return;
  if (prev_ok && !*prev_ok) {  // first CholeskyQR pass already failed
    if (threadIdx.x == 0) *status = 0;
    return;
  }
  const double floor_ = 1e-14 * sqrt(*fro2_first);
  if (threadIdx.x == 0) s_ok = 1;
  for (int64_t e = threadIdx.x; e < p * p; e += blockDim.x) l[(e % p) + (e / p) * ldl] = 0.0;
  __syncthreads();
  for (int64_t j = 0; j < p; ++j) {
    if (threadIdx.x == 0) {
      double d = b[j + j * ldb];
      for (int64_t k = 0; k < j; ++k) d -= l[j + k * ldl] * l[j + k * ldl];
      if (!(d > floor_)) s_ok = 0;
      s_ljj = sqrt(d);
      l[j + j * ldl] = s_ljj;
    }
    __syncthreads();
    if (!s_ok) break;
    const double ljj = s_ljj;
    for (int64_t i = j + 1 + threadIdx.x; i < p; i += blockDim.x) {
      double s = b[j + i * ldb];  // upper triangle: b(j,i) = b(i,j)
      for (int64_t k = 0; k < j; ++k) s -= l[i + k * ldl] * l[j + k * ldl];
      l[i + j * ldl] = s / ljj;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *status = s_ok;
}

// T = (L⁻¹)ᵀ (upper triangular), T[k + c·ldt] = (L⁻¹)[c,k]; one thread per column c
// of L⁻¹ (forward substitution).  Q = X·T then solves Q·Lᵀ = X (solve_right_lt).
__global__ void k_trinv_t(const double* __restrict__ l, int64_t ldl, int64_t p,
                          double* __restrict__ t, int64_t ldt, const int32_t* status) {
  if (!*status) return;
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= p) return;
  for (int64_t i = 0; i < c; ++i) t[c + i * ldt] = 0.0;
  for (int64_t i = c; i < p; ++i) {
    double s = (i == c) ? 1.0 : 0.0;
    for (int64_t k = c; k < i; ++k) s -= l[i + k * ldl] * t[c + k * ldt];
    t[c + i * ldt] = s / l[i + i * ldl];
  }
}

// Cholesky + T = (L⁻¹)ᵀ in ONE block for p ≤ kCholSmemP, with L resident in
// shared memory: left-looking Cholesky (the same recurrence and pivot floor as
// k_cholesky; d_j and the column dots are warp reductions), then forward
// substitution for the columns of L⁻¹, one warp per column (lanes hold the
// solution entries k ≡ lane mod 32).  Replaces k_cholesky + k_trinv_t, whose
// global-memory recurrences are latency-bound (≈0.3 ms each at p = 128).
constexpr int kCholSmemP = 128;
__global__ void __launch_bounds__(1024) k_chol_trinv_small(const double* __restrict__ b,
                                                           int64_t ldb, int p,
                                                           const double* fro2_first,
                                                           double* __restrict__ t, int64_t ldt,
                                                           int32_t* status,
                                                           const int32_t* prev_ok,
                                                           const Ctl* ctl) {
  extern __shared__ double sL[];  // p×p column-major: sL[i + k·p] = L(i, k), i ≥ k
  __shared__ double s_ljj;
  __shared__ int s_ok;
  if (ctl && ctl->done) return;
  if (prev_ok && !*prev_ok) {  // first CholeskyQR pass already failed
    if (threadIdx.x == 0) *status = 0;
    return;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const double floor_ = 1e-14 * sqrt(*fro2_first);
  for (int e = tid; e < p * p; e += blockDim.x) {  // lower triangle of B (from its upper one)
    const int i = e % p, j = e / p;
    sL[e] = i >= j ? b[j + (int64_t)i * ldb] : 0.0;
  }
  if (tid == 0) s_ok = 1;
  __syncthreads();
  for (int j = 0; j < p; ++j) {
    if (warp == 0) {
      double d = 0.0;
      for (int k = lane; k < j; k += 32) d += sL[j + k * p] * sL[j + k * p];
      d = warp_sum(d);
      if (lane == 0) {
        d = sL[j + j * p] - d;
        if (!(d > floor_)) s_ok = 0;
        s_ljj = sqrt(d);
        sL[j + j * p] = s_ljj;
      }
    }
    __syncthreads();
    if (!s_ok) break;
    const double ljj = s_ljj;
    for (int i = j + 1 + warp; i < p; i += nw) {
      double acc = 0.0;
      for (int k = lane; k < j; k += 32) acc += sL[i + k * p] * sL[j + k * p];
      acc = warp_sum(acc);
      if (lane == 0) sL[i + j * p] = (sL[i + j * p] - acc) / ljj;
    }
    __syncthreads();
  }
  if (tid == 0) *status = s_ok;
  if (!s_ok) return;
  // columns c of L⁻¹: x_i = (δ_ic − Σ_{c≤k<i} L(i,k)·x_k) / L(i,i), T(c, i) = x_i
  for (int c = warp; c < p; c += nw) {
    double x[kCholSmemP / 32];
#pragma unroll
    for (int q = 0; q < kCholSmemP / 32; ++q) x[q] = 0.0;
    for (int i = lane; i < c; i += 32) t[c + (int64_t)i * ldt] = 0.0;
    for (int i = c; i < p; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < kCholSmemP / 32; ++q) {
        const int k = lane + 32 * q;
        if (k >= c && k < i) acc += sL[i + k * p] * x[q];
      }
      acc = warp_sum(acc);
      const double xi = ((i == c) ? 1.0 : 0.0) - acc;
      const double v = xi / sL[i + i * p];
#pragma unroll
      for (int q = 0; q < kCholSmemP / 32; ++q)
        if (lane + 32 * q == i) x[q] = v;
      if (lane == (i & 31)) t[c + (int64_t)i * ldt] = v;
    }
  }
}

// Cholesky for kCholSmemP < p ≤ kCholWideP (L does not fit in shared memory):
// the left-looking recurrence of k_cholesky with the factor stored TRANSPOSED,
// u[k + i·ldu] = L(i, k), so every dot Σ_k L(i,k)·L(j,k) reads two contiguous
// rows — one warp per row, lanes over k, fixed-order warp sums — and row j of L
// staged in shared memory for the column's updates.  Same pivot floor.
// (k_cholesky's thread-0 recurrence took ≈ 75 ms at p = 1024.)
constexpr int kCholWideP = 2048;
__global__ void __launch_bounds__(1024) k_cholesky_wide(const double* __restrict__ b,
                                                        int64_t ldb, int p,
                                                        const double* fro2_first,
                                                        double* __restrict__ u, int64_t ldu,
                                                        int32_t* status, const int32_t* prev_ok,
                                                        const Ctl* ctl) {
  __shared__ double s_row[kCholWideP];  // row j of L (k < j)
  __shared__ double s_ljj;
  __shared__ int s_ok;
  if (ctl && ctl->done) return;
  if (prev_ok && !*prev_ok) {
    if (threadIdx.x == 0) *status = 0;
    return;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, nw = blockDim.x >> 5;
  const double floor_ = 1e-14 * sqrt(*fro2_first);
  if (tid == 0) s_ok = 1;
  for (int j = 0; j < p; ++j) {
    // row j of L (written by the earlier columns) into shared memory
    for (int k = tid; k < j; k += blockDim.x) s_row[k] = u[k + (int64_t)j * ldu];
    __syncthreads();
    if (warp == 0) {
      double d = 0.0;
      for (int k = lane; k < j; k += 32) d += s_row[k] * s_row[k];
      d = warp_sum(d);
      if (lane == 0) {
        d = b[j + (int64_t)j * ldb] - d;
        if (!(d > floor_)) s_ok = 0;
        s_ljj = sqrt(d);
        u[j + (int64_t)j * ldu] = s_ljj;
      }
    }
    __syncthreads();
    if (!s_ok) break;
    const double ljj = s_ljj;
    for (int i = j + 1 + warp; i < p; i += nw) {
      const double* ui = u + (int64_t)i * ldu;
      double acc = 0.0;
      for (int k = lane; k < j; k += 32) acc += ui[k] * s_row[k];
      acc = warp_sum(acc);
      if (lane == 0) u[j + (int64_t)i * ldu] = (b[j + (int64_t)i * ldb] - acc) / ljj;  // B(j,i), upper
    }
    __syncthreads();
  }
  if (tid == 0) *status = s_ok;
}

// T = (L⁻¹)ᵀ from the transposed factor of k_cholesky_wide: one warp per column c
// of L⁻¹ (forward substitution, lanes hold x_k for k ≡ lane mod 32, rows of L
// read contiguously), T(c, i) = x_i.
template <int NQ>  // p ≤ 32·NQ
__global__ void __launch_bounds__(256) k_trinv_wide(const double* __restrict__ u, int64_t ldu,
                                                    int p, double* __restrict__ t, int64_t ldt,
                                                    const int32_t* status) {
  if (!*status) return;
  const int lane = threadIdx.x & 31;
  const int c = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (c >= p) return;
  double x[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) x[q] = 0.0;
  for (int i = lane; i < c; i += 32) t[c + (int64_t)i * ldt] = 0.0;
  for (int i = c; i < p; ++i) {
    const double* ui = u + (int64_t)i * ldu;
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int k = lane + 32 * q;
      if (k >= c && k < i) acc += ui[k] * x[q];
    }
    acc = warp_sum(acc);
    const double v = (((i == c) ? 1.0 : 0.0) - acc) / ui[i];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (lane + 32 * q == i) x[q] = v;
    if (lane == (i & 31)) t[c + (int64_t)i * ldt] = v;
  }
}

// mgs2 (kernels.cpp:212-246) fallback: one block, in place on q (= copy of X).
__global__ void k_mgs2(double* __restrict__ q, int64_t n, int64_t ld, int64_t p,
                       const double* fro2_first, int32_t* status) {
  __shared__ double sm[32];
  __shared__ double s_v;
  const double floor_ = 1e-14 * sqrt(*fro2_first);
  for (int pass = 0; pass < 2; ++pass)
    for (int64_t j = 0; j < p; ++j) {
      double* qj = q + j * ld;
      for (int64_t k = 0; k < j; ++k) {
        const double* qk = q + k * ld;
        double acc = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += qk[i] * qj[i];
        const double s = block_sum<1024>(acc, sm);
        if (threadIdx.x == 0) s_v = s;
        __syncthreads();
        const double sv = s_v;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) qj[i] -= sv * qk[i];
        __syncthreads();
      }
      double acc = 0.0;
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += qj[i] * qj[i];
      const double nrm2 = block_sum<1024>(acc, sm);
      if (threadIdx.x == 0) s_v = nrm2;
      __syncthreads();
      if (!(s_v > floor_)) {
        if (threadIdx.x == 0) *status = 0;
        return;
      }
      const double inv = 1.0 / sqrt(s_v);
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) qj[i] *= inv;
      __syncthreads();
    }
  if (threadIdx.x == 0) *status = 1;
}

// In-graph MGS2 fallback of the MOptQR retraction: runs only when a CholeskyQR
// pass failed; a rank-deficient iterate is a rank_error ⇒ Diverged
// (orthonormalize inside solve(), solver.cpp:415-418,464-465).
__global__ void k_mgs2_gated(double* __restrict__ q, int64_t n, int64_t ld, int64_t p,
                             const double* fro2_first, const int32_t* ok1, const int32_t* ok2,
                             int32_t* status, Ctl* ctl) {
  if (ctl->done) return;
  if (*ok1 && *ok2) return;
  __shared__ double sm[32];
  __shared__ double s_v;
  const double floor_ = 1e-14 * sqrt(*fro2_first);
  for (int pass = 0; pass < 2; ++pass)
    for (int64_t j = 0; j < p; ++j) {
      double* qj = q + j * ld;
      for (int64_t k = 0; k < j; ++k) {
        const double* qk = q + k * ld;
        double acc = 0.0;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += qk[i] * qj[i];
        const double s = block_sum<1024>(acc, sm);
        if (threadIdx.x == 0) s_v = s;
        __syncthreads();
        const double sv = s_v;
        for (int64_t i = threadIdx.x; i < n; i += blockDim.x) qj[i] -= sv * qk[i];
        __syncthreads();
      }
      double acc = 0.0;
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += qj[i] * qj[i];
      const double nrm2 = block_sum<1024>(acc, sm);
      if (threadIdx.x == 0) s_v = nrm2;
      __syncthreads();
      if (!(s_v > floor_)) {
        if (threadIdx.x == 0) {
          *status = 0;
          ctl->step_bad = 1;
          ctl->done = 2;
        }
        return;
      }
      const double inv = 1.0 / sqrt(s_v);
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) qj[i] *= inv;
      __syncthreads();
    }
}

// ------------------------------------------------------------------------------
// evaluation bookkeeping kernels
// ------------------------------------------------------------------------------
struct FinishArgs {
  const double* fcol;   // p: Σ over rows of the model's f partials (per column)
  const double* kcol;   // p: Σ kkt² per column
  const double* cpart;  // ncp: Σ C² partials
  int32_t ncp;
  const double* spart;  // KS density scalars partials (nsp × 3) or null
  int32_t nsp;
  int32_t model;
  int64_t p;
  int32_t mode;         // 0 = iteration record, 1 = start point (row 0), 2 = post-orth
  const double* flags;  // sharded: allreduced {step_bad, eval_bad} counts (else null)
  double* trace;
  int32_t* bad;         // evaluation non-finite flag
  double c_xc;          // (3/π)^{1/3}
  const double* fdev;   // device-callback models: f(X) as written by the callback
  double coeff;         // density models: α (P1) / γ (P6)
  int32_t p6;           // density models: the P6 term
  const double* glcol;  // ALM: Σ_i P_ij² per column (‖∇L‖² = their sum), else null
  const double* k2_id;  // XM1 mode: Σ kkt² by the identity (k_kkt_gate) unless *k2_fb
  const int32_t* k2_fb;
};

// ALM inner-loop bookkeeping for the iterate just evaluated (alm_outer,
// solver.cpp:544-561): it is tested while the inner loop and the iteration
// budget allow — best ‖∇L‖ so far (its X is then copied to the best buffer),
// tolerance max(scale·tol, scale^(outer+1))·kkt0 — else the loop ends at a cap.
__device__ void alm_test(Ctl* c, double f, double kkt, double feas, double gl2) {
  c->alm_copy = 0;
  if (c->alm_inner < c->alm_inner_max && c->iter < c->max_iter) {
    const double gl = sqrt(gl2);
    if (gl < c->alm_best) {
      c->alm_best = gl;
      c->alm_copy = 1;
      c->best_f = f;
      c->best_kkt = kkt;
      c->best_feas = feas;
    }
    const double sc = c->alm_tol_scale;
    const double tk = fmax(sc * c->tol, pow(sc, (double)(c->alm_outer + 1))) *
                      (c->kkt_den > 0.0 ? c->kkt_den : 1.0);
    c->alm_met = gl <= tk;
    c->alm_phase = c->alm_met ? 1 : 0;
  } else {
    c->alm_met = 0;
    c->alm_phase = 1;
  }
}

// Thread-0 tail of an evaluation: objective assembly, failure flags, trace
// row, stopping test (solver.cpp:348-359,434-438,460-471).
__device__ void finish_record(const FinishArgs& a, Ctl* ctl, double* post, double f1, double k2,
                              double c2, double vr, double rh, double ex, double gl2 = 0.0) {
  const bool bad_flag = a.flags ? a.flags[1] > 0.0 : *a.bad != 0;
  *a.bad = 0;  // reset for the next evaluation
  if (a.flags && a.mode == 0 && a.flags[0] > 0.0) {  // some rank's pcal_step diverged
    ctl->step_bad = 1;
    ctl->done = 2;
    return;
  }
  double f;
  if (a.model == PCAL_MODEL_KOHN_SHAM) {
    f = 0.25 * f1 + 0.5 * vr + 0.25 * rh - 0.375 * a.c_xc * ex;
  } else if (a.model == PCAL_MODEL_DEVICE_CALLBACK) {
    f = *a.fdev;
  } else if (a.model == PCAL_MODEL_DENSITY) {  // problems.cpp:175-194
    f = a.p6 ? 0.5 * f1 + 0.5 * rh - 0.75 * a.coeff * ex : 0.5 * f1 + 0.25 * a.coeff * rh;
  } else {
    f = 0.5 * f1;
  }
  const double kkt = sqrt(k2), feas = sqrt(c2);
  const bool bad = bad_flag || !isfinite(f);
  if (a.mode == 2) {  // post-orth metrics (solver.cpp:452-455)
    post[0] = f;
    post[1] = kkt;
    post[2] = ctl->kkt_den > 0.0 ? kkt / ctl->kkt_den : (kkt == 0.0 ? 0.0 : INFINITY);
    post[3] = feas;
    post[4] = bad ? 1.0 : 0.0;
    return;
  }
  if (bad) {  // evaluation_error ⇒ Diverged, no trace row (solver.cpp:462-466)
    ctl->eval_bad = 1;
    ctl->done = 2;
    if (a.mode == 0) ctl->degenerate += ctl->step_deg;
    return;
  }
  if (a.mode == 3) {  // ALM multiplier update: a new inner loop starts here (no trace row)
    ctl->f = f;
    ctl->kkt_abs = kkt;
    ctl->feas = feas;
    alm_test(ctl, f, kkt, feas, gl2);
    return;
  }
  int64_t k;
  double eta;
  if (a.mode == 1) {
    k = ctl->iter;
    ctl->kkt_den = ctl->iter == 0 ? kkt : ctl->kkt_den;
    eta = ctl->iter == 0 ? ctl->eta0 : ctl->eta_prev;
  } else {
    k = ctl->iter + 1;
    ctl->degenerate += ctl->step_deg;
    ctl->eta_prev = ctl->eta;
    ctl->have_prev = 1;
    eta = ctl->eta;
  }
  const double rel = ctl->kkt_den > 0.0 ? kkt / ctl->kkt_den : (kkt == 0.0 ? 0.0 : INFINITY);
  double* row = a.trace + ctl->trace_len * kTraceCols;
  row[0] = (double)k;
  row[1] = f;
  row[2] = kkt;
  row[3] = rel;
  row[4] = feas;
  row[5] = eta;
  row[6] = (double)(globaltimer_ns() - ctl->t0_ns) * 1e-9;
  ctl->trace_len += 1;
  ctl->iter = k;
  ctl->f = f;
  ctl->kkt_abs = kkt;
  ctl->feas = feas;
  ctl->rel = rel;
  if (rel < ctl->tol) ctl->done = 1;
  if (ctl->alm && !ctl->done) {
    if (a.mode == 0) ++ctl->alm_inner;
    alm_test(ctl, f, kkt, feas, gl2);
  }
}

// ALM outer step (solver.cpp:562-574), before the multiplier update's
// evaluation: the inner loop's iterate (its best one after a cap) has been
// copied to the other pair; the stepsize memory restarts with the next loop.
// Sharded ALM: the chunk-ordered column sums of the third partial are Σ P²
// (‖∇L‖²), not d; move them to glcol and leave d = 0 for the plain step.
__global__ void k_alm_split(double* __restrict__ d, double* __restrict__ gl, int64_t p,
                            const Ctl* ctl) {
  if (ctl && ctl->done) return;
  for (int64_t j = threadIdx.x; j < p; j += blockDim.x) {
    gl[j] = d[j];
    d[j] = 0.0;
  }
}

__global__ void k_alm_boundary(Ctl* c) {
  if (c->done) return;
  if (!c->alm_met) {
    ++c->alm_caps;
    c->f = c->best_f;
    c->kkt_abs = c->best_kkt;
    c->feas = c->best_feas;
  }
  ++c->alm_outer;
  ++c->alm_flips;
  c->alm_inner = 0;
  c->alm_best = INFINITY;
  c->alm_copy = 0;
  c->have_prev = 0;
  c->eta_prev = 0.0;
  c->iter_base = c->iter;
  if (c->alm_outer >= c->alm_outer_max || c->iter >= c->max_iter) c->done = 4;  // MaxIter
}

__global__ void __launch_bounds__(256) k_finish_eval(FinishArgs a, Ctl* ctl,
                                                     double* post /* 5 */) {
  if (a.mode != 2 && ctl->done) return;
  __shared__ double sm[8];
  double pf = 0.0, pk = 0.0, pc = 0.0, pv = 0.0, pr = 0.0, pe = 0.0;
  for (int64_t j = threadIdx.x; j < a.p; j += blockDim.x) {
    pf += a.fcol[j];
    pk += a.kcol[j];
  }
  for (int i = threadIdx.x; i < a.ncp; i += blockDim.x) pc += a.cpart[i];
  if (a.model == PCAL_MODEL_KOHN_SHAM || a.model == PCAL_MODEL_DENSITY)
    for (int i = threadIdx.x; i < a.nsp; i += blockDim.x) {
      pv += a.spart[3 * i];
      pr += a.spart[3 * i + 1];
      pe += a.spart[3 * i + 2];
    }
  const double f1 = block_sum<256>(pf, sm);
  const double k2s = block_sum<256>(pk, sm);
  const double k2 = (a.k2_id && !*a.k2_fb) ? *a.k2_id : k2s;
  const double c2 = block_sum<256>(pc, sm);
  const double vr = block_sum<256>(pv, sm);
  const double rh = block_sum<256>(pr, sm);
  const double ex = block_sum<256>(pe, sm);
  double pg = 0.0;
  if (a.glcol)
    for (int64_t j = threadIdx.x; j < a.p; j += blockDim.x) pg += a.glcol[j];
  const double gl2 = block_sum<256>(pg, sm);
  if (threadIdx.x != 0) return;
  finish_record(a, ctl, post, f1, k2, c2, vr, rh, ex, gl2);
}

}  // namespace pcal
#include "small.cuh"
#include "small_rows.cuh"
namespace pcal {

// check_finite (problems.cpp:27-30) of a caller-computed gradient.
__global__ void k_check_finite(const double* __restrict__ g, int64_t n, int64_t ld, int64_t p,
                               int32_t* bad, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  bool nonfinite = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * p;
       e += (int64_t)gridDim.x * blockDim.x)
    nonfinite |= !isfinite(g[e % n + (e / n) * ld]);
  if (__syncthreads_or(nonfinite) && threadIdx.x == 0) *bad = 1;
}

__global__ void k_zero_i32(int32_t* p, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  *p = 0;
}

// ------------------------------------------------------------------------------
// Session
// ------------------------------------------------------------------------------
struct DevBuf {
  double* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    free();
    if (count) PCAL_CUDA(cudaMalloc(&p, sizeof(double) * count));
    n = count;
  }
  void zero(cudaStream_t st) {
    if (p) PCAL_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * n, st));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { free(); }
};

}  // namespace pcal

struct pcal_session {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  // sharded grid models (NCCL): the halo exchange runs on hstream while the
  // interior planes of the stencil run on `stream` (ev_x: X ready, ev_h: halos in)
  cudaStream_t hstream = nullptr;
  cudaEvent_t ev_x = nullptr, ev_h = nullptr;
  // row sharding (null comm: the whole problem on this GPU)
  pcal::Comm* comm = nullptr;
  // reproducible reductions (every sharded session): fixed global row chunks
  bool repro = false;
  int64_t chunk_rows = 0;                 // Q: rows per chunk
  int64_t zc_planes = 0;                  // grid models: z-planes per chunk
  int64_t nch = 0, nch_max = 0;           // local / largest per-rank chunk count
  int32_t* rank_nch_d = nullptr;          // chunks per rank (device)
  int grad_splits = 0;                    // dense gradient: fixed K segments per tile
  int gram_sub = 1, orth_sub = 1;         // Gram segments per row chunk (fixed globally)
  bool sym_gx = false;                    // GᵀX symmetric (grid models): upper tiles only
  pcal::DevBuf cc, ccg, bbt, spt;         // chunk partials, gathered, totals
  struct Tree {                           // fixed-tree Gram reduction (0: iteration, 1: orth)
    int maxn = 0, nloc = 0;
    int64_t leaf0 = 0, nleaves = 0;
    int2* nodes_d = nullptr;              // [R][maxn] (level, index)
    int32_t* cnt_d = nullptr;             // [R]
    pcal::DevBuf tn, gath;                // this rank's node sums, all ranks' node sums
    ~Tree() {
      if (nodes_d) cudaFree(nodes_d);
      if (cnt_d) cudaFree(cnt_d);
    }
  } tree[2];
  int64_t n_glob = 0, row0 = 0;  // global row count, first owned row
  int64_t gz = 0;                // grid models: owned z-planes (nz for a single GPU)
  int64_t K_full = 0;            // dense: padded global row count (gradient GEMM K)
  int64_t ld_max = 0;            // common leading dimension of every rank's buffers
  std::vector<int64_t> rank_row0, rank_rows;
  pcal::DevBuf xfull, xgath, halo, rho_gath, rank_rows_d, fkd[2], nrm, xpart;
  pcal_model_desc model{};
  pcal_config cfg{};
  int64_t n = 0, p = 0, pp = 0, ld = 0;
  double beta = 1.0, eta0 = 0.0, c_xc = 0.0;
  // model data
  pcal::DevBuf A, g0, V, u, rho, h, tmpa, tmpb, qx, qy, qz, lx, ly, lz, spart;
  pcal::DevBuf Bm, tb, Minv;  // bilinear B (pp×pp) and A·X; density L⁻¹ rows
  pcal::DevBuf glcol, bestx;  // ALM: column sums of P², the inner loop's best X
  pcal::DevBuf fdev;  // device-callback models: f(X)
  int64_t ldA = 0;
  // iteration state
  pcal::DevBuf pair[2];
  pcal::DevBuf gr, mcat, fpart, kpart, dpart, cpart, bbpart, npart, post;
  pcal::DevBuf colpart, sinv;  // fused normalisation: (chunk, column) sums; 1/‖z_j‖
  int32_t* sfb = nullptr;      // per column: take the exact two-pass normalisation
  // XM1 mode (PCAL / PLAM on one GPU): P = G − X·M1, Σ kkt² by the identity
  // (pcal_kernels.cuh k_kkt_gate); M1 (slot order), W, C, C², the identity's
  // partials, [Σ kkt², fallback count], the fallback flag
  bool xm1 = false;
  double xm1_gate = 1e4;
  pcal::DevBuf m1, wmat, cmat, c2m, kcp, kk;
  int32_t* kfb = nullptr;
  pcal::DevBuf orth_b, orth_l, orth_t, orth_f2;
  int32_t* bad = nullptr;
  int32_t* orth_status = nullptr;
  pcal::Ctl* ctl = nullptr;
  pcal::Ctl* h_ctl = nullptr;  // pinned mirror
  pcal::DevBuf trace;
  int64_t trace_cap = 0;
  // plans
  pcal::GemmPlan grad[2], grad2[2], gram[2], xm[2], orth_gram, orth_mul;
  pcal::GemmPlan c2plan, xmfb[2];  // XM1 mode: C² and the gated two-block fallback
  // MOptQR in-graph retraction (per parity): Gram of Z, Z·T → Q1, Gram of Q1, Q1·T → Q
  pcal::GemmPlan rq_gram_z[2], rq_mul1[2], rq_gram_q[2], rq_mul2[2];
  pcal::DevBuf lam;  // dual-ascent multiplier Λ (p×p, replicated)
  int alg = PCAL_ALG_PCAL;
  int64_t nrb_grad = 0, nrb_xm = 0, nrb_f = 0;  // row-blocks of f/k/d partials
  int64_t pstride_f = 0, pstride_xm = 0;        // column strides of the partial arrays
  int64_t up_chunk = 0, up_nchunks = 0;
  int bb_blocks = 0, cp_blocks = 0, sp_blocks = 0;
  int64_t st_chunk = 0, st_nchunks = 0;
  bool st_march = false;
  bool fused_step = false;  // cooperative k_step_fused fits co-resident on the device
  // stencil model, one GPU: the normalised step's X_{k+1} formed inside the
  // TMA stencil (stencil_tma.cuh FUSE); grad_fused marks an iteration whose
  // gradient already exists except for the exact-rule columns
  bool step_stencil = false, grad_fused = false;
  bool mega = false;        // small dense problem: k_iter_small runs whole batches of iterations
  int mega_grid = 0;
  int64_t mega_lda_s = 0;   // > 0: k_iter_small keeps each CTA's 8 rows of A in shared memory
  pcal::DevBuf at, mpart, mz, mnpb, mbb;  // Aᵀ, Z and the CTA partials of k_iter_small
  bool rows = false;        // n ≤ 8·SMs: k_iter_rows (own rows in registers, 4 barriers)
  int rows_nent = 0, rows_ngroups = 0, rows_csize = 1;
  pcal::DevBuf rgpart, rgtot, rgcnt, rcpart;  // k_iter_rows partials / group sums / counters
  int64_t st_zchunk = 0, st_nzc = 0, st_zpart = 0;  // march z-chunk, count, planes per f partial
  // graphs
  cudaGraphExec_t graph[2] = {nullptr, nullptr};
  int64_t kernels_per_iter = 0;
  int64_t launches = 0;
  int64_t next_k = 0;      // iteration index the next launched graph performs
  int64_t launched = 0;    // iterations enqueued in total
  bool use_graphs = true;
  std::chrono::steady_clock::time_point t_start;
  pcal_category_timers* timers = nullptr;
  cudaEvent_t pev[6] = {};   // phase events (timers / profiling; never inside graphs)
  bool pev_on = false;
  double prof_ms[4] = {0, 0, 0, 0};  // stream, gradient, gram+pxp, xm+reductions
  int64_t prof_iters = 0;
  ~pcal_session();
};

namespace pcal {

// models whose gradient starts with the dense GEMM A·X (A n×n, row-sharded)
static bool dense_family(int32_t kind) {
  return kind == PCAL_MODEL_DENSE || kind == PCAL_MODEL_BILINEAR || kind == PCAL_MODEL_DENSITY;
}
static double* Xof(pcal_session* s, int b) { return s->pair[b].p + s->ld * s->pp; }
static double* Pof(pcal_session* s, int b) { return s->pair[b].p; }
// packed per-column sums of an evaluation: [f | kkt² | d] (one allreduce when sharded)
static double* Fcol(pcal_session* s, int b) { return s->fkd[b].p; }
static double* Kcol(pcal_session* s, int b) { return s->fkd[b].p + s->p; }
static double* Dvec(pcal_session* s, int b) { return s->fkd[b].p + 2 * s->p; }

static void mark(pcal_session* s, int i) {
  if (s->pev_on) PCAL_CUDA(cudaEventRecord(s->pev[i], s->stream));
}

struct LaunchScope {
  int64_t* prev;
  explicit LaunchScope(int64_t* c) : prev(g_launch_counter) { g_launch_counter = c; }
  ~LaunchScope() { g_launch_counter = prev; }
};

// Reproducible sum of per-chunk partials (W values per chunk, `cc` layout
// [nch_max][W]): all-gather in rank order, then the ordered chunk sum.
static void chunk_reduce(pcal_session* s, const double* cc, int64_t W, double* out,
                         const Ctl* ctl, int extra = 0) {
  const int R = s->comm->size;
  const size_t off = (size_t)s->nch_max * W;  // per-rank extras follow the chunk rows
  const size_t cnt = off + extra;
  if (R > 1) s->comm->allgather(cc, s->ccg.p, cnt, s->stream);
  k_chunk_sum<<<(unsigned)ceil_div(W + extra, 128), 128, 0, s->stream>>>(
      R > 1 ? s->ccg.p : cc, R, s->rank_nch_d, (int64_t)cnt, W, out, ctl, extra, (int64_t)off);
  launched("k_chunk_sum");
}

static void chunking(const pcal_model_desc& m, int64_t* Q, int64_t* NC, int64_t* Zc);

// Reproducible Gram: this rank's maximal tree nodes over its chunk partials,
// exchanged (O(log) node sums per rank) and merged into the same fixed tree
// on every rank (gemm_tree_local / gemm_tree_final).
static void gram_reduce(pcal_session* s, const GemmPlan& g, int which) {
  const int R = s->comm->size;
  auto& T = s->tree[which];
  launch_gemm_tree_local(g, T.nodes_d + (size_t)s->comm->rank * T.maxn, T.nloc, T.leaf0,
                         T.nleaves, T.tn.p, s->stream);
  const double* buf = T.tn.p;
  if (R > 1) {
    s->comm->allgather(T.tn.p, T.gath.p, T.tn.n, s->stream);
    buf = T.gath.p;
  }
  launch_gemm_tree_final(g, buf, T.cnt_d, T.nodes_d, R, T.maxn, s->stream);
}

// Maximal fixed-tree nodes inside the leaf range [l0, l1) of nleaves leaves.
static std::vector<int2> tree_nodes(int64_t l0, int64_t l1, int64_t nleaves) {
  int top = 0;
  while (((int64_t)1 << top) < nleaves) ++top;
  std::vector<int2> out;
  for (int64_t cur = l0; cur < l1;) {
    int best = 0;
    for (int l = top; l >= 0; --l) {
      if (cur % ((int64_t)1 << l)) continue;
      if (std::min(cur + ((int64_t)1 << l), nleaves) <= l1) {
        best = l;
        break;
      }
    }
    out.push_back(make_int2(best, (int)(cur >> best)));
    cur = std::min(cur + ((int64_t)1 << best), nleaves);
  }
  return out;
}

// Tree metadata of Gram `which` (m partials per row chunk; ntiles output tiles).
static void tree_setup(pcal_session* s, int which, int m, int64_t ntiles) {
  const int R = s->comm->size;
  auto& T = s->tree[which];
  int64_t NC = 0;
  std::vector<std::vector<int2>> nodes(R);
  std::vector<int64_t> c0(R + 1);
  {
    int64_t Q, Zc;
    chunking(s->model, &Q, &NC, &Zc);
  }
  T.nleaves = NC * m;
  for (int r = 0; r < R; ++r) {
    const int64_t a = (int64_t)r * NC / R * m, b = (int64_t)(r + 1) * NC / R * m;
    nodes[r] = tree_nodes(a, b, T.nleaves);
    T.maxn = std::max<int>(T.maxn, (int)nodes[r].size());
    if (r == s->comm->rank) T.leaf0 = a;
  }
  T.nloc = (int)nodes[s->comm->rank].size();
  std::vector<int2> flat((size_t)R * T.maxn, make_int2(0, 0));
  std::vector<int32_t> cnt(R);
  for (int r = 0; r < R; ++r) {
    cnt[r] = (int32_t)nodes[r].size();
    std::copy(nodes[r].begin(), nodes[r].end(), flat.begin() + (size_t)r * T.maxn);
  }
  PCAL_CUDA(cudaMalloc(&T.nodes_d, sizeof(int2) * flat.size()));
  PCAL_CUDA(cudaMemcpy(T.nodes_d, flat.data(), sizeof(int2) * flat.size(), cudaMemcpyHostToDevice));
  PCAL_CUDA(cudaMalloc(&T.cnt_d, sizeof(int32_t) * R));
  PCAL_CUDA(cudaMemcpy(T.cnt_d, cnt.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice));
  const CfgInfo ci = cfg_info(pick_size(s->pp));
  T.tn.alloc((size_t)T.maxn * ntiles * ci.BM * ci.BN);
  if (R > 1) T.gath.alloc((size_t)R * T.tn.n);
}

// Column sums of the three partial arrays (f, kkt², d), one launch.
static void launch_colsums(pcal_session* s, const double* fp, int64_t nrb_f, const double* kp,
                           const double* dp, int64_t nrb_kd, double* fcol, double* kcol,
                           double* dcol, const Ctl* ctl, const int32_t* gate = nullptr) {
  ColSumArgs a{};
  a.gate = gate;
  a.in[0] = fp;
  a.nrows[0] = nrb_f;
  a.stride[0] = s->pstride_f;
  a.out[0] = fcol;
  a.in[1] = kp;
  a.nrows[1] = nrb_kd;
  a.stride[1] = s->pstride_xm;
  a.out[1] = kcol;
  // d_j only for PCAL with the PCAL formula (solver.cpp:329-330,392-408); else d stays 0
  a.in[2] = (dp && s->alg == PCAL_ALG_PCAL && s->cfg.multiplier_rule == PCAL_MULT_PCAL_FORMULA)
                ? dp
                : nullptr;
  a.nrows[2] = nrb_kd;
  a.stride[2] = s->pstride_xm;
  a.out[2] = dcol;
  if (dp && s->alg == PCAL_ALG_ALM) {  // ALM: ‖∇L‖² column sums; d stays 0
    a.in[2] = dp;
    a.out[2] = s->glcol.p;
  }
  k_colsum3<<<dim3((unsigned)s->p, 3), kStreamThreads, 0, s->stream>>>(a, ctl);
  launched("k_colsum3");
}

// Gradient of the model at X (pair b): G into P(b), f partials into fpart.
// 7-point stencil part of the grid models: z-marching kernel when the grid
// allows it (nx ≤ 128, ny % 8 == 0), else the generic element kernel.
static void launch_stencil_tma(pcal_session* s, int b, const double* u, bool ks, const Ctl* ctl,
                               int xp, const double* hlo, const double* hhi, dim3 grid,
                               int zmode = 0, const int32_t* only_fb = nullptr,
                               const StepFuse* fuse = nullptr) {
  constexpr int TY = 8, NS = 4;
  const auto& m = s->model;
  const int64_t nx = m.nx, ny = m.ny, nz = s->gz, p = s->p;
  // X operand: X of pair b, or (fused step) X_k of pair b with P_k beside it;
  // output G into P of pair b, or (fused) P of the other pair
  const double* xsrc = Xof(s, b);
  double* gout = fuse ? Pof(s, 1 - b) : Pof(s, b);
  StencilMaps mp;
  {
    const int64_t d4[4] = {nx, ny, nz, p}, pt4[3] = {nx * 8, nx * ny * 8, s->ld * 8};
    const int bt[4] = {(int)nx, TY, 1, 1}, br[4] = {(int)nx, 1, 1, 1};
    encode_tensor_map(&mp.x_tile, xsrc, 4, d4, pt4, bt);
    encode_tensor_map(&mp.x_row, xsrc, 4, d4, pt4, br);
    const double* psrc = fuse ? Pof(s, b) : xsrc;  // unused unless fused: any valid map
    encode_tensor_map(&mp.p_tile, psrc, 4, d4, pt4, bt);
    encode_tensor_map(&mp.p_row, psrc, 4, d4, pt4, br);
    const int64_t d3[3] = {nx, ny, nz}, pt3[2] = {nx * 8, nx * ny * 8};
    const int bu[3] = {(int)nx, TY, 1};
    encode_tensor_map(&mp.u_tile, u, 3, d3, pt3, bu);
    const int64_t dh[3] = {nx, ny, p}, pth[2] = {nx * 8, nx * ny * 8};
    const int bht[3] = {(int)nx, TY, 1}, bhr[3] = {(int)nx, 1, 1};
    const double* lo = hlo ? hlo : xsrc;  // unused without halos: any valid map
    const double* hi = hhi ? hhi : xsrc;
    encode_tensor_map(&mp.lo_tile, lo, 3, dh, pth, bht);
    encode_tensor_map(&mp.lo_row, lo, 3, dh, pth, bhr);
    encode_tensor_map(&mp.hi_tile, hi, 3, dh, pth, bht);
    encode_tensor_map(&mp.hi_row, hi, 3, dh, pth, bhr);
  }
  const int smem = (int)(NS * ((TY + 2) * nx * (fuse ? 2 : 1) + TY * nx) * 8 + 2 * NS * 8);
  const dim3 block(32 * (TY + 1));
  const int sh = hlo ? 1 : 0;
  const StepFuse sf = fuse ? *fuse : StepFuse{};
#define PCAL_TMA_ST(KSV, XPV, FV)                                                                 \
  do {                                                                                            \
    auto kern = k_stencil_tma<KSV, XPV, TY, NS, FV>;                                             \
    PCAL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));    \
    kern<<<grid, block, smem, s->stream>>>(mp, gout, (int)nx, (int)ny, (int)nz, s->ld,           \
                                           (int)s->st_zchunk, s->fpart.p, s->pstride_f, s->bad,  \
                                           ctl, sh, (int)s->st_zpart, zmode, only_fb, sf);       \
  } while (0)
  if (fuse) {  // the stencil model only (Kohn–Sham needs ρ of all of X_{k+1} first)
    if (xp == 2) PCAL_TMA_ST(false, 2, true); else PCAL_TMA_ST(false, 4, true);
  } else if (ks) {
    if (xp == 2) PCAL_TMA_ST(true, 2, false); else PCAL_TMA_ST(true, 4, false);
  } else {
    if (xp == 2) PCAL_TMA_ST(false, 2, false); else PCAL_TMA_ST(false, 4, false);
  }
#undef PCAL_TMA_ST
  launched("k_stencil_tma");
  PCAL_CUDA(cudaGetLastError());
}

static void launch_stencil(pcal_session* s, int b, const double* u, bool ks, const Ctl* ctl) {
  const auto& m = s->model;
  const int64_t p = s->p;
  if (s->st_march) {
    const int TY = 8;
    const double* hlo = nullptr;
    const double* hhi = nullptr;
    dim3 grid((unsigned)(m.ny / TY), (unsigned)s->st_nzc, (unsigned)p);
    dim3 block(32, TY);
    const int xp = (int)ceil_div(m.nx, 32);
    const int rxp0 = m.nx % 2 == 0 && m.nx <= 64 ? 2 : m.nx % 4 == 0 && m.nx <= 128 ? 4 : 0;
    const bool tma = rxp0 && m.nx % 16 == 0 && !getenv("PCAL_NO_TMA_STENCIL");
    if (s->comm) {  // C5: exchange the boundary planes with the slab neighbours
      const int64_t nxy = m.nx * m.ny;
      double* h = s->halo.p;
      const size_t cnt = (size_t)p * nxy;
      hlo = h + 2 * cnt;
      hhi = h + 3 * cnt;
      const int64_t zp = s->st_zpart;
      // TMA stencil: the interior planes (no halo read) first, the two boundary
      // row chunks after the exchange — with NCCL the exchange runs on a side
      // stream under the interior planes; emulated ranks keep one stream
      if (tma && s->gz > 2 * zp && !getenv("PCAL_NO_HALO_OVERLAP")) {
        const bool side = s->hstream != nullptr;
        cudaStream_t hs = side ? s->hstream : s->stream;
        if (side) {
          PCAL_CUDA(cudaEventRecord(s->ev_x, s->stream));
          PCAL_CUDA(cudaStreamWaitEvent(hs, s->ev_x, 0));
        }
        const auto pack_and_exchange = [&]() {
          k_pack_planes<<<dim3((unsigned)ceil_div(nxy, 256), (unsigned)p), 256, 0, hs>>>(
              Xof(s, b), s->ld, nxy, s->gz, h, h + cnt, ctl);
          launched("k_pack_planes");
          s->comm->halo(h, h + cnt, h + 2 * cnt, h + 3 * cnt, cnt, hs);
        };
        if (side) pack_and_exchange();
        dim3 gi = grid;
        gi.y = (unsigned)ceil_div(s->gz - 2 * zp, s->st_zchunk);
        launch_stencil_tma(s, b, u, ks, ctl, rxp0, hlo, hhi, gi, 1);
        if (side) {
          PCAL_CUDA(cudaEventRecord(s->ev_h, hs));
          PCAL_CUDA(cudaStreamWaitEvent(s->stream, s->ev_h, 0));
        } else {
          pack_and_exchange();
        }
        dim3 gb = grid;
        gb.y = 2;
        launch_stencil_tma(s, b, u, ks, ctl, rxp0, hlo, hhi, gb, 2);
        return;
      }
      k_pack_planes<<<dim3((unsigned)ceil_div(nxy, 256), (unsigned)p), 256, 0, s->stream>>>(
          Xof(s, b), s->ld, nxy, s->gz, h, h + cnt, ctl);
      launched("k_pack_planes");
      s->comm->halo(h, h + cnt, h + 2 * cnt, h + 3 * cnt, cnt, s->stream);
    }
#define PCAL_MARCH(KSV, XPV)                                                                   \
  k_stencil_march<KSV, XPV, 8><<<grid, block, 0, s->stream>>>(                               \
      Xof(s, b), u, Pof(s, b), (int)m.nx, (int)m.ny, (int)s->gz, s->ld, (int)s->st_zchunk,     \
      s->fpart.p, s->pstride_f, s->bad, ctl, hlo, hhi, (int)s->st_zpart)
#define PCAL_MARCH_ROW(KSV, XPV)                                                               \
  k_stencil_march_row<KSV, XPV, 8><<<grid, block, 0, s->stream>>>(                           \
      Xof(s, b), u, Pof(s, b), (int)m.nx, (int)m.ny, (int)s->gz, s->ld, (int)s->st_zchunk,     \
      s->fpart.p, s->pstride_f, s->bad, ctl, hlo, hhi, (int)s->st_zpart)
    // rows of an even number of points ≤ 64, or a multiple of 4 ≤ 128: the
    // vectorised full-row kernel (XP consecutive points per lane); rows of a
    // multiple of 16 points (128-byte TMA rows): its TMA-staged form
    const int rxp = m.nx % 2 == 0 && m.nx <= 64 ? 2 : m.nx % 4 == 0 && m.nx <= 128 ? 4 : 0;
    if (rxp && m.nx % 16 == 0 && !getenv("PCAL_NO_TMA_STENCIL")) {
      // after the fused step only the exact-rule columns are left
      launch_stencil_tma(s, b, u, ks, ctl, rxp, hlo, hhi, grid, 0, s->grad_fused ? s->sfb : nullptr);
      s->grad_fused = false;
      return;
    }
    if (rxp && !getenv("PCAL_NO_ROW_MARCH")) {
      if (ks) {
        if (rxp == 2) PCAL_MARCH_ROW(true, 2); else PCAL_MARCH_ROW(true, 4);
      } else {
        if (rxp == 2) PCAL_MARCH_ROW(false, 2); else PCAL_MARCH_ROW(false, 4);
      }
    } else if (ks) {
      if (xp == 1) PCAL_MARCH(true, 1); else if (xp == 2) PCAL_MARCH(true, 2);
      else if (xp == 3) PCAL_MARCH(true, 3); else PCAL_MARCH(true, 4);
    } else {
      if (xp == 1) PCAL_MARCH(false, 1); else if (xp == 2) PCAL_MARCH(false, 2);
      else if (xp == 3) PCAL_MARCH(false, 3); else PCAL_MARCH(false, 4);
    }
#undef PCAL_MARCH
#undef PCAL_MARCH_ROW
    launched("k_stencil_march");
  } else {
    dim3 g((unsigned)s->st_nchunks, (unsigned)p);
    if (ks)
      k_stencil_grad<true><<<g, kStencilThreads, 0, s->stream>>>(
          Xof(s, b), u, Pof(s, b), m.nx, m.ny, m.nz, s->ld, p, s->st_chunk, s->fpart.p,
          s->pstride_f, s->bad, ctl);
    else
      k_stencil_grad<false><<<g, kStencilThreads, 0, s->stream>>>(
          Xof(s, b), u, Pof(s, b), m.nx, m.ny, m.nz, s->ld, p, s->st_chunk, s->fpart.p,
          s->pstride_f, s->bad, ctl);
    launched("k_stencil_grad");
  }
}

// DensityModel's terms after G = L·X (problems.cpp:169-203): ρ over all rows
// (the gathered X when sharded), h = L⁻¹ρ on the owned rows, G += w∘X.
static void launch_density(pcal_session* s, int b, const Ctl* ctl) {
  const bool gathered = s->comm && s->comm->size > 1;
  const int64_t ng = s->n_glob;
  k_row_sq_norms<<<(unsigned)ceil_div(ng, 256), 256, 0, s->stream>>>(
      gathered ? s->xfull.p : Xof(s, b), ng, gathered ? s->K_full : s->ld, s->p, s->rho.p, ctl);
  launched("k_row_sq_norms");
  k_density_hartree<<<(unsigned)ceil_div(s->n, 32), 256, 0, s->stream>>>(
      s->Minv.p, s->ld, s->n, ng, s->rho.p, s->h.p, ctl);
  launched("k_density_hartree");
  const int p6 = s->model.density_variant == PCAL_DENSITY_P6;
  if (s->repro) {  // density scalars per row chunk, reduced in chunk order
    k_density_apply<<<(unsigned)s->nch, 256, 0, s->stream>>>(
        Xof(s, b), Pof(s, b), s->ld, s->n, s->p, s->rho.p + s->row0, s->h.p, s->model.coeff, p6,
        s->cc.p, s->bad, ctl, s->chunk_rows);
    launched("k_density_apply");
    chunk_reduce(s, s->cc.p, 3, s->spt.p, ctl);
  } else {
    k_density_apply<<<s->sp_blocks, 256, 0, s->stream>>>(
        Xof(s, b), Pof(s, b), s->ld, s->n, s->p, s->rho.p + s->row0, s->h.p, s->model.coeff, p6,
        s->spart.p, s->bad, ctl);
    launched("k_density_apply");
  }
}

static void launch_gradient(pcal_session* s, int b, const Ctl* ctl) {
  const int64_t p = s->p;
  switch (s->model.kind) {
    case PCAL_MODEL_DENSE:
    case PCAL_MODEL_BILINEAR:
    case PCAL_MODEL_DENSITY:
      if (s->comm && s->comm->size > 1) {  // C5: every rank needs all rows of X for A·X
        const int R = s->comm->size;
        s->comm->allgather(Xof(s, b), s->xgath.p, (size_t)s->ld * s->pp, s->stream);
        k_unpack_rows<<<dim3((unsigned)ceil_div(s->ld, 256), (unsigned)s->pp, (unsigned)R), 256, 0,
                        s->stream>>>(s->xgath.p, s->ld, s->pp, (const int64_t*)s->rank_rows_d.p, R,
                                     s->xfull.p, s->K_full, ctl);
        launched("k_unpack_rows");
      }
      launch_gemm(s->grad[b], s->stream);
      if (s->model.kind == PCAL_MODEL_BILINEAR) launch_gemm(s->grad2[b], s->stream);  // (A·X)·B
      if (s->model.kind == PCAL_MODEL_DENSITY) launch_density(s, b, ctl);
      break;
    case PCAL_MODEL_STENCIL: {
      launch_stencil(s, b, s->V.p, false, ctl);
      break;
    }
    case PCAL_MODEL_KOHN_SHAM: {
      const int64_t n = s->n;
      const unsigned nb = (unsigned)ceil_div(n, 256);
      const auto& m = s->model;
      k_row_sq_norms<<<nb, 256, 0, s->stream>>>(Xof(s, b), n, s->ld, p, s->rho.p, ctl);
      launched("k_row_sq_norms");
      if (s->comm) {  // C5: the spectral solve needs the full density
        const int R = s->comm->size;
        s->comm->allgather(s->rho.p, s->rho_gath.p, (size_t)s->ld, s->stream);
        k_unpack_rows<<<dim3((unsigned)ceil_div(s->ld, 256), 1, (unsigned)R), 256, 0, s->stream>>>(
            s->rho_gath.p, s->ld, 1, (const int64_t*)s->rank_rows_d.p, R, s->rho.p, s->n_glob,
            ctl);
        launched("k_unpack_rows");
      }
      const unsigned ng = (unsigned)ceil_div(s->n_glob, 256);
      k_axis_transform<<<ng, 256, 0, s->stream>>>(s->rho.p, s->tmpa.p, s->qx.p, m.nx, m.nx, m.ny,
                                                  m.nz, 0, 1, ctl);
      launched("k_axis_transform");
      k_axis_transform<<<ng, 256, 0, s->stream>>>(s->tmpa.p, s->tmpb.p, s->qy.p, m.ny, m.nx, m.ny,
                                                  m.nz, 1, 1, ctl);
      launched("k_axis_transform");
      k_axis_transform<<<ng, 256, 0, s->stream>>>(s->tmpb.p, s->tmpa.p, s->qz.p, m.nz, m.nx, m.ny,
                                                  m.nz, 2, 1, ctl);
      launched("k_axis_transform");
      k_spectral_divide<<<ng, 256, 0, s->stream>>>(s->tmpa.p, s->lx.p, s->ly.p, s->lz.p, m.nx,
                                                   m.ny, m.nz, ctl);
      launched("k_spectral_divide");
      k_axis_transform<<<ng, 256, 0, s->stream>>>(s->tmpa.p, s->tmpb.p, s->qz.p, m.nz, m.nx, m.ny,
                                                  m.nz, 2, 0, ctl);
      launched("k_axis_transform");
      k_axis_transform<<<ng, 256, 0, s->stream>>>(s->tmpb.p, s->tmpa.p, s->qy.p, m.ny, m.nx, m.ny,
                                                  m.nz, 1, 0, ctl);
      launched("k_axis_transform");
      k_axis_transform<<<ng, 256, 0, s->stream>>>(s->tmpa.p, s->h.p, s->qx.p, m.nx, m.nx, m.ny,
                                                  m.nz, 0, 0, ctl);
      launched("k_axis_transform");
      if (s->repro) {  // density scalars per row chunk, reduced in chunk order
        k_ks_potential<<<(unsigned)s->nch, 256, 0, s->stream>>>(
            s->V.p, s->rho.p + s->row0, s->h.p + s->row0, s->u.p, n, s->c_xc, s->cc.p, ctl,
            s->chunk_rows);
        launched("k_ks_potential");
        chunk_reduce(s, s->cc.p, 3, s->spt.p, ctl);
      } else {
        k_ks_potential<<<s->sp_blocks, 256, 0, s->stream>>>(s->V.p, s->rho.p + s->row0,
                                                            s->h.p + s->row0, s->u.p, n, s->c_xc,
                                                            s->spart.p, ctl);
        launched("k_ks_potential");
      }
      launch_stencil(s, b, s->u.p, true, ctl);
      break;
    }
    case PCAL_MODEL_DEVICE_CALLBACK: {  // the caller's own gradient, enqueued on our stream
      const int rc = s->model.grad(Xof(s, b), s->ld, s->n, p, Pof(s, b), s->fdev.p,
                                   (void*)s->stream, s->model.grad_ctx);
      if (rc != 0)
        throw Error(PCAL_E_EVALUATION, "gradient callback failed (" + std::to_string(rc) + ")");
      k_check_finite<<<(unsigned)std::min<int64_t>(4 * 148, ceil_div(s->n * p, 256)), 256, 0,
                       s->stream>>>(Pof(s, b), s->n, s->ld, p, s->bad, ctl);
      launched("k_check_finite");
      break;
    }
    default:
      throw Error(PCAL_E_UNSUPPORTED, "unsupported model kind");
  }
}

// eval_iterate(X) for pair b followed by the PCAL multiplier/gradient branch:
// G, [GᵀX; XᵀX], W, C, g_plam = G − XW + βXC (into P), d, kkt, feas, f.
static void launch_eval(pcal_session* s, int b, int mode, const Ctl* ctl_guard) {
  cudaStream_t st = s->stream;
  mark(s, 1);
  launch_gradient(s, b, ctl_guard);
  mark(s, 2);
  launch_gemm(s->gram[b], st);
  if (s->repro) gram_reduce(s, s->gram[b], 0);  // C1
  {
    const bool alm = s->alg == PCAL_ALG_ALM;
    // Λ: W at the start point; dual ascent updates it every evaluation, ALM only
    // at its multiplier updates (mode 3)
    const int lam_mode = mode == 1 ? 1 : alm ? (mode == 3 ? 0 : 2) : 0;
    const int mc = (s->alg == PCAL_ALG_PLAMDA || s->alg == PCAL_ALG_PCALDA || alm) ? MC_DA
                   : s->alg == PCAL_ALG_MOPTQR                               ? MC_MOPTQR
                                                                             : MC_PCAL;
    k_small_pxp<<<s->cp_blocks, kStreamThreads, 0, st>>>(
        s->gr.p, s->pp, s->p, s->mcat.p, s->pp, s->cpart.p, mc, s->beta, s->lam.p, lam_mode,
        ctl_guard, s->sym_gx ? 1 : 0, s->xm[b].size == CFG_XMS ? 1 : 0,
        s->xm1 ? Xm1Out{s->m1.p, s->wmat.p, s->cmat.p} : Xm1Out{nullptr, nullptr, nullptr});
  }
  launched("k_small_pxp");
  if (s->xm1) {  // C² and the identity's inner products
    launch_gemm(s->c2plan, st);
    k_kkt_corr<<<s->cp_blocks, kStreamThreads, 0, st>>>(s->wmat.p, s->cmat.p, s->c2m.p, s->pp,
                                                        s->p, s->kcp.p, ctl_guard);
    launched("k_kkt_corr");
  }
  mark(s, 3);
  launch_gemm(s->xm[b], st);
  // column sums of the f / kkt² (XM1: P²) / d partials; `gate` non-null: the
  // gated recomputation after the XM1 fallback (collectives still run, so every
  // rank issues the same sequence; the gated kernels keep the previous values)
  auto colsums = [&](const int32_t* gate) {
    if (s->repro) {  // C2: per-chunk column sums, gathered and summed in chunk order
      const bool dform =
          s->alg == PCAL_ALG_PCAL && s->cfg.multiplier_rule == PCAL_MULT_PCAL_FORMULA;
      const int64_t wm_xm = cfg_info(pick_size(2 * s->pp)).WM;
      ChunkColArgs a{};
      a.in[0] = s->fpart.p;
      a.nrows[0] = s->nrb_f;
      a.stride[0] = s->pstride_f;
      a.rpc[0] = dense_family(s->model.kind) ? s->chunk_rows / cfg_info(pick_size(s->pp)).WM
                                             : s->model.ny / 8;
      a.in[1] = s->kpart.p;
      const bool alm = s->alg == PCAL_ALG_ALM;
      a.in[2] = (dform || alm) ? s->dpart.p : nullptr;
      for (int w = 1; w < 3; ++w) {
        a.nrows[w] = s->nrb_xm;
        a.stride[w] = s->pstride_xm;
        a.rpc[w] = s->chunk_rows / wm_xm;
      }
      a.out = s->cc.p;
      a.p = s->p;
      a.nch = s->nch;
      a.gate = gate;
      k_chunk_colsum3<<<dim3((unsigned)s->p, 3), 128, 0, st>>>(a, ctl_guard);
      launched("k_chunk_colsum3");
      // + the ranks' failure flags in the same all-gather, so every rank stops
      // together (exact counts)
      if (!gate) {
        k_flags<<<1, 1, 0, st>>>(s->ctl, s->bad, s->cc.p + s->nch_max * 3 * s->p);
        launched("k_flags");
      }
      chunk_reduce(s, s->cc.p, 3 * s->p, s->fkd[b].p, ctl_guard, 2);
      if (alm) {
        k_alm_split<<<1, 256, 0, st>>>(Dvec(s, b), s->glcol.p, s->p, ctl_guard);
        launched("k_alm_split");
      }
    } else {
      launch_colsums(s, s->fpart.p, s->nrb_f, s->kpart.p, s->dpart.p,
                     s->xm1 && !gate ? ceil_div(s->n, (int64_t)cfg_info(CFG_XM1).BM) : s->nrb_xm,
                     Fcol(s, b), Kcol(s, b), Dvec(s, b), ctl_guard, gate);
    }
  };
  colsums(nullptr);
  if (s->xm1) {
    k_kkt_gate<<<1, 256, 0, st>>>(s->kcp.p, s->cp_blocks, Kcol(s, b), s->p, s->beta, s->xm1_gate,
                                  s->kfb, s->kk.p, ctl_guard);
    launched("k_kkt_gate");
    // the identity cancelled too much: kkt = P − X·(βC) directly (gated: no-ops otherwise)
    launch_gemm(s->xmfb[b], st);
    colsums(s->kfb);
  }
  FinishArgs fa{};
  fa.fcol = Fcol(s, b);
  fa.kcol = Kcol(s, b);
  fa.flags = s->comm ? s->fkd[b].p + 3 * s->p : nullptr;
  fa.cpart = s->cpart.p;
  fa.ncp = s->cp_blocks;
  fa.spart = s->repro ? s->spt.p : s->spart.p;
  fa.nsp = s->repro ? 1 : s->sp_blocks;
  fa.model = s->model.kind;
  fa.p = s->p;
  fa.mode = mode;
  fa.trace = s->trace.p;
  fa.bad = s->bad;
  fa.c_xc = s->c_xc;
  fa.fdev = s->fdev.p;
  fa.coeff = s->model.coeff;
  fa.p6 = s->model.density_variant == PCAL_DENSITY_P6;
  fa.glcol = s->alg == PCAL_ALG_ALM ? s->glcol.p : nullptr;
  fa.k2_id = s->xm1 ? s->kk.p : nullptr;
  fa.k2_fb = s->kfb;
  k_finish_eval<<<1, 256, 0, st>>>(fa, s->ctl, s->post.p);
  launched("k_finish_eval");
  mark(s, 4);
  if (s->pev_on) {
    PCAL_CUDA(cudaEventSynchronize(s->pev[4]));
    float g = 0, gm = 0, xm = 0;
    PCAL_CUDA(cudaEventElapsedTime(&g, s->pev[1], s->pev[2]));
    PCAL_CUDA(cudaEventElapsedTime(&gm, s->pev[2], s->pev[3]));
    PCAL_CUDA(cudaEventElapsedTime(&xm, s->pev[3], s->pev[4]));
    if (s->timers) {  // CategoryTimers: products inside evaluate count as func (report.hpp:66-72)
      s->timers->func += g * 1e-3;
      s->timers->blas3 += (gm + xm) * 1e-3;
    }
    s->prof_ms[1] += g;
    s->prof_ms[2] += gm;
    s->prof_ms[3] += xm;
  }
}

// L = chol(B) and T = (L⁻¹)ᵀ with the pivot floor of the first Gram; status = 0 on failure.
static void launch_chol_trinv(cudaStream_t st, const double* b, int64_t ldb, int64_t p,
                              const double* f2, double* l, int64_t ldl, double* t, int64_t ldt,
                              int32_t* status, const int32_t* prev_ok, const Ctl* ctl) {
  if (p <= kCholSmemP) {
    const size_t smem = sizeof(double) * p * p;
    static bool attr = false;
    if (!attr) {
      PCAL_CUDA(cudaFuncSetAttribute(k_chol_trinv_small,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(sizeof(double) * kCholSmemP * kCholSmemP)));
      attr = true;
    }
    k_chol_trinv_small<<<1, 1024, smem, st>>>(b, ldb, (int)p, f2, t, ldt, status, prev_ok, ctl);
    launched("k_chol_trinv_small");
    return;
  }
  if (p <= kCholWideP) {  // l holds Lᵀ here (rows of L contiguous)
    k_cholesky_wide<<<1, 1024, 0, st>>>(b, ldb, (int)p, f2, l, ldl, status, prev_ok, ctl);
    launched("k_cholesky_wide");
    const unsigned g = (unsigned)ceil_div(p, 8);
    if (p <= 256) k_trinv_wide<8><<<g, 256, 0, st>>>(l, ldl, (int)p, t, ldt, status);
    else if (p <= 512) k_trinv_wide<16><<<g, 256, 0, st>>>(l, ldl, (int)p, t, ldt, status);
    else if (p <= 1024) k_trinv_wide<32><<<g, 256, 0, st>>>(l, ldl, (int)p, t, ldt, status);
    else k_trinv_wide<kCholWideP / 32><<<g, 256, 0, st>>>(l, ldl, (int)p, t, ldt, status);
    launched("k_trinv_wide");
    return;
  }
  k_cholesky<<<1, 1024, 0, st>>>(b, ldb, p, f2, l, ldl, status, prev_ok, ctl);
  launched("k_cholesky");
  k_trinv_t<<<(unsigned)ceil_div(p, 128), 128, 0, st>>>(l, ldl, p, t, ldt, status);
  launched("k_trinv_t");
}

// One PCAL iteration from X_k in pair b to X_{k+1} in pair 1−b (solver.cpp:385-438).
// MOptQR retraction inside the iteration graph (solver.cpp:415-418): Z in
// X(nb) → Q = orthonormalize(Z) in X(nb) by CholeskyQR2 with status-gated
// GEMMs (Q1 scratch in P(nb), dead until the next gradient) and the MGS2
// fallback kernel, which only runs when a Cholesky pass failed.
static void launch_retraction(pcal_session* s, int nb) {
  cudaStream_t st = s->stream;
  const int64_t p = s->p, pp = s->pp;
  int32_t* ok1 = s->orth_status;
  int32_t* ok2 = s->orth_status + 1;
  launch_gemm(s->rq_gram_z[nb], st);
  k_sym_fro2<<<1, 1024, 0, st>>>(s->orth_b.p, pp, p, s->orth_f2.p);
  launched("k_sym_fro2");
  launch_chol_trinv(st, s->orth_b.p, pp, p, s->orth_f2.p, s->orth_l.p, pp, s->orth_t.p, pp, ok1,
                    nullptr, s->ctl);
  launch_gemm(s->rq_mul1[nb], st);
  launch_gemm(s->rq_gram_q[nb], st);
  launch_chol_trinv(st, s->orth_b.p, pp, p, s->orth_f2.p, s->orth_l.p, pp, s->orth_t.p, pp, ok2,
                    ok1, s->ctl);
  launch_gemm(s->rq_mul2[nb], st);
  k_mgs2_gated<<<1, 1024, 0, st>>>(Xof(s, nb), s->n, s->ld, p, s->orth_f2.p, ok1, ok2,
                                   s->orth_status + 2, s->ctl);
  launched("k_mgs2_gated");
}

// One iteration from X_k in pair b to X_{k+1} in pair 1−b (solver.cpp:369-439).
static void launch_iteration(pcal_session* s, int b) {
  cudaStream_t st = s->stream;
  const int nb = 1 - b;
  // PLAM, PLAM-DA and the MOptQR pre-retraction step do not normalise columns
  const int plain = !(s->alg == PCAL_ALG_PCAL || s->alg == PCAL_ALG_PCALDA);
  mark(s, 0);
  if (!s->comm && s->fused_step) {  // one cooperative kernel for the whole step phase
    StepArgs a{Xof(s, b), Pof(s, b), Xof(s, nb), Pof(s, nb), Dvec(s, b), Dvec(s, nb),
               Xof(s, nb), s->bbpart.p, s->npart.p, s->n, s->ld, s->p, s->up_chunk,
               s->up_nchunks, s->n_glob, plain};
    Ctl* c = s->ctl;
    void* args[] = {&a, &c};
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3((unsigned)s->bb_blocks);
    lc.blockDim = dim3(kStreamThreads);
    lc.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeCooperative;
    attr.val.cooperative = 1;
    lc.attrs = &attr;
    lc.numAttrs = 1;
    PCAL_CUDA(cudaLaunchKernelExC(&lc, (const void*)k_step_fused, args));
    launched("k_step_fused");
  } else if (s->repro && !plain && !getenv("PCAL_TWO_PASS_NORMALIZE")) {
    // C3 + C4 of the one-pass normalised step: the per-chunk stepsize AND
    // column-norm expansion sums (a, b, c) in one all-gather; flagged columns
    // take the exact rule with their chunk-reduced ‖z_j‖² (a second, tiny
    // all-gather that every rank issues every iteration)
    const unsigned nc = (unsigned)s->nch;
    dim3 gu(nc, (unsigned)s->p);
    k_bb_cols<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Pof(s, b), Xof(s, nb), Pof(s, nb),
                                             Dvec(s, b), Dvec(s, nb), s->n, s->ld, s->p,
                                             s->chunk_rows, s->colpart.p, s->ctl);
    launched("k_bb_cols");
    chunk_reduce(s, s->colpart.p, 6 * s->p, s->bbt.p, s->ctl);  // [j·6 + q], chunk order
    k_bb_cols_sum<<<1, kStreamThreads, 0, st>>>(s->bbt.p, s->p, s->bbpart.p, s->ctl);
    launched("k_bb_cols_sum");
    k_eta<<<1, kStreamThreads, 0, st>>>(s->ctl, s->bbpart.p, 1);
    launched("k_eta");
    k_colscale<<<(unsigned)ceil_div(s->p, 128), 128, 0, st>>>(s->bbt.p, 1, s->p, s->sinv.p,
                                                              s->sfb, s->ctl);
    launched("k_colscale");
    k_update_norm<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Pof(s, b), Dvec(s, b), Xof(s, nb),
                                                 s->n, s->ld, s->p, s->chunk_rows, s->cc.p,
                                                 s->sinv.p, s->sfb, s->ctl, s->cc.p + s->p,
                                                 2 * s->p);
    launched("k_update_norm");
    chunk_reduce(s, s->cc.p, 2 * s->p, s->nrm.p, s->ctl);
    k_normalize<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Xof(s, nb), s->n, s->ld, s->p,
                                               s->chunk_rows, s->nch, s->cc.p, s->nrm.p, s->row0,
                                               s->n_glob, plain, s->ctl, s->sfb);
    launched("k_normalize");
  } else if (s->repro) {  // C3/C4 with chunked, rank-count invariant reductions
    const unsigned nc = (unsigned)s->nch;
    k_bb_chunk<<<dim3(nc, (unsigned)s->p), kStreamThreads, 0, st>>>(
        Xof(s, b), Pof(s, b), Xof(s, nb), Pof(s, nb), Dvec(s, b), Dvec(s, nb), s->n, s->ld, s->p,
        s->chunk_rows, s->cc.p, s->ctl);
    launched("k_bb_chunk");
    chunk_reduce(s, s->cc.p, 3 * s->p, s->bbt.p, s->ctl);
    k_eta<<<1, kStreamThreads, 0, st>>>(s->ctl, s->bbt.p, (int)s->p);
    launched("k_eta");
    dim3 gu(nc, (unsigned)s->p);
    k_update<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Pof(s, b), Dvec(s, b), Xof(s, nb), s->n,
                                            s->ld, s->p, s->chunk_rows, s->cc.p, s->cc.p + s->p,
                                            s->ctl, 2 * s->p);
    launched("k_update");
    chunk_reduce(s, s->cc.p, 2 * s->p, s->nrm.p, s->ctl);
    k_normalize<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Xof(s, nb), s->n, s->ld, s->p,
                                               s->chunk_rows, s->nch, s->cc.p, s->nrm.p, s->row0,
                                               s->n_glob, plain, s->ctl);
    launched("k_normalize");
  } else if (!s->comm && !plain && !getenv("PCAL_TWO_PASS_NORMALIZE")) {
    // normalised step in one pass over Z (pcal_kernels.cuh k_bb_cols): the
    // stepsize kernel also sums x², x·gl, gl² per column, so ‖z_j‖ is known
    // before z is formed; flagged columns fall back to the exact two-pass rule
    dim3 gu((unsigned)s->up_nchunks, (unsigned)s->p);
    k_bb_cols<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Pof(s, b), Xof(s, nb), Pof(s, nb),
                                             Dvec(s, b), Dvec(s, nb), s->n, s->ld, s->p,
                                             s->up_chunk, s->colpart.p, s->ctl);
    launched("k_bb_cols");
    k_bb_cols_sum<<<1, kStreamThreads, 0, st>>>(s->colpart.p, s->up_nchunks * s->p,
                                                s->bbpart.p, s->ctl);
    launched("k_bb_cols_sum");
    k_eta<<<1, kStreamThreads, 0, st>>>(s->ctl, s->bbpart.p, 1);
    launched("k_eta");
    k_colscale<<<(unsigned)ceil_div(s->p, 128), 128, 0, st>>>(s->colpart.p, s->up_nchunks, s->p,
                                                              s->sinv.p, s->sfb, s->ctl);
    launched("k_colscale");
    if (s->step_stencil) {  // X_{k+1} and G_{k+1} in one pass; flagged columns below
      const auto& m = s->model;
      const StepFuse sf{Xof(s, nb), Dvec(s, b), s->sinv.p, s->sfb, s->ctl};
      dim3 grid((unsigned)(m.ny / 8), (unsigned)s->st_nzc, (unsigned)s->p);
      const int rxp = m.nx % 2 == 0 && m.nx <= 64 ? 2 : 4;
      launch_stencil_tma(s, b, s->V.p, false, s->ctl, rxp, nullptr, nullptr, grid, 0, nullptr,
                         &sf);
      s->grad_fused = true;
    }
    k_update_norm<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Pof(s, b), Dvec(s, b), Xof(s, nb),
                                                 s->n, s->ld, s->p, s->up_chunk, s->npart.p,
                                                 s->sinv.p, s->sfb, s->ctl, nullptr, 0,
                                                 s->step_stencil ? 1 : 0);
    launched("k_update_norm");
    k_normalize<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Xof(s, nb), s->n, s->ld, s->p,
                                               s->up_chunk, s->up_nchunks, s->npart.p, nullptr,
                                               s->row0, s->n_glob, plain, s->ctl, s->sfb);
    launched("k_normalize");
  } else {
    k_bb_partials<<<s->bb_blocks, kStreamThreads, 0, st>>>(Xof(s, b), Pof(s, b), Xof(s, nb),
                                                           Pof(s, nb), Dvec(s, b), Dvec(s, nb),
                                                           s->ld, s->p, s->bbpart.p, s->ctl);
    launched("k_bb_partials");
    if (s->comm) s->comm->allreduce(s->bbpart.p, (size_t)3 * s->bb_blocks, st);  // C3
    k_eta<<<1, kStreamThreads, 0, st>>>(s->ctl, s->bbpart.p, s->bb_blocks);
    launched("k_eta");
    dim3 gu((unsigned)s->up_nchunks, (unsigned)s->p);
    k_update<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Pof(s, b), Dvec(s, b), Xof(s, nb), s->n,
                                            s->ld, s->p, s->up_chunk, s->npart.p,
                                            s->comm ? s->xpart.p : nullptr, s->ctl);
    launched("k_update");
    const double* nrm = nullptr;
    if (s->comm && !plain) {  // C4: global column norms
      k_norm_reduce<<<(unsigned)ceil_div(s->p, 128), 128, 0, st>>>(s->npart.p, s->xpart.p,
                                                                   s->up_nchunks, s->p, s->nrm.p,
                                                                   s->ctl);
      launched("k_norm_reduce");
      s->comm->allreduce(s->nrm.p, (size_t)2 * s->p, st);
      nrm = s->nrm.p;
    } else if (s->comm) {
      nrm = s->nrm.p;  // plain steps: only marks the sharded (collective) divergence rule
    }
    k_normalize<<<gu, kStreamThreads, 0, st>>>(Xof(s, b), Xof(s, nb), s->n, s->ld, s->p,
                                               s->up_chunk, s->up_nchunks, s->npart.p, nrm,
                                               s->row0, s->n_glob, plain, s->ctl);
    launched("k_normalize");
  }
  PCAL_CUDA(cudaGetLastError());
  if (s->alg == PCAL_ALG_MOPTQR) launch_retraction(s, nb);
  mark(s, 5);
  launch_eval(s, nb, 0, s->ctl);
  PCAL_CUDA(cudaGetLastError());
  if (s->pev_on) {
    float a = 0;
    PCAL_CUDA(cudaEventElapsedTime(&a, s->pev[0], s->pev[5]));
    s->prof_ms[0] += a;
    s->prof_iters += 1;
  }
}

// GEMM configuration of X·[W|C] (its partial row-block is xm_row_block()).
// XM1 (P = G − X·M1, half the flops): PCAL / PLAM on one GPU with p ≥ 128;
// PCAL_XM_TWO_BLOCK=1 keeps the X·[W|C] product.
static bool xm1_mode(const pcal_session* s) {
  return (s->alg == PCAL_ALG_PCAL || s->alg == PCAL_ALG_PLAM) && pick_size(s->pp) == CFG_BIG &&
         !getenv("PCAL_XM_TWO_BLOCK") && !getenv("PCAL_NO_TMEM_EPI") && !getenv("PCAL_XM_TMEM");
}
static int xm_config(const pcal_session* s) {
  const int xsz = pick_size(2 * s->pp);
  if (xm1_mode(s)) return CFG_XM1;  // whole 64-row tiles: reproducible as well
  if (xsz != CFG_BIG || s->repro || getenv("PCAL_NO_TMEM_EPI")) return xsz;
  return getenv("PCAL_XM_TMEM") ? (int)CFG_XMT : (int)CFG_XMS;
}
static int64_t xm_row_block(const pcal_session* s) {
  const int c = xm_config(s);
  // staged: one partial per tile row (XM1: 64 rows = the fallback GEMM's warp rows)
  return (c == CFG_XMS || c == CFG_XM1) ? cfg_info(c).BM : cfg_info(c).WM;
}

static void build_plans(pcal_session* s) {
  const int dev = s->device;
  const int64_t pp = s->pp, ld = s->ld, n = s->n;
  if (s->alg == PCAL_ALG_MOPTQR) {
    for (int b = 0; b < 2; ++b) {
      auto gram = [&](GemmPlan& g, const double* a) {
        plan_gemm(g, dev, pick_size(pp), A_KCONTIG, EPI_STORE, pp, pp, ld, 0);
        g.args.A = g.args.B = a;
        g.args.lda = g.args.ldb = ld;
        g.args.ep.C = s->orth_b.p;
        g.args.ep.ldc = pp;
        g.args.ep.m_store = g.args.ep.n_store = pp;
        g.args.ctl = s->ctl;
      };
      auto mul = [&](GemmPlan& g, const double* a, double* out, const int32_t* gate) {
        plan_gemm(g, dev, pick_size(pp), A_MCONTIG, EPI_STORE, n, pp, pp);
        g.args.A = a;
        g.args.lda = ld;
        g.args.B = s->orth_t.p;
        g.args.ldb = pp;
        g.args.ep.C = out;
        g.args.ep.ldc = ld;
        g.args.ep.m_store = n;
        g.args.ep.n_store = s->p;
        g.args.ctl = s->ctl;
        g.args.gate = gate;
      };
      gram(s->rq_gram_z[b], Xof(s, b));
      mul(s->rq_mul1[b], Xof(s, b), Pof(s, b), s->orth_status);
      gram(s->rq_gram_q[b], Pof(s, b));
      s->rq_gram_q[b].args.gate = s->orth_status;
      mul(s->rq_mul2[b], Pof(s, b), Xof(s, b), s->orth_status + 1);
    }
  }
  for (int b = 0; b < 2; ++b) {
    // gradient (dense family): G = A·X, A ldA×ldA (MCONTIG), X ld×pp; the
    // bilinear model stores A·X and applies B in a second GEMM with the epilogue
    if (dense_family(s->model.kind)) {
      GemmPlan& g = s->grad[b];
      const int sz = pick_size(pp);
      const bool bil = s->model.kind == PCAL_MODEL_BILINEAR;
      const int epi = bil ? EPI_STORE : EPI_GRAD;
      if (s->repro) {  // fixed K segments (chosen from global sizes in session_create)
        plan_gemm(g, dev, sz, A_MCONTIG, epi, n, pp, s->K_full, -1, 0, s->grad_splits);
      } else {
        plan_gemm(g, dev, sz, A_MCONTIG, epi, n, pp, s->K_full);
      }
      g.args.A = s->A.p;
      g.args.lda = s->ldA;
      g.args.a_stream = 1;  // A streams through once per iteration: keep X resident in L2
      const bool gathered = s->comm && s->comm->size > 1;
      g.args.B = gathered ? s->xfull.p : Xof(s, b);
      g.args.ldb = gathered ? s->K_full : ld;
      EpiParams& e = g.args.ep;
      e.G = Pof(s, b);
      e.X = Xof(s, b);
      e.g0 = s->g0.p;
      e.ld = ld;
      e.fpart = s->fpart.p;
      e.pstride = s->pstride_f;
      e.bad = s->bad;
      e.n = n;
      e.p = s->p;
      g.args.ctl = s->ctl;
      if (bil) {  // T = A·X (all pp columns: X's padding is zero), then G = T·B
        e.C = s->tb.p;
        e.ldc = ld;
        e.m_store = n;
        e.n_store = pp;
        GemmPlan& g2 = s->grad2[b];
        plan_gemm(g2, dev, sz, A_MCONTIG, EPI_GRAD, n, pp, pp, -1, 0, s->repro ? 1 : 0);
        g2.args.A = s->tb.p;
        g2.args.lda = ld;
        g2.args.B = s->Bm.p;
        g2.args.ldb = pp;
        g2.args.ep = e;
        g2.args.ep.C = nullptr;
        g2.args.ctl = s->ctl;
      }
    }
    // Gram: [P|X]ᵀ·X — A = pair (KCONTIG, rows m < 2pp), B = X, K = ld
    {
      GemmPlan& g = s->gram[b];
      if (s->repro)  // one partial per row chunk, summed across ranks in chunk order
        plan_gemm(g, dev, pick_size(pp), A_KCONTIG, EPI_STORE, 2 * pp, pp,
                  s->nch * s->chunk_rows, pp, 0, (int)(s->nch * s->gram_sub), true,
                  (int)(s->nch_max * s->gram_sub), s->sym_gx);
      else
        plan_gemm(g, dev, pick_size(pp), A_KCONTIG, EPI_STORE, 2 * pp, pp, ld, pp, 0, 0, false,
                  0, s->sym_gx);
      g.args.A = s->pair[b].p;
      g.args.lda = ld;
      g.args.B = Xof(s, b);
      g.args.ldb = ld;
      g.args.ep.C = s->gr.p;
      g.args.ep.ldc = 2 * pp;
      g.args.ep.m_store = 2 * pp;
      g.args.ep.n_store = pp;
      g.args.ctl = s->ctl;
    }
    // X·[W|C] with the PCAL epilogue: A = X (MCONTIG, K = pp), B = mcat (pp × 2pp)
    if (s->xm1) {  // P = G − X·M1 (B = M1, pp × pp), fallback X·[βC|C] gated by kfb
      GemmPlan& g = s->xm[b];
      plan_gemm(g, dev, CFG_XM1, A_MCONTIG, EPI_XM, n, pp, pp);
      g.args.A = Xof(s, b);
      g.args.lda = ld;
      g.args.B = s->m1.p;
      g.args.ldb = pp;
      EpiParams& e = g.args.ep;
      e.G = Pof(s, b);
      e.X = Xof(s, b);
      e.ld = ld;
      e.kpart = s->kpart.p;
      e.dpart = s->dpart.p;
      e.pstride = s->pstride_xm;
      e.n = n;
      e.p = s->p;
      g.args.ctl = s->ctl;
      GemmPlan& f = s->xmfb[b];
      plan_gemm(f, dev, CFG_BIG, A_MCONTIG, EPI_XM, n, 2 * pp, pp, -1, 0,
                s->repro ? 1 : 0);  // reproducible: whole tiles, no K split
      f.args.A = Xof(s, b);
      f.args.lda = ld;
      f.args.B = s->mcat.p;
      f.args.ldb = pp;
      f.args.ep = e;
      f.args.ep.beta = s->beta;  // kkt = P − X·(βC); P = kkt + β·XC
      f.args.ctl = s->ctl;
      f.args.gate = s->kfb;
      continue;
    }
    {
      GemmPlan& g = s->xm[b];
      // wide outputs: 128 × 64 tiles whose fused epilogue reads TMA-staged G / X
      // (gemm_xm_staged); PCAL_XM_TMEM=1 selects the TMEM-staged epilogue
      // warpgroup instead (gemm_xm_tmem), PCAL_NO_TMEM_EPI=1 the plain fused one
      const int xsz = xm_config(s);
      plan_gemm(g, dev, xsz, A_MCONTIG, EPI_XM, n, 2 * pp, pp, -1, 0,
                s->repro ? 1 : 0);  // reproducible: whole tiles, no K split
      g.args.A = Xof(s, b);
      g.args.lda = ld;
      g.args.B = s->mcat.p;
      g.args.ldb = pp;
      EpiParams& e = g.args.ep;
      e.G = Pof(s, b);
      e.X = Xof(s, b);
      e.ld = ld;
      e.kpart = s->kpart.p;
      e.dpart = s->dpart.p;
      e.pstride = s->pstride_xm;
      // PCAL/PLAM: P = (G − XW) + β·XC; dual ascent / MOptQR: P = G + X·M
      e.d_sq = s->alg == PCAL_ALG_ALM;
      e.p_from_g = (s->alg == PCAL_ALG_PLAMDA || s->alg == PCAL_ALG_PCALDA || e.d_sq ||
                    s->alg == PCAL_ALG_MOPTQR);
      e.beta = e.p_from_g ? 1.0 : s->beta;
      e.n = n;
      e.p = s->p;
      g.args.ctl = s->ctl;
    }
  }
  if (s->xm1) {  // C² = C·C (C symmetric, pp × pp, zero padded)
    plan_gemm(s->c2plan, dev, pick_size(pp), A_MCONTIG, EPI_STORE, pp, pp, pp);
    GemmArgs& a = s->c2plan.args;
    a.A = a.B = s->cmat.p;
    a.lda = a.ldb = pp;
    a.ep.C = s->c2m.p;
    a.ep.ldc = pp;
    a.ep.m_store = a.ep.n_store = pp;
    a.ctl = s->ctl;
  }
  if (s->repro) tree_setup(s, 0, s->gram_sub, s->gram[0].ntasks);
}


// Fixed global row chunks of the sharded path: every row
// reduction is taken per chunk and the chunk partials are summed in global
// chunk order, so results are bitwise independent of the number of ranks.
//   dense: Q = ⌈n/64⌉ rounded up to the row-block size a (64 for p > 32,
//          else 32: chunk boundaries fall on GEMM warp row-blocks);
//   grid models: Zc = ⌈nz/64⌉ whole z-planes (Q = Zc·nx·ny rows).
static bool is_grid(int32_t kind) {
  return kind == PCAL_MODEL_STENCIL || kind == PCAL_MODEL_KOHN_SHAM;
}

static void chunking(const pcal_model_desc& m, int64_t* Q, int64_t* NC, int64_t* Zc) {
  if (!is_grid(m.kind)) {
    const int64_t a = padded_p(m.p) >= 64 ? 64 : 32;
    *Q = round_up(ceil_div(m.n, 64), a);
    *NC = ceil_div(m.n, *Q);
    *Zc = 0;
  } else {
    *Zc = ceil_div(m.nz, 64);
    *NC = ceil_div(m.nz, *Zc);
    *Q = *Zc * m.nx * m.ny;
  }
}

// Row partition of the sharded path: rank r owns the chunks
// [⌊r·NC/R⌋, ⌊(r+1)·NC/R⌋) — whole z-planes for the grid models.
static void partition(const pcal_model_desc& m, int R, int r, int64_t* row0, int64_t* rows,
                      int64_t* z0, int64_t* nzl) {
  int64_t Q, NC, Zc;
  chunking(m, &Q, &NC, &Zc);
  if (R > NC)
    throw Error(PCAL_E_PARAMETER, "more ranks than row chunks (" + std::to_string(NC) + ")");
  const int64_t c0 = (int64_t)r * NC / R, c1 = (int64_t)(r + 1) * NC / R;
  if (!is_grid(m.kind)) {
    *row0 = c0 * Q;
    *rows = std::min(c1 * Q, m.n) - *row0;
    *z0 = 0;
    *nzl = 0;
  } else {
    *z0 = c0 * Zc;
    *nzl = std::min(c1 * Zc, m.nz) - *z0;
    *row0 = *z0 * m.nx * m.ny;
    *rows = *nzl * m.nx * m.ny;
  }
}

// Segment counts of the reproducible GEMM schedules.  They may depend on
// global sizes only (never on the rank count), so pick the count whose
// modelled time exceeds the ideal (perfectly balanced, no partials) by the
// least over R ∈ {1, 2, 4, 8}.  Model per CTA: ⌈units/148⌉ segments, each
// costing its DMMA time (34 TF/s FP64 over 148 SMs) plus writing and
// re-reading one BM×BN partial at the SM's share of 6.5 TB/s.
static int best_segments(int smax, int64_t nc, int bm, int bn,
                         const std::function<double(int, int)>& units,
                         const std::function<double(int)>& kseg, bool always_store) {
  const double G = 148.0, f_sm = 34e12 / G, bw_sm = 6.5e12 / G;
  const double t_store = 2.0 * bm * bn * 8.0 / bw_sm;
  auto tseg = [&](int S) { return 2.0 * bm * bn * kseg(S) / f_sm; };
  int best = 1;
  double best_excess = 1e300;
  for (int S = 1; S <= smax; ++S) {
    double excess = 0.0;
    for (int R : {1, 2, 4, 8}) {
      if (R > nc) break;
      const double u = units(S, R);
      const double t = std::ceil(u / G) * (tseg(S) + (S > 1 || always_store ? t_store : 0.0));
      const double ideal = units(1, R) * tseg(1) / G;
      excess = std::max(excess, t - ideal);
    }
    if (excess < best_excess * (1.0 - 1e-9)) {
      best_excess = excess;
      best = S;
    }
  }
  return best;
}

static void choose_segments(pcal_session* s, int64_t NC) {
  const int64_t pp = s->pp, Q = s->chunk_rows;
  const CfgInfo ci = cfg_info(pick_size(pp));
  auto rows_R = [&](int R) { return (double)ceil_div(NC, (int64_t)R) * Q; };  // worst rank
  if (dense_family(s->model.kind)) {
    const int64_t ki = s->K_full / ci.BK;
    const double tn = (double)ceil_div(pp, ci.BN);
    s->grad_splits = best_segments(
        (int)std::min<int64_t>(32, ki), NC, ci.BM, ci.BN,
        [&](int S, int R) { return std::ceil(rows_R(R) / ci.BM) * tn * S; },
        [&](int S) { return (double)s->K_full / S; }, false);
  }
  const int smax = (int)std::min<int64_t>(16, Q / ci.BK);
  const double tg = (double)count_tiles(pick_size(pp), 2 * pp, pp, pp, s->sym_gx);
  const double to = (double)count_tiles(pick_size(pp), pp, pp, 0);
  // chunk partials are always stored, so even m = 1 pays the partial traffic
  s->gram_sub = best_segments(
      smax, NC, ci.BM, ci.BN,
      [&](int m, int R) { return tg * (double)ceil_div(NC, (int64_t)R) * m; },
      [&](int m) { return (double)Q / m; }, true);
  s->orth_sub = best_segments(
      smax, NC, ci.BM, ci.BN,
      [&](int m, int R) { return to * (double)ceil_div(NC, (int64_t)R) * m; },
      [&](int m) { return (double)Q / m; }, true);
}

static void alloc_state(pcal_session* s) {
  cudaStream_t st = s->stream;
  const int64_t n = s->n, p = s->p, pp = s->pp, ld = s->ld;
  for (int b = 0; b < 2; ++b) {
    s->pair[b].alloc((size_t)2 * ld * pp);
    s->pair[b].zero(st);
    s->fkd[b].alloc((size_t)3 * p + 2);  // [f | kkt² | d | step_bad, eval_bad]
    s->fkd[b].zero(st);
  }
  s->gr.alloc((size_t)2 * pp * pp);
  s->gr.zero(st);
  s->mcat.alloc((size_t)pp * 2 * pp);
  s->mcat.zero(st);
  s->xm1 = xm1_mode(s);
  if (s->xm1) {
    for (pcal::DevBuf* d : {&s->m1, &s->wmat, &s->cmat, &s->c2m}) {
      d->alloc((size_t)pp * pp);
      d->zero(st);
    }
    s->kk.alloc(2);
    s->kk.zero(st);
    PCAL_CUDA(cudaMalloc(&s->kfb, sizeof(int32_t)));
    PCAL_CUDA(cudaMemsetAsync(s->kfb, 0, sizeof(int32_t), st));
    if (const char* gr = getenv("PCAL_XM1_GATE")) s->xm1_gate = atof(gr);
  }
  // partial arrays: row-block granularities
  const int64_t wm_grad = dense_family(s->model.kind) ? cfg_info(pick_size(pp)).WM : 0;
  const int64_t wm_xm = xm_row_block(s);
  s->st_chunk = 2048;
  s->st_nchunks = ceil_div(n, s->st_chunk);
  {
    const auto& m = s->model;
    s->st_march = is_grid(m.kind) && m.nx <= 128 && m.ny % 8 == 0 && m.ny >= 8 &&
                  s->gz >= 1;
    if (s->comm && is_grid(m.kind) && !s->st_march)
      throw Error(PCAL_E_UNSUPPORTED, "sharded grid models need nx <= 128 and ny % 8 == 0");
    if (s->st_march) {  // enough blocks for ≈ 8 per SM
      const int64_t tiles = (m.ny / 8) * p;
      int64_t nzc = std::max<int64_t>(1, std::min<int64_t>(s->gz, ceil_div(8 * 148, tiles)));
      s->st_zchunk = ceil_div(s->gz, nzc);
      // sharded: z-chunks of whole row chunks, one f partial per (y-tile, row chunk)
      if (s->repro) s->st_zchunk = round_up(s->st_zchunk, s->zc_planes);
      s->st_nzc = ceil_div(s->gz, s->st_zchunk);
      s->st_zpart = s->repro ? s->zc_planes : s->st_zchunk;
    }
  }
  if (s->comm) {
    const int R = s->comm->size;
    const auto& m = s->model;
    if (dense_family(m.kind)) {  // C5: X allgather, unpacked into global row order
      s->xgath.alloc((size_t)R * ld * pp);
      s->xfull.alloc((size_t)s->K_full * pp);
      s->xfull.zero(st);
    } else {  // C5: z-halo planes [send_lo | send_hi | recv_lo | recv_hi], p·nx·ny each
      s->halo.alloc((size_t)4 * p * m.nx * m.ny);
      if (!s->comm->emulated()) {  // exchange overlapped with the interior planes
        PCAL_CUDA(cudaStreamCreateWithFlags(&s->hstream, cudaStreamNonBlocking));
        PCAL_CUDA(cudaEventCreateWithFlags(&s->ev_x, cudaEventDisableTiming));
        PCAL_CUDA(cudaEventCreateWithFlags(&s->ev_h, cudaEventDisableTiming));
      }
      if (m.kind == PCAL_MODEL_KOHN_SHAM) s->rho_gath.alloc((size_t)R * ld);
    }
    std::vector<int64_t> rr(2 * R);
    for (int r = 0; r < R; ++r) {
      rr[r] = s->rank_row0[r];
      rr[R + r] = s->rank_rows[r];
    }
    s->rank_rows_d.alloc((size_t)2 * R);
    PCAL_CUDA(cudaMemcpy(s->rank_rows_d.p, rr.data(), sizeof(int64_t) * 2 * R,
                         cudaMemcpyHostToDevice));
  }
  s->nrb_f = dense_family(s->model.kind) ? ceil_div(n, wm_grad)
             : s->st_march ? (s->model.ny / 8) * ceil_div(s->gz, s->st_zpart)
                           : s->st_nchunks;
  s->nrb_xm = ceil_div(n, wm_xm);
  s->pstride_f = s->nrb_f + 2;
  s->pstride_xm = s->nrb_xm + 2;
  s->fpart.alloc((size_t)s->pstride_f * p);
  s->fpart.zero(st);
  s->kpart.alloc((size_t)s->pstride_xm * p);
  s->kpart.zero(st);
  s->dpart.alloc((size_t)s->pstride_xm * p);
  s->dpart.zero(st);
  s->cp_blocks = (int)std::min<int64_t>(ceil_div(p * p, kStreamThreads), 256);
  s->cpart.alloc(s->cp_blocks);
  if (s->xm1) s->kcp.alloc((size_t)3 * s->cp_blocks);
  s->bb_blocks = 4 * num_sms(s->device);
  {
    int per_sm = 0;
    PCAL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step_fused, kStreamThreads, 0));
    int coop = 0;
    PCAL_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, s->device));
    // the cooperative kernel wins while launch gaps dominate (≤ 8M elements);
    // beyond that the separate kernels stream better
    s->fused_step = coop && per_sm >= 4 && n * p <= (int64_t)8 << 20;
  }
  {
    const auto& m = s->model;
    const int rxp = m.nx % 2 == 0 && m.nx <= 64 ? 2 : m.nx % 4 == 0 && m.nx <= 128 ? 4 : 0;
    s->step_stencil = !s->comm && !s->fused_step && m.kind == PCAL_MODEL_STENCIL && s->st_march &&
                      rxp && m.nx % 16 == 0 && s->alg == PCAL_ALG_PCAL &&
                      !getenv("PCAL_NO_TMA_STENCIL") && !getenv("PCAL_TWO_PASS_NORMALIZE") &&
                      !getenv("PCAL_NO_FUSED_STEP");
  }
  s->bbpart.alloc((size_t)3 * s->bb_blocks);
  s->up_chunk = std::max<int64_t>(1024, round_up(ceil_div(n * p, 8 * 148 * 4), 256));
  s->up_chunk = std::min<int64_t>(s->up_chunk, round_up(n, 256));
  if (s->repro) s->up_chunk = s->chunk_rows;  // norm partials per row chunk
  s->up_nchunks = ceil_div(n, s->up_chunk);
  // (sharded: the all-gathered per-chunk stepsize / norm sums, nch_max rows)
  s->colpart.alloc((size_t)std::max<int64_t>(s->up_nchunks, s->nch_max) * p * 6);
  s->colpart.zero(st);
  s->sinv.alloc((size_t)s->pp);
  PCAL_CUDA(cudaMalloc(&s->sfb, sizeof(int32_t) * s->pp));
  PCAL_CUDA(cudaMemsetAsync(s->sfb, 0, sizeof(int32_t) * s->pp, st));
  if (s->repro) {
    const int R = s->comm->size;
    s->cc.alloc((size_t)s->nch_max * 3 * p + 2);
    s->cc.zero(st);
    s->ccg.alloc((size_t)R * (s->nch_max * 6 * p + 2));
    s->bbt.alloc((size_t)6 * p);
    s->spt.alloc(3);
    s->spt.zero(st);
  }
  s->npart.alloc((size_t)s->up_nchunks * p);
  s->xpart.alloc((size_t)s->up_nchunks * p);
  s->nrm.alloc((size_t)2 * p);
  s->post.alloc(8);
  if (s->alg == PCAL_ALG_ALM) {
    s->glcol.alloc((size_t)p);
    s->glcol.zero(st);
    s->bestx.alloc((size_t)ld * pp);
  }
  s->orth_b.alloc((size_t)pp * pp);
  s->orth_l.alloc((size_t)pp * pp);
  s->orth_t.alloc((size_t)pp * pp);
  s->orth_t.zero(st);
  s->orth_f2.alloc(1);
  s->lam.alloc((size_t)p * p);
  s->lam.zero(st);
  PCAL_CUDA(cudaMalloc(&s->bad, sizeof(int32_t) * 8));
  PCAL_CUDA(cudaMemsetAsync(s->bad, 0, sizeof(int32_t) * 8, st));
  s->orth_status = s->bad + 2;  // [pass-1 ok, pass-2 ok, mgs2 status]
  PCAL_CUDA(cudaMalloc(&s->ctl, sizeof(Ctl)));
  PCAL_CUDA(cudaMallocHost(&s->h_ctl, sizeof(Ctl)));
  s->trace_cap = s->cfg.max_iter + 1;
  s->trace.alloc((size_t)s->trace_cap * kTraceCols);
}

static void upload_matrix(const double* src, int32_t loc, int64_t rows, int64_t cols, double* dst,
                          int64_t ld, cudaStream_t st) {
  if (ld == rows) {  // contiguous: one linear copy (the DMA engines' full rate)
    PCAL_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * rows * cols,
                              loc == PCAL_DEVICE ? cudaMemcpyDeviceToDevice
                                                 : cudaMemcpyHostToDevice,
                              st));
    return;
  }
  PCAL_CUDA(cudaMemcpy2DAsync(dst, sizeof(double) * ld, src, sizeof(double) * rows,
                              sizeof(double) * rows, cols,
                              loc == PCAL_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                              st));
}

// Model data of the rows this session owns.  Sharded sessions receive the
// LOCAL slabs: dense A rows [row0, row0+n) of all n_glob columns (ld = n),
// G0 / V rows of the slab.
static void upload_model(pcal_session* s) {
  const pcal_model_desc& m = s->model;
  cudaStream_t st = s->stream;
  const int64_t n = s->n;
  if (dense_family(m.kind)) {
    if (!m.a) throw Error(PCAL_E_PARAMETER, "dense model: a is NULL");
    s->ldA = s->ld;
    s->A.alloc((size_t)s->ldA * s->K_full);
    s->A.zero(st);
    upload_matrix(m.a, m.location, n, s->n_glob, s->A.p, s->ldA, st);
    if (m.kind == PCAL_MODEL_BILINEAR) {  // B zero-padded to pp×pp; A·X scratch
      if (!m.b) throw Error(PCAL_E_PARAMETER, "bilinear model: b is NULL");
      s->Bm.alloc((size_t)s->pp * s->pp);
      s->Bm.zero(st);
      upload_matrix(m.b, m.location, s->p, s->p, s->Bm.p, s->pp, st);
      s->tb.alloc((size_t)s->ld * s->pp);
      s->tb.zero(st);
    }
    if (m.kind == PCAL_MODEL_DENSITY) {  // L⁻¹ rows of the slab, ρ (all rows), h
      if (!m.linv) throw Error(PCAL_E_PARAMETER, "density model: linv is NULL");
      if (m.density_variant != PCAL_DENSITY_P1 && m.density_variant != PCAL_DENSITY_P6)
        throw Error(PCAL_E_PARAMETER, "density model: unknown variant");
      s->Minv.alloc((size_t)s->ld * s->n_glob);
      s->Minv.zero(st);
      upload_matrix(m.linv, m.location, n, s->n_glob, s->Minv.p, s->ld, st);
      s->rho.alloc((size_t)s->n_glob);
      s->h.alloc((size_t)s->ld);
      s->h.zero(st);
      s->sp_blocks = 4 * 148;
      s->spart.alloc((size_t)3 * s->sp_blocks);
      s->spart.zero(st);
    }
    if (m.kind == PCAL_MODEL_DENSE && m.g0) {
      s->g0.alloc((size_t)s->ld * s->pp);
      s->g0.zero(st);
      upload_matrix(m.g0, m.location, n, s->p, s->g0.p, s->ld, st);
    }
  } else if (m.kind == PCAL_MODEL_STENCIL || m.kind == PCAL_MODEL_KOHN_SHAM) {
    if (m.nx < 1 || m.ny < 1 || m.nz < 1 || m.nx * m.ny * m.nz != s->n_glob)
      throw Error(PCAL_E_DIMENSION, "grid model: n must equal nx*ny*nz");
    if (!m.v) throw Error(PCAL_E_PARAMETER, "grid model: v is NULL");
    s->V.alloc(s->ld);
    s->V.zero(st);
    PCAL_CUDA(cudaMemcpyAsync(s->V.p, m.v, sizeof(double) * n,
                              m.location == PCAL_DEVICE ? cudaMemcpyDeviceToDevice
                                                        : cudaMemcpyHostToDevice,
                              st));
    if (m.kind == PCAL_MODEL_KOHN_SHAM) {
      const int64_t ng = s->n_glob;
      s->u.alloc(s->ld);
      s->rho.alloc(std::max(ng, s->ld));  // local ρ, then the full ρ (sharded)
      s->h.alloc(ng);
      s->tmpa.alloc(ng);
      s->tmpb.alloc(ng);
      auto basis = [&](int64_t N, DevBuf& q, DevBuf& lam) {
        std::vector<double> hq((size_t)N * N), hl((size_t)N);
        pcal_fourier_basis(N, hq.data(), hl.data());
        q.alloc((size_t)N * N);
        lam.alloc((size_t)N);
        PCAL_CUDA(cudaMemcpy(q.p, hq.data(), sizeof(double) * N * N, cudaMemcpyHostToDevice));
        PCAL_CUDA(cudaMemcpy(lam.p, hl.data(), sizeof(double) * N, cudaMemcpyHostToDevice));
      };
      basis(m.nx, s->qx, s->lx);
      basis(m.ny, s->qy, s->ly);
      basis(m.nz, s->qz, s->lz);
      s->sp_blocks = 4 * 148;  // fixed: the partial array is allreduced elementwise
      s->spart.alloc((size_t)3 * s->sp_blocks);
      s->c_xc = std::cbrt(3.0 / 3.14159265358979323846);
    } else {
      s->u.p = nullptr;
    }
  } else if (m.kind == PCAL_MODEL_DEVICE_CALLBACK) {
    if (!m.grad) throw Error(PCAL_E_PARAMETER, "device-callback model: grad is NULL");
    s->fdev.alloc(1);
    s->fdev.zero(st);
  } else {
    throw Error(PCAL_E_UNSUPPORTED, "unsupported model kind " + std::to_string(m.kind));
  }
}

static void init_ctl(pcal_session* s) {
  Ctl c{};
  c.iter = 0;
  c.trace_len = 0;
  c.eta0 = s->eta0;
  c.beta = s->beta;
  c.tol = s->cfg.tol_rel_kkt;
  c.gamma = s->cfg.gamma;
  c.eta_min = s->cfg.eta_min;
  c.eta_max = s->cfg.eta_max;
  c.eta_kind = s->cfg.eta_kind;
  c.mult_rule = s->cfg.multiplier_rule;
  c.max_iter = s->cfg.max_iter;
  c.alm = s->alg == PCAL_ALG_ALM;
  c.alm_inner_max = s->cfg.alm_inner_max;
  c.alm_outer_max = s->cfg.alm_outer_max;
  c.alm_tol_scale = s->cfg.alm_inner_tol_scale;
  c.alm_best = INFINITY;
  *s->h_ctl = c;
  PCAL_CUDA(cudaMemcpyAsync(s->ctl, s->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s->stream));
}

__global__ void k_set_t0(Ctl* c) { c->t0_ns = globaltimer_ns(); }

static void validate(const pcal_config* c) {  // SolverConfig::validate (solver.cpp:106-118)
  if (c->algorithm != PCAL_ALG_PCAL && c->algorithm != PCAL_ALG_PLAM &&
      c->algorithm != PCAL_ALG_MOPTQR && c->algorithm != PCAL_ALG_PLAMDA &&
      c->algorithm != PCAL_ALG_PCALDA && c->algorithm != PCAL_ALG_ALM)
    throw Error(PCAL_E_UNSUPPORTED, "unknown algorithm");
  if (c->beta >= 0.0 && !std::isfinite(c->beta))
    throw Error(PCAL_E_PARAMETER, "SolverConfig: beta must be finite");
  if (!(c->tol_rel_kkt > 0.0))
    throw Error(PCAL_E_PARAMETER, "SolverConfig: tol_rel_kkt must be positive");
  if (c->max_iter < 1) throw Error(PCAL_E_PARAMETER, "SolverConfig: max_iter must be at least 1");
  if (!(c->eta_min < c->eta_max))
    throw Error(PCAL_E_PARAMETER, "SolverConfig: stepsize safeguard interval is empty");
  if (c->eta_kind == PCAL_ETA_CONSTANT && !(c->gamma > 0.0))
    throw Error(PCAL_E_PARAMETER, "SolverConfig: constant stepsize gamma must be positive");
  if (c->eta_kind < 0 || c->eta_kind > 4) throw Error(PCAL_E_PARAMETER, "unknown stepsize rule");
  if (c->multiplier_rule != PCAL_MULT_PCAL_FORMULA && c->multiplier_rule != PCAL_MULT_PLAM_FORMULA)
    throw Error(PCAL_E_PARAMETER, "unknown multiplier rule");
  if (c->alm_inner_max < 1 || c->alm_outer_max < 1)
    throw Error(PCAL_E_PARAMETER, "SolverConfig: ALM iteration caps must be at least 1");
}

static double clamp_eta_h(const pcal_config* c, double v) {
  return std::min(std::max(v, c->eta_min), c->eta_max);
}

static void capture_graphs(pcal_session* s) {
  for (int b = 0; b < 2; ++b) {
    int64_t cnt = 0;
    LaunchScope ls(&cnt);
    cudaGraph_t g;
    PCAL_CUDA(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    launch_iteration(s, b);
    PCAL_CUDA(cudaStreamEndCapture(s->stream, &g));
    PCAL_CUDA(cudaGraphInstantiate(&s->graph[b], g, 0));
    PCAL_CUDA(cudaGraphDestroy(g));
    s->kernels_per_iter = cnt;
  }
}

}  // namespace pcal

pcal_session::~pcal_session() {
  for (auto& g : graph)
    if (g) cudaGraphExecDestroy(g);
  for (auto& e : pev)
    if (e) cudaEventDestroy(e);
  if (bad) cudaFree(bad);
  if (sfb) cudaFree(sfb);
  if (kfb) cudaFree(kfb);
  if (rank_nch_d) cudaFree(rank_nch_d);
  if (ctl) cudaFree(ctl);
  if (h_ctl) cudaFreeHost(h_ctl);
  if (stream && own_stream) cudaStreamDestroy(stream);
  if (hstream) cudaStreamDestroy(hstream);
  if (ev_x) cudaEventDestroy(ev_x);
  if (ev_h) cudaEventDestroy(ev_h);
}

using namespace pcal;

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PCAL_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = "host allocation failed";
    return PCAL_E_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return PCAL_E_CUDA;
  }
}

// k_iter_rows over `iters` iterations (cooperative, one CTA per 8 rows).
static void launch_rows(pcal_session* s, int iters) {
  RowsArgs a{};
  for (int b = 0; b < 2; ++b) {
    a.pair[b] = s->pair[b].p;
    a.fkd[b] = s->fkd[b].p;
  }
  a.at = s->at.p;
  a.ldat = s->ld;
  a.g0 = s->g0.p;
  a.lam = s->lam.p;
  a.z = s->mz.p;
  a.gpart = s->rgpart.p;
  a.gtot = s->rgtot.p;
  a.gcnt = reinterpret_cast<unsigned*>(s->rgcnt.p);
  a.cpart = s->rcpart.p;
  a.bbpart = s->mbb.p;
  a.n = s->n;
  a.ld = s->ld;
  a.p = s->p;
  a.pp = s->pp;
  a.nent = s->rows_nent;
  a.plain = !(s->alg == PCAL_ALG_PCAL || s->alg == PCAL_ALG_PCALDA);
  const bool da = s->alg == PCAL_ALG_PLAMDA || s->alg == PCAL_ALG_PCALDA;
  a.mc_mode = da ? MC_DA : MC_PCAL;
  a.p_from_g = da;
  a.dform = s->alg == PCAL_ALG_PCAL && s->cfg.multiplier_rule == PCAL_MULT_PCAL_FORMULA;
  a.beta = s->beta;
  a.beta_epi = da ? 1.0 : s->beta;
  a.fa.model = s->model.kind;
  a.fa.p = s->p;
  a.fa.mode = 0;
  a.fa.trace = s->trace.p;
  a.fa.bad = s->bad;
  a.fa.c_xc = s->c_xc;
  Ctl* c = s->ctl;
  void* args[] = {&a, &c, &iters};
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)s->mega_grid);
  lc.blockDim = dim3(kRowsThreads);
  a.zld = rows_zld(s->n);
  lc.dynamicSmemBytes = rows_smem_bytes(s->p, a.zld);
  lc.stream = s->stream;
  cudaLaunchAttribute attr[2]{};
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = (unsigned)s->rows_csize;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = s->rows_csize > 1 ? 2 : 1;
  a.csize = s->rows_csize;
  // PCAL_SMALL_PROF=1: per-phase %globaltimer stamps of CTA 0, printed per batch
  static const bool prof = getenv("PCAL_SMALL_PROF") && getenv("PCAL_SMALL_PROF")[0] == '1';
  uint64_t* dprof = nullptr;
  if (prof) {
    PCAL_CUDA(cudaMalloc(&dprof, sizeof(uint64_t) * 16 * iters));
    PCAL_CUDA(cudaMemsetAsync(dprof, 0, sizeof(uint64_t) * 16 * iters, s->stream));
    a.prof = dprof;
  }
  PCAL_CUDA(cudaLaunchKernelExC(&lc, (const void*)k_iter_rows, args));
  launched("k_iter_rows");
  if (prof) {
    std::vector<uint64_t> h((size_t)16 * iters);
    PCAL_CUDA(cudaMemcpyAsync(h.data(), dprof, sizeof(uint64_t) * h.size(), cudaMemcpyDeviceToHost,
                              s->stream));
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
    double acc[16] = {};
    int cnt = 0;
    for (int it = 0; it + 1 < iters; ++it) {
      const uint64_t* r = &h[(size_t)16 * it];
      if (!r[4] || !h[(size_t)16 * (it + 1)]) break;
      for (int q = 0; q < 4; ++q) acc[q] += (double)(r[q + 1] - r[q]);
      acc[4] += (double)(h[(size_t)16 * (it + 1)] - r[4]);
      acc[5] += (double)(r[6] - r[1]);  // phase 2: Y staged
      acc[6] += (double)(r[7] - r[6]);  //          DMMA loop
      acc[7] += (double)(r[5] - r[7]);  //          warp reduction
      for (int q = 8; q <= 13; ++q) acc[q] += (double)(r[q] - r[q == 8 ? 2 : q == 11 ? 3 : q - 1]);
      ++cnt;
    }
    if (cnt)
      fprintf(stderr,
              "k_iter_rows us/iter: 1 eta+Z %.2f  2 A.Z+Gram partials %.2f  3 P epilogue %.2f  "
              "4 sums+record+bb %.2f  (loop %.2f)  [2: stage Y %.2f, DMMA %.2f, reduce %.2f] "
              "grid %d cluster %d\n  3: totals %.2f WCM %.2f rows %.2f | 4: col totals %.2f "
              "record %.2f bb %.2f\n",
              acc[0] / cnt / 1e3, acc[1] / cnt / 1e3, acc[2] / cnt / 1e3, acc[3] / cnt / 1e3,
              acc[4] / cnt / 1e3, acc[5] / cnt / 1e3, acc[6] / cnt / 1e3, acc[7] / cnt / 1e3,
              s->mega_grid, s->rows_csize, acc[8] / cnt / 1e3, acc[9] / cnt / 1e3,
              acc[10] / cnt / 1e3, acc[11] / cnt / 1e3, acc[12] / cnt / 1e3, acc[13] / cnt / 1e3);
    cudaFree(dprof);
  }
}

// k_iter_small over `iters` iterations (cooperative, one CTA per SM).
static void launch_small(pcal_session* s, int iters) {
  if (s->rows) {
    launch_rows(s, iters);
    return;
  }
  SmallArgs a{};
  for (int b = 0; b < 2; ++b) {
    a.pair[b] = s->pair[b].p;
    a.fkd[b] = s->fkd[b].p;
  }
  a.at = s->at.p;
  a.ldat = s->ld;
  a.g0 = s->g0.p;
  a.gr = s->gr.p;
  a.lam = s->lam.p;
  a.z = s->mz.p;
  a.part = s->mpart.p;
  a.npb = s->mnpb.p;
  a.bbpart = s->mbb.p;
  a.n = s->n;
  a.ld = s->ld;
  a.p = s->p;
  a.pp = s->pp;
  a.plain = !(s->alg == PCAL_ALG_PCAL || s->alg == PCAL_ALG_PCALDA);
  const bool da = s->alg == PCAL_ALG_PLAMDA || s->alg == PCAL_ALG_PCALDA;
  a.mc_mode = da ? MC_DA : MC_PCAL;
  a.p_from_g = da;
  a.dform = s->alg == PCAL_ALG_PCAL && s->cfg.multiplier_rule == PCAL_MULT_PCAL_FORMULA;
  a.beta = s->beta;
  a.beta_epi = da ? 1.0 : s->beta;
  a.fa.model = s->model.kind;
  a.fa.p = s->p;
  a.fa.mode = 0;
  a.fa.trace = s->trace.p;
  a.fa.bad = s->bad;
  a.fa.c_xc = s->c_xc;
  a.lda_s = s->mega_lda_s;
  Ctl* c = s->ctl;
  void* args[] = {&a, &c, &iters};
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)s->mega_grid);
  lc.blockDim = dim3(kSmallThreads);
  lc.dynamicSmemBytes = (size_t)8 * s->mega_lda_s * sizeof(double);
  lc.stream = s->stream;
  cudaLaunchAttribute attr{};
  attr.id = cudaLaunchAttributeCooperative;
  attr.val.cooperative = 1;
  lc.attrs = &attr;
  lc.numAttrs = 1;
  // PCAL_SMALL_PROF=1: per-phase %globaltimer stamps of CTA 0, printed per batch
  static const bool prof = getenv("PCAL_SMALL_PROF") && getenv("PCAL_SMALL_PROF")[0] == '1';
  uint64_t* dprof = nullptr;
  if (prof) {
    PCAL_CUDA(cudaMalloc(&dprof, sizeof(uint64_t) * 8 * iters));
    PCAL_CUDA(cudaMemsetAsync(dprof, 0, sizeof(uint64_t) * 8 * iters, s->stream));
    a.prof = dprof;
  }
  PCAL_CUDA(cudaLaunchKernelExC(&lc, (const void*)k_iter_small, args));
  launched("k_iter_small");
  if (prof) {
    std::vector<uint64_t> h((size_t)8 * iters);
    PCAL_CUDA(cudaMemcpyAsync(h.data(), dprof, sizeof(uint64_t) * h.size(), cudaMemcpyDeviceToHost,
                              s->stream));
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
    double acc[6] = {0, 0, 0, 0, 0, 0};
    int cnt = 0;
    for (int it = 0; it + 1 < iters; ++it) {
      const uint64_t* r = &h[(size_t)8 * it];
      if (!r[5] || !h[(size_t)8 * (it + 1)]) break;
      for (int q = 0; q < 5; ++q) acc[q] += (double)(r[q + 1] - r[q]);
      acc[5] += (double)(h[(size_t)8 * (it + 1)] - r[5]);
      ++cnt;
    }
    if (cnt)
      fprintf(stderr,
              "k_iter_small us/iter: B eta+Z %.2f  C norm+grad %.2f  D gram %.2f  E xm %.2f  "
              "A sums+record+bb %.2f  (loop %.2f)\n",
              acc[0] / cnt / 1e3, acc[1] / cnt / 1e3, acc[2] / cnt / 1e3, acc[3] / cnt / 1e3,
              acc[4] / cnt / 1e3, acc[5] / cnt / 1e3);
    cudaFree(dprof);
  }
}

// The persistent small-problem kernel applies to dense PCAL / PLAM / dual-ascent
// runs with p ≤ 32 on one GPU (MOptQR keeps its in-graph retraction).
static void setup_small(pcal_session* s) {
  const char* off = getenv("PCAL_NO_SMALL_KERNEL");
  if ((off && off[0] == '1') || s->comm || s->model.kind != PCAL_MODEL_DENSE ||
      s->p > kSmallP || s->n > 8192 || s->alg == PCAL_ALG_MOPTQR || s->alg == PCAL_ALG_ALM)
    return;
  int coop = 0, per_sm = 0;
  PCAL_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, s->device));
  const int nsm = num_sms(s->device);
  {  // n ≤ 8·SMs (and ≤ 8·4·kRowsKS): one CTA per 8 rows, k_iter_rows
    int64_t g = ceil_div(s->n, 8);
    const char* v1 = getenv("PCAL_SMALL_V1");
    const size_t smem = rows_smem_bytes(s->p, rows_zld(s->n));
    cudaFuncAttributes fa{};
    PCAL_CUDA(cudaFuncGetAttributes(&fa, k_iter_rows));
    int optin = 0;
    PCAL_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->device));
    if (!(v1 && v1[0] == '1') && coop && g <= nsm && g <= kRowsMaxGrid &&
        ceil_div(ceil_div(s->n, 4), 8) <= kRowsKS && smem + fa.sharedSizeBytes <= (size_t)optin) {
      PCAL_CUDA(cudaFuncSetAttribute(k_iter_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
      PCAL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_iter_rows, kRowsThreads,
                                                              smem));
      // clusters of up to 8 CTAs share one L2 read of Y (multicast); the
      // cluster size must divide the grid and every cluster must fit at once
      // (measured at config 1: multicast saves 0.3 us of staging but the
      // rounded-up grid costs as much in the totals; default off)
      int cs = 1;
      const char* ce = getenv("PCAL_ROWS_CLUSTER");
      if (ce) cs = std::max(1, std::min(8, atoi(ce)));
      int64_t gg = g;
      for (; cs > 1; cs /= 2) {
        gg = round_up(g, cs);
        if (gg > nsm || gg > kRowsMaxGrid) continue;
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3((unsigned)gg);
        lc.blockDim = dim3(kRowsThreads);
        lc.dynamicSmemBytes = smem;
        cudaLaunchAttribute at{};
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = (unsigned)cs;
        at.val.clusterDim.y = at.val.clusterDim.z = 1;
        lc.attrs = &at;
        lc.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)k_iter_rows, &lc) == cudaSuccess &&
            (int64_t)ncl * cs >= gg)
          break;
        cudaGetLastError();
      }
      if (cs <= 1) {
        cs = 1;
        gg = g;
      }
      if (per_sm >= 1) {
        s->rows_csize = cs;
        g = gg;
        s->mega_grid = (int)g;
        const int64_t p = s->p, np2 = p * (p + 1) / 2;
        s->rows_nent = (int)(2 * np2 + (s->g0.p ? p * p : 0));
        s->rows_ngroups = (int)ceil_div(g, kRowsGroup);
        s->at.alloc((size_t)s->ld * s->n);
        s->at.zero(s->stream);
        dim3 tg((unsigned)ceil_div(s->n, 32), (unsigned)ceil_div(s->n, 32));
        k_transpose<<<tg, dim3(32, 8), 0, s->stream>>>(s->A.p, s->ldA, s->n, s->at.p, s->ld);
        launched("k_transpose");
        s->rgpart.alloc((size_t)g * s->rows_nent);
        s->rgtot.alloc((size_t)s->rows_ngroups * s->rows_nent);
        s->rgcnt.alloc((size_t)s->rows_ngroups);
        s->rgcnt.zero(s->stream);
        s->rcpart.alloc((size_t)g * 2 * 32);
        s->mbb.alloc((size_t)g * 3);
        s->mz.alloc((size_t)s->ld * s->pp);
        s->mz.zero(s->stream);
        s->rows = true;
        s->mega = true;
        return;
      }
    }
  }
  s->mega_grid = nsm;
  // one 8-row gradient tile per CTA: keep those rows of A resident in shared
  // memory (row stride ≡ 4 mod 16 doubles: conflict-free DMMA fragment loads)
  const int64_t lda_s = round_up(s->n, 16) + 4;
  if (s->n <= 8 * (int64_t)s->mega_grid && 8 * lda_s * 8 <= 160 * 1024) {
    s->mega_lda_s = lda_s;
    PCAL_CUDA(cudaFuncSetAttribute(k_iter_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(8 * lda_s * 8)));
  }
  PCAL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &per_sm, k_iter_small, kSmallThreads, (size_t)8 * s->mega_lda_s * sizeof(double)));
  if (!coop || per_sm < 1) return;
  if (s->mega_grid > 160) return;  // the record phase sums ≤ 160 CTA partials
  s->at.alloc((size_t)s->ld * s->n);
  s->at.zero(s->stream);  // rows k ≥ n are read by the padded k-steps
  dim3 g((unsigned)ceil_div(s->n, 32), (unsigned)ceil_div(s->n, 32));
  k_transpose<<<g, dim3(32, 8), 0, s->stream>>>(s->A.p, s->ldA, s->n, s->at.p, s->ld);
  launched("k_transpose");
  s->mpart.alloc((size_t)s->mega_grid * 3 * kSmallP);
  s->mnpb.alloc((size_t)s->mega_grid * kSmallP);
  s->mbb.alloc((size_t)s->mega_grid * 3);
  s->mz.alloc((size_t)s->ld * s->pp);
  s->mz.zero(s->stream);  // padded rows / columns are read by the DMMA tiles
  s->mega = true;
}

bool orthonormalize_dev(pcal_session* s, const double* x, double* q, double* scratch);

void session_create(const pcal_model_desc* model, const pcal_config* config, const double* x0,
                    int32_t x0_loc, pcal_session** out, pcal_category_timers* timers,
                    Comm* comm = nullptr, cudaStream_t shared_stream = nullptr) {
  if (!model || !config || !x0 || !out) throw Error(PCAL_E_PARAMETER, "NULL argument");
  validate(config);
  if (model->n < 1 || model->p < 1) throw Error(PCAL_E_DIMENSION, "model: n, p must be positive");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
    throw Error(PCAL_E_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  if (config->device < 0 || config->device >= ndev) throw Error(PCAL_E_PARAMETER, "bad device");
  auto s = std::make_unique<pcal_session>();
  s->t_start = std::chrono::steady_clock::now();
  s->device = config->device;
  PCAL_CUDA(cudaSetDevice(s->device));
  s->model = *model;
  s->cfg = *config;
  s->timers = timers;
  s->comm = comm;
  s->n_glob = model->n;
  s->p = model->p;
  s->pp = padded_p(s->p);
  const int R = comm ? comm->size : 1;
  const int rk = comm ? comm->rank : 0;
  if (is_grid(model->kind) && (model->nz < R))
    throw Error(PCAL_E_PARAMETER, "fewer z-planes than ranks");
  if (!is_grid(model->kind) && model->n < R)
    throw Error(PCAL_E_PARAMETER, "fewer rows than ranks");
  int64_t maxrows = 0;
  s->rank_row0.resize(R);
  s->rank_rows.resize(R);
  for (int r = 0; r < R; ++r) {
    int64_t z0, nzl;
    partition(*model, R, r, &s->rank_row0[r], &s->rank_rows[r], &z0, &nzl);
    maxrows = std::max(maxrows, s->rank_rows[r]);
    if (r == rk) s->gz = nzl ? nzl : model->nz;
  }
  s->row0 = s->rank_row0[rk];
  s->n = s->rank_rows[rk];
  s->ld_max = padded_ld(maxrows);
  s->ld = comm ? s->ld_max : padded_ld(s->n);
  s->K_full = padded_ld(s->n_glob);
  if (comm) {  // reproducible chunked reductions
    int64_t Q, NC, Zc;
    chunking(*model, &Q, &NC, &Zc);
    if (is_grid(model->kind) && (model->nx * model->ny) % 64 != 0)
      throw Error(PCAL_E_UNSUPPORTED, "sharded grid models need nx*ny to be a multiple of 64");
    s->repro = true;
    s->chunk_rows = Q;
    s->zc_planes = Zc;
    std::vector<int32_t> nq(R);
    for (int r = 0; r < R; ++r) {
      nq[r] = (int32_t)((int64_t)(r + 1) * NC / R - (int64_t)r * NC / R);
      s->nch_max = std::max<int64_t>(s->nch_max, nq[r]);
    }
    s->nch = nq[rk];
    s->ld_max = s->ld = s->nch_max * Q;  // every chunk's rows fit (zero padded)
    choose_segments(s.get(), NC);
    PCAL_CUDA(cudaMalloc(&s->rank_nch_d, sizeof(int32_t) * R));
    PCAL_CUDA(cudaMemcpy(s->rank_nch_d, nq.data(), sizeof(int32_t) * R, cudaMemcpyHostToDevice));
  }
  s->K_full = padded_ld(s->n_glob);
  s->alg = config->algorithm;
  // the grid models' operators are symmetric, so GᵀX = XᵀLX (+ XᵀVX) is: only its
  // upper triangle is computed (MOptQR uses the unsymmetrised GᵀX)
  s->sym_gx = (model->kind == PCAL_MODEL_STENCIL || model->kind == PCAL_MODEL_KOHN_SHAM) &&
              s->alg != PCAL_ALG_MOPTQR && !getenv("PCAL_FULL_GX");
  if (comm && s->alg == PCAL_ALG_MOPTQR)
    throw Error(PCAL_E_UNSUPPORTED, "MOptQR is single-GPU (its MGS2 fallback is not sharded)");
  if (comm && model->kind == PCAL_MODEL_DEVICE_CALLBACK)
    throw Error(PCAL_E_UNSUPPORTED, "device-callback models are single-GPU");
  // resolve_beta (solver.cpp:120-134)
  s->beta = config->beta >= 0.0                                                ? config->beta
            : (s->alg == PCAL_ALG_PCAL || s->alg == PCAL_ALG_PCALDA) ? 1.0
            : s->alg == PCAL_ALG_MOPTQR                                       ? 0.0
                                                                              : model->s + 0.1;
  s->eta0 = config->eta0 > 0.0 ? clamp_eta_h(config, config->eta0)     // solver.cpp:99-102
                               : clamp_eta_h(config, model->s + 2.0 * s->beta);
  LaunchScope ls(&s->launches);
  if (shared_stream) {
    s->stream = shared_stream;
    s->own_stream = false;
  } else {
    PCAL_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  }
  for (auto& e : s->pev) PCAL_CUDA(cudaEventCreate(&e));
  s->pev_on = timers != nullptr;
  alloc_state(s.get());
  upload_model(s.get());
  build_plans(s.get());
  setup_small(s.get());
  init_ctl(s.get());
  if (x0_loc == PCAL_X0_SEED) {  // initial_point({Qr}, seed) of this rank's rows
    const uint64_t seed = *reinterpret_cast<const uint64_t*>(x0);
    if (2 * s->p > s->n_glob)  // solver.cpp:137-138
      throw Error(PCAL_E_PARAMETER, "initial_point: dimensions must satisfy 2p <= n");
    double* h = nullptr;
    PCAL_CUDA(cudaMallocHost(&h, sizeof(double) * (size_t)s->n * s->p));
    std::unique_ptr<double, decltype(&cudaFreeHost)> hg(h, &cudaFreeHost);
    host_random_normal_rows(s->n_glob, s->p, seed, s->row0, s->n, h,
                            (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
    upload_matrix(h, PCAL_HOST, s->n, s->p, Xof(s.get(), 1), s->ld, s->stream);
    if (!orthonormalize_dev(s.get(), Xof(s.get(), 1), Xof(s.get(), 0), Pof(s.get(), 1)))
      throw Error(PCAL_E_RANK, "initial_point: numerically rank-deficient Gaussian start");
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
  } else {
    upload_matrix(x0, x0_loc, s->n, s->p, Xof(s.get(), 0), s->ld, s->stream);
  }
  k_set_t0<<<1, 1, 0, s->stream>>>(s->ctl);
  launched("k_set_t0");
  launch_eval(s.get(), 0, 1, s->ctl);  // eval_iterate(X0) + record(0) (solver.cpp:363-365)
  PCAL_CUDA(cudaGetLastError());
  s->next_k = 0;
  // graphs: not for timers (events between kernels) nor emulated ranks (host barriers)
  s->use_graphs = timers == nullptr && !(comm && comm->emulated());
  if (s->use_graphs) capture_graphs(s.get());
  *out = s.release();
}

void read_ctl(pcal_session* s) {
  PCAL_CUDA(cudaMemcpyAsync(s->h_ctl, s->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s->stream));
  PCAL_CUDA(cudaStreamSynchronize(s->stream));
}

// ALM (alm_outer, solver.cpp:478-624): the inner steps are the usual iteration
// (graph) with Λ fixed; after each evaluation the device has decided the next
// action (Ctl::alm_phase), which the host reads: an inner step, or the
// multiplier update — the inner loop's iterate (its best after a cap) moves to
// the other pair, Λ ← Λ − β(XᵀX − I) in that pair's evaluation, and the
// stepsize memory restarts.  `iters` bounds the inner steps of this call.
static void run_alm(pcal_session* s, int64_t iters) {
  const size_t xbytes = sizeof(double) * (size_t)s->ld * s->pp;
  int64_t steps = 0;
  for (;;) {
    read_ctl(s);
    const Ctl& c = *s->h_ctl;
    if (c.done || (c.alm_phase == 0 && steps >= iters)) break;
    const int b = (int)(s->next_k % 2);
    if (c.alm_copy)
      PCAL_CUDA(cudaMemcpyAsync(s->bestx.p, Xof(s, b), xbytes, cudaMemcpyDeviceToDevice, s->stream));
    if (c.alm_phase == 0) {
      if (s->use_graphs) {
        PCAL_CUDA(cudaGraphLaunch(s->graph[b], s->stream));
        count_launch(s->kernels_per_iter);
      } else {
        launch_iteration(s, b);
      }
      ++steps;
      s->launched++;
    } else {
      PCAL_CUDA(cudaMemcpyAsync(Xof(s, 1 - b), c.alm_met ? Xof(s, b) : s->bestx.p, xbytes,
                                cudaMemcpyDeviceToDevice, s->stream));
      k_alm_boundary<<<1, 1, 0, s->stream>>>(s->ctl);
      launched("k_alm_boundary");
      launch_eval(s, 1 - b, 3, s->ctl);
    }
    s->next_k++;
  }
}

void session_run(pcal_session* s, int64_t iters) {
  PCAL_CUDA(cudaSetDevice(s->device));
  LaunchScope ls(&s->launches);
  if (s->alg == PCAL_ALG_ALM) {
    run_alm(s, iters);
    return;
  }
  const int64_t batch = 32;
  int64_t remaining = std::min<int64_t>(iters, s->cfg.max_iter - s->launched);
  cudaEvent_t polled = nullptr;
  PCAL_CUDA(cudaEventCreateWithFlags(&polled, cudaEventDisableTiming));
  bool pending = false;
  while (remaining > 0) {
    const int64_t nb = std::min(batch, remaining);
    if (s->mega && !s->pev_on) {  // one persistent launch for the whole batch
      launch_small(s, (int)nb);
      s->next_k += nb;
      s->launched += nb;
    }
    for (int64_t i = 0; i < nb && !(s->mega && !s->pev_on); ++i) {
      const int b = (int)(s->next_k % 2);
      if (s->use_graphs) {
        PCAL_CUDA(cudaGraphLaunch(s->graph[b], s->stream));
        count_launch(s->kernels_per_iter);
      } else {
        launch_iteration(s, b);
      }
      s->next_k++;
      s->launched++;
    }
    remaining -= nb;
    if (s->comm) {  // sharded: every rank must stop after the same batch (collectives)
      PCAL_CUDA(cudaMemcpyAsync(&s->h_ctl->done, &s->ctl->done, sizeof(int32_t),
                                cudaMemcpyDeviceToHost, s->stream));
      PCAL_CUDA(cudaStreamSynchronize(s->stream));
      if (s->h_ctl->done) break;
      continue;
    }
    // poll `done` of the previous batch without stalling the device queue
    if (pending) {
      PCAL_CUDA(cudaEventSynchronize(polled));
      if (s->h_ctl->done) break;
    }
    PCAL_CUDA(cudaMemcpyAsync(&s->h_ctl->done, &s->ctl->done, sizeof(int32_t),
                              cudaMemcpyDeviceToHost, s->stream));
    PCAL_CUDA(cudaEventRecord(polled, s->stream));
    pending = true;
  }
  cudaEventDestroy(polled);
}


// CholeskyQR2 of the n×p matrix at x (ld) into q (ld); MGS2 fallback.  Returns
// false on rank deficiency (rank_error).  q and scratch must not alias x.
bool orthonormalize_dev(pcal_session* s, const double* x, double* q, double* scratch) {
  cudaStream_t st = s->stream;
  const int64_t p = s->p, pp = s->pp, ld = s->ld, n = s->n;
  GemmPlan& gp = s->orth_gram;
  GemmPlan& mp = s->orth_mul;
  if (!gp.d_tiles) {
    if (s->repro) {  // chunked Gram + whole-tile products (rank-count invariant)
      plan_gemm(gp, s->device, pick_size(pp), A_KCONTIG, EPI_STORE, pp, pp,
                s->nch * s->chunk_rows, 0, 0, (int)(s->nch * s->orth_sub), true,
                (int)(s->nch_max * s->orth_sub));
      plan_gemm(mp, s->device, pick_size(pp), A_MCONTIG, EPI_STORE, n, pp, pp, -1, 0, 1);
      tree_setup(s, 1, s->orth_sub, gp.ntasks);
    } else {
      plan_gemm(gp, s->device, pick_size(pp), A_KCONTIG, EPI_STORE, pp, pp, ld, 0);
      plan_gemm(mp, s->device, pick_size(pp), A_MCONTIG, EPI_STORE, n, pp, pp);
    }
  }
  auto gram_of = [&](const double* a) {
    gp.args.A = a;
    gp.args.lda = ld;
    gp.args.B = a;
    gp.args.ldb = ld;
    gp.args.ep.C = s->orth_b.p;
    gp.args.ep.ldc = pp;
    gp.args.ep.m_store = pp;
    gp.args.ep.n_store = pp;
    gp.args.ctl = nullptr;
    launch_gemm(gp, st);
    if (s->repro) gram_reduce(s, gp, 1);  // sharded Gram
  };
  auto mul_t = [&](const double* a, double* out) {  // out = a · T
    mp.args.A = a;
    mp.args.lda = ld;
    mp.args.B = s->orth_t.p;
    mp.args.ldb = pp;
    mp.args.ep.C = out;
    mp.args.ep.ldc = ld;
    mp.args.ep.m_store = n;
    mp.args.ep.n_store = p;
    mp.args.ctl = nullptr;
    launch_gemm(mp, st);
  };
  int32_t ok = 0;
  gram_of(x);
  k_sym_fro2<<<1, 1024, 0, st>>>(s->orth_b.p, pp, p, s->orth_f2.p);
  launched("k_sym_fro2");
  launch_chol_trinv(st, s->orth_b.p, pp, p, s->orth_f2.p, s->orth_l.p, pp, s->orth_t.p, pp,
                    s->orth_status, nullptr, nullptr);
  PCAL_CUDA(cudaMemcpyAsync(&ok, s->orth_status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  PCAL_CUDA(cudaStreamSynchronize(st));
  bool chol_ok = ok != 0;
  g_orth_path = chol_ok ? 0 : 1;
  if (chol_ok) {
    mul_t(x, scratch);  // Q1 = X·L1⁻ᵀ
    gram_of(scratch);
    launch_chol_trinv(st, s->orth_b.p, pp, p, s->orth_f2.p, s->orth_l.p, pp, s->orth_t.p, pp,
                      s->orth_status, nullptr, nullptr);
    PCAL_CUDA(cudaMemcpyAsync(&ok, s->orth_status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    PCAL_CUDA(cudaStreamSynchronize(st));
    chol_ok = ok != 0;
    if (!chol_ok) g_orth_path = 2;
    if (chol_ok) mul_t(scratch, q);  // Q = Q1·L2⁻ᵀ
  }
  if (!chol_ok) {  // mgs2(x) fallback (kernels.cpp:254,258)
    if (s->comm) {
      // sharded: MGS2 is inherently sequential over columns — gather X, run it
      // redundantly on every rank, keep the local rows (rank-deficient path only)
      const int R = s->comm->size;
      const int64_t kf = s->K_full;
      DevBuf gath, full;
      gath.alloc((size_t)R * ld * s->pp);
      full.alloc((size_t)kf * s->pp);
      full.zero(st);
      s->comm->allgather(x, gath.p, (size_t)ld * s->pp, st);
      k_unpack_rows<<<dim3((unsigned)ceil_div(ld, 256), (unsigned)s->pp, (unsigned)R), 256, 0, st>>>(
          gath.p, ld, s->pp, (const int64_t*)s->rank_rows_d.p, R, full.p, kf, nullptr);
      launched("k_unpack_rows");
      k_mgs2<<<1, 1024, 0, st>>>(full.p, s->n_glob, kf, p, s->orth_f2.p, s->orth_status);
      launched("k_mgs2");
      PCAL_CUDA(cudaMemcpy2DAsync(q, sizeof(double) * ld, full.p + s->row0, sizeof(double) * kf,
                                  sizeof(double) * n, p, cudaMemcpyDeviceToDevice, st));
    } else {
      PCAL_CUDA(cudaMemcpy2DAsync(q, sizeof(double) * ld, x, sizeof(double) * ld,
                                  sizeof(double) * ld, p, cudaMemcpyDeviceToDevice, st));
      k_mgs2<<<1, 1024, 0, st>>>(q, n, ld, p, s->orth_f2.p, s->orth_status);
      launched("k_mgs2");
    }
    PCAL_CUDA(cudaMemcpyAsync(&ok, s->orth_status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    PCAL_CUDA(cudaStreamSynchronize(st));
    if (!ok) {
      g_orth_path = -1;
      return false;
    }
  }
  return true;
}

// D2H of an n×p iterate (ld) into a column-major host array; a contiguous
// layout (ld = n) is one linear copy
static void d2h_matrix(const pcal_session* s, const double* dsrc, double* host, cudaStream_t st) {
  if (s->ld == s->n)
    PCAL_CUDA(cudaMemcpyAsync(host, dsrc, sizeof(double) * s->n * s->p, cudaMemcpyDeviceToHost, st));
  else
    PCAL_CUDA(cudaMemcpy2DAsync(host, sizeof(double) * s->n, dsrc, sizeof(double) * s->ld,
                                sizeof(double) * s->n, s->p, cudaMemcpyDeviceToHost, st));
}

void copy_out(pcal_session* s, const double* dsrc, double* host) {
  d2h_matrix(s, dsrc, host, s->stream);
}

void session_finish(pcal_session* s, pcal_report* r) {
  PCAL_CUDA(cudaSetDevice(s->device));
  LaunchScope ls(&s->launches);
  read_ctl(s);
  Ctl& c = *s->h_ctl;
  if (c.step_param) throw Error(PCAL_E_PARAMETER, "pcal_step: eta must be positive");
  const int64_t tl = c.trace_len;
  if (r->trace && r->trace_capacity < tl)
    throw Error(PCAL_E_PARAMETER, "report trace capacity too small");
  if (r->trace && tl)
    PCAL_CUDA(cudaMemcpyAsync(r->trace, s->trace.p, sizeof(double) * tl * kTraceCols,
                              cudaMemcpyDeviceToHost, s->stream));
  r->trace_len = tl;
  r->beta = s->beta;
  r->eta0 = s->eta0;
  r->has_post = 0;
  r->has_x = 0;
  r->degenerate_steps = c.degenerate;
  r->iterations = tl > 0 ? tl - 1 : 0;
  r->outer_iterations = c.alm_outer;
  r->inner_cap_hits = c.alm_caps;
  for (int i = 0; i < 4; ++i) r->final_pre[i] = r->final_post[i] = 0.0;
  int status = c.done == 1 ? PCAL_STATUS_CONVERGED
               : c.done == 2 ? PCAL_STATUS_DIVERGED
                             : PCAL_STATUS_MAX_ITER;
  if (status != PCAL_STATUS_DIVERGED) {
    const int b = (int)((c.iter + c.alm_flips) % 2);
    r->final_pre[0] = c.f;
    r->final_pre[1] = c.kkt_abs;
    r->final_pre[2] = c.rel;
    r->final_pre[3] = c.feas;
    r->has_x = 1;
    // D2H on a side stream: the stop iterate under the final CholeskyQR2, Q
    // under the post-orth evaluation (which only reads it)
    cudaStream_t cs = nullptr;
    auto side_copy = [&](const double* dsrc, double* host) {
      cudaEvent_t ev;
      if (!cs) PCAL_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      PCAL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      PCAL_CUDA(cudaEventRecord(ev, s->stream));
      PCAL_CUDA(cudaStreamWaitEvent(cs, ev, 0));
      PCAL_CUDA(cudaEventDestroy(ev));
      d2h_matrix(s, dsrc, host, cs);
    };
    struct StreamJoin {  // the side copies complete before the report is returned
      cudaStream_t* st;
      ~StreamJoin() {
        if (*st) {
          cudaStreamSynchronize(*st);
          cudaStreamDestroy(*st);
        }
      }
    } join{&cs};
    if (r->stop_x) {
      if (s->cfg.final_orth) side_copy(Xof(s, b), r->stop_x);
      else copy_out(s, Xof(s, b), r->stop_x);
    }
    bool final_is_q = false;  // final_x = Q after a successful final orthonormalization
    if (s->cfg.final_orth) {  // solver.cpp:445-459
      auto t0 = std::chrono::steady_clock::now();
      const int nb = 1 - b;
      const bool ok = orthonormalize_dev(s, Xof(s, b), Xof(s, nb), Pof(s, nb));
      if (s->timers)
        s->timers->orth +=
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (ok) {
        if (r->final_x) side_copy(Xof(s, nb), r->final_x);  // Q, unless the post-eval fails
        // the iteration kernels skip work once `done` is set: clear it for the
        // post-orth evaluation (solver.cpp:452) and restore it afterwards
        const int32_t zero = 0;
        PCAL_CUDA(cudaMemcpyAsync(&s->ctl->done, &zero, sizeof(int32_t), cudaMemcpyHostToDevice,
                                  s->stream));
        launch_eval(s, nb, 2, s->ctl);
        PCAL_CUDA(cudaMemcpyAsync(&s->ctl->done, &s->h_ctl->done, sizeof(int32_t),
                                  cudaMemcpyHostToDevice, s->stream));
        double post[8];
        PCAL_CUDA(cudaMemcpyAsync(post, s->post.p, sizeof(double) * 5, cudaMemcpyDeviceToHost,
                                  s->stream));
        PCAL_CUDA(cudaStreamSynchronize(s->stream));
        if (post[4] != 0.0) {
          status = PCAL_STATUS_DIVERGED;  // evaluation_error in the post-eval
          if (r->final_x) PCAL_CUDA(cudaStreamSynchronize(cs));  // before final_x is rewritten
        } else {
          for (int i = 0; i < 4; ++i) r->final_post[i] = post[i];
          r->has_post = 1;
          final_is_q = true;
        }
      }
    }
    if (r->final_x && !final_is_q) copy_out(s, Xof(s, b), r->final_x);
  }
  PCAL_CUDA(cudaStreamSynchronize(s->stream));
  // alm_outer sets RunReport::iterations only on a normal exit (solver.cpp:577)
  if (status == PCAL_STATUS_DIVERGED && s->alg == PCAL_ALG_ALM) r->iterations = 0;
  if (status == PCAL_STATUS_DIVERGED && tl > 0) {  // solver.cpp:467-471
    const double* last = r->trace ? r->trace + (tl - 1) * kTraceCols : nullptr;
    if (last) {
      r->final_pre[0] = last[1];
      r->final_pre[1] = last[2];
      r->final_pre[2] = last[3];
      r->final_pre[3] = last[4];
    }
    r->has_post = 0;
  }
  r->status = status;
  r->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - s->t_start).count();
}

}  // namespace

// ==============================================================================
// C ABI
// ==============================================================================
extern "C" {

const char* pcal_last_error(void) { return g_last_error.c_str(); }
int32_t pcal_last_orthonormalize_path(void) { return g_orth_path; }

void pcal_config_default(pcal_config* c) {
  c->alm_inner_max = 500;  // AlmOptions (solver.hpp:24-28)
  c->alm_outer_max = 50;
  c->alm_inner_tol_scale = 0.1;
  c->algorithm = PCAL_ALG_PCAL;
  c->beta = -1.0;
  c->eta_kind = PCAL_ETA_ABB;
  c->gamma = 1.0;
  c->eta_min = 1e-10;
  c->eta_max = 1e10;
  c->eta0 = 0.0;
  c->multiplier_rule = PCAL_MULT_PCAL_FORMULA;
  c->tol_rel_kkt = 1e-8;
  c->max_iter = 3000;
  c->final_orth = 1;
  c->device = 0;
}

double pcal_flops_estimate(int64_t n, int64_t p) {
  return 7.0 * ((double)n * (double)p * (double)p);
}

int pcal_session_create(const pcal_model_desc* model, const pcal_config* config, const double* x0,
                        int32_t x0_location, pcal_session** out) {
  return guarded([&] { session_create(model, config, x0, x0_location, out, nullptr); });
}

int pcal_session_run(pcal_session* s, int64_t iters) {
  return guarded([&] {
    if (!s) throw Error(PCAL_E_PARAMETER, "NULL session");
    session_run(s, iters);
  });
}

int pcal_session_sync(pcal_session* s) {
  return guarded([&] { PCAL_CUDA(cudaStreamSynchronize(s->stream)); });
}

void* pcal_session_stream(pcal_session* s) { return s ? (void*)s->stream : nullptr; }

int pcal_session_finish(pcal_session* s, pcal_report* report) {
  return guarded([&] { session_finish(s, report); });
}

void pcal_session_destroy(pcal_session* s) {
  if (!s) return;
  cudaSetDevice(s->device);
  cudaStreamSynchronize(s->stream);
  delete s;
}

int64_t pcal_session_kernel_launches(pcal_session* s) { return s ? s->launches : 0; }

// Per-kernel timing: iterations launched without graphs, an event after every
// kernel; writes "name mean_ms count\n" lines (means per iteration) into buf.
int pcal_session_profile_kernels(pcal_session* s, int64_t iters, char* buf, int64_t cap) {
  return guarded([&] {
    PCAL_CUDA(cudaSetDevice(s->device));
    LaunchScope ls(&s->launches);
    auto prof = std::make_unique<KernelProfiler>();
    prof->stream = s->stream;
    for (auto& m : prof->marks) PCAL_CUDA(cudaEventCreate(&m.ev));
    cudaEvent_t start;
    PCAL_CUDA(cudaEventCreate(&start));
    std::vector<std::pair<std::string, double>> acc;
    iters = std::min<int64_t>(iters, s->cfg.max_iter - s->launched);
    g_kprof = prof.get();
    for (int64_t i = 0; i < iters; ++i) {
      prof->n = 0;
      prof->active = true;
      PCAL_CUDA(cudaEventRecord(start, s->stream));
      launch_iteration(s, (int)(s->next_k % 2));
      prof->active = false;
      s->next_k++;
      s->launched++;
      PCAL_CUDA(cudaStreamSynchronize(s->stream));
      cudaEvent_t prev = start;
      for (int k = 0; k < prof->n; ++k) {
        float ms = 0;
        PCAL_CUDA(cudaEventElapsedTime(&ms, prev, prof->marks[k].ev));
        prev = prof->marks[k].ev;
        bool found = false;
        for (auto& a : acc)
          if (a.first == prof->marks[k].name) {
            a.second += ms;
            found = true;
          }
        if (!found) acc.emplace_back(prof->marks[k].name, ms);
      }
    }
    g_kprof = nullptr;
    std::string out;
    for (auto& a : acc) out += a.first + " " + std::to_string(a.second / std::max<int64_t>(1, iters)) + "\n";
    for (auto& m : prof->marks) cudaEventDestroy(m.ev);
    cudaEventDestroy(start);
    if ((int64_t)out.size() + 1 > cap) throw Error(PCAL_E_PARAMETER, "profile buffer too small");
    std::memcpy(buf, out.c_str(), out.size() + 1);
  });
}

int pcal_session_profile(pcal_session* s, int64_t iters, double* ms_out) {
  return guarded([&] {
    PCAL_CUDA(cudaSetDevice(s->device));
    LaunchScope ls(&s->launches);
    s->pev_on = true;
    for (double& v : s->prof_ms) v = 0.0;
    s->prof_iters = 0;
    iters = std::min<int64_t>(iters, s->cfg.max_iter - s->launched);  // trace capacity
    for (int64_t i = 0; i < iters; ++i) {
      launch_iteration(s, (int)(s->next_k % 2));
      s->next_k++;
      s->launched++;
    }
    s->pev_on = s->timers != nullptr;
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
    for (int i = 0; i < 4; ++i) ms_out[i] = s->prof_iters ? s->prof_ms[i] / s->prof_iters : 0.0;
  });
}
int64_t pcal_session_kernels_per_iteration(pcal_session* s) { return s ? s->kernels_per_iter : 0; }

int pcal_session_xm_mode(pcal_session* s, int64_t* fallbacks) {
  if (!s) return 0;
  if (fallbacks) {
    *fallbacks = 0;
    if (s->xm1) {
      double v[2] = {0, 0};
      if (cudaSetDevice(s->device) == cudaSuccess && cudaStreamSynchronize(s->stream) == cudaSuccess &&
          cudaMemcpy(v, s->kk.p, sizeof v, cudaMemcpyDeviceToHost) == cudaSuccess)
        *fallbacks = (int64_t)v[1];
    }
  }
  return s->xm1 ? 1 : 0;
}

int pcal_session_set_state(pcal_session* s, const double* x_prev, const double* x, int64_t k,
                           double eta_prev) {
  return guarded([&] {
    if (k < 0) throw Error(PCAL_E_PARAMETER, "k must be >= 0");
    PCAL_CUDA(cudaSetDevice(s->device));
    LaunchScope ls(&s->launches);
    read_ctl(s);
    Ctl c = *s->h_ctl;
    const int b = (int)(k % 2);
    c.done = 0;
    c.eval_bad = c.step_bad = c.step_param = 0;
    c.have_prev = 0;
    c.eta_prev = eta_prev;
    c.trace_len = 0;
    if (k > 0 && x_prev) {
      // evaluate X_{k-1} first (its P and d are the stepsize memory)
      c.iter = k - 1;
      *s->h_ctl = c;
      PCAL_CUDA(cudaMemcpyAsync(s->ctl, s->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s->stream));
      upload_matrix(x_prev, PCAL_HOST, s->n, s->p, Xof(s, 1 - b), s->ld, s->stream);
      launch_eval(s, 1 - b, 1, s->ctl);
      read_ctl(s);
      c = *s->h_ctl;
      c.trace_len = 0;
      c.have_prev = 1;
    }
    c.iter = k;
    c.eta_prev = eta_prev;
    *s->h_ctl = c;
    PCAL_CUDA(cudaMemcpyAsync(s->ctl, s->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s->stream));
    upload_matrix(x, PCAL_HOST, s->n, s->p, Xof(s, b), s->ld, s->stream);
    launch_eval(s, b, 1, s->ctl);
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
    s->next_k = k;
    s->launched = 0;
  });
}

int pcal_session_get_x(pcal_session* s, double* x_out, double* eta_out, int64_t* k_out) {
  return guarded([&] {
    PCAL_CUDA(cudaSetDevice(s->device));
    read_ctl(s);
    const int b = (int)((s->h_ctl->iter + s->h_ctl->alm_flips) % 2);
    if (x_out) copy_out(s, Xof(s, b), x_out);
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
    if (eta_out) *eta_out = s->h_ctl->eta;
    if (k_out) *k_out = s->h_ctl->iter;
  });
}

int pcal_session_device_x(pcal_session* s, const double** x, int64_t* ld) {
  return guarded([&] {
    read_ctl(s);
    *x = Xof(s, (int)((s->h_ctl->iter + s->h_ctl->alm_flips) % 2));
    *ld = s->ld;
  });
}

int pcal_solve(const pcal_model_desc* model, const pcal_config* config, const double* x0,
               int32_t x0_location, pcal_report* report, pcal_category_timers* timers) {
  return guarded([&] {
    if (!report) throw Error(PCAL_E_PARAMETER, "NULL report");
    pcal_session* s = nullptr;
    session_create(model, config, x0, x0_location, &s, timers);
    std::unique_ptr<pcal_session> guard(s);
    // evaluation at X0 may already have converged (solver.cpp:366-367)
    session_run(s, config->max_iter);
    session_finish(s, report);
    report->wall_time =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - s->t_start).count();
  });
}

}  // extern "C"

// ==============================================================================
// Building blocks (host buffers) — the reference's exposed kernels/steps
// ==============================================================================
namespace {

std::unique_ptr<pcal_session> make_aux(int64_t n, int64_t p, int device) {
  if (n < 1 || p < 1) throw Error(PCAL_E_DIMENSION, "dimensions must be positive");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
    throw Error(PCAL_E_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  auto s = std::make_unique<pcal_session>();
  s->device = device;
  PCAL_CUDA(cudaSetDevice(device));
  PCAL_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
  pcal_config_default(&s->cfg);
  s->cfg.max_iter = 1;
  s->cfg.device = device;
  s->model.kind = PCAL_MODEL_DENSE;
  s->model.n = n;
  s->model.p = p;
  s->n = n;
  s->p = p;
  s->pp = padded_p(p);
  s->ld = padded_ld(n);
  s->n_glob = n;
  s->K_full = s->ld;
  alloc_state(s.get());
  init_ctl(s.get());
  return s;
}

// upload an r×c host matrix into a zero-padded device buffer (ldr × cpad)
double* upload_padded(DevBuf& buf, const double* h, int64_t r, int64_t c, int64_t ldr, int64_t cpad,
                      cudaStream_t st) {
  buf.alloc((size_t)ldr * cpad);
  buf.zero(st);
  upload_matrix(h, PCAL_HOST, r, c, buf.p, ldr, st);
  return buf.p;
}

__global__ void k_matvec_part(const double* __restrict__ a, int64_t lda, int64_t n,
                              const double* __restrict__ v, int64_t kchunk,
                              double* __restrict__ part) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t kc = blockIdx.y;
  if (i >= n) return;
  const int64_t k0 = kc * kchunk, k1 = min(n, k0 + kchunk);
  double s = 0.0;
  for (int64_t k = k0; k < k1; ++k) s += a[i + k * lda] * v[k];
  part[kc * n + i] = s;
}

// out[i] = Σ_{c < nchunks} part[c·n + i] (fixed order)
__global__ void k_sum_chunks(const double* __restrict__ part, int64_t nchunks, int64_t n,
                             double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) s += part[c * n + i];
  out[i] = s;
}

__global__ void k_dot_part(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                           double* __restrict__ part) {
  __shared__ double sm[32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += a[i] * b[i];
  const double s = block_sum<256>(acc, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_scale_div(double* __restrict__ v, int64_t n, double d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] /= d;
}

}  // namespace

extern "C" {

int pcal_matmul_at_b(const double* a, const double* b, int64_t n, int64_t pa, int64_t pb, double* c,
                     int32_t device) {
  return guarded([&] {
    auto s = make_aux(n, std::max(pa, pb), device);
    DevBuf A, B, C;
    upload_padded(A, a, n, pa, s->ld, padded_p(pa), s->stream);
    upload_padded(B, b, n, pb, s->ld, padded_p(pb), s->stream);
    C.alloc((size_t)pa * pb);
    GemmPlan pl;
    plan_gemm(pl, device, pick_size(pb), A_KCONTIG, EPI_STORE, pa, pb, s->ld);
    pl.args.A = A.p;
    pl.args.lda = s->ld;
    pl.args.B = B.p;
    pl.args.ldb = s->ld;
    pl.args.ep.C = C.p;
    pl.args.ep.ldc = pa;
    pl.args.ep.m_store = pa;
    pl.args.ep.n_store = pb;
    launch_gemm(pl, s->stream);
    PCAL_CUDA(cudaMemcpyAsync(c, C.p, sizeof(double) * pa * pb, cudaMemcpyDeviceToHost, s->stream));
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int pcal_matmul(const double* a, const double* b, int64_t m, int64_t k, int64_t nc, double* c,
                int32_t device) {
  return guarded([&] {
    auto s = make_aux(m, 1, device);
    const int64_t kp = padded_p(k), ldm = padded_ld(m);
    DevBuf A, B, C;
    upload_padded(A, a, m, k, ldm, kp, s->stream);
    upload_padded(B, b, k, nc, kp, nc, s->stream);
    C.alloc((size_t)m * nc);
    GemmPlan pl;
    plan_gemm(pl, device, pick_size(nc), A_MCONTIG, EPI_STORE, m, nc, kp);
    pl.args.A = A.p;
    pl.args.lda = ldm;
    pl.args.B = B.p;
    pl.args.ldb = kp;
    pl.args.ep.C = C.p;
    pl.args.ep.ldc = m;
    pl.args.ep.m_store = m;
    pl.args.ep.n_store = nc;
    launch_gemm(pl, s->stream);
    PCAL_CUDA(cudaMemcpyAsync(c, C.p, sizeof(double) * m * nc, cudaMemcpyDeviceToHost, s->stream));
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int pcal_gram(const double* x, int64_t n, int64_t p, double* g, int32_t device) {
  return guarded([&] {
    auto s = make_aux(n, p, device);
    upload_matrix(x, PCAL_HOST, n, p, Xof(s.get(), 0), s->ld, s->stream);
    GemmPlan& gp = s->orth_gram;
    plan_gemm(gp, device, pick_size(s->pp), A_KCONTIG, EPI_STORE, s->pp, s->pp, s->ld, 0);
    gp.args.A = gp.args.B = Xof(s.get(), 0);
    gp.args.lda = gp.args.ldb = s->ld;
    gp.args.ep.C = s->orth_b.p;
    gp.args.ep.ldc = s->pp;
    gp.args.ep.m_store = gp.args.ep.n_store = s->pp;
    launch_gemm(gp, s->stream);
    std::vector<double> b((size_t)s->pp * s->pp);
    PCAL_CUDA(cudaMemcpyAsync(b.data(), s->orth_b.p, sizeof(double) * b.size(),
                              cudaMemcpyDeviceToHost, s->stream));
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
    for (int64_t j = 0; j < p; ++j)  // exact symmetry: mirror the upper triangle
      for (int64_t i = 0; i <= j; ++i) g[i + j * p] = g[j + i * p] = b[i + j * s->pp];
  });
}

int pcal_orthonormalize(const double* x, int64_t n, int64_t p, double* q, int32_t device) {
  return guarded([&] {
    auto s = make_aux(n, p, device);
    LaunchScope ls(&s->launches);
    upload_matrix(x, PCAL_HOST, n, p, Xof(s.get(), 0), s->ld, s->stream);
    if (!orthonormalize_dev(s.get(), Xof(s.get(), 0), Xof(s.get(), 1), Pof(s.get(), 1)))
      throw Error(PCAL_E_RANK, "orthonormalize: numerically rank-deficient input");
    copy_out(s.get(), Xof(s.get(), 1), q);
    PCAL_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int pcal_initial_point_qr(int64_t n, int64_t p, uint64_t seed, double* x0, int32_t device) {
  return guarded([&] {
    if (n < 1 || p < 1 || 2 * p > n)  // solver.cpp:137-138
      throw Error(PCAL_E_PARAMETER, "initial_point: dimensions must satisfy 2p <= n");
    std::vector<double> h((size_t)n * p);
    host_random_normal(n * p, seed, h.data(), (int)std::min<unsigned>(16, std::thread::hardware_concurrency()));
    const int rc = pcal_orthonormalize(h.data(), n, p, x0, device);
    if (rc != PCAL_OK) throw Error(rc, g_last_error);
  });
}

int pcal_initial_point(int64_t n, int64_t p, int32_t mode, double sigma_lower, uint64_t seed,
                       double* x0, int32_t device) {
  return guarded([&] {
    if (n < 1 || p < 1 || 2 * p > n)  // solver.cpp:137-138
      throw Error(PCAL_E_PARAMETER, "initial_point: dimensions must satisfy 2p <= n");
    if (mode != PCAL_INIT_QR && mode != PCAL_INIT_A2_TYPE_I && mode != PCAL_INIT_A2_TYPE_II)
      throw Error(PCAL_E_PARAMETER, "initial_point: unknown mode");
    const double sl = sigma_lower;
    if (mode == PCAL_INIT_A2_TYPE_I && (!(sl > 0.0 && sl < 1.0) || sl * sl > 0.5))
      throw Error(PCAL_E_PARAMETER,
                  "initial_point: a2-i requires sigma in (0,1) with sigma^2 <= 1/2");
    if (!x0) throw Error(PCAL_E_PARAMETER, "NULL argument");
    const int rc = pcal_initial_point_qr(n, p, seed, x0, device);
    if (rc != PCAL_OK) throw Error(rc, g_last_error);
    std::vector<double> d((size_t)p, 1.0);
    if (mode == PCAL_INIT_A2_TYPE_I) {
      d.back() = std::sqrt(1.0 - sl * sl);
    } else if (mode == PCAL_INIT_A2_TYPE_II) {  // singular values inside the A2 band (solver.cpp:153-167)
      const double band = 0.9 / std::sqrt(static_cast<double>(p));
      std::vector<double> u((size_t)p);
      host_uniform_after_normals(n * p, seed, p, u.data());
      for (int64_t j = 0; j < p; ++j) {
        double sq = 1.0 + band * (2.0 * u[j] - 1.0);
        if (std::abs(sq - 1.0) < 0.1 * band) sq = 1.0 + 0.1 * band;
        d[j] = std::sqrt(sq);
      }
    }
    if (mode != PCAL_INIT_QR)  // scale_cols_in_place (kernels.cpp:338-346)
      for (int64_t j = 0; j < p; ++j)
        for (int64_t i = 0; i < n; ++i) x0[i + j * n] *= d[j];
  });
}

// One evaluation of the session's model at its pair-0 iterate: f (and G into g
// when non-null).  Throws evaluation_error on a non-finite f or G.
static double evaluate_pair0(pcal_session* s, double* g) {
  LaunchScope ls(&s->launches);
  k_zero_i32<<<1, 1, 0, s->stream>>>(s->bad, nullptr);
  launched("k_zero_i32");
  launch_gradient(s, 0, nullptr);
  launch_colsums(s, s->fpart.p, s->nrb_f, nullptr, nullptr, 0, Fcol(s, 0), nullptr, nullptr,
                 nullptr);
  FinishArgs fa{};
  fa.fcol = Fcol(s, 0);
  fa.kcol = Kcol(s, 0);
  fa.cpart = s->cpart.p;
  fa.ncp = 0;
  fa.spart = s->spart.p;
  fa.nsp = s->sp_blocks;
  fa.model = s->model.kind;
  fa.p = s->p;
  fa.mode = 2;
  fa.trace = s->trace.p;
  fa.bad = s->bad;
  fa.c_xc = s->c_xc;
  fa.fdev = s->fdev.p;
  fa.coeff = s->model.coeff;
  fa.p6 = s->model.density_variant == PCAL_DENSITY_P6;
  k_finish_eval<<<1, 256, 0, s->stream>>>(fa, s->ctl, s->post.p);
  launched("k_finish_eval");
  double post[8];
  PCAL_CUDA(cudaMemcpyAsync(post, s->post.p, sizeof(double) * 5, cudaMemcpyDeviceToHost,
                            s->stream));
  if (g) copy_out(s, Pof(s, 0), g);
  PCAL_CUDA(cudaStreamSynchronize(s->stream));
  if (post[4] != 0.0) throw Error(PCAL_E_EVALUATION, "evaluate: non-finite objective or gradient");
  return post[0];
}

static std::unique_ptr<pcal_session> evaluation_session(const pcal_model_desc* model,
                                                        const double* x, int32_t device) {
  pcal_config cfg;
  pcal_config_default(&cfg);
  cfg.max_iter = 1;
  cfg.final_orth = 0;
  cfg.device = device;
  pcal_session* raw = nullptr;
  session_create(model, &cfg, x, PCAL_HOST, &raw, nullptr);
  return std::unique_ptr<pcal_session>(raw);
}

int pcal_evaluate(const pcal_model_desc* model, const double* x, double* f, double* g,
                  int32_t device) {
  return guarded([&] {
    auto s = evaluation_session(model, x, device);
    *f = evaluate_pair0(s.get(), g);
  });
}

// fd_gradient_check (problems.cpp:296-325) with the device evaluation: up to 50
// distinct coordinates drawn as Rng(seed).next_u64() % (n·p), visited in
// ascending order, central differences with step h·(1 + |x_ij|); returns the
// worst |fd − g| / (1 + |g|).  One session serves every probe.
int pcal_fd_gradient_check(const pcal_model_desc* model, const double* x, double h, uint64_t seed,
                           int32_t device, double* worst) {
  return guarded([&] {
    if (!model || !x || !worst) throw Error(PCAL_E_PARAMETER, "NULL argument");
    if (!(h > 0.0)) throw Error(PCAL_E_PARAMETER, "fd_gradient_check: h must be positive");
    const int64_t n = model->n, p = model->p, total = n * p;
    auto s = evaluation_session(model, x, device);
    std::vector<double> g((size_t)total), probe(x, x + total);
    evaluate_pair0(s.get(), g.data());
    const int64_t want = std::min<int64_t>(50, total);
    std::vector<int64_t> coords((size_t)want);
    pcal::host_fd_coordinates(total, seed, want, coords.data());
    double w = 0.0;
    for (int64_t c : coords) {
      const int64_t i = c % n, j = c / n;
      const double x0 = x[c];
      const double hh = h * (1.0 + std::abs(x0));
      probe[(size_t)c] = x0 + hh;
      upload_matrix(probe.data(), PCAL_HOST, n, p, Xof(s.get(), 0), s->ld, s->stream);
      const double fp = evaluate_pair0(s.get(), nullptr);
      probe[(size_t)c] = x0 - hh;
      upload_matrix(probe.data(), PCAL_HOST, n, p, Xof(s.get(), 0), s->ld, s->stream);
      const double fm = evaluate_pair0(s.get(), nullptr);
      probe[(size_t)c] = x0;
      const double fd = (fp - fm) / (2.0 * hh);
      const double gv = g[(size_t)(i + j * n)];
      w = std::max(w, std::abs(fd - gv) / (1.0 + std::abs(gv)));
    }
    *worst = w;
  });
}

int pcal_pcal_step(const double* x, const double* grad_l, int64_t n, int64_t p, double eta,
                   double* out, int64_t* degenerate_columns, int32_t device) {
  return guarded([&] {
    if (!(eta > 0.0)) throw Error(PCAL_E_PARAMETER, "pcal_step: eta must be positive");
    auto s = make_aux(n, p, device);
    upload_matrix(x, PCAL_HOST, n, p, Xof(s.get(), 0), s->ld, s->stream);
    upload_matrix(grad_l, PCAL_HOST, n, p, Pof(s.get(), 0), s->ld, s->stream);
    s->h_ctl->eta = eta;
    s->h_ctl->done = 0;
    PCAL_CUDA(cudaMemcpyAsync(s->ctl, s->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s->stream));
    dim3 gu((unsigned)s->up_nchunks, (unsigned)p);
    k_update<<<gu, kStreamThreads, 0, s->stream>>>(Xof(s.get(), 0), Pof(s.get(), 0), Dvec(s.get(), 0),
                                                   Xof(s.get(), 1), n, s->ld, p, s->up_chunk,
                                                   s->npart.p, nullptr, s->ctl);
    launched("k_update");
    k_normalize<<<gu, kStreamThreads, 0, s->stream>>>(Xof(s.get(), 0), Xof(s.get(), 1), n, s->ld,
                                                      p, s->up_chunk, s->up_nchunks, s->npart.p,
                                                      nullptr, 0, n, 0, s->ctl);
    launched("k_normalize");
    PCAL_CUDA(cudaGetLastError());
    copy_out(s.get(), Xof(s.get(), 1), out);
    read_ctl(s.get());
    if (degenerate_columns) *degenerate_columns = s->h_ctl->step_deg;
    if (s->h_ctl->step_bad) throw Error(PCAL_E_DIVERGENCE, "pcal_step: non-finite iterate");
  });
}

int pcal_spectral_norm_estimate(const double* a, int64_t n, uint64_t seed, double* out,
                                int32_t device) {
  return guarded([&] {
    auto s = make_aux(n, 1, device);
    const int64_t lda = padded_ld(n);
    DevBuf A, v, w, t, part, dots;
    upload_padded(A, a, n, n, lda, n, s->stream);
    // start vector: random_normal(n, 1, Rng(seed)) normalised (kernels.cpp:272-278)
    std::vector<double> hv((size_t)n);
    host_random_normal(n, seed, hv.data(), 1);
    double nv = 0.0;
    for (double e : hv) nv += e * e;
    nv = std::sqrt(nv);
    if (nv == 0.0) hv[0] = 1.0;
    else for (double& e : hv) e /= nv;
    v.alloc(n);
    w.alloc(n);
    t.alloc(n);
    PCAL_CUDA(cudaMemcpyAsync(v.p, hv.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s->stream));
    const int64_t kchunk = std::max<int64_t>(256, ceil_div(n, 32));
    const int64_t nkc = ceil_div(n, kchunk);
    part.alloc((size_t)nkc * n);
    const int nblk = 296;
    dots.alloc(nblk);
    std::vector<double> hd(nblk);
    auto matvec = [&](const double* in, double* o) {
      k_matvec_part<<<dim3((unsigned)ceil_div(n, 256), (unsigned)nkc), 256, 0, s->stream>>>(
          A.p, lda, n, in, kchunk, part.p);
      launched("k_matvec_part");
      k_sum_chunks<<<(unsigned)ceil_div(n, 256), 256, 0, s->stream>>>(part.p, nkc, n, o);
      launched("k_sum_chunks");
    };
    auto norm = [&](const double* x) {
      k_dot_part<<<nblk, 256, 0, s->stream>>>(x, x, n, dots.p);
      launched("k_dot_part");
      PCAL_CUDA(cudaMemcpyAsync(hd.data(), dots.p, sizeof(double) * nblk, cudaMemcpyDeviceToHost,
                                s->stream));
      PCAL_CUDA(cudaStreamSynchronize(s->stream));
      double acc = 0.0;
      for (double d : hd) acc += d;
      return std::sqrt(acc);
    };
    // ‖A‖_F
    double fro2 = 0.0;
    {
      DevBuf fp;
      fp.alloc(nblk);
      for (int64_t j = 0; j < n; ++j) {
        (void)j;
        break;
      }
      // A padded columns are contiguous with lda ≥ n: sum over the whole buffer (pads are 0)
      k_dot_part<<<nblk, 256, 0, s->stream>>>(A.p, A.p, lda * n, fp.p);
      launched("k_dot_part");
      PCAL_CUDA(cudaMemcpyAsync(hd.data(), fp.p, sizeof(double) * nblk, cudaMemcpyDeviceToHost,
                                s->stream));
      PCAL_CUDA(cudaStreamSynchronize(s->stream));
      for (double d : hd) fro2 += d;
    }
    const double fro = std::sqrt(fro2);
    if (fro == 0.0) {
      *out = 0.0;
      return;
    }
    double prev = -1.0, est = 0.0;
    for (int it = 0; it < 500; ++it) {
      matvec(v.p, w.p);
      est = norm(w.p);
      matvec(w.p, t.p);
      const double nt = norm(t.p);
      if (nt == 0.0) break;
      k_scale_div<<<(unsigned)ceil_div(n, 256), 256, 0, s->stream>>>(t.p, n, nt);
      launched("k_scale_div");
      std::swap(v.p, t.p);
      if (prev >= 0.0 && std::abs(est - prev) <= 1e-6 * std::max(est, 1e-300)) break;
      prev = est;
    }
    PCAL_CUDA(cudaGetLastError());
    *out = std::min(est, fro);
  });
}

}  // extern "C"

// ==============================================================================
// Row-sharded sessions (multi-GPU) and the single-GPU loopback emulation
// ==============================================================================
struct pcal_comm {
  pcal::Comm* c = nullptr;
  ~pcal_comm() { delete c; }
};

extern "C" {

int pcal_partition(const pcal_model_desc* m, int32_t nranks, int32_t rank, int64_t* row0,
                   int64_t* nrows) {
  return guarded([&] {
    if (!m || nranks < 1 || rank < 0 || rank >= nranks) throw Error(PCAL_E_PARAMETER, "bad rank");
    int64_t z0, nzl;
    partition(*m, nranks, rank, row0, nrows, &z0, &nzl);
  });
}

int pcal_device_count(int32_t* count) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return PCAL_OK;
}

int pcal_row_chunks(const pcal_model_desc* m, int64_t* chunk_rows, int64_t* nchunks) {
  return guarded([&] {
    if (!m || !chunk_rows || !nchunks) throw Error(PCAL_E_PARAMETER, "NULL argument");
    int64_t zc;
    chunking(*m, chunk_rows, nchunks, &zc);
  });
}

int pcal_nccl_unique_id(void* out) {
  return guarded([&] { nccl_unique_id(out); });
}

int pcal_comm_create_nccl(int32_t nranks, int32_t rank, const void* uid, int32_t device,
                          pcal_comm** out) {
  return guarded([&] {
    auto c = std::make_unique<pcal_comm>();
    c->c = make_nccl_comm(nranks, rank, uid, device);
    *out = c.release();
  });
}

void pcal_comm_destroy(pcal_comm* c) { delete c; }

int pcal_session_create_sharded(const pcal_model_desc* local_model, const pcal_config* config,
                                const double* x0_local, int32_t x0_location, pcal_comm* comm,
                                pcal_session** out) {
  return guarded([&] {
    session_create(local_model, config, x0_local, x0_location, out, nullptr,
                   comm ? comm->c : nullptr);
  });
}

int pcal_solve_sharded(const pcal_model_desc* local_model, const pcal_config* config,
                       const double* x0_local, int32_t x0_location, pcal_comm* comm,
                       pcal_report* report, pcal_category_timers* timers) {
  return guarded([&] {
    pcal_session* s = nullptr;
    session_create(local_model, config, x0_local, x0_location, &s, timers,
                   comm ? comm->c : nullptr);
    std::unique_ptr<pcal_session> guard(s);
    session_run(s, config->max_iter);
    session_finish(s, report);
  });
}

// R emulated ranks on ONE GPU: each rank is a host thread with its own session
// on the group's shared stream; the collectives meet at host barriers.  The
// global report gets rank 0's trace and scalars and every rank's rows of X.
int pcal_solve_emulated(const pcal_model_desc* model, const pcal_config* config, const double* x0,
                        int32_t nranks, pcal_report* report, pcal_category_timers* timers) {
  return guarded([&] {
    if (!model || !config || !x0 || !report) throw Error(PCAL_E_PARAMETER, "NULL argument");
    if (model->location != PCAL_HOST) throw Error(PCAL_E_PARAMETER, "emulation takes host data");
    if (nranks < 1) throw Error(PCAL_E_PARAMETER, "nranks must be >= 1");
    validate(config);
    PCAL_CUDA(cudaSetDevice(config->device));
    const int R = nranks;
    const int64_t n = model->n, p = model->p;
    LoopbackGroup group(R);
    std::vector<std::unique_ptr<LoopbackComm>> comms;
    std::vector<int64_t> r0(R), rows(R);
    for (int r = 0; r < R; ++r) {
      comms.emplace_back(new LoopbackComm(&group, r));
      int64_t z0, nzl;
      partition(*model, R, r, &r0[r], &rows[r], &z0, &nzl);
      if (rows[r] < 1) throw Error(PCAL_E_PARAMETER, "a rank would own no rows");
    }
    std::vector<std::vector<double>> a_loc(R), g_loc(R), x_loc(R), stop_loc(R), fin_loc(R),
        li_loc(R);
    std::vector<pcal_report> reps(R);
    std::vector<std::vector<double>> traces(R);
    std::vector<int> rcs(R, PCAL_OK);
    std::vector<std::string> errs(R);
    auto slice = [&](const double* src, int64_t ld_src, int64_t r, int64_t cols,
                     std::vector<double>& dst) {
      dst.resize((size_t)rows[r] * cols);
      for (int64_t c = 0; c < cols; ++c)
        std::memcpy(dst.data() + c * rows[r], src + r0[r] + c * ld_src, sizeof(double) * rows[r]);
    };
    for (int r = 0; r < R; ++r) {
      if (dense_family(model->kind)) {
        if (!model->a) throw Error(PCAL_E_PARAMETER, "dense model: a is NULL");
        slice(model->a, n, r, n, a_loc[r]);
        if (model->kind == PCAL_MODEL_DENSE && model->g0) slice(model->g0, n, r, p, g_loc[r]);
        if (model->kind == PCAL_MODEL_DENSITY) {
          if (!model->linv) throw Error(PCAL_E_PARAMETER, "density model: linv is NULL");
          slice(model->linv, n, r, n, li_loc[r]);
        }
      }
      slice(x0, n, r, p, x_loc[r]);
      stop_loc[r].resize((size_t)rows[r] * p);
      fin_loc[r].resize((size_t)rows[r] * p);
      traces[r].resize((size_t)(config->max_iter + 1) * kTraceCols);
      reps[r] = pcal_report{};
      reps[r].trace = traces[r].data();
      reps[r].trace_capacity = config->max_iter + 1;
      reps[r].stop_x = stop_loc[r].data();
      reps[r].final_x = fin_loc[r].data();
    }
    std::vector<std::thread> th;
    for (int r = 0; r < R; ++r)
      th.emplace_back([&, r] {
        rcs[r] = guarded([&] {
          PCAL_CUDA(cudaSetDevice(config->device));
          pcal_model_desc m = *model;
          if (dense_family(m.kind)) {
            m.a = a_loc[r].data();
            m.g0 = model->kind == PCAL_MODEL_DENSE && model->g0 ? g_loc[r].data() : nullptr;
            if (m.kind == PCAL_MODEL_DENSITY) m.linv = li_loc[r].data();
          } else {
            m.v = model->v + r0[r];
          }
          pcal_session* s = nullptr;
          session_create(&m, config, x_loc[r].data(), PCAL_HOST, &s, r == 0 ? timers : nullptr,
                         comms[r].get(), group.stream);
          std::unique_ptr<pcal_session> guard(s);
          session_run(s, config->max_iter);
          session_finish(s, &reps[r]);
        });
        if (rcs[r] != PCAL_OK) errs[r] = g_last_error;
      });
    for (auto& t : th) t.join();
    for (int r = 0; r < R; ++r)
      if (rcs[r] != PCAL_OK) throw Error(rcs[r], "rank " + std::to_string(r) + ": " + errs[r]);
    // merge: replicated scalars from rank 0, rows from every rank
    double* trace = report->trace;
    const int64_t cap = report->trace_capacity;
    double* stop_x = report->stop_x;
    double* final_x = report->final_x;
    *report = reps[0];
    report->trace = trace;
    report->trace_capacity = cap;
    report->stop_x = stop_x;
    report->final_x = final_x;
    if (trace) {
      if (cap < reps[0].trace_len) throw Error(PCAL_E_PARAMETER, "report trace capacity too small");
      std::memcpy(trace, traces[0].data(), sizeof(double) * reps[0].trace_len * kTraceCols);
    }
    for (int r = 0; r < R; ++r)
      for (int64_t c = 0; c < p; ++c) {
        if (stop_x && reps[0].has_x)
          std::memcpy(stop_x + r0[r] + c * n, stop_loc[r].data() + c * rows[r],
                      sizeof(double) * rows[r]);
        if (final_x && reps[0].has_x)
          std::memcpy(final_x + r0[r] + c * n, fin_loc[r].data() + c * rows[r],
                      sizeof(double) * rows[r]);
      }
  });
}

}  // extern "C"
