// common.cuh — shared definitions for the B200 PCAL library (sm_100a, FP64).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>

namespace pcal {

// Thrown inside the library, converted to PCAL_E_* at the C ABI.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PCAL_CUDA(call)                                                               \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw ::pcal::Error(-5, std::string(#call) + ": " + cudaGetErrorString(e_) +    \
                                  " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

// Launch bookkeeping: every kernel this library launches is followed by
// launched(name), so sessions can report how many native kernels ran and the
// per-kernel profiler (pcal_session_profile_kernels) can time each one with an
// event recorded right after it on the same stream.
struct KernelProfiler {
  cudaStream_t stream = nullptr;
  bool active = false;
  struct Mark {
    const char* name;
    cudaEvent_t ev;
  };
  Mark marks[512];
  int n = 0;
};
extern thread_local int64_t* g_launch_counter;
extern thread_local KernelProfiler* g_kprof;
inline void launched(const char* name, int64_t k = 1) {
  if (g_launch_counter) *g_launch_counter += k;
  if (g_kprof && g_kprof->active && g_kprof->n < 512) {
    auto& m = g_kprof->marks[g_kprof->n++];
    m.name = name;
    cudaEventRecord(m.ev, g_kprof->stream);
  }
}
inline void count_launch(int64_t k = 1) {
  if (g_launch_counter) *g_launch_counter += k;
}

inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
inline int64_t ceil_div(int64_t v, int64_t m) { return (v + m - 1) / m; }

// Padding of every internal dimension that a GEMM contracts over: a multiple
// of the largest k-slice (32 doubles = 256 B).  Rows/columns are zero padded,
// so 16-byte cp.async chunks are aligned and padding contributes nothing to
// Grams or norms.
constexpr int64_t kPad = 32;
inline int64_t padded_ld(int64_t n) { return round_up(n, kPad); }
inline int64_t padded_p(int64_t p) { return round_up(p, kPad); }

constexpr int kTraceCols = 7;

// Device-resident control block of one PCAL run.  Every iteration kernel
// reads `done` first and exits when the run has stopped, so iteration graphs
// can be launched ahead of the stopping decision without a host round trip.
struct Ctl {
  // run state
  int64_t iter;        // index k of the current iterate X_k (trace row k recorded)
  int64_t trace_len;   // rows recorded
  int64_t degenerate;  // pcal_step degenerate columns (accumulated)
  int32_t done;        // 0 running, 1 converged, 2 diverged
  int32_t have_prev;   // X_{k-1}, GL_{k-1} available (stepsize memory)
  int32_t eval_bad;    // evaluation produced non-finite f/G
  int32_t step_bad;    // pcal_step produced a non-finite iterate
  int32_t step_param;  // pcal_step got eta <= 0 (parameter_error)
  int32_t step_deg;    // degenerate columns of the current step
  // scalars
  double eta;          // stepsize of the current step (η_k)
  double eta_prev;     // SolverState::eta (last stepsize used), 0 before the first step
  double eta0;
  double beta;
  double kkt_den;      // kkt_abs at X_0
  double f, kkt_abs, feas, rel;
  uint64_t t0_ns;      // %globaltimer at session start
  // configuration
  double tol, gamma, eta_min, eta_max;
  int32_t eta_kind;
  int32_t mult_rule;
  // stepsize memory: stepsize_select sees st.iter = iter − iter_base (0 except for
  // ALM, whose SolverState restarts with every inner loop, solver.cpp:540-543)
  int64_t iter_base;
  // ALM (alm_outer, solver.cpp:478-624); alm = 0 for every other algorithm
  int32_t alm;
  int32_t alm_phase;   // next action: 0 = inner step, 1 = multiplier update
  int32_t alm_met;     // the inner loop met its tolerance (else it hit a cap)
  int32_t alm_copy;    // the iterate just evaluated is the inner loop's best so far
  int64_t alm_inner;   // iterates tested in the current inner loop
  int64_t alm_outer;   // multiplier updates (RunReport::outer_iterations)
  int64_t alm_caps;    // inner loops stopped by a cap (RunReport::inner_cap_hits)
  int64_t alm_flips;   // multiplier updates performed (each moves the iterate to the other pair)
  int64_t alm_inner_max, alm_outer_max, max_iter;
  double alm_best, alm_tol_scale;
  double best_f, best_kkt, best_feas;  // data of the best iterate
};

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum in a fixed order (deterministic); result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* sm /* NT/32 */) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sm[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) r += sm[i];
  }
  return r;
}

}  // namespace pcal
