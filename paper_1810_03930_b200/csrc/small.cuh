// small.cuh — the whole PCAL iteration of a small dense problem as ONE
// persistent cooperative kernel (config 1: n = 1000, p = 20).
//
// At config-1 sizes every phase of the iteration is a few microseconds of
// work, so the 9-kernel graph is bound by launch gaps and tails.  This kernel
// keeps one CTA per SM resident for a whole batch of iterations and
// separates the dependent phases with grid-wide barriers
// (phases B, C, D, E, A below; 5 grid barriers per iteration).  The gradient
// runs on DMMA.8x8x4 and is fused with the column normalisation:
// G = (A·Z)·diag(1/‖z‖) — Z is scaled after the product, which changes the
// rounding order only (the parity tolerances of DESIGN.md §5 apply); a step
// with a degenerate column takes one extra barrier and uses X⁺ itself.
//
// Same arithmetic as the multi-kernel path up to summation order (all sums
// fixed-order, no atomics): solver.cpp:369-439 per iteration.
#pragma once

namespace pcal {

constexpr int kSmallThreads = 256;  // 8 warps
constexpr int kSmallP = 32;         // p ≤ 32 (one column per lane)

struct SmallArgs {
  double* pair[2];    // pair b: P = pair[b], X = pair[b] + ld·pp
  double* fkd[2];     // [f | kkt² | d] column sums per parity
  const double* at;   // Aᵀ (ldat × n): at[k + i·ldat] = A(i, k)
  int64_t ldat;
  const double* g0;   // linear term (ld) or null
  double* gr;         // (2pp) × pp: [GᵀX; XᵀX]
  double* lam;        // Λ (p × p) of the dual-ascent variants
  double* z;          // Z = X − (1/η)·GL (ld × p)
  double* part;       // [gridDim][3][kSmallP] CTA column partials (f, KKT², d)
  double* npb;        // [gridDim][kSmallP] CTA column partials of ‖z_j‖²
  double* bbpart;     // [gridDim][3] CTA partials of ⟨S,S⟩, ⟨S,Y⟩, ⟨Y,Y⟩
  int64_t n, ld, p, pp;
  int plain;          // PLAM / PLAM-DA: no column normalisation
  int mc_mode;        // MC_PCAL / MC_DA
  int p_from_g;       // P = G + X·M (dual ascent)
  int dform;          // d_j = X_jᵀP_j (PCAL with the PCAL formula)
  double beta;        // β
  double beta_epi;    // β of the P update (1 for dual ascent)
  FinishArgs fa;      // trace, bad flag, model (mode 0)
  int64_t lda_s;      // > 0: this CTA's 8 rows of A stay in shared memory (row stride)
  uint64_t* prof;     // optional: %globaltimer per phase boundary (CTA 0), [iters][8]
};

// Transposed reduction of 32 per-lane values: afterwards lane L holds
// Σ_lanes v[L] (fixed shuffle pattern ⇒ deterministic).
__device__ __forceinline__ double transpose_reduce32(double (&v)[kSmallP], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int q = 0; q < o; ++q) {
      const double send = upper ? v[q] : v[q + o];
      const double keep = upper ? v[q + o] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
  return v[0];
}

__device__ __forceinline__ void small_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Column sums over the CTAs of src[q·stride + j] (j = lane < p) in two fixed-
// order stages: warp w sums CTAs [20w, 20w+20) with every load issued before
// the first add (one round trip), then thread j sums the 8 warp partials.
// Result in out[j] (shared), valid after the trailing barrier.
__device__ __forceinline__ void cta_column_sums(const double* src, int64_t stride, int64_t p,
                                                double (*wsum)[kSmallP], double* out) {
  constexpr int W8 = kSmallThreads / 32, BPW = 20;  // gridDim ≤ 160
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v[BPW];
#pragma unroll
  for (int u = 0; u < BPW; ++u) {
    const int q = warp * BPW + u;
    v[u] = (q < (int)gridDim.x && lane < p) ? src[(int64_t)q * stride + lane] : 0.0;
  }
  double t = 0.0;
#pragma unroll
  for (int u = 0; u < BPW; ++u) t += v[u];
  wsum[warp][lane] = t;
  __syncthreads();
  if (threadIdx.x < kSmallP) {
    double r = 0.0;
#pragma unroll
    for (int w = 0; w < W8; ++w) r += wsum[w][threadIdx.x];
    out[threadIdx.x] = r;
  }
  __syncthreads();
}

// This CTA's partial ⟨S,S⟩, ⟨S,Y⟩, ⟨Y,Y⟩ over its rows (stepsize_select,
// solver.cpp:218-222): S = X − X_prev, Y = (P − d∘X) − (P_prev − d_prev∘X_prev).
__device__ __forceinline__ void bb_block(const double* x, const double* xp, const double* pg,
                                         const double* pgp, const double* d, const double* dp,
                                         int64_t r0, int64_t r1, int64_t ld, int64_t p,
                                         double* bbpart, double* sm8) {
  double ss = 0.0, sy = 0.0, yy = 0.0;
  const int64_t rows = r1 - r0;
  for (int64_t e = threadIdx.x; e < rows * p; e += blockDim.x) {
    const int64_t i = r0 + e % rows, j = e / rows;
    const int64_t ix = i + j * ld;
    const double xv = x[ix], xpv = xp[ix];
    const double sv = xv - xpv;
    const double yv = (pg[ix] - d[j] * xv) - (pgp[ix] - dp[j] * xpv);
    ss += sv * sv;
    sy += sv * yv;
    yy += yv * yv;
  }
  const double a = block_sum<kSmallThreads>(ss, sm8);
  const double b = block_sum<kSmallThreads>(sy, sm8);
  const double c = block_sum<kSmallThreads>(yy, sm8);
  if (threadIdx.x == 0) {
    bbpart[blockIdx.x * 3 + 0] = a;
    bbpart[blockIdx.x * 3 + 1] = b;
    bbpart[blockIdx.x * 3 + 2] = c;
  }
}

// G rows of 8-row tiles (round-robin over CTAs) = scale_j · (A·Y)(i, j) (+G0):
// the 8 warps split K, DMMA.8x8x4 over the ≤ 4 8-column tiles, K-partials
// summed in warp order; f partial per column accumulated into *fcol (thread j).
// xs_scale != null: the iterate is X = Y·diag(scale) (fused normalisation).
__device__ __forceinline__ void gradient_tiles(const SmallArgs& a, const double* Y,
                                               const double* scale, double* Pn,
                                               double (*sG)[4 * 64], double* sF, double& fcol,
                                               bool& bad, const double* sA) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r8 = lane >> 2, q4 = lane & 3;
  const int64_t n = a.n, ld = a.ld, p = a.p;
  const int ct_n = (int)((p + 7) / 8);
  const int64_t k4n = (n + 3) / 4;
  const int64_t k4b = warp * k4n / 8, k4e = (warp + 1) * k4n / 8;
  for (int64_t rt = blockIdx.x; rt * 8 < n; rt += gridDim.x) {
    const int64_t i0 = rt * 8;
    double c[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) c[t][0] = c[t][1] = 0.0;
    const bool rok = i0 + r8 < n;
    // A rows: resident in shared memory (one tile per CTA) or read from Aᵀ
    const double* arow = sA ? sA + r8 * a.lda_s : a.at + (rok ? (i0 + r8) * a.ldat : 0);
#pragma unroll 8
    for (int64_t k4 = k4b; k4 < k4e; ++k4) {
      const int64_t k = k4 * 4 + q4;
      const double av = rok ? arow[k] : 0.0;
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (t < ct_n) small_dmma(c[t][0], c[t][1], av, Y[k + (t * 8 + r8) * ld]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (t < ct_n) {
        sG[warp][t * 64 + r8 * 8 + 2 * q4] = c[t][0];
        sG[warp][t * 64 + r8 * 8 + 2 * q4 + 1] = c[t][1];
      }
    __syncthreads();
    // thread e = (column j, row r): G(i0 + r, j) = Σ_warps, in warp order
    const int e = threadIdx.x, jj = e >> 3, rr = e & 7;
    double fx = 0.0;
    if (jj < p && i0 + rr < n) {
      const int t = jj >> 3, cc = jj & 7;
      double g = 0.0;
#pragma unroll
      for (int w = 0; w < kSmallThreads / 32; ++w) g += sG[w][t * 64 + rr * 8 + cc];
      const int64_t ix = i0 + rr + jj * ld;
      double xv = Y[ix];
      if (scale) {
        g *= scale[jj];
        xv *= scale[jj];  // = the normalised iterate, as its owner writes it
      }
      double fv = g;
      if (a.g0) {  // f = ½⟨X, AX + 2·G0⟩
        const double g0v = a.g0[ix];
        g += g0v;
        fv = g + g0v;
      }
      Pn[ix] = g;
      fx = xv * fv;
      bad |= !isfinite(g);
    }
    // the 8 rows of column jj sit in 8 consecutive lanes: fixed-order sum
    fx += __shfl_xor_sync(0xffffffffu, fx, 1);
    fx += __shfl_xor_sync(0xffffffffu, fx, 2);
    fx += __shfl_xor_sync(0xffffffffu, fx, 4);
    if (rr == 0 && jj < kSmallP) sF[jj] = fx;
    __syncthreads();
    if (threadIdx.x < p) fcol += sF[threadIdx.x];
  }
}

#define SMALL_STAMP(k) \
  if (a.prof && blockIdx.x == 0 && threadIdx.x == 0) a.prof[it * 8 + (k)] = globaltimer_ns()

// Iterations k → k+1 … of the small dense problem.  Phases per iteration,
// separated by grid barriers (5 per iteration):
//   B  η (every CTA, from the CTA partials of ⟨S,S⟩, ⟨S,Y⟩, ⟨Y,Y⟩), Z rows
//      of this CTA, per-CTA ‖z_j‖² partials
//   C  column norms (every CTA), X⁺ rows of this CTA (pcal_step incl. the
//      degenerate-column rule and the divergence flag), fused gradient
//      G = (A·Z)·diag(1/‖z‖) (+G0) of this CTA's 8-row tiles, f partials
//   D  Gram GᵀX, XᵀX (upper), one warp per entry
//   E  W, M per CTA; X·[W|M] epilogue (kkt, P, d_j, KKT²) per row
//   A  column sums (every CTA), record (CTA 0), stepsize partials of k+1
__global__ void __launch_bounds__(kSmallThreads) k_iter_small(SmallArgs a, Ctl* ctl, int iters) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sW[kSmallP][kSmallP + 1];
  __shared__ double sM[kSmallP][kSmallP + 1];
  __shared__ double sred[3][kSmallThreads / 32][kSmallP];
  __shared__ double sG[kSmallThreads / 32][4 * 64];
  __shared__ double sF[kSmallP];
  __shared__ double sc[3][kSmallP];      // column sums (f, KKT², d) of the last evaluation
  __shared__ double sInv[kSmallP];       // 1/‖z_j‖ (1 for plain steps)
  __shared__ double sm8[kSmallThreads / 32];
  __shared__ double s_eta;
  __shared__ int s_deg[kSmallP];
  __shared__ Ctl sctl;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (kSmallThreads / 32);
  const int gw = blockIdx.x * (kSmallThreads / 32) + warp;
  const int64_t n = a.n, ld = a.ld, p = a.p, pp = a.pp;
  const bool col = lane < p;
  // this CTA's rows of the streaming phases
  const int64_t rpb = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = min(n, (int64_t)blockIdx.x * rpb), r1 = min(n, r0 + rpb);
  extern __shared__ double sA[];  // [8][lda_s]: A rows of this CTA's gradient tile
  if (ctl->done) return;
  if (a.lda_s > 0) {  // n ≤ 8·gridDim: one tile per CTA, loaded once per launch
    const int64_t i0 = (int64_t)blockIdx.x * 8;
    for (int64_t e = threadIdx.x; e < 8 * a.lda_s; e += blockDim.x) {
      const int64_t r = e / a.lda_s, k = e % a.lda_s;
      sA[e] = (i0 + r < n && k < n) ? a.at[k + (i0 + r) * a.ldat] : 0.0;
    }
  }
  {  // stepsize partials of the current step from the stored state (pair b = current)
    const int b = (int)(ctl->iter & 1), nb = b ^ 1;
    double* Pb = a.pair[b];
    double* Pn = a.pair[nb];
    bb_block(Pb + ld * pp, Pn + ld * pp, Pb, Pn, a.fkd[b] + 2 * p, a.fkd[nb] + 2 * p, r0, r1, ld,
             p, a.bbpart, sm8);
  }
  grid.sync();
  for (int it = 0; it < iters; ++it) {
    if (ctl->done) return;  // uniform: written before the last grid barrier
    SMALL_STAMP(0);
    const int b = (int)(ctl->iter & 1), nb = b ^ 1;
    double* Pb = a.pair[b];
    double* Xb = Pb + ld * pp;
    double* Pn = a.pair[nb];
    double* Xn = Pn + ld * pp;
    const double* Db = a.fkd[b] + 2 * p;
    // ---- B: η (solver.cpp:212-251), Z = X − (1/η)(P − d∘X) rows, ‖z_j‖² partials
    {
      const bool need = ctl->eta_kind != 0 && ctl->have_prev && ctl->iter != 0;
      double ss = 0.0, sy = 0.0, yy = 0.0;
      if (threadIdx.x < gridDim.x) {
        ss = a.bbpart[threadIdx.x * 3 + 0];
        sy = a.bbpart[threadIdx.x * 3 + 1];
        yy = a.bbpart[threadIdx.x * 3 + 2];
      }
      ss = block_sum<kSmallThreads>(ss, sm8);
      sy = block_sum<kSmallThreads>(sy, sm8);
      yy = block_sum<kSmallThreads>(yy, sm8);
      if (threadIdx.x == 0) {
        const double eta = select_eta(ctl, ss, sy, yy, need);
        s_eta = eta;
        if (blockIdx.x == 0) {
          ctl->eta = eta;
          ctl->step_deg = 0;
          if (!(eta > 0.0)) {  // pcal_step: parameter_error (solver.cpp:266)
            ctl->step_param = 1;
            ctl->done = 3;
          }
        }
      }
      __syncthreads();
      const double eta = s_eta;
      if (!(eta > 0.0)) return;  // uniform
      const double inv_eta = 1.0 / eta;
      // thread (column j = lane, row group = warp)
      double acc = 0.0;
      if (col) {
        const double dj = Db[lane];
        for (int64_t i = r0 + warp; i < r1; i += kSmallThreads / 32) {
          const int64_t ix = i + lane * ld;
          const double xv = Xb[ix];
          const double gl = Pb[ix] - dj * xv;
          const double v = xv - inv_eta * gl;
          a.z[ix] = v;
          acc += v * v;
        }
      }
      sred[0][warp][lane] = acc;
      __syncthreads();
      if (threadIdx.x < kSmallP) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kSmallThreads / 32; ++w) t += sred[0][w][threadIdx.x];
        a.npb[(int64_t)blockIdx.x * kSmallP + threadIdx.x] = t;
      }
    }
    grid.sync();
    SMALL_STAMP(1);
    // ---- C: pcal_step normalisation (solver.cpp:283-305) + gradient (problems.cpp:130-141)
    bool anydeg = false;
    {
      bool bad = false;
      if (a.plain) {
        if (threadIdx.x < kSmallP) {
          sInv[threadIdx.x] = 1.0;
          s_deg[threadIdx.x] = 0;
        }
        __syncthreads();
      } else {
        cta_column_sums(a.npb, kSmallP, p, sred[1], sF);
        if (threadIdx.x < kSmallP) {
          const double nz = sqrt(sF[threadIdx.x]);
          s_deg[threadIdx.x] = threadIdx.x < p && nz < 1e-14;
          sInv[threadIdx.x] = 1.0 / nz;
        }
        __syncthreads();
        for (int j = 0; j < p; ++j) anydeg |= s_deg[j] != 0;
      }
      // X⁺ rows of this CTA
      if (col) {
        const double inv = sInv[lane];
        double pn = 0.0;
        if (s_deg[lane]) {  // the previous column renormalised, or e_{j mod n}
          for (int64_t i = 0; i < n; ++i) pn += Xb[i + lane * ld] * Xb[i + lane * ld];
          pn = sqrt(pn);
        }
        for (int64_t i = r0 + warp; i < r1; i += kSmallThreads / 32) {
          const int64_t ix = i + lane * ld;
          double v;
          if (!s_deg[lane]) v = a.plain ? a.z[ix] : a.z[ix] * inv;
          else if (pn > 0.0) v = Xb[ix] * (1.0 / pn);
          else v = (i == (lane % n)) ? 1.0 : 0.0;
          Xn[ix] = v;
          bad |= !isfinite(v);
        }
      }
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        int nd = 0;
        for (int j = 0; j < p; ++j) nd += s_deg[j];
        ctl->step_deg = nd;
      }
      if (__syncthreads_or(bad) && threadIdx.x == 0) {
        ctl->step_bad = 1;
        ctl->done = 2;
      }
      double fcol = 0.0;
      bool gbad = false;
      if (!anydeg) {
        gradient_tiles(a, a.z, a.plain ? nullptr : sInv, Pn, sG, sF, fcol, gbad,
                       a.lda_s > 0 ? sA : nullptr);
      } else {  // rare: a degenerate column is not a scaled column of Z
        grid.sync();
        gradient_tiles(a, Xn, nullptr, Pn, sG, sF, fcol, gbad, a.lda_s > 0 ? sA : nullptr);
      }
      if (gbad) *a.fa.bad = 1;
      if (threadIdx.x < kSmallP)
        a.part[((int64_t)blockIdx.x * 3 + 0) * kSmallP + threadIdx.x] = fcol;
    }
    grid.sync();
    SMALL_STAMP(2);
    if (ctl->done) return;  // non-finite step
    // ---- D: Gram GᵀX (all p²) and XᵀX (upper triangle), one warp per entry
    {
      const int64_t ngx = p * p, total = ngx + p * (p + 1) / 2;
      for (int64_t e = gw; e < total; e += nwarps) {
        int64_t r, c;
        const double* ya;
        if (e < ngx) {
          r = e % p;
          c = e / p;
          ya = Pn + r * ld;
        } else {
          const int64_t t = e - ngx;  // t = c(c+1)/2 + r, r ≤ c
          c = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
          while (c * (c + 1) / 2 > t) --c;
          while ((c + 1) * (c + 2) / 2 <= t) ++c;
          r = t - c * (c + 1) / 2;
          ya = Xn + r * ld;
        }
        const double* xc = Xn + c * ld;
        double s = 0.0;
        for (int64_t i = lane; i < n; i += 32) s = fma(ya[i], xc[i], s);
        s = warp_sum(s);
        if (lane == 0) a.gr[(e < ngx ? r : pp + r) + c * 2 * pp] = s;
      }
    }
    grid.sync();
    SMALL_STAMP(3);
    // ---- E: W = Ψ(GᵀX), C = XᵀX − I, M per algorithm (k_small_pxp) in every CTA;
    //         X·[W|M] with the PCAL epilogue, d_j and KKT² partials (solver.cpp:385-409)
    for (int64_t e = threadIdx.x; e < p * p; e += blockDim.x) {
      const int64_t k = e % p, j = e / p;
      const int64_t ldg = 2 * pp;
      const double w = 0.5 * (a.gr[k + j * ldg] + a.gr[j + k * ldg]);
      double c = a.gr[pp + min(k, j) + max(k, j) * ldg];
      if (k == j) c += -1.0;
      double m = c;
      if (a.mc_mode == MC_DA) m = a.beta * c - (a.lam[k + j * p] + -a.beta * c);
      sW[k][j] = w;
      sM[k][j] = m;
    }
    __syncthreads();
    {
      double kacc = 0.0, dacc = 0.0;
      for (int64_t i = gw; i < n; i += nwarps) {
        const double xi = col ? Xn[i + lane * ld] : 0.0;
        double t1 = 0.0, t2 = 0.0;
#pragma unroll 4
        for (int k = 0; k < p; ++k) {
          const double xk = __shfl_sync(0xffffffffu, xi, k);
          if (col) {
            t1 = fma(xk, sW[k][lane], t1);
            t2 = fma(xk, sM[k][lane], t2);
          }
        }
        if (col) {
          const int64_t e = i + lane * ld;
          const double g = Pn[e];
          const double kkt = g - t1;
          const double pv = (a.p_from_g ? g : kkt) + a.beta_epi * t2;
          Pn[e] = pv;
          kacc += kkt * kkt;
          dacc += xi * pv;
        }
      }
      sred[1][warp][lane] = col ? kacc : 0.0;
      sred[2][warp][lane] = col ? dacc : 0.0;
      __syncthreads();
      if (threadIdx.x < 2 * kSmallP) {  // CTA column partials (KKT², d), warps in order
        const int w3 = 1 + threadIdx.x / kSmallP, j = threadIdx.x % kSmallP;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kSmallThreads / 32; ++q) s += sred[w3][q][j];
        a.part[((int64_t)blockIdx.x * 3 + w3) * kSmallP + j] = s;
      }
    }
    grid.sync();
    SMALL_STAMP(4);
    // ---- A: column sums (every CTA), record (CTA 0), stepsize partials of step k+1
    {
      {  // the three arrays at once: all 60 loads of a lane in flight together
        constexpr int W8 = kSmallThreads / 32, BPW = 20;  // gridDim ≤ 160
        double v[3][BPW];
#pragma unroll
        for (int u = 0; u < BPW; ++u) {
          const int q = warp * BPW + u;
          const bool ok = q < (int)gridDim.x && col;
#pragma unroll
          for (int w3 = 0; w3 < 3; ++w3)
            v[w3][u] = ok ? a.part[((int64_t)q * 3 + w3) * kSmallP + lane] : 0.0;
        }
#pragma unroll
        for (int w3 = 0; w3 < 3; ++w3) {
          double t = 0.0;
#pragma unroll
          for (int u = 0; u < BPW; ++u) t += v[w3][u];
          sred[w3][warp][lane] = t;
        }
        __syncthreads();
        if (threadIdx.x < 3 * kSmallP) {
          const int w3 = threadIdx.x / kSmallP, j = threadIdx.x % kSmallP;
          double t = 0.0;
#pragma unroll
          for (int w = 0; w < W8; ++w) t += sred[w3][w][j];
          sc[w3][j] = t;
        }
        __syncthreads();
      }
      if (!a.dform && threadIdx.x < kSmallP) sc[2][threadIdx.x] = 0.0;  // d stays 0
      __syncthreads();
      if (blockIdx.x == 0) {
        constexpr int CW = (int)(sizeof(Ctl) / sizeof(uint32_t));
        static_assert(sizeof(Ctl) % sizeof(uint32_t) == 0, "Ctl copy");
        if (threadIdx.x < CW)
          reinterpret_cast<uint32_t*>(&sctl)[threadIdx.x] =
              reinterpret_cast<const uint32_t*>(ctl)[threadIdx.x];
        if (threadIdx.x < p) {
          double* fk = a.fkd[nb];
          fk[threadIdx.x] = sc[0][threadIdx.x];
          fk[p + threadIdx.x] = sc[1][threadIdx.x];
          fk[2 * p + threadIdx.x] = sc[2][threadIdx.x];
        }
        double cc = 0.0;  // ‖XᵀX − I‖² (from the upper triangle, k_small_pxp)
        for (int64_t e = threadIdx.x; e < p * p; e += blockDim.x) {
          const int64_t k = e % p, j = e / p;
          double c = a.gr[pp + min(k, j) + max(k, j) * 2 * pp];
          if (k == j) c += -1.0;
          cc += c * c;
          if (a.mc_mode == MC_DA) a.lam[e] = a.lam[e] + -a.beta * c;  // Λ ← Λ − β·C
        }
        const double c2 = block_sum<kSmallThreads>(cc, sm8);  // (synchronises the block)
        if (threadIdx.x == 0) {
          double f1 = 0.0, k2 = 0.0;
          for (int64_t j = 0; j < p; ++j) {
            f1 += sc[0][j];
            k2 += sc[1][j];
          }
          finish_record(a.fa, &sctl, nullptr, f1, k2, c2, 0.0, 0.0, 0.0);
        }
        __syncthreads();
        if (threadIdx.x < CW)
          reinterpret_cast<uint32_t*>(ctl)[threadIdx.x] =
              reinterpret_cast<const uint32_t*>(&sctl)[threadIdx.x];
      }
      // stepsize partials for step k+1: S = X⁺ − X, Y = (P⁺ − d⁺∘X⁺) − (P − d∘X)
      bb_block(Xn, Xb, Pn, Pb, sc[2], Db, r0, r1, ld, p, a.bbpart, sm8);
    }
    grid.sync();
    SMALL_STAMP(5);
  }
}
#undef SMALL_STAMP

// Aᵀ for the row-wise gradient (A need not be symmetric in storage).
__global__ void k_transpose(const double* __restrict__ a, int64_t lda, int64_t n,
                            double* __restrict__ at, int64_t ldat) {
  __shared__ double t[32][33];
  const int64_t i0 = (int64_t)blockIdx.x * 32, k0 = (int64_t)blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t k = k0 + r, i = i0 + threadIdx.x;
    t[r][threadIdx.x] = (i < n && k < n) ? a[i + k * lda] : 0.0;  // A(i, k)
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, k = k0 + threadIdx.x;
    if (i < n && k < n) at[k + i * ldat] = t[threadIdx.x][r];
  }
}

}  // namespace pcal
