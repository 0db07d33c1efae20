// pcal_kernels.cuh — streaming / small-matrix / reduction kernels of one PCAL
// iteration (solver.cpp:385-438 restated for HBM).  All reductions are
// deterministic: per-block partials in fixed slots, summed in index order.
#pragma once

#include "common.cuh"

namespace pcal {

constexpr int kStreamThreads = 256;

// Column sums of the row-block partial arrays (part[col·stride + rb]), one
// block per (column, array), fixed-order block reduction:
//   out_a[col] = Σ_{rb < nrows_a} part_a[col·stride_a + rb].
struct ColSumArgs {
  const double* in[3];
  int64_t nrows[3];
  int64_t stride[3];
  double* out[3];
  const int32_t* gate;  // non-null: run only when *gate != 0
};
__global__ void __launch_bounds__(kStreamThreads) k_colsum3(ColSumArgs a, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  if (a.gate && !*a.gate) return;
  __shared__ double sm[kStreamThreads / 32];
  const int which = blockIdx.y;
  if (!a.in[which]) return;
  const int64_t col = blockIdx.x;
  const double* src = a.in[which] + col * a.stride[which];
  double acc = 0.0;
  for (int64_t r = threadIdx.x; r < a.nrows[which]; r += blockDim.x) acc += src[r];
  const double s = block_sum<kStreamThreads>(acc, sm);
  if (threadIdx.x == 0) a.out[which][col] = s;
}

// W = Ψ(GᵀX) = ½(M1 + M1ᵀ), C = XᵀX − I (exactly symmetric, from the computed
// upper triangle), written interleaved as the B operand of the X·[W|M] GEMM:
//   mcat[k + (2j)·ldk] = W[k,j],  mcat[k + (2j+1)·ldk] = M[k,j]
// with the second block per algorithm (solver.cpp:371-409):
//   PCAL / PLAM : M = C                 (epilogue: P = (G − XW) + β·XC)
//   PCAL-DA / PLAM-DA : M = βC − Λ,  Λ ← W at the start point, Λ ← Λ − β·C after
//                 (epilogue: P = G + XM)
//   MOptQR      : M = −GᵀX (not symmetrised)   (epilogue: P = G + XM = G − X·GᵀX)
// cpart[block] = Σ C² over the block (feasibility).
// gr: (2·pp) × pp column-major; rows [0,pp) = GᵀX, rows [pp,2pp) = XᵀX.
// perm32: the column order of gemm_xm_staged (gemm_dmma.cuh xm_out_col): within
// each 32-column block, output column j sits at slot s = nt·4 + q of the
// warp half wn, where t = j mod 16 = 8·(nt>>1) + 2·(nt&1) + (q&1) + 4·(q>>1) —
// the order that makes the staged epilogue's swizzled G / X reads conflict-free.
__host__ __device__ __forceinline__ int64_t xm_slot_of_col(int64_t j) {
  const int64_t t = j & 15;
  const int64_t nt = 2 * ((t >> 3) & 1) + ((t >> 1) & 1), q = 2 * ((t >> 2) & 1) + (t & 1);
  return (j & ~int64_t(15)) + nt * 4 + q;
}

// Column slot of output column j in M1 for gemm_xm1_staged (gemm_dmma.cuh
// xm1_out_col): t = j mod 16 = 8·nt + 2·x + (q & 1) + 4·(q >> 1) sits at MMA
// column 8·nt + 2·q + x.
__host__ __device__ __forceinline__ int64_t xm1_slot_of_col(int64_t j) {
  const int64_t t = j & 15;
  const int64_t nt = (t >> 3) & 1, x = (t >> 1) & 1, q = (t & 1) + 2 * ((t >> 2) & 1);
  return (j & ~int64_t(15)) + 8 * nt + 2 * q + x;
}

// XM1 mode (PCAL / PLAM, gemm_xm1_staged): besides the regular outputs the
// kernel writes M1 = W − β·C in xm1 slot order into m1 (pp × pp), and W and C
// in natural order into wm / cm (the ⟨W, C²⟩, ⟨C, C²⟩ terms of the kkt
// identity), and mcat holds the fallback operand [β·C | C] interleaved.
struct Xm1Out {
  double* m1;
  double* wm;
  double* cm;
};

enum { MC_PCAL = 0, MC_DA = 1, MC_MOPTQR = 2 };
__global__ void k_small_pxp(const double* __restrict__ gr, int64_t pp, int64_t p,
                            double* __restrict__ mcat, int64_t ldk, double* __restrict__ cpart,
                            int mode, double beta, double* __restrict__ lam, int lam_init,
                            const Ctl* ctl, int gx_upper = 0, int perm32 = 0,
                            Xm1Out xm1 = Xm1Out{nullptr, nullptr, nullptr}) {
  if (ctl && ctl->done) return;
  __shared__ double sm[kStreamThreads / 32];
  const int64_t total = p * p;
  const int64_t ldg = 2 * pp;
  double acc = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = e % p, j = e / p;
    const int64_t a = min(k, j), b = max(k, j);
    // symmetric operator: GᵀX = XᵀAX is symmetric, only its upper triangle is
    // computed and Ψ reduces to it (equal to ½(M + Mᵀ) up to rounding)
    const double w = gx_upper ? gr[a + b * ldg] : 0.5 * (gr[k + j * ldg] + gr[j + k * ldg]);
    double c = gr[pp + a + b * ldg];
    if (k == j) c += -1.0;
    double m;
    if (mode == MC_PCAL) {
      m = c;
    } else if (mode == MC_DA) {
      // Λ is updated elementwise from the upper triangle's value, so it stays
      // exactly symmetric (SquareSymmetric::add_scaled, kernels.cpp:38-47)
      // lam_init: 1 = Λ ← W (start point), 0 = dual-ascent update, 2 = keep
      // (ALM inner iterations: Λ changes only at the outer updates)
      double l = lam_init == 1 ? w : lam_init == 2 ? lam[k + j * p] : lam[k + j * p] + -beta * c;
      lam[k + j * p] = l;
      m = beta * c - l;
    } else {
      m = -gr[k + j * ldg];
    }
    if (xm1.m1) {
      xm1.m1[k + xm1_slot_of_col(j) * ldk] = w + -beta * c;
      xm1.wm[k + j * ldk] = w;
      xm1.cm[k + j * ldk] = c;
      mcat[k + (2 * j) * ldk] = beta * c;  // fallback: kkt = P − X·(βC), P = kkt + β·XC
      mcat[k + (2 * j + 1) * ldk] = c;
    } else {
      const int64_t slot = perm32 ? xm_slot_of_col(j) : j;
      mcat[k + (2 * slot) * ldk] = w;
      mcat[k + (2 * slot + 1) * ldk] = m;
    }
    acc += c * c;
  }
  const double s = block_sum<kStreamThreads>(acc, sm);
  if (threadIdx.x == 0) cpart[blockIdx.x] = s;
}

// The kkt identity's p × p inner products (XM1 mode):
// part[block·3 + {0,1,2}] = partial {⟨W, C²⟩, ⟨C, C²⟩, ⟨C, C⟩}.
__global__ void k_kkt_corr(const double* __restrict__ w, const double* __restrict__ c,
                           const double* __restrict__ c2, int64_t ldk, int64_t p,
                           double* __restrict__ part, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  __shared__ double sm[kStreamThreads / 32];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < p * p;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e % p + (e / p) * ldk;
    const double cv = c[i], qv = c2[i];
    a0 += w[i] * qv;
    a1 += cv * qv;
    a2 += cv * cv;
  }
  const double s0 = block_sum<kStreamThreads>(a0, sm);
  const double s1 = block_sum<kStreamThreads>(a1, sm);
  const double s2 = block_sum<kStreamThreads>(a2, sm);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = s0;
    part[3 * blockIdx.x + 1] = s1;
    part[3 * blockIdx.x + 2] = s2;
  }
}

// Σ kkt² = Σ P² + 2β⟨W, C²⟩ − β²(‖C‖² + ⟨C, C²⟩) (gemm_dmma.cuh gemm_xm1_staged).
// The identity is used while its terms cancel by less than a factor `gate_ratio`
// ((Σ P² + |correction terms|) ≤ gate_ratio · result, i.e. the rounding of the
// terms costs < gate_ratio ulps of Σ kkt²); otherwise *fb = 1 and the gated
// two-block product recomputes kkt directly.  kk[0] = Σ kkt² (identity),
// kk[1] counts fallbacks.
__global__ void k_kkt_gate(const double* __restrict__ part, int nb, const double* __restrict__ kcol,
                           int64_t p, double beta, double gate_ratio, int32_t* fb, double* kk,
                           const Ctl* ctl) {
  if (ctl && ctl->done) return;
  __shared__ double sm[8];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, ap = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    a0 += part[3 * i];
    a1 += part[3 * i + 1];
    a2 += part[3 * i + 2];
  }
  for (int64_t j = threadIdx.x; j < p; j += blockDim.x) ap += kcol[j];
  const double wc2 = block_sum<256>(a0, sm);
  const double cc2 = block_sum<256>(a1, sm);
  const double cc = block_sum<256>(a2, sm);
  const double pp2 = block_sum<256>(ap, sm);
  if (threadIdx.x != 0) return;
  const double k2 = pp2 + (2.0 * beta * wc2 - beta * beta * (cc + cc2));
  const double mag = pp2 + 2.0 * fabs(beta * wc2) + beta * beta * (cc + fabs(cc2));
  const bool fall = !(k2 > 0.0) || !isfinite(k2) || mag > gate_ratio * k2;
  *fb = fall ? 1 : 0;
  kk[0] = k2;
  if (fall) kk[1] += 1.0;
}

// Stepsize inner products (stepsize_select, solver.cpp:218-222) with the
// PCAL diagonal correction recomputed in registers (solver.cpp:397-405):
//   GL = P − d∘X,  S = X − X_prev,  Y = GL − GL_prev.
// part[block·3 + {0,1,2}] = partial {⟨S,S⟩, ⟨S,Y⟩, ⟨Y,Y⟩}.
__global__ void k_bb_partials(const double* __restrict__ x, const double* __restrict__ pg,
                              const double* __restrict__ xp, const double* __restrict__ pgp,
                              const double* __restrict__ d, const double* __restrict__ dp,
                              int64_t ld, int64_t p, double* __restrict__ part, const Ctl* ctl) {
  if (ctl->done || ctl->iter == ctl->iter_base || !ctl->have_prev) return;
  __shared__ double sm[kStreamThreads / 32];
  double ss = 0.0, sy = 0.0, yy = 0.0;
  const int64_t half = ld / 2;  // ld is a multiple of 16: double2 vectors never straddle columns
  const int64_t total = half * p;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / half;
    const double2 xv = reinterpret_cast<const double2*>(x)[e];
    const double2 xpv = reinterpret_cast<const double2*>(xp)[e];
    const double2 pv = reinterpret_cast<const double2*>(pg)[e];
    const double2 ppv = reinterpret_cast<const double2*>(pgp)[e];
    const double dj = d[j], dpj = dp[j];
    {
      const double s = xv.x - xpv.x;
      const double y = (pv.x - dj * xv.x) - (ppv.x - dpj * xpv.x);
      ss += s * s;
      sy += s * y;
      yy += y * y;
    }
    {
      const double s = xv.y - xpv.y;
      const double y = (pv.y - dj * xv.y) - (ppv.y - dpj * xpv.y);
      ss += s * s;
      sy += s * y;
      yy += y * y;
    }
  }
  const double a = block_sum<kStreamThreads>(ss, sm);
  const double b = block_sum<kStreamThreads>(sy, sm);
  const double c = block_sum<kStreamThreads>(yy, sm);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = a;
    part[blockIdx.x * 3 + 1] = b;
    part[blockIdx.x * 3 + 2] = c;
  }
}

__device__ __forceinline__ double clamp_eta(const Ctl* c, double v) {
  const double r = v > c->eta_min ? v : c->eta_min;
  return r < c->eta_max ? r : c->eta_max;
}

// The stepsize rule of stepsize_select (solver.cpp:212-251) from the summed
// ⟨S,S⟩, ⟨S,Y⟩, ⟨Y,Y⟩: BB1 / BB2 / ABB (odd k → BB1) / differential, the
// zero-denominator fallback to the previous η (or η0), then the clamp.
__device__ __forceinline__ double select_eta(const Ctl* c, double ss, double sy, double yy,
                                             bool need) {
  if (c->eta_kind == 0) return clamp_eta(c, c->gamma);
  const double fallback = c->eta_prev > 0.0 ? c->eta_prev : c->eta0;
  if (!need) return clamp_eta(c, c->eta0 > 0.0 ? c->eta0 : fallback);
  const double bb1 = (ss == 0.0 || sy == 0.0) ? fallback : fabs(sy) / ss;
  const double bb2 = (sy == 0.0) ? fallback : yy / fabs(sy);
  double v = fallback;
  switch (c->eta_kind) {
    case 2: v = bb1; break;
    case 3: v = bb2; break;
    case 4: v = ((c->iter - c->iter_base) % 2 == 1) ? bb1 : bb2; break;
    case 1: v = (ss == 0.0) ? fallback : sqrt(yy) / sqrt(ss); break;
    default: break;
  }
  return clamp_eta(c, v);
}

// stepsize_select (solver.cpp:212-251) on the device: one block reduces the
// k_bb_partials slots in a fixed order, thread 0 applies the rule.
__global__ void __launch_bounds__(kStreamThreads) k_eta(Ctl* ctl, const double* __restrict__ part,
                                                         int nblocks) {
  if (ctl->done) return;
  __shared__ double sm[kStreamThreads / 32];
  Ctl* c = ctl;
  const bool need = c->eta_kind != 0 && c->have_prev && c->iter != c->iter_base;
  double ss = 0.0, sy = 0.0, yy = 0.0;
  if (need) {
    double a = 0.0, b = 0.0, d = 0.0;
    for (int i = threadIdx.x; i < nblocks; i += blockDim.x) {
      a += part[3 * i + 0];
      b += part[3 * i + 1];
      d += part[3 * i + 2];
    }
    ss = block_sum<kStreamThreads>(a, sm);
    sy = block_sum<kStreamThreads>(b, sm);
    yy = block_sum<kStreamThreads>(d, sm);
  }
  if (threadIdx.x != 0) return;
  const double eta = select_eta(c, ss, sy, yy, need);
  c->eta = eta;
  c->step_deg = 0;
  if (!(eta > 0.0)) {  // pcal_step: parameter_error (solver.cpp:266)
    c->step_param = 1;
    c->done = 3;
  }
}

// pcal_step part 1 (solver.cpp:278-282): Z = X − (1/η)·GL with GL = P − d∘X,
// written over the X_{k-1} buffer; npart[chunk·p + j] = Σ_{chunk rows} z².
__global__ void k_update(const double* __restrict__ x, const double* __restrict__ pg,
                         const double* __restrict__ d, double* __restrict__ z, int64_t n,
                         int64_t ld, int64_t p, int64_t chunk, double* __restrict__ npart,
                         double* __restrict__ xpart, const Ctl* ctl, int64_t cstride = 0) {
  if (ctl->done) return;
  __shared__ double sm[kStreamThreads / 32];
  const int64_t j = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const int64_t r1 = min(n, r0 + chunk);
  const double inv_eta = 1.0 / ctl->eta;
  const double dj = d[j];
  double acc = 0.0, xacc = 0.0;
  const double* xj = x + j * ld;
  const double* pj = pg + j * ld;
  double* zj = z + j * ld;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const double xv = xj[i];
    const double gl = pj[i] - dj * xv;
    const double v = xv - inv_eta * gl;
    zj[i] = v;
    acc += v * v;
    xacc += xv * xv;
  }
  const int64_t cs = cstride ? cstride : p;  // row stride of the chunk-partial arrays
  const double s = block_sum<kStreamThreads>(acc, sm);
  if (threadIdx.x == 0) npart[blockIdx.x * cs + j] = s;
  if (xpart) {  // sharded: ‖x_j‖² partials for the degenerate-column rule
    const double t = block_sum<kStreamThreads>(xacc, sm);
    if (threadIdx.x == 0) xpart[blockIdx.x * cs + j] = t;
  }
}

// ---- normalised step without a separate normalisation pass ----------------
// pcal_step (solver.cpp:278-300) normalises z_j = x_j − (1/η)·gl_j by its
// norm, which the reference takes from a second pass over z.  Here the
// stepsize kernel, which reads X and P anyway, also sums per column
//   a_j = Σ x²,  b_j = Σ x·gl,  c_j = Σ gl²     (gl = p − d_j·x),
// so ‖z_j‖² = a_j + (1/η)·((1/η)·c_j − 2·b_j) is known before Z is formed and
// k_update_norm writes X_{k+1} = z·(1/‖z_j‖) in the same pass that forms z
// (16·n·p fewer bytes per iteration).  With the PCAL multiplier formula gl_j
// is orthogonal to x_j up to ‖x_j‖² − 1, so the three terms add without
// cancellation; a column whose expansion would cancel (terms / result > 1e6)
// or that is near the degenerate threshold is flagged and takes the
// reference's exact two-pass rule in k_normalize (fb mode).  The normalising
// factor differs from the two-pass one by rounding only (the parity
// tolerances of DESIGN.md §5).

// Per (row chunk c, column j): colpart[(c·p + j)·6 + {ss, sy, yy, a, b, cc}].
// 16-byte vector loads (chunks are multiples of 256 rows); the six block sums
// share one shared-memory round (fixed order: lanes, then warps).
__global__ void __launch_bounds__(kStreamThreads)
    k_bb_cols(const double* __restrict__ x, const double* __restrict__ pg,
              const double* __restrict__ xp, const double* __restrict__ pgp,
              const double* __restrict__ d, const double* __restrict__ dp, int64_t n, int64_t ld,
              int64_t p, int64_t chunk, double* __restrict__ colpart, const Ctl* ctl) {
  if (ctl->done) return;
  __shared__ double sm[6][kStreamThreads / 32];
  const bool bb = ctl->iter != ctl->iter_base && ctl->have_prev;
  const int64_t j = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const int64_t r1 = min(n, r0 + chunk);
  const double dj = d[j], dpj = bb ? dp[j] : 0.0;
  const double2* xj = reinterpret_cast<const double2*>(x + j * ld);
  const double2* pj = reinterpret_cast<const double2*>(pg + j * ld);
  const double2* xpj = reinterpret_cast<const double2*>(xp + j * ld);
  const double2* ppj = reinterpret_cast<const double2*>(pgp + j * ld);
  double v[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // ss, sy, yy, a, b, c
  // rows beyond n are zero padding (x = p = 0): they add nothing
  const int64_t h0 = r0 / 2, h1 = (r1 + 1) / 2;  // an odd n ends on a zero padding row
  for (int64_t h = h0 + threadIdx.x; h < h1; h += blockDim.x) {
    const double2 xv = xj[h], pv = pj[h];
    const double g0 = pv.x - dj * xv.x, g1 = pv.y - dj * xv.y;
    v[3] += xv.x * xv.x;
    v[4] += xv.x * g0;
    v[5] += g0 * g0;
    v[3] += xv.y * xv.y;
    v[4] += xv.y * g1;
    v[5] += g1 * g1;
    if (bb) {
      const double2 xpv = xpj[h], ppv = ppj[h];
      const double s0 = xv.x - xpv.x, y0 = g0 - (ppv.x - dpj * xpv.x);
      const double s1 = xv.y - xpv.y, y1 = g1 - (ppv.y - dpj * xpv.y);
      v[0] += s0 * s0;
      v[1] += s0 * y0;
      v[2] += y0 * y0;
      v[0] += s1 * s1;
      v[1] += s1 * y1;
      v[2] += y1 * y1;
    }
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const double t = warp_sum(v[q]);
    if (l == 0) sm[q][w] = t;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < kStreamThreads / 32; ++i) t += sm[threadIdx.x][i];
    colpart[((int64_t)blockIdx.x * p + j) * 6 + threadIdx.x] = t;
  }
}

// Sum of the (chunk, column) stepsize partials in a fixed order → the
// k_eta input layout (one "block" slot holding the totals).
__global__ void __launch_bounds__(kStreamThreads) k_bb_cols_sum(const double* __restrict__ colpart,
                                                                int64_t nslots,
                                                                double* __restrict__ part,
                                                                const Ctl* ctl) {
  if (ctl->done) return;
  __shared__ double sm[kStreamThreads / 32];
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < nslots; i += blockDim.x)
#pragma unroll
    for (int q = 0; q < 3; ++q) v[q] += colpart[i * 6 + q];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double t = block_sum<kStreamThreads>(v[q], sm);
    if (threadIdx.x == 0) part[q] = t;
  }
}

// 1/‖z_j‖ from the expansion (after k_eta), and the fallback flag.
__global__ void k_colscale(const double* __restrict__ colpart, int64_t nchunks, int64_t p,
                           double* __restrict__ inv, int32_t* __restrict__ fb, const Ctl* ctl) {
  if (ctl->done) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p) return;
  double a = 0.0, b = 0.0, c = 0.0;
  for (int64_t k = 0; k < nchunks; ++k) {
    const double* q = colpart + (k * p + j) * 6;
    a += q[3];
    b += q[4];
    c += q[5];
  }
  const double ie = 1.0 / ctl->eta;
  const double nz2 = a + ie * (ie * c - 2.0 * b);
  const double mag = a + ie * (ie * c + 2.0 * fabs(b));
  const bool exact = !(nz2 > 1e-20) || mag > 1e6 * nz2 || !isfinite(nz2);
  fb[j] = exact ? 1 : 0;
  inv[j] = exact ? 1.0 : 1.0 / sqrt(nz2);
}

// One element of the normalised step: z = x − (1/η)·(p − d_j·x) and z·(1/‖z_j‖),
// with explicit roundings so k_update_norm and the fused stencil
// (stencil_tma.cuh, FUSE) produce bitwise the same X_{k+1}.
__device__ __forceinline__ double step_z(double x, double p, double dj, double inv_eta) {
  return __fma_rn(-inv_eta, __fma_rn(-dj, x, p), x);
}
__device__ __forceinline__ double step_value(double x, double p, double dj, double inv_eta,
                                             double sc) {
  return __dmul_rn(step_z(x, p, dj, inv_eta), sc);
}

// X_{k+1} = (x − (1/η)·gl)·inv_j in one pass (flagged columns: z unscaled for
// k_normalize's exact rule); npart as k_update (the exact ‖z‖² partials).
__global__ void __launch_bounds__(kStreamThreads)
    k_update_norm(const double* __restrict__ x, const double* __restrict__ pg,
                  const double* __restrict__ d, double* __restrict__ z, int64_t n, int64_t ld,
                  int64_t p, int64_t chunk, double* __restrict__ npart,
                  const double* __restrict__ inv, const int32_t* __restrict__ fb, Ctl* ctl,
                  double* __restrict__ xpart = nullptr, int64_t cstride = 0, int only_fb = 0) {
  if (ctl->done) return;
  if (only_fb && !fb[blockIdx.y]) return;  // the fused stencil wrote this column
  __shared__ double sm[kStreamThreads / 32];
  const int64_t j = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const int64_t r1 = min(n, r0 + chunk);
  const double inv_eta = 1.0 / ctl->eta;
  const double dj = d[j];
  const bool exact = fb[j] != 0;
  const double sc = exact ? 1.0 : inv[j];  // v·1 = v: flagged columns stay z
  const double2* xj = reinterpret_cast<const double2*>(x + j * ld);
  const double2* pj = reinterpret_cast<const double2*>(pg + j * ld);
  double2* zj = reinterpret_cast<double2*>(z + j * ld);
  double acc = 0.0, xacc = 0.0;
  bool bad = false;
  const int64_t h0 = r0 / 2, h1 = (r1 + 1) / 2;  // an odd n ends on a zero padding row
  for (int64_t h = h0 + threadIdx.x; h < h1; h += blockDim.x) {
    const double2 xv = xj[h], pv = pj[h];
    const double v0 = step_z(xv.x, pv.x, dj, inv_eta);
    const double v1 = step_z(xv.y, pv.y, dj, inv_eta);
    acc += v0 * v0;
    acc += v1 * v1;
    xacc += xv.x * xv.x;
    xacc += xv.y * xv.y;
    const double w0 = __dmul_rn(v0, sc), w1 = __dmul_rn(v1, sc);
    zj[h] = make_double2(w0, w1);
    bad |= !isfinite(w0) || !isfinite(w1);
  }
  const int64_t cs = cstride ? cstride : p;  // row stride of the chunk-partial arrays
  const double s = block_sum<kStreamThreads>(acc, sm);
  if (threadIdx.x == 0) npart[blockIdx.x * cs + j] = s;
  if (xpart) {  // sharded: ‖x_j‖² partials for the degenerate-column rule
    const double t = block_sum<kStreamThreads>(xacc, sm);
    if (threadIdx.x == 0) xpart[blockIdx.x * cs + j] = t;
  }
  if (!exact && __syncthreads_or(bad) && threadIdx.x == 0) {
    ctl->step_bad = 1;
    if (!xpart) ctl->done = 2;  // sharded (xpart given): decided collectively in k_finish_eval
  }
}

// sharded: local column sums of the z² / x² chunk partials → nrm[0:p], nrm[p:2p]
__global__ void k_norm_reduce(const double* __restrict__ npart, const double* __restrict__ xpart,
                              int64_t nchunks, int64_t p, double* __restrict__ nrm,
                              const Ctl* ctl) {
  if (ctl->done) return;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p) return;
  double a = 0.0, b = 0.0;
  for (int64_t c = 0; c < nchunks; ++c) {
    a += npart[c * p + j];
    b += xpart[c * p + j];
  }
  nrm[j] = a;
  nrm[p + j] = b;
}

// ---- reproducible (GPU-count invariant) reductions of the sharded path -----
// Every row reduction is first taken per fixed global row chunk (chunk
// boundaries depend only on the problem), the chunk partials
// are all-gathered in rank order (= global chunk order) and summed
// sequentially by k_chunk_sum, so the result is bitwise independent of the
// number of ranks.

// Stepsize inner products per (chunk, column): out[c·3p + 3j + {0,1,2}].
__global__ void k_bb_chunk(const double* __restrict__ x, const double* __restrict__ pg,
                           const double* __restrict__ xp, const double* __restrict__ pgp,
                           const double* __restrict__ d, const double* __restrict__ dp, int64_t n,
                           int64_t ld, int64_t p, int64_t chunk, double* __restrict__ out,
                           const Ctl* ctl) {
  if (ctl->done || ctl->iter == ctl->iter_base || !ctl->have_prev) return;
  __shared__ double sm[kStreamThreads / 32];
  const int64_t j = blockIdx.y, c = blockIdx.x;
  const int64_t r0 = c * chunk, r1 = min(n, r0 + chunk);
  const double dj = d[j], dpj = dp[j];
  double ss = 0.0, sy = 0.0, yy = 0.0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const int64_t e = i + j * ld;
    const double xv = x[e], xpv = xp[e];
    const double sv = xv - xpv;
    const double yv = (pg[e] - dj * xv) - (pgp[e] - dpj * xpv);
    ss += sv * sv;
    sy += sv * yv;
    yy += yv * yv;
  }
  const double a = block_sum<kStreamThreads>(ss, sm);
  const double b = block_sum<kStreamThreads>(sy, sm);
  const double e = block_sum<kStreamThreads>(yy, sm);
  if (threadIdx.x == 0) {
    double* o = out + c * 3 * p + 3 * j;
    o[0] = a;
    o[1] = b;
    o[2] = e;
  }
}

// Per-chunk column sums of the three row-block partial arrays (f, kkt², d):
// block (j, which) — thread c sums rows [c·rpc, (c+1)·rpc) of column j of
// array `which` sequentially into out[c·3p + which·p + j] (0 where the array
// is absent).
struct ChunkColArgs {
  const double* in[3];
  int64_t nrows[3];   // local row-block count
  int64_t stride[3];  // column stride
  int64_t rpc[3];     // row blocks per chunk
  double* out;
  int64_t p;
  int64_t nch;        // local chunks
  const int32_t* gate;  // non-null: run only when *gate != 0
};
__global__ void __launch_bounds__(128) k_chunk_colsum3(ChunkColArgs a, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  if (a.gate && !*a.gate) return;
  const int which = blockIdx.y;
  const int64_t col = blockIdx.x;
  const double* src = a.in[which] ? a.in[which] + col * a.stride[which] : nullptr;
  for (int64_t c = threadIdx.x; c < a.nch; c += blockDim.x) {
    double acc = 0.0;
    if (src) {
      const int64_t r1 = min(a.nrows[which], (c + 1) * a.rpc[which]);
#pragma unroll 4
      for (int64_t r = c * a.rpc[which]; r < r1; ++r) acc += src[r];
    }
    a.out[c * 3 * a.p + which * a.p + col] = acc;
  }
}

// out[w] = Σ_r Σ_{q < nq[r]} buf[r·rank_stride + q·W + w], in that order;
// out[W + e] = Σ_r buf[r·rank_stride + extra_off + e] for e < extra (per-rank
// values riding along in the same all-gather, e.g. the failure flags).
__global__ void k_chunk_sum(const double* __restrict__ buf, int R, const int32_t* __restrict__ nq,
                            int64_t rank_stride, int64_t W, double* __restrict__ out,
                            const Ctl* ctl, int extra = 0, int64_t extra_off = 0) {
  if (ctl && ctl->done) return;
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= W + extra) return;
  double s = 0.0;
  if (w >= W) {
    for (int r = 0; r < R; ++r) s += buf[r * rank_stride + extra_off + (w - W)];
    out[w] = s;
    return;
  }
  for (int r = 0; r < R; ++r) {
    const double* b = buf + r * rank_stride + w;
    const int q1 = nq[r];
#pragma unroll 8
    for (int q = 0; q < q1; ++q) s += b[(int64_t)q * W];
  }
  out[w] = s;
}

// z[r0:r1) ·= inv in place, 4 loads in flight per thread (an in-place
// read-modify-write loop would otherwise serialise on possible aliasing);
// returns whether a non-finite value was produced.
__device__ __forceinline__ bool scale_range(double* __restrict__ zj, int64_t r0, int64_t r1,
                                            double inv) {
  bool bad = false;
  const int64_t T = blockDim.x;
  int64_t i = r0 + threadIdx.x;
  for (; i + 3 * T < r1; i += 4 * T) {
    const double v0 = zj[i], v1 = zj[i + T], v2 = zj[i + 2 * T], v3 = zj[i + 3 * T];
    const double w0 = v0 * inv, w1 = v1 * inv, w2 = v2 * inv, w3 = v3 * inv;
    zj[i] = w0;
    zj[i + T] = w1;
    zj[i + 2 * T] = w2;
    zj[i + 3 * T] = w3;
    bad |= !isfinite(w0) || !isfinite(w1) || !isfinite(w2) || !isfinite(w3);
  }
  for (; i < r1; i += T) {
    const double v = zj[i] * inv;
    zj[i] = v;
    bad |= !isfinite(v);
  }
  return bad;
}

// pcal_step part 2 (solver.cpp:283-305): z ·= 1/‖z‖; a column with ‖z‖ < 1e-14
// keeps the previous column renormalized (or e_{j mod n}); non-finite ⇒ diverged.
__global__ void k_normalize(const double* __restrict__ x, double* __restrict__ z, int64_t n,
                            int64_t ld, int64_t p, int64_t chunk, int64_t nchunks,
                            const double* __restrict__ npart, const double* __restrict__ nrm,
                            int64_t row0, int64_t n_glob, int plain, Ctl* ctl,
                            const int32_t* __restrict__ only_fb = nullptr) {
  if (ctl->done) return;
  if (only_fb && !only_fb[blockIdx.y]) return;  // k_update_norm already normalised it
  if (plain) {  // plam_step (solver.cpp:253-262): no normalisation, only the finiteness check
    const int64_t j = blockIdx.y;
    const int64_t r0 = (int64_t)blockIdx.x * chunk;
    const int64_t r1 = min(n, r0 + chunk);
    bool bad = false;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) bad |= !isfinite(z[j * ld + i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) {
      ctl->step_bad = 1;
      if (!nrm) ctl->done = 2;
    }
    return;
  }
  __shared__ double sm[kStreamThreads / 32];
  __shared__ double s_inv;
  __shared__ int s_deg;
  const int64_t j = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const int64_t r1 = min(n, r0 + chunk);
  if (threadIdx.x < 32) {  // ‖z_j‖² from the chunk partials: one warp, fixed order
    double nrm2 = 0.0;
    if (nrm) {
      nrm2 = threadIdx.x == 0 ? nrm[j] : 0.0;  // sharded: global column norm (all-reduced)
    } else {
      for (int64_t c = threadIdx.x; c < nchunks; c += 32) nrm2 += npart[c * p + j];
      nrm2 = warp_sum(nrm2);
    }
    if (threadIdx.x == 0) {
      const double nz = sqrt(nrm2);
      s_deg = nz < 1e-14;
      s_inv = 1.0 / nz;
    }
  }
  __syncthreads();
  double* zj = z + j * ld;
  bool bad = false;
  if (!s_deg) {
    bad = scale_range(zj, r0, r1, s_inv);
  } else {
    // degenerate column: whole-column norm of the previous iterate (rare path)
    const double* xj = x + j * ld;
    double pn2;
    if (nrm) {
      pn2 = nrm[p + j];
    } else {
      double acc = 0.0;
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += xj[i] * xj[i];
      pn2 = block_sum<kStreamThreads>(acc, sm);
    }
    if (threadIdx.x == 0) sm[0] = sqrt(pn2);
    __syncthreads();
    const double pn = sm[0];
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
      double v;
      if (pn > 0.0) v = xj[i] * (1.0 / pn);
      else v = (row0 + i == (j % n_glob)) ? 1.0 : 0.0;
      zj[i] = v;
      bad |= !isfinite(v);
    }
  }
  if (s_deg && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&ctl->step_deg, 1);
  if (__syncthreads_or(bad) && threadIdx.x == 0) {
    ctl->step_bad = 1;
    if (!nrm) ctl->done = 2;  // sharded: decided collectively in k_finish_eval
  }
}

}  // namespace pcal

namespace pcal {
// sharded: local failure flags appended to the allreduced column sums
__global__ void k_flags(const Ctl* ctl, const int32_t* bad, double* out) {
  out[0] = ctl->step_bad ? 1.0 : 0.0;
  out[1] = *bad ? 1.0 : 0.0;
}
}  // namespace pcal

#include <cooperative_groups.h>

namespace pcal {

// The whole pcal_step phase of one iteration (stepsize_select + pcal_step,
// solver.cpp:212-307) as ONE cooperative kernel (single GPU): bb partials →
// grid sync → η (every block reduces the partials in the same fixed order;
// block 0 publishes it) → Z = X − GL/η with column-norm partials → grid sync →
// normalisation.  Same arithmetic and reduction order as the separate kernels
// k_bb_partials / k_eta / k_update / k_normalize (bitwise identical results);
// saves three launches and the host-visible gaps between them.
struct StepArgs {
  const double *x, *pg, *xp, *pgp, *d, *dp;
  double* z;
  double* bbpart;
  double* npart;
  int64_t n, ld, p, chunk, nchunks, n_glob;
  int plain;  // 1: plam_step (no normalisation)
};

// The step phase as a device function of a cooperative grid (also the first
// phase of the small-problem iteration kernel, k_iter_small).  Returns false
// when the step must not continue (η ≤ 0); uniform across the grid.
__device__ __forceinline__ bool step_phase(const StepArgs& a, Ctl* ctl) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double sm[kStreamThreads / 32];
  __shared__ double s_eta;
  __shared__ double s_inv;
  __shared__ int s_deg;
  const bool need = ctl->eta_kind != 0 && ctl->have_prev && ctl->iter != ctl->iter_base;
  // ---- phase 1: stepsize inner products (k_bb_partials)
  if (need) {
    double ss = 0.0, sy = 0.0, yy = 0.0;
    const int64_t half = a.ld / 2;
    const int64_t total = half * a.p;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t j = e / half;
      const double2 xv = reinterpret_cast<const double2*>(a.x)[e];
      const double2 xpv = reinterpret_cast<const double2*>(a.xp)[e];
      const double2 pv = reinterpret_cast<const double2*>(a.pg)[e];
      const double2 ppv = reinterpret_cast<const double2*>(a.pgp)[e];
      const double dj = a.d[j], dpj = a.dp[j];
      {
        const double s = xv.x - xpv.x;
        const double y = (pv.x - dj * xv.x) - (ppv.x - dpj * xpv.x);
        ss += s * s;
        sy += s * y;
        yy += y * y;
      }
      {
        const double s = xv.y - xpv.y;
        const double y = (pv.y - dj * xv.y) - (ppv.y - dpj * xpv.y);
        ss += s * s;
        sy += s * y;
        yy += y * y;
      }
    }
    const double bs = block_sum<kStreamThreads>(ss, sm);
    const double by = block_sum<kStreamThreads>(sy, sm);
    const double bc = block_sum<kStreamThreads>(yy, sm);
    if (threadIdx.x == 0) {
      a.bbpart[blockIdx.x * 3 + 0] = bs;
      a.bbpart[blockIdx.x * 3 + 1] = by;
      a.bbpart[blockIdx.x * 3 + 2] = bc;
    }
  }
  grid.sync();
  // ---- phase 2: η (k_eta), redundantly in every block
  {
    double ss = 0.0, sy = 0.0, yy = 0.0;
    if (need) {
      double s1 = 0.0, s2 = 0.0, s3 = 0.0;
      for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
        s1 += a.bbpart[3 * i + 0];
        s2 += a.bbpart[3 * i + 1];
        s3 += a.bbpart[3 * i + 2];
      }
      ss = block_sum<kStreamThreads>(s1, sm);
      sy = block_sum<kStreamThreads>(s2, sm);
      yy = block_sum<kStreamThreads>(s3, sm);
    }
    if (threadIdx.x == 0) s_eta = select_eta(ctl, ss, sy, yy, need);
    __syncthreads();
  }
  const double eta = s_eta;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->eta = eta;
    ctl->step_deg = 0;
    if (!(eta > 0.0)) {
      ctl->step_param = 1;
      ctl->done = 3;
    }
  }
  if (!(eta > 0.0)) return false;  // uniform
  // ---- phase 3: Z = X − (1/η)(P − d∘X), column-norm partials (k_update)
  const double inv_eta = 1.0 / eta;
  const int64_t items = a.nchunks * a.p;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t c = it % a.nchunks, j = it / a.nchunks;
    const int64_t r0 = c * a.chunk, r1 = min(a.n, r0 + a.chunk);
    const double dj = a.d[j];
    const double* xj = a.x + j * a.ld;
    const double* pj = a.pg + j * a.ld;
    double* zj = a.z + j * a.ld;
    double acc = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
      const double xv = xj[i];
      const double gl = pj[i] - dj * xv;
      const double v = xv - inv_eta * gl;
      zj[i] = v;
      acc += v * v;
    }
    const double s = block_sum<kStreamThreads>(acc, sm);
    if (threadIdx.x == 0) a.npart[c * a.p + j] = s;
  }
  grid.sync();
  // ---- phase 4: normalisation + degenerate columns + finiteness (k_normalize)
  bool bad = false;
  if (a.plain) {
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
      const int64_t c = it % a.nchunks, j = it / a.nchunks;
      const int64_t r0 = c * a.chunk, r1 = min(a.n, r0 + a.chunk);
      for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) bad |= !isfinite(a.z[j * a.ld + i]);
    }
  }
  for (int64_t it = blockIdx.x; it < items && !a.plain; it += gridDim.x) {
    const int64_t c = it % a.nchunks, j = it / a.nchunks;
    const int64_t r0 = c * a.chunk, r1 = min(a.n, r0 + a.chunk);
    if (threadIdx.x < 32) {  // same fixed order as k_normalize
      double nrm2 = 0.0;
      for (int64_t q = threadIdx.x; q < a.nchunks; q += 32) nrm2 += a.npart[q * a.p + j];
      nrm2 = warp_sum(nrm2);
      if (threadIdx.x == 0) {
        const double nz = sqrt(nrm2);
        s_deg = nz < 1e-14;
        s_inv = 1.0 / nz;
      }
    }
    __syncthreads();
    double* zj = a.z + j * a.ld;
    if (!s_deg) {
      bad |= scale_range(zj, r0, r1, s_inv);
    } else {
      const double* xj = a.x + j * a.ld;
      double acc = 0.0;
      for (int64_t i = threadIdx.x; i < a.n; i += blockDim.x) acc += xj[i] * xj[i];
      const double pn2 = block_sum<kStreamThreads>(acc, sm);
      if (threadIdx.x == 0) sm[0] = sqrt(pn2);
      __syncthreads();
      const double pn = sm[0];
      for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        double v;
        if (pn > 0.0) v = xj[i] * (1.0 / pn);
        else v = (i == (j % a.n_glob)) ? 1.0 : 0.0;
        zj[i] = v;
        bad |= !isfinite(v);
      }
      if (c == 0 && threadIdx.x == 0) atomicAdd(&ctl->step_deg, 1);
    }
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) {
    ctl->step_bad = 1;
    ctl->done = 2;
  }
  return true;
}

__global__ void __launch_bounds__(kStreamThreads) k_step_fused(StepArgs a, Ctl* ctl) {
  if (ctl->done) return;  // uniform: nothing writes `done` before this kernel ends
  step_phase(a, ctl);
}

}  // namespace pcal
