// small_rows.cuh — the PCAL iteration of a small dense problem (config 1:
// n = 1000, p = 20) as ONE persistent cooperative kernel with FOUR grid
// barriers per iteration (k_iter_small has five and moves every n×p object
// through L2 in every phase).
//
// Ownership: CTA c owns the 8 rows [8c, 8c+8) of every n×p object, and
// thread e of its 256 owns element (row 8c + (e & 7), column e >> 3).  X_k,
// P_k, X_{k−1}, P_{k−1} of that element live in the thread's registers for a
// whole batch of iterations; its 8 rows of A live in registers too, as the
// DMMA A-fragments of the warp's K range.  The only n×p object that crosses
// CTAs is Z = X − (1/η)·GL (the gradient needs all of it); everything else
// crosses as p×p or p-sized partial sums.
//
// Lazy normalisation.  pcal_step normalises z_j by ‖z_j‖ (solver.cpp:283-305)
// and the gradient is then G = A·X⁺ (+G0).  With X⁺ = Z·D, D = diag(1/‖z_j‖):
//   G = (A·Z)·D + G0,   GᵀX⁺ = D·(ZᵀA·Z)·D + G0ᵀZ·D,   X⁺ᵀX⁺ = D·(ZᵀZ)·D,
// so one pass over the rows yields the partials of ZᵀAZ (symmetrised), ZᵀZ
// (whose diagonal gives the norms) and G0ᵀZ, and the norms need no barrier
// of their own.  f = ½ Σ_j d_j² (ZᵀAZ)_jj + 2 d_j (G0ᵀZ)_jj.  The scaling
// changes the rounding order only (DESIGN.md §5 tolerances).  A degenerate
// column (‖z_j‖ < 1e-14) takes a second pass over the same phases with
// Y = X⁺ itself and D = I.
//
// Per iteration (solver.cpp:369-439):
//   1  η from the ⟨S,S⟩, ⟨S,Y⟩, ⟨Y,Y⟩ CTA partials; Z own rows → global   | barrier
//   2  A·Z own rows (DMMA, Z from L2); partials of ZᵀAZ, ZᵀZ, G0ᵀZ; the
//      last CTA of every group of 8 sums its group's partials              | barrier
//   3  totals (group order); D, W, C, M; X⁺, G, P own rows (the X·[W|M]
//      epilogue); KKT² and d_j column partials                             | barrier
//   4  column totals; trace record (CTA 0); ⟨S,S⟩, ⟨S,Y⟩, ⟨Y,Y⟩ partials   | barrier
// Every cross-CTA sum is taken in a fixed order (no atomics in any sum).
#pragma once

namespace pcal {

constexpr int kRowsThreads = 256;  // 8 rows × 32 columns, one element per thread
constexpr int kRowsKS = 32;        // k4-steps per warp (n ≤ 8·4·kRowsKS = 1024)
constexpr int kRowsGroup = 8;      // CTAs per partial-sum group
constexpr int kRowsMaxGrid = 128;  // n ≤ 1024 rows
// dynamic shared memory: warp K-partials of A·Y (8 × 256), three 32 × 33 p×p
// arrays, then Y (p columns of zld doubles)
inline size_t rows_smem_bytes(int64_t p, int64_t zld) {
  return (size_t)(8 * 256 + 3 * 32 * 33 + p * zld) * sizeof(double);
}
inline int64_t rows_zld(int64_t n) { return (n + 15) / 16 * 16 + 4; }

struct RowsArgs {
  double* pair[2];    // pair b: P = pair[b], X = pair[b] + ld·pp
  double* fkd[2];     // [f | kkt² | d] column sums per parity
  const double* at;   // Aᵀ (ldat × n): at[k + i·ldat] = A(i, k)
  int64_t ldat;
  const double* g0;   // linear term (ld) or null
  double* lam;        // Λ (p × p) of the dual-ascent variants
  double* z;          // Z (ld × pp, zero padding): the only n×p object shared by CTAs
  double* gpart;      // [gridDim][nent] CTA partials of [ZᵀAZ | ZᵀZ | G0ᵀZ]
  double* gtot;       // [ngroups][nent] group sums
  unsigned* gcnt;     // [ngroups] arrival counters (monotone)
  double* cpart;      // [gridDim][2][32] CTA column partials (KKT², d)
  double* bbpart;     // [gridDim][3] CTA partials of ⟨S,S⟩, ⟨S,Y⟩, ⟨Y,Y⟩
  int64_t n, ld, p, pp;
  int nent;           // partial entries: 2·p(p+1)/2 (+ p² with G0)
  int64_t zld;        // shared-memory column stride of Y (≡ 4 mod 16 doubles)
  int csize;          // CTAs per cluster (Y multicast), 1 = no cluster
  int plain;          // PLAM / PLAM-DA: no column normalisation
  int mc_mode;        // MC_PCAL / MC_DA
  int p_from_g;       // P = G + X·M (dual ascent)
  int dform;          // d_j = X_jᵀP_j (PCAL with the PCAL formula)
  double beta;        // β
  double beta_epi;    // β of the P update (1 for dual ascent)
  FinishArgs fa;      // trace, bad flag, model (mode 0)
  uint64_t* prof;     // optional: %globaltimer per phase boundary (CTA 0), [iters][8]
};

// A·Y for the warp's K range: CT 8-column tiles, kRowsKS k4-steps, the B
// fragments of 8 k-steps loaded before their DMMAs, eight accumulator sets
// (k-step u → set u mod 8: a DMMA's latency is far longer than its issue
// interval), the sets added in a fixed order at the end.  Steps past n read
// zeros (A's fragments are zero there too).
template <int CT>
__device__ __forceinline__ void rows_dmma(const double* sZ, int64_t zld,
                                          const double (&areg)[kRowsKS], int64_t k4b, int64_t n,
                                          int64_t p, int r8, int q4, double (&out)[4][2]) {
  constexpr int NSET = 8, B = 8;
  double c[NSET][CT][2];
#pragma unroll
  for (int q = 0; q < NSET; ++q)
#pragma unroll
    for (int t = 0; t < CT; ++t) c[q][t][0] = c[q][t][1] = 0.0;
  const double* zr = sZ + (int64_t)r8 * zld + k4b * 4 + q4;
  const int64_t kmax = n - (k4b * 4 + q4);  // k-offsets < kmax are rows of Y
#pragma unroll
  for (int u0 = 0; u0 < kRowsKS; u0 += B) {
    double yb[B][CT];
#pragma unroll
    for (int u = 0; u < B; ++u)
#pragma unroll
      for (int t = 0; t < CT; ++t) {
        const bool ok = (u0 + u) * 4 < kmax && t * 8 + r8 < p;
        yb[u][t] = ok ? zr[(int64_t)t * 8 * zld + (u0 + u) * 4] : 0.0;
      }
#pragma unroll
    for (int u = 0; u < B; ++u)
#pragma unroll
      for (int t = 0; t < CT; ++t)
        small_dmma(c[(u0 + u) % NSET][t][0], c[(u0 + u) % NSET][t][1], areg[u0 + u], yb[u][t]);
  }
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int h = 0; h < 2; ++h)
      out[t][h] = t < CT ? ((c[0][t < CT ? t : 0][h] + c[1][t < CT ? t : 0][h]) +
                            (c[2][t < CT ? t : 0][h] + c[3][t < CT ? t : 0][h])) +
                               ((c[4][t < CT ? t : 0][h] + c[5][t < CT ? t : 0][h]) +
                                (c[6][t < CT ? t : 0][h] + c[7][t < CT ? t : 0][h]))
                         : 0.0;
}

#define ROWS_STAMP(k) \
  if (a.prof && blockIdx.x == 0 && threadIdx.x == 0) a.prof[it * 16 + (k)] = globaltimer_ns()

__global__ void __launch_bounds__(kRowsThreads, 1) k_iter_rows(RowsArgs a, Ctl* ctl, int iters) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  constexpr int P = 32, NW = kRowsThreads / 32;
  extern __shared__ __align__(16) double rows_smem[];
  auto sG = reinterpret_cast<double(*)[4 * 64]>(rows_smem);   // [NW]: warp K-partials of A·Y
  auto sS = reinterpret_cast<double(*)[P + 1]>(rows_smem + NW * 4 * 64);  // YᵀAY (sym sum), then W
  auto sV = sS + P;                                            // YᵀY, then C
  auto sH = sV + P;                                            // G0ᵀY, then M
  double* sZ = rows_smem + NW * 4 * 64 + 3 * P * (P + 1);      // Y, column j at j·zld
  __shared__ __align__(8) uint64_t zbar;
  const unsigned zbar_a = (unsigned)__cvta_generic_to_shared(&zbar);
  unsigned zphase = 0;
  unsigned crank = 0;
  if (a.csize > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(crank));
  __shared__ double sAY[8][P + 1], sY[8][P + 1], sG0[8][P + 1], sX[8][P + 1];
  __shared__ double sd[P], sdp[P], sfc[P], skc[P], sdn[P], ssc[P];
  __shared__ double sred[2][NW][P];
  __shared__ double sm8[NW];
  __shared__ double s_eta;
  __shared__ int s_last, s_deg[P];
  __shared__ int32_t s_bad;
  __shared__ unsigned char s_pj[P * (P + 1) / 2], s_pk[P * (P + 1) / 2];
  __shared__ Ctl sctl;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r = tid & 7, j = tid >> 3;        // own element (row 8c + r, column j)
  const int r8 = lane >> 2, q4 = lane & 3;    // DMMA fragment coordinates
  const int64_t n = a.n, ld = a.ld, p = a.p, pp = a.pp;
  const int64_t i = (int64_t)blockIdx.x * 8 + r;
  const bool own = i < n && j < p;
  const int64_t ix = i + (int64_t)j * ld;
  const int G = gridDim.x, grp = blockIdx.x / kRowsGroup;
  const int gsize = min(kRowsGroup, G - grp * kRowsGroup), ngroups = (G + kRowsGroup - 1) / kRowsGroup;
  const int np2 = (int)(p * (p + 1) / 2);
  const int ct_n = (int)((p + 7) / 8);
  const int64_t k4n = (n + 3) / 4;
  const int64_t ks = (k4n + NW - 1) / NW;     // k4-steps per warp (≤ kRowsKS)
  const int64_t k4b = warp * ks;
  if (ctl->done) return;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(zbar_a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (a.csize > 1) {  // every CTA's barrier is initialised before any multicast lands
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  }
  // (j, k) pairs of the upper triangle, j ≤ k, column by column
  for (int e = tid; e < np2; e += kRowsThreads) {
    int k = 0;
    while ((k + 1) * (k + 2) / 2 <= e) ++k;
    s_pk[e] = (unsigned char)k;
    s_pj[e] = (unsigned char)(e - k * (k + 1) / 2);
  }
  // A fragments of this warp's K range (A is constant for the launch)
  double areg[kRowsKS];
  {
    const int64_t ia = (int64_t)blockIdx.x * 8 + r8;
#pragma unroll
    for (int u = 0; u < kRowsKS; ++u) {
      const int64_t k = (k4b + u) * 4 + q4;
      areg[u] = (u < ks && ia < n && k < n) ? a.at[k + ia * a.ldat] : 0.0;
    }
  }
  // register state of the own element: X_k, P_k, X_{k−1}, P_{k−1}
  double xc = 0.0, pc = 0.0, xo = 0.0, po = 0.0, g0v = 0.0;
  {
    const int b = (int)(ctl->iter & 1), nb = b ^ 1;
    if (own) {
      pc = a.pair[b][ix];
      xc = a.pair[b][ix + ld * pp];
      po = a.pair[nb][ix];
      xo = a.pair[nb][ix + ld * pp];
      if (a.g0) g0v = a.g0[ix];
    }
    if (tid < P) {
      sd[tid] = tid < p ? a.fkd[b][2 * p + tid] : 0.0;
      sdp[tid] = tid < p ? a.fkd[nb][2 * p + tid] : 0.0;
    }
    __syncthreads();
    // stepsize partials of the current step (S = X_k − X_{k−1}, Y = GL_k − GL_{k−1})
    const double sv = own ? xc - xo : 0.0;
    const double yv = own ? (pc - sd[j] * xc) - (po - sdp[j] * xo) : 0.0;
    const double b0 = block_sum<kRowsThreads>(sv * sv, sm8);
    const double b1 = block_sum<kRowsThreads>(sv * yv, sm8);
    const double b2 = block_sum<kRowsThreads>(yv * yv, sm8);
    if (tid == 0) {
      a.bbpart[blockIdx.x * 3 + 0] = b0;
      a.bbpart[blockIdx.x * 3 + 1] = b1;
      a.bbpart[blockIdx.x * 3 + 2] = b2;
    }
  }
  grid.sync();
  for (int it = 0; it < iters; ++it) {
    if (ctl->done) return;  // uniform: written before the last grid barrier
    ROWS_STAMP(0);
    const int b = (int)(ctl->iter & 1), nb = b ^ 1;
    double* Pn = a.pair[nb];
    double* Xn = Pn + ld * pp;
    // ---- 1: η (solver.cpp:212-251); Z = X − (1/η)·(P − d∘X) of the own rows
    double zv = 0.0;
    {
      const bool need = ctl->eta_kind != 0 && ctl->have_prev && ctl->iter != 0;
      double v0 = 0.0, v1 = 0.0, v2 = 0.0;
      if (tid < G) {
        v0 = a.bbpart[tid * 3 + 0];
        v1 = a.bbpart[tid * 3 + 1];
        v2 = a.bbpart[tid * 3 + 2];
      }
      v0 = warp_sum(v0);
      v1 = warp_sum(v1);
      v2 = warp_sum(v2);
      if (lane == 0) {
        sred[0][warp][0] = v0;
        sred[0][warp][1] = v1;
        sred[0][warp][2] = v2;
      }
      __syncthreads();
      if (tid == 0) {
        double ss = 0.0, sy = 0.0, yy = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          ss += sred[0][w][0];
          sy += sred[0][w][1];
          yy += sred[0][w][2];
        }
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
      if (own) {
        zv = xc - inv_eta * (pc - sd[j] * xc);
        a.z[ix] = zv;
      }
    }
    grid.sync();
    ROWS_STAMP(1);
    // ---- 2–3, pass 0 with Y = Z and D = diag(1/‖z_j‖); pass 1 (a degenerate
    //      column) with Y = X⁺ and D = I
    double xn = 0.0, pv = 0.0, gv = 0.0;
    bool gbad = false, sbad = false;
    const double* Y = a.z;
    double yown = zv;
    for (int pass = 0; pass < 2; ++pass) {
      // ---- 2: A·Y of the own rows; partials of YᵀAY (sym), YᵀY, G0ᵀY
      {
        // Y (all rows, p columns) → shared memory by the bulk-copy engine: one
        // copy per column; far fewer L2 requests in flight than per-thread loads
        // With a cluster of CS CTAs every CTA fetches the columns q ≡ its rank
        // (mod CS) once from L2 and multicasts them into all CS CTAs: L2
        // serves Y gridDim/CS times instead of gridDim times.
        if (tid == 0) {
          asm volatile("fence.proxy.async;\n" ::: "memory");  // Y was written by other CTAs
          const unsigned bytes = (unsigned)(((n + 1) / 2) * 16);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(zbar_a),
                       "r"(bytes * (unsigned)p) : "memory");
          if (a.csize == 1) {
            for (int q = 0; q < p; ++q)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                  ::"r"((unsigned)__cvta_generic_to_shared(sZ + (int64_t)q * a.zld)),
                  "l"(Y + (int64_t)q * ld), "r"(bytes), "r"(zbar_a) : "memory");
          } else {
            const unsigned short mask = (unsigned short)((1u << a.csize) - 1u);
            for (int q = (int)crank; q < p; q += a.csize)
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                  " [%0], [%1], %2, [%3], %4;\n"
                  ::"r"((unsigned)__cvta_generic_to_shared(sZ + (int64_t)q * a.zld)),
                  "l"(Y + (int64_t)q * ld), "r"(bytes), "r"(zbar_a), "h"(mask) : "memory");
          }
        }
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            "@!p bra W_%=;\n}\n" ::"r"(zbar_a), "r"(zphase) : "memory");
        zphase ^= 1u;
        if (pass == 0) ROWS_STAMP(6);
        double c[4][2];
        switch (ct_n) {  // block-uniform: one branch-free DMMA stream per tile count
          case 1: rows_dmma<1>(sZ, a.zld, areg, k4b, n, p, r8, q4, c); break;
          case 2: rows_dmma<2>(sZ, a.zld, areg, k4b, n, p, r8, q4, c); break;
          case 3: rows_dmma<3>(sZ, a.zld, areg, k4b, n, p, r8, q4, c); break;
          default: rows_dmma<4>(sZ, a.zld, areg, k4b, n, p, r8, q4, c); break;
        }
        if (pass == 0) ROWS_STAMP(7);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (t < ct_n) {
            sG[warp][t * 64 + r8 * 8 + 2 * q4] = c[t][0];
            sG[warp][t * 64 + r8 * 8 + 2 * q4 + 1] = c[t][1];
          }
        __syncthreads();
        double ay = 0.0;
        if (own) {
          const int t = j >> 3, cc = j & 7;
#pragma unroll
          for (int w = 0; w < NW; ++w) ay += sG[w][t * 64 + r * 8 + cc];
          gbad |= !isfinite(ay);
        }
        if (pass == 0) ROWS_STAMP(5);
        sAY[r][j] = ay;
        sY[r][j] = own ? yown : 0.0;
        sG0[r][j] = own ? g0v : 0.0;
        __syncthreads();
        double* gp = a.gpart + (int64_t)blockIdx.x * a.nent;
        for (int e = tid; e < a.nent; e += kRowsThreads) {
          double s = 0.0;
          if (e < np2) {  // (YᵀAY)_jk + (YᵀAY)_kj
            const int jj = s_pj[e], kk = s_pk[e];
#pragma unroll
            for (int q = 0; q < 8; ++q) s += sAY[q][jj] * sY[q][kk] + sAY[q][kk] * sY[q][jj];
          } else if (e < 2 * np2) {  // (YᵀY)_jk
            const int jj = s_pj[e - np2], kk = s_pk[e - np2];
#pragma unroll
            for (int q = 0; q < 8; ++q) s += sY[q][jj] * sY[q][kk];
          } else {  // (G0ᵀY)_jk, column-major p × p
            const int ee = e - 2 * np2, jj = ee % (int)p, kk = ee / (int)p;
#pragma unroll
            for (int q = 0; q < 8; ++q) s += sG0[q][jj] * sY[q][kk];
          }
          gp[e] = s;
        }
        // the last CTA of the group to arrive sums the group's partials in CTA order
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          const unsigned old = atomicAdd(&a.gcnt[grp], 1u);
          s_last = (old + 1u) % (unsigned)gsize == 0u;
          if (s_last) __threadfence();
        }
        __syncthreads();
        if (s_last) {
          const double* g0p = a.gpart + (int64_t)grp * kRowsGroup * a.nent;
          for (int e = tid; e < a.nent; e += kRowsThreads) {
            double v[kRowsGroup];  // every load in flight before the first add
#pragma unroll
            for (int q = 0; q < kRowsGroup; ++q)
              v[q] = q < gsize ? __ldcg(&g0p[(int64_t)q * a.nent + e]) : 0.0;
            double s = 0.0;
#pragma unroll
            for (int q = 0; q < kRowsGroup; ++q) s += v[q];
            a.gtot[(int64_t)grp * a.nent + e] = s;
          }
        }
        gv = ay;
      }
      grid.sync();
      if (pass == 0) ROWS_STAMP(2);
      // ---- 3: totals; D, W, C, M; X⁺, G, P of the own rows
      {
        for (int e = tid; e < a.nent; e += kRowsThreads) {
          constexpr int MG = kRowsMaxGrid / kRowsGroup;
          double v[MG];  // every load in flight before the first add
#pragma unroll
          for (int q = 0; q < MG; ++q)
            v[q] = q < ngroups ? __ldcg(&a.gtot[(int64_t)q * a.nent + e]) : 0.0;
          double s = 0.0;
#pragma unroll
          for (int q = 0; q < MG; ++q) s += v[q];
          if (e < np2) {
            sS[s_pj[e]][s_pk[e]] = s;
            sS[s_pk[e]][s_pj[e]] = s;
          } else if (e < 2 * np2) {
            sV[s_pj[e - np2]][s_pk[e - np2]] = s;
            sV[s_pk[e - np2]][s_pj[e - np2]] = s;
          } else {
            const int ee = e - 2 * np2;
            sH[ee % (int)p][ee / (int)p] = s;
          }
        }
        __syncthreads();
        if (pass == 0) ROWS_STAMP(8);
        if (tid < P) {
          double sc = 1.0;
          int deg = 0;
          if (tid < p && pass == 0 && !a.plain) {
            const double nz = sqrt(sV[tid][tid]);
            deg = nz < 1e-14;
            sc = 1.0 / nz;
          }
          ssc[tid] = sc;
          s_deg[tid] = deg;
          // column value of f: x_jᵀ(A·x_j + 2·g0_j)
          sfc[tid] = tid < p ? sc * sc * (0.5 * sS[tid][tid]) + (a.g0 ? 2.0 * sc * sH[tid][tid] : 0.0)
                             : 0.0;
        }
        const int nd = __syncthreads_count(tid < P && s_deg[tid]);
        if (nd) {  // pass 0 only: X⁺ with the degenerate-column rule, then pass 1
          if (own) {
            if (!s_deg[j]) {
              xn = zv * ssc[j];
            } else {  // the previous column renormalised, or e_{j mod n}
              const double* xb = a.pair[b] + ld * pp + (int64_t)j * ld;
              double pn = 0.0;
              for (int64_t q = 0; q < n; ++q) pn += xb[q] * xb[q];
              pn = sqrt(pn);
              xn = pn > 0.0 ? xc * (1.0 / pn) : (i == (j % n) ? 1.0 : 0.0);
            }
            Xn[ix] = xn;
            sbad |= !isfinite(xn);
          }
          if (blockIdx.x == 0 && tid == 0) ctl->step_deg = nd;
          grid.sync();
          Y = Xn;
          yown = xn;
          gbad = false;
          continue;
        }
        // W = ½(GᵀX + XᵀG), C = XᵀX − I, M per algorithm (k_small_pxp)
        {
          double wr[4], cr[4], mr[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = tid + u * kRowsThreads;
            if (e >= p * p) continue;
            const int k = e % (int)p, jj = e / (int)p;
            const double dk = ssc[k], dj = ssc[jj];
            double w = 0.5 * (dk * dj * sS[k][jj]);
            if (a.g0) w += 0.5 * (sH[k][jj] * dj + sH[jj][k] * dk);
            double cv = dk * dj * sV[k][jj];
            if (k == jj) cv += -1.0;
            double m = cv;
            if (a.mc_mode == MC_DA) m = a.beta * cv - (a.lam[k + jj * p] + -a.beta * cv);
            wr[u] = w;
            cr[u] = cv;
            mr[u] = m;
          }
          __syncthreads();  // every thread has read its sS / sV / sH entries
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int e = tid + u * kRowsThreads;
            if (e >= p * p) continue;
            const int k = e % (int)p, jj = e / (int)p;
            sS[k][jj] = wr[u];
            sV[k][jj] = cr[u];
            sH[k][jj] = mr[u];
          }
          __syncthreads();
          if (pass == 0) ROWS_STAMP(9);
        }
        if (own) {
          if (pass == 0) xn = yown * ssc[j];
          gv = gv * ssc[j] + g0v;
          sbad |= !isfinite(xn);
          gbad |= !isfinite(gv);
        }
        sX[r][j] = own ? xn : 0.0;
        __syncthreads();
        if (pass == 0) ROWS_STAMP(10);
        double kacc = 0.0, dacc = 0.0;
        if (own) {
          double t1 = 0.0, t2 = 0.0;
          for (int k = 0; k < p; ++k) {
            t1 = fma(sX[r][k], sS[k][j], t1);
            t2 = fma(sX[r][k], sH[k][j], t2);
          }
          const double kkt = gv - t1;
          pv = (a.p_from_g ? gv : kkt) + a.beta_epi * t2;
          Xn[ix] = xn;
          Pn[ix] = pv;
          kacc = kkt * kkt;
          dacc = xn * pv;
        }
        // the 8 rows of column j sit in 8 consecutive lanes: fixed-order sums
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          kacc += __shfl_xor_sync(0xffffffffu, kacc, o);
          dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
        }
        if (r == 0) {
          a.cpart[((int64_t)blockIdx.x * 2 + 0) * P + j] = kacc;
          a.cpart[((int64_t)blockIdx.x * 2 + 1) * P + j] = dacc;
        }
        if (__syncthreads_or(sbad) && tid == 0) {
          ctl->step_bad = 1;
          ctl->done = 2;
        }
        if (__syncthreads_or(gbad) && tid == 0) *a.fa.bad = 1;
        break;
      }
    }
    grid.sync();
    ROWS_STAMP(3);
    // non-finite step (not `done`: CTA 0 may already be recording below)
    if (ctl->step_bad) return;
    // ---- 4: column totals, record (CTA 0), stepsize partials of step k+1
    {
      constexpr int CW = (int)(sizeof(Ctl) / sizeof(uint32_t));
      static_assert(sizeof(Ctl) % sizeof(uint32_t) == 0, "Ctl copy");
      if (blockIdx.x == 0) {  // CTA 0 records: its loads overlap the column totals'
        if (tid < CW)
          reinterpret_cast<uint32_t*>(&sctl)[tid] = __ldcg(reinterpret_cast<const uint32_t*>(ctl) + tid);
        if (tid == CW) s_bad = __ldcg(a.fa.bad);
      }
      constexpr int BPW = kRowsMaxGrid / NW;
      double v[2][BPW];
#pragma unroll
      for (int u = 0; u < BPW; ++u) {
        const int q = warp * BPW + u;
        const bool ok = q < G && lane < p;
#pragma unroll
        for (int w2 = 0; w2 < 2; ++w2)
          v[w2][u] = ok ? __ldcg(&a.cpart[((int64_t)q * 2 + w2) * P + lane]) : 0.0;
      }
#pragma unroll
      for (int w2 = 0; w2 < 2; ++w2) {
        double t = 0.0;
#pragma unroll
        for (int u = 0; u < BPW; ++u) t += v[w2][u];
        sred[w2][warp][lane] = t;
      }
      __syncthreads();
      if (tid < 2 * P) {
        const int w2 = tid / P, jj = tid % P;
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) t += sred[w2][w][jj];
        if (w2 == 0) skc[jj] = t;
        else sdn[jj] = a.dform ? t : 0.0;  // d stays 0 without the PCAL formula
      }
      __syncthreads();
      ROWS_STAMP(11);
      if (blockIdx.x == 0) {
        if (tid < p) {
          double* fk = a.fkd[nb];
          fk[tid] = sfc[tid];
          fk[p + tid] = skc[tid];
          fk[2 * p + tid] = sdn[tid];
        }
        double cc = 0.0;  // ‖XᵀX − I‖²
        for (int e = tid; e < p * p; e += kRowsThreads) {
          const int k = e % (int)p, jj = e / (int)p;
          const double cv = sV[k][jj];
          cc += cv * cv;
          if (a.mc_mode == MC_DA) a.lam[e] = a.lam[e] + -a.beta * cv;  // Λ ← Λ − β·C
        }
        const double c2 = block_sum<kRowsThreads>(cc, sm8);  // (synchronises the block)
        if (tid == 0) {
          double f1 = 0.0, k2 = 0.0;
          for (int64_t q = 0; q < p; ++q) {
            f1 += sfc[q];
            k2 += skc[q];
          }
          FinishArgs fa = a.fa;
          fa.bad = &s_bad;  // prefetched above; finish_record clears it
          const int32_t was_bad = s_bad;
          finish_record(fa, &sctl, nullptr, f1, k2, c2, 0.0, 0.0, 0.0);
          if (was_bad) *a.fa.bad = 0;
        }
        __syncthreads();
        if (tid < CW)
          reinterpret_cast<uint32_t*>(ctl)[tid] = reinterpret_cast<const uint32_t*>(&sctl)[tid];
      }
      ROWS_STAMP(12);
      // S = X⁺ − X, Y = (P⁺ − d⁺∘X⁺) − (P − d∘X)
      const double sv = own ? xn - xc : 0.0;
      const double yv = own ? (pv - sdn[j] * xn) - (pc - sd[j] * xc) : 0.0;
      const double b0 = block_sum<kRowsThreads>(sv * sv, sm8);
      const double b1 = block_sum<kRowsThreads>(sv * yv, sm8);
      const double b2 = block_sum<kRowsThreads>(yv * yv, sm8);
      if (tid == 0) {
        a.bbpart[blockIdx.x * 3 + 0] = b0;
        a.bbpart[blockIdx.x * 3 + 1] = b1;
        a.bbpart[blockIdx.x * 3 + 2] = b2;
      }
      xo = xc;
      po = pc;
      xc = xn;
      pc = pv;
      __syncthreads();
      ROWS_STAMP(13);
      if (tid < P) {
        sdp[tid] = sd[tid];
        sd[tid] = sdn[tid];
      }
    }
    grid.sync();
    ROWS_STAMP(4);
  }
}
#undef ROWS_STAMP

}  // namespace pcal
