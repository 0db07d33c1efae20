// operators.cuh — device gradient evaluation for the grid models (the
// ObjectiveModel::evaluate callback of problems.hpp:39, restated for the
// configs without a reference implementation; definitions in DESIGN.md §3).
//
// Arithmetic uses explicit round-to-nearest intrinsics (no FMA contraction) in
// the same left-to-right order as the oracle (oracle/pcal_oracle.c
// orc_laplacian_apply / orc_evaluate), so the stencil gradient is bitwise equal
// to the oracle's; only the objective's reduction order differs.
#pragma once

#include "common.cuh"

namespace pcal {

constexpr int kStencilThreads = 256;
constexpr int kStreamThreadsOps = 256;

// G = L X + V∘X with L = −Δ_h (7-point, periodic, h = 1) and, for the
// Kohn–Sham model, G = ½ L X + u∘X (scale_l = 0.5, u = V + L†ρ − c ρ^{1/3}).
// fpart[j·pstride + chunk] = Σ_{rows of chunk} X∘G (X∘LX for the KS model).
// Grid: (n / chunk, p); one thread per row element, x-fastest for coalescing.
template <bool KS>
__global__ void __launch_bounds__(kStencilThreads)
    k_stencil_grad(const double* __restrict__ x, const double* __restrict__ u,
                   double* __restrict__ g, int64_t nx, int64_t ny, int64_t nz, int64_t ld,
                   int64_t p, int64_t chunk, double* __restrict__ fpart, int64_t pstride,
                   int32_t* bad, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  __shared__ double sm[kStencilThreads / 32];
  const int64_t n = nx * ny * nz;
  const int64_t j = blockIdx.y;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  const int64_t r1 = min(n, r0 + chunk);
  const double* xj = x + j * ld;
  double* gj = g + j * ld;
  const int64_t nxy = nx * ny;
  double acc = 0.0;
  bool nonfinite = false;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    const int64_t xx = i % nx;
    const int64_t y = (i / nx) % ny;
    const int64_t z = i / nxy;
    const int64_t xm = i + (xx == 0 ? nx - 1 : -1);
    const int64_t xp = i + (xx == nx - 1 ? 1 - nx : 1);
    const int64_t ym = i + (y == 0 ? (ny - 1) * nx : -nx);
    const int64_t yp = i + (y == ny - 1 ? (1 - ny) * nx : nx);
    const int64_t zm = i + (z == 0 ? (nz - 1) * nxy : -nxy);
    const int64_t zp = i + (z == nz - 1 ? (1 - nz) * nxy : nxy);
    const double xv = __ldg(xj + i);
    double lx = __dmul_rn(6.0, xv);
    lx = __dsub_rn(lx, __ldg(xj + xm));
    lx = __dsub_rn(lx, __ldg(xj + xp));
    lx = __dsub_rn(lx, __ldg(xj + ym));
    lx = __dsub_rn(lx, __ldg(xj + yp));
    lx = __dsub_rn(lx, __ldg(xj + zm));
    lx = __dsub_rn(lx, __ldg(xj + zp));
    double gv;
    if (KS) gv = __dadd_rn(__dmul_rn(0.5, lx), __dmul_rn(__ldg(u + i), xv));
    else gv = __dadd_rn(lx, __dmul_rn(__ldg(u + i), xv));
    gj[i] = gv;
    acc += KS ? xv * lx : xv * gv;
    nonfinite |= !isfinite(gv);
  }
  const double s = block_sum<kStencilThreads>(acc, sm);
  if (threadIdx.x == 0) fpart[j * pstride + blockIdx.x] = s;
  if (__syncthreads_or(nonfinite) && threadIdx.x == 0) *bad = 1;
}

// z-marching 2.5D stencil for grids with nx ≤ 32·XP and ny % TY == 0: a block
// owns an nx × TY tile of the xy-plane of one column j and walks a z-range;
// each thread keeps its points of planes z−1, z, z+1 in registers and the
// current plane (+ periodic y-halo rows) in shared memory, so every X value is
// read from HBM once (halo rows: 2/TY extra, mostly L2 hits).  Same operation
// order as k_stencil_grad (bitwise identical results).
#ifndef PCAL_STENCIL_MINB
#define PCAL_STENCIL_MINB 4  // ≤ 64 registers: 32 resident warps per SM for the plane pipeline
#endif
template <bool KS, int XP, int TY>
__global__ void __launch_bounds__(32 * TY, PCAL_STENCIL_MINB)
    k_stencil_march(const double* __restrict__ x, const double* __restrict__ u,
                    double* __restrict__ g, int nx, int ny, int nz, int64_t ld, int zchunk,
                    double* __restrict__ fpart, int64_t pstride, int32_t* bad, const Ctl* ctl,
                    const double* __restrict__ hlo, const double* __restrict__ hhi, int zpart) {
  if (ctl && ctl->done) return;
  constexpr int W = 32 * XP;  // smem row width (≥ nx)
  __shared__ double pl[TY + 2][W];
  __shared__ double sm[TY];
  const int lane = threadIdx.x, ty = threadIdx.y;
  const int y0 = blockIdx.x * TY;
  const int zc = blockIdx.y;
  const int64_t j = blockIdx.z;
  const int z0 = zc * zchunk;
  const int z1 = min(nz, z0 + zchunk);
  const int y = y0 + ty;
  const int64_t nxy = (int64_t)nx * ny;
  const double* xj = x + j * ld;
  double* gj = g + j * ld;
  const int yh = ty == 0 ? (y0 == 0 ? ny - 1 : y0 - 1) : (y0 + TY == ny ? 0 : y0 + TY);
  // all global loads run one z-step ahead: planes z+1 (interior), the y-halo
  // rows of plane z+1 and the potential u of plane z+1 are fetched while
  // plane z is computed
  // halo rows are consumed at the START of an iteration (smem fill), so they
  // are fetched two planes ahead; interior planes and u one plane ahead
  double below[XP], cur[XP], above[XP], halo[XP], halo_n[XP], uc[XP];
  // plane z of column j: periodic wrap on a single GPU; on a z-slab of a
  // sharded grid, planes −1 and nz come from the neighbours' halo planes
  auto src = [&](int z) -> const double* {
    if (hlo) {
      if (z < 0) return hlo + j * nxy;
      if (z >= nz) return hhi + j * nxy;
      return xj + (int64_t)z * nxy;
    }
    return xj + (int64_t)((z % nz + nz) % nz) * nxy;
  };
  const bool hrow = ty == 0 || ty == TY - 1;
#pragma unroll
  for (int k = 0; k < XP; ++k) {
    const int xx = lane + 32 * k;
    const bool ok = xx < nx;
    below[k] = ok ? __ldg(src(z0 - 1) + (int64_t)y * nx + xx) : 0.0;
    cur[k] = ok ? __ldg(src(z0) + (int64_t)y * nx + xx) : 0.0;
    above[k] = ok ? __ldg(src(z0 + 1) + (int64_t)y * nx + xx) : 0.0;
    halo[k] = (ok && hrow) ? __ldg(src(z0) + (int64_t)yh * nx + xx) : 0.0;
    halo_n[k] = (ok && hrow && z0 + 1 < z1) ? __ldg(src(z0 + 1) + (int64_t)yh * nx + xx) : 0.0;
    uc[k] = ok ? __ldg(u + (int64_t)z0 * nxy + (int64_t)y * nx + xx) : 0.0;
  }
  double acc = 0.0;
  bool nonfinite = false;
  // plane z+2 (wrapped) and the f-partial counters advance incrementally: no
  // integer division on the per-plane path (the kernel is issue-bound otherwise)
  int zw = (z0 + 2) % nz;
  int zp_cnt = z0 % zpart, zp_idx = z0 / zpart;
  for (int z = z0; z < z1; ++z) {
    const double* sa = hlo ? src(z + 2) : xj + (int64_t)zw * nxy;
    zw = zw + 1 == nz ? 0 : zw + 1;
    const int64_t pz = (int64_t)z * nxy, pn = pz + nxy;
#pragma unroll
    for (int k = 0; k < XP; ++k) {
      const int xx = lane + 32 * k;
      if (xx < nx) {
        pl[ty + 1][xx] = cur[k];
        if (hrow) pl[ty == 0 ? 0 : TY + 1][xx] = halo[k];
      }
    }
    __syncthreads();
    double above2[XP], halo_nn[XP], u_n[XP];
    const bool more = z + 1 < z1, more2 = z + 2 < z1;
#pragma unroll
    for (int k = 0; k < XP; ++k) {
      const int xx = lane + 32 * k;
      const bool ok = xx < nx && more;
      above2[k] = ok ? __ldg(sa + (int64_t)y * nx + xx) : 0.0;
      halo_nn[k] = (xx < nx && more2 && hrow) ? __ldg(sa + (int64_t)yh * nx + xx) : 0.0;
      u_n[k] = ok ? __ldg(u + pn + (int64_t)y * nx + xx) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < XP; ++k) {
      const int xx = lane + 32 * k;
      if (xx < nx) {
        const int xm = xx == 0 ? nx - 1 : xx - 1;
        const int xp = xx == nx - 1 ? 0 : xx + 1;
        const double xv = cur[k];
        double lx = __dmul_rn(6.0, xv);
        lx = __dsub_rn(lx, pl[ty + 1][xm]);
        lx = __dsub_rn(lx, pl[ty + 1][xp]);
        lx = __dsub_rn(lx, pl[ty][xx]);
        lx = __dsub_rn(lx, pl[ty + 2][xx]);
        lx = __dsub_rn(lx, below[k]);
        lx = __dsub_rn(lx, above[k]);
        const int64_t i = pz + (int64_t)y * nx + xx;
        double gv;
        if (KS) gv = __dadd_rn(__dmul_rn(0.5, lx), __dmul_rn(uc[k], xv));
        else gv = __dadd_rn(lx, __dmul_rn(uc[k], xv));
        gj[i] = gv;
        acc += KS ? xv * lx : xv * gv;
        // stencil model: a non-finite G makes Σ X∘G non-finite (x·±inf and
        // 0·inf are never finite), so the partial sum is checked at its flush
        if (KS) nonfinite |= !isfinite(gv);
      }
      below[k] = cur[k];
      cur[k] = above[k];
      above[k] = above2[k];
      halo[k] = halo_n[k];
      halo_n[k] = halo_nn[k];
      uc[k] = u_n[k];
    }
    // block reduction (fixed order) → one f partial per (tile, zpart planes):
    // once per z-chunk (zpart = zchunk), or per row chunk on the sharded path
    if (++zp_cnt == zpart || z + 1 == z1) {
      if (!KS) nonfinite |= !isfinite(acc);
      const double v = warp_sum(acc);
      if (lane == 0) sm[ty] = v;
      __syncthreads();
      if (lane == 0 && ty == 0) {
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < TY; ++t) s += sm[t];
        fpart[j * pstride + blockIdx.x + (int64_t)gridDim.x * zp_idx] = s;
      }
      acc = 0.0;
      if (zp_cnt == zpart) {
        zp_cnt = 0;
        ++zp_idx;
      }
    }
    __syncthreads();
  }
  if (__syncthreads_or(nonfinite) && lane == 0 && ty == 0) *bad = 1;
}

// Full-row variant (nx = L·XP with L ≤ 32 active lanes, XP even): lane l owns
// the XP consecutive points x = XP·l … XP·l + XP − 1, so X, u and G move as
// 16-byte vectors and the x-neighbours come from registers and two warp
// shuffles (one row per warp: the periodic wrap is the wrap over the L active
// lanes); shared memory carries only the y-neighbour rows.  Same operands in the same order as
// k_stencil_march: G is bitwise identical; the f partial sums its terms in a
// different (fixed) per-thread order.
template <bool KS, int XP, int TY>
__global__ void __launch_bounds__(32 * TY, PCAL_STENCIL_MINB)
    k_stencil_march_row(const double* __restrict__ x, const double* __restrict__ u,
                        double* __restrict__ g, int nx, int ny, int nz, int64_t ld, int zchunk,
                        double* __restrict__ fpart, int64_t pstride, int32_t* bad, const Ctl* ctl,
                        const double* __restrict__ hlo, const double* __restrict__ hhi,
                        int zpart) {
  static_assert(XP % 2 == 0, "full-row march: XP even (16-byte vectors)");
  constexpr int V = XP / 2;
  if (ctl && ctl->done) return;
  __shared__ __align__(16) double pl[TY + 2][32 * XP];
  __shared__ double sm[TY];
  const int lane = threadIdx.x, ty = threadIdx.y;
  const int L = nx / XP;      // active lanes
  const int ln = lane < L ? lane : L - 1;  // idle lanes shadow the last one (no stores)
  const bool act = lane < L;
  const int y0 = blockIdx.x * TY;
  const int z0 = blockIdx.y * zchunk;
  const int z1 = min(nz, z0 + zchunk);
  const int64_t j = blockIdx.z;
  const int y = y0 + ty;
  const int64_t nxy = (int64_t)nx * ny;
  const double* xj = x + j * ld;
  double* gj = g + j * ld;
  const int yh = ty == 0 ? (y0 == 0 ? ny - 1 : y0 - 1) : (y0 + TY == ny ? 0 : y0 + TY);
  const bool hrow = ty == 0 || ty == TY - 1;
  const int64_t row = (int64_t)y * nx + XP * ln, hrw = (int64_t)yh * nx + XP * ln;
  auto src = [&](int z) -> const double* {
    if (hlo) {
      if (z < 0) return hlo + j * nxy;
      if (z >= nz) return hhi + j * nxy;
      return xj + (int64_t)z * nxy;
    }
    return xj + (int64_t)((z % nz + nz) % nz) * nxy;
  };
  auto ld2 = [](const double* p, double (&d)[XP]) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(p) + v);
      d[2 * v] = t.x;
      d[2 * v + 1] = t.y;
    }
  };
  double below[XP], cur[XP], above[XP], halo[XP], halo_n[XP], uc[XP];
  ld2(src(z0 - 1) + row, below);
  ld2(src(z0) + row, cur);
  ld2(src(z0 + 1) + row, above);
  ld2(u + (int64_t)z0 * nxy + row, uc);
#pragma unroll
  for (int k = 0; k < XP; ++k) halo[k] = halo_n[k] = 0.0;
  if (hrow) {
    ld2(src(z0) + hrw, halo);
    if (z0 + 1 < z1) ld2(src(z0 + 1) + hrw, halo_n);
  }
  double acc = 0.0;
  bool nonfinite = false;
  int zw = (z0 + 2) % nz;
  int zp_cnt = z0 % zpart, zp_idx = z0 / zpart;
  double2* prow = reinterpret_cast<double2*>(&pl[ty + 1][XP * lane]);
  double2* phal = reinterpret_cast<double2*>(&pl[ty == 0 ? 0 : TY + 1][XP * lane]);
  const double2* pdn = reinterpret_cast<const double2*>(&pl[ty][XP * lane]);
  const double2* pup = reinterpret_cast<const double2*>(&pl[ty + 2][XP * lane]);
  const int lsrc = ln == 0 ? L - 1 : ln - 1, rsrc = ln == L - 1 ? 0 : ln + 1;
  for (int z = z0; z < z1; ++z) {
    const double* sa = hlo ? src(z + 2) : xj + (int64_t)zw * nxy;
    zw = zw + 1 == nz ? 0 : zw + 1;
    const int64_t pz = (int64_t)z * nxy, pn = pz + nxy;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      prow[v] = make_double2(cur[2 * v], cur[2 * v + 1]);
      if (hrow) phal[v] = make_double2(halo[2 * v], halo[2 * v + 1]);
    }
    __syncthreads();
    double above2[XP], halo_nn[XP], u_n[XP];
#pragma unroll
    for (int k = 0; k < XP; ++k) above2[k] = halo_nn[k] = u_n[k] = 0.0;
    if (z + 1 < z1) {
      ld2(sa + row, above2);
      ld2(u + pn + row, u_n);
    }
    if (hrow && z + 2 < z1) ld2(sa + hrw, halo_nn);
    double dn[XP], up[XP];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double2 a = pdn[v], b = pup[v];
      dn[2 * v] = a.x;
      dn[2 * v + 1] = a.y;
      up[2 * v] = b.x;
      up[2 * v + 1] = b.y;
    }
    const double left = __shfl_sync(0xffffffffu, cur[XP - 1], lsrc);
    const double right = __shfl_sync(0xffffffffu, cur[0], rsrc);
    double gv[XP];
#pragma unroll
    for (int k = 0; k < XP; ++k) {
      const double xv = cur[k];
      double lx = __dmul_rn(6.0, xv);
      lx = __dsub_rn(lx, k == 0 ? left : cur[k - 1]);
      lx = __dsub_rn(lx, k == XP - 1 ? right : cur[k + 1]);
      lx = __dsub_rn(lx, dn[k]);
      lx = __dsub_rn(lx, up[k]);
      lx = __dsub_rn(lx, below[k]);
      lx = __dsub_rn(lx, above[k]);
      if (KS) gv[k] = __dadd_rn(__dmul_rn(0.5, lx), __dmul_rn(uc[k], xv));
      else gv[k] = __dadd_rn(lx, __dmul_rn(uc[k], xv));
      if (act) {
        acc += KS ? xv * lx : xv * gv[k];
        if (KS) nonfinite |= !isfinite(gv[k]);
      }
    }
    if (act) {
      double2* gout = reinterpret_cast<double2*>(gj + pz + row);
#pragma unroll
      for (int v = 0; v < V; ++v) gout[v] = make_double2(gv[2 * v], gv[2 * v + 1]);
    }
#pragma unroll
    for (int k = 0; k < XP; ++k) {
      below[k] = cur[k];
      cur[k] = above[k];
      above[k] = above2[k];
      halo[k] = halo_n[k];
      halo_n[k] = halo_nn[k];
      uc[k] = u_n[k];
    }
    if (++zp_cnt == zpart || z + 1 == z1) {
      if (!KS) nonfinite |= !isfinite(acc);
      const double v = warp_sum(acc);
      if (lane == 0) sm[ty] = v;
      __syncthreads();
      if (lane == 0 && ty == 0) {
        double sacc = 0.0;
#pragma unroll
        for (int t = 0; t < TY; ++t) sacc += sm[t];
        fpart[j * pstride + blockIdx.x + (int64_t)gridDim.x * zp_idx] = sacc;
      }
      acc = 0.0;
      if (zp_cnt == zpart) {
        zp_cnt = 0;
        ++zp_idx;
      }
    }
    __syncthreads();
  }
  if (__syncthreads_or(nonfinite) && lane == 0 && ty == 0) *bad = 1;
}

// Halo send planes of a z-slab: lo = plane 0, hi = plane nzl−1 of every column.
__global__ void k_pack_planes(const double* __restrict__ x, int64_t ld, int64_t nxy, int64_t nzl,
                              double* __restrict__ lo, double* __restrict__ hi, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t j = blockIdx.y;
  if (e >= nxy) return;
  lo[j * nxy + e] = x[j * ld + e];
  hi[j * nxy + e] = x[j * ld + (nzl - 1) * nxy + e];
}

// Gathered rank blocks (R × [ld_blk × cols]) → global row order (ld_out × cols):
// out[row0_r + i + c·ld_out] = in[r·ld_blk·cols + c·ld_blk + i], i < rows_r.
__global__ void k_unpack_rows(const double* __restrict__ in, int64_t ld_blk, int64_t cols,
                              const int64_t* __restrict__ rr /* row0[R], rows[R] */, int R,
                              double* __restrict__ out, int64_t ld_out, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c = blockIdx.y;
  const int r = blockIdx.z;
  if (i >= rr[R + r]) return;
  out[rr[r] + i + c * ld_out] = in[(int64_t)r * ld_blk * cols + c * ld_blk + i];
}

// ρ_i = Σ_j X_ij² (row_sq_norms, kernels.cpp:295-303 order: column-outer).
__global__ void k_row_sq_norms(const double* __restrict__ x, int64_t n, int64_t ld, int64_t p,
                               double* __restrict__ rho, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t j = 0; j < p; ++j) {
    const double v = x[i + j * ld];
    s = __dadd_rn(s, __dmul_rn(v, v));
  }
  rho[i] = s;
}

// One axis of the separable real Fourier transform of an n-vector on the grid
// (oracle axis_transform): forward out[..o..] = Σ_i Q[i,o]·in[..i..],
// inverse out[..o..] = Σ_m Q[o,m]·in[..m..], index order, no contraction.
__global__ void k_axis_transform(const double* __restrict__ in, double* __restrict__ out,
                                 const double* __restrict__ q, int64_t N, int64_t nx, int64_t ny,
                                 int64_t nz, int axis, int forward, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  const int64_t n = nx * ny * nz;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int64_t stride = axis == 0 ? 1 : (axis == 1 ? nx : nx * ny);
  const int64_t o = (e / stride) % N;
  const int64_t base = e - o * stride;
  double s = 0.0;
  for (int64_t i = 0; i < N; ++i) {
    const double qv = forward ? q[i + N * o] : q[o + N * i];
    s = __dadd_rn(s, __dmul_rn(qv, in[base + i * stride]));
  }
  out[e] = s;
}

// Spectral division by λx+λy+λz with the constant mode removed (L† of the
// periodic Laplacian), then (after the inverse transform, separate launch)
// the KS potential.  Also accumulates the density scalars per block:
//   spart[b·3 + {0,1,2}] = {Σ V ρ, Σ ρ h, Σ ρ^{4/3}}.
__global__ void k_spectral_divide(double* __restrict__ a, const double* __restrict__ lx,
                                  const double* __restrict__ ly, const double* __restrict__ lz,
                                  int64_t nx, int64_t ny, int64_t nz, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  const int64_t n = nx * ny * nz;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t x = i % nx, y = (i / nx) % ny, z = i / (nx * ny);
  const double lam = __dadd_rn(__dadd_rn(lx[x], ly[y]), lz[z]);
  a[i] = (i == 0) ? 0.0 : __ddiv_rn(a[i], lam);
}

__global__ void k_ks_potential(const double* __restrict__ v, const double* __restrict__ rho,
                               const double* __restrict__ h, double* __restrict__ u, int64_t n,
                               double c /* (3/π)^{1/3} */, double* __restrict__ spart,
                               const Ctl* ctl, int64_t chunk = 0) {
  if (ctl && ctl->done) return;
  __shared__ double sm[kStreamThreadsOps / 32];
  double vr = 0.0, rh = 0.0, ex = 0.0;
  // chunk > 0: block b owns rows [b·chunk, (b+1)·chunk) (reproducible sharded
  // path); else a grid-stride loop
  const int64_t i0 = chunk ? (int64_t)blockIdx.x * chunk + threadIdx.x
                           : (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i1 = chunk ? min(n, (int64_t)(blockIdx.x + 1) * chunk) : n;
  const int64_t di = chunk ? (int64_t)blockDim.x : (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0; i < i1; i += di) {
    const double r = rho[i];
    const double cr = cbrt(r);
    vr += v[i] * r;
    rh += r * h[i];
    ex += r * cr;
    u[i] = __dsub_rn(__dadd_rn(v[i], h[i]), __dmul_rn(c, cr));
  }
  const double a = block_sum<kStreamThreadsOps>(vr, sm);
  const double b = block_sum<kStreamThreadsOps>(rh, sm);
  const double d = block_sum<kStreamThreadsOps>(ex, sm);
  if (threadIdx.x == 0) {
    spart[blockIdx.x * 3 + 0] = a;
    spart[blockIdx.x * 3 + 1] = b;
    spart[blockIdx.x * 3 + 2] = d;
  }
}

// h = L⁻¹ρ of the density models (DensityModel::evaluate, problems.cpp:170;
// LinearSolver::solve through the precomputed inverse): rows [0, n) of the
// slab m (ld ldm), all nk columns.  A block covers 32 rows with 8 column
// groups: a warp reads one 256-byte row segment per column, each thread sums
// its columns k ≡ g (mod 8) in order and the group sums are added in group
// order, so h is independent of the grid and of the row partition.
__global__ void __launch_bounds__(256) k_density_hartree(const double* __restrict__ m, int64_t ldm,
                                                         int64_t n, int64_t nk,
                                                         const double* __restrict__ rho,
                                                         double* __restrict__ h, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t i = (int64_t)blockIdx.x * 32 + lane;
  double s = 0.0;
  if (i < n) {
    const double* mi = m + i;
#pragma unroll 4
    for (int64_t k = g; k < nk; k += 8) s = fma(__ldg(mi + k * ldm), __ldg(rho + k), s);
  }
  part[g][lane] = s;
  __syncthreads();
  if (g == 0 && i < n) {
    double t = part[0][lane];
#pragma unroll
    for (int q = 1; q < 8; ++q) t += part[q][lane];
    h[i] = t;
  }
}

// The density term of DensityModel::evaluate (problems.cpp:179-203) on the
// owned rows, after G = L·X: P1 G += (coeff·h)∘X, P6 G += (2h − 2coeff·ρ^{1/3})∘X;
// block partials of ρᵀh and Σρ^{4/3} into spart[3b + 1], [3b + 2] (slot 0 = 0,
// the Kohn–Sham layout).  Non-finite G sets *bad (check_finite, problems.cpp:27-30).
// chunk > 0: block b owns rows [b·chunk, (b+1)·chunk) (reproducible sharded path).
__global__ void k_density_apply(const double* __restrict__ x, double* __restrict__ g, int64_t ld,
                                int64_t n, int64_t p, const double* __restrict__ rho,
                                const double* __restrict__ h, double coeff, int p6,
                                double* __restrict__ spart, int32_t* bad, const Ctl* ctl,
                                int64_t chunk = 0) {
  if (ctl && ctl->done) return;
  __shared__ double sm[kStreamThreadsOps / 32];
  double rh = 0.0, ex = 0.0;
  bool nonfinite = false;
  const int64_t i0 = chunk ? (int64_t)blockIdx.x * chunk + threadIdx.x
                           : (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i1 = chunk ? min(n, (int64_t)(blockIdx.x + 1) * chunk) : n;
  const int64_t di = chunk ? (int64_t)blockDim.x : (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0; i < i1; i += di) {
    const double r = rho[i], hi = h[i];
    double w;
    rh = __dadd_rn(rh, __dmul_rn(r, hi));
    if (p6) {
      const double cr = cbrt(r);
      ex = __dadd_rn(ex, __dmul_rn(r, cr));
      w = __dsub_rn(__dmul_rn(2.0, hi), __dmul_rn(__dmul_rn(2.0, coeff), cr));
    } else {
      w = __dmul_rn(coeff, hi);
    }
    for (int64_t j = 0; j < p; ++j) {
      const double v = __dadd_rn(g[i + j * ld], __dmul_rn(w, x[i + j * ld]));
      g[i + j * ld] = v;
      nonfinite |= !isfinite(v);
    }
  }
  if (nonfinite) *bad = 1;
  const double b = block_sum<kStreamThreadsOps>(rh, sm);
  const double d = block_sum<kStreamThreadsOps>(ex, sm);
  if (threadIdx.x == 0) {
    spart[blockIdx.x * 3 + 0] = 0.0;
    spart[blockIdx.x * 3 + 1] = b;
    spart[blockIdx.x * 3 + 2] = d;
  }
}

}  // namespace pcal
