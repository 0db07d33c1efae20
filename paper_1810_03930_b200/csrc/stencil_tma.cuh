// stencil_tma.cuh — the z-marching 7-point stencil of the grid models with its
// planes staged by the Tensor Memory Accelerator.
//
// A block owns an nx × TY tile of the xy-plane of one column j over a z-range.
// One producer warp streams, per plane z, the tile's TY rows plus the two
// periodic y-halo rows of X and the TY rows of the potential u into a ring of
// NS shared-memory slots (cp.async.bulk.tensor, mbarrier complete_tx); the TY
// consumer warps (one per row, lane l owning the XP consecutive points
// x = XP·l …) keep planes z−1, z, z+1 of their own points in registers, take
// the x-neighbours from warp shuffles and the y-neighbours from the slot, and
// write G with 16-byte vector stores.  No per-element global load is issued by
// the compute warps, so the kernel is limited by HBM, not by instruction issue
// (the register-pipelined k_stencil_march_row issues ≈3 loads per point).
// The arithmetic is k_stencil_march_row's, operand for operand: G is bitwise
// identical (round-to-nearest intrinsics, oracle order); the f partial sums
// its terms in a different fixed order.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace pcal {

// X as {nx, ny, nz, p} (row pitch nx, plane pitch nx·ny, column pitch ld);
// halo planes of a sharded slab as {nx, ny, p}; u as {nx, ny, nz}.  Two box
// shapes per tensor: the TY-row tile and a single halo row.
struct alignas(64) StencilMaps {
  CUtensorMap x_tile, x_row;    // box {nx, TY, 1, 1} / {nx, 1, 1, 1}
  CUtensorMap lo_tile, lo_row;  // plane −1 of the slab (sharded), box {nx, TY, 1} / {nx, 1, 1}
  CUtensorMap hi_tile, hi_row;  // plane nz
  CUtensorMap u_tile;           // box {nx, TY, 1}
  CUtensorMap p_tile, p_row;    // STEP: P_k as X (the fused normalised step)
};

// The fused normalised step (FUSE): the kernel reads X_k and P_k instead of
// X_{k+1} and forms every X_{k+1} value it uses as k_update_norm does,
// x⁺ = (x − (1/η)·(p − d_j·x))·(1/‖z_j‖) — one expression shared by both
// kernels, so X_{k+1} and G are bitwise the unfused path's — writing X_{k+1}
// of its own rows beside G: the step's write of X_{k+1} and the stencil's
// re-read of it become one pass (16np instead of 24np + 16np bytes).  Columns
// flagged for the exact two-pass rule (k_colscale) are skipped here and take
// k_update_norm → k_normalize → the plain stencil.
struct StepFuse {
  double* xplus;        // X_{k+1} (ld)
  const double* d;      // d_j of X_k
  const double* inv;    // 1/‖z_j‖
  const int32_t* fb;    // exact-rule flags (skipped columns)
  Ctl* ctl;             // η; step_bad / done on a non-finite X_{k+1}
};

template <bool KS, int XP, int TY, int NS, bool FUSE = false>
__global__ void __launch_bounds__(32 * (TY + 1))
    k_stencil_tma(const __grid_constant__ StencilMaps maps, double* __restrict__ g, int nx, int ny,
                  int nz, int64_t ld, int zchunk, double* __restrict__ fpart, int64_t pstride,
                  int32_t* bad, const Ctl* ctl, int sharded, int zpart, int zmode,
                  const int32_t* only_fb, StepFuse sf) {
  static_assert(XP % 2 == 0, "full-row march: XP even (16-byte vectors)");
  constexpr int V = XP / 2;
  if (ctl && ctl->done) return;
  const int j = blockIdx.z;
  if (only_fb && !only_fb[j]) return;  // the fused step already produced this column
  if (FUSE && sf.fb[j]) return;        // exact-rule column: the unfused path
  extern __shared__ __align__(128) double st_smem[];
  const int W = nx;                              // doubles per row
  const int XT = (TY + 2) * W, UT = TY * W;      // slot sizes (doubles)
  double* xs = st_smem;                          // [NS][TY + 2][nx]
  double* us = xs + NS * XT;                     // [NS][TY][nx]
  double* ps = us + NS * UT;                     // FUSE: [NS][TY + 2][nx] of P_k
  uint64_t* full = reinterpret_cast<uint64_t*>(FUSE ? ps + NS * XT : us + NS * UT);
  uint64_t* empty = full + NS;
  __shared__ double sm[TY];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int y0 = blockIdx.x * TY;
  // zmode 0: z-chunks of the whole slab; 1: the interior planes [zpart, nz − zpart)
  // (no halo plane read — they run while the halo exchange is in flight);
  // 2: the two boundary row chunks [0, zpart) and [nz − zpart, nz).  Chunks
  // start on multiples of zpart, so every f partial (zpart planes) is summed
  // inside one CTA exactly as in mode 0.
  int z0, z1;
  if (zmode == 0) {
    z0 = blockIdx.y * zchunk;
    z1 = min(nz, z0 + zchunk);
  } else if (zmode == 1) {
    z0 = zpart + blockIdx.y * zchunk;
    z1 = min(nz - zpart, z0 + zchunk);
  } else {
    z0 = blockIdx.y ? nz - zpart : 0;
    z1 = z0 + zpart;
  }
  const int nplanes = z1 - z0 + 2;  // planes z0 − 1 … z1
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(&full[i])) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(
                       (unsigned)__cvta_generic_to_shared(&empty[i])),
                   "r"(TY) : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto bar_addr = [](uint64_t* b) { return (unsigned)__cvta_generic_to_shared(b); };
  auto wait = [&](uint64_t* b, unsigned par) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" ::"r"(bar_addr(b)),
        "r"(par)
        : "memory");  // the slot's shared-memory reads must not move above the wait
  };
  if (warp == TY) {  // ---- producer: one lane drives the TMA unit
    if (lane != 0) return;
    const int yl = y0 == 0 ? ny - 1 : y0 - 1, yh = y0 + TY == ny ? 0 : y0 + TY;
    const unsigned bytes = (unsigned)((XT + UT + (FUSE ? XT : 0)) * 8);
    for (int i = 0; i < nplanes; ++i) {
      const int s = i % NS;
      wait(&empty[s], ((unsigned)(i / NS) & 1u) ^ 1u);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                       bar_addr(&full[s])),
                   "r"(bytes)
                   : "memory");
      const int z = z0 - 1 + i;
      double* xd = xs + s * XT;
      double* ud = us + s * UT;
      const unsigned fb = bar_addr(&full[s]);
      auto ld4 = [&](double* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3) {
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(fb)
            : "memory");
      };
      auto ld3 = [&](double* dst, const CUtensorMap* m, int c0, int c1, int c2) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
            "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(c2), "r"(fb)
            : "memory");
      };
      if (sharded && z < 0) {          // the lower neighbour's boundary plane
        ld3(xd + W, &maps.lo_tile, 0, y0, j);
        ld3(xd, &maps.lo_row, 0, yl, j);
        ld3(xd + (TY + 1) * W, &maps.lo_row, 0, yh, j);
      } else if (sharded && z >= nz) {  // the upper neighbour's boundary plane
        ld3(xd + W, &maps.hi_tile, 0, y0, j);
        ld3(xd, &maps.hi_row, 0, yl, j);
        ld3(xd + (TY + 1) * W, &maps.hi_row, 0, yh, j);
      } else {
        const int zz = z < 0 ? z + nz : (z >= nz ? z - nz : z);  // periodic wrap
        ld4(xd + W, &maps.x_tile, 0, y0, zz, j);
        ld4(xd, &maps.x_row, 0, yl, zz, j);
        ld4(xd + (TY + 1) * W, &maps.x_row, 0, yh, zz, j);
        if (FUSE) {
          double* pd = ps + s * XT;
          ld4(pd + W, &maps.p_tile, 0, y0, zz, j);
          ld4(pd, &maps.p_row, 0, yl, zz, j);
          ld4(pd + (TY + 1) * W, &maps.p_row, 0, yh, zz, j);
        }
      }
      // u of plane z (needed for z0 … z1−1; the two end planes load a valid
      // plane so every slot carries the same byte count)
      const int zu = z < 0 ? 0 : (z >= nz ? nz - 1 : z);
      ld3(ud, &maps.u_tile, 0, y0, zu);
    }
    return;
  }
  // ---- consumers: warp ty = row y0 + ty
  const int ty = warp;
  const int L = nx / XP;
  const int ln = lane < L ? lane : L - 1;
  const bool act = lane < L;
  const int y = y0 + ty;
  const int64_t nxy = (int64_t)nx * ny;
  double* gj = g + (int64_t)j * ld;
  // FUSE: the step's scalars of column j
  double f_ie = 0.0, f_dj = 0.0, f_sc = 1.0;
  if (FUSE) {
    f_ie = 1.0 / sf.ctl->eta;
    f_dj = sf.d[j];
    f_sc = sf.inv[j];
  }
  // X values of a slot (FUSE: X_{k+1} formed from the X_k and P_k slots)
  auto rd = [&](const double* p, double (&d)[XP]) {
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double2 t = reinterpret_cast<const double2*>(p)[v];
      if (FUSE) {
        const double2 q = reinterpret_cast<const double2*>(p + (ps - xs))[v];
        d[2 * v] = step_value(t.x, q.x, f_dj, f_ie, f_sc);
        d[2 * v + 1] = step_value(t.y, q.y, f_dj, f_ie, f_sc);
      } else {
        d[2 * v] = t.x;
        d[2 * v + 1] = t.y;
      }
    }
  };
  auto rdu = [&](const double* p, double (&d)[XP]) {  // potential (never transformed)
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const double2 t = reinterpret_cast<const double2*>(p)[v];
      d[2 * v] = t.x;
      d[2 * v + 1] = t.y;
    }
  };
  const int own = (ty + 1) * W + XP * ln;  // this lane's points in an X slot
  const int lsrc = ln == 0 ? L - 1 : ln - 1, rsrc = ln == L - 1 ? 0 : ln + 1;
  double below[XP], cur[XP], above[XP];
  // A slot is released only after the values read from it have been consumed
  // by the plane's arithmetic and stored: mbarrier.arrive does not wait for
  // this warp's outstanding shared-memory loads, and a release straight after
  // the loads let the producer's next TMA fill of the slot overtake them
  // (observed: plane z0+3 read as plane z0−1 in a few rows at config 5).
  wait(&full[0], 0u);
  rd(xs + own, below);
  wait(&full[1 % NS], (unsigned)(1 / NS) & 1u);
  rd(xs + (1 % NS) * XT + own, cur);
  double acc = 0.0;
  bool nonfinite = false, xbad = false;
  int zp_cnt = z0 % zpart, zp_idx = z0 / zpart;
  for (int z = z0; z < z1; ++z) {
    const int ic = z - z0 + 1, ia = ic + 1;  // slots of planes z and z + 1
    const int sc = ic % NS, sa = ia % NS;
    wait(&full[sa], (unsigned)(ia / NS) & 1u);
    rd(xs + sa * XT + own, above);
    const double* xc = xs + sc * XT;
    double dn[XP], up[XP], uc[XP];
    rd(xc + ty * W + XP * ln, dn);
    rd(xc + (ty + 2) * W + XP * ln, up);
    rdu(us + sc * UT + ty * W + XP * ln, uc);
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
      double2* gout = reinterpret_cast<double2*>(gj + (int64_t)z * nxy + (int64_t)y * nx + XP * ln);
#pragma unroll
      for (int v = 0; v < V; ++v) gout[v] = make_double2(gv[2 * v], gv[2 * v + 1]);
      if (FUSE) {  // X_{k+1} of the own points (k_update_norm's store)
        double2* xout = reinterpret_cast<double2*>(sf.xplus + (int64_t)j * ld + (int64_t)z * nxy +
                                                   (int64_t)y * nx + XP * ln);
#pragma unroll
        for (int v = 0; v < V; ++v) {
          xout[v] = make_double2(cur[2 * v], cur[2 * v + 1]);
          xbad |= !isfinite(cur[2 * v]) || !isfinite(cur[2 * v + 1]);
        }
      }
    }
    // every lane has consumed what it read from slot sc (plane z) — and, at the
    // first plane, from slot 0 (plane z0 − 1): the stores above depend on it
    __syncwarp();
    if (lane == 0) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar_addr(&empty[sc])) : "memory");
      if (z == z0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar_addr(&empty[0])) : "memory");
    }
#pragma unroll
    for (int k = 0; k < XP; ++k) {
      below[k] = cur[k];
      cur[k] = above[k];
    }
    if (++zp_cnt == zpart || z + 1 == z1) {  // one f partial per (tile, zpart planes)
      if (!KS) nonfinite |= !isfinite(acc);
      const double v = warp_sum(acc);
      if (lane == 0) sm[ty] = v;
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * TY) : "memory");
      if (lane == 0 && ty == 0) {
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < TY; ++t) s += sm[t];
        fpart[(int64_t)j * pstride + blockIdx.x + (int64_t)gridDim.x * zp_idx] = s;
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(32 * TY) : "memory");
      acc = 0.0;
      if (zp_cnt == zpart) {
        zp_cnt = 0;
        ++zp_idx;
      }
    }
  }
  {  // the last plane (z1) was only read as `above`: release its slot
    const int il = z1 - z0 + 1;
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar_addr(&empty[il % NS])) : "memory");
  }
  if (__any_sync(0xffffffffu, nonfinite) && lane == 0) *bad = 1;
  if (FUSE && __any_sync(0xffffffffu, xbad) && lane == 0) {  // k_update_norm's divergence rule
    sf.ctl->step_bad = 1;
    sf.ctl->done = 2;
  }
}

}  // namespace pcal
