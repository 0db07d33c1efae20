// gemm_dmma.cuh — FP64 tensor-core GEMM for sm_100a with stream-K scheduling
// and fused PCAL epilogues.
//
// Blackwell has no FP64 tcgen05 kind (ptxas rejects kind::f64),
// so FP64 tensor math is the warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4,
// measured 37.1 TFLOP/s peak on B200: profiles/fp64_peaks_r01.txt).  Tiles are
// staged global→shared by the Tensor Memory Accelerator (cp.async.bulk.tensor,
// 128-byte swizzled boxes, mbarrier complete_tx) into a STAGES-deep ring that
// ONE producer thread keeps full; the schedule is stream-K: the linearised (tile, k-iteration) space is cut into
// `grid` equal contiguous ranges, one per CTA (grid = SM count), so the
// tall-skinny contractions of PCAL (K = n up to 2M, M·N = p×p) and the dense
// gradient (M = n, N = p, K = n) both fill all 148 SMs.  A tile completed by
// one CTA gets its epilogue in-kernel; a tile shared by several CTAs has its
// partial accumulators written to a workspace and summed in a FIXED order
// (CTA order) by gemm_fixup — results never depend on timing, and the
// direct and fixup paths run the same epilogue code.
//
// Operands (FP64, column-major device buffers):
//   A_MCONTIG: A(m,k) = A[m + k·lda]     (dense operator A; X in X·M)
//   A_KCONTIG: A(m,k) = A[k + m·lda]     (Xᵀ / [G|X]ᵀ in the Grams)
//   B        : B(k,n) = B[k + n·ldb]     (X, Y, or the p×2p multiplier block)
#pragma once

#include <cuda.h>  // CUtensorMap

#include "gemm_types.h"

namespace pcal {

template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int STAGES_, int AMODE_, int BK_ = 16>
struct GemmCfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_;
  static constexpr int WARPS_M = WARPS_M_, WARPS_N = WARPS_N_;
  static constexpr int WARPS = WARPS_M * WARPS_N, THREADS = WARPS * 32;
  static constexpr int STAGES = STAGES_;
  static constexpr int AMODE = AMODE_;
  static constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;  // warp tile
  static constexpr int MT = WM / 8, NT = WN / 8;              // 8×8 mma tiles per warp
  static constexpr int FRAG = MT * NT * 2;                    // accumulators per thread
  // Shared layouts (TMA boxes, SWIZZLE_128B: 128-byte rows, the 16-byte chunk
  // c of row R stored at chunk c ^ (R mod 8), every box 1024-byte aligned):
  //   A_MCONTIG: BM/16 boxes {16 m, BK k}: rows = k, 16 consecutive m per row
  //   A_KCONTIG and B: BK/16 boxes {16 k, BM or BN rows}: rows = m (n), 16 k per row
  static constexpr int A_STAGE = BM * BK;   // doubles per stage
  static constexpr int B_STAGE = BN * BK;
  static constexpr int STAGE_BYTES = (A_STAGE + B_STAGE) * 8;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 1024;  // + align slack
  static_assert(WM % 16 == 0 && WN % 8 == 0, "warp tile: WM multiple of 16, WN of 8");
  static_assert(BK % 16 == 0 && BM % 16 == 0, "TMA boxes are 16 doubles wide");
};

// Tensor maps of one launch (encoded on the host per launch, gemm.cu; kernel
// parameter, so graph capture keeps the pointers of the captured launch).
struct alignas(64) GemmMaps {
  CUtensorMap a;  // A_MCONTIG: {M, K} box {16, BK};  A_KCONTIG: {K, M} box {16, BM}
  CUtensorMap b;  // {K, N} box {16, BN}
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// Same with an L2 cache policy: the streamed dense operator is marked
// evict-first so it does not push the reused X out of L2.
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// predicated DMMA (a warp-uniform predicate, no branch)
__device__ __forceinline__ void dmma_8x8x4_if(bool on, double& c0, double& c1, double a, double b) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "@p mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n}\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b), "r"((int)on));
}

// k-slice order inside one 16-k box.  DMMA.8x8x4 lane (r, q) holds A(m = r, k_q)
// and B(k_q, n = r); which four k of the slice form k-step s is free as long as
// A and B agree.  Step s of a box uses k = kq(q) ^ t(s) with kq = {0, 3, 12, 15}
// and t = {0, 1, 4, 5}: the four sets partition 0..15, and under the 128-byte
// swizzle each 16-lane half of a fragment load hits 16 distinct bank pairs
//   * A_MCONTIG (rows = k): k mod 8 of the four q differ in bits 1–2, so the
//     four rows' 32-byte segments land in four different chunk pairs;
//   * rows = m / n (A_KCONTIG, B): two q per 8-byte half-chunk (k & 1), and
//     within a half their chunks k >> 1 differ in bit 2, so rows r = 0..3
//     (XOR r) never collide.
__device__ __forceinline__ int kq_of(int q) { return (q & 1) * 3 + (q >> 1) * 12; }
// ---- one BK slice of MMAs (swizzled TMA layout, permuted k order) ------------
template <class Cfg>
__device__ __forceinline__ void mma_stage(const char* As, const char* Bs, int wm, int wn, int lane,
                                          double (&acc)[Cfg::MT][Cfg::NT][2]) {
  const int r = lane >> 2, q = lane & 3;
  const int kq = kq_of(q);
#pragma unroll
  for (int st = 0; st < Cfg::BK / 4; ++st) {
    const int box = st >> 2;
    const int kl = kq ^ ((st & 1) | ((st & 2) << 1));  // k within the box: kq ^ {0,1,4,5}
    double a[Cfg::MT], b[Cfg::NT];
    if constexpr (Cfg::AMODE == A_MCONTIG) {
      // element (m, k): box m/16, row k, chunk ((m & 15) >> 1) ^ (k & 7), half m & 1
      const int k = box * 16 + kl;
      const char* rowp = As + k * 128 + (r & 1) * 8;
      const int ce = ((r >> 1) ^ (k & 7)) << 4;   // even mt (m & 15 < 8)
      const int co = ce ^ 64;                      // odd mt: chunk ^ 4
#pragma unroll
      for (int mt = 0; mt < Cfg::MT; ++mt) {
        const int mb = (wm * Cfg::WM + mt * 8) >> 4;
        a[mt] = *reinterpret_cast<const double*>(rowp + mb * (Cfg::BK * 128) + ((mt & 1) ? co : ce));
      }
    } else {
      // element (m, k): box k/16, row m, chunk ((k & 15) >> 1) ^ (m & 7), half k & 1
      const char* bx = As + box * (Cfg::BM * 128) + (kl & 1) * 8 + ((((kl >> 1) ^ r)) << 4);
#pragma unroll
      for (int mt = 0; mt < Cfg::MT; ++mt) {
        const int m = wm * Cfg::WM + mt * 8 + r;
        a[mt] = *reinterpret_cast<const double*>(bx + m * 128);
      }
    }
    {
      const char* bx = Bs + box * (Cfg::BN * 128) + (kl & 1) * 8 + ((((kl >> 1) ^ r)) << 4);
#pragma unroll
      for (int nt = 0; nt < Cfg::NT; ++nt) {
        const int n = wn * Cfg::WN + nt * 8 + r;
        b[nt] = *reinterpret_cast<const double*>(bx + n * 128);
      }
    }
#pragma unroll
    for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < Cfg::NT; ++nt) dmma_8x8x4(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
  }
}

// ---- diagonal tiles of a symmetric Gram: only the upper triangle -------------
// A 128 × 128 tile on the diagonal of a block whose upper triangle is all that
// is needed (XᵀX; GᵀX of a symmetric operator) holds 136 of its 256 8×8
// sub-blocks at or above the diagonal.  Warp w computes sub-block rows w and
// 15 − w from the diagonal to the right edge — 16 − w and w + 1 sub-blocks,
// 17 DMMAs per k-step for every warp (warps w and w + 4 share an SM
// sub-partition: 34 each, balanced) instead of 32: the tile costs 136/256 of a
// full one.  Sub-block (R, C) accumulates in acc[c/4 (+4 for row 15 − w)][c % 4],
// the registers of the full tile, and is stored in the full tile's fragment
// layout (frag_index of its owner in the full schedule), so partial tiles go
// through the same fixup / tree reductions.  Same k order as mma_stage: the
// computed elements are bitwise those of the full tile.
#ifndef PCAL_TRI_UNROLL
#define PCAL_TRI_UNROLL 2
#endif
constexpr int kTriUnroll = PCAL_TRI_UNROLL;
template <class Cfg, int W>
__device__ __forceinline__ void mma_stage_tri_w(const char* As, const char* Bs, int lane,
                                                double (&acc)[Cfg::MT][Cfg::NT][2]) {
  static_assert(Cfg::AMODE == A_KCONTIG && Cfg::BM == 128 && Cfg::BN == 128 && Cfg::MT == 8 &&
                    Cfg::NT == 4 && Cfg::WARPS == 8,
                "triangular tiles: the 128 × 128 K-contiguous Gram configuration");
  constexpr int R1 = W, R2 = 15 - W;
  const int r = lane >> 2, q = lane & 3;
  const int kq = kq_of(q);
  // partially unrolled: eight specialised warp bodies fully unrolled over the
  // k-steps overflow the instruction cache (stall_no_inst at config 3)
#pragma unroll kTriUnroll
  for (int st = 0; st < Cfg::BK / 4; ++st) {
    const int box = st >> 2;
    const int kl = kq ^ ((st & 1) | ((st & 2) << 1));
    const int sw = (kl & 1) * 8 + (((kl >> 1) ^ r) << 4);
    const char* ax = As + box * (Cfg::BM * 128) + sw;
    const char* bx = Bs + box * (Cfg::BN * 128) + sw;
    const double a1 = *reinterpret_cast<const double*>(ax + (R1 * 8 + r) * 128);
    const double a2 = *reinterpret_cast<const double*>(ax + (R2 * 8 + r) * 128);
    double b[16 - R1];
#pragma unroll
    for (int c = R1; c < 16; ++c)
      b[c - R1] = *reinterpret_cast<const double*>(bx + (c * 8 + r) * 128);
#pragma unroll
    for (int c = R1; c < 16; ++c) {
      dmma_8x8x4(acc[c >> 2][c & 3][0], acc[c >> 2][c & 3][1], a1, b[c - R1]);
      if constexpr (true) {
        if (c >= R2)  // compile-time after unrolling
          dmma_8x8x4(acc[4 + (c >> 2)][c & 3][0], acc[4 + (c >> 2)][c & 3][1], a2, b[c - R1]);
      }
    }
  }
}

// Warp w of a triangular tile: sub-block rows w and 15 − w (exactly 17 DMMAs
// and 18 − w fragment loads per k-step: one code path per warp, no predication).
template <class Cfg>
__device__ __forceinline__ void mma_stage_tri(const char* As, const char* Bs, int warp, int lane,
                                              double (&acc)[Cfg::MT][Cfg::NT][2]) {
  switch (warp) {
    case 0: mma_stage_tri_w<Cfg, 0>(As, Bs, lane, acc); break;
    case 1: mma_stage_tri_w<Cfg, 1>(As, Bs, lane, acc); break;
    case 2: mma_stage_tri_w<Cfg, 2>(As, Bs, lane, acc); break;
    case 3: mma_stage_tri_w<Cfg, 3>(As, Bs, lane, acc); break;
    case 4: mma_stage_tri_w<Cfg, 4>(As, Bs, lane, acc); break;
    case 5: mma_stage_tri_w<Cfg, 5>(As, Bs, lane, acc); break;
    case 6: mma_stage_tri_w<Cfg, 6>(As, Bs, lane, acc); break;
    default: mma_stage_tri_w<Cfg, 7>(As, Bs, lane, acc); break;
  }
}

// ---- epilogues ---------------------------------------------------------------
// Fragment (mt, nt, e) of lane `lane` in warp (wm, wn) is output element
//   row = m0 + wm·WM + mt·8 + lane/4,   col = n0 + wn·WN + nt·8 + 2·(lane%4) + e.
// Column partial sums are reduced over the warp's WM rows (fixed shuffle
// order) and stored per row-block rb = (m0 + wm·WM)/WM.
template <class Cfg, int EPI>
__device__ __forceinline__ void epilogue(const GemmArgs& g, int tm, int tn, int wm, int wn,
                                         int lane, double (&acc)[Cfg::MT][Cfg::NT][2]) {
  const EpiParams& e = g.ep;
  const int r = lane >> 2, q = lane & 3;
  const int64_t mw0 = (int64_t)tm * Cfg::BM + wm * Cfg::WM;
  const int64_t nw0 = (int64_t)tn * Cfg::BN + wn * Cfg::WN;
  if constexpr (EPI == EPI_STORE) {
#pragma unroll
    for (int mt = 0; mt < Cfg::MT; ++mt) {
      const int64_t row = mw0 + mt * 8 + r;
#pragma unroll
      for (int nt = 0; nt < Cfg::NT; ++nt)
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const int64_t col = nw0 + nt * 8 + 2 * q + x;
          if (row < e.m_store && col < e.n_store) e.C[row + col * e.ldc] = acc[mt][nt][x];
        }
    }
  } else if constexpr (EPI == EPI_GRAD) {
    const int64_t rb = mw0 / Cfg::WM;
    const bool interior = (mw0 + Cfg::WM <= e.n) && (nw0 + Cfg::WN <= e.p) && !e.g0;
    bool bad = false;
#pragma unroll
    for (int nt = 0; nt < Cfg::NT; ++nt) {
      double xv[2][Cfg::MT];
      if (interior) {  // batch the X loads of this column pair
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int mt = 0; mt < Cfg::MT; ++mt)
            xv[x][mt] = e.X[mw0 + mt * 8 + r + (nw0 + nt * 8 + 2 * q + x) * e.ld];
      }
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int64_t col = nw0 + nt * 8 + 2 * q + x;
        double fs = 0.0;
#pragma unroll
        for (int mt = 0; mt < Cfg::MT; ++mt) {
          const int64_t row = mw0 + mt * 8 + r;
          if (interior) {
            const double gv = acc[mt][nt][x];
            e.G[row + col * e.ld] = gv;
            fs += xv[x][mt] * gv;
            bad |= !isfinite(gv);
          } else if (row < e.n && col < e.p) {
            double gv = acc[mt][nt][x];
            double fv = gv;  // f = ½⟨X, AX + 2·G0⟩ = ½⟨X,AX⟩ + ⟨G0,X⟩
            if (e.g0) {
              const double g0v = e.g0[row + col * e.ld];
              gv += g0v;
              fv = gv + g0v;
            }
            e.G[row + col * e.ld] = gv;
            fs += e.X[row + col * e.ld] * fv;
            bad |= !isfinite(gv);
          }
        }
        fs += __shfl_xor_sync(0xffffffffu, fs, 4);
        fs += __shfl_xor_sync(0xffffffffu, fs, 8);
        fs += __shfl_xor_sync(0xffffffffu, fs, 16);
        if (r == 0 && col < e.p) e.fpart[col * e.pstride + rb] = fs;
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) *e.bad = 1;
  } else {  // EPI_XM
    const int64_t rb = mw0 / Cfg::WM;
    // interior warp tiles: issue every G/X load of a batch of NB column groups
    // before any use (one memory round trip per batch instead of one per element)
    const bool interior = (mw0 + Cfg::WM <= e.n) && (((nw0 + Cfg::WN) >> 1) <= e.p);
    constexpr int NB = Cfg::NT >= 2 ? 2 : 1;
#pragma unroll
    for (int nb0 = 0; nb0 < Cfg::NT; nb0 += NB) {
      double gv[NB][Cfg::MT], xv[NB][Cfg::MT];
      if (interior) {
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          const int64_t j = (nw0 + (nb0 + b) * 8 + 2 * q) >> 1;
#pragma unroll
          for (int mt = 0; mt < Cfg::MT; ++mt) {
            const int64_t idx = mw0 + mt * 8 + r + j * e.ld;
            gv[b][mt] = e.G[idx];
            xv[b][mt] = e.X[idx];
          }
        }
      }
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int nt = nb0 + b;
        const int64_t j = (nw0 + nt * 8 + 2 * q) >> 1;  // output column
        double ks = 0.0, ds = 0.0;
#pragma unroll
        for (int mt = 0; mt < Cfg::MT; ++mt) {
          const int64_t row = mw0 + mt * 8 + r;
          const int64_t idx = row + j * e.ld;
          if (interior) {
            const double kkt = gv[b][mt] - acc[mt][nt][0];
            const double pv = (e.p_from_g ? gv[b][mt] : kkt) + e.beta * acc[mt][nt][1];
            e.G[idx] = pv;
            ks += kkt * kkt;
            ds += (e.d_sq ? pv : xv[b][mt]) * pv;
          } else if (row < e.n && j < e.p) {
            const double g0 = e.G[idx];
            const double kkt = g0 - acc[mt][nt][0];
            const double pv = (e.p_from_g ? g0 : kkt) + e.beta * acc[mt][nt][1];
            e.G[idx] = pv;
            ks += kkt * kkt;
            ds += (e.d_sq ? pv : e.X[idx]) * pv;
          }
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          ks += __shfl_xor_sync(0xffffffffu, ks, o);
          ds += __shfl_xor_sync(0xffffffffu, ds, o);
        }
        if (r == 0 && j < e.p) {
          e.kpart[j * e.pstride + rb] = ks;
          e.dpart[j * e.pstride + rb] = ds;
        }
      }
    }
  }
}

template <class Cfg>
__device__ __forceinline__ size_t frag_index(int warp, int mt, int nt, int x, int lane) {
  return ((((size_t)warp * Cfg::MT + mt) * Cfg::NT + nt) * 2 + x) * 32 + lane;
}

// ---- mbarrier helpers ------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");  // shared-memory reads of the stage must not move above the wait
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// ---- producer: ONE thread streams the CTA's unit range into the smem ring.
// Per stage it waits for the consumers to free the slot, announces the stage's
// bytes on the slot's `full` barrier and issues the TMA box loads (A: BM/16
// or BK/16 boxes, B: BK/16 boxes); the TMA unit completes the transaction
// count, zero-filling every element outside the logical extents (edge tiles).
constexpr int kProducerRegs = 40;  // per producer thread after setmaxnreg
template <class Cfg>
__device__ __forceinline__ void produce_tma(const GemmArgs& g, const GemmMaps& maps, char* As,
                                            char* Bs, uint64_t* full, uint64_t* empty, int64_t u0,
                                            int64_t u1) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, S = Cfg::STAGES;
  const bool a_stream = Cfg::AMODE == A_MCONTIG && g.a_stream;
  const uint64_t pol = a_stream ? l2_evict_first_policy() : 0;
  int t = (int)(u0 / g.ki), kk = (int)(u0 % g.ki);
  int2 tc = g.tiles[t];
  int s = 0;
  unsigned ph = 0;
  for (int64_t u = u0; u < u1; ++u) {
    mbar_wait(&empty[s], ph ^ 1u);
    mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
    char* as = As + s * (Cfg::A_STAGE * 8);
    char* bs = Bs + s * (Cfg::B_STAGE * 8);
    const int m0 = tc.x * BM, n0 = tc.y * BN, k0 = kk * BK;
    if constexpr (Cfg::AMODE == A_MCONTIG) {
#pragma unroll
      for (int mb = 0; mb < BM / 16; ++mb) {
        if (a_stream)
          tma_load_2d_hint(as + mb * (BK * 128), &maps.a, m0 + 16 * mb, k0, &full[s], pol);
        else
          tma_load_2d(as + mb * (BK * 128), &maps.a, m0 + 16 * mb, k0, &full[s]);
      }
    } else {
#pragma unroll
      for (int kh = 0; kh < BK / 16; ++kh)
        tma_load_2d(as + kh * (BM * 128), &maps.a, k0 + 16 * kh, m0, &full[s]);
    }
#pragma unroll
    for (int kh = 0; kh < BK / 16; ++kh)
      tma_load_2d(bs + kh * (BN * 128), &maps.b, k0 + 16 * kh, n0, &full[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
    if (++kk == g.ki) {
      kk = 0;
      if (u + 1 < u1) tc = g.tiles[++t];
    }
  }
}

// Smem carve-up shared by both kernels: 1024-byte aligned ring, then barriers.
// (offset arithmetic on the __shared__ array itself, so the compiler keeps the
// shared address space: LDS with 32-bit addresses, not generic loads)
template <class Cfg>
__device__ __forceinline__ char* smem_ring(char* raw) {
  return raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
}

// Store the upper-triangle sub-blocks of a triangular tile (mma_stage_tri):
// straight into C (whole tile) or into the partial slot w in the full tile's
// fragment layout.
template <class Cfg>
__device__ __forceinline__ void flush_tri(const GemmArgs& g, int2 tc, bool whole, double* w,
                                          int warp, int lane,
                                          const double (&acc)[Cfg::MT][Cfg::NT][2]) {
  const int r = lane >> 2, q = lane & 3;
  const EpiParams& e = g.ep;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int R = h == 0 ? warp : 15 - warp;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      if (c < R) continue;
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const double v = acc[4 * h + (c >> 2)][c & 3][x];
        if (whole) {
          const int64_t row = (int64_t)tc.x * Cfg::BM + R * 8 + r;
          const int64_t col = (int64_t)tc.y * Cfg::BN + c * 8 + 2 * q + x;
          if (row < e.m_store && col < e.n_store) e.C[row + col * e.ldc] = v;
        } else {
          const int owner = (R >> 3) * Cfg::WARPS_N + (c >> 2);  // full-schedule warp of (R, c)
          w[frag_index<Cfg>(owner, R & 7, c & 3, x, lane)] = v;
        }
      }
    }
  }
}

// ---- main kernel ----------------------------------------------------------------
// Warp-specialized: warps [0, WARPS) consume (LDS + DMMA + epilogue), warp
// WARPS produces (cp.async ring, one mbarrier pair per stage); the rest of
// the producer warpgroup only donates its registers.
template <class Cfg, int EPI>
__global__ void __launch_bounds__(Cfg::THREADS + 128, 1)
    gemm_streamk(GemmArgs g, const __grid_constant__ GemmMaps maps) {
  if (g.ctl && g.ctl->done) return;
  if (g.gate && !*g.gate) return;
  extern __shared__ __align__(1024) char smem_raw[];
  char* As = smem_ring<Cfg>(smem_raw);
  char* Bs = As + Cfg::STAGES * Cfg::A_STAGE * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + Cfg::STAGES * Cfg::B_STAGE * 8);
  uint64_t* empty = full + Cfg::STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t cta = blockIdx.x;
  // explicit (weighted) CTA ranges first: whole segments in segmented mode
  const int64_t u0 = g.cta_begin ? g.cta_begin[cta]
                     : g.segs    ? seg_unit_begin(cta, g.ntiles, g.ki, g.segs, g.grid)
                                 : cta_unit_begin(cta, g.units, g.grid, g.upc);
  const int64_t u1 = g.cta_begin ? g.cta_begin[cta + 1]
                     : g.segs    ? seg_unit_begin(cta + 1, g.ntiles, g.ki, g.segs, g.grid)
                                 : cta_unit_begin(cta + 1, g.units, g.grid, g.upc);
  if (u0 >= u1) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // The producer owns a whole warpgroup (setmaxnreg is warpgroup-collective):
  // with 8 consumer warps, consumers take 232 registers and the producer
  // group kProducerRegs = 40 (8·32·232 + 4·32·40 ≤ 64K).
  if (warp >= Cfg::WARPS) {
    if constexpr (Cfg::WARPS >= 8) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
    if (warp == Cfg::WARPS && lane == 0) produce_tma<Cfg>(g, maps, As, Bs, full, empty, u0, u1);
    return;
  }
  if constexpr (Cfg::WARPS >= 8) {
    // (64K − 128·40) / consumer threads, rounded down to a multiple of 8, ≤ 232
    constexpr int R = (65536 - 128 * kProducerRegs) / Cfg::THREADS / 8 * 8 > 232
                          ? 232
                          : (65536 - 128 * kProducerRegs) / Cfg::THREADS / 8 * 8;
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(R));
  }
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;

  double acc[Cfg::MT][Cfg::NT][2];
#pragma unroll
  for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < Cfg::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

  // tile / k-iteration / segment counters advance incrementally (no 64-bit
  // divisions on the DMMA issue path)
  int t = (int)(u0 / g.ki);
  int kk = (int)(u0 % g.ki);
  const int S = g.segs;
  int cur_seg = S > 1 ? seg_of(kk, g.ki, S) : 0;
  int seg_stop = S > 1 ? (int)((int64_t)(cur_seg + 1) * g.ki / S) : g.ki;  // exclusive, in kk
  bool tile_start = kk == 0;  // this CTA's current tile segment began at the tile's k = 0
  int stage = 0;
  unsigned phase = 0;
  constexpr bool kTriCfg = Cfg::AMODE == A_KCONTIG && EPI == EPI_STORE && Cfg::BM == 128 &&
                           Cfg::BN == 128 && Cfg::WARPS == 8;
  bool tri = kTriCfg && g.tile_tri && g.tile_tri[t];
  for (int64_t u = u0; u < u1; ++u) {
    mbar_wait(&full[stage], phase);
    if constexpr (kTriCfg) {
      if (tri)
        mma_stage_tri<Cfg>(As + stage * (Cfg::A_STAGE * 8), Bs + stage * (Cfg::B_STAGE * 8), warp,
                           lane, acc);
      else
        mma_stage<Cfg>(As + stage * (Cfg::A_STAGE * 8), Bs + stage * (Cfg::B_STAGE * 8), wm, wn,
                       lane, acc);
    } else {
      mma_stage<Cfg>(As + stage * (Cfg::A_STAGE * 8), Bs + stage * (Cfg::B_STAGE * 8), wm, wn,
                     lane, acc);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == Cfg::STAGES) {
      stage = 0;
      phase ^= 1u;
    }

    const bool tile_end = kk == g.ki - 1;
    const bool seg_end = kk + 1 == seg_stop;  // == tile_end without segments
    if (tile_end || seg_end || u == u1 - 1) {
      const int2 tc = g.tiles[t];
      const bool whole = tile_start && tile_end && !g.force_ws && S <= 1;
      if (kTriCfg && tri) {
        flush_tri<Cfg>(g, tc, whole, whole ? nullptr
                       : g.ws + ((size_t)g.split_slot[t] * g.qmax +
                                 (S ? cur_seg
                                    : cta - (g.tile_cta0 ? g.tile_cta0[t]
                                                         : cta_of_unit((int64_t)t * g.ki, g.units,
                                                                       g.grid)))) *
                                    (size_t)(Cfg::BM * Cfg::BN),
                       warp, lane, acc);
      } else if (whole) {
        epilogue<Cfg, EPI>(g, tc.x, tc.y, wm, wn, lane, acc);
      } else {
        const int slot = g.split_slot[t];
        const int q = S ? cur_seg
                        : cta - (g.tile_cta0 ? g.tile_cta0[t]
                                             : cta_of_unit((int64_t)t * g.ki, g.units, g.grid));
        double* w = g.ws + ((size_t)slot * g.qmax + q) * (size_t)(Cfg::BM * Cfg::BN);
#pragma unroll
        for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
          for (int nt = 0; nt < Cfg::NT; ++nt)
#pragma unroll
            for (int x = 0; x < 2; ++x) w[frag_index<Cfg>(warp, mt, nt, x, lane)] = acc[mt][nt][x];
      }
#pragma unroll
      for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < Cfg::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
      tile_start = tile_end;
    }
    if (tile_end) {
      kk = 0;
      ++t;
      cur_seg = 0;
      seg_stop = S > 1 ? g.ki / S : g.ki;
      if constexpr (kTriCfg) tri = g.tile_tri && u + 1 < u1 && g.tile_tri[t];
    } else {
      ++kk;
      if (seg_end) {
        ++cur_seg;
        seg_stop = (int)((int64_t)(cur_seg + 1) * g.ki / S);
      }
    }
  }
}

// ---- X·[W|C] with the epilogue off the DMMA path (TMEM-staged accumulators) ------
// K = 2p is only 8–16 k-slices per tile, so the fused epilogue (G/X loads, P
// stores, column partials) idles the DMMA pipe ≈20% of the time.  Here the 8
// consumer warps hand each finished tile to tensor memory (tcgen05.st, two
// 128 KB buffers = all 512 TMEM columns) and go straight on to the next tile,
// while a fourth warpgroup reads the tile back (tcgen05.ld) and runs the same
// epilogue code.  TMEM lane quarter q (= warp % 4) holds consumer warps
// (wm, wn) = (0, q) and (1, q); epilogue warp q processes exactly their
// fragments, so every element, partial and shuffle order is the one of
// gemm_streamk — results are bitwise identical.  Data-parallel whole tiles.
__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n"
               ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31]) : "r"(addr) : "memory");
}

// tcgen05.wait::ld with the loaded registers as operands: no use of them can be
// scheduled before the wait.
__device__ __forceinline__ void tmem_wait_ld(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :: "memory");
}

// XM epilogue of one 8-column group nt of warp tile (wm, wn): EPI_XM of
// epilogue<> with NB = 1 (same element / partial / shuffle order).
template <class Cfg>
__device__ __forceinline__ void epilogue_xm_group(const GemmArgs& g, int tm, int tn, int wm, int wn,
                                                  int lane, int nt, const double (&a)[Cfg::MT][2]) {
  const EpiParams& e = g.ep;
  const int r = lane >> 2, q = lane & 3;
  const int64_t mw0 = (int64_t)tm * Cfg::BM + wm * Cfg::WM;
  const int64_t nw0 = (int64_t)tn * Cfg::BN + wn * Cfg::WN;
  const int64_t rb = mw0 / Cfg::WM;
  const bool interior = (mw0 + Cfg::WM <= e.n) && (((nw0 + Cfg::WN) >> 1) <= e.p);
  const int64_t j = (nw0 + nt * 8 + 2 * q) >> 1;
  double gv[Cfg::MT], xv[Cfg::MT];
  if (interior) {
#pragma unroll
    for (int mt = 0; mt < Cfg::MT; ++mt) {
      const int64_t idx = mw0 + mt * 8 + r + j * e.ld;
      gv[mt] = e.G[idx];
      xv[mt] = e.X[idx];
    }
  }
  double ks = 0.0, ds = 0.0;
#pragma unroll
  for (int mt = 0; mt < Cfg::MT; ++mt) {
    const int64_t row = mw0 + mt * 8 + r;
    const int64_t idx = row + j * e.ld;
    if (interior) {
      const double kkt = gv[mt] - a[mt][0];
      const double pv = (e.p_from_g ? gv[mt] : kkt) + e.beta * a[mt][1];
      e.G[idx] = pv;
      ks += kkt * kkt;
      ds += (e.d_sq ? pv : xv[mt]) * pv;
    } else if (row < e.n && j < e.p) {
      const double g0 = e.G[idx];
      const double kkt = g0 - a[mt][0];
      const double pv = (e.p_from_g ? g0 : kkt) + e.beta * a[mt][1];
      e.G[idx] = pv;
      ks += kkt * kkt;
      ds += (e.d_sq ? pv : e.X[idx]) * pv;
    }
  }
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    ks += __shfl_xor_sync(0xffffffffu, ks, o);
    ds += __shfl_xor_sync(0xffffffffu, ds, o);
  }
  if (r == 0 && j < e.p) {
    e.kpart[j * e.pstride + rb] = ks;
    e.dpart[j * e.pstride + rb] = ds;
  }
}

constexpr int kTmemEpiRegs = 104;  // epilogue warpgroup after setmaxnreg
template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS + 256, 1)
    gemm_xm_tmem(GemmArgs g, const __grid_constant__ GemmMaps maps) {
  static_assert(Cfg::WARPS == 8 && Cfg::WARPS_N == 4 && Cfg::MT * Cfg::NT * 4 == 128,
                "TMEM staging: 8 consumer warps (2 × 4), 64 doubles each");
  if (g.ctl && g.ctl->done) return;
  extern __shared__ __align__(1024) char smem_raw[];
  constexpr int S = Cfg::STAGES;
  char* As = smem_ring<Cfg>(smem_raw);
  char* Bs = As + S * Cfg::A_STAGE * 8;
  uint64_t* full = reinterpret_cast<uint64_t*>(Bs + S * Cfg::B_STAGE * 8);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;   // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int w = (int)(g.upc / g.ki);
  const int t0 = blockIdx.x * w, t1 = min(g.ntiles, t0 + w);
  if (t0 >= t1) return;  // uniform over the CTA, before any TMEM allocation
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], Cfg::WARPS);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], Cfg::WARPS);
      mbar_init(&acc_empty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {  // all 512 columns: two 128 × (2 × 128) accumulator buffers
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n"
                 ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = *tslot;
  if (warp >= Cfg::WARPS && warp < Cfg::WARPS + 4) {  // producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
    const int64_t u0 = (int64_t)t0 * g.ki, u1 = (int64_t)t1 * g.ki;
    if (warp == Cfg::WARPS && lane == 0) produce_tma<Cfg>(g, maps, As, Bs, full, empty, u0, u1);
    return;
  }
  const uint32_t quarter = (uint32_t)(warp & 3) * 32u;
  if (warp >= Cfg::WARPS + 4) {  // epilogue warpgroup: warp q reads TMEM lanes [32q, 32q+32)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kTmemEpiRegs));
    const int wn = warp & 3;
    const EpiParams& e = g.ep;
    for (int t = t0; t < t1; ++t) {
      const int buf = (t - t0) & 1;
      const unsigned ph = (unsigned)((t - t0) >> 1) & 1u;
      {  // while the tile is still being multiplied: its G / X columns into L2
        // (lane c: column j0 + c/2 of G or X, the tile's 128 rows, one bulk prefetch)
        const int2 tp = g.tiles[t];
        const int64_t m0 = (int64_t)tp.x * Cfg::BM;
        const int64_t rows = e.n - m0 < Cfg::BM ? e.n - m0 : Cfg::BM;
        const int64_t j = ((int64_t)tp.y * Cfg::BN + wn * Cfg::WN) / 2 + (lane >> 1);
        if (rows > 0 && j < e.p) {
          const double* src = ((lane & 1) ? e.X : e.G) + m0 + j * e.ld;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src),
                       "r"((unsigned)((rows * 8 + 15) & ~15ll)) : "memory");
        }
      }
      mbar_wait(&acc_full[buf], ph);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const int2 tc = g.tiles[t];
#pragma unroll 1
      for (int wm = 0; wm < 2; ++wm)
#pragma unroll 1
        for (int nt = 0; nt < Cfg::NT; ++nt) {
          uint32_t v[32];
          tmem_ld32(tbase + (quarter << 16) + (uint32_t)(buf * 256 + wm * 128 + nt * 32), v);
          tmem_wait_ld(v);
          double a[Cfg::MT][2];
#pragma unroll
          for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
            for (int x = 0; x < 2; ++x)
              a[mt][x] = __hiloint2double((int)v[(mt * 2 + x) * 2 + 1], (int)v[(mt * 2 + x) * 2]);
          epilogue_xm_group<Cfg>(g, tc.x, tc.y, wm, wn, lane, nt, a);
        }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(Cfg::THREADS + 128) : "memory");  // consumers + epilogue
    return;
  }
  {  // consumers
    constexpr int R = (65536 - 128 * kProducerRegs - 128 * kTmemEpiRegs) / Cfg::THREADS / 8 * 8;
    // setmaxnreg only redistributes the registers the CTA was launched with
    // (65536 / 512 threads = 128 each): an increase that the decreases do not
    // cover blocks forever
    constexpr int kLaunchRegs = 65536 / (Cfg::THREADS + 256) / 8 * 8;
    static_assert(128 * kProducerRegs + 128 * kTmemEpiRegs + Cfg::THREADS * (R > 232 ? 232 : R) <=
                      kLaunchRegs * (Cfg::THREADS + 256),
                  "register pool of the CTA exceeded");
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(R > 232 ? 232 : R));
  }
  const int wm = warp / Cfg::WARPS_N;
  const int wn = warp % Cfg::WARPS_N;
  double acc[Cfg::MT][Cfg::NT][2];
  int stage = 0;
  unsigned phase = 0;
  for (int t = t0; t < t1; ++t) {
#pragma unroll
    for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < Cfg::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    for (int kk = 0; kk < g.ki; ++kk) {
      mbar_wait(&full[stage], phase);
      mma_stage<Cfg>(As + stage * (Cfg::A_STAGE * 8), Bs + stage * (Cfg::B_STAGE * 8), wm, wn,
                     lane, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == S) {
        stage = 0;
        phase ^= 1u;
      }
    }
    const int buf = (t - t0) & 1;
    const unsigned ph = (unsigned)((t - t0) >> 1) & 1u;
    mbar_wait(&acc_empty[buf], ph ^ 1u);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
    for (int nt = 0; nt < Cfg::NT; ++nt) {
      uint32_t v[32];
#pragma unroll
      for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          v[(mt * 2 + x) * 2] = (uint32_t)__double2loint(acc[mt][nt][x]);
          v[(mt * 2 + x) * 2 + 1] = (uint32_t)__double2hiint(acc[mt][nt][x]);
        }
      tmem_st32(tbase + (quarter << 16) + (uint32_t)(buf * 256 + wm * 128 + nt * 32), v);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&acc_full[buf]);
  }
  asm volatile("bar.sync 1, %0;\n" ::"n"(Cfg::THREADS + 128) : "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase));
  }
}

// ---- X·[W|C] with a fused epilogue whose operands are staged by TMA -------------
// The epilogue of X·[W|C] needs, per output element, G and X (kkt = G − XW,
// P = kkt + β·XC, column partials Σkkt², ΣX∘P).  Here the producer thread also
// loads each tile's G and X blocks (128 rows × 32 output columns) into shared
// memory with TMA while the tile is multiplied, so the consumers run the
// epilogue straight after their last DMMA with every operand on chip: no
// global-load latency, and the FP64 epilogue instructions run in one burst per
// tile instead of being interleaved with (and starved by) the DMMA stream of a
// separate epilogue warpgroup.  128 × 64 tiles (32 output columns) keep the
// ring (3 × 48 KB) plus the staging (2 × 32 KB) inside 227 KB.
// Column partials are reduced over the tile's 128 rows in a fixed order
// (warp shuffles, then the four warp rows in order): one partial per
// (128-row block, column).
// The staging boxes are {16 rows, 32 columns} with the 128-byte swizzle (box b
// of rows [16b, 16b+16) at b·4 KB; "row" of the swizzle = the column): the
// epilogue's lanes (r, q) read rows r(+8·mt) of four columns, and with the
// columns of one 8-wide fragment chosen as {0, 1, 4, 5} + base (mcat column
// order perm32, pcal_kernels.cuh xm_slot_of_col) two of them XOR into each
// 64-byte half of the bank space: 2 wavefronts, the minimum for 256 bytes.
struct alignas(64) XmMaps {
  CUtensorMap a;  // X  {n, K = pp}, box {16, BK}
  CUtensorMap b;  // [W|C] interleaved (perm32 column order) {K = pp, 2pp}, box {16, BN}
  CUtensorMap g;  // G  {n, p}, box {16, BN/2}, 128-byte swizzle
  CUtensorMap x;  // X  {n, p}, box {16, BN/2}, 128-byte swizzle
};
// output column (within the tile) of fragment (wn, nt) lane column q
__device__ __forceinline__ int xm_out_col(int wn, int nt, int q) {
  return wn * 16 + 8 * (nt >> 1) + 2 * (nt & 1) + (q & 1) + 4 * (q >> 1);
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS + 128, 1)
    gemm_xm_staged(GemmArgs g, const __grid_constant__ XmMaps maps) {
  constexpr int S = Cfg::STAGES, BM = Cfg::BM, BNO = Cfg::BN / 2;
  static_assert(Cfg::WARPS == 8 && Cfg::WARPS_M == 4 && Cfg::WARPS_N == 2 && BM == 128 &&
                    BNO == 32,
                "staged XM: 128 × 64 tiles (32 output columns), 4 × 2 consumer warps");
  if (g.ctl && g.ctl->done) return;
  extern __shared__ __align__(1024) char smem_raw[];
  char* As = smem_ring<Cfg>(smem_raw);
  char* Bs = As + S * Cfg::A_STAGE * 8;
  double* Gs = reinterpret_cast<double*>(Bs + S * Cfg::B_STAGE * 8);  // [col][row]
  double* Xs = Gs + BM * BNO;
  double* red = Xs + BM * BNO;                                        // [2][8][BNO]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * 8 * BNO);
  uint64_t* empty = full + S;
  uint64_t* efull = empty + S;
  uint64_t* eempty = efull + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // tiles round-robin over the CTAs: at any time the grid works on ~148
  // consecutive (tm-major) tiles, so each 128-row block of X (the A operand,
  // K = pp) is fetched from DRAM once and served from L2 to the CTAs of its
  // 2pp/64 column tiles (a contiguous tile range per CTA keeps 148 different
  // row blocks live — more than L2 holds at p = 1024)
  if ((int)blockIdx.x >= g.ntiles) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], Cfg::WARPS);
    }
    mbar_init(efull, 1);
    mbar_init(eempty, Cfg::WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp >= Cfg::WARPS) {  // producer warpgroup: one thread drives the TMA unit
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
    if (warp != Cfg::WARPS || lane != 0) return;
    const int kload = min(S, g.ki - 1);  // when the previous tile's epilogue is surely done
    int s = 0;
    unsigned ph = 0;
    int it = 0;
    for (int t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++it) {
      const int2 tc = g.tiles[t];
      const int m0 = tc.x * BM, n0 = tc.y * Cfg::BN, j0 = tc.y * BNO;
      for (int kk = 0; kk < g.ki; ++kk) {
        if (kk == kload) {  // this tile's G / X blocks (after the previous tile's epilogue released them)
          mbar_wait(eempty, (unsigned)(it & 1) ^ 1u);
          mbar_arrive_expect_tx(efull, 2 * BM * BNO * 8);
#pragma unroll
          for (int rb = 0; rb < BM / 16; ++rb) {
            tma_load_2d(Gs + rb * 16 * BNO, &maps.g, m0 + 16 * rb, j0, efull);
            tma_load_2d(Xs + rb * 16 * BNO, &maps.x, m0 + 16 * rb, j0, efull);
          }
        }
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        char* as = As + s * (Cfg::A_STAGE * 8);
        char* bs = Bs + s * (Cfg::B_STAGE * 8);
        const int k0 = kk * Cfg::BK;
#pragma unroll
        for (int mb = 0; mb < BM / 16; ++mb)
          tma_load_2d(as + mb * (Cfg::BK * 128), &maps.a, m0 + 16 * mb, k0, &full[s]);
#pragma unroll
        for (int kh = 0; kh < Cfg::BK / 16; ++kh)
          tma_load_2d(bs + kh * (Cfg::BN * 128), &maps.b, k0 + 16 * kh, n0, &full[s]);
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(232));
  const EpiParams& e = g.ep;
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  const int r = lane >> 2, q = lane & 3;
  double acc[Cfg::MT][Cfg::NT][2];
  int stage = 0;
  unsigned phase = 0;
  int it = 0;
  for (int t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++it) {
#pragma unroll
    for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < Cfg::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    for (int kk = 0; kk < g.ki; ++kk) {
      mbar_wait(&full[stage], phase);
      mma_stage<Cfg>(As + stage * (Cfg::A_STAGE * 8), Bs + stage * (Cfg::B_STAGE * 8), wm, wn,
                     lane, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == S) {
        stage = 0;
        phase ^= 1u;
      }
    }
    // ---- epilogue: every operand in shared memory
    const int2 tc = g.tiles[t];
    const int64_t m0 = (int64_t)tc.x * BM;
    const int64_t j0 = (int64_t)tc.y * BNO;
    mbar_wait(efull, (unsigned)(it & 1));
    double* rk = red + (it & 1) * (8 * BNO);  // per-tile double buffer: [k rows 0-3 | d rows 0-3]
    const char* gsb = reinterpret_cast<const char*>(Gs);
    const char* xsb = reinterpret_cast<const char*>(Xs);
#pragma unroll
    for (int nt = 0; nt < Cfg::NT; ++nt) {
      const int jl = xm_out_col(wn, nt, q);  // output column within the tile
      const int64_t j = j0 + jl;
      double ks = 0.0, ds = 0.0;
#pragma unroll
      for (int mt = 0; mt < Cfg::MT; ++mt) {
        const int rl = wm * Cfg::WM + mt * 8 + r;
        const int64_t row = m0 + rl;
        // swizzled staging: box rl/16, swizzle row jl, chunk ((rl & 15) >> 1) ^ (jl & 7)
        const int off = (rl >> 4) * (16 * BNO * 8) + jl * 128 +
                        ((((rl & 15) >> 1) ^ (jl & 7)) << 4) + (rl & 1) * 8;
        const double gv = *reinterpret_cast<const double*>(gsb + off);
        const double xv = *reinterpret_cast<const double*>(xsb + off);
        if (row < e.n && j < e.p) {
          const double kkt = gv - acc[mt][nt][0];
          const double pv = (e.p_from_g ? gv : kkt) + e.beta * acc[mt][nt][1];
          e.G[row + j * e.ld] = pv;
          ks += kkt * kkt;
          ds += (e.d_sq ? pv : xv) * pv;
        }
      }
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        ks += __shfl_xor_sync(0xffffffffu, ks, o);
        ds += __shfl_xor_sync(0xffffffffu, ds, o);
      }
      if (r == 0) {
        rk[wm * BNO + jl] = ks;
        rk[(4 + wm) * BNO + jl] = ds;  // second half of the buffer: d partials
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(eempty);  // Gs / Xs of this tile are no longer read
    // the four warp rows' partials of each column, summed in row order
    asm volatile("bar.sync 1, %0;\n" ::"n"(Cfg::THREADS) : "memory");
    if (warp == 0) {
      const int jl = lane;  // BNO == 32 columns
      const int64_t j = j0 + jl;
      if (j < e.p) {
        const double kv = ((rk[jl] + rk[BNO + jl]) + rk[2 * BNO + jl]) + rk[3 * BNO + jl];
        const double dv = ((rk[4 * BNO + jl] + rk[5 * BNO + jl]) + rk[6 * BNO + jl]) +
                          rk[7 * BNO + jl];
        e.kpart[j * e.pstride + tc.x] = kv;
        e.dpart[j * e.pstride + tc.x] = dv;
      }
    }
  }
}

// ---- P = G − X·M1 with M1 = W − β·C: the single-block X·[W|C] -------------------
// PCAL / PLAM need P = (G − XW) + β·XC and the column sums of kkt² with
// kkt = G − XW.  Multiplying by the one p × p matrix M1 = W − β·C gives P with
// half the flops of X·[W|C]; Σ kkt² then follows from Σ P² by the identity
// (X has XᵀX = I + C, C and W symmetric):
//   ‖G − XW‖² = ‖P‖² + 2β⟨W, C²⟩ − β²(‖C‖² + ⟨C, C²⟩)
// (session.cu k_kkt_gate, with a gated fallback to the two-block product when
// the correction cancels too much of ‖P‖²).  64 × 64 tiles, all 64 MMA
// columns are output columns: the G / X staging (64 rows × 64 columns, 2 ×
// 32 KB) fits beside a 4 × 32 KB ring.  Output column of (wn, nt, x, q):
// wn·16 + 8·nt + 2·x + {0,1,4,5}[q] (M1 stored in that slot order,
// pcal_kernels.cuh xm1_slot_of_col): each 8-lane row group of a fragment
// column reads four columns whose (jl mod 8) are {b, b^1, b^4, b^5} — the
// swizzled staging reads are conflict-free (2 wavefronts per 256 bytes).
__device__ __forceinline__ int xm1_out_col(int wn, int nt, int x, int q) {
  return wn * 16 + 8 * nt + 2 * x + (q & 1) + 4 * (q >> 1);
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::THREADS + 128, 1)
    gemm_xm1_staged(GemmArgs g, const __grid_constant__ XmMaps maps) {
  constexpr int S = Cfg::STAGES, BM = Cfg::BM, BN = Cfg::BN;
  static_assert(Cfg::WARPS == 8 && Cfg::WARPS_M == 2 && Cfg::WARPS_N == 4 && BM == 64 &&
                    BN == 64 && Cfg::NT == 2 && Cfg::MT == 4,
                "XM1: 64 × 64 tiles, 2 × 4 consumer warps");
  if (g.ctl && g.ctl->done) return;
  extern __shared__ __align__(1024) char smem_raw[];
  char* As = smem_ring<Cfg>(smem_raw);
  char* Bs = As + S * Cfg::A_STAGE * 8;
  double* Gs = reinterpret_cast<double*>(Bs + S * Cfg::B_STAGE * 8);  // [col][row], swizzled
  double* Xs = Gs + BM * BN;
  double* red = Xs + BM * BN;  // [2 parity][k wm0, k wm1, d wm0, d wm1][BN]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 2 * 4 * BN);
  uint64_t* empty = full + S;
  uint64_t* efull = empty + S;
  uint64_t* eempty = efull + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if ((int)blockIdx.x >= g.ntiles) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], Cfg::WARPS);
    }
    mbar_init(efull, 1);
    mbar_init(eempty, Cfg::WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp >= Cfg::WARPS) {  // producer warpgroup: one thread drives the TMA unit
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
    if (warp != Cfg::WARPS || lane != 0) return;
    const int kload = min(S, g.ki - 1);
    int s = 0;
    unsigned ph = 0;
    int it = 0;
    for (int t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++it) {
      const int2 tc = g.tiles[t];
      const int m0 = tc.x * BM, n0 = tc.y * BN;
      for (int kk = 0; kk < g.ki; ++kk) {
        if (kk == kload) {
          mbar_wait(eempty, (unsigned)(it & 1) ^ 1u);
          mbar_arrive_expect_tx(efull, 2 * BM * BN * 8);
#pragma unroll
          for (int rb = 0; rb < BM / 16; ++rb) {
            tma_load_2d(Gs + rb * 16 * BN, &maps.g, m0 + 16 * rb, n0, efull);
            tma_load_2d(Xs + rb * 16 * BN, &maps.x, m0 + 16 * rb, n0, efull);
          }
        }
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], Cfg::STAGE_BYTES);
        char* as = As + s * (Cfg::A_STAGE * 8);
        char* bs = Bs + s * (Cfg::B_STAGE * 8);
        const int k0 = kk * Cfg::BK;
#pragma unroll
        for (int mb = 0; mb < BM / 16; ++mb)
          tma_load_2d(as + mb * (Cfg::BK * 128), &maps.a, m0 + 16 * mb, k0, &full[s]);
#pragma unroll
        for (int kh = 0; kh < Cfg::BK / 16; ++kh)
          tma_load_2d(bs + kh * (BN * 128), &maps.b, k0 + 16 * kh, n0, &full[s]);
        if (++s == S) {
          s = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(232));
  const EpiParams& e = g.ep;
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  const int r = lane >> 2, q = lane & 3;
  double acc[Cfg::MT][Cfg::NT][2];
  int stage = 0;
  unsigned phase = 0;
  int it = 0;
  for (int t = blockIdx.x; t < g.ntiles; t += gridDim.x, ++it) {
#pragma unroll
    for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < Cfg::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
    for (int kk = 0; kk < g.ki; ++kk) {
      mbar_wait(&full[stage], phase);
      mma_stage<Cfg>(As + stage * (Cfg::A_STAGE * 8), Bs + stage * (Cfg::B_STAGE * 8), wm, wn,
                     lane, acc);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == S) {
        stage = 0;
        phase ^= 1u;
      }
    }
    const int2 tc = g.tiles[t];
    const int64_t m0 = (int64_t)tc.x * BM;
    const int64_t j0 = (int64_t)tc.y * BN;
    mbar_wait(efull, (unsigned)(it & 1));
    double* rk = red + (it & 1) * (4 * BN);
    const char* gsb = reinterpret_cast<const char*>(Gs);
    const char* xsb = reinterpret_cast<const char*>(Xs);
#pragma unroll
    for (int nt = 0; nt < Cfg::NT; ++nt)
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        const int jl = xm1_out_col(wn, nt, x, q);
        const int64_t j = j0 + jl;
        double ks = 0.0, ds = 0.0;
#pragma unroll
        for (int mt = 0; mt < Cfg::MT; ++mt) {
          const int rl = wm * Cfg::WM + mt * 8 + r;
          const int64_t row = m0 + rl;
          const int off = (rl >> 4) * (16 * BN * 8) + jl * 128 +
                          ((((rl & 15) >> 1) ^ (jl & 7)) << 4) + (rl & 1) * 8;
          const double gv = *reinterpret_cast<const double*>(gsb + off);
          const double xv = *reinterpret_cast<const double*>(xsb + off);
          if (row < e.n && j < e.p) {
            const double pv = gv - acc[mt][nt][x];
            e.G[row + j * e.ld] = pv;
            ks += pv * pv;
            ds += xv * pv;
          }
        }
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          ks += __shfl_xor_sync(0xffffffffu, ks, o);
          ds += __shfl_xor_sync(0xffffffffu, ds, o);
        }
        if (r == 0) {
          rk[wm * BN + jl] = ks;
          rk[(2 + wm) * BN + jl] = ds;
        }
      }
    __syncwarp();
    if (lane == 0) mbar_arrive(eempty);  // Gs / Xs of this tile are no longer read
    asm volatile("bar.sync 1, %0;\n" ::"n"(Cfg::THREADS) : "memory");
    if (threadIdx.x < BN) {
      const int jl = threadIdx.x;
      const int64_t j = j0 + jl;
      if (j < e.p) {
        e.kpart[j * e.pstride + tc.x] = rk[jl] + rk[BN + jl];
        e.dpart[j * e.pstride + tc.x] = rk[2 * BN + jl] + rk[3 * BN + jl];
      }
    }
  }
}

// Sums the partials of split tiles in CTA order (q = 0, 1, …) and applies the
// epilogue with the consumer-warp geometry of the main kernel.  q-outer loop:
// every partial contributes FRAG independent coalesced loads per thread.
template <class Cfg, int EPI>
__global__ void __launch_bounds__(Cfg::THREADS) gemm_fixup(GemmArgs g, const FixupTask* tasks) {
  if (g.ctl && g.ctl->done) return;
  if (g.gate && !*g.gate) return;
  const FixupTask tk = tasks[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  double acc[Cfg::MT][Cfg::NT][2];
#pragma unroll
  for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < Cfg::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  const double* base = g.ws + (size_t)tk.slot * g.qmax * (size_t)(Cfg::BM * Cfg::BN);
#pragma unroll 2
  for (int q = 0; q < tk.nq; ++q) {
    const double* w = base + (size_t)q * (Cfg::BM * Cfg::BN);
#pragma unroll
    for (int mt = 0; mt < Cfg::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < Cfg::NT; ++nt)
#pragma unroll
        for (int x = 0; x < 2; ++x) acc[mt][nt][x] += w[frag_index<Cfg>(warp, mt, nt, x, lane)];
  }
  const int2 tc = g.tiles[tk.tile];
  epilogue<Cfg, EPI>(g, tc.x, tc.y, wm, wn, lane, acc);
}

// Plain-store fixup spread over the whole chip: one thread per output element
// of every split tile (heavily split tall-skinny Grams have ~70 partials per tile).
template <class Cfg>
__global__ void __launch_bounds__(256) gemm_fixup_store(GemmArgs g, const FixupTask* tasks,
                                                        int ntasks) {
  if (g.ctl && g.ctl->done) return;
  if (g.gate && !*g.gate) return;
  constexpr int TILE = Cfg::BM * Cfg::BN;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ntasks * TILE) return;
  const int task = (int)(e / TILE);
  const int f = (int)(e % TILE);
  const FixupTask tk = tasks[task];
  const double* base = g.ws + (size_t)tk.slot * g.qmax * (size_t)TILE + f;
  double s = 0.0;
  for (int q = 0; q < tk.nq; ++q) s += base[(size_t)q * TILE];
  // decode the fragment-native index (frag_index)
  const int lane = f & 31;
  int r = f >> 5;
  const int x = r & 1;
  r >>= 1;
  const int nt = r % Cfg::NT;
  r /= Cfg::NT;
  const int mt = r % Cfg::MT;
  const int warp = r / Cfg::MT;
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  const int2 tc = g.tiles[tk.tile];
  const int64_t row = (int64_t)tc.x * Cfg::BM + wm * Cfg::WM + mt * 8 + (lane >> 2);
  const int64_t col = (int64_t)tc.y * Cfg::BN + wn * Cfg::WN + nt * 8 + 2 * (lane & 3) + x;
  const EpiParams& ep = g.ep;
  if (row < ep.m_store && col < ep.n_store) ep.C[row + col * ep.ldc] = s;
}

// ---- fixed-tree reduction of chunk partials (reproducible Gram) -------------
// The S_glob chunk partials (leaves, in global chunk order) are summed over a
// fixed binary tree: node (ℓ, i) covers leaves [i·2^ℓ, min((i+1)·2^ℓ, S_glob))
// and equals left + right (left alone when the right child is empty).  Each
// rank sums the maximal nodes inside its own leaf range (gemm_tree_local), the
// ranks exchange only those O(log S) node sums, and every rank finishes the
// same tree (gemm_tree_final): bitwise the same Gram for every rank count.

// Sum of the n leaves of one aligned node: binary counter + right fold.
__device__ __forceinline__ double tree_leaves(const double* leaf, int64_t stride, int n) {
  double st[24];
  int sp = 0;
  int j = 0;
  for (; j + 8 <= n; j += 8) {  // aligned 8-leaf blocks: 8 loads in flight, pairwise in registers
    double l[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) l[q] = leaf[(int64_t)(j + q) * stride];
    double v = ((l[0] + l[1]) + (l[2] + l[3])) + ((l[4] + l[5]) + (l[6] + l[7]));
    for (int k = (j + 8) >> 3; (k & 1) == 0; k >>= 1) v = st[--sp] + v;
    st[sp++] = v;
  }
  for (; j < n; ++j) {
    double v = leaf[(int64_t)j * stride];
    for (int k = j + 1; (k & 1) == 0; k >>= 1) v = st[--sp] + v;
    st[sp++] = v;
  }
  double acc = st[sp - 1];
  for (int q = sp - 2; q >= 0; --q) acc = st[q] + acc;
  return acc;
}

// out[k][task][f] = sum of this rank's maximal node k over its leaves
// ws[task][q][f] (q = local leaf index, leaf0 = first global leaf of the rank).
__global__ void __launch_bounds__(256) gemm_tree_local(const double* __restrict__ ws, int qmax,
                                                       int ntasks, int tile, const int2* nodes,
                                                       int nnodes, int64_t leaf0, int64_t nleaves,
                                                       double* __restrict__ out, const Ctl* ctl) {
  if (ctl && ctl->done) return;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ntasks * tile) return;
  const int task = (int)(e / tile), f = (int)(e % tile);
  for (int k = 0; k < nnodes; ++k) {
    const int2 nd = nodes[k];
    const int64_t a = (int64_t)nd.y << nd.x;
    const int64_t b = min(a + ((int64_t)1 << nd.x), nleaves);
    const double* leaf = ws + ((int64_t)task * qmax + (a - leaf0)) * tile + f;
    out[((int64_t)k * ntasks + task) * tile + f] = tree_leaves(leaf, tile, (int)(b - a));
  }
}

// Merges every rank's node sums (buf[r][k][task][f], labels nodes[r·maxn + k])
// in global order into the tree root and stores it (fragment-native decode).
template <class Cfg>
__global__ void __launch_bounds__(256) gemm_tree_final(GemmArgs g, const FixupTask* tasks,
                                                       int ntasks, const double* buf,
                                                       const int32_t* cnt, const int2* nodes,
                                                       int R, int maxn) {
  if (g.ctl && g.ctl->done) return;
  constexpr int TILE = Cfg::BM * Cfg::BN;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)ntasks * TILE) return;
  const int task = (int)(e / TILE);
  const int f = (int)(e % TILE);
  double sv[24];
  int sl[24], si[24];
  int sp = 0;
  for (int r = 0; r < R; ++r) {
    const int nk = cnt[r];
    for (int k = 0; k < nk; ++k) {
      const int2 nd = nodes[r * maxn + k];
      double v = buf[(((int64_t)r * maxn + k) * ntasks + task) * TILE + f];
      int l = nd.x, i = nd.y;
      while (sp > 0 && sl[sp - 1] == l && (si[sp - 1] & 1) == 0 && si[sp - 1] + 1 == i) {
        v = sv[sp - 1] + v;  // left sibling + right sibling = parent
        --sp;
        ++l;
        i >>= 1;
      }
      sv[sp] = v;
      sl[sp] = l;
      si[sp] = i;
      ++sp;
    }
  }
  double s = sv[sp - 1];
  for (int q = sp - 2; q >= 0; --q) s = sv[q] + s;  // truncated right spine
  const FixupTask tk = tasks[task];
  const int lane = f & 31;
  int rr = f >> 5;
  const int x = rr & 1;
  rr >>= 1;
  const int nt = rr % Cfg::NT;
  rr /= Cfg::NT;
  const int mt = rr % Cfg::MT;
  const int warp = rr / Cfg::MT;
  const int wm = warp / Cfg::WARPS_N, wn = warp % Cfg::WARPS_N;
  const int2 tc = g.tiles[tk.tile];
  const int64_t row = (int64_t)tc.x * Cfg::BM + wm * Cfg::WM + mt * 8 + (lane >> 2);
  const int64_t col = (int64_t)tc.y * Cfg::BN + wn * Cfg::WN + nt * 8 + 2 * (lane & 3) + x;
  const EpiParams& ep = g.ep;
  if (row < ep.m_store && col < ep.n_store) ep.C[row + col * ep.ldc] = s;
}

}  // namespace pcal
