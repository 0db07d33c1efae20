// gemm_types.h — host/device shared types of the stream-K DMMA GEMM.
#pragma once

#include <cuda.h>  // CUtensorMap

#include "common.cuh"

namespace pcal {

enum AMode { A_MCONTIG = 0, A_KCONTIG = 1 };
enum EpiKind { EPI_STORE = 0, EPI_GRAD = 1, EPI_XM = 2 };

struct EpiParams {
  // EPI_STORE: C[row + col·ldc] = acc for row < m_store, col < n_store
  double* C;
  int64_t ldc, m_store, n_store;
  // EPI_GRAD: G = acc (+g0); fpart[rb·p + col] = Σ_rows X∘G over a warp row-block
  // EPI_XM:   acc columns interleave (X·W, X·C) per output column j:
  //           kkt = G − XW; P = kkt + β·XC (written over G);
  //           kpart[rb·p + j] = Σ kkt², dpart[rb·p + j] = Σ X∘P
  double* G;
  const double* X;
  const double* g0;
  int64_t ld;        // leading dimension of G, X, g0
  double* fpart;
  double* kpart;
  double* dpart;
  int32_t* bad;      // set to 1 if a non-finite value is produced (GRAD)
  double beta;
  int64_t n, p;
  int64_t pstride;   // column stride of the partial arrays: part[col·pstride + rb]
  int32_t p_from_g;  // EPI_XM: P = G + β·acc1 (dual-ascent / MOptQR) instead of kkt + β·acc1
  int32_t d_sq;      // EPI_XM: dpart accumulates Σ P² (ALM's ‖∇L‖) instead of Σ X∘P
};

struct GemmArgs {
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  int64_t M, N;       // logical extents (loads beyond are zero-filled)
  int64_t K;          // multiple of BK (operands zero-padded)
  const int2* tiles;  // (tm, tn) per tile
  const int32_t* split_slot;  // per tile: workspace slot or -1 (owned by one CTA)
  int32_t ntiles;
  int32_t ki;         // k-iterations per tile
  int64_t units;      // ntiles · ki
  int32_t grid;
  int64_t upc;        // > 0: data-parallel (whole tiles per CTA), 0: stream-K
  double* ws;         // [slot][q][BM·BN] partials, fragment-native layout
  int32_t qmax;
  EpiParams ep;
  const Ctl* ctl;     // early exit when ctl->done (may be null)
  const int32_t* gate;  // early exit when non-null and *gate == 0 (in-graph CholeskyQR)
  int32_t force_ws;     // chunk-partial plans: every CTA stores its partial (no epilogue)
  int32_t segs;         // > 0: segmented schedule, S fixed K segments per tile (see below)
  int32_t a_stream;     // A is read exactly once (dense gradient): L2 evict-first loads
  const uint8_t* tile_tri;  // per tile: 1 = diagonal tile of an upper-triangle-only block
  const int64_t* cta_begin; // stream-K with weighted tiles: unit range start of each CTA (G+1)
  const int32_t* tile_cta0; //   and the first CTA of each tile (its partial slot q = cta − cta0)
};

struct FixupTask {   // one split tile
  int32_t tile;
  int32_t slot;
  int32_t nq;
};

// CTA whose contiguous unit range contains unit x: max c with ⌊c·U/G⌋ ≤ x.
__host__ __device__ inline int32_t cta_of_unit(int64_t x, int64_t U, int32_t G) {
  int64_t c = ((x + 1) * (int64_t)G + U - 1) / U - 1;
  return (int32_t)(c < 0 ? 0 : (c >= G ? G - 1 : c));
}
// upc > 0: data-parallel schedule, each CTA owns upc consecutive units (whole tiles)
__host__ __device__ inline int64_t cta_unit_begin(int32_t c, int64_t U, int32_t G, int64_t upc) {
  if (upc > 0) return (int64_t)c * upc < U ? (int64_t)c * upc : U;
  return (int64_t)c * U / G;
}
// Segmented schedule (reproducible plans): the K range of every tile is cut
// into S segments at k-iterations ⌊s·ki/S⌋, independent of the tile count;
// CTA c owns the whole segments [⌊c·T·S/G⌋, ⌊(c+1)·T·S/G⌋) and flushes one
// partial per segment, so each output is (((0 + P₀) + P₁) + …) over the same
// segments whatever the number of tiles or CTAs.
__host__ __device__ inline int32_t seg_of(int32_t kk, int32_t ki, int32_t S) {
  return (int32_t)(((int64_t)(kk + 1) * S - 1) / ki);
}
__host__ __device__ inline int64_t seg_unit_begin(int32_t c, int32_t ntiles, int32_t ki,
                                                  int32_t S, int32_t G) {
  const int64_t sg = (int64_t)c * ntiles * S / G;
  return (sg / S) * ki + (sg % S) * ki / S;
}


// ---- host-side plans -----------------------------------------------------------
// CFG_XMT: the CFG_BIG tiles of X·[W|C] with the TMEM-staged epilogue
// (gemm_xm_tmem; data-parallel whole tiles).  CFG_XMS: 128 × 64 tiles of
// X·[W|C] with the fused epilogue reading TMA-staged G / X (gemm_xm_staged;
// column partials per 128-row tile block).  CFG_XM1: 64 × 64 tiles of the
// single-block P = G − X·M1 (gemm_xm1_staged; column partials per 64-row block).
enum CfgSize { CFG_BIG = 0, CFG_MID = 1, CFG_SMALL = 2, CFG_XMT = 3, CFG_XMS = 4, CFG_XM1 = 5 };

struct CfgInfo {
  int BM, BN, WM, BK;
};
CfgInfo cfg_info(int size);
int pick_size(int64_t N);

// A GEMM with a static stream-K schedule (tile list, split tiles, workspace).
struct GemmPlan {
  int size = CFG_BIG, amode = A_MCONTIG, epi = EPI_STORE;
  GemmArgs args{};
  int2* d_tiles = nullptr;
  uint8_t* d_tri = nullptr;   // triangular (diagonal) tiles of symmetric Grams
  int64_t* d_cta_begin = nullptr;
  int32_t* d_tile_cta0 = nullptr;
  int32_t* d_split = nullptr;
  FixupTask* d_tasks = nullptr;
  int ntasks = 0;
  double* ws = nullptr;
  size_t ws_doubles = 0;
  bool no_fixup = false;  // chunk-partial plans: the caller reduces ws (launch_gemm_tree_*)
  GemmPlan() = default;
  GemmPlan(const GemmPlan&) = delete;
  GemmPlan& operator=(const GemmPlan&) = delete;
  ~GemmPlan() { release(); }
  void release();
};

// Build a plan.  `sym_row0` >= 0 skips tiles lying strictly below the diagonal
// of the block starting at row sym_row0 (the XᵀX half of the Gram); with
// `sym_first` also those of the block at row 0 (GᵀX of a symmetric operator).
//
// Reproducible schedules (the sharded path):
//   fixed_splits = S > 0: every tile's K range is cut into the same S segments
//     (segment boundaries ⌊s·ki/S⌋ depend only on K and S, not on the number
//     of tiles), fixed up in segment order — per-element results independent
//     of M, hence of the row partition.
//   chunk_partials: S = K / chunk segments whose partials are all kept in ws
//     ([task][q][BM·BN], q padded to qmax_min) for an ordered sum across ranks.
void plan_gemm(GemmPlan& pl, int device, int size, int amode, int epi, int64_t M, int64_t N,
               int64_t K, int64_t sym_row0 = -1, int grid_override = 0, int fixed_splits = 0,
               bool chunk_partials = false, int qmax_min = 0, bool sym_first = false);
void launch_gemm(const GemmPlan& pl, cudaStream_t st);
// Tiles plan_gemm schedules for an M×N output (same skipping rule).
int64_t count_tiles(int size, int64_t M, int64_t N, int64_t sym_row0 = -1,
                    bool sym_first = false);
// Fixed-tree reduction of a chunk-partial plan's ws (gemm_dmma.cuh):
// local maximal-node sums into `out` ([nnodes][ntasks][BM·BN]), then the
// merge of every rank's node sums (buf = [R][maxn][ntasks][BM·BN]) into ep.C.
void launch_gemm_tree_local(const GemmPlan& pl, const int2* nodes, int nnodes, int64_t leaf0,
                            int64_t nleaves, double* out, cudaStream_t st);
void launch_gemm_tree_final(const GemmPlan& pl, const double* buf, const int32_t* cnt,
                            const int2* nodes, int R, int maxn, cudaStream_t st);
int num_sms(int device);
// A rank-`rank` FP64 TMA descriptor (no swizzle, zero fill): dims innermost
// first, pitches (bytes) of dims 1…rank−1, box extents.
void encode_tensor_map(CUtensorMap* m, const void* base, int rank, const int64_t* dims,
                       const int64_t* pitches_bytes, const int* box);

}  // namespace pcal
