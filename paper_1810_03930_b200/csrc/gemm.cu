// gemm.cu — stream-K DMMA GEMM: configurations, schedules, launches.
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "../../include/pcal_b200.h"
#include "gemm_dmma.cuh"

namespace pcal {

// ------------------------------------------------------------------------------
// GEMM configurations and launch plumbing
// ------------------------------------------------------------------------------

template <int AM>
using CfgBig = GemmCfg<128, 128, 2, 4, 3, AM, 32>;  // BK = 32: 3 × 64 KB stages
using CfgXms = GemmCfg<128, 64, 4, 2, 3, A_MCONTIG, 32>;  // staged X·[W|C]: 3 × 48 KB + 64 KB
using CfgXm1 = GemmCfg<64, 64, 2, 4, 4, A_MCONTIG, 32>;   // staged X·M1: 4 × 32 KB + 64 KB
template <int AM>
using CfgMid = GemmCfg<64, 64, 2, 2, 4, AM>;
template <int AM>
using CfgSmall = GemmCfg<64, 32, 2, 2, 4, AM>;

int num_sms(int device) {
  int v = 0;
  PCAL_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  return v;
}

CfgInfo cfg_info(int size) {
  switch (size) {
    case CFG_BIG:
    case CFG_XMT: return {128, 128, CfgBig<A_MCONTIG>::WM, CfgBig<A_MCONTIG>::BK};
    case CFG_XMS: return {128, 64, CfgXms::WM, CfgXms::BK};
    case CFG_XM1: return {64, 64, CfgXm1::WM, CfgXm1::BK};
    case CFG_MID: return {64, 64, 32, CfgMid<A_MCONTIG>::BK};
    default: return {64, 32, 32, CfgSmall<A_MCONTIG>::BK};
  }
}

void GemmPlan::release() {
  if (d_tiles) cudaFree(d_tiles);
  if (d_tri) cudaFree(d_tri);
  d_tri = nullptr;
  if (d_cta_begin) cudaFree(d_cta_begin);
  if (d_tile_cta0) cudaFree(d_tile_cta0);
  d_cta_begin = nullptr;
  d_tile_cta0 = nullptr;
  if (d_split) cudaFree(d_split);
  if (d_tasks) cudaFree(d_tasks);
  if (ws) cudaFree(ws);
  d_tiles = nullptr;
  d_split = nullptr;
  d_tasks = nullptr;
  ws = nullptr;
}

int pick_size(int64_t N) {
  if (N >= 128) return CFG_BIG;
  if (N > 32) return CFG_MID;
  return CFG_SMALL;
}

// Tile (tm, tn) lies strictly below the diagonal of a symmetric square block:
// the block starting at row sym_row0, and with sym_first also the one at row 0.
static bool below_diagonal(const CfgInfo& ci, int64_t tm, int64_t tn, int64_t sym_row0,
                           bool sym_first) {
  if (sym_row0 < 0) return false;
  const int64_t r0 = tm * ci.BM, c1 = (tn + 1) * ci.BN - 1;
  if (r0 >= sym_row0) return (r0 - sym_row0) > c1;
  return sym_first && r0 > c1;
}

int64_t count_tiles(int size, int64_t M, int64_t N, int64_t sym_row0, bool sym_first) {
  const CfgInfo ci = cfg_info(size);
  int64_t c = 0;
  for (int64_t tm = 0; tm < ceil_div(M, ci.BM); ++tm)
    for (int64_t tn = 0; tn < ceil_div(N, ci.BN); ++tn)
      if (!below_diagonal(ci, tm, tn, sym_row0, sym_first)) ++c;
  return c;
}

void plan_gemm(GemmPlan& pl, int device, int size, int amode, int epi, int64_t M,
                      int64_t N, int64_t K, int64_t sym_row0, int grid_override, int fixed_splits,
                      bool chunk_partials, int qmax_min, bool sym_first) {
  pl.release();
  pl.size = size;
  pl.amode = amode;
  pl.epi = epi;
  const CfgInfo ci = cfg_info(size);
  const int BK = ci.BK;
  if (K % BK) throw Error(PCAL_E_DIMENSION, "gemm: K must be a multiple of the k-slice");
  const int64_t tm_n = ceil_div(M, ci.BM), tn_n = ceil_div(N, ci.BN);
  std::vector<int2> tiles;
  // tm-major: consecutive tiles share the A row-block (L2 reuse across tn)
  for (int64_t tm = 0; tm < tm_n; ++tm)
    for (int64_t tn = 0; tn < tn_n; ++tn) {
      if (below_diagonal(ci, tm, tn, sym_row0, sym_first)) continue;
      tiles.push_back(make_int2((int)tm, (int)tn));
    }
  const int ntiles = (int)tiles.size();
  const int ki = (int)(K / BK);
  const int64_t units = (int64_t)ntiles * ki;
  int grid = grid_override > 0 ? grid_override : num_sms(device);
  if (units < grid) grid = (int)std::max<int64_t>(1, units);
  int64_t upc = 0;
  int segs = 0;
  if (fixed_splits > 0) {
    // segmented schedule: S fixed K segments per tile, whole segments per CTA
    if (fixed_splits > ki) throw Error(PCAL_E_DIMENSION, "gemm: more segments than k-slices");
    segs = fixed_splits;
    const int64_t nseg = (int64_t)ntiles * segs;
    const int g0 = grid_override > 0 ? grid_override : num_sms(device);
    // persistent CTAs walk whole segments (one pipeline per SM, no per-segment
    // CTA start-up; measured 5% faster than one CTA per segment)
    grid = (int)std::min<int64_t>(nseg, g0);
  } else {
    // Enough tiles for every SM: data-parallel whole tiles (no partials, no
    // fixup); otherwise stream-K so tall-skinny / few-tile products fill the chip.
    // Cost model in k-iterations on the busiest CTA: data-parallel costs
    // ⌈T/G⌉·ki; stream-K costs ⌈T·ki/G⌉ plus ≈4 k-iterations of fixup (partial
    // stores, the extra launch, the re-read).
    const int64_t g0 = grid;
    const int64_t dp_cost = ceil_div(ntiles, g0) * ki;
    const int64_t sk_cost = ceil_div(units, g0) + 4;
    const bool xm_only = size == CFG_XMT || size == CFG_XMS || size == CFG_XM1;
    if (xm_only && (amode != A_MCONTIG || epi != EPI_XM))
      throw Error(PCAL_E_STATE, "gemm: the TMEM / staged-epilogue kernels are X·[W|C] only");
    if (dp_cost <= sk_cost || xm_only) {  // gemm_xm_tmem / gemm_xm_staged: whole tiles only
      const int64_t w = ceil_div(ntiles, g0);
      upc = w * ki;
      // gemm_xm_staged walks the tiles round-robin (one CTA per SM)
      grid = (size == CFG_XMS || size == CFG_XM1) ? (int)std::min<int64_t>(ntiles, g0)
                                                  : (int)ceil_div(ntiles, w);
    } else if (epi != EPI_STORE && grid > 4 * (int64_t)ntiles) {
      // fused epilogues are fixed up one tile per CTA: keep ≤ 4 partials per tile
      grid = (int)(4 * (int64_t)ntiles);
    }
    // Tall-skinny Grams (K = n, up to 2M rows at config 5): one CTA range would
    // sum ≈ 1M rows in a single DMMA accumulator chain, whose rounding error
    // (≈ eps·√chain on the unit diagonal of XᵀX) then dominates ‖XᵀX − I‖ and the
    // CholeskyQR2 result.  Cap the chain at kGramChain k-iterations: more,
    // shorter CTA ranges (whole waves of g0), their partials summed in CTA order
    // by the fixup.  Cost: one partial tile store per range (< 0.3 % at config 5).
    if (upc == 0 && amode == A_KCONTIG && epi == EPI_STORE) {
      const char* ev = getenv("PCAL_GRAM_CHAIN");
      const int64_t kmax = ev ? atoll(ev) : 2048;
      if (kmax > 0 && ceil_div(units, (int64_t)grid) > kmax)
        grid = (int)(ceil_div(ceil_div(units, kmax), g0) * g0);
    }
  }
  // diagonal tiles of the upper-triangle-only blocks: triangular work (mma_stage_tri)
  std::vector<uint8_t> tri(ntiles, 0);
  bool any_tri = false;
  if (sym_row0 >= 0 && size == CFG_BIG && amode == A_KCONTIG && epi == EPI_STORE &&
      ci.BM == ci.BN && !getenv("PCAL_NO_TRI_TILES")) {
    for (int t = 0; t < ntiles; ++t) {
      const int64_t r0 = (int64_t)tiles[t].x * ci.BM, c0 = (int64_t)tiles[t].y * ci.BN;
      const bool d = r0 >= sym_row0 ? (r0 - sym_row0 == c0) : (sym_first && r0 == c0);
      tri[t] = d ? 1 : 0;
      any_tri |= d;
    }
  }
  // stream-K over tiles of unequal cost (triangular tiles ≈ 136/256 of a full
  // one): the CTA ranges split the WEIGHTED unit sequence evenly, so no CTA
  // waits on another's extra full tiles; explicit range starts replace ⌊c·U/G⌋
  std::vector<int64_t> cta_begin;
  // Cost of a triangular tile in units of a full one: 17 of 32 DMMAs, but
  // the full A and B panels still stream in.  Measured best with the
  // partially unrolled triangular k-loop (tools/kernel_times.py,
  // PCAL_TRI_COST sweep 0.5 … 0.9): 0.6 for configs 3 (67 % triangular
  // tiles), 4 (40 %) and 5 (22 %).
  const double kTriCost = getenv("PCAL_TRI_COST") ? atof(getenv("PCAL_TRI_COST")) : 0.6;
  if (segs > 0 && any_tri && (int64_t)grid < (int64_t)ntiles * segs) {
    // persistent CTAs over whole fixed segments (reproducible schedules): runs
    // of equal WEIGHT, not equal count — with equal counts the CTAs on
    // triangular tiles idle while the others finish (config 5 sharded: +10 %).
    // Which CTA computes a segment never changes its value.
    const int64_t nseg = (int64_t)ntiles * segs;
    std::vector<double> cum(nseg + 1, 0.0);
    for (int64_t sg = 0; sg < nseg; ++sg)
      cum[sg + 1] = cum[sg] + (tri[sg / segs] ? kTriCost : 1.0);
    cta_begin.assign(grid + 1, units);
    cta_begin[0] = 0;
    int64_t sg = 0;
    for (int c = 1; c < grid; ++c) {
      const double target = cum[nseg] * c / grid;
      while (sg < nseg && cum[sg + 1] <= target) ++sg;
      // the segment containing the target goes to whichever side holds more of it
      int64_t b = sg;
      if (sg < nseg && target - cum[sg] > 0.5 * (cum[sg + 1] - cum[sg])) b = sg + 1;
      cta_begin[c] = b >= nseg ? units : (b / segs) * ki + (b % segs) * ki / segs;
    }
    for (int c = 0; c < grid; ++c)
      if (cta_begin[c + 1] <= cta_begin[c]) {
        cta_begin.clear();
        break;
      }
  }
  if (segs == 0 && upc == 0 && any_tri) {
    std::vector<double> cum(ntiles + 1, 0.0);
    for (int t = 0; t < ntiles; ++t) cum[t + 1] = cum[t] + (tri[t] ? kTriCost : 1.0) * ki;
    cta_begin.assign(grid + 1, units);
    cta_begin[0] = 0;
    int t = 0;
    for (int c = 1; c < grid; ++c) {
      const double target = cum[ntiles] * c / grid;
      while (t < ntiles && cum[t + 1] <= target) ++t;
      if (t >= ntiles) {
        cta_begin[c] = units;
        continue;
      }
      const double per = (tri[t] ? kTriCost : 1.0);
      const int64_t within = std::min<int64_t>(ki, (int64_t)std::ceil((target - cum[t]) / per));
      cta_begin[c] = std::max<int64_t>(cta_begin[c - 1], (int64_t)t * ki + within);
    }
    // every range non-empty (a partial slot per CTA of a split tile), else
    // keep the plain equal split
    for (int c = 0; c < grid; ++c)
      if (cta_begin[c + 1] <= cta_begin[c]) {
        cta_begin.clear();
        break;
      }
  }
  auto cta_of = [&](int64_t u) -> int32_t {  // CTA whose range contains unit u
    if (cta_begin.empty()) return cta_of_unit(u, units, grid);
    return (int32_t)(std::upper_bound(cta_begin.begin(), cta_begin.end() - 1, u) -
                     cta_begin.begin() - 1);
  };
  std::vector<int32_t> tile_cta0;
  if (!cta_begin.empty()) {
    tile_cta0.resize(ntiles);
    for (int t2 = 0; t2 < ntiles; ++t2) tile_cta0[t2] = cta_of((int64_t)t2 * ki);
  }
  std::vector<int32_t> split(ntiles, -1);
  std::vector<FixupTask> tasks;
  int qmax = 1;
  if (segs > 0) {
    if (segs > 1 || chunk_partials)
      for (int t = 0; t < ntiles; ++t) {
        split[t] = t;
        tasks.push_back({t, t, segs});
      }
    qmax = segs;
  } else {
    for (int t = 0; t < ntiles && upc == 0; ++t) {
      const int32_t cf = cta_of((int64_t)t * ki);
      const int32_t cl = cta_of((int64_t)(t + 1) * ki - 1);
      if (cf != cl || chunk_partials) {
        split[t] = (int32_t)tasks.size();
        tasks.push_back({t, (int32_t)tasks.size(), cl - cf + 1});
        qmax = std::max(qmax, cl - cf + 1);
      }
    }
  }
  if (chunk_partials) qmax = std::max(qmax, qmax_min);
  PCAL_CUDA(cudaMalloc(&pl.d_tiles, sizeof(int2) * ntiles));
  PCAL_CUDA(cudaMemcpy(pl.d_tiles, tiles.data(), sizeof(int2) * ntiles, cudaMemcpyHostToDevice));
  if (any_tri) {
    PCAL_CUDA(cudaMalloc(&pl.d_tri, ntiles));
    PCAL_CUDA(cudaMemcpy(pl.d_tri, tri.data(), ntiles, cudaMemcpyHostToDevice));
  }
  if (!cta_begin.empty()) {
    PCAL_CUDA(cudaMalloc(&pl.d_cta_begin, sizeof(int64_t) * cta_begin.size()));
    PCAL_CUDA(cudaMemcpy(pl.d_cta_begin, cta_begin.data(), sizeof(int64_t) * cta_begin.size(),
                         cudaMemcpyHostToDevice));
    PCAL_CUDA(cudaMalloc(&pl.d_tile_cta0, sizeof(int32_t) * ntiles));
    PCAL_CUDA(cudaMemcpy(pl.d_tile_cta0, tile_cta0.data(), sizeof(int32_t) * ntiles,
                         cudaMemcpyHostToDevice));
  }
  PCAL_CUDA(cudaMalloc(&pl.d_split, sizeof(int32_t) * ntiles));
  PCAL_CUDA(cudaMemcpy(pl.d_split, split.data(), sizeof(int32_t) * ntiles, cudaMemcpyHostToDevice));
  pl.ntasks = (int)tasks.size();
  if (pl.ntasks) {
    PCAL_CUDA(cudaMalloc(&pl.d_tasks, sizeof(FixupTask) * pl.ntasks));
    PCAL_CUDA(cudaMemcpy(pl.d_tasks, tasks.data(), sizeof(FixupTask) * pl.ntasks,
                         cudaMemcpyHostToDevice));
    pl.ws_doubles = (size_t)pl.ntasks * qmax * ci.BM * ci.BN;
    PCAL_CUDA(cudaMalloc(&pl.ws, sizeof(double) * pl.ws_doubles));
  }
  GemmArgs& g = pl.args;
  g = GemmArgs{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.tiles = pl.d_tiles;
  g.tile_tri = pl.d_tri;
  g.cta_begin = pl.d_cta_begin;
  g.tile_cta0 = pl.d_tile_cta0;
  g.split_slot = pl.d_split;
  g.ntiles = ntiles;
  g.ki = ki;
  g.units = units;
  g.grid = grid;
  g.upc = upc;
  g.ws = pl.ws;
  g.qmax = qmax;
  g.force_ws = chunk_partials ? 1 : 0;
  g.segs = segs;
  pl.no_fixup = chunk_partials;
}

// ---- TMA descriptors ------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    PCAL_CUDA(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000,
                                               cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p)
      throw Error(PCAL_E_CUDA, "cuTensorMapEncodeTiled unavailable in the driver");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

void encode_tensor_map(CUtensorMap* m, const void* base, int rank, const int64_t* dims,
                       const int64_t* pitches_bytes, const int* box) {
  cuuint64_t d[5], st[4];
  cuuint32_t bx[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = (cuuint64_t)dims[i];
    bx[i] = (cuuint32_t)box[i];
    es[i] = 1u;
    if (i + 1 < rank) st[i] = (cuuint64_t)pitches_bytes[i];
  }
  if (reinterpret_cast<uintptr_t>(base) & 15)
    throw Error(PCAL_E_STATE, "tensor map: base not 16-byte aligned");
  const CUresult r = tensor_map_encoder()(
      m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, (cuuint32_t)rank, const_cast<void*>(base), d, st, bx, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(PCAL_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

// 2-D FP64 tensor {inner, outer} with row pitch ld (elements), box
// {box_inner, box_outer} (default {16, ·} with the 128-byte swizzle of the GEMM
// rings), zero fill outside the extents.
static void encode_map(CUtensorMap* m, const double* base, int64_t inner, int64_t outer,
                       int64_t ld, int box_outer, int box_inner = 16,
                       CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld * 8) % 16 || inner < 1 || outer < 1 ||
      inner > ld)
    throw Error(PCAL_E_STATE, "gemm: operand not TMA-addressable (16-byte aligned base / pitch)");
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)(ld * 8)};
  const cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = tensor_map_encoder()(
      m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw Error(PCAL_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
}

template <class Cfg>
static GemmMaps make_maps(const GemmArgs& g) {
  GemmMaps m;
  if (Cfg::AMODE == A_MCONTIG)
    encode_map(&m.a, g.A, g.M, g.K, g.lda, Cfg::BK);   // A(m, k) = A[m + k·lda]
  else
    encode_map(&m.a, g.A, g.K, g.M, g.lda, Cfg::BM);   // A(m, k) = A[k + m·lda]
  encode_map(&m.b, g.B, g.K, g.N, g.ldb, Cfg::BN);      // B(k, n) = B[k + n·ldb]
  return m;
}

template <class Cfg, int EPI>
static void launch_cfg(const GemmPlan& pl, cudaStream_t st) {
  static bool attr_set = false;  // per (Cfg, EPI)
  if (!attr_set) {
    PCAL_CUDA(cudaFuncSetAttribute(gemm_streamk<Cfg, EPI>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES));
    attr_set = true;
  }
  const GemmMaps maps = make_maps<Cfg>(pl.args);
  gemm_streamk<Cfg, EPI><<<pl.args.grid, Cfg::THREADS + 128, Cfg::SMEM_BYTES, st>>>(pl.args, maps);
  launched(EPI == EPI_GRAD ? "gemm_grad" : EPI == EPI_XM ? "gemm_xm" : Cfg::AMODE == A_KCONTIG ? "gemm_gram" : "gemm_store");
  PCAL_CUDA(cudaGetLastError());
  if (pl.ntasks && !pl.no_fixup) {
    if (EPI == EPI_STORE) {
      const int64_t total = (int64_t)pl.ntasks * Cfg::BM * Cfg::BN;
      gemm_fixup_store<Cfg><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(pl.args, pl.d_tasks,
                                                                            pl.ntasks);
      launched(Cfg::AMODE == A_KCONTIG ? "fixup_gram" : "fixup_store");
    } else {
      gemm_fixup<Cfg, EPI><<<pl.ntasks, Cfg::THREADS, 0, st>>>(pl.args, pl.d_tasks);
      launched(EPI == EPI_GRAD ? "fixup_grad" : "fixup_xm");
    }
    PCAL_CUDA(cudaGetLastError());
  }
}

static void launch_xm_tmem(const GemmPlan& pl, cudaStream_t st) {
  using Cfg = CfgBig<A_MCONTIG>;
  constexpr int smem = Cfg::SMEM_BYTES + 4 * 8 + 16;  // + acc_full/acc_empty, TMEM slot
  static bool attr_set = false;
  if (!attr_set) {
    PCAL_CUDA(cudaFuncSetAttribute(gemm_xm_tmem<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   smem));
    attr_set = true;
  }
  const GemmMaps maps = make_maps<Cfg>(pl.args);
  gemm_xm_tmem<Cfg><<<pl.args.grid, Cfg::THREADS + 256, smem, st>>>(pl.args, maps);
  launched("gemm_xm");
  PCAL_CUDA(cudaGetLastError());
}

static void launch_xm_staged(const GemmPlan& pl, cudaStream_t st) {
  using Cfg = CfgXms;
  constexpr int kOut = Cfg::BN / 2;
  constexpr int smem = Cfg::SMEM_BYTES + (2 * Cfg::BM * kOut + 2 * 8 * kOut) * 8 + 2 * 8;
  static_assert(smem <= 232448, "staged XM: shared memory budget");
  static bool attr_set = false;
  if (!attr_set) {
    PCAL_CUDA(cudaFuncSetAttribute(gemm_xm_staged<Cfg>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  const GemmArgs& g = pl.args;
  XmMaps maps;
  encode_map(&maps.a, g.A, g.M, g.K, g.lda, Cfg::BK);
  encode_map(&maps.b, g.B, g.K, g.N, g.ldb, Cfg::BN);
  encode_map(&maps.g, g.ep.G, g.ep.n, g.ep.p, g.ep.ld, kOut);
  encode_map(&maps.x, g.ep.X, g.ep.n, g.ep.p, g.ep.ld, kOut);
  gemm_xm_staged<Cfg><<<g.grid, Cfg::THREADS + 128, smem, st>>>(g, maps);
  launched("gemm_xm");
  PCAL_CUDA(cudaGetLastError());
}

static void launch_xm1_staged(const GemmPlan& pl, cudaStream_t st) {
  using Cfg = CfgXm1;
  constexpr int smem = Cfg::SMEM_BYTES + (2 * Cfg::BM * Cfg::BN + 2 * 4 * Cfg::BN) * 8 + 2 * 8;
  static_assert(smem <= 232448, "XM1: shared memory budget");
  static bool attr_set = false;
  if (!attr_set) {
    PCAL_CUDA(cudaFuncSetAttribute(gemm_xm1_staged<Cfg>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = true;
  }
  const GemmArgs& g = pl.args;
  XmMaps maps;
  encode_map(&maps.a, g.A, g.M, g.K, g.lda, Cfg::BK);
  encode_map(&maps.b, g.B, g.K, g.N, g.ldb, Cfg::BN);
  encode_map(&maps.g, g.ep.G, g.ep.n, g.ep.p, g.ep.ld, Cfg::BN);
  encode_map(&maps.x, g.ep.X, g.ep.n, g.ep.p, g.ep.ld, Cfg::BN);
  gemm_xm1_staged<Cfg><<<g.grid, Cfg::THREADS + 128, smem, st>>>(g, maps);
  launched("gemm_xm1");
  PCAL_CUDA(cudaGetLastError());
}

template <int AM, int EPI>
static void launch_sized(const GemmPlan& pl, cudaStream_t st) {
  if constexpr (AM == A_MCONTIG && EPI == EPI_XM) {
    if (pl.size == CFG_XMT) {
      launch_xm_tmem(pl, st);
      return;
    }
    if (pl.size == CFG_XMS) {
      launch_xm_staged(pl, st);
      return;
    }
    if (pl.size == CFG_XM1) {
      launch_xm1_staged(pl, st);
      return;
    }
  }
  switch (pl.size) {
    case CFG_BIG: launch_cfg<CfgBig<AM>, EPI>(pl, st); break;
    case CFG_MID: launch_cfg<CfgMid<AM>, EPI>(pl, st); break;
    default: launch_cfg<CfgSmall<AM>, EPI>(pl, st); break;
  }
}

void launch_gemm(const GemmPlan& pl, cudaStream_t st) {
  if (pl.amode == A_MCONTIG) {
    switch (pl.epi) {
      case EPI_STORE: launch_sized<A_MCONTIG, EPI_STORE>(pl, st); break;
      case EPI_GRAD: launch_sized<A_MCONTIG, EPI_GRAD>(pl, st); break;
      default: launch_sized<A_MCONTIG, EPI_XM>(pl, st); break;
    }
  } else {
    if (pl.epi != EPI_STORE) throw Error(PCAL_E_STATE, "gemm: K-contiguous A only with stores");
    launch_sized<A_KCONTIG, EPI_STORE>(pl, st);
  }
  (void)0;
}

void launch_gemm_tree_local(const GemmPlan& pl, const int2* nodes, int nnodes, int64_t leaf0,
                            int64_t nleaves, double* out, cudaStream_t st) {
  const CfgInfo ci = cfg_info(pl.size);
  const int tile = ci.BM * ci.BN;
  const int64_t total = (int64_t)pl.ntasks * tile;
  gemm_tree_local<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      pl.ws, pl.args.qmax, pl.ntasks, tile, nodes, nnodes, leaf0, nleaves, out, pl.args.ctl);
  launched("gram_tree_local");
  PCAL_CUDA(cudaGetLastError());
}

template <class Cfg>
static void tree_final_cfg(const GemmPlan& pl, const double* buf, const int32_t* cnt,
                           const int2* nodes, int R, int maxn, cudaStream_t st) {
  const int64_t total = (int64_t)pl.ntasks * Cfg::BM * Cfg::BN;
  gemm_tree_final<Cfg><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
      pl.args, pl.d_tasks, pl.ntasks, buf, cnt, nodes, R, maxn);
  launched("gram_tree_final");
  PCAL_CUDA(cudaGetLastError());
}

void launch_gemm_tree_final(const GemmPlan& pl, const double* buf, const int32_t* cnt,
                            const int2* nodes, int R, int maxn, cudaStream_t st) {
  if (pl.amode != A_KCONTIG || pl.epi != EPI_STORE || !pl.no_fixup)
    throw Error(PCAL_E_STATE, "gemm: tree sums need a K-contiguous chunk-partial plan");
  switch (pl.size) {
    case CFG_BIG: tree_final_cfg<CfgBig<A_KCONTIG>>(pl, buf, cnt, nodes, R, maxn, st); break;
    case CFG_MID: tree_final_cfg<CfgMid<A_KCONTIG>>(pl, buf, cnt, nodes, R, maxn, st); break;
    default: tree_final_cfg<CfgSmall<A_KCONTIG>>(pl, buf, cnt, nodes, R, maxn, st); break;
  }
}

}  // namespace pcal
