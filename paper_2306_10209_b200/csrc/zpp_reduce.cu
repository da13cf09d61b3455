// Host launchers for the f64 reduce kernels: K3 (dequant -> reduce,
// BlockCodec.reduce_final, zs/collectives.py:71-75) and K2 (dequant -> reduce
// -> requant, fused_dequant_reduce_quant, zs/quantizer.py:241-258).  Each has a
// 16-element fast path (block % 16 == 0, n % 16 == 0, aligned codes) and the
// general 8-element kernels for odd block sizes and alignments.  `validate`
// turns the IntegrityError code check on (API calls) or off (internal qgZ hops,
// whose codes come from this library's own quantizer).
#include <algorithm>
#include <cstdlib>

#include "zpp_internal.h"
#include "zpp_kernels.cuh"
#include "zpp_launch.cuh"

namespace zpp {

// ZPP_NO_SPAN=1 (development A/B only): fp32 outputs of the INT4 folds in the
// per-lane layout instead of the warp-coalesced span layout
static bool span_on() {
  static const bool v = [] {
    const char* e = getenv("ZPP_NO_SPAN");
    return !(e && e[0] == '1');
  }();
  return v;
}


// ZPP_FORCE_TMA=1 (development only): route the public K2/K3 entry points to
// the TMA-fed kernels so they can be timed on local buffers.  Those kernels
// may read up to 16 bytes past each source slice, which stays inside torch's
// 512-byte allocation granules.
static bool force_tma() {
  static const bool on = [] {
    const char* e = getenv("ZPP_FORCE_TMA");
    return e && e[0] == '1';
  }();
  return on;
}

static bool codes_aligned(const SrcTable& t, int n_src, int bits) {
  for (int i = 0; i < n_src; ++i)
    if ((reinterpret_cast<uintptr_t>(t.codes[i]) % (2 * bits)) != 0) return false;
  return true;
}

// ---------------------------------------------------------------------------
// K3

// K3 fixed fan-in fast path: 2/4/8 sources, power-of-two block, fp32/f64 out
bool tbl_off();

template <int BITS, int NS, typename A, typename O>
static int run_reduce_fast(const SrcTable& t, int64_t n, int lg, void* out, double post_scale, uint32_t* flag,
                           cudaStream_t st) {
  // INT4 sources with one scale per warp tile: product tables
  auto k = (BITS == 4 && lg >= 9 && !tbl_off()) ? dr_fast_kernel<BITS, NS, A, O, BITS == 4>
                                                : dr_fast_kernel<BITS, NS, A, O, false>;
  const int grid = grid_for(k, 256, ceil_div(n / 16, 256));
  launch_k(k, grid, 256, 0, st, t, n, lg, reinterpret_cast<O*>(out), post_scale, flag, span_on() ? 1 : 0);
  return check_cuda(cudaGetLastError(), "dr_fast_kernel launch");
}

template <int BITS, typename A, typename O>
static int run_reduce(const SrcTable& t, int n_src, int64_t n, int64_t block, void* out, double post_scale,
                      bool validate, uint32_t* flag, cudaStream_t st) {
  if constexpr (sizeof(O) >= 4) {
    if (n % 16 == 0 && block % 16 == 0 && (block & (block - 1)) == 0 && aligned16(out) &&
        codes_aligned(t, n_src, BITS)) {
      const int lg = __builtin_ctzll((unsigned long long)block);
      switch (n_src) {
        case 2: return run_reduce_fast<BITS, 2, A, O>(t, n, lg, out, post_scale, flag, st);
        case 4: return run_reduce_fast<BITS, 4, A, O>(t, n, lg, out, post_scale, flag, st);
        case 8: return run_reduce_fast<BITS, 8, A, O>(t, n, lg, out, post_scale, flag, st);
        default: break;
      }
    }
  }
  if (n % 16 == 0 && block % 16 == 0 && aligned16(out) && codes_aligned(t, n_src, BITS)) {
    auto k = validate ? dequant_reduce16_kernel<BITS, A, O, true> : dequant_reduce16_kernel<BITS, A, O, false>;
    const int grid = grid_for(k, 256, ceil_div(n / 16, 256));
    launch_k(k, grid, 256, 0, st, t, n_src, n, block, reinterpret_cast<O*>(out), post_scale, flag);
    return check_cuda(cudaGetLastError(), "dequant_reduce16_kernel launch");
  }
  auto k = dequant_reduce_kernel<BITS, A, O>;
  const int grid = grid_for(k, 256, ceil_div(n, 8 * 32 * 2 * 8));
  launch_k(k, grid, 256, 0, st, t, n_src, n, block, reinterpret_cast<O*>(out), post_scale, aligned16(out), flag);
  return check_cuda(cudaGetLastError(), "dequant_reduce_kernel launch");
}

int launch_dequant_reduce(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src, int64_t n,
                          int bits, int64_t block, void* out, int out_dtype, double post_scale, uint32_t* flag,
                          cudaStream_t st, bool validate) {
  if (n == 0) return ZPP_OK;
  if (force_tma() && absmax_dtype == ZPP_F64 && post_scale == 1.0) {  // development: time the TMA K3 locally
    bool handled = false;
    int rc = launch_dr_tma(codes, absmax, n_src, n, bits, block, out, out_dtype, flag, st, &handled);
    if (rc || handled) return rc;
  }
  SrcTable t;
  int rc = fill_table(t, codes, absmax, n_src);
  if (rc) return rc;
  ZPP_DISPATCH_BA_O(run_reduce, t, n_src, n, block, out, post_scale, validate, flag, st);
}

// ---------------------------------------------------------------------------
// K2

bool drq_has_reg_path(int64_t out_block) {
  return out_block == 16 || out_block == 32 || out_block == 64 || out_block == 128 || out_block == 256 ||
         out_block == 512;
}

size_t drq_workspace_bytes(int64_t n, int64_t out_block) {
  return (size_t)(ceil_div(n, out_block) * out_block) * sizeof(double);
}

// fixed fan-in fast path (drq_fast_kernel): fp32 absmax, 512-element output
// blocks, power-of-two input blocks, 1/2/4/8 sources (the qgZ hop-1 shapes)
static bool drq_fast_ok(int n_src, int64_t n, int64_t in_block, int64_t out_block, bool a64) {
  return !a64 && out_block == 512 && n % 16 == 0 && in_block % 16 == 0 &&
         (in_block & (in_block - 1)) == 0 && (n_src == 1 || n_src == 2 || n_src == 4 || n_src == 8);
}

// ZPP_K2=est (opt-in): K2 through the certified fp32 estimate
// (drq_est_kernel) instead of the f64 product tables.  Bit-exact (tests), but
// measured slower: X = 4 62.6 vs 51.2 us, X = 2 87.2 vs 56.2 us, qgZ 2x2
// bucket 224.7 vs 194.5 us (profiles/r2/k2_est_ab_r2.jsonl): the block's
// argmax is always an absmax candidate, so every warp runs a divergent exact
// f64 fold per block, which costs more than the fp32 fold saves.
static bool k2_est_on() {
  static const bool v = [] {
    const char* e = getenv("ZPP_K2");
    return e && e[0] == 'e';
  }();
  return v;
}

// ZPP_NO_TBL=1 (development A/B only): INT4 folds without product tables
bool tbl_off() {
  static const bool off = [] {
    const char* e = getenv("ZPP_NO_TBL");
    return e && e[0] == '1';
  }();
  return off;
}

// ZPP_TBL_SPLIT=2 (development A/B only): 4-source K2 with 2 table sources
static int tbl_split() {
  static const int v = [] {
    const char* e = getenv("ZPP_TBL_SPLIT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

template <int IBITS, int OBITS, typename FO>
static int run_drq_fast(const SrcTable& t, int n_src, int64_t n, int64_t in_block, int64_t nbo, uint8_t* codes,
                        double* absmax, FO* final_out, uint32_t* flag, cudaStream_t st) {
  const int lg1 = __builtin_ctzll((unsigned long long)in_block);
  // INT4 sources with one scale per 512-element warp tile: product tables
  const bool tbl = IBITS == 4 && in_block % 512 == 0 && !tbl_off();
  // INT4 -> INT4/512 through the certified fp32 estimate (drq_est_kernel)
  // only with ZPP_K2=est (measured slower than the f64 product tables)
  constexpr bool can_est = IBITS == 4 && OBITS == 4 && (std::is_void<FO>::value || std::is_same<FO, float>::value);
  const bool est = can_est && tbl && k2_est_on();
#define ZPP_FAST(NS)                                                                            \
  {                                                                                             \
    if constexpr (can_est) {                                                                    \
      if (est) {                                                                                \
        auto k = drq_est_kernel<NS, FO>;                                                        \
        const int grid = grid_for(k, 256, ceil_div(nbo, 8));                                    \
        launch_k(k, grid, 256, 0, st, t, n, lg1, nbo, codes, absmax, flag, final_out, span_on() ? 1 : 0); \
        return check_cuda(cudaGetLastError(), "drq_est_kernel launch");                         \
      }                                                                                         \
    }                                                                                           \
    if (tbl) {                                                                                  \
      auto k = tbl_split() == 2 && NS == 4 ? drq_tbl_kernel<OBITS, NS, FO, (NS == 4 ? 2 : NS)>   \
                                             : drq_tbl_kernel<OBITS, NS, FO>;                   \
      const int grid = grid_for(k, 256, ceil_div(nbo, 8));                                      \
      launch_k(k, grid, 256, 0, st, t, n, lg1, nbo, codes, absmax, flag, final_out, span_on() ? 1 : 0, HopDst{}); \
      return check_cuda(cudaGetLastError(), "drq_tbl_kernel launch");                           \
    }                                                                                           \
    auto k = drq_fast_kernel<IBITS, OBITS, NS, FO>;                                             \
    const int grid = grid_for(k, 256, ceil_div(nbo, 8));                                        \
    launch_k(k, grid, 256, 0, st, t, n, lg1, nbo, codes, absmax, flag, final_out);                    \
    return check_cuda(cudaGetLastError(), "drq_fast_kernel launch");                            \
  }
  switch (n_src) {
    case 1: ZPP_FAST(1)
    case 2: ZPP_FAST(2)
    case 4: ZPP_FAST(4)
    case 8: ZPP_FAST(8)
  }
#undef ZPP_FAST
  return fail(ZPP_ERR_VALIDATION, "no fast K2 for this fan-in");
}

template <int IBITS, typename IA, int OBITS, int LANES>
static int run_drq(const SrcTable& t, int n_src, int64_t n, int64_t in_block, int64_t nbo, uint8_t* codes,
                   double* absmax, bool validate, uint32_t* flag, cudaStream_t st) {
  if (LANES == 32 && drq_fast_ok(n_src, n, in_block, 512, sizeof(IA) == 8) &&
      codes_aligned(t, n_src, IBITS))
    return run_drq_fast<IBITS, OBITS, void>(t, n_src, n, in_block, nbo, codes, absmax, nullptr, flag, st);
  if (n % 16 == 0 && in_block % 16 == 0 && codes_aligned(t, n_src, IBITS)) {
    auto k = validate ? drq16_kernel<IBITS, IA, OBITS, LANES, true> : drq16_kernel<IBITS, IA, OBITS, LANES, false>;
    const int grid = grid_for(k, 256, ceil_div(nbo, 256 / LANES));
    launch_k(k, grid, 256, 0, st, t, n_src, n, in_block, nbo, codes, absmax, flag, nullptr);
    return check_cuda(cudaGetLastError(), "drq16_kernel launch");
  }
  auto k = drq_reg_kernel<IBITS, IA, OBITS, LANES>;
  const int grid = grid_for(k, 256, ceil_div(nbo, 256 / LANES));
  launch_k(k, grid, 256, 0, st, t, n_src, n, in_block, nbo, codes, absmax, flag);
  return check_cuda(cudaGetLastError(), "drq_reg_kernel launch");
}

template <int IBITS, typename IA, int OBITS>
static int drq_block(const SrcTable& t, int n_src, int64_t n, int64_t in_block, int64_t out_block, uint8_t* codes,
                     double* absmax, bool validate, uint32_t* flag, cudaStream_t st) {
  const int64_t nbo = ceil_div(n, out_block);
#define ZPP_RUN(L) return run_drq<IBITS, IA, OBITS, L>(t, n_src, n, in_block, nbo, codes, absmax, validate, flag, st)
  switch (out_block) {
    case 16: ZPP_RUN(1);
    case 32: ZPP_RUN(2);
    case 64: ZPP_RUN(4);
    case 128: ZPP_RUN(8);
    case 256: ZPP_RUN(16);
    case 512: ZPP_RUN(32);
  }
#undef ZPP_RUN
  return fail(ZPP_ERR_VALIDATION, "no register path for this output block");
}

// K2 with its output pushed to the hop-2 receivers (HopDst): INT4 -> INT4/512
// through the product tables only; *handled = false otherwise.
int launch_drq_hop(const void* const* codes, const void* const* absmax, int n_src, int64_t n, int in_bits,
                   int64_t in_block, int out_bits, int64_t out_block, const HopDst& hop, uint32_t* flag,
                   cudaStream_t st, bool* handled) {
  *handled = false;
  if (n == 0 || in_bits != 4 || out_bits != 4 || out_block != 512 || in_block % 512 != 0 || tbl_off()) return ZPP_OK;
  if (n % 512 != 0 || hop.seg_blocks <= 0) return ZPP_OK;
  for (int i = 0; i < n_src; ++i)
    if (reinterpret_cast<uintptr_t>(codes[i]) % 8) return ZPP_OK;
  SrcTable t;
  int rc = fill_table(t, codes, absmax, n_src);
  if (rc) return rc;
  const int lg1 = __builtin_ctzll((unsigned long long)in_block);
  const int64_t nbo = n / 512;
#define ZPP_HOP(NS)                                                                              \
  {                                                                                              \
    auto k = drq_tbl_kernel<4, NS, void, NS, true>;                                              \
    const int grid = grid_for(k, 256, ceil_div(nbo, 8));                                         \
    launch_k(k, grid, 256, 0, st, t, n, lg1, nbo, nullptr, nullptr, flag, nullptr, 1, hop);      \
    *handled = true;                                                                             \
    return check_cuda(cudaGetLastError(), "drq_tbl_kernel<hop> launch");                         \
  }
  switch (n_src) {
    case 1: ZPP_HOP(1)
    case 2: ZPP_HOP(2)
    case 4: ZPP_HOP(4)
    case 8: ZPP_HOP(8)
  }
#undef ZPP_HOP
  return ZPP_OK;
}

int launch_drq(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src, int64_t n,
               int in_bits, int64_t in_block, int out_bits, int64_t out_block, uint8_t* out_codes,
               double* out_absmax, void* workspace, size_t ws_bytes, uint32_t* flag, cudaStream_t st,
               bool validate) {
  if (n == 0) return ZPP_OK;
  SrcTable t;
  int rc = fill_table(t, codes, absmax, n_src);
  if (rc) return rc;
  if (absmax_dtype != ZPP_F32 && absmax_dtype != ZPP_F64)
    return fail(ZPP_ERR_VALIDATION, "absmax dtype must be F32 or F64");
  if (force_tma() && absmax_dtype == ZPP_F32) {  // development: time the TMA K2 locally
    bool handled = false;
    rc = launch_drq_tma(codes, absmax, n_src, n, in_bits, in_block, out_bits, out_block, out_codes, out_absmax,
                        nullptr, 0, flag, st, &handled);
    if (rc || handled) return rc;
  }
  const bool a64 = absmax_dtype == ZPP_F64;
  bool aligned = true;  // 8-element chunk loads need 8 B (INT8) / 4 B (INT4) aligned codes
  for (int i = 0; i < n_src; ++i) aligned = aligned && (reinterpret_cast<uintptr_t>(codes[i]) % in_bits) == 0;
  if (drq_has_reg_path(out_block) && aligned) {
#define ZPP_DRQ(IB, OB)                                                                                        \
  return a64 ? drq_block<IB, double, OB>(t, n_src, n, in_block, out_block, out_codes, out_absmax, validate,  \
                                         flag, st)                                                           \
             : drq_block<IB, float, OB>(t, n_src, n, in_block, out_block, out_codes, out_absmax, validate,   \
                                        flag, st);
    if (in_bits == 8 && out_bits == 8) ZPP_DRQ(8, 8)
    if (in_bits == 8 && out_bits == 4) ZPP_DRQ(8, 4)
    if (in_bits == 4 && out_bits == 8) ZPP_DRQ(4, 8)
    ZPP_DRQ(4, 4)
#undef ZPP_DRQ
  }
  // generic: f64 fold into the workspace (K3 with f64 output), then the
  // generic f64 quantizer -- identical arithmetic, three launches.
  const size_t need = drq_workspace_bytes(n, out_block);
  if (!workspace || ws_bytes < need) return fail(ZPP_ERR_VALIDATION, "workspace too small for fused requantize");
  rc = launch_dequant_reduce(codes, absmax, absmax_dtype, n_src, n, in_bits, in_block, workspace, ZPP_F64, 1.0, flag,
                             st, validate);
  if (rc) return rc;
  AddrSpec a;
  a.n = n;
  return launch_quantize(workspace, ZPP_F64, a, n, out_bits, out_block, out_codes, out_absmax, flag, st);
}

// K2 whose hop-2 destination is itself (Y = 1): writes the final dequantized
// partition instead of codes.  Fast-path shapes only (16-element lanes,
// 512-element output blocks, validate off -- internal qgZ use).
int launch_drq_final(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src, int64_t n,
                     int in_bits, int64_t in_block, int out_bits, int64_t out_block, double* out_absmax, void* out,
                     int out_dtype, uint32_t* flag, cudaStream_t st, bool* handled) {
  *handled = false;
  if (n == 0 || out_block != 512 || n % 16 || in_block % 16 || !aligned16(out)) return ZPP_OK;
  if (out_dtype != ZPP_F32 && out_dtype != ZPP_F64) return ZPP_OK;
  SrcTable t;
  int rc = fill_table(t, codes, absmax, n_src);
  if (rc) return rc;
  if (!codes_aligned(t, n_src, in_bits)) return ZPP_OK;
  if (absmax_dtype != ZPP_F32 && absmax_dtype != ZPP_F64) return ZPP_OK;
  const int64_t nbo = ceil_div(n, out_block);
  const bool a64 = absmax_dtype == ZPP_F64;
#define ZPP_F(IB, IA, OB, FO)                                                                         \
  {                                                                                                   \
    if (drq_fast_ok(n_src, n, in_block, out_block, a64)) {                                     \
      *handled = true;                                                                                \
      return run_drq_fast<IB, OB, FO>(t, n_src, n, in_block, nbo, nullptr, out_absmax,                \
                                      reinterpret_cast<FO*>(out), flag, st);                          \
    }                                                                                                 \
    auto k = drq16_kernel<IB, IA, OB, 32, false, FO>;                                                 \
    const int grid = grid_for(k, 256, ceil_div(nbo, 8));                                              \
    launch_k(k, grid, 256, 0, st, t, n_src, n, in_block, nbo, nullptr, out_absmax, flag,                    \
                            reinterpret_cast<FO*>(out));                                              \
    *handled = true;                                                                                  \
    return check_cuda(cudaGetLastError(), "drq16_kernel<final> launch");                              \
  }
#define ZPP_FO(IB, IA, OB) \
  if (out_dtype == ZPP_F32) ZPP_F(IB, IA, OB, float) else ZPP_F(IB, IA, OB, double)
#define ZPP_FA(IB, OB) \
  if (a64) { ZPP_FO(IB, double, OB) } else { ZPP_FO(IB, float, OB) }
  if (in_bits == 4 && out_bits == 4) { ZPP_FA(4, 4) }
  if (in_bits == 8 && out_bits == 4) { ZPP_FA(8, 4) }
  if (in_bits == 4 && out_bits == 8) { ZPP_FA(4, 8) }
  if (in_bits == 8 && out_bits == 8) { ZPP_FA(8, 8) }
#undef ZPP_FA
#undef ZPP_FO
#undef ZPP_F
  return ZPP_OK;
}

// ---------------------------------------------------------------------------
// TMA-fed K2 / K3 (multi-GPU qgZ hops)

static constexpr int kTmaStages = 3;

static TmaTile tma_tile(int n_src, int bits, int64_t block, size_t abs_size) {
  TmaTile tt;
  const int ub = 2 * bits;
  // code bytes of all sources per ring stage: 12 KB measured best on 4 B200s
  // (qgZ 1x4 K2 97 us vs 103-110 at 24 KB and 124 at 48 KB; 2x2 K3 54 vs 64 us)
  static const int64_t budget = [] {
    const char* e = getenv("ZPP_TMA_STAGE_BYTES");
    return (int64_t)(e ? atoi(e) : 12288);
  }();
  int tu = 4096;
  while (tu > 32 && (int64_t)n_src * tu * ub > budget) tu >>= 1;
  tt.tu = tu;
  tt.lg = __builtin_ctzll((unsigned long long)block);
  tt.code_slot = (int)((tu * ub + 15) & ~15);
  tt.abs_slot = (int)((((int64_t)tu * 16 / block + 2) * (int64_t)abs_size + 32 + 15) & ~15);
  tt.stage_bytes = n_src * (tt.code_slot + tt.abs_slot);
  return tt;
}

template <typename K>
static int tma_grid(K k, const TmaTile& tt, int64_t tiles, size_t* smem) {
  *smem = (size_t)kTmaStages * tt.stage_bytes + kTmaStages * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)*smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, *smem);
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sm_budget() * occ_capped(occ), tiles));
}

template <int IB, int OB, int NS, typename FO>
static int run_drq_tma(const SrcTable& t, int64_t n, int64_t in_block, uint8_t* codes, double* absmax, FO* fo,
                       uint32_t* flag, cudaStream_t st) {
  const TmaTile tt = tma_tile(NS, IB, in_block, sizeof(float));
  // INT4 sources with one scale per warp tile: product tables
  constexpr bool can_span = IB == 4 && OB == 4 && std::is_same<FO, float>::value;
  const bool tbl = IB == 4 && in_block % 512 == 0 && !tbl_off();
  auto k = tbl ? (can_span && n % 512 == 0 && span_on() ? drq_tma_kernel<IB, OB, NS, FO, kTmaStages, IB == 4, can_span>
                                                       : drq_tma_kernel<IB, OB, NS, FO, kTmaStages, IB == 4>)
               : drq_tma_kernel<IB, OB, NS, FO, kTmaStages, false>;
  size_t smem = 0;
  const int grid = tma_grid(k, tt, ceil_div(n / 16, tt.tu), &smem);
  launch_k(k, grid, 256, smem, st, t, n, tt, codes, absmax, flag, fo);
  return check_cuda(cudaGetLastError(), "drq_tma_kernel launch");
}

template <int IB, int OB, typename FO>
static int drq_tma_ns(const SrcTable& t, int n_src, int64_t n, int64_t in_block, uint8_t* codes, double* absmax,
                      FO* fo, uint32_t* flag, cudaStream_t st) {
  switch (n_src) {
    case 2: return run_drq_tma<IB, OB, 2, FO>(t, n, in_block, codes, absmax, fo, flag, st);
    case 4: return run_drq_tma<IB, OB, 4, FO>(t, n, in_block, codes, absmax, fo, flag, st);
    case 8: return run_drq_tma<IB, OB, 8, FO>(t, n, in_block, codes, absmax, fo, flag, st);
  }
  return fail(ZPP_ERR_VALIDATION, "no TMA K2 for this fan-in");
}

template <typename FO>
static int drq_tma_bits(const SrcTable& t, int n_src, int64_t n, int in_bits, int64_t in_block, int out_bits,
                        uint8_t* codes, double* absmax, FO* fo, uint32_t* flag, cudaStream_t st) {
  if (in_bits == 4 && out_bits == 4) return drq_tma_ns<4, 4, FO>(t, n_src, n, in_block, codes, absmax, fo, flag, st);
  if (in_bits == 8 && out_bits == 4) return drq_tma_ns<8, 4, FO>(t, n_src, n, in_block, codes, absmax, fo, flag, st);
  if (in_bits == 4 && out_bits == 8) return drq_tma_ns<4, 8, FO>(t, n_src, n, in_block, codes, absmax, fo, flag, st);
  return drq_tma_ns<8, 8, FO>(t, n_src, n, in_block, codes, absmax, fo, flag, st);
}

int launch_drq_tma(const void* const* codes, const void* const* absmax, int n_src, int64_t n, int in_bits,
                   int64_t in_block, int out_bits, int64_t out_block, uint8_t* out_codes, double* out_absmax,
                   void* final_out, int final_dtype, uint32_t* flag, cudaStream_t st, bool* handled) {
  *handled = false;
  if (n <= 0 || n % 16 || out_block != 512 || in_block % 16 || (in_block & (in_block - 1)) ||
      !(n_src == 2 || n_src == 4 || n_src == 8))
    return ZPP_OK;
  if (final_out && final_dtype != ZPP_F32 && final_dtype != ZPP_F64) return ZPP_OK;
  SrcTable t;
  int rc = fill_table(t, codes, absmax, n_src);
  if (rc) return rc;
  for (int i = 0; i < n_src; ++i)
    if (reinterpret_cast<uintptr_t>(codes[i]) % 16) return ZPP_OK;
  *handled = true;
  if (!final_out)
    return drq_tma_bits<void>(t, n_src, n, in_bits, in_block, out_bits, out_codes, out_absmax, nullptr, flag, st);
  if (final_dtype == ZPP_F32)
    return drq_tma_bits<float>(t, n_src, n, in_bits, in_block, out_bits, nullptr, out_absmax,
                               reinterpret_cast<float*>(final_out), flag, st);
  return drq_tma_bits<double>(t, n_src, n, in_bits, in_block, out_bits, nullptr, out_absmax,
                              reinterpret_cast<double*>(final_out), flag, st);
}

template <int B, int NS, typename O>
static int run_dr_tma(const SrcTable& t, int64_t n, int64_t block, O* out, uint32_t* flag, cudaStream_t st) {
  const TmaTile tt = tma_tile(NS, B, block, sizeof(double));
  constexpr bool can_span = B == 4 && sizeof(O) == 4;
  const bool tbl = B == 4 && block % 512 == 0 && !tbl_off();
  auto k = tbl ? (can_span && n % 512 == 0 && span_on() ? dr_tma_kernel<B, NS, O, kTmaStages, B == 4, can_span>
                                                       : dr_tma_kernel<B, NS, O, kTmaStages, B == 4>)
               : dr_tma_kernel<B, NS, O, kTmaStages, false>;
  size_t smem = 0;
  const int grid = tma_grid(k, tt, ceil_div(n / 16, tt.tu), &smem);
  launch_k(k, grid, 256, smem, st, t, n, tt, out, flag);
  return check_cuda(cudaGetLastError(), "dr_tma_kernel launch");
}

template <int B, typename O>
static int dr_tma_ns(const SrcTable& t, int n_src, int64_t n, int64_t block, O* out, uint32_t* flag,
                     cudaStream_t st) {
  switch (n_src) {
    case 2: return run_dr_tma<B, 2, O>(t, n, block, out, flag, st);
    case 4: return run_dr_tma<B, 4, O>(t, n, block, out, flag, st);
    case 8: return run_dr_tma<B, 8, O>(t, n, block, out, flag, st);
  }
  return fail(ZPP_ERR_VALIDATION, "no TMA K3 for this fan-in");
}

int launch_dr_tma(const void* const* codes, const void* const* absmax_f64, int n_src, int64_t n, int bits,
                  int64_t block, void* out, int out_dtype, uint32_t* flag, cudaStream_t st, bool* handled) {
  *handled = false;
  if (n <= 0 || n % 16 || block % 16 || (block & (block - 1)) || !(n_src == 2 || n_src == 4 || n_src == 8) ||
      (out_dtype != ZPP_F32 && out_dtype != ZPP_F64) || !aligned16(out))
    return ZPP_OK;
  SrcTable t;
  int rc = fill_table(t, codes, absmax_f64, n_src);
  if (rc) return rc;
  for (int i = 0; i < n_src; ++i)
    if (reinterpret_cast<uintptr_t>(codes[i]) % 16) return ZPP_OK;
  *handled = true;
  if (out_dtype == ZPP_F32)
    return bits == 8 ? dr_tma_ns<8, float>(t, n_src, n, block, reinterpret_cast<float*>(out), flag, st)
                     : dr_tma_ns<4, float>(t, n_src, n, block, reinterpret_cast<float*>(out), flag, st);
  return bits == 8 ? dr_tma_ns<8, double>(t, n_src, n, block, reinterpret_cast<double*>(out), flag, st)
                   : dr_tma_ns<4, double>(t, n_src, n, block, reinterpret_cast<double*>(out), flag, st);
}

}  // namespace zpp
