// Launch helpers shared by the host translation units.
#pragma once

#include <cstdlib>
#include <utility>

#include "zpp_internal.h"
#include "zpp_kernels.cuh"

namespace zpp {

// SM budget for the next launches on this host thread (0 = the whole GPU).
// Lets two stream-concurrent kernels (qgZ K1 of stage s+1 beside K2 of stage
// s) split the SMs instead of the first launched one taking a full wave.
inline thread_local int t_sm_cap = 0;

struct SmBudget {
  int saved;
  explicit SmBudget(int sms) : saved(t_sm_cap) { t_sm_cap = sms; }
  ~SmBudget() { t_sm_cap = saved; }
};

// SMs available to the next launch under the current budget
inline int sm_budget() { return (t_sm_cap > 0 && t_sm_cap < sm_count()) ? t_sm_cap : sm_count(); }

// Resident CTAs per SM for the next launches on this host thread (0 = the
// kernel's occupancy).  Lets two stream-concurrent persistent grids share
// every SM instead of splitting the SMs: the qwZ gather capped below its
// occupancy leaves room for one CTA of the prefetched K0 on each SM.
inline thread_local int t_occ_cap = 0;

struct OccCap {
  int saved;
  explicit OccCap(int ctas) : saved(t_occ_cap) { t_occ_cap = ctas; }
  ~OccCap() { t_occ_cap = saved; }
};

inline int occ_capped(int occ) { return (t_occ_cap > 0 && t_occ_cap < occ) ? t_occ_cap : (occ > 0 ? occ : 1); }

// ZPP_BALANCED_GRID=0 turns the balanced grid-stride sizing off (A/B)
inline bool balanced_grids() {
  static const bool v = [] {
    const char* e = getenv("ZPP_BALANCED_GRID");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Programmatic dependent launch for the communicator's kernel chains
// (K0 -> barrier -> gather, K1 -> barrier -> K2 -> barrier -> K3): under a
// PdlScope, launch_k sets cudaLaunchAttributeProgrammaticStreamSerialization,
// so each kernel's launch and CTA ramp overlap the tail of the one before it;
// every such kernel waits for its predecessor at entry (comm_aborted).
// Opt-in (ZPP_PDL=1): measured no faster on 4 B200s (qgZ bucket 2x2 195.3 vs
// 192.8 us, 1x4 130.7 vs 132.2, 2x1 258.8 vs 255.4; 40-layer qwZ forward
// 16.1 ms both; profiles/r2/pdl_ab_r2.jsonl) -- the gaps between the chain's
// kernels are barrier skew, not launch latency.
inline thread_local bool t_pdl = false;

inline bool pdl_enabled() {
  static const bool v = [] {
    const char* e = getenv("ZPP_PDL");
    return e && e[0] == '1';
  }();
  return v;
}

struct PdlScope {
  bool saved;
  explicit PdlScope(bool on) : saved(t_pdl) { t_pdl = on && pdl_enabled(); }
  ~PdlScope() { t_pdl = saved; }
};

template <typename... KArgs, typename... Args>
inline void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  if (!t_pdl) {
    k<<<grid, block, smem, st>>>(std::forward<Args>(args)...);
    return;
  }
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// one resident wave of CTAs (persistent-style grid-stride), capped by work
template <typename K>
inline int grid_for(K kernel, int threads, int64_t needed_ctas) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, 0) != cudaSuccess || occ <= 0) occ = 1;
  occ = occ_capped(occ);
  int64_t g = (int64_t)sm_budget() * occ;
  if (needed_ctas < g) {
    g = needed_ctas;
  } else if (balanced_grids()) {
    // the same number of grid-stride rounds with every CTA doing every round:
    // a small job (config 1: 1024 CTA-rounds over 296 slots) otherwise ends
    // with a round at 46% of the GPU
    const int64_t rounds = ceil_div(needed_ctas, g);
    g = ceil_div(needed_ctas, rounds);
  }
  return (int)(g < 1 ? 1 : g);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

inline int fill_table(SrcTable& t, const void* const* codes, const void* const* absmax, int n_src) {
  if (n_src < 1 || n_src > kMaxSrc) return fail(ZPP_ERR_VALIDATION, "n_src must be in [1, 64]");
  for (int i = 0; i < n_src; ++i) {
    if (!codes[i] || !absmax[i]) return fail(ZPP_ERR_VALIDATION, "null source pointer");
    t.codes[i] = reinterpret_cast<const uint8_t*>(codes[i]);
    t.absmax[i] = absmax[i];
  }
  for (int i = n_src; i < kMaxSrc; ++i) {
    t.codes[i] = nullptr;
    t.absmax[i] = nullptr;
  }
  return ZPP_OK;
}

}  // namespace zpp

#define ZPP_DISPATCH_BA_O(FN, ...)                                                                  \
  do {                                                                                              \
    if (absmax_dtype != ZPP_F32 && absmax_dtype != ZPP_F64)                                         \
      return fail(ZPP_ERR_VALIDATION, "absmax dtype must be F32 or F64");                           \
    const bool a64 = absmax_dtype == ZPP_F64;                                                       \
    switch (out_dtype) {                                                                            \
      case ZPP_F32:                                                                                 \
        if (bits == 8) return a64 ? FN<8, double, float>(__VA_ARGS__) : FN<8, float, float>(__VA_ARGS__); \
        return a64 ? FN<4, double, float>(__VA_ARGS__) : FN<4, float, float>(__VA_ARGS__);          \
      case ZPP_F16:                                                                                 \
        if (bits == 8) return a64 ? FN<8, double, __half>(__VA_ARGS__) : FN<8, float, __half>(__VA_ARGS__); \
        return a64 ? FN<4, double, __half>(__VA_ARGS__) : FN<4, float, __half>(__VA_ARGS__);        \
      case ZPP_BF16:                                                                                \
        if (bits == 8)                                                                              \
          return a64 ? FN<8, double, __nv_bfloat16>(__VA_ARGS__) : FN<8, float, __nv_bfloat16>(__VA_ARGS__); \
        return a64 ? FN<4, double, __nv_bfloat16>(__VA_ARGS__) : FN<4, float, __nv_bfloat16>(__VA_ARGS__); \
      case ZPP_F64:                                                                                 \
        if (bits == 8) return a64 ? FN<8, double, double>(__VA_ARGS__) : FN<8, float, double>(__VA_ARGS__); \
        return a64 ? FN<4, double, double>(__VA_ARGS__) : FN<4, float, double>(__VA_ARGS__);        \
    }                                                                                               \
    return fail(ZPP_ERR_VALIDATION, "unknown output dtype");                                        \
  } while (0)

