// Host launchers + C ABI for the codec kernels (K0..K4).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "zpp_internal.h"
#include "zpp_kernels.cuh"
#include "zpp_launch.cuh"

namespace zpp {

// ---------------------------------------------------------------------------
// error plumbing

static thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int check_cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ZPP_OK;
  return fail(ZPP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int sm_count() {
  static int cached = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  });
  return cached;
}

static size_t dtype_size(int dt) {
  switch (dt) {
    case ZPP_F32: return 4;
    case ZPP_F16: return 2;
    case ZPP_BF16: return 2;
    case ZPP_F64: return 8;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// K0 / K1

template <typename T, int BITS, int LANES, typename Addr, int EPL = Raw<T>::kEPL>
static int run_qreg(const T* x, const Addr& addr, int64_t n_blocks, uint8_t* codes, float* absmax, uint32_t* flag,
                    cudaStream_t st) {
  auto k = quantize_reg_kernel<T, BITS, LANES, EPL, Addr>;
  const int grid = grid_for(k, 256, ceil_div(n_blocks, 256 / LANES));
  launch_k(k, grid, 256, 0, st, x, addr, n_blocks, codes, absmax, flag, nullptr);
  return check_cuda(cudaGetLastError(), "quantize_reg_kernel launch");
}

// register path: block = LANES * Raw<T>::kEPL with LANES a power of two <= 32
template <typename T, int BITS, typename Addr>
static int dispatch_qreg(const T* x, const Addr& addr, int64_t n_blocks, int64_t block, uint8_t* codes,
                         float* absmax, uint32_t* flag, cudaStream_t st, bool* handled) {
  *handled = true;
  constexpr int64_t EPL = Raw<T>::kEPL;
  if (block == EPL) return run_qreg<T, BITS, 1>(x, addr, n_blocks, codes, absmax, flag, st);
  if (block == 2 * EPL) return run_qreg<T, BITS, 2>(x, addr, n_blocks, codes, absmax, flag, st);
  if (block == 4 * EPL) return run_qreg<T, BITS, 4>(x, addr, n_blocks, codes, absmax, flag, st);
  if (block == 8 * EPL) return run_qreg<T, BITS, 8>(x, addr, n_blocks, codes, absmax, flag, st);
  if (block == 16 * EPL) return run_qreg<T, BITS, 16>(x, addr, n_blocks, codes, absmax, flag, st);
  if (block == 32 * EPL) return run_qreg<T, BITS, 32>(x, addr, n_blocks, codes, absmax, flag, st);
  if (EPL == 32 && block == 2048) return run_qreg<T, BITS, 32, Addr, 64>(x, addr, n_blocks, codes, absmax, flag, st);
  *handled = false;
  return ZPP_OK;
}

template <typename T, int BITS, typename Addr>
static int run_qgeneric(const T* x, const Addr& addr, int64_t n_out, int64_t block, uint8_t* codes, void* absmax,
                        uint32_t* flag, cudaStream_t st) {
  using Bits = typename GenTraits<T>::Bits;
  const int64_t nb = ceil_div(n_out, block);
  const int64_t n_chunks = nb * block / 8;
  int rc = check_cuda(cudaMemsetAsync(absmax, 0, nb * sizeof(Bits), st), "absmax memset");
  if (rc) return rc;
  auto k1 = absmax_generic_kernel<T, Addr>;
  const int g1 = grid_for(k1, 256, ceil_div(n_chunks, 256));
  k1<<<g1, 256, 0, st>>>(x, addr, n_chunks, block, reinterpret_cast<Bits*>(absmax), flag);
  rc = check_cuda(cudaGetLastError(), "absmax_generic_kernel launch");
  if (rc) return rc;
  auto k2 = quantize_generic_kernel<T, BITS, Addr>;
  const int g2 = grid_for(k2, 256, ceil_div(n_chunks, 256));
  k2<<<g2, 256, 0, st>>>(x, addr, n_chunks, block, reinterpret_cast<const Bits*>(absmax), codes);
  return check_cuda(cudaGetLastError(), "quantize_generic_kernel launch");
}

template <typename T, int BITS, typename Addr>
static int quantize_t(const void* xv, const Addr& addr, int64_t n_out, int64_t block, uint8_t* codes, void* absmax,
                      uint32_t* flag, cudaStream_t st) {
  const T* x = reinterpret_cast<const T*>(xv);
  const int64_t nb = ceil_div(n_out, block);
  if constexpr (!std::is_same<T, double>::value) {
    if (aligned16(x)) {
      bool handled = false;
      int rc = dispatch_qreg<T, BITS>(x, addr, nb, block, codes, reinterpret_cast<float*>(absmax), flag, st,
                                      &handled);
      if (handled) return rc;
    }
  }
  return run_qgeneric<T, BITS>(x, addr, n_out, block, codes, absmax, flag, st);
}

template <typename Addr>
static int quantize_dispatch(const void* x, int dtype, const Addr& addr, int64_t n_out, int bits, int64_t block,
                             uint8_t* codes, void* absmax, uint32_t* flag, cudaStream_t st) {
#define ZPP_Q(T)                                                                            \
  return bits == 8 ? quantize_t<T, 8>(x, addr, n_out, block, codes, absmax, flag, st)      \
                   : quantize_t<T, 4>(x, addr, n_out, block, codes, absmax, flag, st);
  switch (dtype) {
    case ZPP_F32: ZPP_Q(float)
    case ZPP_F16: ZPP_Q(__half)
    case ZPP_BF16: ZPP_Q(__nv_bfloat16)
    case ZPP_F64: ZPP_Q(double)
  }
#undef ZPP_Q
  return fail(ZPP_ERR_VALIDATION, "unknown input dtype");
}

// quantize + write dequantize(quantize(x)) in one pass (fp16/bf16 in = out,
// register-path blocks, aligned).  Returns false when not applicable.
template <typename T, int BITS>
static bool qdeq_t(const T* x, int64_t n, int64_t block, uint8_t* codes, float* absmax, T* out, uint32_t* flag,
                   cudaStream_t st, int* rc) {
  constexpr int64_t EPL = Raw<T>::kEPL;
  const int64_t nb = ceil_div(n, block);
  PlainAddr addr{n, block};
#define ZPP_QD(L)                                                                         \
  {                                                                                       \
    auto k = quantize_reg_kernel<T, BITS, L, (int)EPL, PlainAddr, true>;                  \
    const int grid = grid_for(k, 256, ceil_div(nb, 256 / L));                             \
    launch_k(k, grid, 256, 0, st, x, addr, nb, codes, absmax, flag, out);                  \
    *rc = check_cuda(cudaGetLastError(), "quantize_reg_kernel<deq> launch");              \
    return true;                                                                          \
  }
  if (block == 8 * EPL) ZPP_QD(8)
  if (block == 16 * EPL) ZPP_QD(16)
  if (block == 32 * EPL) ZPP_QD(32)
#undef ZPP_QD
  return false;
}

int launch_quantize_deq(const void* x, int dtype, int64_t n, int bits, int64_t block, uint8_t* codes, void* absmax,
                        void* out, uint32_t* flag, cudaStream_t st, bool* handled) {
  *handled = false;
  if (n == 0 || !aligned16(x) || !aligned16(out) || n % 8 != 0) return ZPP_OK;
  int rc = ZPP_OK;
  float* am = reinterpret_cast<float*>(absmax);
  if (dtype == ZPP_F16) {
    auto xx = reinterpret_cast<const __half*>(x);
    auto oo = reinterpret_cast<__half*>(out);
    *handled = bits == 8 ? qdeq_t<__half, 8>(xx, n, block, codes, am, oo, flag, st, &rc)
                         : qdeq_t<__half, 4>(xx, n, block, codes, am, oo, flag, st, &rc);
  } else if (dtype == ZPP_BF16) {
    auto xx = reinterpret_cast<const __nv_bfloat16*>(x);
    auto oo = reinterpret_cast<__nv_bfloat16*>(out);
    *handled = bits == 8 ? qdeq_t<__nv_bfloat16, 8>(xx, n, block, codes, am, oo, flag, st, &rc)
                         : qdeq_t<__nv_bfloat16, 4>(xx, n, block, codes, am, oo, flag, st, &rc);
  }
  return rc;
}

int launch_quantize(const void* x, int dtype, const AddrSpec& a, int64_t n_out, int bits, int64_t block,
                    uint8_t* codes, void* absmax, uint32_t* flag, cudaStream_t st) {
  if (n_out == 0) return ZPP_OK;
  if (a.swizzle) {
    if (a.L / block >= (1ll << 31) || (int64_t)a.X * a.Y * (a.L / block) >= (1ll << 31))
      return fail(ZPP_ERR_VALIDATION, "qgZ bucket too large (more than 2^31 blocks)");
    SwizzleAddr addr{a.L, a.part, a.stage_off, block, a.X, a.Y, a.reorder,
                     FastDiv::make((uint32_t)(a.L / block)), FastDiv::make((uint32_t)a.Y)};
    return quantize_dispatch(x, dtype, addr, n_out, bits, block, codes, absmax, flag, st);
  }
  PlainAddr addr{a.n, block};
  return quantize_dispatch(x, dtype, addr, n_out, bits, block, codes, absmax, flag, st);
}

// K1 with the hop-1 push (quantize_push_kernel): register-path blocks only
template <typename T, int BITS, int LANES, int EPL = Raw<T>::kEPL>
static int run_qpush(const T* x, const SwizzleAddr& addr, int n_msg, int first, const PushDst& dst, uint32_t* flag,
                     cudaStream_t st) {
  auto k = quantize_push_kernel<T, BITS, LANES, EPL>;
  const int64_t tiles = ceil_div((int64_t)dst.mb.d, PushTile<LANES, EPL, BITS>::WT) * n_msg;
  const int grid = grid_for(k, 256, ceil_div(tiles, 8));
  launch_k(k, grid, 256, 0, st, x, addr, n_msg, first, dst, flag);
  return check_cuda(cudaGetLastError(), "quantize_push_kernel launch");
}

template <typename T, int BITS>
static int dispatch_qpush(const T* x, const SwizzleAddr& addr, int n_msg, int first, int64_t block,
                          const PushDst& dst, uint32_t* flag, cudaStream_t st, bool* handled) {
  *handled = true;
  constexpr int64_t EPL = Raw<T>::kEPL;
  // LANES >= 2 keeps every block's codes a 16-byte multiple (INT4, 16-bit input)
  if (block == 2 * EPL) return run_qpush<T, BITS, 2>(x, addr, n_msg, first, dst, flag, st);
  if (block == 4 * EPL) return run_qpush<T, BITS, 4>(x, addr, n_msg, first, dst, flag, st);
  if (block == 8 * EPL) return run_qpush<T, BITS, 8>(x, addr, n_msg, first, dst, flag, st);
  if (block == 16 * EPL) return run_qpush<T, BITS, 16>(x, addr, n_msg, first, dst, flag, st);
  if (block == 32 * EPL) return run_qpush<T, BITS, 32>(x, addr, n_msg, first, dst, flag, st);
  *handled = false;
  return ZPP_OK;
}

int launch_quantize_push(const void* x, int dtype, const AddrSpec& a, int64_t n_out, int bits, int64_t block,
                         uint8_t* const* dst_codes, uint8_t* const* dst_absmax, int64_t msg_blocks, int first,
                         int self_msg, uint32_t* flag, cudaStream_t st, bool* handled) {
  *handled = false;
  if (n_out == 0 || !a.swizzle || !aligned16(x) || a.X > kMaxPush) return ZPP_OK;
  if (a.L / block >= (1ll << 31) || (int64_t)a.X * a.Y * (a.L / block) >= (1ll << 31)) return ZPP_OK;
  for (int j = 0; j < a.X; ++j)
    if (!aligned16(dst_codes[j])) return ZPP_OK;
  SwizzleAddr addr{a.L, a.part, a.stage_off, block, a.X, a.Y, a.reorder,
                   FastDiv::make((uint32_t)(a.L / block)), FastDiv::make((uint32_t)a.Y)};
  PushDst d;
  for (int j = 0; j < kMaxPush; ++j) {
    d.codes[j] = j < a.X ? dst_codes[j] : nullptr;
    d.absmax[j] = j < a.X ? dst_absmax[j] : nullptr;
  }
  d.mb = FastDiv::make((uint32_t)msg_blocks);
  // ZPP_PUSH_STAGE_SELF=1 (A/B): stage and bulk-store the kept message too
  static const bool stage_self = [] {
    const char* e = getenv("ZPP_PUSH_STAGE_SELF");
    return e && e[0] == '1';
  }();
  d.self_msg = stage_self ? -1 : self_msg;
  if (ceil_div(n_out, block) != (int64_t)a.X * msg_blocks) return fail(ZPP_ERR_VALIDATION, "push: bad message size");
  const auto* xx = x;
#define ZPP_P(T)                                                                                                 \
  return bits == 8                                                                                               \
             ? dispatch_qpush<T, 8>(reinterpret_cast<const T*>(xx), addr, a.X, first, block, d, flag, st, handled) \
             : dispatch_qpush<T, 4>(reinterpret_cast<const T*>(xx), addr, a.X, first, block, d, flag, st, handled);
  switch (dtype) {
    case ZPP_F32: ZPP_P(float)
    case ZPP_F16: ZPP_P(__half)
    case ZPP_BF16: ZPP_P(__nv_bfloat16)
  }
#undef ZPP_P
  return ZPP_OK;
}

// ---------------------------------------------------------------------------
// K4 gather-dequantize and K3 dequant-reduce

template <int BITS, typename A, typename O>
static int run_gather(const SrcTable& t, int n_src, int rot, int64_t shard_len, int64_t block, void* out,
                      void* sec_out, int64_t sec_lo, int64_t sec_len, uint32_t* flag, cudaStream_t st,
                      int64_t out_stride) {
  const int vec_ok = aligned16(out) && (shard_len % 8 == 0) && (out_stride % 8 == 0) &&
                     (sec_out == nullptr || (aligned16(sec_out) && sec_lo % 8 == 0));
  constexpr bool k16 = sizeof(O) == 2 && std::is_same<A, float>::value;
  if constexpr (k16) {
    // fast 16-bit output path: one scale per 16-byte code load, aligned loads
    bool fast = block % (128 / BITS) == 0;
    for (int i = 0; i < n_src; ++i) fast = fast && aligned16(t.codes[i]);
    if (fast && n_src > 1) {
      // peers involved: TMA bulk copies of each source's codes into a 4-stage
      // shared ring hide the NVLink latency (4 x 512 units of 16 code bytes)
      constexpr int S = 4, TU = 512;
      auto k = dequant16_tma_kernel<BITS, O, S, TU>;
      const int smem = S * TU * 16 + S * 8;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, smem);
      const int64_t units = ceil_div(shard_len, 128 / BITS);
      const int grid = (int)std::min<int64_t>((int64_t)sm_budget() * occ_capped(occ), ceil_div(units, TU) * n_src);
      launch_k(k, grid, 256, smem, st, t, n_src, rot, shard_len, block, reinterpret_cast<O*>(out),
                                 reinterpret_cast<O*>(sec_out), sec_lo, sec_len, vec_ok, flag, out_stride);
      return check_cuda(cudaGetLastError(), "dequant16_tma_kernel launch");
    }
    if (fast) {
      auto k = dequant16_kernel<BITS, O>;
      const int64_t tiles = ceil_div(ceil_div(shard_len, 128 / BITS), 32 * (BITS == 8 ? 2 : 1)) * n_src;
      const int grid = grid_for(k, 256, ceil_div(tiles, 8));
      launch_k(k, grid, 256, 0, st, t, n_src, rot, shard_len, block, reinterpret_cast<O*>(out),
                              reinterpret_cast<O*>(sec_out), sec_lo, sec_len, vec_ok, flag, out_stride);
      return check_cuda(cudaGetLastError(), "dequant16_kernel launch");
    }
  }
  if constexpr (BITS == 8 && std::is_same<O, float>::value && std::is_same<A, float>::value) {
    // INT8 -> fp32 (config 1): 4-element groups, warp-contiguous stores
    bool ok = aligned16(out) && sec_out == nullptr && shard_len % 4 == 0 && (out_stride % 4 == 0);
    for (int i = 0; i < n_src; ++i) ok = ok && (reinterpret_cast<uintptr_t>(t.codes[i]) & 3) == 0;
    if (ok) {
      auto k = dequant8_f32_kernel<8>;
      const int grid = grid_for(k, 256, ceil_div(shard_len / 4, 256 * 4));
      launch_k(k, grid, 256, 0, st, t, n_src, shard_len, block, reinterpret_cast<float*>(out),
                              out_stride ? out_stride : shard_len, flag);
      return check_cuda(cudaGetLastError(), "dequant8_f32_kernel launch");
    }
  }
  if constexpr (sizeof(O) >= 4 && std::is_same<A, float>::value) {
    // fp32 / f64 outputs, whole 16-byte code units, no write-through
    constexpr int64_t E = 128 / BITS;
    bool wide = vec_ok && sec_out == nullptr && shard_len % E == 0 && block % E == 0 &&
                (out_stride == 0 || out_stride % E == 0);
    for (int i = 0; i < n_src; ++i) wide = wide && aligned16(t.codes[i]);
    if (wide) {
      auto k = dequant_wide_kernel<BITS, O>;
      const int grid = grid_for(k, 256, ceil_div(shard_len / E, 256));
      launch_k(k, grid, 256, 0, st, t, n_src, shard_len, block, reinterpret_cast<O*>(out),
                              out_stride ? out_stride : shard_len, flag);
      return check_cuda(cudaGetLastError(), "dequant_wide_kernel launch");
    }
  }
  auto k = dequant_gather_kernel<BITS, A, O>;
  const int64_t tiles = ceil_div(ceil_div(shard_len, 8), 32 * 4) * n_src;
  const int grid = grid_for(k, 256, ceil_div(tiles, 8));
  launch_k(k, grid, 256, 0, st, t, n_src, rot, shard_len, block, reinterpret_cast<O*>(out), reinterpret_cast<O*>(sec_out),
                          sec_lo, sec_len, vec_ok, flag, out_stride);
  return check_cuda(cudaGetLastError(), "dequant_gather_kernel launch");
}

int launch_gather_dequant(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src, int rot,
                          int64_t shard_len, int bits, int64_t block, void* out, int out_dtype, void* sec_out,
                          int64_t sec_lo, int64_t sec_len, uint32_t* flag, cudaStream_t st, int64_t out_stride) {
  if (shard_len == 0) return ZPP_OK;
  if (out_stride == 0) out_stride = shard_len;
  if (out_stride < shard_len) return fail(ZPP_ERR_VALIDATION, "out_stride smaller than shard_len");
  SrcTable t;
  int rc = fill_table(t, codes, absmax, n_src);
  if (rc) return rc;
  rot = ((rot % n_src) + n_src) % n_src;
  ZPP_DISPATCH_BA_O(run_gather, t, n_src, rot, shard_len, block, out, sec_out, sec_lo, sec_len, flag, st,
                    out_stride);
}

}  // namespace zpp

// ===========================================================================
// C ABI

using namespace zpp;

static int check_cfg(int bits, int64_t block) {
  if (bits != 4 && bits != 8) return fail(ZPP_ERR_CONFIG, "bit_width must be 4 or 8");
  if (block < 8 || block % 8 != 0) return fail(ZPP_ERR_CONFIG, "block_size must be a positive multiple of 8");
  return ZPP_OK;
}

static int check_dtype(int dt) {
  if (dtype_size(dt) == 0) return fail(ZPP_ERR_VALIDATION, "unknown dtype");
  return ZPP_OK;
}

extern "C" {

int zpp_version(void) { return 10000; }

const char* zpp_last_error(void) { return g_last_error.c_str(); }

int zpp_device_sm_count(void) { return sm_count(); }

int zpp_quantize(const void* x, int dtype, int64_t n, int bits, int64_t block, void* codes, void* absmax,
                 void* errflag, void* stream) {
  int rc = check_cfg(bits, block);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (n < 0) return fail(ZPP_ERR_VALIDATION, "negative length");
  if (n > 0 && (!x || !codes || !absmax)) return fail(ZPP_ERR_VALIDATION, "null pointer");
  AddrSpec a;
  a.n = n;
  return launch_quantize(x, dtype, a, n, bits, block, reinterpret_cast<uint8_t*>(codes), absmax,
                         reinterpret_cast<uint32_t*>(errflag), reinterpret_cast<cudaStream_t>(stream));
}

int zpp_swizzle_quantize(const void* grad, int dtype, int64_t n, int X, int Y, int S, int stage, int reorder, int bits,
                         int64_t block, void* codes, void* absmax, void* errflag, void* stream) {
  int rc = check_cfg(bits, block);
  if (rc || (rc = check_dtype(dtype))) return rc;
  if (X < 1 || Y < 1 || S < 1) return fail(ZPP_ERR_VALIDATION, "X, Y, S must be >= 1");
  if (stage < 0 || stage >= S) return fail(ZPP_ERR_VALIDATION, "stage out of range");
  const int64_t T = (int64_t)X * Y;
  if (n < 0 || n % (S * T)) return fail(ZPP_ERR_VALIDATION, "input length not divisible by stages*world");
  const int64_t L = n / (S * T);
  if (L % block) return fail(ZPP_ERR_VALIDATION, "slice length is not a multiple of block_size");
  if (n > 0 && (!grad || !codes || !absmax)) return fail(ZPP_ERR_VALIDATION, "null pointer");
  AddrSpec a;
  a.swizzle = true;
  a.L = L;
  a.part = (int64_t)S * L;
  a.stage_off = (int64_t)stage * L;
  a.X = X;
  a.Y = Y;
  a.reorder = reorder ? 1 : 0;
  return launch_quantize(grad, dtype, a, T * L, bits, block, reinterpret_cast<uint8_t*>(codes), absmax,
                         reinterpret_cast<uint32_t*>(errflag), reinterpret_cast<cudaStream_t>(stream));
}

int zpp_dequantize(const void* codes, const void* absmax, int absmax_dtype, int64_t n, int bits, int64_t block,
                   void* out, int out_dtype, void* errflag, void* stream) {
  int rc = check_cfg(bits, block);
  if (rc || (rc = check_dtype(out_dtype))) return rc;
  if (n < 0) return fail(ZPP_ERR_VALIDATION, "negative length");
  if (n == 0) return ZPP_OK;
  if (!out) return fail(ZPP_ERR_VALIDATION, "null pointer");
  const void* c[1] = {codes};
  const void* a[1] = {absmax};
  return launch_gather_dequant(c, a, absmax_dtype, 1, 0, n, bits, block, out, out_dtype, nullptr, 0, 0,
                               reinterpret_cast<uint32_t*>(errflag), reinterpret_cast<cudaStream_t>(stream), n);
}

int zpp_gather_dequantize(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src, int rot,
                          int64_t shard_len, int bits, int64_t block, void* out, int out_dtype, int64_t out_stride,
                          void* sec_out, int64_t sec_lo, int64_t sec_len, void* errflag, void* stream) {
  int rc = check_cfg(bits, block);
  if (rc || (rc = check_dtype(out_dtype))) return rc;
  if (shard_len < 0 || !codes || !absmax) return fail(ZPP_ERR_VALIDATION, "bad arguments");
  if (shard_len > 0 && !out) return fail(ZPP_ERR_VALIDATION, "null pointer");
  return launch_gather_dequant(codes, absmax, absmax_dtype, n_src, rot, shard_len, bits, block, out, out_dtype,
                               sec_out, sec_lo, sec_len, reinterpret_cast<uint32_t*>(errflag),
                               reinterpret_cast<cudaStream_t>(stream), out_stride);
}

int zpp_dequant_reduce(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src, int64_t n,
                       int bits, int64_t block, void* out, int out_dtype, double post_scale, void* errflag,
                       void* stream) {
  int rc = check_cfg(bits, block);
  if (rc || (rc = check_dtype(out_dtype))) return rc;
  if (n < 0 || !codes || !absmax) return fail(ZPP_ERR_VALIDATION, "bad arguments");
  if (n > 0 && !out) return fail(ZPP_ERR_VALIDATION, "null pointer");
  return launch_dequant_reduce(codes, absmax, absmax_dtype, n_src, n, bits, block, out, out_dtype, post_scale,
                               reinterpret_cast<uint32_t*>(errflag), reinterpret_cast<cudaStream_t>(stream));
}

int zpp_dequant_reduce_quant(const void* const* codes, const void* const* absmax, int absmax_dtype, int n_src,
                             int64_t n, int in_bits, int64_t in_block, int out_bits, int64_t out_block,
                             void* out_codes, void* out_absmax, void* workspace, size_t workspace_bytes,
                             void* errflag, void* stream) {
  int rc = check_cfg(in_bits, in_block);
  if (rc || (rc = check_cfg(out_bits, out_block))) return rc;
  if (n < 0 || !codes || !absmax) return fail(ZPP_ERR_VALIDATION, "bad arguments");
  if (n > 0 && (!out_codes || !out_absmax)) return fail(ZPP_ERR_VALIDATION, "null pointer");
  return launch_drq(codes, absmax, absmax_dtype, n_src, n, in_bits, in_block, out_bits, out_block,
                    reinterpret_cast<uint8_t*>(out_codes), reinterpret_cast<double*>(out_absmax), workspace,
                    workspace_bytes, reinterpret_cast<uint32_t*>(errflag), reinterpret_cast<cudaStream_t>(stream));
}

size_t zpp_drq_workspace_bytes(int64_t n, int64_t out_block) {
  if (n <= 0 || out_block < 8) return 0;
  return drq_workspace_bytes(n, out_block);
}

int zpp_scales(const void* absmax, int absmax_dtype, int64_t n_blocks, int bits, void* out_f64, void* stream) {
  if (bits != 4 && bits != 8) return fail(ZPP_ERR_CONFIG, "bit_width must be 4 or 8");
  if (n_blocks <= 0) return ZPP_OK;
  if (!absmax || !out_f64) return fail(ZPP_ERR_VALIDATION, "null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int grid = (int)std::min<int64_t>(ceil_div(n_blocks, 256), 4 * sm_count());
  double* o = reinterpret_cast<double*>(out_f64);
  if (absmax_dtype == ZPP_F32) {
    if (bits == 8) scales_kernel<8, float><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(absmax), n_blocks, o);
    else scales_kernel<4, float><<<grid, 256, 0, st>>>(reinterpret_cast<const float*>(absmax), n_blocks, o);
  } else if (absmax_dtype == ZPP_F64) {
    if (bits == 8) scales_kernel<8, double><<<grid, 256, 0, st>>>(reinterpret_cast<const double*>(absmax), n_blocks, o);
    else scales_kernel<4, double><<<grid, 256, 0, st>>>(reinterpret_cast<const double*>(absmax), n_blocks, o);
  } else {
    return fail(ZPP_ERR_VALIDATION, "absmax dtype must be F32 or F64");
  }
  return check_cuda(cudaGetLastError(), "scales_kernel launch");
}

int zpp_wire_pack(const void* codes, const void* absmax, int absmax_dtype, int64_t n, int bits, int64_t block,
                  void* out, void* stream) {
  int rc = check_cfg(bits, block);
  if (rc) return rc;
  if (n < 0 || (n > 0 && (!codes || !absmax)) || !out) return fail(ZPP_ERR_VALIDATION, "bad arguments");
  if (absmax_dtype != ZPP_F32 && absmax_dtype != ZPP_F64)
    return fail(ZPP_ERR_VALIDATION, "absmax dtype must be F32 or F64");
  const int64_t nb = ceil_div(n, block);
  const int64_t cb = code_bytes(n, bits, block);
  // '<QBI': u64 original_len, u8 bit_width, u32 block_size, little endian
  const uint64_t lo = (uint64_t)n;
  const uint64_t hi = (uint64_t)(uint8_t)bits | ((uint64_t)(uint32_t)block << 8);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nb + 13, 256), 8 * sm_count()));
  uint8_t* o = reinterpret_cast<uint8_t*>(out);
  if (absmax_dtype == ZPP_F32) {
    auto a = reinterpret_cast<const float*>(absmax);
    if (bits == 8) wire_pack_kernel<8, float><<<grid, 256, 0, st>>>(a, nb, lo, hi, o);
    else wire_pack_kernel<4, float><<<grid, 256, 0, st>>>(a, nb, lo, hi, o);
  } else {
    auto a = reinterpret_cast<const double*>(absmax);
    if (bits == 8) wire_pack_kernel<8, double><<<grid, 256, 0, st>>>(a, nb, lo, hi, o);
    else wire_pack_kernel<4, double><<<grid, 256, 0, st>>>(a, nb, lo, hi, o);
  }
  rc = check_cuda(cudaGetLastError(), "wire_pack_kernel launch");
  if (rc || cb == 0) return rc;
  return check_cuda(cudaMemcpyAsync(o + 13 + 2 * nb, codes, (size_t)cb, cudaMemcpyDeviceToDevice, st),
                    "wire codes copy");
}

int zpp_wire_unpack(const void* raw, int64_t n, int bits, int64_t block, void* codes, void* absmax_f64, void* stream) {
  int rc = check_cfg(bits, block);
  if (rc) return rc;
  if (n < 0 || !raw || (n > 0 && (!codes || !absmax_f64))) return fail(ZPP_ERR_VALIDATION, "bad arguments");
  const int64_t nb = ceil_div(n, block);
  const int64_t cb = code_bytes(n, bits, block);
  if (nb == 0) return ZPP_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nb, 256), 8 * sm_count()));
  auto r = reinterpret_cast<const uint8_t*>(raw);
  auto a = reinterpret_cast<double*>(absmax_f64);
  if (bits == 8) wire_unpack_kernel<8><<<grid, 256, 0, st>>>(r, nb, a);
  else wire_unpack_kernel<4><<<grid, 256, 0, st>>>(r, nb, a);
  rc = check_cuda(cudaGetLastError(), "wire_unpack_kernel launch");
  if (rc) return rc;
  return check_cuda(cudaMemcpyAsync(codes, r + 13 + 2 * nb, (size_t)cb, cudaMemcpyDeviceToDevice, st),
                    "wire codes copy");
}

}  // extern "C"
