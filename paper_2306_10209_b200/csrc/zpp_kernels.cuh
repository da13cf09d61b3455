// ZeRO++ codec kernels for sm_100a.  All are HBM/NVLink-bound streaming
// kernels (no tensor-core work exists on this path): 16-byte vector loads,
// coalesced per warp, per-block absmax by warp shuffles, grid = one resident
// wave over the 148 SMs with grid-stride loops.
//
//   K0 quantize          zs/quantizer.py:204-228   (register path + generic path)
//   K1 swizzle-quantize  zs/collectives.py:509-518 + reorder_mapping :407-417
//   K2 dequant-reduce-requant  zs/quantizer.py:241-258 (BlockCodec.fuse)
//   K3 dequant-reduce    zs/collectives.py:71-75 (BlockCodec.reduce_final)
//   K4 dequantize / gather-dequantize  zs/quantizer.py:231-238, collectives.py:264
#pragma once

#include <cfloat>
#include "zpp_common.cuh"

namespace zpp {

constexpr int kMaxSrc = 64;

// A table of (codes, absmax) sources, passed by value as a kernel parameter.
// Peer pointers (NVLink P2P) and local pointers are treated alike.
struct SrcTable {
  const uint8_t* codes[kMaxSrc];
  const void* absmax[kMaxSrc];
};

// ---------------------------------------------------------------------------
// addressing: output element o (a multiple of 8) -> source element

struct PlainAddr {
  int64_t n;
  __device__ __forceinline__ int64_t src(int64_t o) const { return o; }
  __device__ __forceinline__ int64_t valid(int64_t o) const { return n - o; }
};

// qgZ hop-1 send buffer [j][c][e]: slice k = j*Y + c holds the source slice at
// residue resid_at[k] of this stage (zs/collectives.py:509-514):
//   reorder: resid = c*X + j  (inverse of reorder_mapping(X, Y, 1))
//   else   : resid = k
struct SwizzleAddr {
  int64_t L;         // slice length
  int64_t part;      // S * L: one rank's final partition
  int64_t stage_off; // stage * L
  int X, Y;
  int reorder;
  __device__ __forceinline__ int64_t src(int64_t o) const {
    int64_t k = o / L;
    int64_t e = o - k * L;
    int64_t j = k / Y, c = k - j * Y;
    int64_t resid = reorder ? c * X + j : k;
    return resid * part + stage_off + e;
  }
  __device__ __forceinline__ int64_t valid(int64_t) const { return INT64_MAX; }
};

// ---------------------------------------------------------------------------
// raw 8-element chunks of the input types

template <typename T> struct Raw;

template <> struct Raw<__half> {
  static constexpr int W = 4;
  __device__ static void load(const __half* p, uint32_t (&r)[W]) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
  }
  __device__ static void load_scalar(const __half* p, int cnt, uint32_t (&r)[W]) {
    const uint16_t* q = reinterpret_cast<const uint16_t*>(p);
#pragma unroll
    for (int i = 0; i < W; ++i) {
      uint32_t lo = (2 * i < cnt) ? q[2 * i] : 0u;
      uint32_t hi = (2 * i + 1 < cnt) ? q[2 * i + 1] : 0u;
      r[i] = lo | (hi << 16);
    }
  }
  __device__ static uint32_t absmax_bits(const uint32_t (&r)[W], uint32_t acc) {
#pragma unroll
    for (int i = 0; i < W; ++i) acc = __vmaxu2(acc, r[i] & 0x7fff7fffu);
    return acc;
  }
  __device__ static uint32_t finish(uint32_t acc) { return max(acc & 0xffffu, acc >> 16); }
  __device__ static bool nonfinite(uint32_t m) { return m >= 0x7c00u; }
  __device__ static float m_to_float(uint32_t m) { return __half2float(__ushort_as_half((unsigned short)m)); }
  __device__ static void to_float(const uint32_t (&r)[W], float (&v)[8]) {
#pragma unroll
    for (int i = 0; i < W; ++i) {
      float2 f = __half22float2(*reinterpret_cast<const __half2*>(&r[i]));
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
};

template <> struct Raw<__nv_bfloat16> {
  static constexpr int W = 4;
  __device__ static void load(const __nv_bfloat16* p, uint32_t (&r)[W]) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
  }
  __device__ static void load_scalar(const __nv_bfloat16* p, int cnt, uint32_t (&r)[W]) {
    const uint16_t* q = reinterpret_cast<const uint16_t*>(p);
#pragma unroll
    for (int i = 0; i < W; ++i) {
      uint32_t lo = (2 * i < cnt) ? q[2 * i] : 0u;
      uint32_t hi = (2 * i + 1 < cnt) ? q[2 * i + 1] : 0u;
      r[i] = lo | (hi << 16);
    }
  }
  __device__ static uint32_t absmax_bits(const uint32_t (&r)[W], uint32_t acc) {
#pragma unroll
    for (int i = 0; i < W; ++i) acc = __vmaxu2(acc, r[i] & 0x7fff7fffu);
    return acc;
  }
  __device__ static uint32_t finish(uint32_t acc) { return max(acc & 0xffffu, acc >> 16); }
  __device__ static bool nonfinite(uint32_t m) { return m >= 0x7f80u; }
  __device__ static float m_to_float(uint32_t m) { return __uint_as_float(m << 16); }
  __device__ static void to_float(const uint32_t (&r)[W], float (&v)[8]) {
#pragma unroll
    for (int i = 0; i < W; ++i) {
      v[2 * i] = __uint_as_float(r[i] << 16);
      v[2 * i + 1] = __uint_as_float(r[i] & 0xffff0000u);
    }
  }
};

template <> struct Raw<float> {
  static constexpr int W = 8;
  __device__ static void load(const float* p, uint32_t (&r)[W]) {
    uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
    uint4 b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
    r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
    r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
  }
  __device__ static void load_scalar(const float* p, int cnt, uint32_t (&r)[W]) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
#pragma unroll
    for (int i = 0; i < W; ++i) r[i] = (i < cnt) ? q[i] : 0u;
  }
  __device__ static uint32_t absmax_bits(const uint32_t (&r)[W], uint32_t acc) {
#pragma unroll
    for (int i = 0; i < W; ++i) acc = max(acc, r[i] & 0x7fffffffu);
    return acc;
  }
  __device__ static uint32_t finish(uint32_t acc) { return acc; }
  __device__ static bool nonfinite(uint32_t m) { return m >= 0x7f800000u; }
  __device__ static float m_to_float(uint32_t m) { return __uint_as_float(m); }
  __device__ static void to_float(const uint32_t (&r)[W], float (&v)[8]) {
#pragma unroll
    for (int i = 0; i < W; ++i) v[i] = __uint_as_float(r[i]);
  }
};

// store the packed codes of one 8-element chunk
template <int BITS>
__device__ __forceinline__ void store_codes8(uint8_t* dst, const uint32_t (&b)[8]) {
  if constexpr (BITS == 8) {
    *reinterpret_cast<uint2*>(dst) = pack8_int8(b);
  } else {
    *reinterpret_cast<uint32_t*>(dst) = pack8_int4(b);
  }
}

// quantize 8 floats of one block: fp32 fast path, exact f64 redo near ties
template <int BITS>
__device__ __forceinline__ void quant8(const float (&v)[8], float inv32, double inv64, bool slow,
                                       uint32_t (&q)[8]) {
  constexpr int QMAX = Codes<BITS>::kQmax;
  bool redo = slow;
  if (!slow) {
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = q_fast(v[i], inv32, redo);
  }
  if (redo) {
#pragma unroll
    for (int i = 0; i < 8; ++i) q[i] = q_exact<QMAX>((double)v[i], inv64);
  }
}

// ---------------------------------------------------------------------------
// K0/K1 register path: a team of LANES lanes owns one quantization block of
// B = LANES * EPL elements; lane l loads 8-element chunks c*LANES + l so each
// warp-wide load instruction covers one contiguous 512 B (fp16) span.

template <typename T, int BITS, int LANES, int EPL, bool VEC, typename Addr>
__global__ void __launch_bounds__(256)
quantize_reg_kernel(const T* __restrict__ x, Addr addr, int64_t n_blocks, uint8_t* __restrict__ codes,
                    float* __restrict__ absmax, uint32_t* __restrict__ flag) {
  static_assert(EPL % 8 == 0 && 32 % LANES == 0, "team shape");
  constexpr int B = LANES * EPL;
  constexpr int CH = EPL / 8;
  constexpr int RW = Raw<T>::W;
  constexpr int QMAX = Codes<BITS>::kQmax;
  constexpr int TPW = 32 / LANES;
  const int lane = threadIdx.x & 31;
  const int tl = lane % LANES;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;

  for (int64_t wb = gwarp * TPW; wb < n_blocks; wb += nwarp * TPW) {
    const int64_t b = wb + lane / LANES;
    const bool active = b < n_blocks;
    const int64_t o0 = b * B;
    int64_t src = 0, valid = 0;
    if (active) {
      src = addr.src(o0);
      valid = addr.valid(o0);
    }
    uint32_t raw[CH][RW];
    uint32_t acc = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int e = (c * LANES + tl) * 8;
      if (VEC && active && e + 8 <= valid) {
        Raw<T>::load(x + src + e, raw[c]);
      } else {
        const int cnt = active ? (int)max((int64_t)0, min((int64_t)8, valid - e)) : 0;
        Raw<T>::load_scalar(x + src + e, cnt, raw[c]);
      }
      acc = Raw<T>::absmax_bits(raw[c], acc);
    }
    uint32_t mb = Raw<T>::finish(acc);
#pragma unroll
    for (int off = LANES / 2; off >= 1; off >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, off));
    const float m = Raw<T>::m_to_float(mb);
    if (active && tl == 0) {
      absmax[b] = m;
      if (Raw<T>::nonfinite(mb)) raise_flag(flag, FLAG_NONFINITE);
    }
    const double inv64 = m > 0.0f ? __ddiv_rn((double)QMAX, (double)m) : 0.0;
    const float inv32 = __double2float_rn(inv64);
    const bool slow = !(inv32 <= FLT_MAX);
    if (active) {
      uint8_t* out = codes + b * (int64_t)(B * BITS / 8);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float v[8];
        Raw<T>::to_float(raw[c], v);
        uint32_t q[8];
        quant8<BITS>(v, inv32, inv64, slow, q);
        store_codes8<BITS>(out + (c * LANES + tl) * BITS, q);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K0/K1 generic path (any block size, any dtype incl. f64): pass 1 reduces
// per-block absmax with atomics (bits of |x| are monotone as unsigned),
// pass 2 quantizes 8-element chunks.  8-element chunks never straddle a
// block because block % 8 == 0.

template <typename T> struct GenTraits;
template <> struct GenTraits<float> { using Bits = uint32_t; };
template <> struct GenTraits<__half> { using Bits = uint32_t; };
template <> struct GenTraits<__nv_bfloat16> { using Bits = uint32_t; };
template <> struct GenTraits<double> { using Bits = unsigned long long; };

// load 8 elements (zero beyond cnt) as doubles/floats
template <typename T>
__device__ __forceinline__ void load8_generic(const T* p, int cnt, float (&v)[8], uint32_t& bits) {
  uint32_t r[Raw<T>::W];
  Raw<T>::load_scalar(p, cnt, r);
  bits = Raw<T>::finish(Raw<T>::absmax_bits(r, 0u));
  Raw<T>::to_float(r, v);
}

template <typename T, typename Addr>
__global__ void __launch_bounds__(256)
absmax_generic_kernel(const T* __restrict__ x, Addr addr, int64_t n_chunks, int64_t B,
                      typename GenTraits<T>::Bits* __restrict__ absmax_bits, uint32_t* __restrict__ flag) {
  using Bits = typename GenTraits<T>::Bits;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t per_warp = ((n_chunks + nwarp - 1) / nwarp + 31) / 32 * 32;
  const int64_t c0 = gwarp * per_warp;
  const int64_t c1 = min(n_chunks, c0 + per_warp);
  int64_t cur = -1;
  Bits curmax = 0;
  bool bad = false;
  for (int64_t cb = c0; cb < c1; cb += 32) {
    const int64_t ch = cb + lane;
    if (ch < c1) {
      const int64_t o = ch * 8;
      const int64_t blk = o / B;
      const int64_t valid = addr.valid(o);
      const int cnt = (int)max((int64_t)0, min((int64_t)8, valid));
      Bits m;
      if constexpr (sizeof(Bits) == 8) {
        const unsigned long long* q = reinterpret_cast<const unsigned long long*>(x + addr.src(o));
        m = 0;
        for (int i = 0; i < cnt; ++i) m = max(m, q[i] & 0x7fffffffffffffffull);
        bad |= m >= 0x7ff0000000000000ull;
      } else {
        float v[8];
        uint32_t mb;
        load8_generic<T>(x + addr.src(o), cnt, v, mb);
        bad |= Raw<T>::nonfinite(mb);
        m = __float_as_uint(Raw<T>::m_to_float(mb));
      }
      if (blk != cur) {
        if (cur >= 0) atomicMax(absmax_bits + cur, curmax);
        cur = blk;
        curmax = m;
      } else {
        curmax = max(curmax, m);
      }
    }
  }
  // merge lanes that end on the same block, one atomic per distinct block
  const int64_t first = __shfl_sync(0xffffffffu, cur, 0);
  const bool same = __all_sync(0xffffffffu, cur == first);
  if (same) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      Bits o = __shfl_xor_sync(0xffffffffu, curmax, off);
      curmax = max(curmax, o);
    }
    if (lane == 0 && cur >= 0) atomicMax(absmax_bits + cur, curmax);
  } else if (cur >= 0) {
    atomicMax(absmax_bits + cur, curmax);
  }
  if (bad) raise_flag(flag, FLAG_NONFINITE);
}

template <typename T, int BITS, typename Addr>
__global__ void __launch_bounds__(256)
quantize_generic_kernel(const T* __restrict__ x, Addr addr, int64_t n_chunks, int64_t B,
                        const typename GenTraits<T>::Bits* __restrict__ absmax_bits,
                        uint8_t* __restrict__ codes) {
  constexpr int QMAX = Codes<BITS>::kQmax;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ch < n_chunks; ch += stride) {
    const int64_t o = ch * 8;
    const int64_t blk = o / B;
    const int64_t valid = addr.valid(o);
    const int cnt = (int)max((int64_t)0, min((int64_t)8, valid));
    uint32_t q[8];
    if constexpr (sizeof(typename GenTraits<T>::Bits) == 8) {
      const double m = __longlong_as_double((long long)absmax_bits[blk]);
      const double inv64 = m > 0.0 ? __ddiv_rn((double)QMAX, m) : 0.0;
      const double* p = reinterpret_cast<const double*>(x) + addr.src(o);
#pragma unroll
      for (int i = 0; i < 8; ++i) q[i] = q_exact<QMAX>(i < cnt ? p[i] : 0.0, inv64);
    } else {
      const float m = __uint_as_float(absmax_bits[blk]);
      const double inv64 = m > 0.0f ? __ddiv_rn((double)QMAX, (double)m) : 0.0;
      const float inv32 = __double2float_rn(inv64);
      float v[8];
      uint32_t mb;
      load8_generic<T>(x + addr.src(o), cnt, v, mb);
      quant8<BITS>(v, inv32, inv64, !(inv32 <= FLT_MAX), q);
    }
    store_codes8<BITS>(codes + ch * BITS, q);
  }
}

// ---------------------------------------------------------------------------
// decode helpers: one 8-element chunk of codes -> 8 exact doubles

template <int BITS>
__device__ __forceinline__ void decode8(const uint8_t* p, double s, double (&v)[8], bool& bad) {
  if constexpr (BITS == 8) {
    uint2 w = *reinterpret_cast<const uint2*>(p);
    bad |= has_byte_0x80(w.x) | has_byte_0x80(w.y);
    uint32_t u[4];
    constexpr double mb = kMagic52 + 128.0;
    unpack4_int8(w.x, u);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __dmul_rn(biased_to_f64(u[i], mb), s);
    unpack4_int8(w.y, u);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[4 + i] = __dmul_rn(biased_to_f64(u[i], mb), s);
  } else {
    uint32_t w = *reinterpret_cast<const uint32_t*>(p);
    bad |= has_nibble_8(w);
    uint32_t u[8];
    constexpr double mb = kMagic52 + 8.0;
    unpack8_int4(w, u);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __dmul_rn(biased_to_f64(u[i], mb), s);
  }
}

template <int BITS>
__device__ __forceinline__ void decode8_acc(const uint8_t* p, double s, double (&acc)[8], bool& bad) {
  double v[8];
  decode8<BITS>(p, s, v, bad);
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = __dadd_rn(acc[i], v[i]);
}

template <typename O>
__device__ __forceinline__ void store8(O* dst, const double (&v)[8], int cnt, bool vec) {
  if (vec && cnt == 8) {
    if constexpr (sizeof(O) == 2) {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        O a = from_f64<O>(v[2 * i]), b = from_f64<O>(v[2 * i + 1]);
        w[i] = (uint32_t)(*reinterpret_cast<uint16_t*>(&a)) | ((uint32_t)(*reinterpret_cast<uint16_t*>(&b)) << 16);
      }
      *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    } else if constexpr (sizeof(O) == 4) {
      float f[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = from_f64<float>(v[i]);
      reinterpret_cast<float4*>(dst)[0] = make_float4(f[0], f[1], f[2], f[3]);
      reinterpret_cast<float4*>(dst)[1] = make_float4(f[4], f[5], f[6], f[7]);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) reinterpret_cast<double2*>(dst)[i] = make_double2(v[2 * i], v[2 * i + 1]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < cnt) dst[i] = from_f64<O>(v[i]);
  }
}

// ---------------------------------------------------------------------------
// K4: dequantize / gather-dequantize.  Output = concatenation of the n_src
// sources' decoded shards (shard_len each), the qwZ receive side
// (zs/collectives.py:264).  Warps walk 32-chunk groups with the source index
// fastest-varying and rotated by `rot`, so at any moment every peer's NVLink
// egress is being read.  Optional hpZ write-through: output range
// [sec_lo, sec_lo + sec_len) is also written to sec_out (the secondary
// partition, zs/engine.py:364-367).

template <int BITS, typename A, typename O>
__global__ void __launch_bounds__(256)
dequant_gather_kernel(SrcTable src, int n_src, int rot, int64_t shard_len, int64_t B, O* __restrict__ out,
                      O* __restrict__ sec_out, int64_t sec_lo, int64_t sec_len, int vec_ok,
                      uint32_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t chunks = (shard_len + 7) / 8;
  const int64_t groups_per_src = (chunks + 31) / 32;
  const int64_t n_groups = groups_per_src * n_src;
  const bool pow2 = (B & (B - 1)) == 0;
  const int lg = pow2 ? __ffsll(B) - 1 : 0;
  bool bad = false;
  for (int64_t g = gwarp; g < n_groups; g += nwarp) {
    int s = (int)(g % n_src);
    s = (s + rot) % n_src;
    const int64_t ch = (g / n_src) * 32 + lane;
    if (ch >= chunks) continue;
    const int64_t e = ch * 8;
    const int64_t blk = pow2 ? (e >> lg) : e / B;
    const double sc = scale_of<BITS>(absmax_f64<A>(reinterpret_cast<const A*>(src.absmax[s]), blk));
    double v[8];
    decode8<BITS>(src.codes[s] + ch * BITS, sc, v, bad);
    const int cnt = (int)min((int64_t)8, shard_len - e);
    const int64_t oi = (int64_t)s * shard_len + e;
    store8<O>(out + oi, v, cnt, vec_ok);
    if (sec_out != nullptr && oi + cnt > sec_lo && oi < sec_lo + sec_len) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t k = oi + i - sec_lo;
        if (i < cnt && k >= 0 && k < sec_len) sec_out[k] = from_f64<O>(v[i]);
      }
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K3: dequantize n_src sources of n elements each and fold them in f64 from
// +0.0 in source order; optional f64 post-scale (1.0 = the reference's sum).

template <int BITS, typename A, typename O>
__global__ void __launch_bounds__(256)
dequant_reduce_kernel(SrcTable src, int n_src, int64_t n, int64_t B, O* __restrict__ out, double post_scale,
                      int vec_ok, uint32_t* __restrict__ flag) {
  const int64_t chunks = (n + 7) / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool pow2 = (B & (B - 1)) == 0;
  const int lg = pow2 ? __ffsll(B) - 1 : 0;
  bool bad = false;
  for (int64_t ch = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ch < chunks; ch += stride) {
    const int64_t e = ch * 8;
    const int64_t blk = pow2 ? (e >> lg) : e / B;
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.0;
    for (int s = 0; s < n_src; ++s) {
      const double sc = scale_of<BITS>(absmax_f64<A>(reinterpret_cast<const A*>(src.absmax[s]), blk));
      decode8_acc<BITS>(src.codes[s] + ch * BITS, sc, acc, bad);
    }
    if (post_scale != 1.0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = __dmul_rn(acc[i], post_scale);
    }
    store8<O>(out + e, acc, (int)min((int64_t)8, n - e), vec_ok);
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K2 register path: a team of LANES lanes owns one OUTPUT block of
// B2 = LANES * EPL elements; for each source (ascending) it dequantizes the
// 8-element chunks (input block size B1 arbitrary) and folds them into f64
// accumulators, then requantizes from the exact f64 block absmax.  The output
// absmax is stored in f64, so the next hop decodes bit-exactly.

template <int IBITS, typename IA, int OBITS, int LANES, int EPL>
__global__ void __launch_bounds__(256)
drq_reg_kernel(SrcTable src, int n_src, int64_t n, int64_t B1, int64_t n_blocks_out, uint8_t* __restrict__ codes,
               double* __restrict__ absmax, uint32_t* __restrict__ flag) {
  constexpr int B2 = LANES * EPL;
  constexpr int CH = EPL / 8;
  constexpr int TPW = 32 / LANES;
  constexpr int QMAX = Codes<OBITS>::kQmax;
  const int lane = threadIdx.x & 31;
  const int tl = lane % LANES;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool pow2 = (B1 & (B1 - 1)) == 0;
  const int lg = pow2 ? __ffsll(B1) - 1 : 0;
  bool bad = false;
  for (int64_t wb = gwarp * TPW; wb < n_blocks_out; wb += nwarp * TPW) {
    const int64_t b = wb + lane / LANES;
    const bool active = b < n_blocks_out;
    double acc[CH][8];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[c][i] = 0.0;
    for (int s = 0; s < n_src; ++s) {
      const IA* am = reinterpret_cast<const IA*>(src.absmax[s]);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        const int64_t e = b * B2 + (c * LANES + tl) * 8;
        if (active && e < n) {
          const int64_t ib = pow2 ? (e >> lg) : e / B1;
          const double sc = scale_of<IBITS>(absmax_f64<IA>(am, ib));
          decode8_acc<IBITS>(src.codes[s] + (e / 8) * IBITS, sc, acc[c], bad);
        }
      }
    }
    // n is a multiple of 8 except possibly in the generic fused API; zero the
    // tail of a partial chunk like the reference's zero padding
    double mx = 0.0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int64_t e = b * B2 + (c * LANES + tl) * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (e + i >= n) acc[c][i] = 0.0;
        mx = fmax(mx, fabs(acc[c][i]));
      }
    }
#pragma unroll
    for (int off = LANES / 2; off >= 1; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (active && tl == 0) {
      absmax[b] = mx;
      if (!(mx <= DBL_MAX)) raise_flag(flag, FLAG_NONFINITE);
    }
    const double inv = mx > 0.0 ? __ddiv_rn((double)QMAX, mx) : 0.0;
    if (active) {
      uint8_t* out = codes + b * (int64_t)(B2 * OBITS / 8);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        uint32_t q[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) q[i] = q_exact<QMAX>(acc[c][i], inv);
        store_codes8<OBITS>(out + (c * LANES + tl) * OBITS, q);
      }
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// f64 scales from absmax (QuantizedTensor.scales; zs/quantizer.py:219)
template <int BITS, typename A>
__global__ void scales_kernel(const A* __restrict__ absmax, int64_t nb, double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += stride)
    out[i] = scale_of<BITS>(absmax_f64<A>(absmax, i));
}

}  // namespace zpp
