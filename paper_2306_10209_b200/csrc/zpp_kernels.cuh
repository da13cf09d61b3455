// ZeRO++ codec kernels for sm_100a.  All are HBM/NVLink-bound streaming
// kernels (no tensor-core work exists on this path).  Design rules, from ncu
// on B200: keep every lane >= 64-128 B of loads in flight, keep registers
// <= ~64 for >= 50% occupancy, and spend < ~6 ALU + ~6 FMA-pipe thread
// instructions per element (the ALU and FMA pipes each take a warp
// instruction every 2 cycles per SMSP).  The inner loops therefore use
// Blackwell's packed fp32x2 FFMA2/FADD2/FMUL2 and HMNMX2, and fall back to
// exact f64 arithmetic only for elements an error bound cannot decide.
//
//   K0 quantize          zs/quantizer.py:204-228   (register path + generic path)
//   K1 swizzle-quantize  zs/collectives.py:509-518 + reorder_mapping :407-417
//   K2 dequant-reduce-requant  zs/quantizer.py:241-258 (BlockCodec.fuse)
//   K3 dequant-reduce    zs/collectives.py:71-75 (BlockCodec.reduce_final)
//   K4 dequantize / gather-dequantize  zs/quantizer.py:231-238, collectives.py:264
#pragma once

#include <cfloat>
#include <type_traits>
#include "zpp_common.cuh"

namespace zpp {

constexpr int kMaxSrc = 64;

// A table of (codes, absmax) sources, passed by value as a kernel parameter.
// Peer pointers (NVLink P2P) and local pointers are treated alike.
struct SrcTable {
  const uint8_t* codes[kMaxSrc];
  const void* absmax[kMaxSrc];
  __device__ __forceinline__ const uint8_t* code_ptr(int s) const { return codes[s]; }
  __device__ __forceinline__ const void* abs_ptr(int s) const { return absmax[s]; }
};

// ---------------------------------------------------------------------------
// addressing: where the input of output block b / output element o lives

struct PlainAddr {
  int64_t n;
  int64_t B;
  __device__ __forceinline__ int64_t block_src(int64_t b) const { return b * B; }
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
  int64_t B;
  int X, Y;
  int reorder;
  FastDiv bps;       // blocks per slice (L / B)
  FastDiv fy;        // Y
  __device__ __forceinline__ int64_t resid_of(int64_t k) const {
    const int64_t j = fy.div((uint32_t)k), c = k - j * Y;
    return reorder ? c * X + j : k;
  }
  __device__ __forceinline__ int64_t block_src(int64_t b) const {
    const int64_t k = bps.div((uint32_t)b);
    const int64_t eb = b - k * (int64_t)bps.d;
    return resid_of(k) * part + stage_off + eb * B;
  }
  __device__ __forceinline__ int64_t src(int64_t o) const {
    const int64_t k = o / L;
    return resid_of(k) * part + stage_off + (o - k * L);
  }
  __device__ __forceinline__ int64_t valid(int64_t) const { return INT64_MAX; }
};

// ---------------------------------------------------------------------------
// raw 8-element chunks of the input types

template <typename T> struct Raw;

template <> struct Raw<__half> {
  static constexpr int W = 4;
  static constexpr int kEPL = 64;  // elements per lane in the register path
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
  // running max of |x| over packed pairs (NaN-propagating); sign bits garbage
  __device__ static uint32_t absacc(const uint32_t (&r)[W], uint32_t acc) {
    return absmax_f16x2(acc, absmax_f16x2(absmax_f16x2(r[0], r[1]), absmax_f16x2(r[2], r[3])));
  }
  __device__ static uint32_t finish(uint32_t acc) {
    acc &= 0x7fff7fffu;
    return max(acc & 0xffffu, acc >> 16);
  }
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
  static constexpr int kEPL = 64;
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
  __device__ static uint32_t absacc(const uint32_t (&r)[W], uint32_t acc) {
    return absmax_bf16x2(acc, absmax_bf16x2(absmax_bf16x2(r[0], r[1]), absmax_bf16x2(r[2], r[3])));
  }
  __device__ static uint32_t finish(uint32_t acc) {
    acc &= 0x7fff7fffu;
    return max(acc & 0xffffu, acc >> 16);
  }
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
  static constexpr int kEPL = 32;
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
  __device__ static uint32_t absacc(const uint32_t (&r)[W], uint32_t acc) {
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

// Fast 16-bit output of a unit: p = RN32(code * s32) with s32 = RN32(m * RN32(1/q))
// is within 3 fp32 ulps of the exact f64 product code*s64, so RN16(p) equals
// RN16(RN64(code*s64)) unless p lies within 64 ulps of a 16-bit rounding
// midpoint; the unit is then redone in f64.  Out-of-range scales (16-bit
// subnormal results, overflow) take the f64 path up front.
template <typename O> struct Out16;
template <> struct Out16<__half> {
  // zero iff the 13 bits below the fp16 mantissa are within [-64, +64) of 0x1000
  __device__ static uint32_t near_mid(uint32_t bits) { return ((bits + 0x40u) & 0x1F80u) ^ 0x1000u; }
  __device__ static bool scale_ok(float s, int qmax) { return s >= 0x1p-14f && s * (float)qmax < 65504.0f; }
  static constexpr uint32_t kLowMask = 0x1FFFu;  // absmax has <= 11 significant bits
  __device__ static bool in_range(float m) { return m <= 65504.0f; }
  __device__ static uint32_t pack2(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};
template <> struct Out16<__nv_bfloat16> {
  __device__ static uint32_t near_mid(uint32_t bits) { return ((bits + 0x40u) & 0xFF80u) ^ 0x8000u; }
  __device__ static bool scale_ok(float s, int qmax) { return s >= 0x1p-125f && s * (float)qmax < 0x1p127f; }
  static constexpr uint32_t kLowMask = 0xFFFFu;  // absmax has <= 8 significant bits
  __device__ static bool in_range(float m) { return m >= 0x1p-100f && m < 0x1p127f; }
  __device__ static uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
};

// Quantize one chunk of 8 floats.  Fast path (fp32, packed):
//   u = RN(x*inv32 + 1.5*2^23) = 1.5*2^23 + k with k = rint(x*inv32)  (FFMA2)
//   e = RN(x*inv32 - k)                                                (FFMA2)
// With inv32 = RN32(qmax/m), |x*inv32 - RN64(x*RN64(qmax/m))| < 7.6e-6 and
// |e - (x*inv32 - k)| <= 2^-25, so |e| <= 0.5 - 2^-15 proves k equals the
// reference's rint of the f64 product.  Elements failing that test (near or
// exact ties: ~0.3% of bf16 inputs, whose 8-bit mantissas make exact ties
// common) are recomputed with the reference's f64 arithmetic, element by
// element.  The low byte of each returned word is the code in two's complement.
template <int QMAX>
__device__ __forceinline__ void quant_chunk(const float (&v)[8], float inv32, double inv64, uint32_t (&q)[8]) {
  const float2 inv2 = make_float2(inv32, inv32);
  const float2 m2 = make_float2(kMagic23, kMagic23);
  float e[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = make_float2(v[2 * i], v[2 * i + 1]);
    const float2 u = ffma2(x, inv2, m2);
    float2 nk;
    asm("sub.rn.f32x2 %0, %1, %2;"
        : "=l"(*reinterpret_cast<unsigned long long*>(&nk))
        : "l"(*reinterpret_cast<const unsigned long long*>(&m2)), "l"(*reinterpret_cast<const unsigned long long*>(&u)));
    const float2 ee = ffma2(x, inv2, nk);
    e[2 * i] = ee.x;
    e[2 * i + 1] = ee.y;
    q[2 * i] = __float_as_uint(u.x);
    q[2 * i + 1] = __float_as_uint(u.y);
  }
  const float emax = fmaxf(fmaxf(fmaxf(fabsf(e[0]), fabsf(e[1])), fmaxf(fabsf(e[2]), fabsf(e[3]))),
                           fmaxf(fmaxf(fabsf(e[4]), fabsf(e[5])), fmaxf(fabsf(e[6]), fabsf(e[7]))));
  if (emax > kTieGuard) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (fabsf(e[i]) > kTieGuard) q[i] = (uint32_t)rint_f64(__dmul_rn((double)v[i], inv64));
  }
}

// Fast part of quant_chunk only: returns true when some element is a near or
// exact tie whose code must be recomputed with the reference's f64 arithmetic
// (the caller redoes that chunk later, see quant_team).
template <int QMAX>
__device__ __forceinline__ bool quant_chunk_fast(const float (&v)[8], float inv32, uint32_t (&q)[8]) {
  const float2 inv2 = make_float2(inv32, inv32);
  const float2 m2 = make_float2(kMagic23, kMagic23);
  float e[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = make_float2(v[2 * i], v[2 * i + 1]);
    const float2 u = ffma2(x, inv2, m2);
    float2 nk;
    asm("sub.rn.f32x2 %0, %1, %2;"
        : "=l"(*reinterpret_cast<unsigned long long*>(&nk))
        : "l"(*reinterpret_cast<const unsigned long long*>(&m2)), "l"(*reinterpret_cast<const unsigned long long*>(&u)));
    const float2 ee = ffma2(x, inv2, nk);
    e[2 * i] = ee.x;
    e[2 * i + 1] = ee.y;
    q[2 * i] = __float_as_uint(u.x);
    q[2 * i + 1] = __float_as_uint(u.y);
  }
  const float emax = fmaxf(fmaxf(fmaxf(fabsf(e[0]), fabsf(e[1])), fmaxf(fabsf(e[2]), fabsf(e[3]))),
                           fmaxf(fmaxf(fabsf(e[4]), fabsf(e[5])), fmaxf(fabsf(e[6]), fabsf(e[7]))));
  return emax > kTieGuard;
}

// ---------------------------------------------------------------------------
// K0/K1 register path: a team of LANES lanes owns one quantization block of
// B = LANES * EPL elements (EPL = 64 for 16-bit inputs, 32 for fp32, so each
// lane issues eight 16-byte loads before reducing); lane l loads 8-element
// chunks c*LANES + l, so each team-wide load covers one contiguous span of
// >= 128 B.

// DEQ = true additionally writes dequantize(quantize(x)) to deq_out (same
// 16-bit type as the input): the qwZ self-gather of a 1-GPU world in one pass
// (5 instead of 6 bytes of HBM traffic per element).  For fp16/bf16 sources
// the block absmax fits the output significand, so by the exact16 argument
// (see decode16_any) the fp32 product rounds to the reference's value.
// One team of LANES lanes quantizes output block b (EPL elements per lane).
// Shared by the K0/K1 grid-stride kernel and the fused qgZ kernel.
#ifndef ZPP_DEQ_FAST_LOOP
#define ZPP_DEQ_FAST_LOOP 1
#endif
constexpr bool kDeqFastLoop = ZPP_DEQ_FAST_LOOP;

// The loaded input of one team block: raw 16-byte chunks plus where it came from.
template <typename T, int EPL>
struct TeamIn {
  uint32_t raw[EPL / 8][Raw<T>::W];
  int64_t src, valid;
};

template <typename T, int LANES, int EPL, typename Addr>
__device__ __forceinline__ void quant_load(const T* __restrict__ x, const Addr& addr, int64_t b, bool active, int tl,
                                           TeamIn<T, EPL>& in) {
  constexpr int B = LANES * EPL;
  constexpr int CH = EPL / 8;
  int64_t src = 0, valid = 0;
  if (active) {
    src = addr.block_src(b);
    valid = addr.valid(b * B);
  }
  in.src = src;
  in.valid = valid;
  auto& raw = in.raw;
  if (active && valid >= B) {  // full block: unconditional vector loads
    const T* xb = x + src + tl * 8;
#pragma unroll
    for (int c = 0; c < CH; ++c) Raw<T>::load(xb + c * LANES * 8, raw[c]);
  } else {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int e = (c * LANES + tl) * 8;
      if (active && e + 8 <= valid) {
        Raw<T>::load(x + src + e, raw[c]);
      } else {
        const int cnt = active ? (int)max((int64_t)0, min((int64_t)8, valid - e)) : 0;
        Raw<T>::load_scalar(x + src + e, cnt, raw[c]);
      }
    }
  }
}

template <typename T, int BITS, int LANES, int EPL, bool DEQ>
__device__ __forceinline__ void quant_compute(const T* __restrict__ x, const TeamIn<T, EPL>& in, int64_t b,
                                              bool active, int tl, uint8_t* __restrict__ codes,
                                              float* __restrict__ absmax, uint32_t* __restrict__ flag,
                                              T* __restrict__ deq_out) {
  constexpr int B = LANES * EPL;
  constexpr int CH = EPL / 8;
  constexpr int RW = Raw<T>::W;
  constexpr int QMAX = Codes<BITS>::kQmax;
  const auto& raw = in.raw;
  const int64_t src = in.src, valid = in.valid;
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc = Raw<T>::absacc(raw[c], acc);
  uint32_t mb = Raw<T>::finish(acc);
#pragma unroll
  for (int off = LANES / 2; off >= 1; off >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, off));
  const float m = Raw<T>::m_to_float(mb);
  if (active && tl == 0) {
    absmax[b] = m;
    if (Raw<T>::nonfinite(mb)) raise_flag(flag, FLAG_NONFINITE);
  }
  const float inv32 = m > 0.0f ? __fdiv_rn((float)QMAX, m) : 0.0f;
  const bool slow = !(inv32 <= 0x1p100f);  // reciprocal of a (sub)normal tiny absmax
  // Without the fused dequantize, chunks holding a near tie are redone after
  // the chunk loop: a lane loops only over its own flagged chunks (~2% of
  // bf16 chunks), so a warp runs ~1.4 exact redos per block instead of
  // diverging into the f64 path at every chunk where any lane has a tie; the
  // f64 reciprocal (a long dependent chain) is then only computed for them.
  constexpr bool DEFER = !DEQ;
  auto inv64_of = [&]() { return m > 0.0f ? __ddiv_rn((double)QMAX, (double)m) : 0.0; };
  const double inv64 = (DEFER && !slow) ? 0.0 : inv64_of();
  uint8_t* out = codes + b * (int64_t)(B * BITS / 8);
  uint32_t need = 0;
  // warp-uniform fast loop when no team of the warp has a tiny absmax: no
  // per-chunk branch on `slow` (each costs a BSSY/BSYNC pair in SASS).  INT4
  // only: K1 69.8 -> 66.7 us; the INT8 K0 grows from 116 to 128 registers
  // and loses 5%.
  bool general = true;
  if constexpr (DEFER && BITS == 4) {
    if (!__any_sync(0xffffffffu, slow)) {
      general = false;
      if (__all_sync(0xffffffffu, active)) {
        // every team of the warp holds a block (all but the grid's last
        // wave): unconditional stores from one hoisted base address, no
        // per-chunk branch region
        uint8_t* const ob = out + tl * BITS;
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          float v[8];
          uint32_t q[8];
          Raw<T>::to_float(raw[c], v);
          if (quant_chunk_fast<QMAX>(v, inv32, q)) need |= 1u << c;
          store_codes8<BITS>(ob + c * LANES * BITS, q);
        }
      } else {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          float v[8];
          uint32_t q[8];
          Raw<T>::to_float(raw[c], v);
          if (quant_chunk_fast<QMAX>(v, inv32, q)) need |= 1u << c;
          if (active) store_codes8<BITS>(out + (c * LANES + tl) * BITS, q);
        }
      }
    }
  }
  if constexpr (DEQ && kDeqFastLoop) {
    // the fused N = 1 qwZ pass: one warp-uniform loop when every team has a
    // normal absmax that fits the 16-bit output, and the whole warp's chunks
    // are full (all but the last, ragged block of the input)
    const bool full = active && valid >= B && !slow && Out16<T>::in_range(m);
    if (__all_sync(0xffffffffu, full)) {
      general = false;
      const float s32 = __fmul_rn(m, 1.0f / QMAX);
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float v[8];
        uint32_t q[8];
        Raw<T>::to_float(raw[c], v);
        quant_chunk<QMAX>(v, inv32, inv64, q);
        store_codes8<BITS>(out + (c * LANES + tl) * BITS, q);
        uint32_t h[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float c0 = (float)(int)(int8_t)(q[2 * i] & 0xFFu);
          const float c1 = (float)(int)(int8_t)(q[2 * i + 1] & 0xFFu);
          const float2 p = fmul2(make_float2(c0, c1), make_float2(s32, s32));
          h[i] = Out16<T>::pack2(p.x, p.y);
        }
        *reinterpret_cast<uint4*>(deq_out + b * (int64_t)B + (c * LANES + tl) * 8) = make_uint4(h[0], h[1], h[2], h[3]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CH && general; ++c) {
    float v[8];
    uint32_t q[8];
    Raw<T>::to_float(raw[c], v);
    if (!slow) {
      if constexpr (DEFER) {
        if (quant_chunk_fast<QMAX>(v, inv32, q)) need |= 1u << c;
      } else {
        quant_chunk<QMAX>(v, inv32, inv64, q);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) q[i] = q_exact<QMAX>((double)v[i], inv64);
    }
    if (active) store_codes8<BITS>(out + (c * LANES + tl) * BITS, q);
    if constexpr (DEQ) {
      if (active) {
        // code as an exact float: the low byte of q is the two's complement code
        const float s32 = __fmul_rn(m, 1.0f / QMAX);
        const bool ok16 = Out16<T>::in_range(m);
        uint32_t h[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float c0 = (float)(int)(int8_t)(q[2 * i] & 0xFFu);
          const float c1 = (float)(int)(int8_t)(q[2 * i + 1] & 0xFFu);
          if (ok16) {
            const float2 p = fmul2(make_float2(c0, c1), make_float2(s32, s32));
            h[i] = Out16<T>::pack2(p.x, p.y);
          } else {
            const double s64 = scale_of<BITS>((double)m);
            T a = from_f64<T>(__dmul_rn((double)c0, s64)), bb = from_f64<T>(__dmul_rn((double)c1, s64));
            h[i] = (uint32_t)(*reinterpret_cast<uint16_t*>(&a)) | ((uint32_t)(*reinterpret_cast<uint16_t*>(&bb)) << 16);
          }
        }
        const int e = (c * LANES + tl) * 8;
        T* dst = deq_out + b * (int64_t)B + e;
        if (e + 8 <= valid) {
          *reinterpret_cast<uint4*>(dst) = make_uint4(h[0], h[1], h[2], h[3]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (e + i < valid) reinterpret_cast<uint16_t*>(dst)[i] = (uint16_t)(h[i / 2] >> (16 * (i & 1)));
        }
      }
    }
  }
  if constexpr (DEFER) {
    const double inv64r = need ? inv64_of() : 0.0;
    while (need) {  // exact redo of this lane's flagged chunks (reference arithmetic)
      const int c = __ffs(need) - 1;
      need &= need - 1;
      const int e = (c * LANES + tl) * 8;
      uint32_t r[RW];
      if (e + 8 <= valid) {
        Raw<T>::load(x + src + e, r);
      } else {
        Raw<T>::load_scalar(x + src + e, (int)max((int64_t)0, min((int64_t)8, valid - e)), r);
      }
      float v[8];
      uint32_t q[8];
      Raw<T>::to_float(r, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) q[i] = (uint32_t)rint_f64(__dmul_rn((double)v[i], inv64r));
      store_codes8<BITS>(out + e * BITS / 8, q);
    }
  }
}

template <typename T, int BITS, int LANES, int EPL, typename Addr, bool DEQ>
__device__ __forceinline__ void quant_team(const T* __restrict__ x, const Addr& addr, int64_t b, bool active, int tl,
                                           uint8_t* __restrict__ codes, float* __restrict__ absmax,
                                           uint32_t* __restrict__ flag, T* __restrict__ deq_out) {
  TeamIn<T, EPL> in;
  quant_load<T, LANES, EPL, Addr>(x, addr, b, active, tl, in);
  quant_compute<T, BITS, LANES, EPL, DEQ>(x, in, b, active, tl, codes, absmax, flag, deq_out);
}

template <typename T, int BITS, int LANES, int EPL, typename Addr, bool DEQ = false>
__global__ void __launch_bounds__(256)
quantize_reg_kernel(const T* __restrict__ x, Addr addr, int64_t n_blocks, uint8_t* __restrict__ codes,
                    float* __restrict__ absmax, uint32_t* __restrict__ flag, T* __restrict__ deq_out = nullptr) {
  if (comm_aborted(flag)) return;
  static_assert(32 % LANES == 0 && EPL % 8 == 0, "team shape");
  constexpr int TPW = 32 / LANES;
  const int lane = threadIdx.x & 31;
  const int tl = lane % LANES;
  const int team = lane / LANES;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // INT8 (qwZ K0): software-pipelined, measured 673 -> 619 us (89% -> 96.5% of
  // the copy peak) on a 1.3B fp16 buffer.  INT4 (qgZ K1, more ALU work per
  // byte) keeps the single buffer: the pipelined version's 116 registers halve
  // occupancy and measured 68 -> 74 us (16 lanes x 32 elements, 78
  // registers: 78 us).
  // The pipeline keeps two input buffers live: only when one buffer is at
  // most 32 registers (fp16/bf16 x 64, fp32 x 32).  fp32 x 64 (config 1's
  // INT8/2048 blocks) pipelined took 170 registers, one CTA per SM and 45% of
  // the DRAM peak.
  constexpr bool PIPE = !DEQ && BITS == 8 && sizeof(T) * EPL <= 128;
  if constexpr (!PIPE) {
    for (int64_t wb = gwarp * TPW; wb < n_blocks; wb += nwarp * TPW) {
      const int64_t b = wb + team;
      quant_team<T, BITS, LANES, EPL, Addr, DEQ>(x, addr, b, b < n_blocks, tl, codes, absmax, flag, deq_out);
    }
  } else {
    // software pipeline: the next block's chunks are loaded before this block
    // is quantized (two register buffers, alternating), so every warp keeps a
    // block of loads in flight while it computes
    const int64_t step = nwarp * TPW;
    TeamIn<T, EPL> bufA, bufB;
    int64_t b = gwarp * TPW + team;
    quant_load<T, LANES, EPL, Addr>(x, addr, b, b < n_blocks, tl, bufA);
    for (int64_t wb = gwarp * TPW; wb < n_blocks; wb += 2 * step) {
      quant_load<T, LANES, EPL, Addr>(x, addr, b + step, b + step < n_blocks, tl, bufB);
      quant_compute<T, BITS, LANES, EPL, false>(x, bufA, b, b < n_blocks, tl, codes, absmax, flag, nullptr);
      b += step;
      if (wb + step >= n_blocks) break;
      quant_load<T, LANES, EPL, Addr>(x, addr, b + step, b + step < n_blocks, tl, bufA);
      quant_compute<T, BITS, LANES, EPL, false>(x, bufB, b, b < n_blocks, tl, codes, absmax, flag, nullptr);
      b += step;
    }
  }
}

// ---------------------------------------------------------------------------
// K0/K1 generic path (any block size, any dtype incl. f64, any alignment):
// pass 1 reduces per-block absmax with atomics (bits of |x| are monotone as
// unsigned), pass 2 quantizes 8-element chunks.  8-element chunks never
// straddle a block because block % 8 == 0.

template <typename T> struct GenTraits;
template <> struct GenTraits<float> { using Bits = uint32_t; };
template <> struct GenTraits<__half> { using Bits = uint32_t; };
template <> struct GenTraits<__nv_bfloat16> { using Bits = uint32_t; };
template <> struct GenTraits<double> { using Bits = unsigned long long; };

template <typename T>
__device__ __forceinline__ void load8_generic(const T* p, int cnt, float (&v)[8], uint32_t& bits) {
  uint32_t r[Raw<T>::W];
  Raw<T>::load_scalar(p, cnt, r);
  bits = Raw<T>::finish(Raw<T>::absacc(r, 0u));
  Raw<T>::to_float(r, v);
}

template <typename T, typename Addr>
__global__ void __launch_bounds__(256)
absmax_generic_kernel(const T* __restrict__ x, Addr addr, int64_t n_chunks, int64_t B,
                      typename GenTraits<T>::Bits* __restrict__ absmax_bits, uint32_t* __restrict__ flag) {
  if (comm_aborted(flag)) return;
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
      float v[8];
      uint32_t mb;
      load8_generic<T>(x + addr.src(o), cnt, v, mb);
      const float inv32 = m > 0.0f ? __fdiv_rn((float)QMAX, m) : 0.0f;
      const double inv64 = m > 0.0f ? __ddiv_rn((double)QMAX, (double)m) : 0.0;
      if (inv32 <= 0x1p100f) {
        quant_chunk<QMAX>(v, inv32, inv64, q);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) q[i] = q_exact<QMAX>((double)v[i], inv64);
      }
    }
    store_codes8<BITS>(codes + ch * BITS, q);
  }
}

// ---------------------------------------------------------------------------
// decode helpers

// elements per 16-byte code load
template <int BITS> struct Unit16B {
  static constexpr int E = 128 / BITS;
};

__device__ __forceinline__ bool bad_codes(uint4 w, int bits) {
  if (bits == 8)
    return has_byte_0x80(w.x) | has_byte_0x80(w.y) | has_byte_0x80(w.z) | has_byte_0x80(w.w);
  return has_nibble_8(w.x) | has_nibble_8(w.y) | has_nibble_8(w.z) | has_nibble_8(w.w);
}

// codes -> "magic float" bits 0x4B400000 | (code + bias): the float
// 1.5*2^23 + code + bias, exact
__device__ __forceinline__ void magic_int8(uint32_t w, uint32_t (&f)[4]) {
  const uint32_t b = w ^ 0x80808080u;
  f[0] = __byte_perm(b, 0x4B400000u, 0x7650);
  f[1] = __byte_perm(b, 0x4B400000u, 0x7651);
  f[2] = __byte_perm(b, 0x4B400000u, 0x7652);
  f[3] = __byte_perm(b, 0x4B400000u, 0x7653);
}
// 8 INT4 codes (low nibble first)
__device__ __forceinline__ void magic_int4(uint32_t w, uint32_t (&f)[8]) {
  const uint32_t b = w ^ 0x88888888u;
  const uint32_t ev = b & 0x0F0F0F0Fu, od = (b >> 4) & 0x0F0F0F0Fu;
  f[0] = __byte_perm(ev, 0x4B400000u, 0x7650);
  f[1] = __byte_perm(od, 0x4B400000u, 0x7650);
  f[2] = __byte_perm(ev, 0x4B400000u, 0x7651);
  f[3] = __byte_perm(od, 0x4B400000u, 0x7651);
  f[4] = __byte_perm(ev, 0x4B400000u, 0x7652);
  f[5] = __byte_perm(od, 0x4B400000u, 0x7652);
  f[6] = __byte_perm(ev, 0x4B400000u, 0x7653);
  f[7] = __byte_perm(od, 0x4B400000u, 0x7653);
}

template <int BITS>
__device__ __forceinline__ void magic_word(uint32_t w, uint32_t (&f)[32 / BITS]) {
  if constexpr (BITS == 8) magic_int8(w, f);
  else magic_int4(w, f);
}

template <int BITS> struct Bias;
template <> struct Bias<8> {
  static constexpr float kF = 12582912.0f + 128.0f;
  static constexpr double kD = kMagic52 + 128.0;
};
template <> struct Bias<4> {
  static constexpr float kF = 12582912.0f + 8.0f;
  static constexpr double kD = kMagic52 + 8.0;
};

// exact code value from magic-float bits
template <int BITS> __device__ __forceinline__ double code_f64(uint32_t fbits) {
  return __dsub_rn(__hiloint2double(0x43380000, (int)(fbits & 0xFFu)), Bias<BITS>::kD);
}

template <typename O>
__device__ __forceinline__ void store_scalar(O* dst, int i, uint32_t bits16) {
  reinterpret_cast<uint16_t*>(dst)[i] = (uint16_t)bits16;
}

// ---------------------------------------------------------------------------
// K4 (16-bit outputs): dequantize / gather-dequantize.  Output = concatenation
// of the n_src sources' decoded shards (shard_len each), the qwZ receive side
// (zs/collectives.py:264).  Lane unit = one 16-byte code load (E elements,
// one block scale: the host guarantees B % E == 0 and fp32 absmax); U units
// per lane per iteration, all loads issued first.  Tiles walk the sources
// fastest, rotated by `rot`, so every peer's NVLink egress is read at once.
// Optional hpZ write-through of output range [sec_lo, sec_lo+sec_len) into
// sec_out (the secondary partition, zs/engine.py:364-367).

// decode one 16-byte unit (E elements) into packed 16-bit outputs h[E/2].
// CHECKED = false: the exact16 proof applies, pure packed fp32 math.
// CHECKED = true : per-element midpoint test with an exact f64 redo.
template <int BITS, typename O, bool CHECKED>
__device__ __forceinline__ void decode16_unit(uint4 w, float m, float s32, uint32_t (&h)[Unit16B<BITS>::E / 2]) {
  const uint32_t wa[4] = {w.x, w.y, w.z, w.w};
  uint32_t risky = 0xFFFFFFFFu;
  if constexpr (CHECKED) risky = Out16<O>::scale_ok(s32, Codes<BITS>::kQmax) ? 0xFFFFFFFFu : 0u;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    uint32_t f[32 / BITS];
    magic_word<BITS>(wa[i], f);
#pragma unroll
    for (int j = 0; j < 32 / BITS; j += 2) {
      const float2 c = fadd2(make_float2(__uint_as_float(f[j]), __uint_as_float(f[j + 1])),
                             make_float2(-Bias<BITS>::kF, -Bias<BITS>::kF));
      const float2 p = fmul2(c, make_float2(s32, s32));
      if constexpr (CHECKED)
        risky = min(risky, min(Out16<O>::near_mid(__float_as_uint(p.x)), Out16<O>::near_mid(__float_as_uint(p.y))));
      h[(i * (32 / BITS) + j) / 2] = Out16<O>::pack2(p.x, p.y);
    }
  }
  if constexpr (CHECKED) {
    if (risky == 0u) {  // exact f64 redo of this unit
      const double s64 = scale_of<BITS>((double)m);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t f[32 / BITS];
        magic_word<BITS>(wa[i], f);
#pragma unroll
        for (int j = 0; j < 32 / BITS; j += 2) {
          O a = from_f64<O>(__dmul_rn(code_f64<BITS>(f[j]), s64));
          O b = from_f64<O>(__dmul_rn(code_f64<BITS>(f[j + 1]), s64));
          h[(i * (32 / BITS) + j) / 2] =
              (uint32_t)(*reinterpret_cast<uint16_t*>(&a)) | ((uint32_t)(*reinterpret_cast<uint16_t*>(&b)) << 16);
        }
      }
    }
  }
}

// exact16: absmax fits the output format's significand (fp16-sourced scales
// for fp16 output, bf16-sourced for bf16/fp16).  Then z = code*absmax/qmax is
// either representable or a rational whose distance to every output rounding
// midpoint is >= 2^-(p+1)/qmax relative (p = 11 or 8 significand bits; qmax
// prime), while the fp32 product is within 1.5*2^-23 of z and RN64(z) within
// 2^-52: both round to the same 16-bit value, so no per-element check.
template <int BITS, typename O>
__device__ __forceinline__ void decode16_any(uint4 w, float m, uint32_t (&h)[Unit16B<BITS>::E / 2]) {
  constexpr float RQ = 1.0f / Codes<BITS>::kQmax;
  const float s32 = __fmul_rn(m, RQ);
  if (((__float_as_uint(m) & Out16<O>::kLowMask) == 0u) && Out16<O>::in_range(m))
    decode16_unit<BITS, O, false>(w, m, s32, h);
  else
    decode16_unit<BITS, O, true>(w, m, s32, h);
}

template <int N>
__device__ __forceinline__ void store_words(void* dst, const uint32_t (&h)[N]) {
#pragma unroll
  for (int i = 0; i < N / 4; ++i)
    reinterpret_cast<uint4*>(dst)[i] = make_uint4(h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
}

template <int BITS, typename O>
__global__ void __launch_bounds__(256, 4)
dequant16_kernel(SrcTable src, int n_src, int rot, int64_t shard_len, int64_t B, O* __restrict__ out,
                 O* __restrict__ sec_out, int64_t sec_lo, int64_t sec_len, int vec_ok, uint32_t* __restrict__ flag,
                 int64_t out_stride) {
  if (comm_aborted(flag)) return;
  constexpr int E = Unit16B<BITS>::E;
  constexpr int U = BITS == 8 ? 2 : 1;  // 16-byte code loads per lane per tile
  constexpr int TU = 32 * U;            // units per warp tile
  const int lane = threadIdx.x & 31;
  const int gwarp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarp = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  const int units = (int)((shard_len + E - 1) / E);
  const int full_units = vec_ok ? (int)(shard_len / E) : 0;
  const int tiles = (units + TU - 1) / TU;
  const int n_tiles = tiles * n_src;
  const bool pow2 = (B & (B - 1)) == 0;
  const int lg = pow2 ? __ffsll(B) - 1 : 0;
  bool bad = false;
  for (int g = gwarp; g < n_tiles; g += nwarp) {
    const int t = g / n_src;
    int s = g - t * n_src + rot;
    if (s >= n_src) s -= n_src;
    const int t0 = t * TU;
    const uint4* cs = reinterpret_cast<const uint4*>(src.codes[s]);
    const float* am = reinterpret_cast<const float*>(src.absmax[s]);
    const int64_t obase = (int64_t)s * out_stride;
    // tile fully inside the shard, vector-aligned and not touching the hpZ
    // secondary range: branch-free fast path
    const int64_t te0 = obase + (int64_t)t0 * E, te1 = te0 + (int64_t)TU * E;
    const bool sec_touch = sec_out != nullptr && te1 > sec_lo && te0 < sec_lo + sec_len;
    if (t0 + TU <= full_units && !sec_touch) {
      uint4 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = __ldg(cs + t0 + u * 32 + lane);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int unit = t0 + u * 32 + lane;
        bad |= bad_codes(w[u], BITS);
        const int64_t e0 = (int64_t)unit * E;
        const float m = __ldg(am + (pow2 ? (e0 >> lg) : e0 / B));
        uint32_t h[E / 2];
        decode16_any<BITS, O>(w[u], m, h);
        store_words<E / 2>(out + obase + e0, h);
      }
      continue;
    }
    // edge tiles: bounds, partial units, scalar stores, hpZ write-through
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int unit = t0 + u * 32 + lane;
      if (unit >= units) continue;
      const uint4 w = __ldg(cs + unit);
      bad |= bad_codes(w, BITS);
      const int64_t e0 = (int64_t)unit * E;
      const float m = __ldg(am + (pow2 ? (e0 >> lg) : e0 / B));
      uint32_t h[E / 2];
      decode16_any<BITS, O>(w, m, h);
      const int cnt = (int)min((int64_t)E, shard_len - e0);
      const int64_t oi = obase + e0;
      if (vec_ok && cnt == E) {
        store_words<E / 2>(out + oi, h);
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i)
          if (i < cnt) store_scalar<O>(out + oi, i, h[i / 2] >> (16 * (i & 1)));
      }
      if (sec_out != nullptr && oi + cnt > sec_lo && oi < sec_lo + sec_len) {
        const int64_t k0 = oi - sec_lo;
        if (vec_ok && cnt == E && k0 >= 0 && k0 + E <= sec_len) {
          store_words<E / 2>(sec_out + k0, h);
        } else {
#pragma unroll
          for (int i = 0; i < E; ++i)
            if (i < cnt && k0 + i >= 0 && k0 + i < sec_len) store_scalar<O>(sec_out + k0, i, h[i / 2] >> (16 * (i & 1)));
        }
      }
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K4, INT8 codes -> fp32 (config 1's dequantize): the same arithmetic as
// dequant_wide_kernel, but a lane owns one 4-element group (one 32-bit code
// word, one float4 of output) per step, consecutive lanes consecutive groups:
// every warp-wide store writes 512 contiguous bytes.  (With 16-element units
// a lane's four float4 stores sit 64 B apart from its neighbours', so each
// store instruction half-fills 32-byte sectors: 26 us for 16M elements, DRAM
// at 15% of peak, 77% of cycles with no eligible warp.)  Four groups per lane
// are loaded before any is converted, to keep loads in flight.
// Requires shard_len % 4 == 0 and 16-byte aligned output rows.
template <int BITS = 8>  // a template: the header is compiled into several translation units
__global__ void __launch_bounds__(256)
dequant8_f32_kernel(SrcTable src, int n_src, int64_t shard_len, int64_t B, float* __restrict__ out,
                    int64_t out_stride, uint32_t* __restrict__ flag) {
  if (comm_aborted(flag)) return;
  const int64_t groups = shard_len >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool pow2 = (B & (B - 1)) == 0;
  const int lg = pow2 ? __ffsll(B) - 1 : 0;
  bool bad = false;
  for (int s = 0; s < n_src; ++s) {
    const uint32_t* cs = reinterpret_cast<const uint32_t*>(src.codes[s]);
    const float* am = reinterpret_cast<const float*>(src.absmax[s]);
    float4* o = reinterpret_cast<float4*>(out + (int64_t)s * out_stride);
    for (int64_t g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g0 < groups; g0 += 4 * stride) {
      uint32_t w[4];
      float a[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t g = g0 + i * stride;
        const bool ok = g < groups;
        w[i] = ok ? __ldg(cs + g) : 0u;
        const int64_t e0 = g << 2;
        a[i] = ok ? __ldg(am + (pow2 ? (e0 >> lg) : e0 / B)) : 0.0f;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t g = g0 + i * stride;
        if (g >= groups) break;
        bad |= has_byte_0x80(w[i]);
        const double sc = scale_of<8>((double)a[i]);
        const uint32_t b = w[i] ^ 0x80808080u;
        float v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[j] = __double2float_rn(
              __dmul_rn(__dsub_rn(__hiloint2double(0x43380000, (int)__byte_perm(b, 0, 0x4440 + j)), Bias<8>::kD), sc));
        o[g] = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K4 (fp32 / f64 outputs), fp32 absmax, 16-byte code units: each element is
// the reference's f64 product RN64(code * RN64(absmax/qmax)) (one DMUL, the
// code made exact by the 2^52+2^51 trick), rounded once to the output type.
// Lane = one unit (E = 16 INT8 or 32 INT4 elements); sources one after the
// other, grid-stride over units; all-unit-aligned shards only (the host
// guarantees shard_len % E == 0 and 16-byte aligned codes/output), no hpZ
// write-through.  Replaces the 8-element exact kernel on these shapes
// (config 1's fp32 round trip).
template <int BITS, typename O>
__global__ void __launch_bounds__(256)
dequant_wide_kernel(SrcTable src, int n_src, int64_t shard_len, int64_t B, O* __restrict__ out, int64_t out_stride,
                    uint32_t* __restrict__ flag) {
  if (comm_aborted(flag)) return;
  constexpr int E = Unit16B<BITS>::E;
  const int64_t units = shard_len / E;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool pow2 = (B & (B - 1)) == 0;
  const int lg = pow2 ? __ffsll(B) - 1 : 0;
  bool bad = false;
  for (int s = 0; s < n_src; ++s) {
    const uint4* cs = reinterpret_cast<const uint4*>(src.codes[s]);
    const float* am = reinterpret_cast<const float*>(src.absmax[s]);
    O* o = out + (int64_t)s * out_stride;
    for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units; u += stride) {
      const uint4 w = __ldg(cs + u);
      bad |= bad_codes(w, BITS);
      const int64_t e0 = u * E;
      const double sc = scale_of<BITS>((double)__ldg(am + (pow2 ? (e0 >> lg) : e0 / B)));
      const uint32_t* ww = reinterpret_cast<const uint32_t*>(&w);
      double v[E];
      if constexpr (BITS == 8) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t b = ww[k] ^ 0x80808080u;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            v[4 * k + j] = __dmul_rn(__dsub_rn(__hiloint2double(0x43380000, (int)__byte_perm(b, 0, 0x4440 + j)),
                                               Bias<8>::kD), sc);
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t b = ww[k] ^ 0x88888888u;
          const uint32_t ev = b & 0x0F0F0F0Fu, od = (b >> 4) & 0x0F0F0F0Fu;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            v[8 * k + 2 * j] = __dmul_rn(
                __dsub_rn(__hiloint2double(0x43380000, (int)__byte_perm(ev, 0, 0x4440 + j)), Bias<4>::kD), sc);
            v[8 * k + 2 * j + 1] = __dmul_rn(
                __dsub_rn(__hiloint2double(0x43380000, (int)__byte_perm(od, 0, 0x4440 + j)), Bias<4>::kD), sc);
          }
        }
      }
      O* dst = o + e0;
      if constexpr (sizeof(O) == 4) {
#pragma unroll
        for (int i = 0; i < E / 4; ++i)
          reinterpret_cast<float4*>(dst)[i] = make_float4(__double2float_rn(v[4 * i]), __double2float_rn(v[4 * i + 1]),
                                                          __double2float_rn(v[4 * i + 2]), __double2float_rn(v[4 * i + 3]));
      } else {
#pragma unroll
        for (int i = 0; i < E / 2; ++i) reinterpret_cast<double2*>(dst)[i] = make_double2(v[2 * i], v[2 * i + 1]);
      }
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K4 over NVLink, TMA variant: one elected thread streams TILE-byte tiles of
// codes from the (peer) source with cp.async.bulk into a STAGES-deep shared
// ring, completion tracked by mbarrier transaction counts; all 256 threads
// decode from shared memory.  Large bulk requests cut per-request overhead on
// the NVLink read path.

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

// TMA bulk stores (shared -> global, local or a peer's NVLink-mapped memory)
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
               "r"((uint32_t)__cvta_generic_to_shared(smem)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// order this thread's generic-proxy shared-memory writes before later
// async-proxy (bulk copy) reads of them
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int BITS, typename O, int STAGES, int TILE_U>
__global__ void __launch_bounds__(256)
dequant16_tma_kernel(SrcTable src, int n_src, int rot, int64_t shard_len, int64_t B, O* __restrict__ out,
                     O* __restrict__ sec_out, int64_t sec_lo, int64_t sec_len, int vec_ok,
                     uint32_t* __restrict__ flag, int64_t out_stride) {
  if (comm_aborted(flag)) return;
  constexpr int E = Unit16B<BITS>::E;
  constexpr int UPT = TILE_U / 256;  // units per thread per tile
  extern __shared__ __align__(128) uint8_t dsm[];  // [STAGES][TILE_U] uint4 ring, then STAGES mbarriers
  uint4 (*ring)[TILE_U] = reinterpret_cast<uint4 (*)[TILE_U]>(dsm);
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)STAGES * TILE_U * 16);
  const int tid = threadIdx.x;
  const int units = (int)((shard_len + E - 1) / E);
  const int tiles = (units + TILE_U - 1) / TILE_U;
  const int n_tiles = tiles * n_src;
  const bool pow2 = (B & (B - 1)) == 0;
  const int lg = pow2 ? __ffsll(B) - 1 : 0;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto locate = [&](int g, int& s, int& t) {
    t = g / n_src;
    s = g - t * n_src + rot;
    if (s >= n_src) s -= n_src;
  };
  auto issue = [&](int g, int slot) {  // thread 0 only
    if (g < n_tiles) {
      int s, t;
      locate(g, s, t);
      const int u0 = t * TILE_U;
      const uint32_t bytes = (uint32_t)min(TILE_U, units - u0) * 16u;
      mbar_expect_tx(&full[slot], bytes);
      bulk_g2s(&ring[slot][0], reinterpret_cast<const uint4*>(src.codes[s]) + u0, bytes, &full[slot]);
    }
  };
  const int G = gridDim.x;
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < STAGES - 1; ++k) issue(blockIdx.x + k * G, k);
  }
  bool bad = false;
  int k = 0;
  for (int g = blockIdx.x; g < n_tiles; g += G, ++k) {
    const int slot = k % STAGES;
    if (tid == 0) issue(g + (STAGES - 1) * G, (k + STAGES - 1) % STAGES);
    mbar_wait(&full[slot], (uint32_t)((k / STAGES) & 1));
    int s, t;
    locate(g, s, t);
    const float* am = reinterpret_cast<const float*>(src.absmax[s]);
#pragma unroll
    for (int j = 0; j < UPT; ++j) {
      const int lu = j * 256 + tid;
      const int unit = t * TILE_U + lu;
      if (unit >= units) continue;
      const uint4 w = ring[slot][lu];
      bad |= bad_codes(w, BITS);
      const int64_t e0 = (int64_t)unit * E;
      const float m = __ldg(am + (pow2 ? (e0 >> lg) : e0 / B));
      uint32_t h[E / 2];
      decode16_any<BITS, O>(w, m, h);
      const int cnt = (int)min((int64_t)E, shard_len - e0);
      const int64_t oi = (int64_t)s * out_stride + e0;
      if (vec_ok && cnt == E) {
        store_words<E / 2>(out + oi, h);
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i)
          if (i < cnt) store_scalar<O>(out + oi, i, h[i / 2] >> (16 * (i & 1)));
      }
      if (sec_out != nullptr && oi + cnt > sec_lo && oi < sec_lo + sec_len) {
        const int64_t k0 = oi - sec_lo;
        if (vec_ok && cnt == E && k0 >= 0 && k0 + E <= sec_len) {
          store_words<E / 2>(sec_out + k0, h);
        } else {
#pragma unroll
          for (int i = 0; i < E; ++i)
            if (i < cnt && k0 + i >= 0 && k0 + i < sec_len) store_scalar<O>(sec_out + k0, i, h[i / 2] >> (16 * (i & 1)));
        }
      }
    }
    __syncthreads();  // every thread is done with this slot before it is refilled
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// exact (f64) decode of 8-element chunks, for fp32/f64 outputs, f64 absmax,
// odd block sizes and odd alignments

template <int BITS>
__device__ __forceinline__ void decode8(const uint8_t* p, double s, double (&v)[8], bool& bad) {
  if constexpr (BITS == 8) {
    uint2 w = *reinterpret_cast<const uint2*>(p);
    bad |= has_byte_0x80(w.x) | has_byte_0x80(w.y);
    uint32_t f[4];
    magic_int8(w.x, f);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = __dmul_rn(code_f64<8>(f[i]), s);
    magic_int8(w.y, f);
#pragma unroll
    for (int i = 0; i < 4; ++i) v[4 + i] = __dmul_rn(code_f64<8>(f[i]), s);
  } else {
    uint32_t w = *reinterpret_cast<const uint32_t*>(p);
    bad |= has_nibble_8(w);
    uint32_t f[8];
    magic_int4(w, f);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __dmul_rn(code_f64<4>(f[i]), s);
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
      reinterpret_cast<float4*>(dst)[0] = make_float4(from_f64<float>(v[0]), from_f64<float>(v[1]),
                                                      from_f64<float>(v[2]), from_f64<float>(v[3]));
      reinterpret_cast<float4*>(dst)[1] = make_float4(from_f64<float>(v[4]), from_f64<float>(v[5]),
                                                      from_f64<float>(v[6]), from_f64<float>(v[7]));
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

// K4 exact path: 8-element chunks, U chunks per lane per iteration (loads first)
template <int BITS, typename A, typename O>
__global__ void __launch_bounds__(256)
dequant_gather_kernel(SrcTable src, int n_src, int rot, int64_t shard_len, int64_t B, O* __restrict__ out,
                      O* __restrict__ sec_out, int64_t sec_lo, int64_t sec_len, int vec_ok,
                      uint32_t* __restrict__ flag, int64_t out_stride) {
  if (comm_aborted(flag)) return;
  constexpr int U = 4;
  using CW = typename std::conditional<BITS == 8, uint2, uint32_t>::type;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t chunks = (shard_len + 7) / 8;
  const int64_t tiles = (chunks + 32 * U - 1) / (32 * U);
  const int64_t n_tiles = tiles * n_src;
  const bool pow2 = (B & (B - 1)) == 0;
  const int lg = pow2 ? __ffsll(B) - 1 : 0;
  bool bad = false;
  for (int64_t tile = gwarp; tile < n_tiles; tile += nwarp) {
    const int s = (int)((tile % n_src + rot) % n_src);
    const int64_t t0 = (tile / n_src) * 32 * U;
    const A* am = reinterpret_cast<const A*>(src.absmax[s]);
    CW w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t ch = t0 + u * 32 + lane;
      w[u] = ch < chunks ? __ldg(reinterpret_cast<const CW*>(src.codes[s] + ch * BITS)) : CW{};
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t ch = t0 + u * 32 + lane;
      if (ch >= chunks) continue;
      const int64_t e = ch * 8;
      const double sc = scale_of<BITS>(absmax_f64<A>(am, pow2 ? (e >> lg) : e / B));
      double v[8];
      decode8<BITS>(reinterpret_cast<const uint8_t*>(&w[u]), sc, v, bad);
      const int cnt = (int)min((int64_t)8, shard_len - e);
      const int64_t oi = (int64_t)s * out_stride + e;
      store8<O>(out + oi, v, cnt, vec_ok);
      if (sec_out != nullptr && oi + cnt > sec_lo && oi < sec_lo + sec_len) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int64_t k = oi + i - sec_lo;
          if (i < cnt && k >= 0 && k < sec_len) sec_out[k] = from_f64<O>(v[i]);
        }
      }
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K3: dequantize n_src sources of n elements each and fold them in f64 from
// +0.0 in source order; optional f64 post-scale (1.0 = the reference's sum).
// Lane unit: 8-element chunk; each lane owns 2 chunks per iteration and issues
// the code loads of up to 4 sources before decoding them.

template <int BITS, typename A, typename O>
__global__ void __launch_bounds__(256)
dequant_reduce_kernel(SrcTable src, int n_src, int64_t n, int64_t B, O* __restrict__ out, double post_scale,
                      int vec_ok, uint32_t* __restrict__ flag) {
  if (comm_aborted(flag)) return;
  constexpr int U = 2;
  constexpr int SB = 4;
  using CW = typename std::conditional<BITS == 8, uint2, uint32_t>::type;
  const int lane = threadIdx.x & 31;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t chunks = (n + 7) / 8;
  const int64_t tiles = (chunks + 32 * U - 1) / (32 * U);
  const bool pow2 = (B & (B - 1)) == 0;
  const int lg = pow2 ? __ffsll(B) - 1 : 0;
  bool bad = false;
  for (int64_t tile = gwarp; tile < tiles; tile += nwarp) {
    const int64_t t0 = tile * 32 * U;
    double acc[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[u][i] = 0.0;
    for (int s0 = 0; s0 < n_src; s0 += SB) {
      CW w[SB][U];
#pragma unroll
      for (int j = 0; j < SB; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t ch = t0 + u * 32 + lane;
          if (s0 + j < n_src && ch < chunks)
            w[j][u] = __ldg(reinterpret_cast<const CW*>(src.codes[s0 + j] + ch * BITS));
          else
            w[j][u] = CW{};
        }
#pragma unroll
      for (int j = 0; j < SB; ++j) {
        if (s0 + j >= n_src) break;
        const A* am = reinterpret_cast<const A*>(src.absmax[s0 + j]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t ch = t0 + u * 32 + lane;
          if (ch >= chunks) continue;
          const int64_t e = ch * 8;
          const double sc = scale_of<BITS>(absmax_f64<A>(am, pow2 ? (e >> lg) : e / B));
          decode8_acc<BITS>(reinterpret_cast<const uint8_t*>(&w[j][u]), sc, acc[u], bad);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t ch = t0 + u * 32 + lane;
      if (ch >= chunks) continue;
      const int64_t e = ch * 8;
      if (post_scale != 1.0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[u][i] = __dmul_rn(acc[u][i], post_scale);
      }
      store8<O>(out + e, acc[u], (int)min((int64_t)8, n - e), vec_ok);
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K2 register path: a team of LANES lanes owns one OUTPUT block of
// B2 = LANES * 16 elements (lane = 16 contiguous elements = two 8-chunks).
// For each source (ascending, loads of up to 4 sources in flight) the codes
// are dequantized (input block size B1 arbitrary, multiple of 8) and folded
// into f64 accumulators; then the block is requantized from its exact f64
// absmax, which is stored in f64 so the next hop decodes bit-exactly.

template <int IBITS, typename IA, int OBITS, int LANES>
__global__ void __launch_bounds__(256)
drq_reg_kernel(SrcTable src, int n_src, int64_t n, int64_t B1, int64_t n_blocks_out, uint8_t* __restrict__ codes,
               double* __restrict__ absmax, uint32_t* __restrict__ flag) {
  if (comm_aborted(flag)) return;
  constexpr int B2 = LANES * 16;
  constexpr int TPW = 32 / LANES;
  constexpr int QMAX = Codes<OBITS>::kQmax;
  constexpr int SB = 4;
  using CW = typename std::conditional<IBITS == 8, uint2, uint32_t>::type;  // one 8-chunk of codes
  const int lane = threadIdx.x & 31;
  const int tl = lane % LANES;
  const int team = lane / LANES;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool pow2 = (B1 & (B1 - 1)) == 0;
  const int lg = pow2 ? __ffsll(B1) - 1 : 0;
  const int64_t chunks_in = (n + B1 - 1) / B1 * B1 / 8;  // padded input chunks
  bool bad = false;
  for (int64_t wb = gwarp * TPW; wb < n_blocks_out; wb += nwarp * TPW) {
    const int64_t b = wb + team;
    const bool active = b < n_blocks_out;
    const int64_t c0 = (b * B2 + (int64_t)tl * 16) / 8;  // first of this lane's two chunks
    double acc[2][8];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[h][i] = 0.0;
    for (int s0 = 0; s0 < n_src; s0 += SB) {
      CW w[SB][2];
#pragma unroll
      for (int j = 0; j < SB; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t ch = c0 + h;
          if (active && s0 + j < n_src && ch < chunks_in)
            w[j][h] = __ldg(reinterpret_cast<const CW*>(src.codes[s0 + j] + ch * IBITS));
          else
            w[j][h] = CW{};
        }
#pragma unroll
      for (int j = 0; j < SB; ++j) {
        if (s0 + j >= n_src) break;
        const IA* am = reinterpret_cast<const IA*>(src.absmax[s0 + j]);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t ch = c0 + h;
          if (!active || ch >= chunks_in) continue;
          const int64_t e = ch * 8;
          const double sc = scale_of<IBITS>(absmax_f64<IA>(am, pow2 ? (e >> lg) : e / B1));
          decode8_acc<IBITS>(reinterpret_cast<const uint8_t*>(&w[j][h]), sc, acc[h], bad);
        }
      }
    }
    double mx = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if ((c0 + h) * 8 + i >= n) acc[h][i] = 0.0;  // zero padding like the reference
        mx = dmax_nn(mx, fabs(acc[h][i]));
      }
#pragma unroll
    for (int off = LANES / 2; off >= 1; off >>= 1) mx = dmax_nn(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    if (active && tl == 0) {
      absmax[b] = mx;
      if (!(mx <= DBL_MAX)) raise_flag(flag, FLAG_NONFINITE);
    }
    const double inv = mx > 0.0 ? __ddiv_rn((double)QMAX, mx) : 0.0;
    if (active) {
      uint32_t q0[8], q1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        q0[i] = q_exact<QMAX>(acc[0][i], inv);
        q1[i] = q_exact<QMAX>(acc[1][i], inv);
      }
      uint8_t* dst = codes + c0 * OBITS;
      if constexpr (OBITS == 8) {
        const uint2 a = pack8_int8(q0), c = pack8_int8(q1);
        *reinterpret_cast<uint4*>(dst) = make_uint4(a.x, a.y, c.x, c.y);
      } else {
        *reinterpret_cast<uint2*>(dst) = make_uint2(pack8_int4(q0), pack8_int4(q1));
      }
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// 16-element lanes for the f64 reduce kernels (K2 fast path, K3 fast path):
// one load of 16 codes per source (INT8: 16 B, INT4: 8 B), one block scale per
// source (host guarantees block % 16 == 0 and aligned code pointers).

template <int BITS> struct Vec16;
template <> struct Vec16<8> { using T = uint4; };
template <> struct Vec16<4> { using T = uint2; };

// Source loads: read-only path (__ldg) when the sources cannot change during
// the kernel, L2-coherent loads (ld.global.cg) when peers may still be
// writing other parts of the same buffers.
enum { kLdNC = 0, kLdCG = 1 };
template <int MODE, typename V>
__device__ __forceinline__ V ld_src(const V* p) {
  if constexpr (MODE == kLdCG) return __ldcg(p);
  else return __ldg(p);
}
template <int MODE, typename A>
__device__ __forceinline__ double ld_absmax(const A* p, int64_t i) {
  if constexpr (MODE == kLdCG) return (double)__ldcg(p + i);
  else return absmax_f64<A>(p, i);
}

// acc[i] = RN64(acc[i] + RN64(code_i * s)) for the 16 codes in w -- the
// reference's fold step (zs/quantizer.py:255-257, zs/collectives.py:71-75).
// Each code becomes an exact double as 2^52+2^51+(code+bias) - (2^52+2^51+bias):
// one PRMT builds the low word, one DADD removes the bias.
// ASSIGN (first source of a fold): acc[i] = RN64(code_i * s), which equals
// RN64(+0.0 + RN64(code_i * s)) because the product is never -0.0 (s > 0 and
// codes are integers), so the reference's fold from +0.0 is reproduced exactly.
template <int BITS, bool VALIDATE, bool ASSIGN = false>
__device__ __forceinline__ void fold16(const typename Vec16<BITS>::T& w, double s, double (&acc)[16], bool& bad) {
  const uint32_t* ww = reinterpret_cast<const uint32_t*>(&w);
  if constexpr (BITS == 8) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (VALIDATE) bad |= has_byte_0x80(ww[k]);
      const uint32_t b = ww[k] ^ 0x80808080u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double c = __dsub_rn(__hiloint2double(0x43380000, (int)__byte_perm(b, 0, 0x4440 + j)), Bias<8>::kD);
        if constexpr (ASSIGN) acc[4 * k + j] = __dmul_rn(c, s);
        else acc[4 * k + j] = __dadd_rn(acc[4 * k + j], __dmul_rn(c, s));
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if constexpr (VALIDATE) bad |= has_nibble_8(ww[k]);
      const uint32_t b = ww[k] ^ 0x88888888u;
      const uint32_t ev = b & 0x0F0F0F0Fu, od = (b >> 4) & 0x0F0F0F0Fu;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double c0 = __dsub_rn(__hiloint2double(0x43380000, (int)__byte_perm(ev, 0, 0x4440 + j)), Bias<4>::kD);
        const double c1 = __dsub_rn(__hiloint2double(0x43380000, (int)__byte_perm(od, 0, 0x4440 + j)), Bias<4>::kD);
        if constexpr (ASSIGN) {
          acc[8 * k + 2 * j] = __dmul_rn(c0, s);
          acc[8 * k + 2 * j + 1] = __dmul_rn(c1, s);
        } else {
          acc[8 * k + 2 * j] = __dadd_rn(acc[8 * k + 2 * j], __dmul_rn(c0, s));
          acc[8 * k + 2 * j + 1] = __dadd_rn(acc[8 * k + 2 * j + 1], __dmul_rn(c1, s));
        }
      }
    }
  }
}

// K3 fast path: lane = 16 contiguous elements, loads of up to 4 sources in
// flight, f64 fold in source order from +0.0, one rounding to the output type.
// One lane: 16 output elements of K3 starting at 16*u (see dequant_reduce16_kernel).
template <int BITS, typename A, typename O, bool VALIDATE, int CG>
__device__ __forceinline__ void dr_unit(const SrcTable& src, int n_src, int64_t u, int64_t B, bool pow2, int lg,
                                        O* __restrict__ out, double post_scale, bool& bad) {
  using V = typename Vec16<BITS>::T;
  constexpr int SB = 4;
  const int64_t e0 = u * 16;
  const int64_t blk = pow2 ? (e0 >> lg) : e0 / B;
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  for (int s0 = 0; s0 < n_src; s0 += SB) {
    V w[SB];
    double sc[SB];
#pragma unroll
    for (int j = 0; j < SB; ++j) {
      if (s0 + j < n_src) {
        w[j] = ld_src<CG>(reinterpret_cast<const V*>(src.codes[s0 + j]) + u);
        sc[j] = ld_absmax<CG, A>(reinterpret_cast<const A*>(src.absmax[s0 + j]), blk);
      }
    }
#pragma unroll
    for (int j = 0; j < SB; ++j) {
      if (s0 + j >= n_src) break;
      fold16<BITS, VALIDATE>(w[j], scale_of<BITS>(sc[j]), acc, bad);
    }
  }
  if (post_scale != 1.0) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = __dmul_rn(acc[i], post_scale);
  }
  O* dst = out + e0;
  if constexpr (sizeof(O) == 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      reinterpret_cast<float4*>(dst)[i] = make_float4(from_f64<float>(acc[4 * i]), from_f64<float>(acc[4 * i + 1]),
                                                      from_f64<float>(acc[4 * i + 2]), from_f64<float>(acc[4 * i + 3]));
  } else if constexpr (sizeof(O) == 8) {
#pragma unroll
    for (int i = 0; i < 8; ++i) reinterpret_cast<double2*>(dst)[i] = make_double2(acc[2 * i], acc[2 * i + 1]);
  } else {
    uint32_t h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      O a = from_f64<O>(acc[2 * i]), b = from_f64<O>(acc[2 * i + 1]);
      h[i] = (uint32_t)(*reinterpret_cast<uint16_t*>(&a)) | ((uint32_t)(*reinterpret_cast<uint16_t*>(&b)) << 16);
    }
    store_words<8>(dst, h);
  }
}

template <int BITS, typename A, typename O, bool VALIDATE>
__global__ void __launch_bounds__(256)
dequant_reduce16_kernel(SrcTable src, int n_src, int64_t n, int64_t B, O* __restrict__ out, double post_scale,
                        uint32_t* __restrict__ flag) {
  if (comm_aborted(flag)) return;
  const int64_t units = n / 16;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool pow2 = (B & (B - 1)) == 0;
  const int lg = pow2 ? __ffsll(B) - 1 : 0;
  bool bad = false;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units; u += stride)
    dr_unit<BITS, A, O, VALIDATE, kLdNC>(src, n_src, u, B, pow2, lg, out, post_scale, bad);
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// One team of LANES lanes: output block b of K2 (see drq16_kernel).
template <int IBITS, typename IA, int OBITS, int LANES, bool VALIDATE, typename FO, int CG, int CGA = CG,
          typename Src = SrcTable>
__device__ __forceinline__ void drq_team(const Src& src, int n_src, int64_t n, int64_t B1, bool pow2, int lg,
                                         int64_t b, int64_t n_blocks_out, int tl, uint8_t* __restrict__ codes,
                                         double* __restrict__ absmax, uint32_t* __restrict__ flag,
                                         FO* __restrict__ final_out, bool& bad) {
  using V = typename Vec16<IBITS>::T;
  constexpr int B2 = LANES * 16;
  constexpr int QMAX = Codes<OBITS>::kQmax;
  constexpr int SB = 4;
  const int64_t e0 = b * B2 + (int64_t)tl * 16;
  const bool active = b < n_blocks_out && e0 < n;  // n % 16 == 0: lanes are all-valid or all-empty
  const int64_t u = e0 / 16;
  const int64_t ib = pow2 ? (e0 >> lg) : e0 / B1;
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  for (int s0 = 0; s0 < n_src; s0 += SB) {
    V w[SB];
    double sc[SB];
#pragma unroll
    for (int j = 0; j < SB; ++j) {
      if (active && s0 + j < n_src) {
        w[j] = ld_src<CG>(reinterpret_cast<const V*>(src.code_ptr(s0 + j)) + u);
        sc[j] = ld_absmax<CGA, IA>(reinterpret_cast<const IA*>(src.abs_ptr(s0 + j)), ib);
      }
    }
    if (active) {
#pragma unroll
      for (int j = 0; j < SB; ++j) {
        if (s0 + j >= n_src) break;
        fold16<IBITS, VALIDATE>(w[j], scale_of<IBITS>(sc[j]), acc, bad);
      }
    }
  }
  double mx = absmax16(acc);
#pragma unroll
  for (int off = LANES / 2; off >= 1; off >>= 1) mx = dmax_nn(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (b < n_blocks_out && tl == 0) {
    absmax[b] = mx;
    if (!(mx <= DBL_MAX)) raise_flag(flag, FLAG_NONFINITE);
  }
  if (active) {
    const double inv = mx > 0.0 ? __ddiv_rn((double)QMAX, mx) : 0.0;
    uint32_t q0[8], q1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {  // |acc*inv| <= qmax: no clamp needed
      q0[i] = (uint32_t)rint_f64(__dmul_rn(acc[i], inv));
      q1[i] = (uint32_t)rint_f64(__dmul_rn(acc[8 + i], inv));
    }
    if constexpr (std::is_void<FO>::value) {
      uint8_t* dst = codes + u * 2 * OBITS;
      if constexpr (OBITS == 8) {
        const uint2 a = pack8_int8(q0), c = pack8_int8(q1);
        *reinterpret_cast<uint4*>(dst) = make_uint4(a.x, a.y, c.x, c.y);
      } else {
        *reinterpret_cast<uint2*>(dst) = make_uint2(pack8_int4(q0), pack8_int4(q1));
      }
    } else {
      const double s2 = scale_of<OBITS>(mx);
      double v[16];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[i] = __dadd_rn(0.0, __dmul_rn((double)(int)q0[i], s2));
        v[8 + i] = __dadd_rn(0.0, __dmul_rn((double)(int)q1[i], s2));
      }
      FO* dst = final_out + e0;
      if constexpr (sizeof(FO) == 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          reinterpret_cast<float4*>(dst)[i] = make_float4(from_f64<float>(v[4 * i]), from_f64<float>(v[4 * i + 1]),
                                                          from_f64<float>(v[4 * i + 2]), from_f64<float>(v[4 * i + 3]));
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) reinterpret_cast<double2*>(dst)[i] = make_double2(v[2 * i], v[2 * i + 1]);
      }
    }
  } else if (b < n_blocks_out && std::is_void<FO>::value) {
    // zero padding of a partial last block (zs/quantizer.py:215-217)
    uint8_t* dst = codes + u * 2 * OBITS;
    if constexpr (OBITS == 8) *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    else *reinterpret_cast<uint2*>(dst) = make_uint2(0, 0);
  }
}

// K2 fast path: a team of LANES lanes owns one output block of B2 = 16*LANES
// elements, lane = 16 contiguous elements; sources folded in order (loads of
// up to 4 in flight); requantized from the exact f64 block absmax (stored in
// f64).  Requires n % 16 == 0, input block % 16 == 0, aligned code pointers.
//
// FO != void (qgZ with a single group, Y = 1): hop 2 is a self-send, so instead
// of storing the requantized codes the kernel emits what K3 would compute from
// them -- fold(+0.0, code * RN64(absmax/qmax)) rounded once to FO.
template <int IBITS, typename IA, int OBITS, int LANES, bool VALIDATE, typename FO = void>
__global__ void __launch_bounds__(256)
drq16_kernel(SrcTable src, int n_src, int64_t n, int64_t B1, int64_t n_blocks_out, uint8_t* __restrict__ codes,
             double* __restrict__ absmax, uint32_t* __restrict__ flag, FO* __restrict__ final_out = nullptr) {
  if (comm_aborted(flag)) return;
  constexpr int TPW = 32 / LANES;
  const int lane = threadIdx.x & 31;
  const int tl = lane % LANES;
  const int team = lane / LANES;
  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool pow2 = (B1 & (B1 - 1)) == 0;
  const int lg = pow2 ? __ffsll(B1) - 1 : 0;
  bool bad = false;
  for (int64_t wb = gwarp * TPW; wb < n_blocks_out; wb += nwarp * TPW)
    drq_team<IBITS, IA, OBITS, LANES, VALIDATE, FO, kLdNC>(src, n_src, n, B1, pow2, lg, wb + team, n_blocks_out, tl,
                                                           codes, absmax, flag, final_out, bad);
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K2 fixed fan-in fast path (the qgZ hop-1 reduce, zs/collectives.py:519-527):
// NSRC sources known at compile time, fp32 absmax from K1, 512-element output
// blocks (one warp per block, lane = 16 contiguous elements).  Codes are
// always validated (-8 / -128 raise IntegrityError, zs/quantizer.py:233-235):
// a few integer ops per 16 codes.
// Against drq16_kernel it drops the runtime source loop and its predicates,
// the +0.0 initialisation (first source assigns, see fold16), and the
// small-absmax branch of the scale division (fp32 absmax is never below
// 2^-149, inside div_q's exactness premise).  Same arithmetic, same bits.
template <int Q>
__device__ __forceinline__ double div_q_f32(float m) {
  constexpr double r = 1.0 / Q;
  const double md = (double)m;
  const double q0 = __dmul_rn(md, r);
  const double e = __fma_rn(-q0, (double)Q, md);
  return __fma_rn(e, r, q0);
}

// K2 epilogue for one 512-element output block b held by a warp (lane tl owns
// elements e0 .. e0+15): the exact f64 block absmax (stored in f64), then
// either the requantized codes (inactive lanes write the zero padding of a
// partial last block, zs/quantizer.py:215-217) or, when hop 2 is a self-send
// (FO != void), K3's fold of that one source rounded once to FO.
// fo_tbl (FO = float, OBITS = 4): the warp's 16-float shared table of the
// final values, fo_tbl[c + 8] = RN32(RN64(+0.0 + RN64(c * s2))), so a code
// costs one IMAD + one LDS.32 instead of DSUB + DMUL + F2F (same values).
template <int OBITS, typename FO>
__device__ __forceinline__ void drq_epilogue(const double (&acc)[16], int64_t b, int tl, int64_t e0, bool active,
                                             int64_t u, uint8_t* __restrict__ codes, double* __restrict__ absmax,
                                             uint32_t* __restrict__ flag, FO* __restrict__ final_out,
                                             float* fo_tbl = nullptr, bool span = false) {
  constexpr int QMAX = Codes<OBITS>::kQmax;
  double mx = absmax16(acc);
  mx = warp_max_nonneg(mx);
  if (tl == 0) {
    absmax[b] = mx;
    if (!(mx <= DBL_MAX)) raise_flag(flag, FLAG_NONFINITE);
  }
  const double inv = mx > 0.0 ? __ddiv_rn((double)QMAX, mx) : 0.0;
  // r = RN(acc*inv) + 2^52+2^51: its low word is rint-even(acc*inv) (|.| <= qmax,
  // no clamp needed) and r - (2^52+2^51) is that code as an exact double
  double r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = __dadd_rn(__dmul_rn(acc[i], inv), kMagic52);
  if constexpr (std::is_void<FO>::value) {
    uint32_t q0[8], q1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      q0[i] = (uint32_t)__double2loint(r[i]);
      q1[i] = (uint32_t)__double2loint(r[8 + i]);
    }
    // inactive lanes hold zeros: they write the zero padding of a partial
    // last block (zs/quantizer.py:215-217)
    uint8_t* dst = codes + u * 2 * OBITS;
    if constexpr (OBITS == 8) {
      const uint2 a = pack8_int8(q0), c = pack8_int8(q1);
      *reinterpret_cast<uint4*>(dst) = make_uint4(a.x, a.y, c.x, c.y);
    } else {
      *reinterpret_cast<uint2*>(dst) = make_uint2(pack8_int4(q0), pack8_int4(q1));
    }
  } else if (OBITS == 4 && sizeof(FO) == 4 && fo_tbl != nullptr) {
    const double s2 = scale_of<OBITS>(mx);
    __syncwarp();  // the previous block's lookups are done
    if (tl < 16) fo_tbl[tl] = __double2float_rn(__dadd_rn(0.0, __dmul_rn((double)(tl - 8), s2)));
    __syncwarp();
    if (active) {
      const uint32_t base = (uint32_t)__cvta_generic_to_shared(fo_tbl) + 32;  // entry of code 0
      float v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t a = base + (uint32_t)(__double2loint(r[i]) * 4);
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[i]) : "r"(a) : "memory");
      }
      if (span) {  // coalesced layout (store_span_f32): the block's 512 outputs are contiguous
        float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(final_out) + b * 512);
#pragma unroll
        for (int k = 0; k < 4; ++k) dst[k * 32 + tl] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
      } else {
        float* dst = reinterpret_cast<float*>(final_out) + e0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
          reinterpret_cast<float4*>(dst)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
    }
  } else if (active) {
    // hop 2 to itself: K3's fold of one source, RN(+0.0 + RN(code*s2)) = RN(code*s2)
    const double s2 = scale_of<OBITS>(mx);
    double v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __dmul_rn(__dsub_rn(r[i], kMagic52), s2);
    FO* dst = final_out + e0;
    if constexpr (sizeof(FO) == 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        reinterpret_cast<float4*>(dst)[i] = make_float4(from_f64<float>(v[4 * i]), from_f64<float>(v[4 * i + 1]),
                                                        from_f64<float>(v[4 * i + 2]), from_f64<float>(v[4 * i + 3]));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) reinterpret_cast<double2*>(dst)[i] = make_double2(v[2 * i], v[2 * i + 1]);
    }
  }
}

template <int IBITS, int OBITS, int NSRC, typename FO = void>
__global__ void __launch_bounds__(256)
drq_fast_kernel(SrcTable src, int64_t n, int lg1, int64_t n_blocks_out, uint8_t* __restrict__ codes,
                double* __restrict__ absmax, uint32_t* __restrict__ flag, FO* __restrict__ final_out = nullptr) {
  if (comm_aborted(flag)) return;
  using V = typename Vec16<IBITS>::T;
  const int tl = threadIdx.x & 31;
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool bad = false;
  // the sources live in peers' HBM (NVLink): the next block's codes and absmax
  // are loaded before this block is folded (register double buffer), so each
  // warp keeps its loads in flight across the compute
  V w[NSRC], wn[NSRC];
  float m[NSRC], mn[NSRC];
  auto load = [&](int64_t b, V (&wv)[NSRC], float (&mv)[NSRC]) {
    const int64_t e0 = b * 512 + (int64_t)tl * 16;
    const bool ok = b < n_blocks_out && e0 < n;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      if (ok) {
        wv[j] = __ldg(reinterpret_cast<const V*>(src.codes[j]) + (e0 >> 4));
        mv[j] = __ldg(reinterpret_cast<const float*>(src.absmax[j]) + (e0 >> lg1));
      } else {
        wv[j] = V{};
        mv[j] = 0.0f;
      }
    }
  };
  int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  load(b, wn, mn);
  for (; b < n_blocks_out; b += nwarp) {
    const int64_t e0 = b * 512 + (int64_t)tl * 16;
    const bool active = e0 < n;  // n % 16 == 0: lanes are all-valid or all-empty
    const int64_t u = e0 >> 4;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      w[j] = wn[j];
      m[j] = mn[j];
    }
    load(b + nwarp, wn, mn);
    double acc[16];
    fold16<IBITS, true, true>(w[0], div_q_f32<Codes<IBITS>::kQmax>(m[0]), acc, bad);
#pragma unroll
    for (int j = 1; j < NSRC; ++j) fold16<IBITS, true>(w[j], div_q_f32<Codes<IBITS>::kQmax>(m[j]), acc, bad);
    drq_epilogue<OBITS, FO>(acc, b, tl, e0, active, u, codes, absmax, flag, final_out);
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K1 with the hop-1 all-to-all fused in (push).  The qgZ send buffer [j][c][e]
// is message j = send blocks [j*mb, (j+1)*mb), destined for
// local peer j; instead of writing it to this rank's HBM for the peers to
// pull, each CTA quantizes a tile of TILE consecutive send blocks into shared
// memory (two alternating staging buffers) and one thread streams the tile's
// codes and absmax straight into the receiving peers' buffers with TMA bulk
// stores over NVLink, slot `loc` of peer j's [src_loc][c][e] receive region
// (zs/collectives.py:519-523: the receiver folds its X messages in ascending
// source order).  The quantize arithmetic is quant_compute's, unchanged; only
// the destination differs.  The NVLink transfer thus overlaps the (issue-
// bound) quantization instead of following it, and K2 reads local HBM.
constexpr int kMaxPush = 8;
template <int LANES, int EPL, int BITS>
struct PushTile {  // a warp tile carries about 2 KB of codes
  static constexpr int kBB = LANES * EPL * BITS / 8;
  static constexpr int R = (2048 / kBB) / (32 / LANES) > 1 ? (2048 / kBB) / (32 / LANES) : 1;
  static constexpr int WT = (32 / LANES) * R;
};
struct PushDst {
  uint8_t* codes[kMaxPush];  // peer j's receive slot for this rank's message (codes)
  uint8_t* absmax[kMaxPush]; // ... and its fp32 absmax
  FastDiv mb;                // send blocks per message
  int self_msg;              // the message this rank keeps (its own slot): stored directly, not staged
};

template <typename T, int BITS, int LANES, int EPL>
__global__ void __launch_bounds__(256)
quantize_push_kernel(const T* __restrict__ x, SwizzleAddr addr, int n_msg, int first, PushDst dst,
                     uint32_t* __restrict__ flag) {
  if (comm_aborted(flag)) return;
  constexpr int TPW = 32 / LANES;
  constexpr int BB = LANES * EPL * BITS / 8;     // code bytes per block
  constexpr int R = PushTile<LANES, EPL, BITS>::R;   // team rounds per warp tile
  constexpr int WT = TPW * R;                    // send blocks per warp tile (~2 KB of codes)
  static_assert(BB % 16 == 0, "bulk copies move 16-byte multiples");
  // per-warp staging, two alternating buffers: warps never wait for each other
  __shared__ __align__(128) uint8_t st_codes[8][2][WT * BB];
  __shared__ __align__(16) float st_abs[8][2][WT];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int tl = lane % LANES, team = lane / LANES;
  // Warp tiles never straddle a message, and consecutive tiles go to
  // different peers (message (first + v) mod n_msg for virtual tile v), so at
  // any moment the grid's stores are spread over every peer's NVLink ingress
  // instead of all ranks pushing message 0 to the same GPU first.
  const int64_t mbs = dst.mb.d;
  const int64_t tpm = (mbs + WT - 1) / WT;  // warp tiles per message
  const int64_t tiles = tpm * n_msg;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int it = 0;  // staged tiles so far
  for (int64_t v = gw; v < tiles; v += nw) {
    int j = (int)(v % n_msg) + first;
    if (j >= n_msg) j -= n_msg;
    const int64_t off0 = (v / n_msg) * WT;  // first block of the tile inside message j
    const int nb = (int)min((int64_t)WT, mbs - off0);
    if (j == dst.self_msg) {
      // the message this rank keeps: quantize straight into its slot in local
      // HBM, like K1 without the push (no staging, no bulk store)
      uint8_t* const cb = dst.codes[j] + off0 * BB;
      float* const ab = reinterpret_cast<float*>(dst.absmax[j]) + off0;
#pragma unroll 1
      for (int r = 0; r < R; ++r) {
        const int bl = r * TPW + team;
        TeamIn<T, EPL> in;
        quant_load<T, LANES, EPL, SwizzleAddr>(x, addr, (int64_t)j * mbs + off0 + bl, bl < nb, tl, in);
        quant_compute<T, BITS, LANES, EPL, false>(x, in, bl, bl < nb, tl, cb, ab, flag, nullptr);
      }
      continue;
    }
    const int buf = it & 1;
    if (it >= 2) {
      if (lane == 0) bulk_wait_read<1>();  // the stores issued from this buffer two tiles ago have read it
      __syncwarp();
    }
    ++it;
#pragma unroll 1
    for (int r = 0; r < R; ++r) {
      const int bl = r * TPW + team;
      TeamIn<T, EPL> in;
      quant_load<T, LANES, EPL, SwizzleAddr>(x, addr, (int64_t)j * mbs + off0 + bl, bl < nb, tl, in);
      quant_compute<T, BITS, LANES, EPL, false>(x, in, bl, bl < nb, tl, st_codes[wid][buf], st_abs[wid][buf], flag,
                                                nullptr);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      bulk_s2g(dst.codes[j] + off0 * BB, st_codes[wid][buf], (uint32_t)(nb * BB));
      float* da = reinterpret_cast<float*>(dst.absmax[j]) + off0;
      if ((reinterpret_cast<uintptr_t>(da) & 15) == 0 && nb % 4 == 0) {
        bulk_s2g(da, st_abs[wid][buf], (uint32_t)(nb * 4));
      } else {
        for (int i = 0; i < nb; ++i) da[i] = st_abs[wid][buf][i];
      }
      bulk_commit();
    }
  }
  if (lane == 0) {
    bulk_wait<0>();           // every store performed before the grid completes ...
    __threadfence_system();   // ... and ordered before the group barrier's release that follows
  }
}

// ---------------------------------------------------------------------------
// Product tables for INT4 folds.  The reference's fold step adds RN64(c * s)
// for a code c in [-7, 7] and its block scale s (zs/quantizer.py:237,
// :255-257; zs/collectives.py:71-75): 15 possible products per (source,
// block).  When one block scale covers a whole warp's 512 elements, the warp
// computes them once into shared memory --
//     T[c + 8] = RN64(+0.0 + RN64(c * s))
// (the +0.0 turns the -0.0 product of a negative code with s == 0 into the
// +0.0 that the reference's fold from +0.0 produces; the fold never holds
// -0.0, so adding +0.0 instead of -0.0 later is the same) -- and each code then
// costs one PRMT (its byte offset into the table), one LDS.64 and one DADD,
// instead of fold16's PRMT + MOV + DSUB + DMUL + DADD.  Same products, same
// fold order: the same bits.  A table is 16 doubles = 128 contiguous bytes, so
// any mix of lanes' entries touches each of the 32 banks at most once.

// Table layout: one 256-byte-aligned slot per (warp, source), entries at the
// slot start, so the shared address of entry k is one PRMT: the slot address
// with its low byte replaced by 8k (8k <= 120) -- no address add per code.
constexpr int kTblSlotDoubles = 32;  // 256 bytes

// lanes 16*h .. 16*h+15 build source 2p+h's table (entry lane & 15) from the
// block absmax m[j] (identical in every lane): one scale division and one
// product per lane per pass
template <int NSRC, typename A>
__device__ __forceinline__ void tbl4_build(double* __restrict__ tbl, const A (&m)[NSRC], int lane) {
#pragma unroll
  for (int p = 0; p < (NSRC + 1) / 2; ++p) {
    const int h = lane >> 4;
    const int j = 2 * p + h;
    const A mj = h ? m[2 * p + 1 < NSRC ? 2 * p + 1 : 2 * p] : m[2 * p];
    if (j < NSRC) {
      double sj;
      if constexpr (sizeof(A) == 4) sj = div_q_f32<7>(mj);
      else sj = scale_of<4>(mj);
      tbl[j * kTblSlotDoubles + (lane & 15)] = __dadd_rn(0.0, __dmul_rn((double)((lane & 15) - 8), sj));
    }
  }
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr) : "memory");
  return v;
}

// Warp-coalesced fp32 output for K3 (and any fold whose warp covers 512
// contiguous elements, 32 units of 16): instead of lane l folding elements
// 16l..16l+15 and storing four float4s 64 B apart from its neighbours' (each
// store instruction then half-fills every 32-byte sector it touches: ncu on
// K3 showed the L1/L2 store path 70% busy at 14% of the DRAM peak), lane l
// folds elements k*128 + 4l .. +3 for k = 0..3, whose codes are four 16-bit
// pieces at byte k*64 + 2l of the warp's 256-byte INT4 span, and store k of
// the warp writes 512 contiguous bytes.  The 16 nibbles are packed in that
// order, so acc[4k + e] is element k*128 + 4l + e.  Arithmetic per element is
// unchanged.
__device__ __forceinline__ uint2 int4_span_pieces_g(const uint8_t* __restrict__ span, int lane) {
  const uint16_t* p = reinterpret_cast<const uint16_t*>(span) + lane;
  const uint32_t p0 = __ldg(p), p1 = __ldg(p + 32), p2 = __ldg(p + 64), p3 = __ldg(p + 96);
  return make_uint2(p0 | (p1 << 16), p2 | (p3 << 16));
}
__device__ __forceinline__ uint2 int4_span_pieces_s(const uint8_t* span, int lane) {
  const uint16_t* p = reinterpret_cast<const uint16_t*>(span) + lane;
  const uint32_t p0 = p[0], p1 = p[32], p2 = p[64], p3 = p[96];
  return make_uint2(p0 | (p1 << 16), p2 | (p3 << 16));
}
__device__ __forceinline__ void store_span_f32(float* __restrict__ span, const double (&acc)[16], int lane) {
#pragma unroll
  for (int k = 0; k < 4; ++k)
    reinterpret_cast<float4*>(span)[k * 32 + lane] =
        make_float4(from_f64<float>(acc[4 * k]), from_f64<float>(acc[4 * k + 1]), from_f64<float>(acc[4 * k + 2]),
                    from_f64<float>(acc[4 * k + 3]));
}

// acc[i] (+)= T[code_i + 8] for the 16 INT4 codes in w (element order as
// fold16); `slot` = shared address of the source's table (256-byte aligned)
template <bool ASSIGN>
__device__ __forceinline__ void fold16_tbl4(const uint2& w, uint32_t slot, double (&acc)[16], bool& bad) {
  const uint32_t ww[2] = {w.x, w.y};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    bad |= has_nibble_8(ww[k]);
    const uint32_t b = ww[k] ^ 0x88888888u;     // biased nibbles c + 8
    const uint32_t ev = (b << 3) & 0x78787878u;  // 8 * (low nibble) in each byte
    const uint32_t od = (b >> 1) & 0x78787878u;  // 8 * (high nibble) in each byte
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const double v0 = lds_f64(__byte_perm(ev, slot, 0x7650 + j));
      const double v1 = lds_f64(__byte_perm(od, slot, 0x7650 + j));
      if constexpr (ASSIGN) {
        acc[8 * k + 2 * j] = v0;
        acc[8 * k + 2 * j + 1] = v1;
      } else {
        acc[8 * k + 2 * j] = __dadd_rn(acc[8 * k + 2 * j], v0);
        acc[8 * k + 2 * j + 1] = __dadd_rn(acc[8 * k + 2 * j + 1], v1);
      }
    }
  }
}

// K2 with INT4 sources through product tables (the qgZ hop-1 reduce with the
// INT4/512 intra codec): as drq_fast_kernel, for input blocks that are
// multiples of 512 (one scale per warp and source).  Every lane loads the
// block absmax even past the end of a partial last block, so the table inputs
// are warp-uniform.
// Hop-2 destinations of K2's output when hop 2 is pushed: segment c (L
// elements = seg_blocks output blocks of 512) of this rank's K2 output goes to
// rank (c, loc)'s hop-2 receive slot for this rank's node, so that rank's K3
// folds local HBM.  Pointers may be peers' symmetric memory (NVLink stores).
constexpr int kMaxHop = 8;
struct HopDst {
  uint8_t* codes[kMaxHop];   // slot start of segment c's codes (256 B per output block)
  double* absmax[kMaxHop];   // ... and of its f64 absmax
  int64_t seg_blocks;        // output blocks per segment (L / 512)
};

template <int OBITS, int NSRC, typename FO = void, int NT = NSRC, bool HOP = false>
__global__ void __launch_bounds__(256)
drq_tbl_kernel(SrcTable src, int64_t n, int lg1, int64_t n_blocks_out, uint8_t* __restrict__ codes,
               double* __restrict__ absmax, uint32_t* __restrict__ flag, FO* __restrict__ final_out = nullptr,
               int span_ok = 1, HopDst hop = HopDst{}) {
  if (comm_aborted(flag)) return;
  __shared__ __align__(256) double tbl_all[8][NT * kTblSlotDoubles];
  __shared__ __align__(64) float fo_all[8][16];
  const int tl = threadIdx.x & 31;
  double* tbl = tbl_all[threadIdx.x >> 5];
  const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(tbl);
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  bool bad = false;
  uint2 w[NSRC], wn[NSRC];
  float m[NSRC], mn[NSRC];
  // final fp32 output and whole blocks: coalesced layout (store_span_f32);
  // the fp32 table path of drq_epilogue is the only consumer, codes outputs
  // keep the per-lane order their packing needs
  // (not with one source: the four 16-bit loads cost more than the coalesced
  // stores gain there, 231 vs 224 us for the 1-GPU qgZ bucket)
  const bool span = span_ok && NSRC > 1 && std::is_same<FO, float>::value && OBITS == 4 && (n & 511) == 0;
  auto load = [&](int64_t b, uint2 (&wv)[NSRC], float (&mv)[NSRC]) {
    const int64_t e0 = b * 512 + (int64_t)tl * 16;
    const bool blk = b < n_blocks_out, ok = blk && e0 < n;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      wv[j] = !ok ? make_uint2(0, 0)
              : span ? int4_span_pieces_g(src.codes[j] + b * 256, tl)
                     : __ldg(reinterpret_cast<const uint2*>(src.codes[j]) + (e0 >> 4));
      mv[j] = blk ? __ldg(reinterpret_cast<const float*>(src.absmax[j]) + ((b * 512) >> lg1)) : 0.0f;
    }
  };
  int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  load(b, wn, mn);
  for (; b < n_blocks_out; b += nwarp) {
    const int64_t e0 = b * 512 + (int64_t)tl * 16;
    const bool active = e0 < n;
    const int64_t u = e0 >> 4;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      w[j] = wn[j];
      m[j] = mn[j];
    }
    load(b + nwarp, wn, mn);
    __syncwarp();  // the previous block's lookups are done before the tables change
    {
      float mt[NT];
#pragma unroll
      for (int j = 0; j < NT; ++j) mt[j] = m[j];
      tbl4_build<NT>(tbl, mt, tl);
    }
    __syncwarp();
    double acc[16];
    fold16_tbl4<true>(w[0], slot0, acc, bad);
#pragma unroll
    for (int j = 1; j < NSRC; ++j) {
      // sources past NT (development split): the plain product path
      if (j < NT) fold16_tbl4<false>(w[j], slot0 + j * 256, acc, bad);
      else fold16<4, true>(w[j], div_q_f32<7>(m[j]), acc, bad);
    }
    if constexpr (HOP) {
      // block b of segment c lands at block b - c*seg_blocks of c's slot (the
      // epilogue indexes codes by unit, 32 per block, and absmax by block)
      const int64_t c = b / hop.seg_blocks;
      const int64_t shift = c * hop.seg_blocks;
      drq_epilogue<OBITS, FO>(acc, b - shift, tl, e0, active, u - shift * 32, hop.codes[c], hop.absmax[c], flag,
                              final_out, fo_all[threadIdx.x >> 5], span);
    } else {
      drq_epilogue<OBITS, FO>(acc, b, tl, e0, active, u, codes, absmax, flag, final_out, fo_all[threadIdx.x >> 5],
                              span);
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
  if constexpr (HOP) __threadfence_system();  // the stores to peers are performed before the cross barrier's release
}

// K2 through a certified fp32 estimate (INT4 sources with fp32 absmax,
// 512-multiple input blocks, INT4/512 output).  The reference's value per
// element is the f64 fold acc = RN64(...RN64(T0[c0] + T1[c1])...) of the
// products Tj[c] = RN64(+0.0 + RN64(c * s_j)) (zs/quantizer.py:237,255-257),
// and only two things about it reach the output: the block's exact
// absmax M = max |acc| (stored in f64) and each code rint(RN64(acc * inv)),
// inv = RN64(7/M) (:218-226).  Here every element is first folded in fp32
// from per-block fp32 tables RN32(Tj[c]) (one LDS.32 per code, half the
// shared-memory wavefronts of the f64 tables); with S = sum_j 7 s_j,
//     |acc32 - acc| <= E = NSRC * 2^-22 * S
// (NSRC fp32 roundings of the tables and the adds, each <= 2^-24 S, plus the
// reference's own f64 roundings).  Then:
//   * absmax: the true argmax has |acc32| >= m32 - 2E (m32 = max |acc32|),
//     so the exact f64 fold of just those candidates (usually one element)
//     gives M bit-exactly;
//   * codes: with t = acc32 * RN32(inv) and e = t - rint(t) from one FFMA,
//     |t - acc*inv| < E*inv + 2^-20 =: G, so |e| <= 0.5 - G proves the code;
//     any other element (a near tie, ~G of them) is redone with the exact f64
//     fold and the reference's f64 requantization.
// Blocks whose scales are outside [2^-100, 2^100] (fp32 range/subnormal
// effects) take the exact f64 fold for every element.  Same bits as drq_tbl.
template <int NSRC, typename FO = void>
__global__ void __launch_bounds__(256, std::is_void<FO>::value ? 3 : 2)  // codes out: <= 85 registers, 3 CTAs/SM
drq_est_kernel(SrcTable src, int64_t n, int lg1, int64_t n_blocks_out, uint8_t* __restrict__ codes,
               double* __restrict__ absmax, uint32_t* __restrict__ flag, FO* __restrict__ final_out, int span_ok) {
  if (comm_aborted(flag)) return;
  constexpr int QMAX = 7;
  __shared__ __align__(256) float tbl_all[8][NSRC][64];  // 256-byte slot per (warp, source), 16 entries used
  __shared__ __align__(64) float fo_all[8][16];
  const int tl = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(&tbl_all[wid][0][0]);
  float* fo_tbl = fo_all[wid];
  const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool span = span_ok && NSRC > 1 && std::is_same<FO, float>::value && (n & 511) == 0;
  bool bad = false;
  uint2 w[NSRC], wn[NSRC];
  float m[NSRC], mn[NSRC];
  auto load = [&](int64_t b, uint2 (&wv)[NSRC], float (&mv)[NSRC]) {
    const int64_t e0 = b * 512 + (int64_t)tl * 16;
    const bool blk = b < n_blocks_out, ok = blk && e0 < n;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      wv[j] = !ok ? make_uint2(0, 0)
              : span ? int4_span_pieces_g(src.codes[j] + b * 256, tl)
                     : __ldg(reinterpret_cast<const uint2*>(src.codes[j]) + (e0 >> 4));
      mv[j] = blk ? __ldg(reinterpret_cast<const float*>(src.absmax[j]) + ((b * 512) >> lg1)) : 0.0f;
    }
  };
  int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  load(b, wn, mn);
  for (; b < n_blocks_out; b += nwarp) {
    const int64_t e0 = b * 512 + (int64_t)tl * 16;
    const bool active = e0 < n;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      w[j] = wn[j];
      m[j] = mn[j];
    }
    load(b + nwarp, wn, mn);
#pragma unroll
    for (int j = 0; j < NSRC; ++j) bad |= has_nibble_8(w[j].x) | has_nibble_8(w[j].y);
    // exact f64 scales (warp-uniform) and the error budget
    double sc[NSRC];
    double S = 0.0;
    bool wild = false;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      sc[j] = div_q_f32<QMAX>(m[j]);
      S += 7.0 * sc[j];
      wild |= sc[j] != 0.0 && !(sc[j] >= 0x1p-100 && sc[j] <= 0x1p100);
    }
    const double E = S * (double)NSRC * 0x1p-22 * (1.0 + 0x1p-20);
    // fp32 tables: lanes 16h + k build entry k of source 2p + h
    __syncwarp();  // the previous block's lookups are done
#pragma unroll
    for (int p = 0; p < (NSRC + 1) / 2; ++p) {
      const int j = 2 * p + (tl >> 4);
      if (j < NSRC) {
        const double sj = (tl >> 4) ? sc[2 * p + 1 < NSRC ? 2 * p + 1 : 2 * p] : sc[2 * p];
        tbl_all[wid][j][tl & 15] = __double2float_rn(__dadd_rn(0.0, __dmul_rn((double)((tl & 15) - 8), sj)));
      }
    }
    __syncwarp();
    // exact f64 fold of element i of this lane (the reference's arithmetic)
    auto exact = [&](int i) -> double {
      const int sh = 4 * (i & 7);
      double a = 0.0;
#pragma unroll
      for (int j = 0; j < NSRC; ++j) {
        const uint32_t word = (i < 8) ? w[j].x : w[j].y;
        const int c = (int)(((word >> sh) & 0xFu) ^ 8u) - 8;
        const double pr = __dmul_rn((double)c, sc[j]);
        a = j == 0 ? __dadd_rn(0.0, pr) : __dadd_rn(a, pr);
      }
      return a;
    };
    // fp32 fold through the tables (element order as fold16_tbl4)
    float acc[16];
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      const uint32_t slot = slot0 + j * 256;
      const uint32_t ww[2] = {w[j].x, w[j].y};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const uint32_t bb = ww[k] ^ 0x88888888u;
        const uint32_t ev = (bb << 2) & 0x3C3C3C3Cu;  // 4 * (low nibble) per byte
        const uint32_t od = (bb >> 2) & 0x3C3C3C3Cu;  // 4 * (high nibble) per byte
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float v0, v1;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v0) : "r"(__byte_perm(ev, slot, 0x7650 + q)) : "memory");
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v1) : "r"(__byte_perm(od, slot, 0x7650 + q)) : "memory");
          if (j == 0) {
            acc[8 * k + 2 * q] = v0;
            acc[8 * k + 2 * q + 1] = v1;
          } else {  // one FADD2 for the pair
            const float2 r = fadd2(make_float2(acc[8 * k + 2 * q], acc[8 * k + 2 * q + 1]), make_float2(v0, v1));
            acc[8 * k + 2 * q] = r.x;
            acc[8 * k + 2 * q + 1] = r.y;
          }
        }
      }
    }
    // exact absmax: candidates within 2E of the estimated max
    float lm = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) lm = fmaxf(lm, fabsf(acc[i]));
    const float m32 = __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(lm)));
    const double thr = wild ? -1.0 : (double)m32 - 2.0 * E;
    double lmax = 0.0;
    if ((double)lm >= thr) {  // rare: the lanes holding a candidate (every lane of a wild block)
#pragma unroll
      for (int i = 0; i < 16; ++i)  // unrolled: acc[] stays in registers
        if (wild || (double)fabsf(acc[i]) >= thr) lmax = dmax_nn(lmax, fabs(exact(i)));
    }
    const double mx = warp_max_nonneg(lmax);
    if (tl == 0) {
      absmax[b] = mx;
      if (!(mx <= DBL_MAX)) raise_flag(flag, FLAG_NONFINITE);
    }
    const double inv = mx > 0.0 ? __ddiv_rn((double)QMAX, mx) : 0.0;
    const float inv32 = __double2float_rn(inv);
    // |e| <= 0.5 - G proves the code; G >= 0.5 (heavy cancellation) sends every element to the exact path
    const float guard = wild ? -1.0f : __double2float_rd(0.5 - (E * inv + 0x1p-20));
    uint32_t q[16];
    float emax = 0.0f;
    {
      const float2 inv2 = make_float2(inv32, inv32), m2 = make_float2(kMagic23, kMagic23);
#pragma unroll
      for (int i = 0; i < 8; ++i) {  // FFMA2 / FADD2 / FFMA2 per pair
        const float2 x = make_float2(acc[2 * i], acc[2 * i + 1]);
        const float2 u = ffma2(x, inv2, m2);
        const float2 nk = fadd2(m2, make_float2(-u.x, -u.y));
        const float2 ee = ffma2(x, inv2, nk);
        q[2 * i] = __float_as_uint(u.x);
        q[2 * i + 1] = __float_as_uint(u.y);
        emax = fmaxf(emax, fmaxf(fabsf(ee.x), fabsf(ee.y)));
      }
    }
    if (!(emax <= guard)) {  // rare: the reference's requantization for the unproven elements
#pragma unroll
      for (int i = 0; i < 16; ++i) {  // unrolled: q[] stays in registers
        const float ei = __fmaf_rn(acc[i], inv32, kMagic23 - __uint_as_float(q[i]));
        if (!(fabsf(ei) <= guard)) q[i] = (uint32_t)__double2loint(__dadd_rn(__dmul_rn(exact(i), inv), kMagic52));
      }
    }
    if constexpr (std::is_void<FO>::value) {
      // inactive lanes hold zero codes: the zero padding of a partial last block
      uint32_t q0[8], q1[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        q0[i] = q[i];
        q1[i] = q[8 + i];
      }
      *reinterpret_cast<uint2*>(codes + (e0 >> 4) * 8) = make_uint2(pack8_int4(q0), pack8_int4(q1));
    } else {
      static_assert(sizeof(FO) == 4, "fp32 final output");
      const double s2 = scale_of<4>(mx);
      __syncwarp();  // the previous block's FO lookups are done
      if (tl < 16) fo_tbl[tl] = __double2float_rn(__dadd_rn(0.0, __dmul_rn((double)(tl - 8), s2)));
      __syncwarp();
      if (active) {
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = fo_tbl[((int)(q[i] << 28) >> 28) + 8];  // low nibble = code
        if (span) {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(final_out) + b * 512);
#pragma unroll
          for (int k = 0; k < 4; ++k) dst[k * 32 + tl] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        } else {
          float* dst = reinterpret_cast<float*>(final_out) + e0;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            reinterpret_cast<float4*>(dst)[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        }
      }
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// qgZ with one GPU per group (X = 1): hop 1 is a self-send, and K2 would
// requantize the dequantized codes of a single source with the same block
// (zs/quantizer.py:241-258).  That reproduces every code exactly -- the max
// element's code is +-QMAX, so maxabs = RN64(QMAX*s) and
// RN64(RN64(c*s) * RN64(QMAX/maxabs)) = c*(1 + e) with |c*e| <= QMAX*2^-50 --
// so hop 2 sends K1's codes as they are, and this kernel writes only the f64
// block absmax RN64(QMAX * RN64(m/QMAX)) that K2 would have produced.
template <int QMAX>
__global__ void __launch_bounds__(256)
hop_absmax_x1_kernel(const float* __restrict__ m, int64_t nb, double* __restrict__ out, uint32_t* __restrict__ flag) {
  if (comm_aborted(flag)) return;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    out[b] = __dmul_rn((double)QMAX, div_q_f32<QMAX>(__ldg(m + b)));
}

// K3 fixed fan-in fast path (the qgZ hop-2 fold, zs/collectives.py:536-544):
// NSRC sources known at compile time, power-of-two block, fp32/f64 output;
// lane = 16 contiguous elements, grid-stride, next unit's codes and absmax
// loaded before this unit is folded (the sources are peers' HBM).  The first
// source assigns (see fold16).  Same arithmetic as dr_unit.
template <int BITS, int NSRC, typename A, typename O, bool TBL = false>
__global__ void __launch_bounds__(256)
dr_fast_kernel(SrcTable src, int64_t n, int lg, O* __restrict__ out, double post_scale, uint32_t* __restrict__ flag,
               int span_ok = 1) {
  if (comm_aborted(flag)) return;
  static_assert(!TBL || BITS == 4, "product tables are for INT4 sources");
  using V = typename Vec16<BITS>::T;
  // TBL (INT4, blocks of >= 512 elements): a warp's 32 units share one block
  // per source, whose absmax every lane loads (warp-uniform table inputs)
  __shared__ __align__(256) double tbl_all[TBL ? 8 : 1][TBL ? NSRC * kTblSlotDoubles : 1];
  const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(&tbl_all[TBL ? (threadIdx.x >> 5) : 0][0]);
  const int64_t units = n / 16;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  V w[NSRC], wn[NSRC];
  A m[NSRC], mn[NSRC];
  // TBL with fp32 output and whole 512-element warp spans: coalesced layout
  // (see store_span_f32); warp-uniform
  constexpr bool CAN_SPAN = TBL && sizeof(O) == 4;
  const bool span = CAN_SPAN && span_ok && (n & 511) == 0;
  const int lane = threadIdx.x & 31;
  auto load = [&](int64_t u, V (&wv)[NSRC], A (&mv)[NSRC]) {
    const int64_t ua = TBL ? (u & ~int64_t(31)) : u;
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      if constexpr (CAN_SPAN) {
        if (span) {
          wv[j] = u < units ? int4_span_pieces_g(src.codes[j] + ua * 8, lane) : V{};
        } else {
          wv[j] = u < units ? __ldg(reinterpret_cast<const V*>(src.codes[j]) + u) : V{};
        }
      } else {
        wv[j] = u < units ? __ldg(reinterpret_cast<const V*>(src.codes[j]) + u) : V{};
      }
      mv[j] = ua < units ? __ldg(reinterpret_cast<const A*>(src.absmax[j]) + ((ua * 16) >> lg)) : A(0);
    }
  };
  int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  load(u, wn, mn);
  for (; (TBL ? (u & ~int64_t(31)) : u) < units; u += stride) {
#pragma unroll
    for (int j = 0; j < NSRC; ++j) {
      w[j] = wn[j];
      m[j] = mn[j];
    }
    load(u + stride, wn, mn);
    double acc[16];
    if constexpr (TBL) {
      double md[NSRC];
#pragma unroll
      for (int j = 0; j < NSRC; ++j) md[j] = (double)m[j];
      __syncwarp();
      tbl4_build<NSRC>(&tbl_all[threadIdx.x >> 5][0], md, threadIdx.x & 31);
      __syncwarp();
      if (u >= units) continue;
      fold16_tbl4<true>(w[0], slot0, acc, bad);
#pragma unroll
      for (int j = 1; j < NSRC; ++j) fold16_tbl4<false>(w[j], slot0 + j * 256, acc, bad);
    } else {
      fold16<BITS, true, true>(w[0], scale_of<BITS>((double)m[0]), acc, bad);
#pragma unroll
      for (int j = 1; j < NSRC; ++j) fold16<BITS, true>(w[j], scale_of<BITS>((double)m[j]), acc, bad);
    }
    if (post_scale != 1.0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = __dmul_rn(acc[i], post_scale);
    }
    O* dst = out + u * 16;
    if constexpr (CAN_SPAN) {
      if (span) {
        store_span_f32(reinterpret_cast<float*>(out + (u & ~int64_t(31)) * 16), acc, lane);
        continue;
      }
    }
    if constexpr (sizeof(O) == 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        reinterpret_cast<float4*>(dst)[i] = make_float4(from_f64<float>(acc[4 * i]), from_f64<float>(acc[4 * i + 1]),
                                                        from_f64<float>(acc[4 * i + 2]), from_f64<float>(acc[4 * i + 3]));
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) reinterpret_cast<double2*>(dst)[i] = make_double2(acc[2 * i], acc[2 * i + 1]);
    }
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// ---------------------------------------------------------------------------
// K2 / K3 fed by TMA (the multi-GPU qgZ hops).  Their sources are slices of
// peers' symmetric buffers: plain per-thread loads over NVLink stall at a few
// hundred GB/s, so one elected thread streams each tile's codes and absmax of
// every source with cp.async.bulk into a STAGES-deep shared ring (mbarrier
// transaction counts), and all 256 threads fold from shared memory.  A tile
// is `tu` 16-element units of every source.  Bulk copies need 16-byte aligned
// addresses and sizes, so each absmax slice is widened to 16-byte bounds and
// the last codes slice rounded up: the host only uses these kernels on the
// communicator's symmetric regions, which are padded to 256 bytes.

struct TmaTile {
  int tu;             // units (16 elements) per tile
  int lg;             // log2 of the input block size
  int code_slot;      // bytes per source codes slot (16-aligned)
  int abs_slot;       // bytes per source absmax slot (16-aligned)
  int stage_bytes;    // NSRC * (code_slot + abs_slot)
};

template <int BITS, int NSRC, typename A>
__device__ __forceinline__ void tma_issue_tile(const SrcTable& src, const TmaTile& tt, int64_t units, int64_t t,
                                               uint8_t* stage, uint64_t* bar) {
  constexpr int UB = 2 * BITS;  // bytes per unit of codes
  const int64_t u0 = t * tt.tu;
  const int64_t nu = min((int64_t)tt.tu, units - u0);
  const uint32_t cbytes = (uint32_t)((nu * UB + 15) & ~15);
  const int64_t b_first = (u0 * 16) >> tt.lg, b_last = ((u0 + nu) * 16 - 1) >> tt.lg;
  uint32_t total = 0;
#pragma unroll
  for (int j = 0; j < NSRC; ++j) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(src.absmax[j]) + (uintptr_t)b_first * sizeof(A);
    const uintptr_t a1 = reinterpret_cast<uintptr_t>(src.absmax[j]) + (uintptr_t)(b_last + 1) * sizeof(A);
    total += cbytes + (uint32_t)(((a1 + 15) & ~(uintptr_t)15) - (a0 & ~(uintptr_t)15));
  }
  mbar_expect_tx(bar, total);
#pragma unroll
  for (int j = 0; j < NSRC; ++j) {
    uint8_t* slot = stage + j * (tt.code_slot + tt.abs_slot);
    bulk_g2s(slot, src.codes[j] + u0 * UB, cbytes, bar);
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(src.absmax[j]) + (uintptr_t)b_first * sizeof(A);
    const uintptr_t a1 = reinterpret_cast<uintptr_t>(src.absmax[j]) + (uintptr_t)(b_last + 1) * sizeof(A);
    const uintptr_t lo = a0 & ~(uintptr_t)15;
    bulk_g2s(slot + tt.code_slot, reinterpret_cast<const void*>(lo), (uint32_t)(((a1 + 15) & ~(uintptr_t)15) - lo), bar);
  }
}

// absmax of input block b (first block of tile: b_first) of source j in a stage
template <typename A>
__device__ __forceinline__ double tma_absmax(const SrcTable& src, int j, const uint8_t* slot_abs, int64_t b_first,
                                             int64_t b) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(src.absmax[j]) + (uintptr_t)b_first * sizeof(A);
  const int skew = (int)(a0 & 15);
  return (double)*reinterpret_cast<const A*>(slot_abs + skew + (b - b_first) * sizeof(A));
}

// K2 (hop-1 fold + requant into 512-element blocks, or the final partition
// when hop 2 is a self-send): fp32 absmax sources, warp = output block.
template <int IBITS, int OBITS, int NSRC, typename FO, int STAGES, bool TBL = false, bool SPAN = false>
__global__ void __launch_bounds__(256)
drq_tma_kernel(SrcTable src, int64_t n, TmaTile tt, uint8_t* __restrict__ codes, double* __restrict__ absmax,
               uint32_t* __restrict__ flag, FO* __restrict__ final_out) {
  if (comm_aborted(flag)) return;
  static_assert(!TBL || IBITS == 4, "product tables are for INT4 sources");
  using V = typename Vec16<IBITS>::T;
  constexpr int UB = 2 * IBITS;
  extern __shared__ __align__(128) uint8_t dsm[];
  // TBL (INT4 sources, input blocks of >= 512 elements): one product table per
  // (warp, source), see tbl4_build
  __shared__ __align__(256) double tbl_all[TBL ? 8 : 1][TBL ? NSRC * kTblSlotDoubles : 1];
  __shared__ __align__(64) float fo_all[8][16];
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)STAGES * tt.stage_bytes);
  const int tid = threadIdx.x, tl = tid & 31, wid = tid >> 5;
  const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(&tbl_all[TBL ? wid : 0][0]);
  const int64_t units = n / 16;
  const int64_t tiles = (units + tt.tu - 1) / tt.tu;
  const int64_t G = gridDim.x;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < STAGES - 1; ++k)
      if (blockIdx.x + k * G < tiles)
        tma_issue_tile<IBITS, NSRC, float>(src, tt, units, blockIdx.x + k * G, dsm + (size_t)k * tt.stage_bytes,
                                           &full[k]);
  }
  bool bad = false;
  // final fp32 output through the product tables, whole blocks: coalesced
  // layout (store_span_f32); a template choice (the host checks n % 512 == 0)
  // because a runtime switch took the kernel from 80 to 124 registers
  static_assert(!SPAN || (TBL && std::is_same<FO, float>::value && OBITS == 4), "span layout: fp32 table path only");
  constexpr bool span = SPAN;
  int k = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += G, ++k) {
    const int slot = k % STAGES;
    if (tid == 0) {
      const int64_t tn = t + (STAGES - 1) * G;
      const int sn = (k + STAGES - 1) % STAGES;
      if (tn < tiles) tma_issue_tile<IBITS, NSRC, float>(src, tt, units, tn, dsm + (size_t)sn * tt.stage_bytes, &full[sn]);
    }
    mbar_wait(&full[slot], (uint32_t)((k / STAGES) & 1));
    const uint8_t* stage = dsm + (size_t)slot * tt.stage_bytes;
    const int64_t u0 = t * tt.tu;
    const int64_t b_first = (u0 * 16) >> tt.lg;
    for (int ob = wid; ob < tt.tu / 32; ob += 8) {  // output block = 32 units
      const int lu = ob * 32 + tl;
      const int64_t unit = u0 + lu;
      const bool active = unit < units;
      if (u0 + ob * 32 >= units) break;  // warp-uniform: block entirely past the end
      double acc[16];
      if constexpr (TBL) {
        // the warp's 512 elements share one input block per source
        const int64_t bw = ((u0 + ob * 32) * 16) >> tt.lg;
        float m[NSRC];
#pragma unroll
        for (int j = 0; j < NSRC; ++j)
          m[j] = (float)tma_absmax<float>(src, j, stage + j * (tt.code_slot + tt.abs_slot) + tt.code_slot, b_first, bw);
        __syncwarp();  // the previous block's lookups are done before the tables change
        tbl4_build<NSRC>(&tbl_all[wid][0], m, tl);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < NSRC; ++j) {
          const uint8_t* sl = stage + j * (tt.code_slot + tt.abs_slot);
          const uint2 w = !active ? make_uint2(0, 0)
                          : span ? int4_span_pieces_s(sl + (lu & ~31) * UB, tl)
                                 : *reinterpret_cast<const uint2*>(sl + lu * UB);
          if (j == 0) fold16_tbl4<true>(w, slot0, acc, bad);
          else fold16_tbl4<false>(w, slot0 + j * 256, acc, bad);
        }
      } else {
#pragma unroll
        for (int j = 0; j < NSRC; ++j) {
          const uint8_t* sl = stage + j * (tt.code_slot + tt.abs_slot);
          V w = active ? *reinterpret_cast<const V*>(sl + lu * UB) : V{};
          const double m = active ? tma_absmax<float>(src, j, sl + tt.code_slot, b_first, (unit * 16) >> tt.lg) : 0.0;
          const double sc = div_q_f32<Codes<IBITS>::kQmax>((float)m);
          if (j == 0) fold16<IBITS, true, true>(w, sc, acc, bad);
          else fold16<IBITS, true>(w, sc, acc, bad);
        }
      }
      if (!active) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0.0;  // zero padding of a partial last block
      }
      drq_epilogue<OBITS, FO>(acc, (u0 + ob * 32) / 32, tl, unit * 16, active, unit, codes, absmax, flag, final_out,
                              TBL ? fo_all[wid] : nullptr, span);
    }
    __syncthreads();  // every thread is done with this slot before it is refilled
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// K3 (hop-2 fold into the rank's partition): f64 absmax sources from K2.
template <int BITS, int NSRC, typename O, int STAGES, bool TBL = false, bool SPAN = false>
__global__ void __launch_bounds__(256)
dr_tma_kernel(SrcTable src, int64_t n, TmaTile tt, O* __restrict__ out, uint32_t* __restrict__ flag) {
  if (comm_aborted(flag)) return;
  static_assert(!TBL || BITS == 4, "product tables are for INT4 sources");
  using V = typename Vec16<BITS>::T;
  constexpr int UB = 2 * BITS;
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(256) double tbl_all[TBL ? 8 : 1][TBL ? NSRC * kTblSlotDoubles : 1];
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)STAGES * tt.stage_bytes);
  const int tid = threadIdx.x;
  const int wid = tid >> 5;
  const uint32_t slot0 = (uint32_t)__cvta_generic_to_shared(&tbl_all[TBL ? wid : 0][0]);
  const int64_t units = n / 16;
  const int64_t tiles = (units + tt.tu - 1) / tt.tu;
  const int64_t G = gridDim.x;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < STAGES - 1; ++k)
      if (blockIdx.x + k * G < tiles)
        tma_issue_tile<BITS, NSRC, double>(src, tt, units, blockIdx.x + k * G, dsm + (size_t)k * tt.stage_bytes,
                                           &full[k]);
  }
  bool bad = false;
  // TBL with fp32 output and whole 512-element warp spans: coalesced layout
  // (a template choice; the host checks n % 512 == 0)
  static_assert(!SPAN || (TBL && sizeof(O) == 4), "span layout: fp32 table path only");
  constexpr bool span = SPAN;
  int k = 0;
  for (int64_t t = blockIdx.x; t < tiles; t += G, ++k) {
    const int slot = k % STAGES;
    if (tid == 0) {
      const int64_t tn = t + (STAGES - 1) * G;
      const int sn = (k + STAGES - 1) % STAGES;
      if (tn < tiles) tma_issue_tile<BITS, NSRC, double>(src, tt, units, tn, dsm + (size_t)sn * tt.stage_bytes, &full[sn]);
    }
    mbar_wait(&full[slot], (uint32_t)((k / STAGES) & 1));
    const uint8_t* stage = dsm + (size_t)slot * tt.stage_bytes;
    const int64_t u0 = t * tt.tu;
    const int64_t b_first = (u0 * 16) >> tt.lg;
    for (int lu = tid; lu < tt.tu; lu += 256) {
      const int64_t unit = u0 + lu;
      double acc[16];
      if constexpr (TBL) {
        // warp = 32 units = 512 elements inside one block of every source
        const int64_t uw = u0 + (lu & ~31);
        if (uw >= units) break;  // warp-uniform
        const int64_t bw = (uw * 16) >> tt.lg;
        double m[NSRC];
#pragma unroll
        for (int j = 0; j < NSRC; ++j)
          m[j] = tma_absmax<double>(src, j, stage + j * (tt.code_slot + tt.abs_slot) + tt.code_slot, b_first, bw);
        __syncwarp();
        tbl4_build<NSRC>(&tbl_all[wid][0], m, tid & 31);
        __syncwarp();
        if (unit >= units) continue;  // past the end (the warp's last loop trip)
#pragma unroll
        for (int j = 0; j < NSRC; ++j) {
          const uint8_t* sj = stage + j * (tt.code_slot + tt.abs_slot);
          const uint2 w = span ? int4_span_pieces_s(sj + (lu & ~31) * UB, tid & 31)
                               : *reinterpret_cast<const uint2*>(sj + lu * UB);
          if (j == 0) fold16_tbl4<true>(w, slot0, acc, bad);
          else fold16_tbl4<false>(w, slot0 + j * 256, acc, bad);
        }
        if constexpr (sizeof(O) == 4) {
          if (span) {  // coalesced layout, see store_span_f32
            store_span_f32(reinterpret_cast<float*>(out + (u0 + (lu & ~31)) * 16), acc, tid & 31);
            continue;
          }
        }
      } else {
        if (unit >= units) break;
#pragma unroll
        for (int j = 0; j < NSRC; ++j) {
          const uint8_t* sl = stage + j * (tt.code_slot + tt.abs_slot);
          const V w = *reinterpret_cast<const V*>(sl + lu * UB);
          const double sc = scale_of<BITS>(tma_absmax<double>(src, j, sl + tt.code_slot, b_first, (unit * 16) >> tt.lg));
          if (j == 0) fold16<BITS, true, true>(w, sc, acc, bad);
          else fold16<BITS, true>(w, sc, acc, bad);
        }
      }
      O* dst = out + unit * 16;
      if constexpr (sizeof(O) == 4) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          reinterpret_cast<float4*>(dst)[i] = make_float4(from_f64<float>(acc[4 * i]), from_f64<float>(acc[4 * i + 1]),
                                                          from_f64<float>(acc[4 * i + 2]), from_f64<float>(acc[4 * i + 3]));
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) reinterpret_cast<double2*>(dst)[i] = make_double2(acc[2 * i], acc[2 * i + 1]);
      }
    }
    __syncthreads();
  }
  if (bad) raise_flag(flag, FLAG_BADCODE);
}

// Wire format on the device (QuantizedTensor.to_bytes / from_bytes,
// zs/quantizer.py:121-149): 13-byte '<QBI' header, fp16 scales, packed codes
// (incl. padding), contiguous and unaligned after the header.

// f64 -> fp16 bits, round to nearest even, subnormals and overflow to inf
// included (numpy's float64.astype(float16), zs/quantizer.py:130), in integer
// arithmetic so no intermediate rounding can intervene.
__device__ __forceinline__ uint16_t f64_to_f16_bits(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  const uint16_t sign = (uint16_t)((b >> 48) & 0x8000u);
  const int e = (int)((b >> 52) & 0x7FF);
  const uint64_t man = b & ((1ull << 52) - 1);
  if (e == 0x7FF) return sign | (man ? 0x7E00u : 0x7C00u);
  const int ue = e - 1023;        // unbiased exponent
  if (ue < -25) return sign;      // below half the smallest subnormal (2^-25 ties to even: 0)
  const uint64_t sig = (1ull << 52) | man;  // e > 0 here (f64 subnormals are < 2^-25)
  // fp16 value = sig * 2^(ue-52); in units of 2^-24 (subnormal ulp) when
  // ue < -14, else with an implicit bit and a 10-bit mantissa
  const int shift = ue < -14 ? (52 - (ue + 24)) : 42;
  uint64_t m = sig >> shift;
  const uint64_t rem = sig & ((1ull << shift) - 1), half = 1ull << (shift - 1);
  if (rem > half || (rem == half && (m & 1))) ++m;
  if (ue < -14) return sign | (uint16_t)m;  // m <= 1024: 1024 is the smallest normal, 0x0400
  int E = ue + 15;
  if (m == (1ull << 11)) {  // mantissa overflowed into the next binade
    m >>= 1;
    ++E;
  }
  if (E >= 31) return sign | 0x7C00u;
  return sign | (uint16_t)(E << 10) | (uint16_t)(m & 0x3FF);
}

__device__ __forceinline__ void st_u8(uint8_t* p, uint32_t v) {
  asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// pack: header + fp16 scales (the codes follow by a device-to-device copy)
template <int BITS, typename A>
__global__ void wire_pack_kernel(const A* __restrict__ absmax, int64_t nb, uint64_t hdr_lo, uint64_t hdr_hi,
                                 uint8_t* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i0 < 13) st_u8(out + i0, (uint32_t)((i0 < 8 ? (hdr_lo >> (8 * i0)) : (hdr_hi >> (8 * (i0 - 8)))) & 0xFF));
  for (int64_t b = i0; b < nb; b += stride) {
    const uint32_t u = f64_to_f16_bits(scale_of<BITS>(absmax_f64<A>(absmax, b)));
    st_u8(out + 13 + 2 * b, u & 0xFF);
    st_u8(out + 14 + 2 * b, u >> 8);
  }
}

// unpack: fp16 wire scales -> f64 absmax = scale16 * qmax (exact), codes copied
// (the codes are copied device-to-device by the host)
template <int BITS>
__global__ void wire_unpack_kernel(const uint8_t* __restrict__ raw, int64_t nb, double* __restrict__ absmax) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t b = i0; b < nb; b += stride) {
    const uint32_t lo = raw[13 + 2 * b], hi = raw[14 + 2 * b];
    const uint16_t u = (uint16_t)(lo | (hi << 8));
    absmax[b] = __dmul_rn((double)__half2float(__ushort_as_half(u)), (double)Codes<BITS>::kQmax);
  }
}

// f64 scales from absmax (QuantizedTensor.scales; zs/quantizer.py:219)
template <int BITS, typename A>
__global__ void scales_kernel(const A* __restrict__ absmax, int64_t nb, double* __restrict__ out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += stride)
    out[i] = scale_of<BITS>(absmax_f64<A>(absmax, i));
}

}  // namespace zpp
