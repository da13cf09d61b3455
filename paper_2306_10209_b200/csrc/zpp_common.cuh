// Shared device helpers for the ZeRO++ codec kernels (sm_100a).
//
// Numerics contract (reference: zs/quantizer.py:204-258):
//   scale = f64(absmax) / qmax,  inv = qmax / f64(absmax) (0 if absmax == 0)
//   code  = clip(rint_even(f64(x) * inv), -qmax, qmax)
//   value = f64(code) * scale ; reductions fold in f64 from +0.0, ascending source.
// Every operation below is an explicit _rn intrinsic or an exactness-preserving
// integer trick, so nvcc can neither contract nor reorder them.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace zpp {

enum DType : int { F32 = 0, F16 = 1, BF16 = 2, F64 = 3 };

enum Flag : uint32_t {
  FLAG_NONFINITE = 1u,  // non-finite input value (reference: ValidationError)
  FLAG_BADCODE = 2u,    // code outside the symmetric range (reference: IntegrityError)
  FLAG_TIMEOUT = 4u,    // a peer never arrived at a device barrier
};

__device__ __forceinline__ void raise_flag(uint32_t* flag, uint32_t bit) {
  if (flag) atomicOr(flag, bit);
}

// A device barrier of this flag's communicator timed out: the ranks' epochs
// are out of step and peers' buffers may be stale or half written, so every
// data kernel sharing the flag returns without touching its buffers until the
// host clears the condition (Communicator.recover()).  One load per thread at
// kernel entry.
//
// It is also every kernel's programmatic-dependent-launch point: a kernel the
// communicator launches with programmatic stream serialization (launch_k under
// PdlScope) may be scheduled while its predecessor is still finishing, so it
// first waits for the predecessor grid to complete and its memory to be
// visible (griddepcontrol.wait), then lets its own successor be scheduled
// (griddepcontrol.launch_dependents).  Both are no-ops for a normal launch.
__device__ __forceinline__ bool comm_aborted(const uint32_t* flag) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  return flag && (*reinterpret_cast<const volatile uint32_t*>(flag) & FLAG_TIMEOUT);
}

// ---------------------------------------------------------------------------
// exact helpers

// f64 division by the constant qmax (127 or 7), correctly rounded.
// q0 = RN(m * RN(1/Q)); e = m - q0*Q (exact through FMA); RN(q0 + e * RN(1/Q))
// is the correctly rounded quotient for normal m (Markstein); verified against
// __ddiv_rn on every positive fp32 value and 2^30 random doubles in
// tests/test_gpu_codec.py.
template <int Q>
__device__ __forceinline__ double div_q(double m) {
  constexpr double r = 1.0 / Q;
  if (m < 1e-290) return __ddiv_rn(m, (double)Q);  // keep the proof's no-underflow premise
  double q0 = __dmul_rn(m, r);
  double e = __fma_rn(-q0, (double)Q, m);
  return __fma_rn(e, r, q0);
}

// int code c in [-128, 127] given as the byte (c + 128) -> exact double c.
// 2^52 + 2^51 has an all-zero low word, so OR-ing an unsigned value u < 2^31
// into it gives exactly 2^52 + 2^51 + u; one exact subtraction recovers u - bias.
__device__ __forceinline__ double biased_to_f64(uint32_t u, double magic_plus_bias) {
  return __dsub_rn(__hiloint2double(0x43380000, (int)u), magic_plus_bias);
}
constexpr double kMagic52 = 6755399441055744.0;  // 2^52 + 2^51

// round-half-even of a double to int via the 2^52+2^51 trick (|t| < 2^31).
__device__ __forceinline__ int rint_f64(double t) {
  return __double2loint(__dadd_rn(t, kMagic52));
}

// max(mx, a) for a running absmax mx >= 0 as one DSETP and two selects (fmax
// also handles signaling NaNs: 8 instructions in SASS).  Like fmax it keeps mx
// when a is NaN and keeps +inf, so the callers' !(mx <= DBL_MAX) flag is unchanged.
__device__ __forceinline__ double dmax_nn(double mx, double a) { return a > mx ? a : mx; }

// max |acc[i]| over 16 values, carrying the signed value and comparing
// magnitudes (DSETP with |.| operands, then one select per word), so no fabs
// is materialised per element (the compiler emits it as a DADD); the
// magnitude is taken once at the end.  A sequential chain: a pairwise tree
// keeps 8 more doubles live and took K2 from 80 to 104 registers.  NaNs lose
// every comparison (kept only in slot 0); the callers test !(mx <= DBL_MAX).
// Warp-wide max of non-negative doubles (or NaN/inf) in two redux.sync
// integer reductions: a non-negative double's bit pattern orders like its
// value, so the max has the largest high word and, among the lanes holding
// that high word, the largest low word.  Replaces five shuffle + DSETP +
// 2 select levels (25 instructions per lane).  NaN high words (0x7FF8...)
// exceed every finite and infinite one, so a NaN anywhere gives NaN, which the
// callers' !(mx <= DBL_MAX) test flags.
__device__ __forceinline__ double warp_max_nonneg(double x) {
  const unsigned hi = (unsigned)__double2hiint(x), lo = (unsigned)__double2loint(x);
  const unsigned H = __reduce_max_sync(0xffffffffu, hi);
  const unsigned L = __reduce_max_sync(0xffffffffu, hi == H ? lo : 0u);
  return __hiloint2double((int)H, (int)L);
}

__device__ __forceinline__ double absmax16(const double (&a)[16]) {
  double m = a[0];
#pragma unroll
  for (int i = 1; i < 16; ++i) m = fabs(a[i]) > fabs(m) ? a[i] : m;
  return fabs(m);
}

constexpr float kMagic23 = 12582912.0f;  // 1.5 * 2^23: x + kMagic23 rounds x to an integer
// quantize fast-path guard: |e| <= 0.5 - 2^-15 (see quant_chunk in zpp_kernels.cuh)
constexpr float kTieGuard = 0.5f - 3.0517578125e-05f;

template <int QMAX>
__device__ __forceinline__ uint32_t q_exact(double x, double inv64) {
  int k = rint_f64(__dmul_rn(x, inv64));
  k = k > QMAX ? QMAX : (k < -QMAX ? -QMAX : k);
  return (uint32_t)k;
}

// ---------------------------------------------------------------------------
// packing: 8 codes (low byte of each word = two's complement code)

__device__ __forceinline__ uint2 pack8_int8(const uint32_t (&b)[8]) {
  uint32_t lo = __byte_perm(__byte_perm(b[0], b[1], 0x0040), __byte_perm(b[2], b[3], 0x0040), 0x5410);
  uint32_t hi = __byte_perm(__byte_perm(b[4], b[5], 0x0040), __byte_perm(b[6], b[7], 0x0040), 0x5410);
  return make_uint2(lo, hi);
}

// byte i = (c[2i] & 0xF) | (c[2i+1] & 0xF) << 4   (zs/quantizer.py:188-189)
__device__ __forceinline__ uint32_t pack8_int4(const uint32_t (&b)[8]) {
  uint32_t ev = __byte_perm(__byte_perm(b[0], b[2], 0x0040), __byte_perm(b[4], b[6], 0x0040), 0x5410);
  uint32_t od = __byte_perm(__byte_perm(b[1], b[3], 0x0040), __byte_perm(b[5], b[7], 0x0040), 0x5410);
  return (ev & 0x0F0F0F0Fu) | ((od << 4) & 0xF0F0F0F0u);
}

// ---------------------------------------------------------------------------
// unpacking: codes -> biased unsigned (c + 128 for INT8, c + 8 for INT4) and
// validity (the reference rejects -128 / -8, zs/quantizer.py:233-235)

__device__ __forceinline__ bool has_byte_0x80(uint32_t w) {
  uint32_t v = w ^ 0x80808080u;  // zero byte <=> code == -128
  return ((v - 0x01010101u) & ~v & 0x80808080u) != 0;
}
__device__ __forceinline__ bool has_nibble_8(uint32_t w) {
  uint32_t v = w ^ 0x88888888u;  // zero nibble <=> code == -8
  return ((v - 0x11111111u) & ~v & 0x88888888u) != 0;
}

// 4 INT8 codes in w -> biased bytes u[i] = code_i + 128
__device__ __forceinline__ void unpack4_int8(uint32_t w, uint32_t (&u)[4]) {
  uint32_t f = w ^ 0x80808080u;
  u[0] = __byte_perm(f, 0, 0x4440);
  u[1] = __byte_perm(f, 0, 0x4441);
  u[2] = __byte_perm(f, 0, 0x4442);
  u[3] = __byte_perm(f, 0, 0x4443);
}
// 8 INT4 codes in w (low nibble first) -> biased nibbles code_i + 8
__device__ __forceinline__ void unpack8_int4(uint32_t w, uint32_t (&u)[8]) {
  uint32_t f = w ^ 0x88888888u;
#pragma unroll
  for (int i = 0; i < 8; ++i) u[i] = (f >> (4 * i)) & 0xFu;
}

// ---------------------------------------------------------------------------
// element types

template <int BITS> struct Codes {
  static constexpr int kQmax = (1 << (BITS - 1)) - 1;
  static constexpr int kBytesPer8 = BITS;  // 8 elements -> 8 or 4 bytes
};

// output conversion from an exact double
template <typename O> __device__ __forceinline__ O from_f64(double v);
template <> __device__ __forceinline__ float from_f64<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double from_f64<double>(double v) { return v; }
template <> __device__ __forceinline__ __half from_f64<__half>(double v) { return __double2half(v); }
template <> __device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double v) {
  return __double2bfloat16(v);
}

// absmax storage: fp32 (exact for fp16/bf16/fp32 inputs) or f64
template <typename A> __device__ __forceinline__ double absmax_f64(const A* p, int64_t i);
template <> __device__ __forceinline__ double absmax_f64<float>(const float* p, int64_t i) {
  return (double)__ldg(p + i);
}
template <> __device__ __forceinline__ double absmax_f64<double>(const double* p, int64_t i) {
  return __ldg(p + i);
}

template <int BITS>
__device__ __forceinline__ double scale_of(double m) {
  return div_q<Codes<BITS>::kQmax>(m);
}

// ---------------------------------------------------------------------------
// Blackwell packed fp32x2 arithmetic (FFMA2 / FADD2 / FMUL2), round-to-nearest

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(*reinterpret_cast<unsigned long long*>(&d))
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return d;
}

// max(|a|,|b|) per 16-bit lane, NaN-propagating (HMNMX2.NAN.XORSIGN |a|,|b|);
// the sign bits of the result are garbage and must be masked by the caller.
__device__ __forceinline__ uint32_t absmax_bf16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.NaN.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t absmax_f16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.NaN.xorsign.abs.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// unsigned 32-bit division by an invariant divisor (n < 2^31):
// q = (umulhi(n, mul) + n) >> shift
struct FastDiv {
  uint32_t d, mul, shift;
  __host__ static FastDiv make(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint32_t s = 0;
    while ((1ull << s) < d) ++s;
    f.shift = s;
    f.mul = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
    return f;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, mul) + n) >> shift; }
};

// global timer for bounded spins
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace zpp
