// quant.cuh -- per-tile precision casts on the device ("on-the-fly
// data type up/down-casting", P:335 MxP; G10/G11).
//
// Storage model: every tile lives in an fp64 container holding the values of
// its storage precision p (deq(q_p(X))) plus its amax.  q_p:
//   FP64  identity;  FP32  RNE to binary32;
//   FP16  codes = RNE_binary16(x*s), s = 2^clamp(14 - floor(log2 amax), -127, 127)
//   FP8   codes = RNE_E4M3_satfinite(x*s), s = 2^clamp(7 - floor(log2 amax), -127, 127)
//   (amax = 0 -> s = 1); value = code / s, exact in fp64.
// cast_c(T) = deq(q_c(T)) for a stored tile T: the identity when T's precision
// is no finer than c (exact up-cast), a re-quantization with T's own amax
// otherwise.
#pragma once
#include <math.h>
#include <stdint.h>

namespace mxp {

enum { P_FP64 = 0, P_FP32 = 1, P_FP16 = 2, P_FP8 = 3 };

// RNE of |v| to a binary format with `mb` explicit mantissa bits and minimum
// normal exponent `emin` (gradual underflow), then overflow handling.
__device__ __forceinline__ double rne_format(double v, int mb, int emin, double maxfin, bool saturate) {
    if (v == 0.0 || v != v) return v;
    double a = fabs(v);
    int e = ilogb(a);
    if (e < emin) e = emin;
    double quantum = scalbn(1.0, e - mb);
    double r = rint(a / quantum) * quantum;  // a/quantum exact (power of two); rint = RNE
    if (r > maxfin) r = saturate ? maxfin : INFINITY;
    return copysign(r, v);
}

// Fast exact paths: hardware cvt.rn for binary32/binary16 (IEEE RNE with
// gradual underflow, overflow to inf); E4M3 by integer mantissa rounding on
// the fp64 bit pattern (normal range) and a magic-number add (subnormal
// range, quantum 2^-9), then satfinite.  Equal to rne_format() for every input.
__device__ __forceinline__ double round_fp32(double v) { return (double)__double2float_rn(v); }
__device__ __forceinline__ double round_fp16(double v) {
    unsigned short h;
    asm("cvt.rn.f16.f64 %0, %1;" : "=h"(h) : "d"(v));
    float f;
    asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
    return (double)f;
}
__device__ __forceinline__ double round_e4m3(double v) {
    double a = fabs(v);
    if (!(a == a)) return v;
    double r;
    if (a > 448.0) {
        r = 448.0;  // satfinite: everything above the largest finite rounds/saturates to it
    } else if (a < 0.015625) {  // below 2^-6: fixed quantum 2^-9 (RNE via the 1.5*2^43 shifter)
        const double M = 13194139533312.0;  // 1.5 * 2^43
        r = (a + M) - M;
    } else {  // keep 3 explicit mantissa bits: RNE on bit 49 of the fp64 pattern
        unsigned long long b = (unsigned long long)__double_as_longlong(a);
        b += 0x0000FFFFFFFFFFFFull + ((b >> 49) & 1ull);
        b &= ~0x0001FFFFFFFFFFFFull;
        r = __longlong_as_double((long long)b);
        if (r > 448.0) r = 448.0;
    }
    return copysign(r, v);
}

// power-of-two scale of a tile with max-abs `amax` for precision p (G11)
__device__ __forceinline__ double tile_scale(int p, double amax) {
    if (p != P_FP16 && p != P_FP8) return 1.0;
    if (!(amax > 0.0)) return 1.0;
    int k = (p == P_FP16 ? 14 : 7) - ilogb(amax);
    k = k > 127 ? 127 : (k < -127 ? -127 : k);
    return scalbn(1.0, k);
}

// q then deq of one value with the tile scale s (s = 1 for FP64/FP32);
// s is a power of two, so dividing by it is the exact multiply by 1/s.
__device__ __forceinline__ double quantize_value(int p, double x, double s, double inv_s) {
    switch (p) {
    case P_FP32: return round_fp32(x);
    case P_FP16: return round_fp16(x * s) * inv_s;
    case P_FP8: return round_e4m3(x * s) * inv_s;
    default: return x;
    }
}
__device__ __forceinline__ double quantize_value(int p, double x, double s) {
    return quantize_value(p, x, s, 1.0 / s);
}

// A cast applied while staging an operand tile: mode = target precision when
// the stored precision is finer than the compute precision, else FP64 (none).
struct Cast {
    int mode;
    double s, inv_s;
};
__device__ __forceinline__ Cast make_cast(int stored, int compute, double amax) {
    Cast c;
    c.mode = (stored < compute) ? compute : P_FP64;  // codes: lower = finer
    c.s = tile_scale(c.mode, amax);
    c.inv_s = 1.0 / c.s;
    return c;
}
__device__ __forceinline__ double apply_cast(const Cast& c, double x) {
    return quantize_value(c.mode, x, c.s, c.inv_s);
}

// value of element e of a tile stored as codes at precision p (FP32 float, FP16
// binary16, FP8 E4M3) with scale s: code / s (exact)
__device__ __forceinline__ double decode_code(int p, const uint8_t* codes, int64_t e, double inv_s) {
    if (p == P_FP32) return (double)__ldcg(reinterpret_cast<const float*>(codes) + e);
    if (p == P_FP16) {
        const unsigned short h = __ldcg(reinterpret_cast<const unsigned short*>(codes) + e);
        float f;
        asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"(h));
        return (double)f * inv_s;
    }
    const unsigned short b = (unsigned short)__ldcg(codes + e);
    unsigned int h2;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(b));
    float f;
    asm("cvt.f32.f16 %0, %1;" : "=f"(f) : "h"((unsigned short)(h2 & 0xFFFFu)));
    return (double)f * inv_s;
}

// amax of non-negative doubles via their bit patterns (monotone for x >= 0)
__device__ __forceinline__ void atomic_max_abs(unsigned long long* slot, double v) {
    atomicMax(slot, (unsigned long long)__double_as_longlong(fabs(v)));
}
__device__ __forceinline__ double amax_of(const unsigned long long* slot) {
    return __longlong_as_double((long long)__ldcg(slot));
}

}  // namespace mxp
