// Device arithmetic of the bit-exact sampling rule (DESIGN.md §2 "exp_spec" and "Bit-exact
// sampling"; reading Z7). Every float op is an explicit round-to-nearest intrinsic so the
// compiler cannot contract or reorder it; integer weights make every reduction associative.
#pragma once

#include <stdint.h>

namespace rs {

typedef unsigned __int128 u128;

// Philox4x32-10 (Salmon et al., SC'11): 10 rounds of the (0xD2511F53, 0xCD9E8D57) multiply
// rounds with Weyl key increments (0x9E3779B9, 0xBB67AE85).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

// Uniform word for (trial, node) of sample gid at (seed, step): counter (trial, node,
// lo32(step), lo32(gid)), key (lo32(seed), hi32(seed)), output word 0.
__device__ __forceinline__ uint32_t uniform_word(uint64_t seed, uint64_t step, int64_t gid,
                                                 uint32_t trial, uint32_t node) {
    uint4 c = make_uint4(trial, node, (uint32_t)step, (uint32_t)(uint64_t)gid);
    uint2 k = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    return philox4x32_10(c, k).x;
}

// exp_spec(x) for x <= 0 (0 for x < -32 or NaN). Sequence of single RN fp32 operations
// (DESIGN.md "exp_spec"). Branch-free, so the compiler can interleave the independent chains of
// a vector's elements: the polynomial is evaluated for every x and the x < -32 / NaN lanes are
// selected to 0 at the end (their intermediate values are discarded, no trap). n = rint(v) is
// taken as fl(v + 1.5*2^23) - 1.5*2^23: for |v| < 2^22 the sum lies in [2^23, 2^24), where the
// floats are the integers, so its round-to-nearest-even IS rint(v) (1.5*2^23 is even) and the
// subtraction is exact; the integer n is then the sum's low mantissa bits (no FRND / F2I).
// Returns y (the polynomial part) and n with exp_spec(x) = y * 2^n for x in [-32, 0].
__device__ __forceinline__ float exp_spec_parts(float x, int& ni) {
    const float LOG2E = 1.44269502735137939453125f;
    const float C1 = 0.693359375f;
    const float C2 = -2.12194440e-4f;
    const float SHIFT = 12582912.0f;   // 1.5 * 2^23
    const float t = __fadd_rn(__fmul_rn(x, LOG2E), SHIFT);
    const float n = __fsub_rn(t, SHIFT);
    ni = __float_as_int(t) - 0x4B400000;
    float r = __fsub_rn(x, __fmul_rn(n, C1));
    r = __fsub_rn(r, __fmul_rn(n, C2));
    float p = 1.9875691500e-4f;
    p = __fadd_rn(__fmul_rn(p, r), 1.3981999507e-3f);
    p = __fadd_rn(__fmul_rn(p, r), 8.3334519073e-3f);
    p = __fadd_rn(__fmul_rn(p, r), 4.1665795894e-2f);
    p = __fadd_rn(__fmul_rn(p, r), 1.6666665459e-1f);
    p = __fadd_rn(__fmul_rn(p, r), 5.0000001201e-1f);
    float y = __fmul_rn(p, __fmul_rn(r, r));
    y = __fadd_rn(y, r);
    return __fadd_rn(y, 1.0f);
}

__device__ __forceinline__ float exp_spec(float x) {
    int ni;
    const float y = exp_spec_parts(x, ni);
    // y * 2^n, n in [-47, 0]: the power of two is a normal float, the product is exact.
    const float e = __fmul_rn(y, __int_as_float((127 + ni) << 23));
    return (x >= -32.0f) ? e : 0.0f;
}

// trunc(exp_spec(x) * 2^32) ENCODED as u32 (2^32 -> 0xFFFFFFFF, the f2w code of the MSS kernel).
// exp_spec(x) * 2^32 = (y * 2^n) * 2^32 = y * 2^(n+32) exactly (both scalings are exact: y * 2^n
// is a normal float for n >= -47), so one multiply; cvt.rzi.u32 saturates 2^32 to 0xFFFFFFFF.
__device__ __forceinline__ uint32_t exp_spec_w32(float x) {
    int ni;
    const float y = exp_spec_parts(x, ni);
    const uint32_t w = __float2uint_rz(__fmul_rn(y, __int_as_float((127 + 32 + ni) << 23)));
    return (x >= -32.0f) ? w : 0u;
}

// Target weight: trunc(exp_spec((l - m) * inv_tau) * 2^32).
__device__ __forceinline__ uint64_t target_weight(float l, float m, float inv_tau) {
    float x = __fmul_rn(__fsub_rn(l, m), inv_tau);
    float e = exp_spec(x);
    return __float2ull_rz(__fmul_rn(e, 4294967296.0f));
}

// Draft weight: trunc(q * 2^32) (q in [0, 1]).
__device__ __forceinline__ uint64_t draft_weight(float q) {
    return (q > 0.0f) ? __float2ull_rz(__fmul_rn(q, 4294967296.0f)) : 0ull;
}

__device__ __forceinline__ int bitlen128(u128 x) {
    uint64_t hi = (uint64_t)(x >> 64), lo = (uint64_t)x;
    if (hi) return 128 - __clzll((long long)hi);
    if (lo) return 64 - __clzll((long long)lo);
    return 0;
}

__device__ __forceinline__ float bf16_bits_to_f32(uint16_t h) {
    return __uint_as_float(((uint32_t)h) << 16);
}

}  // namespace rs
