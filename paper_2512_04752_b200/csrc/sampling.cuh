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

// exp_spec(x) for x <= 0 (0 for x < -32 or NaN). Sequence of single RN fp32 operations.
__device__ __forceinline__ float exp_spec(float x) {
    if (!(x >= -32.0f)) return 0.0f;
    const float LOG2E = 1.44269502735137939453125f;
    const float C1 = 0.693359375f;
    const float C2 = -2.12194440e-4f;
    float n = rintf(__fmul_rn(x, LOG2E));
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
    y = __fadd_rn(y, 1.0f);
    // y * 2^n, n in [-47, 0]: the power of two is a normal float, the product is exact.
    int ni = __float2int_rn(n);
    return __fmul_rn(y, __int_as_float((127 + ni) << 23));
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
