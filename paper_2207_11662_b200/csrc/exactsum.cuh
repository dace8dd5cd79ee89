// Exact, correctly rounded sums of non-negative doubles -- device helpers (exactsum.cu has the
// method; reading Z6 of DESIGN.md §3: mean = RN(exact sum) / n, math.fsum semantics).
#pragma once
#include <stdint.h>

namespace hm {

constexpr int EXACT_LO = -1088;     // limb i weighs 2^(32 i + EXACT_LO)
constexpr int EXACT_NLIMB = 70;     // covers 2^-1088 .. 2^1152

// Adds v (finite, >= 0; checked by the caller) exactly into block-local 32-bit shared counters, two per limb (its low and high 16 bits), so every
// update is a native 32-bit shared atomic (64-bit shared atomicAdd compiles to a CAS loop, and all
// values of similar magnitude hit the same three limbs).  A counter receives < 2^16 per value:
// exact for fewer than 2^16 values per block.
constexpr int EXACT_MAX_PER_BLOCK = 65535;
__device__ __forceinline__ void exact_add16(unsigned *s16, double v) {
    const uint64_t bits = (uint64_t)__double_as_longlong(v);
    const int ef = (int)((bits >> 52) & 0x7ff);
    uint64_t m = bits & ((1ull << 52) - 1);
    int e;
    if (ef == 0) {
        e = -1074;
    } else {
        m |= (1ull << 52);
        e = ef - 1075;
    }
    if (m == 0) return;
    const int pos = e - EXACT_LO;
    const int li = pos >> 5, off = pos & 31;
    const unsigned __int128 t = (unsigned __int128)m << off;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const uint32_t l = (uint32_t)(t >> (32 * q));
        if (l & 0xffffu) atomicAdd(&s16[2 * (li + q)], l & 0xffffu);
        if (l >> 16) atomicAdd(&s16[2 * (li + q) + 1], l >> 16);
    }
}
// limb i of a block's 16-bit-half counters as a 64-bit value
__device__ __forceinline__ unsigned long long exact_limb16(const unsigned *s16, int i) {
    return (unsigned long long)s16[2 * i] + ((unsigned long long)s16[2 * i + 1] << 16);
}

// One thread: carry-normalise the limbs and round the integer once to binary64 (round half to even).
__device__ __forceinline__ double exact_round(const unsigned long long *acc_in) {
    uint32_t L[EXACT_NLIMB + 2];
    unsigned long long carry = 0;
    for (int i = 0; i < EXACT_NLIMB; ++i) {
        const unsigned long long v = acc_in[i] + carry;   // < 2^64 (acc < 2^63, carry < 2^32)
        L[i] = (uint32_t)(v & 0xffffffffull);
        carry = v >> 32;
    }
    L[EXACT_NLIMB] = (uint32_t)(carry & 0xffffffffull);
    L[EXACT_NLIMB + 1] = (uint32_t)(carry >> 32);
    int t = EXACT_NLIMB + 1;
    while (t >= 0 && L[t] == 0) --t;
    if (t < 0) return 0.0;
    const uint32_t hi = L[t];
    const uint32_t mid = t >= 1 ? L[t - 1] : 0u;
    const uint32_t lo = t >= 2 ? L[t - 2] : 0u;
    bool sticky = false;
    for (int i = t - 3; i >= 0; --i)
        if (L[i]) { sticky = true; break; }
    const unsigned __int128 X = ((unsigned __int128)hi << 64) | ((unsigned __int128)mid << 32) | lo;
    const int p = 64 + (31 - __clz((int)hi));           // index of X's top bit
    const int shift = p - 52;                             // >= 12
    uint64_t q = (uint64_t)(X >> shift);
    const unsigned __int128 rem = X & ((((unsigned __int128)1) << shift) - 1);
    const unsigned __int128 half = ((unsigned __int128)1) << (shift - 1);
    if (rem > half || (rem == half && (sticky || (q & 1ull)))) ++q;
    // value = q * 2^(shift + 32 (t-2) + LO); q <= 2^53 is exact in binary64
    return ldexp((double)q, shift + 32 * (t - 2) + EXACT_LO);
}

}  // namespace hm
