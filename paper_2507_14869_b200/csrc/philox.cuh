// Philox4x32-10 counter-based generator (Salmon et al., SC'11), device side.
// RNG contract: DESIGN.md section 4.  Round keys are precomputed on the host
// (rk[2i], rk[2i+1] = key + i*(W0, W1)) and passed as uniform kernel parameters,
// so the 10 rounds are 2 IMAD.WIDE + 2 LOP3 each with no key schedule in the loop.
#pragma once
#include <cstdint>

namespace pcab200 {

struct PhiloxKeys {
    uint32_t rk[20];
};

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, const PhiloxKeys& k) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t lo0 = 0xD2511F53u * c.x;
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.rk[2 * i], lo1, hi0 ^ c.w ^ k.rk[2 * i + 1], lo0);
    }
    return c;
}

}  // namespace pcab200
