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

namespace pcab200 {

// The same Philox4x32-10 with the counter's row word y split off.  For a counter
// (x, y, z, w) whose x, z, w are fixed while y (the lattice row) varies -- a thread walking a
// run of rows -- the row-independent part of rounds 0..2 is computed once (philox_pre) and each
// row costs 6 instead of 12 instructions for those rounds (philox_row).  Derivation (M0, M1 the
// multipliers, k_j the round keys, hi/lo the halves of the products):
//   round 0: (hi1(z)^y^k0, lo1(z), hi0(x)^w^k1, lo0(x))            = (Y1^y, Z1, W1, X1)
//   round 1: (hi1(W1)^Z1^k2, lo1(W1), hi0(Y1^y)^X1^k3, lo0(Y1^y))  = (Y2, Z2, hi0'^W2, lo0')
//   round 2: (hi1(z2)^Z2^k4, lo1(z2), hi0(Y2)^lo0'^k5, lo0(Y2))    = (hi1(z2)^C1, lo1(z2), lo0'^C2, C3)
// with z2 = hi0' ^ W2; rounds 3..9 as philox4x32_10.  Bit-identical by construction (the
// tests compare every chain with the oracle's Philox).
struct PhiloxPre {
    uint32_t y1, w2, c1, c2, c3;
};

__device__ __forceinline__ PhiloxPre philox_pre(uint32_t x, uint32_t z, uint32_t w, const PhiloxKeys& k) {
    PhiloxPre p;
    const uint32_t lo0 = 0xD2511F53u * x, hi0 = __umulhi(0xD2511F53u, x);
    const uint32_t lo1 = 0xCD9E8D57u * z, hi1 = __umulhi(0xCD9E8D57u, z);
    p.y1 = hi1 ^ k.rk[0];
    const uint32_t Z1 = lo1, W1 = hi0 ^ w ^ k.rk[1], X1 = lo0;
    const uint32_t lo1b = 0xCD9E8D57u * W1, hi1b = __umulhi(0xCD9E8D57u, W1);
    const uint32_t Y2 = hi1b ^ Z1 ^ k.rk[2], Z2 = lo1b;
    p.w2 = X1 ^ k.rk[3];
    p.c1 = Z2 ^ k.rk[4];
    p.c2 = __umulhi(0xD2511F53u, Y2) ^ k.rk[5];
    p.c3 = 0xD2511F53u * Y2;
    return p;
}

// lo/hi halves of m * x: WIDE = one 64-bit product (ptxas emits IMAD.WIDE.U32), else __umulhi and
// a 32-bit product (which ptxas may emit as IMAD.HI + IMAD, or fuse).  Which is faster depends on
// the kernel around it, so the callers choose (measured: the table kernel and the packed and byte
// kernels on a torus gain 0.7-1.5% with WIDE; the packed kernel on a free boundary loses 1%).
template <bool WIDE>
__device__ __forceinline__ void philox_mulhilo(uint32_t m, uint32_t x, uint32_t& lo, uint32_t& hi) {
    if (WIDE) {
        const unsigned long long p = (unsigned long long)m * x;
        lo = (uint32_t)p;
        hi = (uint32_t)(p >> 32);
    } else {
        lo = m * x;
        hi = __umulhi(m, x);
    }
}

template <bool WIDE = false>
__device__ __forceinline__ uint4 philox_row(const PhiloxPre& p, uint32_t y, const PhiloxKeys& k) {
    const uint32_t x1 = p.y1 ^ y;
    uint32_t lo0, hi0, lo1, hi1;
    philox_mulhilo<WIDE>(0xD2511F53u, x1, lo0, hi0);
    const uint32_t z2 = hi0 ^ p.w2;
    philox_mulhilo<WIDE>(0xCD9E8D57u, z2, lo1, hi1);
    uint4 c = make_uint4(hi1 ^ p.c1, lo1, lo0 ^ p.c2, p.c3);
#pragma unroll
    for (int i = 3; i < 10; ++i) {
        uint32_t l0, h0, l1, h1;
        philox_mulhilo<WIDE>(0xD2511F53u, c.x, l0, h0);
        philox_mulhilo<WIDE>(0xCD9E8D57u, c.z, l1, h1);
        c = make_uint4(h1 ^ c.y ^ k.rk[2 * i], l1, h0 ^ c.w ^ k.rk[2 * i + 1], l0);
    }
    return c;
}

}  // namespace pcab200
