// general_decide.cuh -- the fp64 per-site decision of the multi-level PCA law (PAPER.md:462-477
// with R1), used by sweep_general.cu: w_s = A[n_s] D[g][s] I[x][s],
// Z = sum_s w_s, new label = min{k < L-1 : u Z < sum_{s<=k} w_s}, else L-1 (R14); the
// log-domain max-subtracted form when the factorised weights under/overflow.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "kernels.cuh"

namespace pcab200 {

// a queued fp64 site: neighbour labels (NB <= 8 bytes), x_i, g_i, the Philox word
struct SiteJob {
    uint32_t nb_lo, nb_hi;
    uint32_t xg;  // x_i | g_i << 8
    uint32_t r;
};

// fp64 decision with L known at compile time (L <= 16): the neighbour histogram is built once
// as 16 nibbles, the L weights stay in registers, and the CDF scan is branch-free.
template <int NB, int L>
__device__ __forceinline__ int decide_fp64_fixed(const GeneralSweepParams& p, const double* sA,
                                                 const double* sD, const double* sI,
                                                 const SiteJob& j) {
    uint64_t hist = 0;
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const uint32_t v = ((q < 4 ? j.nb_lo : j.nb_hi) >> (8 * (q & 3))) & 0xFFu;
        hist += (v < (uint32_t)L) ? (1ull << (4 * v)) : 0ull;  // sentinel 0xFF never counts
    }
    const int xi = (int)(j.xg & 0xFFu), gi = (int)((j.xg >> 8) & 0xFFu);
    const double Cw = p.Cw;
    const double* Drow = sD + gi * L;
    const double* Irow = sI + xi * L;
    const bool l0 = p.inertia_p == 0;
    double w[L];
    double Z = 0.0;
#pragma unroll
    for (int s = 0; s < L; ++s) {
        const int n = (int)((hist >> (4 * s)) & 0xFull);
        w[s] = sA[n] * Drow[s] * (l0 ? (s == xi ? 1.0 : Cw) : Irow[s]);
        Z += w[s];
    }
    if (!(Z >= 1e-290 && Z <= 1e290)) return -1;  // caller takes the log-domain path
    const double target = (double)j.r * (1.0 / 4294967296.0) * Z;
    double F = 0.0;
    int res = L - 1;
#pragma unroll
    for (int s = 0; s < L - 1; ++s) {
        F += w[s];
        res = (res == L - 1 && target < F) ? s : res;
    }
    return res;
}

// L <= 8 known at compile time, W0[g][x][s] = D[g][s] I[x][s] staged in shared memory:
// w_s = A[n_s] W0[g][x][s].  The site is byte sb of the staged quad words (w0 = UL UC UR ML,
// w1 = MR DL DC DR; 4 neighbours: UC ML MR DC).  The neighbour histogram (one nibble per
// label, L <= 8 fits 32 bits) uses the PTX shift's clamp: the sentinel 0xFF shifts the 1 out.
__device__ __forceinline__ uint32_t shl_clamp(uint32_t a, uint32_t n) {
    uint32_t r;
    asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(n));
    return r;
}

template <int NB, int L>
__device__ __forceinline__ int decide_fp64_w0(const double* sA, const double* sW0, uint4 w0, uint4 w1,
                                              uint32_t xw, uint32_t gw, uint32_t r, int sb) {
    static_assert(L <= 8, "nibble histogram in 32 bits");
    const uint32_t sel = 0x4440u + (uint32_t)sb;
    auto one = [&](uint32_t w) { return shl_clamp(1u, __byte_perm(w, 0u, sel) << 2); };
    uint32_t h;
    if (NB == 8)
        h = one(w0.x) + one(w0.y) + one(w0.z) + one(w0.w) + one(w1.x) + one(w1.y) + one(w1.z) + one(w1.w);
    else
        h = one(w0.y) + one(w0.w) + one(w1.x) + one(w1.z);
    const int xi = (int)__byte_perm(xw, 0u, sel), gi = (int)__byte_perm(gw, 0u, sel);
    const double* Wrow = sW0 + (gi * L + xi) * L;
    double w[L];
    double Z = 0.0;
#pragma unroll
    for (int s = 0; s < L; ++s) {
        w[s] = sA[(h >> (4 * s)) & 0xFu] * Wrow[s];
        Z += w[s];
    }
    if (!(Z >= 1e-290 && Z <= 1e290)) return -1;  // caller takes the log-domain path
    const double target = (double)r * (1.0 / 4294967296.0) * Z;
    // F_k is non-decreasing, so min{k < L-1 : target < F_k} (else L-1) = #{k < L-1 : F_k <= target}
    double F = 0.0;
    int res = 0;
#pragma unroll
    for (int s = 0; s < L - 1; ++s) {
        F += w[s];
        res += (F <= target) ? 1 : 0;
    }
    return res;
}

template <int NB>
__device__ int decide_fp64(const GeneralSweepParams& p, const double* sA, const SiteJob& j) {
    const int L = p.c.geo.levels;
    int nb[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) nb[q] = (int)(((q < 4 ? j.nb_lo : j.nb_hi) >> (8 * (q & 3))) & 0xFFu);
    const int xi = (int)(j.xg & 0xFFu), gi = (int)((j.xg >> 8) & 0xFFu);
    const double Cw = p.Cw;
    const double* Drow = p.dtab + (size_t)gi * L;
    const double* Irow = p.itab + (size_t)xi * L;
    const bool l0 = p.inertia_p == 0;
    double Z = 0.0;
    for (int s = 0; s < L; ++s) {
        int n = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) n += (nb[q] == s);
        Z += sA[n] * __ldg(Drow + s) * (l0 ? (s == xi ? 1.0 : Cw) : __ldg(Irow + s));
    }
    const double u = (double)j.r * (1.0 / 4294967296.0);
    if (Z >= 1e-290 && Z <= 1e290) {
        const double target = u * Z;
        double F = 0.0;
        for (int s = 0; s < L - 1; ++s) {
            int n = 0;
#pragma unroll
            for (int q = 0; q < NB; ++q) n += (nb[q] == s);
            F += sA[n] * __ldg(Drow + s) * (l0 ? (s == xi ? 1.0 : Cw) : __ldg(Irow + s));
            if (target < F) return s;
        }
        return L - 1;
    }
    // Rare slow path (extreme beta, q or sigma: the factorised weights under- or overflow):
    // E_s = a n_s - b d_s^2 - c pen(x_i, s), softmax with the max subtracted.
    const double lg = (double)gi / (double)(L - 1);
    const double lx = (double)xi / (double)(L - 1);
    auto pen = [&](int s) {
        if (s == xi) return 0.0;
        if (p.inertia_p == 0) return 1.0;
        const double e = lx - (double)s / (double)(L - 1);
        return p.inertia_p == 1 ? fabs(e) : e * e;
    };
    double Emax = -INFINITY;
    for (int s = 0; s < L; ++s) {
        int n = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) n += (nb[q] == s);
        const double d = lg - (double)s / (double)(L - 1);
        Emax = fmax(Emax, p.coef_a * n - p.coef_b * d * d - p.coef_c * pen(s));
    }
    double Zs = 0.0;
    for (int s = 0; s < L; ++s) {
        int n = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) n += (nb[q] == s);
        const double d = lg - (double)s / (double)(L - 1);
        Zs += exp(p.coef_a * n - p.coef_b * d * d - p.coef_c * pen(s) - Emax);
    }
    const double target = u * Zs;
    double F = 0.0;
    for (int s = 0; s < L - 1; ++s) {
        int n = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) n += (nb[q] == s);
        const double d = lg - (double)s / (double)(L - 1);
        F += exp(p.coef_a * n - p.coef_b * d * d - p.coef_c * pen(s) - Emax);
        if (target < F) return s;
    }
    return L - 1;
}

}  // namespace pcab200
