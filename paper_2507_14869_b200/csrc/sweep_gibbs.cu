// sweep_gibbs.cu -- the Gibbs sampler of PAPER.md:148-158 / 417-435 on the GPU: a systematic
// scan in checkerboard colour order.  Sites of one colour are never neighbours (4-neighbour:
// 2 colours (r + c) mod 2; Moore-8: 4 colours 2 (r mod 2) + (c mod 2); on a torus H and W
// must be even), so updating a colour class at once equals updating its sites one after the
// other: one launch per colour, in place, is exactly the sequential scan "colour 0, colour
// 1, ..." of oracle/orc_gibbs_sweep_coloured (the paper's own scan is column-major,
// PAPER.md:435; the order changes the chain, not its stationary law pi_GS, R21).
//
// Per site of colour k: the Gibbs conditional p_i(s) ∝ exp(a n_i(s) - b (lum g_i - lum s)^2)
// (no inertia term), inverse-CDF draw with the site's Philox word of tag
// GIBBS.  levels == 2: integer thresholds for every (n_present, n_1,
// g_i) -- exact; levels > 2: the uniform-neighbourhood threshold table (levels <= 16) or
// fp64 weights, as in sweep_general.cu, specialised at compile time for 3, 5, 9 and 16
// levels (tables in shared memory, unrolled fp64 path).
//
// Thread = 4 consecutive sites of a row (one Philox call), walking a run of rows with a
// rolling window (as sweep_general.cu).  Moore-8 launches cover only the rows of the
// colour's parity.  levels == 2 uses SWAR byte sums for the label-1 and present neighbours
// of the 4 sites and one table lookup per site.  A thread rewrites its whole 4-byte word:
// the bytes of other colours are rewritten with the values it read, which no thread of this
// launch changes, so concurrent readers see the same neighbour labels either way.  MPM counts
// are taken in the launch after which a row is final (colours 1 and 3), with fire-and-forget
// 64-bit reductions.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "tma_ring.cuh"  // from_left / from_right byte funnels

namespace pcab200 {
namespace {

namespace cg = cooperative_groups;

#ifndef PCA_GB_MINB
#define PCA_GB_MINB 6  // blocks per SM the register budget is sized for (8192^2 l=5: 4 -> 1465, 6 -> 1265, 8 -> 1324 us)
#endif
constexpr int GB_THREADS = 128;
constexpr int GB_WARPS = GB_THREADS / 32;
constexpr unsigned FULL = 0xFFFFFFFFu;

// plain (coherent) loads: the buffer is written by this same launch, so not the read-only path
__device__ __forceinline__ uint32_t ld4(const uint8_t* p) {
    return *reinterpret_cast<const uint32_t*>(p);
}

struct GibbsJob {
    uint32_t nb_lo, nb_hi;
    uint32_t g;
    uint32_t r;
};

template <int NB>
__device__ int gibbs_fp64(const GibbsSweepParams& p, const double* sA, const GibbsJob& j) {
    const int L = p.c.geo.levels;
    int nb[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) nb[q] = (int)(((q < 4 ? j.nb_lo : j.nb_hi) >> (8 * (q & 3))) & 0xFFu);
    const int gi = (int)j.g;
    const double* Drow = p.dtab + (size_t)gi * L;
    double Z = 0.0;
    for (int s = 0; s < L; ++s) {
        int n = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) n += (nb[q] == s);
        Z += sA[n] * __ldg(Drow + s);
    }
    const double u = (double)j.r * (1.0 / 4294967296.0);
    if (Z >= 1e-290 && Z <= 1e290) {
        const double target = u * Z;
        double F = 0.0;
        for (int s = 0; s < L - 1; ++s) {
            int n = 0;
#pragma unroll
            for (int q = 0; q < NB; ++q) n += (nb[q] == s);
            F += sA[n] * __ldg(Drow + s);
            if (target < F) return s;
        }
        return L - 1;
    }
    // log domain (extreme beta or sigma): E_s = a n_s - b d_s^2, max subtracted
    const double lg = (double)gi / (double)(L - 1);
    double Emax = -INFINITY;
    for (int s = 0; s < L; ++s) {
        int n = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) n += (nb[q] == s);
        const double d = lg - (double)s / (double)(L - 1);
        Emax = fmax(Emax, p.coef_a * n - p.coef_b * d * d);
    }
    double Zs = 0.0;
    for (int s = 0; s < L; ++s) {
        int n = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) n += (nb[q] == s);
        const double d = lg - (double)s / (double)(L - 1);
        Zs += exp(p.coef_a * n - p.coef_b * d * d - Emax);
    }
    const double target = u * Zs;
    double F = 0.0;
    for (int s = 0; s < L - 1; ++s) {
        int n = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q) n += (nb[q] == s);
        const double d = lg - (double)s / (double)(L - 1);
        F += exp(p.coef_a * n - p.coef_b * d * d - Emax);
        if (target < F) return s;
    }
    return L - 1;
}

// levels known at compile time (3, 5, 9, 16): the neighbour histogram is built once as
// nibbles, the weights A[n_s] D[g][s] stay in registers, the CDF scan is branch-free (the
// products and sums are those of gibbs_fp64, so the decisions are the same).  Returns -1 when
// Z under/overflows (the caller takes the log-domain path).
constexpr int GB_LMAX = 16;   // D table in shared memory up to 16 levels
constexpr int GB_UMAX = 9;    // uniform thresholds in shared memory up to 9 levels
template <int NB, int L>
__device__ __forceinline__ int gibbs_fp64_fixed(const double* sA, const double* sD, const GibbsJob& j) {
    uint64_t hist = 0;
#pragma unroll
    for (int q = 0; q < NB; ++q) {
        const uint32_t v = ((q < 4 ? j.nb_lo : j.nb_hi) >> (8 * (q & 3))) & 0xFFu;
        hist += (v < (uint32_t)L) ? (1ull << (4 * v)) : 0ull;  // sentinel 0xFF never counts
    }
    const double* Drow = sD + (int)j.g * L;
    double w[L];
    double Z = 0.0;
#pragma unroll
    for (int s = 0; s < L; ++s) {
        w[s] = sA[(int)((hist >> (4 * s)) & 0xFull)] * Drow[s];
        Z += w[s];
    }
    if (!(Z >= 1e-290 && Z <= 1e290)) return -1;
    const double target = (double)j.r * (1.0 / 4294967296.0) * Z;
    // F_k is non-decreasing: min{k < L-1 : target < F_k} (else L-1) = #{k < L-1 : F_k <= target}
    double F = 0.0;
    int res = 0;
#pragma unroll
    for (int s = 0; s < L - 1; ++s) {
        F += w[s];
        res += (F <= target) ? 1 : 0;
    }
    return res;
}

struct GibbsSmem {
    double A[9];
    double D[GB_LMAX * GB_LMAX];
    uint32_t T[GIBBS_THR2];
    uint32_t U[GB_UMAX * GB_UMAX * (GB_UMAX - 1)];
    GibbsJob jobs[GB_WARPS][64];
    uint8_t res[GB_WARPS][64];
};

// stage the launch's tables: A, and per level count the binary thresholds, or D and the
// uniform-neighbourhood thresholds
template <int LT>
__device__ __forceinline__ void gibbs_load_tables(const GibbsSweepParams& p, GibbsSmem& sm) {
    if (threadIdx.x < 9) sm.A[threadIdx.x] = p.A[threadIdx.x];
    if (LT == 2)
        for (int i = threadIdx.x; i < GIBBS_THR2; i += GB_THREADS) sm.T[i] = p.thr2[i];
    if (LT > 2 && LT <= GB_LMAX)
        for (int i = threadIdx.x; i < LT * LT; i += GB_THREADS) sm.D[i] = p.dtab[i];
    if (LT > 2 && LT <= GB_UMAX && p.uthr != nullptr)
        for (int i = threadIdx.x; i < LT * LT * (LT - 1); i += GB_THREADS) sm.U[i] = p.uthr[i];
}

// One launch's work for x-block xb, row block rb of chain `chain`: colour k (FUSED: row parity
// k), sweep t.  COH: x is read through L2 (ld.global.cg) because earlier phases of the same
// cooperative launch wrote it.
template <int NB, int LT, bool FUSED, bool COH>  // LT: levels at compile time (2 = binary), 0 = any
__device__ __forceinline__ void gibbs_rows(const GibbsSweepParams& p, GibbsSmem& sm, int k, uint32_t t,
                                           int count_enable, int xb, int rb, int chain, int R) {
    constexpr bool BIN = LT == 2;
    constexpr bool SMEM_U = LT > 2 && LT <= GB_UMAX;
    const double* sA = sm.A;
    const uint32_t* sT = sm.T;
    const Geometry& G = p.c.geo;
    const int L = G.levels;
    const int nquads = (G.W + 3) >> 2;
    const int qd = xb * GB_THREADS + threadIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool active = qd < nquads;
    if (__ballot_sync(FULL, active) == 0) return;
    const uint32_t tagchain = (TAG_GIBBS << 24) | (p.c.chain0 + (uint32_t)chain);
    const unsigned lt = (1u << lane) - 1u;
    GibbsJob* jobs = sm.jobs[warp];
    uint8_t* res = sm.res[warp];
    // rows of this block: Moore-8 visits only rows whose global parity is k >> 1 (FUSED: k is
    // the row parity itself, both colours of the row in one launch)
    const int rstep = NB == 8 ? 2 : 1;
    const int par = FUSED ? k : (k >> 1);
    int rfirst = p.c.rlo;
    if (NB == 8 && ((G.row0 + rfirst) & 1) != par) ++rfirst;
    const int rbeg = rfirst + rstep * R * rb;
    const int rend = min(rbeg + rstep * R, p.c.rhi);
    if (rbeg >= rend) return;
    const int c0 = 4 * qd;
    const int nvalid = active ? min(4, G.W - c0) : 0;
    uint8_t* xcol = p.c.x_out + chain * G.xchain + XOFF + c0;
    const uint8_t* gcol = p.c.g + chain * G.gchain + XOFF + c0;
    auto load_row = [&](int r, uint32_t (&w)[3]) {
        if (!active) return;
        const uint8_t* xr = xcol + (long long)(r + HALO) * G.xpitch;
        if (COH) {
            w[0] = __ldcg(reinterpret_cast<const uint32_t*>(xr - 4));
            w[1] = __ldcg(reinterpret_cast<const uint32_t*>(xr));
            w[2] = __ldcg(reinterpret_cast<const uint32_t*>(xr + 4));
        } else {
            w[0] = ld4(xr - 4);
            w[1] = ld4(xr);
            w[2] = ld4(xr + 4);
        }
    };
    // rolling window; the rows a launch reads around its rows never change in the launch
    // (4-neighbour: only the other colour's bytes are used; Moore-8: the other row parity)
    uint32_t up[3] = {0, 0, 0}, mid[3] = {0, 0, 0}, dn[3] = {0, 0, 0};
    load_row(rbeg - 1, up);
    load_row(rbeg, mid);
    load_row(rbeg + 1, dn);

    for (int r = rbeg; r < rend; r += rstep) {
        const int grow = G.row0 + r;
        uint32_t gword = 0;
        uint4 rnd = make_uint4(0, 0, 0, 0);
        if (active) {
            gword = __ldg(reinterpret_cast<const uint32_t*>(gcol + (long long)(r + GHALO) * G.gpitch));
            rnd = philox4x32_10(make_uint4((uint32_t)qd, (uint32_t)grow, t, tagchain), p.c.keys);
        }
        const uint32_t rr[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
        uint32_t outw = mid[1];  // start from the current labels of the 4 sites
        // decide the sites in `mask` from the neighbour words (byte b = neighbour of site b)
        auto decide4 = [&](uint32_t UL, uint32_t UC, uint32_t UR, uint32_t ML, uint32_t MR,
                           uint32_t DL, uint32_t DC, uint32_t DR, unsigned mask) {
            if (BIN) {
                // SWAR over the 4 sites: label-1 neighbours and present neighbours per byte
                auto one = [](uint32_t w) { return w & ~(w >> 1) & 0x01010101u; };  // 0xFF -> 0
                auto pres = [](uint32_t w) { return (~w >> 7) & 0x01010101u; };     // 0xFF -> 0
                uint32_t n1, np;
                if (NB == 8) {
                    n1 = one(UL) + one(UC) + one(UR) + one(ML) + one(MR) + one(DL) + one(DC) + one(DR);
                    np = G.periodic ? 0x08080808u
                                    : pres(UL) + pres(UC) + pres(UR) + pres(ML) + pres(MR) + pres(DL) + pres(DC) + pres(DR);
                } else {
                    n1 = one(UC) + one(ML) + one(MR) + one(DC);
                    np = G.periodic ? 0x04040404u : pres(UC) + pres(ML) + pres(MR) + pres(DC);
                }
                const uint32_t idx4 = ((np * 9u + n1) << 1) | gword;  // (np*9 + n1)*2 + g per byte
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    if ((mask >> b) & 1u) {
                        const uint32_t w = rr[b] > sT[(idx4 >> (8 * b)) & 0xFFu] ? 1u : 0u;
                        outw = (outw & ~(0xFFu << (8 * b))) | (w << (8 * b));
                    }
                }
            } else {
                int qpos[4] = {-1, -1, -1, -1};
                int qbase = 0;
                uint32_t D;
                if (NB == 8)
                    D = (UL ^ UC) | (UC ^ UR) | (UR ^ ML) | (ML ^ MR) | (MR ^ DL) | (DL ^ DC) | (DC ^ DR);
                else
                    D = (UC ^ ML) | (ML ^ MR) | (MR ^ DC);
                const uint32_t differ = (((D & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | D) & 0x80808080u;
                const uint32_t S0 = NB == 8 ? UL : UC;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const bool my = (mask >> b) & 1u;
                    const int gi = (int)((gword >> (8 * b)) & 0xFFu);
                    const int s0 = (int)((S0 >> (8 * b)) & 0xFFu);
                    const bool uniform = p.uthr != nullptr && ((differ >> (8 * b + 7)) & 1u) == 0u && s0 < L;
                    if (SMEM_U) {
                        // branch-free: every lane reads a row (row 0 unless its site is a uniform
                        // one of this colour) and counts the thresholds T_k >= r with borrow bits
                        const bool uni = my && uniform;
                        const uint32_t* T = sm.U + (uni ? (s0 * LT + gi) * (LT - 1) : 0);
                        uint32_t ge = 0;
#pragma unroll
                        for (int kk = 0; kk < (SMEM_U ? LT - 1 : 1); ++kk)
                            asm("{\n\t.reg .u32 d;\n\tsub.cc.u32 d, %1, %2;\n\taddc.u32 %0, %0, 0;\n\t}"
                                : "+r"(ge) : "r"(T[kk]), "r"(rr[b]));
                        if (uni) outw = (outw & ~(0xFFu << (8 * b))) | (((uint32_t)(LT - 1) - ge) << (8 * b));
                    } else if (my && uniform) {
                        const uint32_t* T = p.uthr + (size_t)(s0 * L + gi) * (L - 1);
                        int w = 0;
                        for (int kk = 0; kk < L - 1; ++kk) w += (rr[b] > __ldg(T + kk)) ? 1 : 0;
                        outw = (outw & ~(0xFFu << (8 * b))) | ((uint32_t)w << (8 * b));
                    }
                    const bool need = my && !uniform;
                    const unsigned m = __ballot_sync(FULL, need);
                    if (need) {
                        qpos[b] = qbase + __popc(m & lt);
                        const uint32_t sel = (uint32_t)b | ((uint32_t)(b + 4) << 4);
                        GibbsJob jb;
                        if (NB == 8) {
                            jb.nb_lo = __byte_perm(__byte_perm(UL, UC, sel), __byte_perm(UR, ML, sel), 0x5410);
                            jb.nb_hi = __byte_perm(__byte_perm(MR, DL, sel), __byte_perm(DC, DR, sel), 0x5410);
                        } else {
                            jb.nb_lo = __byte_perm(__byte_perm(UC, ML, sel), __byte_perm(MR, DC, sel), 0x5410);
                            jb.nb_hi = 0u;
                        }
                        jb.g = (uint32_t)gi;
                        jb.r = rr[b];
                        jobs[qpos[b]] = jb;
                    }
                    qbase += __popc(m);
                }
                if (qbase > 0) {
                    __syncwarp();
                    for (int i = lane; i < qbase; i += 32) {
                        int w = -1;
                        if (LT > 2) w = gibbs_fp64_fixed<NB, (LT > 2 ? LT : 3)>(sA, sm.D, jobs[i]);
                        if (w < 0) w = gibbs_fp64<NB>(p, sA, jobs[i]);
                        res[i] = (uint8_t)w;
                    }
                    __syncwarp();
#pragma unroll
                    for (int b = 0; b < 4; ++b)
                        if (qpos[b] >= 0) outw = (outw & ~(0xFFu << (8 * b))) | ((uint32_t)res[qpos[b]] << (8 * b));
                    __syncwarp();
                }
            }
        };
        const unsigned valid = nvalid >= 4 ? 0xFu : ((1u << nvalid) - 1u);
        const uint32_t UL = from_left(up[0], up[1]), UC = up[1], UR = from_right(up[1], up[2]);
        const uint32_t ML = from_left(mid[0], mid[1]), MR = from_right(mid[1], mid[2]);
        const uint32_t DL = from_left(dn[0], dn[1]), DC = dn[1], DR = from_right(dn[1], dn[2]);
        if (!FUSED) {
            // sites of colour k in this quad (c0 is a multiple of 4)
            const unsigned mine = (NB == 4 ? (((grow + k) & 1) ? 0xAu : 0x5u) : ((k & 1) ? 0xAu : 0x5u)) & valid;
            decide4(UL, UC, UR, ML, MR, DL, DC, DR, mine);
        } else {
            // Moore-8, one row parity per launch: colour 2p (even columns) from the old labels,
            // then colour 2p+1 (odd columns) from the new even-column labels of the same row
            // (the rows above and below have the other parity and do not change)
            decide4(UL, UC, UR, ML, MR, DL, DC, DR, 0x5u & valid);
            // new label of column c0+4 (colour 2p): from the next lane, or recomputed here when
            // the next quad belongs to another warp (or wraps around the torus)
            const uint32_t nb0 = __shfl_down_sync(FULL, outw & 0xFFu, 1);
            uint32_t v4 = (mid[2] & 0xFFu);  // sentinel 0xFF past a free boundary
            const bool has_next = c0 + 4 < G.W;
            const bool wraps = G.periodic && c0 + 4 == G.W;
            if (active && (has_next || wraps)) {
                if (lane < 31 && has_next && qd + 1 < nquads) {
                    v4 = nb0;
                } else {
                    // site c0+4 (or column 0 on a torus): neighbours from the window, Philox
                    // word 0 of its quad, its g
                    const int qn = wraps ? 0 : qd + 1;
                    const uint4 rn = philox4x32_10(make_uint4((uint32_t)qn, (uint32_t)grow, t, tagchain), p.c.keys);
                    const int gn = (int)__ldg(gcol + (long long)(r + GHALO) * G.gpitch + (wraps ? -c0 : 4));
                    // neighbour bytes of site c0+4: columns c0+3, c0+4, c0+5 of the rows above /
                    // below and c0+3, c0+5 of this row (old: colour 2p+1 is decided later)
                    auto b3 = [&](const uint32_t (&w)[3]) { return (w[1] >> 24) & 0xFFu; };
                    auto b4 = [&](const uint32_t (&w)[3]) { return w[2] & 0xFFu; };
                    auto b5 = [&](const uint32_t (&w)[3]) { return (w[2] >> 8) & 0xFFu; };
                    const uint32_t nbs[8] = {b3(up), b4(up), b5(up), b3(mid), b5(mid), b3(dn), b4(dn), b5(dn)};
                    if (BIN) {
                        int n1 = 0, np = 0;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            n1 += nbs[q] == 1u;
                            np += nbs[q] != 0xFFu;
                        }
                        if (G.periodic) np = 8;
                        v4 = rn.x > sT[(np * 9 + n1) * 2 + gn] ? 1u : 0u;
                    } else {
                        bool uni = p.uthr != nullptr && nbs[0] < (uint32_t)L;
#pragma unroll
                        for (int q = 1; q < 8; ++q) uni = uni && nbs[q] == nbs[0];
                        if (uni) {
                            const uint32_t* T = p.uthr + (size_t)((int)nbs[0] * L + gn) * (L - 1);
                            int w = 0;
                            for (int kk = 0; kk < L - 1; ++kk) w += (rn.x > __ldg(T + kk)) ? 1 : 0;
                            v4 = (uint32_t)w;
                        } else {
                            GibbsJob jb;
                            jb.nb_lo = nbs[0] | (nbs[1] << 8) | (nbs[2] << 16) | (nbs[3] << 24);
                            jb.nb_hi = nbs[4] | (nbs[5] << 8) | (nbs[6] << 16) | (nbs[7] << 24);
                            jb.g = (uint32_t)gn;
                            jb.r = rn.x;
                            v4 = (uint32_t)gibbs_fp64<NB>(p, sA, jb);
                        }
                    }
                }
            }
            const uint32_t MLn = from_left(mid[0], outw);
            const uint32_t MRn = from_right(outw, (mid[2] & ~0xFFu) | v4);
            decide4(UL, UC, UR, MLn, MRn, DL, DC, DR, 0xAu & valid);
        }
        if (active) {
            uint8_t* xr = xcol + (long long)(r + HALO) * G.xpitch;
            auto store = [&](uint8_t* dst) {
                if (nvalid == 4) *reinterpret_cast<uint32_t*>(dst) = outw;
                else for (int b = 0; b < nvalid; ++b) dst[b] = (uint8_t)(outw >> (8 * b));
                if (G.periodic) {  // column pads (W even on a torus)
                    if ((G.W & 15) == 0) {
                        if (c0 < 16) *reinterpret_cast<uint32_t*>(dst + G.W) = outw;
                        if (c0 >= G.W - 16) *reinterpret_cast<uint32_t*>(dst - G.W) = outw;
                    } else {
                        if (c0 == 0) dst[G.W] = (uint8_t)outw;
                        if (c0 + nvalid == G.W) dst[-c0 - 1] = (uint8_t)(outw >> (8 * (nvalid - 1)));
                    }
                }
            };
            store(xr);
            if (G.periodic && G.self_halo_rows) {
                if (r < HALO) store(xr + (long long)G.rows * G.xpitch);
                if (r >= G.rows - HALO) store(xr - (long long)G.rows * G.xpitch);
            }
            if (count_enable) {  // the row is final after this colour (1 or 3) / parity launch
                uint16_t* cp = p.c.counts + chain * G.cchain + (long long)r * G.cpitch + c0;
                if (nvalid == 4) {
                    if (L == 2) {
                        const unsigned long long inc =
                            (unsigned long long)__byte_perm(outw, 0u, 0x4140) |
                            ((unsigned long long)__byte_perm(outw, 0u, 0x4342) << 32);
                        if (inc) atomicAdd(reinterpret_cast<unsigned long long*>(cp), inc);
                    } else {
                        unsigned todo = 0xFu;
                        while (todo) {
                            const int b0 = __ffs(todo) - 1;
                            const uint32_t kk = (outw >> (8 * b0)) & 0xFFu;
                            const uint32_t e = outw ^ (kk * 0x01010101u);
                            const uint32_t nz = (((e & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | e) & 0x80808080u;
                            const uint32_t eq = (~nz >> 7) & 0x01010101u;
                            const unsigned long long inc =
                                (unsigned long long)__byte_perm(eq, 0u, 0x4140) |
                                ((unsigned long long)__byte_perm(eq, 0u, 0x4342) << 32);
                            atomicAdd(reinterpret_cast<unsigned long long*>(cp + (long long)kk * G.cplane), inc);
                            todo &= ~(unsigned)(((eq & 1u) ? 1u : 0u) | ((eq & 0x100u) ? 2u : 0u) |
                                                ((eq & 0x10000u) ? 4u : 0u) | ((eq & 0x1000000u) ? 8u : 0u));
                        }
                    }
                } else {
                    for (int b = 0; b < nvalid; ++b) {
                        const int w = (int)((outw >> (8 * b)) & 0xFFu);
                        if (L == 2) cp[b] += (uint16_t)w;
                        else cp[(long long)w * G.cplane + b] += 1;
                    }
                }
            }
        }
        // slide the window by rstep rows
        if (r + rstep < rend) {
            if (NB == 8) {
#pragma unroll
                for (int j = 0; j < 3; ++j) up[j] = dn[j];
                load_row(r + 2, mid);
                load_row(r + 3, dn);
            } else {
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    up[j] = mid[j];
                    mid[j] = dn[j];
                }
                load_row(r + 2, dn);
            }
        }
    }
}

template <int NB, int LT, bool FUSED>
__global__ void __launch_bounds__(GB_THREADS, PCA_GB_MINB)
    sweep_gibbs_kernel(const __grid_constant__ GibbsSweepParams p, int R) {
    __shared__ GibbsSmem sm;
    pdl_begin();  // programmatic dependent launch (kernels.cuh): nothing is read before it
    gibbs_load_tables<LT>(p, sm);
    __syncthreads();
    gibbs_rows<NB, LT, FUSED, false>(p, sm, p.colour, p.c.t, p.c.count_enable, blockIdx.x,
                                      blockIdx.y, blockIdx.z, R);
}

// Small lattices: `nsweeps` Gibbs sweeps (one beta stage; p.c.count_enable = counting in the
// whole run) in one cooperative launch, every colour phase followed by a grid barrier.
template <int NB, int LT, bool FUSED>
__global__ void __launch_bounds__(GB_THREADS, PCA_GB_MINB)
    gibbs_multi_kernel(const __grid_constant__ GibbsSweepParams p, int R, int nrb, int nsweeps, int batch) {
    __shared__ GibbsSmem sm;
    gibbs_load_tables<LT>(p, sm);
    __syncthreads();
    const int xblocks = (((p.c.geo.W + 3) >> 2) + GB_THREADS - 1) / GB_THREADS;
    const int items = xblocks * nrb * batch;
    const int nph = (NB == 4 || FUSED) ? 2 : 4;
    for (int sw = 0; sw < nsweeps; ++sw) {
        for (int k = 0; k < nph; ++k) {
            const int cnt = p.c.count_enable && (FUSED || (k & 1));
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                const int xb = it % xblocks, rb = (it / xblocks) % nrb, chain = it / (xblocks * nrb);
                gibbs_rows<NB, LT, FUSED, true>(p, sm, k, p.c.t + (uint32_t)sw, cnt, xb, rb, chain, R);
            }
            if (gridDim.x == 1) {
                __syncthreads();
            } else {
                __threadfence();
                cg::this_grid().sync();
            }
        }
    }
}

template <int NB, int LT, bool FUSED>
int launch_gb(const GibbsSweepParams& p, int batch, int nsweeps, cudaStream_t s) {
    static LaunchInfo info[MAX_DEVICES];
    LaunchInfo& li = info[current_device()];
    if (!li.ok.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lock(launch_info_mutex());
        if (!li.ok.load(std::memory_order_relaxed)) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&li.sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.occ, sweep_gibbs_kernel<NB, LT, FUSED>, GB_THREADS, 0);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.mocc, gibbs_multi_kernel<NB, LT, FUSED>, GB_THREADS, 0);
            if (li.occ < 1) li.occ = 1;
            if (li.mocc < 1) li.mocc = 1;
            li.ok.store(true, std::memory_order_release);
        }
    }
    const int occ = li.occ, mocc = li.mocc, sms = li.sms;
    const Geometry& G = p.c.geo;
    const int nquads = (G.W + 3) / 4;
    int nr = p.c.rhi - p.c.rlo;
    if (G.nbhd == 8) nr = (nr + 1) / 2;  // rows of one parity
    if (nr <= 0) return 0;
    const long long xblocks = (nquads + GB_THREADS - 1) / GB_THREADS;
    const long long target = nsweeps > 1 ? (long long)sms * mocc : 4LL * sms * occ;
    long long R = ((long long)nr * xblocks * batch + target - 1) / target;
    if (R < 1) R = 1;
    long long nrb = (nr + R - 1) / R;
    if (nrb > 65535) {
        nrb = 65535;
        R = (nr + nrb - 1) / nrb;
    }
    if (nsweeps > 1) {
        const long long items = xblocks * nrb * batch;
        const long long slots = (long long)sms * mocc;
        const int grid = (int)(items < slots ? items : slots);
        GibbsSweepParams pp = p;
        int Ri = (int)R, nrbi = (int)nrb, ns = nsweeps, b = batch;
        void* args[] = {&pp, &Ri, &nrbi, &ns, &b};
        return (int)cudaLaunchCooperativeKernel((const void*)gibbs_multi_kernel<NB, LT, FUSED>, dim3(grid),
                                                dim3(GB_THREADS), args, 0, s);
    }
    dim3 grid((unsigned)xblocks, (unsigned)nrb, batch);
    return (int)launch_pdl(sweep_gibbs_kernel<NB, LT, FUSED>, grid, dim3(GB_THREADS), 0, s, p, (int)R);
}

}  // namespace

int launch_sweep_gibbs(const GibbsSweepParams& p, int batch, int nsweeps, void* stream) {
    const Geometry& G = p.c.geo;
    cudaStream_t s = (cudaStream_t)stream;
#define PCA_GB_LAUNCH(LTV)                                                                     \
    return G.nbhd == 8 ? (p.fused ? launch_gb<8, LTV, true>(p, batch, nsweeps, s)              \
                                  : launch_gb<8, LTV, false>(p, batch, nsweeps, s))            \
                       : launch_gb<4, LTV, false>(p, batch, nsweeps, s)
    switch (G.levels) {  // two levels: the exact binary path; the paper's level counts (and 3)
        case 2: PCA_GB_LAUNCH(2);  // get fully unrolled fp64 paths
        case 3: PCA_GB_LAUNCH(3);
        case 5: PCA_GB_LAUNCH(5);
        case 9: PCA_GB_LAUNCH(9);
        case 16: PCA_GB_LAUNCH(16);
        default: PCA_GB_LAUNCH(0);
    }
#undef PCA_GB_LAUNCH
}

}  // namespace pcab200
