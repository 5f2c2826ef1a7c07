// sweep_general.cu -- one synchronous lazy-PCA sweep for any number of levels (2..255).
//
// Uniform neighbourhood (all NB neighbours carry the same label s*, ~75-85% of the sites of
// a restored MRF image): p_i depends only on (s*, g_i, x_i), so the host tabulates for the
// current beta the integer thresholds T_k = ceil(F_k 2^32) - 1 of the cumulative
// probabilities (fp64, accumulated exactly as the oracle does, levels <= 16) and the new
// label is #{k : r > T_k} -- integer-exact, like the binary kernel.
//
// Otherwise, per site i (PAPER.md:462-477 with R1), in fp64:
//   w_s = e^{a n_i(s)} * e^{-b (lum g_i - lum s)^2} * e^{-c pen(x_i, s)}
//       = A[n_i(s)] * D[g_i][s] * I[x_i][s],   I[x][s] = (s == x ? 1 : Cw) for the paper's
// L0 inertia, the host table exp(-c |lum x - lum s|^p) for L1 / L2
// (the factorised form of exp(E_i(s)); A, D, Cw, I tabulated on the host in fp64),
// Z = sum_s w_s; the new label is min{k < l-1 : u Z < sum_{s<=k} w_s}, else l-1 (R14),
// with u = r 2^-32 from the site's Philox word.  Rounding differs from the oracle's
// exp(E - max E)/Z only in the last bits, so decisions can differ only when u lies within
// ~1e-15 of a cumulative probability (an allowed near-tie, R19).  When the factorised
// weights under/overflow (extreme beta, q, sigma) the site uses the oracle's log-domain form.
//
// One thread = 4 consecutive sites of a row (one Philox4x32-10 call).  The 3x12-byte
// neighbourhood window is fetched as 9 aligned 32-bit loads (L1-resident across the warp).
// Load balance: the fp64 sites of a warp are compacted into a per-warp shared-memory queue
// (ballot + popc) and processed round-robin by all 32 lanes, so a warp pays
// ceil(#fp64 sites / 32) fp64 evaluations instead of one per site slot that any lane needs.
// The free-boundary sentinel 0xFF never equals a label, so n_i(s) needs no position test.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "general_decide.cuh"
#include "kernels.cuh"
#include "tma_ring.cuh"  // from_left / from_right byte funnels

namespace pcab200 {
namespace {

namespace cg = cooperative_groups;

// resident 128-thread blocks per SM the register budget is sized for (measured on C5:
// 4 -> 262 us, 6 -> 238 us, 8 -> 245 us per sweep)
#ifndef PCA_GEN_MINB
#define PCA_GEN_MINB 6
#endif
constexpr int GEN_THREADS = 128;
constexpr int GEN_WARPS = GEN_THREADS / 32;
constexpr unsigned FULL = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t ldg4(const uint8_t* p) {
    return __ldg(reinterpret_cast<const uint32_t*>(p));
}

// Many levels (16 < L <= 64): the weights of the labels no neighbour carries are the stage
// table W0[g][x][s] = D[g][s] I[x][s], with prefix sums pfx[g][x][k].  Only the (at most NB)
// distinct neighbour labels change the weights, by (A[n_s] - 1) W0[s], so
//   Z = pfx[L-1] + sum_j corr_j,  F_k = pfx[k] + (sum of corr_j over neighbour labels <= k);
// the decision walks the segments between neighbour labels in ascending order and
// binary-searches the prefix table inside the segment that holds u Z: O(NB + log L) per site
// instead of O(L NB).  Rounding differs from the oracle's sequential sum only in the last
// bits (the fp64 path's near-tie semantics, R19).  Returns -1 when Z under/overflows.
template <int NB>
__device__ int decide_sparse(const GeneralSweepParams& p, const double* sA, const SiteJob& j) {
    const int L = p.c.geo.levels;
    const int xi = (int)(j.xg & 0xFFu), gi = (int)((j.xg >> 8) & 0xFFu);
    const size_t row = ((size_t)gi * L + xi) * L;
    const double* W0 = p.w0 + row;
    const double* PF = p.pfx + row;
    // the smallest neighbour label above `prev` (L when none) and how many neighbours carry it
    auto next_label = [&](int prev, int& n) {
        int best = L;
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const int v = (int)(((q < 4 ? j.nb_lo : j.nb_hi) >> (8 * (q & 3))) & 0xFFu);
            best = (v > prev && v < best) ? v : best;  // the sentinel 0xFF >= L never wins
        }
        n = 0;
#pragma unroll
        for (int q = 0; q < NB; ++q)
            n += (int)((((q < 4 ? j.nb_lo : j.nb_hi) >> (8 * (q & 3))) & 0xFFu) == (uint32_t)best);
        return best;
    };
    double Z = __ldg(PF + L - 1);
    for (int prev = -1;;) {
        int n;
        const int lab = next_label(prev, n);
        if (lab >= L) break;
        Z += (sA[n] - 1.0) * __ldg(W0 + lab);
        prev = lab;
    }
    if (!(Z >= 1e-290 && Z <= 1e290)) return -1;
    const double target = (double)j.r * (1.0 / 4294967296.0) * Z;
    double C = 0.0;
    int a = 0;
    for (int prev = -1;;) {
        int n;
        const int lab = next_label(prev, n);
        // labels a .. min(lab, L-1)-1 carry no neighbour: F_k = PF[k] + C
        const int b = min(lab, L - 1) - 1;
        if (b >= a && target < __ldg(PF + b) + C) {
            int lo = a, hi = b;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (target < __ldg(PF + mid) + C) hi = mid;
                else lo = mid + 1;
            }
            return lo;
        }
        if (lab >= L) break;
        C += (sA[n] - 1.0) * __ldg(W0 + lab);
        if (lab < L - 1 && target < __ldg(PF + lab) + C) return lab;
        a = lab + 1;
        prev = lab;
    }
    return L - 1;
}

// Uniform-neighbourhood thresholds staged in shared memory when the table is small.
__host__ __device__ constexpr int uthr_smem_entries(int LT) { return (LT > 0 && LT <= 9) ? LT * LT * LT * (LT - 1) : 1; }

// levels <= 8 known at compile time: the fp64 queue uses W0[g][x][s] = D[g][s] I[x][s] (the
// part of the weight that does not depend on the neighbours), built per block in shared
// memory (at 9 levels the table would cost a resident block per SM)
__host__ __device__ constexpr bool w0_smem(int LT) { return LT > 2 && LT <= 8; }

template <int LT>
struct GenSmem {
    double A[9];
    double D[LT > 2 ? LT * LT : 1];
    double I[LT > 2 ? LT * LT : 1];
    double W0[w0_smem(LT) ? LT * LT * LT : 1];
    uint32_t U[LT == 2 ? THR_ENTRIES : uthr_smem_entries(LT)];  // levels == 2: binary table
    // per lane, the quad's words a queued site needs (STAGE_WORDS: a stride that keeps the
    // 128-bit stores of a quarter-warp on distinct banks): UL UC UR ML | MR DL DC DR | x g - - |
    // r0 r1 r2 r3; the per-warp queue holds lane*4 + site
    alignas(16) uint32_t stage[GEN_WARPS][32 * 20];
    uint8_t queue[GEN_WARPS][128];
    uint8_t res[GEN_WARPS][128];
};

template <int LT>
__device__ __forceinline__ void gen_load_tables(const GeneralSweepParams& p, GenSmem<LT>& sm) {
    if (threadIdx.x < 9) sm.A[threadIdx.x] = p.A[threadIdx.x];
    if (LT > 2)
        for (int i = threadIdx.x; i < LT * LT; i += blockDim.x) {
            sm.D[i] = p.dtab[i];
            sm.I[i] = p.inertia_p != 0 ? p.itab[i] : 0.0;
        }
    if (w0_smem(LT))
        for (int i = threadIdx.x; i < LT * LT * LT; i += blockDim.x) {
            const int g = i / (LT * LT), x = (i / LT) % LT, s = i % LT;
            const double I = p.inertia_p != 0 ? p.itab[x * LT + s] : (s == x ? 1.0 : p.Cw);
            sm.W0[i] = p.dtab[g * LT + s] * I;
        }
    if (LT == 2)
        for (int i = threadIdx.x; i < THR_ENTRIES; i += blockDim.x) sm.U[i] = p.bthr[i];
    else if (LT > 0 && LT <= 9 && p.uthr != nullptr)
        for (int i = threadIdx.x; i < uthr_smem_entries(LT); i += blockDim.x) sm.U[i] = p.uthr[i];
}

// Work decomposition shared by both kernels: a block of GEN_THREADS threads covers QW
// consecutive quads (QW = the quad count rounded up to a power of two, at most GEN_THREADS)
// times RS = GEN_THREADS / QW row runs of R rows, so narrow lattices keep every lane busy.
struct Decomp {
    int QW, RS, R;  // quads per block row, row runs per block, rows per run
    int nxb, nrb;   // x-blocks, run-blocks (each RS runs)
};
__host__ __device__ inline Decomp make_decomp(int nquads, int nrows, int R) {
    Decomp d;
    d.QW = 1;
    while (d.QW < nquads && d.QW < GEN_THREADS) d.QW <<= 1;
    d.RS = GEN_THREADS / d.QW;
    d.R = R < 1 ? 1 : R;
    d.nxb = (nquads + d.QW - 1) / d.QW;
    const int runs = (nrows + d.R - 1) / d.R;
    d.nrb = (runs + d.RS - 1) / d.RS;
    return d;
}

// One quad column (4 sites, quad qd) of chain `chain` over local rows [rbeg, rend), sweep t:
// x_in -> x_out.  Every thread of the block calls it with the same `iters` (the warp-level
// queue needs uniform trip counts); lanes past their rows idle.  COH: x is read through L2
// (ld.global.cg) because an earlier sweep of the same launch wrote it; otherwise through the
// read-only path.
template <int NB, int LT, bool COH, bool PEERS = false>  // PEERS: edge rows also to the peers' halos
__device__ __forceinline__ void gen_rows(const GeneralSweepParams& p, GenSmem<LT>& sm,
                                         const uint8_t* __restrict__ x_in, uint8_t* __restrict__ x_out,
                                         uint32_t t, int count_enable, int qd, int chain, int rbeg,
                                         int rend, int iters) {
    constexpr bool SMEM_U = LT > 0 && LT <= 9;
    const Geometry& G = p.c.geo;
    const int L = LT > 0 ? LT : G.levels;  // a compile-time constant when LT fixes it
    const int nquads = (G.W + 3) >> 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool active = qd < nquads && rbeg < rend;
    if (__ballot_sync(FULL, active) == 0) return;  // warp-uniform exit
    const uint32_t tagchain = (TAG_PCA << 24) | (p.c.chain0 + (uint32_t)chain);
    const unsigned lt = (1u << lane) - 1u;
    uint32_t* stage = sm.stage[warp];
    uint8_t* queue = sm.queue[warp];
    uint8_t* res = sm.res[warp];
    // the uniform table exists for every level count <= 16 (UTHR_MAX_LEVELS)
    const bool use_u = (LT >= 2 && LT <= 16) || p.uthr != nullptr;
    const uint32_t* U = (SMEM_U || LT == 2) ? sm.U : p.uthr;
    const int c0 = 4 * qd;
    const int nvalid = active ? min(4, G.W - c0) : 0;
    const uint8_t* xcol = x_in + chain * G.xchain + XOFF + c0;
    const uint8_t* gcol = p.c.g + chain * G.gchain + XOFF + c0;

    // rolling 3-row window of the words left of / at / right of the quad
    uint32_t up[3] = {0, 0, 0}, mid[3] = {0, 0, 0}, dn[3] = {0, 0, 0};
    auto load_row = [&](const uint8_t* xr, uint32_t (&w)[3]) {
        if (COH) {
            w[0] = __ldcg(reinterpret_cast<const uint32_t*>(xr - 4));
            w[1] = __ldcg(reinterpret_cast<const uint32_t*>(xr));
            w[2] = __ldcg(reinterpret_cast<const uint32_t*>(xr + 4));
        } else {
            w[0] = ldg4(xr - 4);
            w[1] = ldg4(xr);
            w[2] = ldg4(xr + 4);
        }
    };
    // software pipeline: the x row r+2 and the g row r+1 are loaded one iteration ahead, so
    // the load latency overlaps a row of work (rows rbeg-1 .. rend+1 exist: HALO = 2)
    // (running row pointers: the next x row to fetch, the next g row, this row's output and
    // count words)
    uint32_t nxt[3] = {0, 0, 0}, gnext = 0;
    const uint8_t* xp = xcol + (long long)(rbeg - 1 + HALO) * G.xpitch;
    const uint8_t* gp = gcol + (long long)(rbeg + GHALO) * G.gpitch;
    if (active) {
        load_row(xp, up);
        load_row(xp + G.xpitch, mid);
        load_row(xp + 2 * G.xpitch, nxt);
        gnext = ldg4(gp);
    }
    xp += 3 * G.xpitch;
    gp += G.gpitch;
    uint8_t* op = x_out + chain * G.xchain + (long long)(rbeg + HALO) * G.xpitch + XOFF + c0;
    uint16_t* cp = p.c.counts + chain * G.cchain + (long long)rbeg * G.cpitch + c0;

    for (int it = 0; it < iters; ++it) {
        const int r = rbeg + it;
        const bool act = active && r < rend;
#pragma unroll
        for (int j = 0; j < 3; ++j) dn[j] = nxt[j];
        const uint32_t gword = gnext;
        if (act && r + 1 < rend) {
            load_row(xp, nxt);
            gnext = ldg4(gp);
        }
        xp += G.xpitch;
        gp += G.gpitch;
        const int grow = G.row0 + r;
        uint4 rnd = make_uint4(0, 0, 0, 0);
        if (act)
            rnd = philox4x32_10(make_uint4((uint32_t)qd, (uint32_t)grow, t, tagchain), p.c.keys);
        // the neighbours of the 4 sites, one byte per site (byte b = neighbour of site b)
        const uint32_t UL = from_left(up[0], up[1]), UC = up[1], UR = from_right(up[1], up[2]);
        const uint32_t ML = from_left(mid[0], mid[1]), MR = from_right(mid[1], mid[2]);
        const uint32_t DL = from_left(dn[0], dn[1]), DC = dn[1], DR = from_right(dn[1], dn[2]);
        const uint32_t rr[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
        const uint32_t xw = mid[1];
        uint32_t outw = 0u;
        if (LT == 2) {
            // two levels: every site is an integer-threshold decision (as sweep_binary.cu):
            // T[((np*9 + n1)*2 + g)*2 + x], n1 / np = label-1 / present neighbours (SWAR)
            auto one = [](uint32_t w) { return w & ~(w >> 1) & 0x01010101u; };  // 0xFF -> 0
            auto pres = [](uint32_t w) { return (~w >> 7) & 0x01010101u; };     // 0xFF -> 0
            uint32_t n1, np;
            if (NB == 8) {
                n1 = one(UL) + one(UC) + one(UR) + one(ML) + one(MR) + one(DL) + one(DC) + one(DR);
                np = pres(UL) + pres(UC) + pres(UR) + pres(ML) + pres(MR) + pres(DL) + pres(DC) + pres(DR);
            } else {
                n1 = one(UC) + one(ML) + one(MR) + one(DC);
                np = pres(UC) + pres(ML) + pres(MR) + pres(DC);
            }
            const uint32_t lo4 = (((n1 << 1) | gword) << 1) | xw;  // (n1*2 + g)*2 + x <= 35
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const uint32_t idx = ((np >> (8 * b)) & 0xFFu) * 36u + ((lo4 >> (8 * b)) & 0xFFu);
                outw |= (rr[b] > U[idx] ? 1u : 0u) << (8 * b);
            }
        } else {
            // uniform neighbourhood: all NB neighbour bytes equal (chain of XORs), SWAR zero test
            uint32_t D;
            if (NB == 8)
                D = (UL ^ UC) | (UC ^ UR) | (UR ^ ML) | (ML ^ MR) | (MR ^ DL) | (DL ^ DC) | (DC ^ DR);
            else
                D = (UC ^ ML) | (ML ^ MR) | (MR ^ DC);
            const uint32_t differ = (((D & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | D) & 0x80808080u;
            const uint32_t S0 = NB == 8 ? UL : UC;  // s* when uniform
            // <= 5 levels: the uniform-table rows (s*, g, x) of the 4 sites in one SWAR word
            // (s* masked to 3 bits: a non-uniform site's byte may be the sentinel; <= 199)
            const uint32_t IDX4 = LT > 2 && LT <= 5 ? (S0 & 0x07070707u) * (uint32_t)(LT * LT) + gword * (uint32_t)LT + xw : 0u;
            uint32_t needm = 0;  // bit b: site b goes to the warp's fp64 queue
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int s0 = (int)__byte_perm(S0, 0u, 0x4440 + b);
                const bool valid = act && b < nvalid;
                const bool uniform = use_u && ((differ >> (8 * b + 7)) & 1u) == 0u && s0 < L;
                if (SMEM_U) {
                    // branch-free: every lane reads a table row (row 0 when its site is not a
                    // valid uniform one) and counts the thresholds T_k >= r with borrow bits
                    const bool uni = valid && uniform;
                    int row;
                    if (LT <= 5) {
                        row = (int)__byte_perm(IDX4, 0u, 0x4440 + b);
                    } else {
                        const int xi = (int)__byte_perm(xw, 0u, 0x4440 + b);
                        const int gi = (int)__byte_perm(gword, 0u, 0x4440 + b);
                        row = (s0 * LT + gi) * LT + xi;
                    }
                    const uint32_t* T = U + (uni ? row * (LT - 1) : 0);
                    uint32_t ge = 0;
#pragma unroll
                    for (int k = 0; k < (SMEM_U ? LT - 1 : 1); ++k)
                        asm("{\n\t.reg .u32 d;\n\tsub.cc.u32 d, %1, %2;\n\taddc.u32 %0, %0, 0;\n\t}"
                            : "+r"(ge) : "r"(T[k]), "r"(rr[b]));
                    outw |= (uni ? (uint32_t)(LT - 1) - ge : 0u) << (8 * b);
                } else if (valid && uniform) {
                    // every neighbour carries s* = s0 (so all NB exist): integer thresholds
                    const int xi = (int)__byte_perm(xw, 0u, 0x4440 + b);
                    const int gi = (int)__byte_perm(gword, 0u, 0x4440 + b);
                    const uint32_t* T = U + (size_t)((s0 * L + gi) * L + xi) * (L - 1);
                    int w = 0;
                    if (LT > 0) {
#pragma unroll
                        for (int k = 0; k < (LT > 0 ? LT - 1 : 1); ++k) w += (rr[b] > __ldg(T + k)) ? 1 : 0;
                    } else {
                        for (int k = 0; k < L - 1; ++k) w += (rr[b] > __ldg(T + k)) ? 1 : 0;
                    }
                    outw |= (uint32_t)w << (8 * b);
                }
                needm |= (valid && !uniform) ? 1u << b : 0u;
            }
            if (__ballot_sync(FULL, needm != 0u)) {  // warp-uniform
                // a lane with queued sites stages its quad's words once; the queue holds
                // (lane, site) and the consumer lane reads the words it needs
                if (needm) {
                    uint4* st = reinterpret_cast<uint4*>(stage + lane * 20);
                    st[0] = make_uint4(UL, UC, UR, ML);
                    st[1] = make_uint4(MR, DL, DC, DR);
                    st[2] = make_uint4(xw, gword, 0u, 0u);
                    st[3] = make_uint4(rnd.x, rnd.y, rnd.z, rnd.w);
                }
                int qpos[4];
                int qbase = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const bool need = (needm >> b) & 1u;
                    const unsigned m = __ballot_sync(FULL, need);
                    const int pos = qbase + __popc(m & lt);
                    PCA_DCHECK(!need || pos < 128);
                    if (need) queue[pos] = (uint8_t)(lane * 4 + b);
                    qpos[b] = need ? pos : -1;
                    qbase += __popc(m);
                }
                __syncwarp();
                for (int i = lane; i < qbase; i += 32) {
                    const int e = queue[i];
                    const int sb = e & 3;
                    const uint32_t* sw = stage + (e >> 2) * 20;
                    const uint4 w0 = *reinterpret_cast<const uint4*>(sw);
                    const uint4 w1 = *reinterpret_cast<const uint4*>(sw + 4);
                    const uint2 xg = *reinterpret_cast<const uint2*>(sw + 8);
                    const uint32_t rs = sw[12 + sb];
                    int w = -1;
                    if (w0_smem(LT))
                        w = decide_fp64_w0<NB, (w0_smem(LT) ? LT : 3)>(sm.A, sm.W0, w0, w1, xg.x, xg.y, rs, sb);
                    if (w < 0) {
                        const uint32_t sel = (uint32_t)sb | ((uint32_t)(sb + 4) << 4);  // byte sb of a, of b
                        SiteJob jb;
                        if (NB == 8) {
                            jb.nb_lo = __byte_perm(__byte_perm(w0.x, w0.y, sel), __byte_perm(w0.z, w0.w, sel), 0x5410);
                            jb.nb_hi = __byte_perm(__byte_perm(w1.x, w1.y, sel), __byte_perm(w1.z, w1.w, sel), 0x5410);
                        } else {  // UC, ML, MR, DC
                            jb.nb_lo = __byte_perm(__byte_perm(w0.y, w0.w, sel), __byte_perm(w1.x, w1.z, sel), 0x5410);
                            jb.nb_hi = 0u;
                        }
                        jb.xg = __byte_perm(xg.x, xg.y, sel) & 0xFFFFu;
                        jb.r = rs;
                        if (!w0_smem(LT) && LT > 2) w = decide_fp64_fixed<NB, (LT > 2 ? LT : 3)>(p, sm.A, sm.D, sm.I, jb);
                        else if (LT == 0 && p.pfx != nullptr) w = decide_sparse<NB>(p, sm.A, jb);
                        if (w < 0) w = decide_fp64<NB>(p, sm.A, jb);
                    }
                    PCA_DCHECK(w >= 0 && w < L);
                    res[i] = (uint8_t)w;
                }
                __syncwarp();
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (qpos[b] >= 0) outw |= (uint32_t)res[qpos[b]] << (8 * b);
                __syncwarp();
            }
        }
        if (act) {
            auto store = [&](uint8_t* dst) {
                if (nvalid == 4) *reinterpret_cast<uint32_t*>(dst) = outw;
                else for (int b = 0; b < nvalid; ++b) dst[b] = (uint8_t)(outw >> (8 * b));
                if (G.periodic) {  // column pads (see kernels.cuh)
                    if ((G.W & 15) == 0) {
                        if (c0 < 16) *reinterpret_cast<uint32_t*>(dst + G.W) = outw;
                        if (c0 >= G.W - 16) *reinterpret_cast<uint32_t*>(dst - G.W) = outw;
                    } else {
                        if (c0 == 0) dst[G.W] = (uint8_t)outw;
                        if (c0 + nvalid == G.W) dst[-c0 - 1] = (uint8_t)(outw >> (8 * (nvalid - 1)));
                    }
                }
            };
            store(op);
            if (G.periodic && G.self_halo_rows) {
                if (r < HALO) store(op + (long long)G.rows * G.xpitch);
                if (r >= G.rows - HALO) store(op - (long long)G.rows * G.xpitch);
            }
            // device-initiated halo exchange: the edge rows straight into the peers' halo rows
            // (compiled out otherwise: even never-taken checks cost ~5% of a C5 sweep)
            if (PEERS) {
                if (p.c.peer_up != nullptr && r == 0) store(p.c.peer_up + chain * p.c.peer_up_chain + XOFF + c0);
                if (p.c.peer_dn != nullptr && r == G.rows - 1)
                    store(p.c.peer_dn + chain * p.c.peer_dn_chain + XOFF + c0);
            }
            if (count_enable) {
                if (nvalid == 4) {
                    // the quad's 4 counters of a plane form one 8-byte word; each distinct label
                    // of the quad adds its per-site increments with one fire-and-forget 64-bit
                    // reduction (no lane carries: counts stay <= 65535), so the count update
                    // costs no load latency
                    if (L == 2) {
                        const unsigned long long inc =
                            (unsigned long long)__byte_perm(outw, 0u, 0x4140) |
                            ((unsigned long long)__byte_perm(outw, 0u, 0x4342) << 32);
                        if (inc) atomicAdd(reinterpret_cast<unsigned long long*>(cp), inc);
                    } else {
                        uint32_t rem = 0x01010101u;  // bit 8b: site b still to count
                        do {
                            const uint32_t k = __byte_perm(outw, 0u, 0x4440u + ((__ffs(rem) - 1) >> 3));
                            // bytes equal to k -> 0x01 per byte
                            const uint32_t e = outw ^ (k * 0x01010101u);
                            const uint32_t nz = (((e & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | e) & 0x80808080u;
                            const uint32_t eq = (~nz >> 7) & 0x01010101u;
                            const unsigned long long inc =
                                (unsigned long long)__byte_perm(eq, 0u, 0x4140) |
                                ((unsigned long long)__byte_perm(eq, 0u, 0x4342) << 32);
                            atomicAdd(reinterpret_cast<unsigned long long*>(cp + (long long)k * G.cplane), inc);
                            rem &= ~eq;
                        } while (rem);
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
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            up[j] = mid[j];
            mid[j] = dn[j];
        }
        op += G.xpitch;
        cp += G.cpitch;
    }
}

template <int NB, int LT, bool PEERS>  // LT: levels known at compile time, 0 = any
__global__ void __launch_bounds__(GEN_THREADS, PCA_GEN_MINB)
    sweep_general_kernel(const __grid_constant__ GeneralSweepParams p, int R) {
    __shared__ GenSmem<LT> sm;
    pdl_begin();  // programmatic dependent launch (kernels.cuh): nothing is read before it
    gen_load_tables<LT>(p, sm);
    __syncthreads();
    const Decomp d = make_decomp(((p.c.geo.W + 3) >> 2), p.c.rhi - p.c.rlo, R);
    const int qd = blockIdx.x * d.QW + (threadIdx.x & (d.QW - 1));
    const int rbeg = p.c.rlo + (blockIdx.y * d.RS + threadIdx.x / d.QW) * d.R;
    const int rend = min(rbeg + d.R, p.c.rhi);
    gen_rows<NB, LT, false, PEERS>(p, sm, p.c.x_in, p.c.x_out, p.c.t, p.c.count_enable, qd, blockIdx.z,
                            rbeg, rend, d.R);
}

// Small lattices: `nsweeps` consecutive sweeps (one beta stage, one counting mode) in ONE
// cooperative launch, the grid synchronising between sweeps, instead of one launch per sweep
// (a 64^2 or 256^2 sweep is a few microseconds of launch latency and under a microsecond of
// work).  Work items (x-block, row block, chain) are distributed grid-stride; the double
// buffer alternates in the kernel.  Same per-site code, same chain.
template <int NB, int LT>
__global__ void __launch_bounds__(GEN_THREADS, PCA_GEN_MINB)
    sweep_multi_kernel(const __grid_constant__ GeneralSweepParams p, int R, int nsweeps, int batch) {
    __shared__ GenSmem<LT> sm;
    gen_load_tables<LT>(p, sm);
    __syncthreads();
    const Decomp d = make_decomp(((p.c.geo.W + 3) >> 2), p.c.rhi - p.c.rlo, R);
    const int items = d.nxb * d.nrb * batch;
    for (int sw = 0; sw < nsweeps; ++sw) {
        const uint8_t* xi = (sw & 1) ? p.c.x_out : p.c.x_in;
        uint8_t* xo = (sw & 1) ? const_cast<uint8_t*>(p.c.x_in) : p.c.x_out;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            const int xb = it % d.nxb;
            const int rb = (it / d.nxb) % d.nrb;
            const int chain = it / (d.nxb * d.nrb);
            const int qd = xb * d.QW + (threadIdx.x & (d.QW - 1));
            const int rbeg = p.c.rlo + (rb * d.RS + threadIdx.x / d.QW) * d.R;
            const int rend = min(rbeg + d.R, p.c.rhi);
            gen_rows<NB, LT, true>(p, sm, xi, xo, p.c.t + (uint32_t)sw, p.c.count_enable, qd, chain,
                                   rbeg, rend, d.R);
        }
        // every store of this sweep (x, halos, count reductions) before any read of the next;
        // a one-block grid needs only the block barrier
        if (gridDim.x == 1) {
            __syncthreads();
        } else {
            __threadfence();
            cg::this_grid().sync();
        }
    }
}

template <int NB, int LT>
struct GenLaunch {
    // per device: occupancy of both kernels at their dynamic shared memory, SM count
    static LaunchInfo& get() {
        static LaunchInfo info[MAX_DEVICES];
        LaunchInfo& li = info[current_device()];
        if (!li.ok.load(std::memory_order_acquire)) {
            std::lock_guard<std::mutex> lock(launch_info_mutex());
            if (!li.ok.load(std::memory_order_relaxed)) {
                int dev = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&li.sms, cudaDevAttrMultiProcessorCount, dev);
                const int smem = (int)sizeof(GenSmem<LT>);
                cudaFuncSetAttribute(sweep_general_kernel<NB, LT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                cudaFuncSetAttribute(sweep_general_kernel<NB, LT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                cudaFuncSetAttribute(sweep_multi_kernel<NB, LT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                // NB: the tables are static shared memory, so passing `smem` as dynamic shared memory
            // counts them twice; that halves occ at 9 and 16 levels, and the resulting longer
            // row runs measured faster (2048^2, 9 levels: 77.8 vs 114-117 us per sweep with the
            // exact occupancy), so occ is used as a sizing heuristic, not a residency count
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.occ, sweep_general_kernel<NB, LT, false>, GEN_THREADS, smem);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.mocc, sweep_multi_kernel<NB, LT>, GEN_THREADS, smem);
                if (li.occ < 1) li.occ = 1;
                if (li.mocc < 1) li.mocc = 1;
                li.ok.store(true, std::memory_order_release);
            }
        }
        return li;
    }
};

template <int NB, int LT>
int launch_g(const GeneralSweepParams& p, int batch, int nsweeps, cudaStream_t s) {
    const LaunchInfo& GL = GenLaunch<NB, LT>::get();
    const Geometry& G = p.c.geo;
    const int nquads = (G.W + 3) / 4;
    const int nr = p.c.rhi - p.c.rlo;
    if (nr <= 0) return 0;
    const Decomp d1 = make_decomp(nquads, nr, 1);
    const long long quadrows = (long long)d1.nxb * d1.QW * nr * batch;  // thread-rows of work
    if (nsweeps > 1) {
        // spread the thread-rows over the co-resident blocks, one row per thread when they fit
        const long long slots = (long long)GL.sms * GL.mocc;
        long long R = (quadrows + slots * GEN_THREADS - 1) / (slots * GEN_THREADS);
        if (R < 1) R = 1;
        const Decomp d = make_decomp(nquads, nr, (int)R);
        const long long items = (long long)d.nxb * d.nrb * batch;
        const int grid = (int)(items < slots ? items : slots);
        GeneralSweepParams pp = p;
        int Ri = (int)R, ns = nsweeps, b = batch;
        void* args[] = {&pp, &Ri, &ns, &b};
        return (int)cudaLaunchCooperativeKernel((const void*)sweep_multi_kernel<NB, LT>, dim3(grid),
                                                dim3(GEN_THREADS), args, 0, s);
    }
    // rows per run: about four waves of blocks (the fp64 share of a row varies, so several
    // waves balance the tail), each thread walking a run of rows with a rolling window
    const long long target = 4LL * GL.sms * GL.occ * GEN_THREADS;
    long long R = (quadrows + target - 1) / target;
    if (R < 1) R = 1;
    Decomp d = make_decomp(nquads, nr, (int)R);
    while (d.nrb > 65535) d = make_decomp(nquads, nr, d.R * 2);
    dim3 grid((unsigned)d.nxb, (unsigned)d.nrb, batch);
    if (p.c.peer_up != nullptr || p.c.peer_dn != nullptr)
        return (int)launch_pdl(sweep_general_kernel<NB, LT, true>, grid, dim3(GEN_THREADS), 0, s, p, d.R);
    return (int)launch_pdl(sweep_general_kernel<NB, LT, false>, grid, dim3(GEN_THREADS), 0, s, p, d.R);
}

}  // namespace

int launch_sweep_general(const GeneralSweepParams& p, int batch, int nsweeps, void* stream) {
    // the table kernel sweeps one launch per sweep; runs of sweeps on small lattices (one
    // cooperative launch, latency-bound) stay on the general kernel's multi-sweep variant:
    // C2 256^2, l = 5: 3.9 us per sweep against 6.2 us for the table kernel's (256-thread
    // blocks, fewer of them, and a queue drain at the end of every one-row run)
    if (p.tab != nullptr && nsweeps <= 1) return launch_sweep_table(p, batch, nsweeps, stream);
    const Geometry& G = p.c.geo;
    cudaStream_t s = (cudaStream_t)stream;
#define PCA_GEN_LAUNCH(LTV) \
    return G.nbhd == 8 ? launch_g<8, LTV>(p, batch, nsweeps, s) : launch_g<4, LTV>(p, batch, nsweeps, s)
    switch (G.levels) {  // two levels: exact integer path; the paper's level counts (and 3)
        case 2: PCA_GEN_LAUNCH(2);  // get fully unrolled fp64 paths
        case 3: PCA_GEN_LAUNCH(3);
        case 5: PCA_GEN_LAUNCH(5);
        case 9: PCA_GEN_LAUNCH(9);
        case 16: PCA_GEN_LAUNCH(16);
        default: PCA_GEN_LAUNCH(0);
    }
#undef PCA_GEN_LAUNCH
}

}  // namespace pcab200
