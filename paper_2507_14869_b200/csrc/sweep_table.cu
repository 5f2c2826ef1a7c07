// sweep_table.cu -- the synchronous lazy-PCA sweep for 3..5 levels (the paper's 5-level images,
// PAPER.md:504-506) driven by neighbour-histogram tables.
//
// Per site i (R1) the law of the new label depends on x_t only through the
// neighbour histogram n_i(.), g_i and x_i.  Here every site's histogram is formed as ONE
// 32-bit word h of 4-bit counts (nibble s = n_i(s)), from one-hot nibble words of the window
// (1 << 4 label; the free-boundary sentinel 0xFF shifts the 1 out): vertical sums of three
// rows per column, then three columns per site -- a few integer instructions per site for the
// whole histogram.
//
// Interior sites whose neighbours carry at most two distinct labels (~97% of a restored image,
// all uniform and two-label neighbourhoods) are decided exactly as the binary kernel decides
// two-level sites: the host tabulates, once per beta stage and in the oracle's fp64
// arithmetic, the integer thresholds T_k = ceil(F_k 2^32) - 1 of the cumulative law for every
// such histogram and every (g, x); the device finds the histogram's row with a multiplicative
// hash (h * magic) >> (32 - hbits) into a collision-free slot table whose tag check also
// detects the other sites, and the new label is #{k : r > T_k} (borrow bits), bit-exact with
// the oracle's u < F_k.
//
// The remaining sites (three or more neighbour labels, fewer neighbours at a free boundary)
// are queued: a lane whose quad has such sites appends one record (histograms, Philox words,
// g and x words, position, site mask) to its warp's queue in shared memory (ballot
// compaction), and once 32 records are pending (or at the end of the run) the 32 lanes decide
// them in fp64 -- w_s = A[n_s] W0[g][x][s], the general kernel's CDF count (near-tie semantics
// R19; stages where those weights could under/overflow run on the general kernel, which has
// the oracle's log-domain form).  The producer stores the
// quad's word with a placeholder byte; the drain patches the byte (and its torus pads / halo
// rows / peer rows) and adds its MPM count after a __syncwarp, which orders the two in the
// warp.
//
// MPM counts: uint8 deltas per level plane (GeneralSweepParams.tdc), one 32-bit reduction per
// distinct label of a quad with the per-site byte increments (half the count bytes of the
// uint16 planes, no 64-bit increment assembly); the runtime folds them into the uint16 counts
// at most every 255 counted sweeps and at the end of every pca_sweep call.
//
// Data movement: a thread owns a quad of 4 sites (one Philox4x32-10 call) and walks a run of
// rows with a rolling 3-row window of one-hot words (the next x row and g row prefetched one
// row ahead, as in sweep_general.cu); the table blob reaches each block's shared memory with
// one TMA bulk copy.  One launch per sweep: runs of sweeps on small lattices (one cooperative
// launch) use the general kernel's multi-sweep variant, which is faster there.
#include <cuda_runtime.h>

#include <cmath>

#include "kernels.cuh"
#include "tma_ring.cuh"

namespace pcab200 {
namespace {

constexpr int TB_THREADS = 256;
constexpr int TB_WARPS = TB_THREADS / 32;
constexpr unsigned FULL = 0xFFFFFFFFu;
#ifndef PCA_TAB_MINB
#define PCA_TAB_MINB 3
#endif
// 1: the threshold rows are read from the workspace copy of the blob (L1/L2-cached) instead of
// the block's shared-memory copy, so a block's shared memory is only A, W0, slots and queues
#ifndef PCA_TAB_THR_GLOBAL
#define PCA_TAB_THR_GLOBAL 0
#endif
// waves of resident blocks the row runs are sized for (measured, us per sweep at C5 t = 700 /
// t = 900 / 8192^2 l = 5 t = 0 / t = 1000: 1 150/190/428/302, 2 111/139/400/263, 3 107/134/
// 402/263, 4 101/127/392/259, 5 105/130/393/261, 6 104/129/392/264, 8 104/130/397/266, 12 108/
// 132/398/269)
#ifndef PCA_TAB_PDL
#define PCA_TAB_PDL 1  // programmatic dependent launch between consecutive sweep launches
#endif
#ifndef PCA_TAB_WAVES
#define PCA_TAB_WAVES 4
#endif
constexpr int TAB_MAX_BYTES = 48 * 1024;  // blob limit (3..5 levels: <= 42 KB)

__host__ __device__ constexpr int tab_tp(int L) { return L == 3 ? 2 : 4; }

__device__ __forceinline__ uint32_t shl_clamp1(uint32_t n) {  // 1 << n, 0 when n >= 32
    uint32_t r;
    asm("shl.b32 %0, 1, %1;" : "=r"(r) : "r"(n));
    return r;
}

// one-hot nibble words of the 6 columns c0-1 .. c0+4 of a row from its 3 label words
// (left of, at, right of the quad); a label byte v <= 7 becomes 1 << 4v, the sentinel 0xFF
// (0x3F << 2 = 252) becomes 0
__device__ __forceinline__ void onehots(const uint32_t (&w)[3], uint32_t (&o)[6]) {
    const uint32_t c4 = (w[1] & 0x3F3F3F3Fu) << 2;
    o[0] = shl_clamp1(((w[0] >> 24) & 0x3Fu) << 2);
#pragma unroll
    for (int b = 0; b < 4; ++b) o[1 + b] = shl_clamp1(__byte_perm(c4, 0u, 0x4440u + b));
    o[5] = shl_clamp1((w[2] & 0x3Fu) << 2);
}

// A queued quad: a lane whose quad has sites without a table row stores one record (its four
// histograms, its Philox words, its g and x words, row << 16 | first column, the mask of the
// queued sites); the drain decides the masked sites.
struct Rec {
    uint4 h, r;
    uint32_t gw, xw, rc0, mask;
};
constexpr int QCAP = 64;  // records per warp: < 32 pending before a row adds at most 32

// the block's table blob and record queues live in the dynamic shared memory below; offsets
// are 32-bit so every access is an LDS/STS with a 32-bit address
extern __shared__ __align__(16) uint8_t tab_smem_buf[];
constexpr int BLOB = 16;  // the blob follows the bulk copy's mbarrier
struct TabShared {
    uint32_t slot, thr, queue;  // byte offsets in tab_smem_buf (queue: this warp's)
    const uint8_t* gthr;        // PCA_TAB_THR_GLOBAL: the workspace copy of the rows
};
__device__ __forceinline__ const double* sm_A() {
    return reinterpret_cast<const double*>(tab_smem_buf + BLOB);
}
__device__ __forceinline__ const double* sm_AW() {
    return reinterpret_cast<const double*>(tab_smem_buf + BLOB + TAB_OFF_W0);
}

// fp64 decision of a queued site from its histogram: the general kernel's factorised weights
// w_s = A[n_s] W0[g][x][s] and CDF count (near-tie semantics R19).  The runtime selects this
// kernel only for beta stages where the factorised weights cannot under/overflow
// (Z >= A[n_x] D[g][x] >= exp(-b) >= 1e-290 and Z <= L A[NB] <= 1e290, build_tables), so the
// general kernel's log-domain fallback is never needed here.
template <int L>
__device__ __forceinline__ int decide_hist_fp64(uint32_t h, int gi, int xi, uint32_t r) {
    // w_s = A[n_s] W0[g][x][s], read as the stage's precomputed products AW[g][x][s][n_s]
    const double* AWrow = sm_AW() + (gi * L + xi) * L * 9;
    double w[L];
    double Z = 0.0;
#pragma unroll
    for (int s = 0; s < L; ++s) {
        w[s] = AWrow[s * 9 + ((h >> (4 * s)) & 0xFu)];
        Z += w[s];
    }
    const double target = (double)r * (1.0 / 4294967296.0) * Z;
    double F = 0.0;
    int res = 0;
#pragma unroll
    for (int s = 0; s < L - 1; ++s) {
        F += w[s];
        res += (F <= target) ? 1 : 0;
    }
    return res;
}

// Decomposition (as sweep_general.cu's, for TB_THREADS-thread blocks): a block covers QW
// quads x RS row runs of R rows.
struct TDecomp {
    int QW, RS, R, nxb, nrb;
};
__host__ __device__ inline TDecomp tdecomp(int nquads, int nrows, int R) {
    TDecomp d;
    d.QW = 1;
    while (d.QW < nquads && d.QW < TB_THREADS) d.QW <<= 1;
    d.RS = TB_THREADS / d.QW;
    d.R = R < 1 ? 1 : R;
    d.nxb = (nquads + d.QW - 1) / d.QW;
    const int runs = (nrows + d.R - 1) / d.R;
    d.nrb = (runs + d.RS - 1) / d.RS;
    return d;
}

// Store one byte of the new state (a queued site's label) at local (row, col) of a padded
// buffer, with the torus column pads / row halos and the peers' halo rows (as the quad store)
template <bool PEERS>
__device__ __forceinline__ void put_site(const GeneralSweepParams& p, uint8_t* x_out, int chain,
                                         int row, int col, uint8_t v) {
    const Geometry& G = p.c.geo;
    auto put = [&](uint8_t* rp) {  // rp: padded row base
        rp[XOFF + col] = v;
        if (G.periodic) {
            if ((G.W & 15) == 0) {
                if (col < 16) rp[XOFF + G.W + col] = v;
                if (col >= G.W - 16) rp[XOFF + col - G.W] = v;
            } else {
                if (col == 0) rp[XOFF + G.W] = v;
                if (col == G.W - 1) rp[XOFF - 1] = v;
            }
        }
    };
    uint8_t* rp = x_out + chain * G.xchain + (long long)(row + HALO) * G.xpitch;
    put(rp);
    if (G.periodic && G.self_halo_rows) {
        if (row < HALO) put(rp + (long long)G.rows * G.xpitch);
        if (row >= G.rows - HALO) put(rp - (long long)G.rows * G.xpitch);
    }
    if (PEERS) {
        if (p.c.peer_up != nullptr && row == 0) put(p.c.peer_up + chain * p.c.peer_up_chain);
        if (p.c.peer_dn != nullptr && row == G.rows - 1) put(p.c.peer_dn + chain * p.c.peer_dn_chain);
    }
}

// the warp decides the queued sites of its qn pending records (a record per lane per round),
// patches their bytes and counts them
template <int L, bool PEERS>
__device__ __forceinline__ void drain(const GeneralSweepParams& p, uint32_t qoff, uint8_t* x_out,
                                      int chain, int count_enable, int qn, int lane) {
    __syncwarp();  // the records and the producers' quad stores are visible to the whole warp
    const Geometry& G = p.c.geo;
    PCA_DCHECK(qn <= QCAP);
    for (int i = lane; i < qn; i += 32) {
        const uint8_t* rec = tab_smem_buf + qoff + i * (uint32_t)sizeof(Rec);
        const uint4 tail = *reinterpret_cast<const uint4*>(rec + 32);  // gw, xw, rc0, mask
        const int row = (int)(tail.z >> 16), c0 = (int)(tail.z & 0xFFFFu);
        // the record's row bases, once per record; a quad away from the torus column pads, the
        // wrapped halo rows and the peers' rows stores its bytes plainly (put_site otherwise)
        uint8_t* xq = x_out + chain * G.xchain + (long long)(row + HALO) * G.xpitch + XOFF + c0;
        unsigned* dq = reinterpret_cast<unsigned*>(p.tdc + chain * p.tdc_chain + (long long)row * G.cpitch + c0);
        const bool special =
            (G.periodic && (c0 < 16 || c0 + 4 > G.W - 16 ||
                            (G.self_halo_rows && (row < HALO || row >= G.rows - HALO)))) ||
            (PEERS && (row == 0 || row == G.rows - 1));
        for (uint32_t m = tail.w; m != 0u; m &= m - 1u) {
            const int b = __ffs(m) - 1;
            const uint32_t h = *reinterpret_cast<const uint32_t*>(rec + 4 * b);
            const uint32_t r = *reinterpret_cast<const uint32_t*>(rec + 16 + 4 * b);
            const int gi = (int)__byte_perm(tail.x, 0u, 0x4440u + b);
            const int xi = (int)__byte_perm(tail.y, 0u, 0x4440u + b);
            const int w = decide_hist_fp64<L>(h, gi, xi, r);
            PCA_DCHECK(w >= 0 && w < L && gi < L && xi < L && row >= 0 && row < G.rows && c0 + b < G.W);
            if (special) put_site<PEERS>(p, x_out, chain, row, c0 + b, (uint8_t)w);
            else xq[b] = (uint8_t)w;
            if (count_enable) atomicAdd(dq + (long long)w * (p.tdc_plane >> 2), 1u << (8 * b));
        }
    }
    __syncwarp();  // the queue is free again
}

template <int NB, int L, bool COH, bool PEERS>
__device__ __forceinline__ void tab_rows(const GeneralSweepParams& p, const TabShared& S,
                                         const uint8_t* __restrict__ x_in, uint8_t* __restrict__ x_out,
                                         uint32_t t, int count_enable, int qd, int chain, int rbeg,
                                         int rend, int iters) {
    constexpr int TP = tab_tp(L);
    const Geometry& G = p.c.geo;
    const int nquads = (G.W + 3) >> 2;
    const int lane = threadIdx.x & 31;
    const bool active = qd < nquads && rbeg < rend;
    if (__ballot_sync(FULL, active) == 0) return;  // warp-uniform exit
    const uint32_t tagchain = (TAG_PCA << 24) | (p.c.chain0 + (uint32_t)chain);
    const unsigned lt = (1u << lane) - 1u;
    const int c0 = 4 * qd;
    const int nvalid = active ? min(4, G.W - c0) : 0;
    const uint32_t vmask = (1u << nvalid) - 1u;  // valid sites of the quad
    const uint8_t* xcol = x_in + chain * G.xchain + XOFF + c0;
    const uint8_t* gcol = p.c.g + chain * G.gchain + XOFF + c0;
    const uint32_t hmul = p.tab_magic;
    const int hsh = 32 - p.tab_hbits;
    // the row-independent Philox prefix of the quad's counter (qd, row, t, tag|chain)
    const PhiloxPre ppre = philox_pre((uint32_t)qd, t, tagchain, p.c.keys);

    auto load_row = [&](const uint8_t* xr, uint32_t (&w)[3]) {
        if (COH) {
            w[0] = __ldcg(reinterpret_cast<const uint32_t*>(xr - 4));
            w[1] = __ldcg(reinterpret_cast<const uint32_t*>(xr));
            w[2] = __ldcg(reinterpret_cast<const uint32_t*>(xr + 4));
        } else {
            w[0] = __ldg(reinterpret_cast<const uint32_t*>(xr - 4));
            w[1] = __ldg(reinterpret_cast<const uint32_t*>(xr));
            w[2] = __ldg(reinterpret_cast<const uint32_t*>(xr + 4));
        }
    };
    // rolling window: one-hot words of rows r-1 (OU), r (OM); the raw centre word of row r
    // (x_i); the next x row and g row prefetched one iteration ahead
    uint32_t OU[6] = {0, 0, 0, 0, 0, 0}, OM[6] = {0, 0, 0, 0, 0, 0};
    uint32_t xmid = 0, nxt[3] = {0, 0, 0}, gnext = 0;
    const uint8_t* xp = xcol + (long long)(rbeg - 1 + HALO) * G.xpitch;
    const uint8_t* gp = gcol + (long long)(rbeg + GHALO) * G.gpitch;
    if (active) {
        uint32_t w[3];
        load_row(xp, w);
        onehots(w, OU);
        load_row(xp + G.xpitch, w);
        onehots(w, OM);
        xmid = w[1];
        load_row(xp + 2 * G.xpitch, nxt);
        gnext = __ldg(reinterpret_cast<const uint32_t*>(gp));
    }
    xp += 3 * G.xpitch;
    gp += G.gpitch;
    uint8_t* op = x_out + chain * G.xchain + (long long)(rbeg + HALO) * G.xpitch + XOFF + c0;
    // the MPM count deltas of this quad column (uint8 [levels] planes; sweep_table.cu header)
    PCA_DCHECK(!count_enable || p.tdc != nullptr);
    uint8_t* dp = p.tdc + chain * p.tdc_chain + (long long)rbeg * G.cpitch + c0;
    int qn = 0;  // pending records of the warp (warp-uniform)

    for (int it = 0; it < iters; ++it) {
        const int r = rbeg + it;
        const bool act = active && r < rend;
        uint32_t OD[6];
        onehots(nxt, OD);
        const uint32_t xdn = nxt[1];
        const uint32_t gword = gnext;
        if (act) {  // (the last row's prefetch reads x row rend+1 and g row rend: halo rows, unused)
            load_row(xp, nxt);
            gnext = __ldg(reinterpret_cast<const uint32_t*>(gp));
        }
        xp += G.xpitch;
        gp += G.gpitch;
        const int grow = G.row0 + r;
        uint4 rnd = make_uint4(0, 0, 0, 0);
        if (act) rnd = philox_row<true>(ppre, (uint32_t)grow, p.c.keys);
        const uint32_t rr[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
        // ---- neighbour histograms, one 32-bit word of nibbles per site ----
        uint32_t h[4];
        if (NB == 8) {
            uint32_t V[6], Wc[6];
#pragma unroll
            for (int j = 0; j < 6; ++j) {
                Wc[j] = OU[j] + OD[j];
                V[j] = Wc[j] + OM[j];
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) h[b] = V[b] + V[b + 2] + Wc[b + 1];
        } else {
#pragma unroll
            for (int b = 0; b < 4; ++b) h[b] = OU[b + 1] + OD[b + 1] + OM[b] + OM[b + 2];
        }
        // ---- table decisions (integer-exact) for histograms with a slot ----
        const uint32_t GX = gword * (uint32_t)L + xmid;  // byte b: g*L + x (<= 24)
        uint32_t outw = 0u, rare = 0u;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint2 sl = *reinterpret_cast<const uint2*>(tab_smem_buf + S.slot + 8 * ((h[b] * hmul) >> hsh));
            rare |= (sl.x != h[b]) ? (1u << b) : 0u;
            const uint32_t off = sl.y + __byte_perm(GX, 0u, 0x4440u + b) * (uint32_t)(4 * TP);
            PCA_DCHECK(!(sl.x == h[b] && ((vmask >> b) & 1u) && act) || off + 4 * TP <= p.tab_bytes - p.tab_thr);
            uint32_t T[4];
            if (TP == 2) {
                const uint2 v = PCA_TAB_THR_GLOBAL ? __ldg(reinterpret_cast<const uint2*>(S.gthr + off))
                                                   : *reinterpret_cast<const uint2*>(tab_smem_buf + S.thr + off);
                T[0] = v.x; T[1] = v.y; T[2] = T[3] = 0u;
            } else {
                const uint4 v = PCA_TAB_THR_GLOBAL ? __ldg(reinterpret_cast<const uint4*>(S.gthr + off))
                                                   : *reinterpret_cast<const uint4*>(tab_smem_buf + S.thr + off);
                T[0] = v.x; T[1] = v.y; T[2] = v.z; T[3] = v.w;
            }
            uint32_t ge = 0;  // #{k : T_k >= r}
#pragma unroll
            for (int k = 0; k < L - 1; ++k)
                asm("{\n\t.reg .u32 d;\n\tsub.cc.u32 d, %1, %2;\n\taddc.u32 %0, %0, 0;\n\t}"
                    : "+r"(ge) : "r"(T[k]), "r"(rr[b]));
            outw |= ((uint32_t)(L - 1) - ge) << (8 * b);
        }
        rare &= act ? vmask : 0u;
        // queued sites: placeholder 0 (the drain stores their labels)
        outw &= ~(((rare * 0x00204081u) & 0x01010101u) * 0xFFu);
        // ---- one record per lane with queued sites (ballot compaction) ----
        {
            const unsigned m = __ballot_sync(FULL, rare != 0u);
            if (rare) {
                PCA_DCHECK(qn + __popc(m & lt) < QCAP);
                uint8_t* rec = tab_smem_buf + S.queue + (qn + __popc(m & lt)) * (uint32_t)sizeof(Rec);
                *reinterpret_cast<uint4*>(rec) = make_uint4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<uint4*>(rec + 16) = rnd;
                *reinterpret_cast<uint4*>(rec + 32) =
                    make_uint4(gword, xmid, ((uint32_t)r << 16) | (uint32_t)c0, rare);
            }
            qn += __popc(m);
        }
        // ---- store x_{t+1} (+ torus pads / row halos, + the peers' halo rows) ----
        if (act) {
            auto store = [&](uint8_t* dst) {
                if (nvalid == 4) *reinterpret_cast<uint32_t*>(dst) = outw;
                else for (int b = 0; b < nvalid; ++b) dst[b] = (uint8_t)(outw >> (8 * b));
                if (G.periodic) {
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
            if (PEERS) {
                if (p.c.peer_up != nullptr && r == 0) store(p.c.peer_up + chain * p.c.peer_up_chain + XOFF + c0);
                if (p.c.peer_dn != nullptr && r == G.rows - 1)
                    store(p.c.peer_dn + chain * p.c.peer_dn_chain + XOFF + c0);
            }
            // ---- fused MPM counts of the table-decided sites (queued ones: at the drain) ----
            if (count_enable) {
                // one reduction per distinct label of the quad's valid table-decided sites (a
                // uniform quad, the common case, is the loop's single iteration: no separate path,
                // so a warp with mixed quads does not run both); byte b of rem/eq: site b
                // (byte b of rem / eq: site b; the uint8 deltas take eq as the increment)
                uint32_t rem = ((vmask & ~rare) * 0x00204081u) & 0x01010101u;
                while (rem) {
                    const uint32_t k = __byte_perm(outw, 0u, 0x4440u + ((__ffs(rem) - 1) >> 3));
                    const uint32_t e = outw ^ (k * 0x01010101u);
                    const uint32_t nz = (((e & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | e) & 0x80808080u;
                    const uint32_t eq = (~nz >> 7) & rem;
                    atomicAdd(reinterpret_cast<unsigned*>(dp + (long long)k * p.tdc_plane), eq);
                    rem &= ~eq;
                }
            }
        }
        if (qn >= 32 || it == iters - 1) {
            if (qn > 0) drain<L, PEERS>(p, S.queue, x_out, chain, count_enable, qn, lane);
            qn = 0;
        }
#pragma unroll
        for (int j = 0; j < 6; ++j) {
            OU[j] = OM[j];
            OM[j] = OD[j];
        }
        xmid = xdn;
        op += G.xpitch;
        dp += G.cpitch;
    }
}

// bytes of the blob a block copies: all of it, or without the threshold rows
__host__ __device__ inline uint32_t tab_smem_blob(const GeneralSweepParams& p) {
    return PCA_TAB_THR_GLOBAL ? p.tab_thr : p.tab_bytes;
}
__host__ __device__ inline int tab_smem(const GeneralSweepParams& p) {
    return 16 + (int)tab_smem_blob(p) + TB_WARPS * QCAP * (int)sizeof(Rec);
}
constexpr int TAB_SMEM_MAX = 16 + TAB_MAX_BYTES + TB_WARPS * QCAP * (int)sizeof(Rec);

// the block's copy of the table blob (one bulk copy) and its warps' queues
__device__ __forceinline__ TabShared tab_setup(const GeneralSweepParams& p) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(tab_smem_buf);
    // programmatic dependent launch (as sweep_packed.cu): the next sweep's blocks may be
    // scheduled once every block of this one is resident; they read the stage's table blob and
    // the previous sweep's output only after the previous grid completed (griddepcontrol.wait)
    if (PCA_TAB_PDL) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_expect_tx(bar, tab_smem_blob(p));
        bulk_g2s(tab_smem_buf + BLOB, p.tab, tab_smem_blob(p), bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    TabShared S;
    S.slot = BLOB + p.tab_slots;
    S.thr = BLOB + p.tab_thr;
    S.queue = BLOB + tab_smem_blob(p) + (threadIdx.x >> 5) * QCAP * (uint32_t)sizeof(Rec);
    S.gthr = p.tab + p.tab_thr;
    return S;
}

template <int NB, int L, bool PEERS>
__global__ void __launch_bounds__(TB_THREADS, PCA_TAB_MINB)
    sweep_table_kernel(const __grid_constant__ GeneralSweepParams p, int R) {
    const TabShared S = tab_setup(p);
    const TDecomp d = tdecomp((p.c.geo.W + 3) >> 2, p.c.rhi - p.c.rlo, R);
    const int qd = blockIdx.x * d.QW + (threadIdx.x & (d.QW - 1));
    const int rbeg = p.c.rlo + (blockIdx.y * d.RS + threadIdx.x / d.QW) * d.R;
    const int rend = min(rbeg + d.R, p.c.rhi);
    tab_rows<NB, L, false, PEERS>(p, S, p.c.x_in, p.c.x_out, p.c.t, p.c.count_enable, qd, blockIdx.z,
                                  rbeg, rend, d.R);
}

template <int NB, int L>
struct TabLaunch {
    static LaunchInfo& get(int smem) {
        static LaunchInfo info[MAX_DEVICES];
        LaunchInfo& li = info[current_device()];
        if (!li.ok.load(std::memory_order_acquire)) {
            std::lock_guard<std::mutex> lock(launch_info_mutex());
            if (!li.ok.load(std::memory_order_relaxed)) {
                int dev = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&li.sms, cudaDevAttrMultiProcessorCount, dev);
                cudaFuncSetAttribute(sweep_table_kernel<NB, L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_SMEM_MAX);
                cudaFuncSetAttribute(sweep_table_kernel<NB, L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TAB_SMEM_MAX);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.occ, sweep_table_kernel<NB, L, false>, TB_THREADS, smem);
                if (li.occ < 1) li.occ = 1;
                li.ok.store(true, std::memory_order_release);
            }
        }
        return li;
    }
};

template <int NB, int L>
int launch_tab(const GeneralSweepParams& p, int batch, int nsweeps, cudaStream_t s) {
    if ((int)p.tab_bytes > TAB_MAX_BYTES) return (int)cudaErrorInvalidValue;
    const int smem = tab_smem(p);
    const LaunchInfo& TL = TabLaunch<NB, L>::get(smem);
    const Geometry& G = p.c.geo;
    const int nquads = (G.W + 3) / 4;
    const int nr = p.c.rhi - p.c.rlo;
    if (nr <= 0) return 0;
    const TDecomp d1 = tdecomp(nquads, nr, 1);
    const long long quadrows = (long long)d1.nxb * d1.QW * nr * batch;
    if (nsweeps > 1) return (int)cudaErrorInvalidValue;  // runs of sweeps: the general kernel's
    const long long target = (long long)PCA_TAB_WAVES * TL.sms * TL.occ * TB_THREADS;
    long long R = (quadrows + target - 1) / target;
    if (R < 1) R = 1;
    TDecomp d = tdecomp(nquads, nr, (int)R);
    while (d.nrb > 65535) d = tdecomp(nquads, nr, d.R * 2);
    dim3 grid((unsigned)d.nxb, (unsigned)d.nrb, batch);
    const bool peers = p.c.peer_up != nullptr || p.c.peer_dn != nullptr;
    if (PCA_TAB_PDL) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(TB_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return (int)(peers ? cudaLaunchKernelEx(&cfg, sweep_table_kernel<NB, L, true>, p, d.R)
                           : cudaLaunchKernelEx(&cfg, sweep_table_kernel<NB, L, false>, p, d.R));
    }
    if (peers)
        sweep_table_kernel<NB, L, true><<<grid, TB_THREADS, smem, s>>>(p, d.R);
    else
        sweep_table_kernel<NB, L, false><<<grid, TB_THREADS, smem, s>>>(p, d.R);
    return (int)cudaGetLastError();
}

}  // namespace

int launch_sweep_table(const GeneralSweepParams& p, int batch, int nsweeps, void* stream) {
    const Geometry& G = p.c.geo;
    cudaStream_t s = (cudaStream_t)stream;
#define PCA_TAB_LAUNCH(LV) \
    return G.nbhd == 8 ? launch_tab<8, LV>(p, batch, nsweeps, s) : launch_tab<4, LV>(p, batch, nsweeps, s)
    switch (G.levels) {
        case 3: PCA_TAB_LAUNCH(3);
        case 4: PCA_TAB_LAUNCH(4);
        case 5: PCA_TAB_LAUNCH(5);
        default: return (int)cudaErrorInvalidValue;
    }
#undef PCA_TAB_LAUNCH
}

}  // namespace pcab200
