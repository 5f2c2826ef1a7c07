// sweep_binary.cu -- one synchronous lazy-PCA sweep for levels == 2 on the byte state (round 1's
// headline kernel; since round 2 the bit-packed kernel, sweep_packed.cu, runs whole lattices and
// strips with W % 512 == 0, and this one the other two-level cases and strips with peers).
//
// Per site i (R1): new label w_i = 0 iff u_i < p_i(0; x), with
//   p_i(0) = e^{E(0)} / (e^{E(0)} + e^{E(1)}),
//   E(s) = a n_i(s) - b (lum g_i - s)^2 - c 1{s != x_i},  n_i(0) = np_i - n_i(1),
// where np_i is the number of lattice neighbours of i (8/4 inside, fewer at a free
// boundary).  p_i(0) depends only on (np, n_i(1), g_i, x_i), so the host
// tabulates the exact integer threshold T = ceil(p0 * 2^32) in fp64 for the current beta
// (324 entries) and the device decision is the integer compare r > T - 1 on the Philox
// word r (u = r 2^-32): bit-exact with the fp64 oracle whenever the host's p0 equals it.
//
// Data movement (Blackwell-native): one warp per CTA owns a 512-column segment (16 sites
// per lane) of a run of R rows and streams it through a private KSTAGES-deep shared-memory
// ring filled by 1-D TMA bulk copies (cp.async.bulk, SASS UBLKCP) that complete on
// per-stage mbarriers.  A stage carries TWO rows: two padded x rows (544 B each, incl. the
// words left/right of the segment) and two g rows (512 B); the two rows of uint16 MPM
// counts (1 KiB each) ride in the stage too on a free boundary, while on a torus each lane
// prefetches its counts into registers one item ahead, which halves the stage and lets 16
// instead of 12 warps share an SM (RingCfg).  The per-stage bookkeeping (wait, refill,
// fence, address arithmetic) is paid once per two rows.  The 4-row neighbourhood window lives in registers; neighbour counts
// are SWAR byte sums (vertical sum of 3 rows, then funnel-shifted left/right sums); the table
// index of each site is one byte of a pre-scaled SWAR word, extracted with one PRMT.  One
// Philox4x32-10 call serves 4 sites.  The MPM count of label 1 (uint16) is updated in the
// same pass (R15) and stored with x_{t+1}.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "tma_ring.cuh"

namespace pcab200 {
namespace {

// Ring depth x resident CTAs x where the MPM counts travel, per boundary kind, measured on
// B200 with tools/tune_variants.py at 8192^2 (us per sweep, MPM on):
//   torus: counts prefetched into registers one item ahead (stage = x + g rows only),
//          4 stages x 14 CTAs/SM: 84.3 (4 x 16: 84.8; counts in the ring, 4 x 12: 86.2;
//          3 x 20: 94.4; 5 x 16: 94.1; 6 x 14: 97.1; 8 x 12: 93.8)
//   free:  counts in the ring, 4 x 12: 90.8 (registers, 4 x 16: 98.7)
#ifndef PCA_T_K
#define PCA_T_K 4
#endif
#ifndef PCA_T_CTAS
#define PCA_T_CTAS 14  // 14 (84.3 us, MPM off 76.1) edged out 16 (85.1, 78.5) and 18 (97.8)
#endif
#ifndef PCA_T_CREG
#define PCA_T_CREG 1
#endif
// PCA_T_RED = 1: torus counts by fire-and-forget 64-bit reductions (no load): measured
// 138 us per sweep (16.8 M RED.64 per sweep saturate the L2 atomic units), so it stays off.
#ifndef PCA_CARRY
#define PCA_CARRY 1  // decisions as borrow bits (sub.cc / addc): 84.5 -> 83.8 us (0 = compare)
#endif
#ifndef PCA_T_RED
#define PCA_T_RED 0
#endif
// Philox products as one wide multiply (philox.cuh) on a torus (8192^2 torus with MPM: 81.9 ->
// 81.35 us per sweep), the split form on a free boundary (as sweep_packed.cu)
#ifndef PCA_B_WIDE
#define PCA_B_WIDE PER
#endif
#ifndef PCA_B_PDL
#define PCA_B_PDL 1  // programmatic dependent launch between consecutive sweeps (kernels.cuh)
#endif
#ifndef PCA_B_WAVES
#define PCA_B_WAVES 4  // waves of resident warps the row runs are sized for (8192^2 torus MPM on, us per
                       // sweep: 1 wave 84.6, 2 84.2, 4 83.5; MPM off 71.7 / 70.6 / 70.9)
#endif
#ifndef PCA_B_PRE
#define PCA_B_PRE 1  // the row-independent Philox prefix in registers (philox.cuh)
#endif
#ifndef PCA_F_K
#define PCA_F_K 4
#endif
#ifndef PCA_F_CTAS
#define PCA_F_CTAS 12
#endif
#ifndef PCA_F_CREG
#define PCA_F_CREG 0
#endif
// 16-site chunks per warp segment (one per lane).  Two chunks per lane (1024-column segments,
// halving the per-row bookkeeping per site) measured 114.6 us per sweep at best (4 x 12):
// the doubled register window cut occupancy more than it saved.
constexpr int SEG_CHUNKS = 32;
constexpr int XROW_BYTES = 16 * SEG_CHUNKS + 32;       // 544: [col0-16, col0+528)
constexpr int GROW_BYTES = 16 * SEG_CHUNKS;            // 512
constexpr int CROW_BYTES = 32 * SEG_CHUNKS;            // 1024
constexpr int XOFS = 0, GOFS = 2 * XROW_BYTES, COFS = GOFS + 2 * GROW_BYTES;

template <bool PER>
struct RingCfg {
    static constexpr int K = PER ? PCA_T_K : PCA_F_K;           // ring depth (2 rows per stage)
    static constexpr int CTAS = PER ? PCA_T_CTAS : PCA_F_CTAS;  // resident one-warp CTAs per SM
    static constexpr bool RED = PER ? PCA_T_RED : 0;              // counts via reductions
    static constexpr bool CREG = !RED && (PER ? PCA_T_CREG : PCA_F_CREG); // counts via registers
    static constexpr int STAGE = COFS + ((CREG || RED) ? 0 : 2 * CROW_BYTES);  // 2112 or 4160
    static constexpr int RING_OFF = ((K + 1) * 8 + 63) / 64 * 64;    // mbarriers, then the ring
    static constexpr int SMEM = RING_OFF + K * STAGE;                // dynamic smem per CTA
    static_assert(K + 1 <= RING_OFF / 8, "mbarrier slots");
};
static_assert(THR_ENTRIES * 4 % 16 == 0, "bulk copy size");

// Map label bytes to {0,1}: 0 -> 0, 1 -> 1, free-boundary sentinel 0xFF -> 0.
__device__ __forceinline__ uint32_t to01(uint32_t w) { return w & ~(w >> 1) & 0x01010101u; }

template <int NB>
__device__ __forceinline__ int neighbours_present(int grow, int H, int c, int W) {
    const int er = (grow == 0) + (grow == H - 1);
    const int ec = (c == 0) + (c == W - 1);
    return NB == 8 ? (3 - er) * (3 - ec) - 1 : 4 - er - ec;
}

struct XRow {
    uint32_t w[4];  // the lane's 16 labels
    uint32_t l, r;  // the words left / right of the chunk
};

// One warp per CTA: every per-warp quantity (segment, row range, stage addresses) derives
// from blockIdx and kernel parameters only, so the compiler keeps it in uniform registers and
// the bulk-copy issue needs no per-lane address handling.
// F: compile-time launch flags.  This kernel's schedule is sensitive to code it never runs:
// two never-taken peer-pointer tests cost 3.5 us per 8192^2 sweep, and making the counting
// or the torus self-halo compile-time in the counting variant cost 2 (torus) to 7.5 (free
// boundary) us through a different register allocation, so only the peer stores and the
// no-counting variant (76.1 -> 73.9 us) are separate instantiations.
constexpr int BF_PEERS = 1;    // edge rows also stored into the peers' halo rows
constexpr int BF_NOCOUNT = 2;  // no MPM counting in this sweep
template <int NB, bool PER, int F>
__global__ void __launch_bounds__(32, RingCfg<PER>::CTAS)
    sweep_binary_kernel(const __grid_constant__ BinarySweepParams p, int R) {
    constexpr bool PEERS = (F & BF_PEERS) != 0;
    constexpr bool NOCOUNT = (F & BF_NOCOUNT) != 0;
    using C = RingCfg<PER>;
    constexpr int KSTAGES = C::K;
    constexpr int STAGE_BYTES = C::STAGE;
    constexpr bool CREG = C::CREG;  // counts prefetched into registers (no ring slot)
    constexpr bool RED = C::RED;    // counts added by reductions (no ring slot, no load)
    __shared__ __align__(16) uint32_t s_thr[THR_ENTRIES];  // static: LDS [reg + imm]
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    uint8_t* ring = smem + C::RING_OFF;
    const int lane = threadIdx.x;
    if (PCA_B_PDL) pdl_begin();
    if (lane == 0) {
        for (int s = 0; s <= KSTAGES; ++s) mbar_init(&bars[s], 1);  // bars[KSTAGES]: the table
        fence_mbar_init();
    }
    __syncwarp();

    const Geometry& G = p.c.geo;
    const int seg = blockIdx.x;
    const int chain = blockIdx.z;
    const int rbeg = p.c.rlo + blockIdx.y * R;
    const int rend = min(rbeg + R, p.c.rhi);
    if (rbeg >= rend) return;
    // item i carries x rows rbeg-1+2i, rbeg+2i and g / count rows rbeg+2i-2, rbeg+2i-1
    const int nitems = (rend - rbeg + 3) >> 1;
    const int nch = min(SEG_CHUNKS, G.nchunks - seg * SEG_CHUNKS);
    const int col0 = 16 * SEG_CHUNKS * seg;
    const int k = seg * SEG_CHUNKS + lane;  // this lane's chunk
    const bool active = lane < nch;
    const int ccol = col0 + 16 * lane;      // first column of the chunk
    const uint32_t xbytes = 16 * nch + 32, gbytes = 16 * nch;
    const uint32_t cbytes = (!NOCOUNT && p.c.count_enable) ? 32 * nch : 0;
    // padded x row j starts at (j+HALO)*xpitch; byte col0 of it is column col0-16; xin points
    // at x row rbeg-1 (item 0)
    const uint8_t* xin = p.c.x_in + chain * G.xchain + col0 + (long long)(rbeg - 1 + HALO) * G.xpitch;
    const uint8_t* gin = p.c.g + chain * G.gchain + XOFF + col0 + (long long)(rbeg + GHALO) * G.gpitch;
    const uint16_t* cin = p.c.counts + chain * G.cchain + col0 + (long long)rbeg * G.cpitch;
    uint8_t* xo = p.c.x_out + chain * G.xchain + (long long)(rbeg + HALO) * G.xpitch;  // row rbeg
    uint16_t* co = p.c.counts + chain * G.cchain + ccol + (long long)rbeg * G.cpitch;
    const uint32_t tagchain = (TAG_PCA << 24) | (p.c.chain0 + (uint32_t)chain);
    const uint8_t* thr_b = reinterpret_cast<const uint8_t*>(s_thr);
    // the lane's 4 Philox counters (4k+i, row, t, tagchain): rounds 0..2 minus the row, once
    // (philox.cuh philox_pre / philox_row: 34 instead of 40 instructions per call)
    PhiloxPre ppre[4];
    if (PCA_B_PRE) {
#pragma unroll
        for (int i = 0; i < 4; ++i) ppre[i] = philox_pre((uint32_t)(4 * k + i), p.c.t, tagchain, p.c.keys);
    }
    // CREG: the count rows of the next two updated rows, loaded one item ahead
    uint4 CR[2][2];
    auto load_counts = [&](int rfirst) {
        if (!CREG || !cbytes || !active) return;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (rfirst + q < rend) {
                const uint4* src = reinterpret_cast<const uint4*>(co + (long long)(rfirst + q - rbeg) * G.cpitch);
                CR[q][0] = __ldcs(src);
                CR[q][1] = __ldcs(src + 1);
            }
        }
    };

    // elected lane: load item `it` into stage s (rows past the run are skipped)
    auto issue = [&](int it, int s) {
        uint8_t* st = ring + s * STAGE_BYTES;
        const int jx = 2 * it;             // x row rbeg-1+jx relative to xin
        const int nx = (rbeg - 1 + jx + 1 <= rend) ? 2 : 1;
        const int jr = 2 * it - 2;         // g / count row rbeg+jr
        const int nr = it == 0 ? 0 : min(2, rend - rbeg - jr);
        PCA_DCHECK(nx * XROW_BYTES + nr * (GROW_BYTES + ((CREG || RED) ? 0 : CROW_BYTES)) <= STAGE_BYTES);
        PCA_DCHECK(rbeg - 1 + jx >= -HALO && rbeg - 1 + jx + nx - 1 < G.rows + HALO);
        mbar_expect_tx(&bars[s], nx * xbytes + nr * (gbytes + ((CREG || RED) ? 0u : cbytes)));
        for (int q = 0; q < nx; ++q)
            bulk_g2s(st + XOFS + q * XROW_BYTES, xin + (long long)(jx + q) * G.xpitch, xbytes, &bars[s]);
        for (int q = 0; q < nr; ++q) {
            bulk_g2s(st + GOFS + q * GROW_BYTES, gin + (long long)(jr + q) * G.gpitch, gbytes, &bars[s]);
            if (!CREG && !RED && cbytes)
                bulk_g2s(st + COFS + q * CROW_BYTES, cin + (long long)(jr + q) * G.cpitch, cbytes,
                         &bars[s]);
        }
    };
    if (elect_one()) {
        mbar_expect_tx(&bars[KSTAGES], THR_ENTRIES * 4);
        bulk_g2s(s_thr, p.thr, THR_ENTRIES * 4, &bars[KSTAGES]);
        for (int it = 0; it < min(KSTAGES, nitems); ++it) issue(it, it);
    }
    mbar_wait(&bars[KSTAGES], 0);

    auto read_x = [&](const uint8_t* st, int q, XRow& x) {
        const uint8_t* xr = st + XOFS + q * XROW_BYTES;
        const uint4 xv = *reinterpret_cast<const uint4*>(xr + 16 + 16 * lane);
        x.l = *reinterpret_cast<const uint32_t*>(xr + 12 + 16 * lane);
        x.r = *reinterpret_cast<const uint32_t*>(xr + 32 + 16 * lane);
        x.w[0] = xv.x; x.w[1] = xv.y; x.w[2] = xv.z; x.w[3] = xv.w;
        if (!PER) {
#pragma unroll
            for (int i = 0; i < 4; ++i) x.w[i] = to01(x.w[i]);
            x.l = to01(x.l);
            x.r = to01(x.r);
        }
    };

    // device-initiated halo exchange: the edge rows also go straight into the neighbouring
    // ranks' halo rows (peer memory over NVLink), written by the lanes that computed them
    auto store_peer_rows = [&](int r, const uint32_t (&O)[4]) {
        if (!PEERS) return;
        if (p.c.peer_up != nullptr && r == 0)
            store_row_chunk<HALO, XOFF>(p.c.peer_up + chain * p.c.peer_up_chain, O, ccol, G.W - ccol, k, r,
                                        G.W, G.nchunks, G.rows, G.xpitch, PER, false);
        if (p.c.peer_dn != nullptr && r == G.rows - 1)
            store_row_chunk<HALO, XOFF>(p.c.peer_dn + chain * p.c.peer_dn_chain, O, ccol, G.W - ccol, k, r,
                                        G.W, G.nchunks, G.rows, G.xpitch, PER, false);
    };

    // update local row r from the window (U = row r-1, M = row r, D = row r+1); its g row
    // and counts row are slot q of stage st
    auto update = [&](int r, const uint8_t* st, int q, const XRow& U, const XRow& M, const XRow& D) {
        const int grow = G.row0 + r;
        const uint4 gv = *reinterpret_cast<const uint4*>(st + GOFS + q * GROW_BYTES + 16 * lane);
        // ---- n_i(1): SWAR neighbour counts, one byte per site ----
        uint32_t S[4];
        if (NB == 8) {
            uint32_t V[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) V[i] = U.w[i] + M.w[i] + D.w[i];
            const uint32_t VL = U.l + M.l + D.l, VR = U.r + M.r + D.r;
            S[0] = from_left(VL, V[0]) + V[0] + from_right(V[0], V[1]) - M.w[0];
            S[1] = from_left(V[0], V[1]) + V[1] + from_right(V[1], V[2]) - M.w[1];
            S[2] = from_left(V[1], V[2]) + V[2] + from_right(V[2], V[3]) - M.w[2];
            S[3] = from_left(V[2], V[3]) + V[3] + from_right(V[3], VR) - M.w[3];
        } else {
            S[0] = U.w[0] + D.w[0] + from_left(M.l, M.w[0]) + from_right(M.w[0], M.w[1]);
            S[1] = U.w[1] + D.w[1] + from_left(M.w[0], M.w[1]) + from_right(M.w[1], M.w[2]);
            S[2] = U.w[2] + D.w[2] + from_left(M.w[1], M.w[2]) + from_right(M.w[2], M.w[3]);
            S[3] = U.w[3] + D.w[3] + from_left(M.w[2], M.w[3]) + from_right(M.w[3], M.r);
        }
        // byte offset into the threshold table: 4 * (n1*4 + g*2 + x) <= 140, one byte per site
        const uint32_t Gw[4] = {gv.x, gv.y, gv.z, gv.w};
        uint32_t IDX4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) IDX4[i] = (S[i] << 4) | (Gw[i] << 3) | (M.w[i] << 2);
        const bool edge = !PER && (k == 0 || k == G.nchunks - 1 || grow == 0 || grow == G.H - 1);

        // ---- Philox (one call per 4 sites) + integer-threshold decisions ----
        uint32_t O[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 rnd = PCA_B_PRE ? philox_row<PCA_B_WIDE>(ppre[i], (uint32_t)grow, p.c.keys)
                                        : philox4x32_10(make_uint4((uint32_t)(4 * k + i), (uint32_t)grow, p.c.t,
                                                                   tagchain), p.c.keys);
            const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
            // sub.cc sets the carry of T + ~r + 1, i.e. T >= r: the complement of the decision
            // w = (r > T); shifted into a 4-bit word (site b -> bit b, sites taken 3..0)
            uint32_t bits = 0u;
#pragma unroll
            for (int b = 3; b >= 0; --b) {
                uint32_t off = __byte_perm(IDX4[i], 0u, 0x4440 + b);
                if (PER) {
                    off += NB * 36 * 4;
                } else {
                    const int np = edge ? neighbours_present<NB>(grow, G.H, ccol + 4 * i + b, G.W) : NB;
                    off += (uint32_t)np * 144u;
                }
                const uint32_t T = *reinterpret_cast<const uint32_t*>(thr_b + off);
                uint32_t dummy;
                asm("sub.cc.u32 %1, %2, %3;\n\taddc.u32 %0, %0, %0;"
                    : "+r"(bits), "=r"(dummy)
                    : "r"(T), "r"(rw[b]));
            }
            O[i] = ((~bits & 0xFu) * 0x00204081u) & 0x01010101u;  // bit b -> byte b
        }
        // ---- fused MPM counts of label 1 (uint16 per site) ----
        if (cbytes) {
            uint4 c0, c1;
            if (CREG) {
                c0 = CR[q][0];
                c1 = CR[q][1];
            } else {
                const uint4* cs = reinterpret_cast<const uint4*>(st + COFS + q * CROW_BYTES + 32 * lane);
                c0 = cs[0];
                c1 = cs[1];
            }
            c0.x += __byte_perm(O[0], 0u, 0x4140); c0.y += __byte_perm(O[0], 0u, 0x4342);
            c0.z += __byte_perm(O[1], 0u, 0x4140); c0.w += __byte_perm(O[1], 0u, 0x4342);
            c1.x += __byte_perm(O[2], 0u, 0x4140); c1.y += __byte_perm(O[2], 0u, 0x4342);
            c1.z += __byte_perm(O[3], 0u, 0x4140); c1.w += __byte_perm(O[3], 0u, 0x4342);
            uint4* cp = reinterpret_cast<uint4*>(co + (long long)(r - rbeg) * G.cpitch);
            cp[0] = c0;
            cp[1] = c1;
        }
        // ---- store x_{t+1} (+ torus halos, + the peers' halo rows) ----
        store_row_chunk<HALO, XOFF>(xo + (long long)(r - rbeg) * G.xpitch, O, ccol, G.W - ccol, k, r,
                                    G.W, G.nchunks, G.rows, G.xpitch, PER, G.self_halo_rows);
        store_peer_rows(r, O);
    };

    // Torus: update local rows r0 and (when nrow == 2) r0+1 together from the window rows
    // x rows r0-1 .. r0+2; their g rows and count rows are slots 0, 1 of stage st.  Both
    // rows' table indices are formed first and their 8 Philox calls are independent, so the
    // dependent IMAD/LOP3 chains of the rounds interleave (instruction-level parallelism is
    // what the one-warp CTAs lack): 2.7% (MPM on) / 3.6% (MPM off) faster at 8192^2.  The
    // free boundary keeps the row-by-row `update` (its edge logic made the joint form 4-6%
    // slower).
    auto update2 = [&](int r0, int nrow, const uint8_t* st, const XRow& X0, const XRow& X1,
                       const XRow& X2, const XRow& X3) {
        const XRow* Wn[4] = {&X0, &X1, &X2, &X3};
        uint32_t IDX4[2][4];
        bool edge[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const XRow& U = *Wn[q];
            const XRow& M = *Wn[q + 1];
            const XRow& D = *Wn[q + 2];
            const int grow = G.row0 + r0 + q;
            const uint4 gv = *reinterpret_cast<const uint4*>(st + GOFS + q * GROW_BYTES + 16 * lane);
            // ---- n_i(1): SWAR neighbour counts, one byte per site ----
            uint32_t S[4];
            if (NB == 8) {
                uint32_t V[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) V[i] = U.w[i] + M.w[i] + D.w[i];
                const uint32_t VL = U.l + M.l + D.l, VR = U.r + M.r + D.r;
                S[0] = from_left(VL, V[0]) + V[0] + from_right(V[0], V[1]) - M.w[0];
                S[1] = from_left(V[0], V[1]) + V[1] + from_right(V[1], V[2]) - M.w[1];
                S[2] = from_left(V[1], V[2]) + V[2] + from_right(V[2], V[3]) - M.w[2];
                S[3] = from_left(V[2], V[3]) + V[3] + from_right(V[3], VR) - M.w[3];
            } else {
                S[0] = U.w[0] + D.w[0] + from_left(M.l, M.w[0]) + from_right(M.w[0], M.w[1]);
                S[1] = U.w[1] + D.w[1] + from_left(M.w[0], M.w[1]) + from_right(M.w[1], M.w[2]);
                S[2] = U.w[2] + D.w[2] + from_left(M.w[1], M.w[2]) + from_right(M.w[2], M.w[3]);
                S[3] = U.w[3] + D.w[3] + from_left(M.w[2], M.w[3]) + from_right(M.w[3], M.r);
            }
            // byte offset into the threshold table: 4 * (n1*4 + g*2 + x) <= 140, one byte per site
            const uint32_t Gw[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) IDX4[q][i] = (S[i] << 4) | (Gw[i] << 3) | (M.w[i] << 2);
            edge[q] = !PER && (k == 0 || k == G.nchunks - 1 || grow == 0 || grow == G.H - 1);
        }
        if (nrow < 2) {  // row r0+1 is past the run: its stage slot holds stale bytes, whose
#pragma unroll           // table offsets could be misaligned; decide on index 0 and discard
            for (int i = 0; i < 4; ++i) IDX4[1][i] = 0u;
        }

        // ---- Philox (one call per 4 sites) + integer-threshold decisions ----
        uint32_t O[2][4];
        auto decide = [&](int q, int i) {
            const int grow = G.row0 + r0 + q;
            const uint4 rnd = PCA_B_PRE ? philox_row<PCA_B_WIDE>(ppre[i], (uint32_t)grow, p.c.keys)
                                        : philox4x32_10(make_uint4((uint32_t)(4 * k + i), (uint32_t)grow, p.c.t,
                                                                   tagchain), p.c.keys);
            const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
#if PCA_CARRY
            // sub.cc sets the carry of T + ~r + 1, i.e. T >= r: the complement of the decision
            // w = (r > T); shifted into a 4-bit word (site b -> bit b, sites taken 3..0), then
            // complemented and spread to bytes
            uint32_t bits = 0u;
#pragma unroll
            for (int b = 3; b >= 0; --b) {
                uint32_t off = __byte_perm(IDX4[q][i], 0u, 0x4440 + b);
                if (PER) {
                    off += NB * 36 * 4;
                } else {
                    const int np = edge[q] ? neighbours_present<NB>(grow, G.H, ccol + 4 * i + b, G.W) : NB;
                    off += (uint32_t)np * 144u;
                }
                const uint32_t T = *reinterpret_cast<const uint32_t*>(thr_b + off);
                uint32_t dummy;
                asm("sub.cc.u32 %1, %2, %3;\n\taddc.u32 %0, %0, %0;"
                    : "+r"(bits), "=r"(dummy)
                    : "r"(T), "r"(rw[b]));
            }
            O[q][i] = ((~bits & 0xFu) * 0x00204081u) & 0x01010101u;
#else
            uint32_t o = 0u;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                uint32_t off = __byte_perm(IDX4[q][i], 0u, 0x4440 + b);
                if (PER) {
                    off += NB * 36 * 4;
                } else {
                    const int np = edge[q] ? neighbours_present<NB>(grow, G.H, ccol + 4 * i + b, G.W) : NB;
                    off += (uint32_t)np * 144u;
                }
                const uint32_t T = *reinterpret_cast<const uint32_t*>(thr_b + off);
                if (rw[b] > T) o += 1u << (8 * b);
            }
            O[q][i] = o;
#endif
        };
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int q = 0; q < 2; ++q) decide(q, i);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (q == 1 && nrow < 2) break;
            const int r = r0 + q;
            // ---- fused MPM counts of label 1 (uint16 per site) ----
            if (cbytes && RED) {
                unsigned long long* cp =
                    reinterpret_cast<unsigned long long*>(co + (long long)(r - rbeg) * G.cpitch);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const unsigned long long inc =
                        (unsigned long long)__byte_perm(O[q][i], 0u, 0x4140) |
                        ((unsigned long long)__byte_perm(O[q][i], 0u, 0x4342) << 32);
                    atomicAdd(cp + i, inc);
                }
            } else if (cbytes) {
                uint4 c0, c1;
                if (CREG) {
                    c0 = CR[q][0];
                    c1 = CR[q][1];
                } else {
                    const uint4* cs = reinterpret_cast<const uint4*>(st + COFS + q * CROW_BYTES + 32 * lane);
                    c0 = cs[0];
                    c1 = cs[1];
                }
                c0.x += __byte_perm(O[q][0], 0u, 0x4140); c0.y += __byte_perm(O[q][0], 0u, 0x4342);
                c0.z += __byte_perm(O[q][1], 0u, 0x4140); c0.w += __byte_perm(O[q][1], 0u, 0x4342);
                c1.x += __byte_perm(O[q][2], 0u, 0x4140); c1.y += __byte_perm(O[q][2], 0u, 0x4342);
                c1.z += __byte_perm(O[q][3], 0u, 0x4140); c1.w += __byte_perm(O[q][3], 0u, 0x4342);
                uint4* cp = reinterpret_cast<uint4*>(co + (long long)(r - rbeg) * G.cpitch);
                cp[0] = c0;
                cp[1] = c1;
            }
            // ---- store x_{t+1} (+ torus halos, + the peers' halo rows) ----
            store_row_chunk<HALO, XOFF>(xo + (long long)(r - rbeg) * G.xpitch, O[q], ccol, G.W - ccol, k,
                                        r, G.W, G.nchunks, G.rows, G.xpitch, PER, G.self_halo_rows);
            store_peer_rows(r, O[q]);
        }
    };

    // window: A0 = x row r0-1, A1 = x row r0 (previous item), B0 = r0+1, B1 = r0+2 (current)
    XRow A0, A1, B0, B1;
    load_counts(rbeg);
    int s = 0;
    uint32_t phase = 0;
    for (int it = 0; it < nitems; ++it) {
        mbar_wait(&bars[s], phase);
        const uint8_t* st = ring + s * STAGE_BYTES;
        if (active) {
            read_x(st, 0, B0);
            read_x(st, 1, B1);  // (stale data when past the run: then never used)
            if (it > 0) {
                const int r0 = rbeg + 2 * it - 2;
                if (PER) {
                    update2(r0, r0 + 1 < rend ? 2 : 1, st, A0, A1, B0, B1);
                } else {
                    update(r0, st, 0, A0, A1, B0);
                    if (r0 + 1 < rend) update(r0 + 1, st, 1, A1, B0, B1);
                }
                load_counts(r0 + 2);
            }
        }
        // every lane is done with this stage: refill it with item it + KSTAGES
        __syncwarp();
        if (it + KSTAGES < nitems && elect_one()) {
            fence_proxy_async();
            issue(it + KSTAGES, s);
        }
        A0 = B0;
        A1 = B1;
        if (++s == KSTAGES) {
            s = 0;
            phase ^= 1u;
        }
    }
}

template <int NB, bool PER, int F>
int launch_t(const BinarySweepParams& p, int batch, int R, cudaStream_t s) {
    const Geometry& G = p.c.geo;
    static LaunchInfo info[MAX_DEVICES];
    LaunchInfo& li = info[current_device()];
    if (!li.ok.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lock(launch_info_mutex());
        if (!li.ok.load(std::memory_order_relaxed)) {
            cudaError_t e = cudaFuncSetAttribute(sweep_binary_kernel<NB, PER, F>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, RingCfg<PER>::SMEM);
            if (e != cudaSuccess) return (int)e;
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&li.sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.occ, sweep_binary_kernel<NB, PER, F>, 32,
                                                          RingCfg<PER>::SMEM);
            if (li.occ < 1) li.occ = 1;
            li.ok.store(true, std::memory_order_release);
        }
    }
    const int occ = li.occ, sms = li.sms;
    if (R <= 0) {
        // size R so the grid is PCA_B_WAVES waves of resident warps: every warp walks one
        // contiguous run of rows with its pipeline primed once (several waves balance the tail)
        const long long segs = (G.nchunks + SEG_CHUNKS - 1) / SEG_CHUNKS;
        const long long target = (long long)sms * occ * PCA_B_WAVES;
        const long long work = (long long)(p.c.rhi - p.c.rlo) * segs * batch;
        R = (int)((work + target - 1) / target);
        if (R < 2) R = 2;
    }
    const int nrb = (p.c.rhi - p.c.rlo + R - 1) / R;
    if (nrb <= 0) return 0;
    if (nrb > 65535) return (int)cudaErrorInvalidConfiguration;
    dim3 grid((G.nchunks + SEG_CHUNKS - 1) / SEG_CHUNKS, nrb, batch);
    if (PCA_B_PDL) return (int)launch_pdl(sweep_binary_kernel<NB, PER, F>, grid, dim3(32), RingCfg<PER>::SMEM, s, p, R);
    sweep_binary_kernel<NB, PER, F><<<grid, 32, RingCfg<PER>::SMEM, s>>>(p, R);
    return (int)cudaGetLastError();
}

template <int NB, bool PER>
int launch_f(const BinarySweepParams& p, int batch, int R, cudaStream_t s) {
    const bool peers = p.c.peer_up != nullptr || p.c.peer_dn != nullptr;
    const int f = (peers ? BF_PEERS : 0) | (p.c.count_enable ? 0 : BF_NOCOUNT);
    switch (f) {
        case 0: return launch_t<NB, PER, 0>(p, batch, R, s);
        case 1: return launch_t<NB, PER, 1>(p, batch, R, s);
        case 2: return launch_t<NB, PER, 2>(p, batch, R, s);
        default: return launch_t<NB, PER, 3>(p, batch, R, s);
    }
}

}  // namespace

int launch_sweep_binary(const BinarySweepParams& p, int batch, int rows_per_thread, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int R = rows_per_thread;  // 0 = auto (PCA_B_WAVES waves)
    if (p.c.geo.nbhd == 8)
        return p.c.geo.periodic ? launch_f<8, true>(p, batch, R, s) : launch_f<8, false>(p, batch, R, s);
    return p.c.geo.periodic ? launch_f<4, true>(p, batch, R, s) : launch_f<4, false>(p, batch, R, s);
}

}  // namespace pcab200
