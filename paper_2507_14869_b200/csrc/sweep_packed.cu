// sweep_packed.cu -- the two-level sweep on bit-packed multi-spin state (north star (2):
// "bit-packed multi-spin words for the binary case").
//
// The state x_t, x_{t+1} and the observation g live in HBM at ONE BIT per site (32 sites per
// 32-bit word, column c at bit c % 8 of byte c / 8 of its row, LSB first), so a sweep moves
// 3 bits of state per site-update instead of 3 bytes (plus the uint8 MPM count-delta read-
// modify-write when counting, below): 2.375 B/SU with MPM counts, 0.375 B/SU without.
//
// The chain is the byte kernel's (sweep_binary.cu) bit for bit: the same Philox words
// (counter (col >> 2, row, t, tag << 24 | chain)), the same host-tabulated integer thresholds
// T[(np, n1, g, x)] = ceil(p0 2^32) - 1 of PAPER.md:462-477, the same decision w = (r > T).
// Per lane and row the 16 packed bits (+ the columns left and right) are expanded to SWAR
// bytes (two lookups in a 256-entry shared table) and the byte kernel's neighbour sums and table lookups run
// unchanged; the decisions are packed back to 16 bits.  A spin-level bit-sliced evaluation was
// not used: the exact per-site law needs the 32-bit uniform and a table row per site, so
// bit-slicing the neighbour counts saves little and the bits -> table-index transposition costs
// more than it saves.
//
// Layout (one context, a whole lattice or a row strip, W % 512 == 0): xp[2]: uint8
// [batch][rows + 2 HALO][pp],
// pp = W/8 + 32: packed row j at (j + HALO) pp, column c at bit c%8 of byte 16 + c/8; bytes
// [0, 16) / [16 + W/8, pp) are the column pads (on a torus the lane owning columns W-16..W-1
// also writes them to bytes 14..15 and the lane owning 0..15 to bytes W/8+16..+17, the only pad
// bits any lane reads; zero on a free boundary).  Halo rows: wrapped rows rewritten by every
// sweep on a torus, zero on a free boundary, the neighbours' packed rows on a strip (the
// runtime's NCCL exchange, or the caller's).  gp: uint8 [batch][rows][W/8].
//
// Launch shape: row runs sized for 4 waves of resident CTAs, programmatic dependent launch
// between consecutive sweeps.
//
// Data movement: one warp per CTA owns a 512-column segment of a run of rows; rows stream
// through a 4-stage shared-memory ring of TMA bulk copies (96 B of packed x and 64 B of packed
// g per row, two rows per stage: 320 B against the byte kernel's 2112 B); each lane prefetches
// its 16 B of uint8 count deltas per row into registers one item ahead.
//
// MPM counts: the kernel adds each sweep's labels into a uint8 delta plane (one byte-wise add
// per 4 sites, 2 B/SU of read-modify-write instead of the uint16 plane's 4 B/SU); the runtime
// folds the deltas into the canonical uint16 counts (fold_counts_kernel) before 255 counted
// sweeps accumulate and at the end of every run of sweeps, so every other reader sees the
// usual counts.  Per site-update the kernel moves 3/8 B of state + 2 B of counts.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "tma_ring.cuh"

namespace pcab200 {
namespace {

#ifndef PCA_P_K
#define PCA_P_K 4
#endif
#ifndef PCA_P_CTAS
#define PCA_P_CTAS 16
#endif
#ifndef PCA_P_QN
#define PCA_P_QN 1  // rows updated together (2: their Philox chains interleaved, more registers)
#endif
#ifndef PCA_P_PRE
// 1: the row-independent Philox prefix of the lane's 4 counters kept in registers (philox.cuh
// philox_pre / philox_row: 34 instead of 40 instructions per call).  Measured with 50-sweep
// calls, torus MPM on / off / free boundary, us per sweep: prefix + 1 row per update + 16 CTAs
// 74.3 / 68.9 / 82.4; prefix + 2 joint rows + 14 CTAs 74.3 / 67.1 / 88.6; no prefix + 2 joint
// rows + 14 CTAs (round-2 first version) 76.3 / 70.7 / 82.4
#define PCA_P_PRE 1
#endif
#ifndef PCA_P_LUT
#define PCA_P_LUT 1  // a row's 16 bits to label bytes by two 256-entry shared-memory lookups
#endif
#ifndef PCA_P_LUT_G
#define PCA_P_LUT_G 1  // g's bits by the same table
#endif
#ifndef PCA_P_LUT_O
#define PCA_P_LUT_O 0  // the new labels' count increments by the same table (measured slower)
#endif
// Philox products as one wide multiply (philox.cuh) on a torus; the split form on a free
// boundary (us per direct 8192^2 sweep, wide / split: torus 65.4 / 66.4, strip shape 124.6 /
// 126.8, free boundary 75.8 / 75.0)
#ifndef PCA_P_WIDE
#define PCA_P_WIDE PER
#endif
#ifndef PCA_P_PDL
#define PCA_P_PDL 1  // programmatic dependent launch between consecutive sweep launches
#endif
#ifndef PCA_P_WAVES
#define PCA_P_WAVES 4  // waves of resident CTAs the row runs are sized for
#endif
constexpr int P_XROW = 96;                  // packed x bytes staged per row: cols [c0-128, c0+640)
constexpr int P_GROW = 64;                  // packed g bytes per row: cols [c0, c0+512)
constexpr int P_STAGE = 2 * P_XROW + 2 * P_GROW;  // 320
constexpr int P_GOFS = 2 * P_XROW;
constexpr int P_RING_OFF = ((PCA_P_K + 1) * 8 + 63) / 64 * 64;
constexpr int P_SMEM = P_RING_OFF + PCA_P_K * P_STAGE;

// 4 sites' 0/1 bits (nibble n) -> 4 label bytes
__device__ __forceinline__ uint32_t spread4(uint32_t n) { return (n * 0x00204081u) & 0x01010101u; }

template <int NB>
__device__ __forceinline__ int p_neighbours_present(int grow, int H, int c, int W) {
    const int er = (grow == 0) + (grow == H - 1);
    const int ec = (c == 0) + (c == W - 1);
    return NB == 8 ? (3 - er) * (3 - ec) - 1 : 4 - er - ec;
}

struct PRow {
    uint32_t w[4];  // the lane's 16 labels as bytes
    uint32_t l, r;  // byte 3 of l: column c0 - 1; byte 0 of r: column c0 + 16
};

template <int NB, bool PER, bool NOCOUNT>
__global__ void __launch_bounds__(32, PCA_P_CTAS)
    sweep_packed_kernel(const __grid_constant__ PackedSweepParams p, int R) {
    __shared__ __align__(16) uint32_t s_thr[THR_ENTRIES];
    // byte -> its 8 bits as 8 label bytes (two words), filled once per CTA (PCA_P_LUT)
    __shared__ __align__(16) uint2 s_spread[PCA_P_LUT ? 256 : 1];
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    uint8_t* ring = smem + P_RING_OFF;
    const int lane = threadIdx.x;
    // programmatic dependent launch: the next sweep's CTAs may be scheduled as soon as every CTA
    // of this one is resident (they set up, then wait for this grid to complete: griddepcontrol.
    // wait returns when the prerequisite grid has completed and its memory is visible)
    if (PCA_P_PDL) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (lane == 0) {
        for (int s = 0; s <= PCA_P_K; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    if (PCA_P_LUT)
        for (int v = lane; v < 256; v += 32) s_spread[v] = make_uint2(spread4(v & 0xFu), spread4(v >> 4));
    __syncwarp();
    const Geometry& G = p.c.geo;
    const int seg = blockIdx.x;
    const int chain = blockIdx.z;
    const int rbeg = p.c.rlo + blockIdx.y * R;
    const int rend = min(rbeg + R, p.c.rhi);
    if (rbeg >= rend) return;
    const int nitems = (rend - rbeg + 3) >> 1;  // item i: x rows rbeg-1+2i, rbeg+2i; g rows rbeg+2i-2, +1
    const int col0 = 512 * seg;
    const int ccol = col0 + 16 * lane;
    const int k = seg * 32 + lane;  // 16-site chunk index
    const int nchunks = G.W >> 4;
    const bool cnt = !NOCOUNT && p.c.count_enable;
    const uint8_t* xin = p.x_in + chain * p.xchain + 64 * seg + (long long)(rbeg - 1 + HALO) * p.pp;
    const uint8_t* gin = p.g + chain * p.gchain + 64 * seg + (long long)rbeg * p.gpp;
    uint8_t* xo = p.x_out + chain * p.xchain + (long long)(rbeg + HALO) * p.pp + 16 + 2 * (ccol >> 4);
    // MPM counts of label 1: uint8 deltas [batch][rows][cpitch] (folded into the uint16 counts
    // by the runtime at most every 255 counted sweeps and at the end of every run)
    uint8_t* co = p.dcounts + chain * p.dchain + ccol + (long long)rbeg * G.cpitch;
    const uint32_t tagchain = (TAG_PCA << 24) | (p.c.chain0 + (uint32_t)chain);
    const uint8_t* thr_b = reinterpret_cast<const uint8_t*>(s_thr);
    // the lane's 4 Philox counters (4k+i, row, t, tagchain): rounds 0..2 minus the row, once
    PhiloxPre ppre[4];
    if (PCA_P_PRE) {
#pragma unroll
        for (int i = 0; i < 4; ++i) ppre[i] = philox_pre((uint32_t)(4 * k + i), p.c.t, tagchain, p.c.keys);
    }

    // shared-window addresses of the ring and its barriers, computed once
    const uint32_t ring_s = smem_u32(ring), bars_s = smem_u32(bars);
    // everything above reads only the parameters; the previous sweep's output (x_in, the count
    // deltas) and the stage's thresholds only after the previous grid completed
    if (PCA_P_PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    auto issue = [&](int it, int s) {
        const uint32_t st = ring_s + s * P_STAGE, bar = bars_s + 8 * s;
        const int jx = 2 * it;
        const bool two_x = rbeg + jx <= rend;
        const int jr = 2 * it - 2;
        const int nr = it == 0 ? 0 : min(2, rend - rbeg - jr);
        PCA_DCHECK(rbeg - 1 + jx >= -HALO && rbeg + jx + (two_x ? 1 : 0) - 1 < G.rows + HALO);
        PCA_DCHECK(nr == 0 || (rbeg + jr >= 0 && rbeg + jr + nr - 1 < G.rows));
        PCA_DCHECK(64 * seg + P_XROW <= p.pp && 64 * seg + P_GROW <= p.gpp);
        mbar_expect_tx_s(bar, (two_x ? 2 : 1) * P_XROW + nr * P_GROW);
        const uint8_t* xs = xin + (long long)jx * p.pp;
        bulk_g2s_s(st, xs, P_XROW, bar);
        if (two_x) bulk_g2s_s(st + P_XROW, xs + p.pp, P_XROW, bar);
        if (nr > 0) {
            const uint8_t* gs = gin + (long long)jr * p.gpp;
            bulk_g2s_s(st + P_GOFS, gs, P_GROW, bar);
            if (nr > 1) bulk_g2s_s(st + P_GOFS + P_GROW, gs + p.gpp, P_GROW, bar);
        }
    };
    if (elect_one()) {
        mbar_expect_tx(&bars[PCA_P_K], THR_ENTRIES * 4);
        bulk_g2s(s_thr, p.thr, THR_ENTRIES * 4, &bars[PCA_P_K]);
        for (int it = 0; it < min(PCA_P_K, nitems); ++it) issue(it, it);
    }
    mbar_wait(&bars[PCA_P_K], 0);

    // counts of the next two rows prefetched into registers one item ahead
    uint4 CR[2];
    auto load_counts = [&](int rfirst) {
        if (!cnt) return;
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (rfirst + q < rend)
                CR[q] = __ldcs(reinterpret_cast<const uint4*>(co + (long long)(rfirst + q - rbeg) * G.cpitch));
    };
    auto read_x = [&](const uint8_t* st, int q, PRow& x) {
        const uint8_t* xr = st + q * P_XROW;
        const int j0 = 16 + 2 * lane;
        const uint32_t h16 = *reinterpret_cast<const uint16_t*>(xr + j0);
        x.l = ((uint32_t)xr[j0 - 1] & 0x80u) << 17;  // bit 7 -> byte 3 bit 0
        x.r = (uint32_t)xr[j0 + 2] & 1u;
        if (PCA_P_LUT) {
            const uint2 lo = s_spread[h16 & 0xFFu], hi = s_spread[h16 >> 8];
            x.w[0] = lo.x;
            x.w[1] = lo.y;
            x.w[2] = hi.x;
            x.w[3] = hi.y;
        } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) x.w[i] = spread4((h16 >> (4 * i)) & 0xFu);
        }
    };
    // store the 16 new bits of local row r (+ torus pad copies, + wrapped halo rows)
    // (the pad / halo copies are one rarely taken branch: lanes at the torus seam or rows next
    // to the wrapped halos)
    const bool seam = PER && (k == 0 || k == nchunks - 1);
    // only runs that touch the first or last HALO rows of a self-wrapped torus write halo rows
    const bool near_halo = PER && G.self_halo_rows && (rbeg < HALO || rend > G.rows - HALO);
    auto store_row = [&](int r, uint32_t bits16) {
        uint8_t* dst = xo + (long long)(r - rbeg) * p.pp;
        *reinterpret_cast<uint16_t*>(dst) = (uint16_t)bits16;
        const bool hrow = near_halo && (r < HALO || r >= G.rows - HALO);
        if (seam || hrow) {
            auto put = [&](uint8_t* d) {
                *reinterpret_cast<uint16_t*>(d) = (uint16_t)bits16;
                if (k == 0) *reinterpret_cast<uint16_t*>(d + (G.W >> 3)) = (uint16_t)bits16;
                if (k == nchunks - 1) *reinterpret_cast<uint16_t*>(d - (G.W >> 3)) = (uint16_t)bits16;
            };
            if (seam) put(dst);
            if (hrow) put(r < HALO ? dst + (long long)G.rows * p.pp : dst - (long long)G.rows * p.pp);
        }
    };

    // update QN local rows r0 + q0 + qq (qq < QN, rows past nrow skipped) from the window X0..X3
    // (x rows r0-1 .. r0+2); QN = 2 interleaves the two rows' Philox chains (more ILP, more
    // registers), QN = 1 updates one row per call
    auto updq = [&](int r0, int nrow, int q0, const uint8_t* st, const PRow& X0, const PRow& X1,
                    const PRow& X2, const PRow& X3) {
        constexpr int QN = PCA_P_QN;
        const PRow* Wn[4] = {&X0, &X1, &X2, &X3};
        uint32_t IDX4[QN][4];
        bool edge[QN];
#pragma unroll
        for (int qq = 0; qq < QN; ++qq) {
            const int q = q0 + qq;
            const PRow& U = *Wn[q];
            const PRow& M = *Wn[q + 1];
            const PRow& D = *Wn[q + 2];
            const int grow = G.row0 + r0 + q;
            const uint32_t g16 = *reinterpret_cast<const uint16_t*>(st + P_GOFS + q * P_GROW + 2 * lane);
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
            // byte b: n1 << 4 | g << 3 | x << 2 (the fields do not overlap, so as multiply-adds on
            // the FMA pipe: the ALU pipe is the busier one); g's 4 bits spread to bit 3 of each
            // byte by one multiply (gn < 16: the shifted copies neither overlap nor carry)
            if (PCA_P_LUT_G) {  // g's label bytes from the shared table, x 8 in the multiply-add
                const uint2 glo = s_spread[g16 & 0xFFu], ghi = s_spread[g16 >> 8];
                const uint32_t gw[4] = {glo.x, glo.y, ghi.x, ghi.y};
#pragma unroll
                for (int i = 0; i < 4; ++i) IDX4[qq][i] = S[i] * 16u + (gw[i] * 8u + M.w[i] * 4u);
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t gsp = (((g16 >> (4 * i)) & 0xFu) * 0x01020408u) & 0x08080808u;
                    IDX4[qq][i] = S[i] * 16u + M.w[i] * 4u + gsp;
                }
            }
            edge[qq] = !PER && (k == 0 || k == nchunks - 1 || grow == 0 || grow == G.H - 1);
            if (q >= nrow) {  // past the run: its stage slot holds stale bytes; decide on index 0
#pragma unroll
                for (int i = 0; i < 4; ++i) IDX4[qq][i] = 0u;
            }
        }
        uint32_t O[QN][4], B[QN];
#pragma unroll
        for (int qq = 0; qq < QN; ++qq) B[qq] = 0u;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int qq = 0; qq < QN; ++qq) {
                const int q = q0 + qq;
                const int grow = G.row0 + r0 + q;
                const uint4 rnd = PCA_P_PRE ? philox_row<PCA_P_WIDE>(ppre[i], (uint32_t)grow, p.c.keys)
                                            : philox4x32_10(make_uint4((uint32_t)(4 * k + i), (uint32_t)grow,
                                                                       p.c.t, tagchain), p.c.keys);
                const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
                uint32_t bits = 0u;
#pragma unroll
                for (int b = 3; b >= 0; --b) {
                    uint32_t off = __byte_perm(IDX4[qq][i], 0u, 0x4440 + b);
                    if (PER) {
                        off += NB * 36 * 4;
                    } else {
                        const int np = edge[qq] ? p_neighbours_present<NB>(grow, G.H, ccol + 4 * i + b, G.W) : NB;
                        off += (uint32_t)np * 144u;
                    }
                    const uint32_t T = *reinterpret_cast<const uint32_t*>(thr_b + off);
                    uint32_t dummy;
                    asm("sub.cc.u32 %1, %2, %3;\n\taddc.u32 %0, %0, %0;" : "+r"(bits), "=r"(dummy)
                        : "r"(T), "r"(rw[b]));
                }
                const uint32_t nib = ~bits & 0xFu;  // bit b: site 4i + b is 1
                B[qq] |= nib << (4 * i);
                if (!PCA_P_LUT_O) O[qq][i] = spread4(nib);
            }
        if (PCA_P_LUT_O && cnt) {  // the new labels as count increments: the 16 bits by the table
#pragma unroll
            for (int qq = 0; qq < QN; ++qq) {
                const uint2 lo = s_spread[B[qq] & 0xFFu], hi = s_spread[B[qq] >> 8];
                O[qq][0] = lo.x;
                O[qq][1] = lo.y;
                O[qq][2] = hi.x;
                O[qq][3] = hi.y;
            }
        }
#pragma unroll
        for (int qq = 0; qq < QN; ++qq) {
            const int q = q0 + qq;
            if (q >= nrow) break;
            const int r = r0 + q;
            if (cnt) {  // byte-wise adds: no carries, deltas stay <= 255 between folds
                const uint4 c = CR[q];
                *reinterpret_cast<uint4*>(co + (long long)(r - rbeg) * G.cpitch) =
                    make_uint4(c.x + O[qq][0], c.y + O[qq][1], c.z + O[qq][2], c.w + O[qq][3]);
            }
            store_row(r, B[qq]);
        }
    };

    PRow A0, A1, B0, B1;
    load_counts(rbeg);
    int s = 0;
    uint32_t phase = 0;
    for (int it = 0; it < nitems; ++it) {
        mbar_wait(&bars[s], phase);
        const uint8_t* st = ring + s * P_STAGE;
        read_x(st, 0, B0);
        read_x(st, 1, B1);
        if (it > 0) {
            const int r0 = rbeg + 2 * it - 2;
            const int nrow = r0 + 1 < rend ? 2 : 1;
            updq(r0, nrow, 0, st, A0, A1, B0, B1);
            if (PCA_P_QN == 1 && nrow == 2) updq(r0, nrow, 1, st, A0, A1, B0, B1);
            load_counts(r0 + 2);
        }
        __syncwarp();
        if (it + PCA_P_K < nitems && elect_one()) {
            fence_proxy_async();
            issue(it + PCA_P_K, s);
        }
        A0 = B0;
        A1 = B1;
        if (++s == PCA_P_K) {
            s = 0;
            phase ^= 1u;
        }
    }
}

template <int NB, bool PER, bool NOCOUNT>
int launch_p(const PackedSweepParams& p, int batch, cudaStream_t s) {
    static LaunchInfo info[MAX_DEVICES];
    LaunchInfo& li = info[current_device()];
    if (!li.ok.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lock(launch_info_mutex());
        if (!li.ok.load(std::memory_order_relaxed)) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&li.sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.occ, sweep_packed_kernel<NB, PER, NOCOUNT>, 32, P_SMEM);
            if (li.occ < 1) li.occ = 1;
            li.ok.store(true, std::memory_order_release);
        }
    }
    const Geometry& G = p.c.geo;
    const long long segs = G.W / 512 + ((G.W % 512) ? 1 : 0);
    const long long target = (long long)li.sms * li.occ * PCA_P_WAVES;
    const int nr = p.c.rhi - p.c.rlo;
    if (nr <= 0) return 0;
    long long R = ((long long)nr * segs * batch + target - 1) / target;
    if (R < 2) R = 2;
    const int nrb = (int)((nr + R - 1) / R);
    if (nrb > 65535) return (int)cudaErrorInvalidConfiguration;
    dim3 grid((unsigned)segs, nrb, batch);
    if (PCA_P_PDL) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(32);
        cfg.dynamicSmemBytes = P_SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return (int)cudaLaunchKernelEx(&cfg, sweep_packed_kernel<NB, PER, NOCOUNT>, p, (int)R);
    }
    sweep_packed_kernel<NB, PER, NOCOUNT><<<grid, 32, P_SMEM, s>>>(p, (int)R);
    return (int)cudaGetLastError();
}

// padded byte state (kernels.cuh layout) <-> packed state; one thread per 16 columns of one
// padded row.  to_packed reads labels 0/1 (free-boundary sentinels 0xFF -> 0).
__global__ void to_packed_kernel(Geometry G, const uint8_t* __restrict__ xb, uint8_t* __restrict__ xp,
                                 int pp, long long pchain) {
    const int chain = blockIdx.z;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;  // 16-column chunk
    const int j = blockIdx.y;                             // padded row index 0 .. rows + 2 HALO - 1
    const int nch = G.W >> 4;
    if (k >= nch) return;
    const uint4 v = *reinterpret_cast<const uint4*>(xb + chain * G.xchain + (long long)j * G.xpitch + XOFF + 16 * k);
    auto nib = [](uint32_t w) { return (((w & ~(w >> 1) & 0x01010101u) * 0x01020408u) >> 24) & 0xFu; };
    const uint32_t b16 = nib(v.x) | (nib(v.y) << 4) | (nib(v.z) << 8) | (nib(v.w) << 12);
    uint8_t* row = xp + chain * pchain + (long long)j * pp;
    *reinterpret_cast<uint16_t*>(row + 16 + 2 * k) = (uint16_t)b16;
    if (G.periodic) {
        if (k == 0) *reinterpret_cast<uint16_t*>(row + 16 + (G.W >> 3)) = (uint16_t)b16;
        if (k == nch - 1) *reinterpret_cast<uint16_t*>(row + 14) = (uint16_t)b16;
    }
}

__global__ void from_packed_kernel(Geometry G, const uint8_t* __restrict__ xp, int pp, long long pchain,
                                   uint8_t* __restrict__ xb, int halo_up, int halo_dn) {
    const int chain = blockIdx.z;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;  // padded row index
    const int nch = G.W >> 4;
    if (k >= nch) return;
    // halo rows: written where a neighbour's rows live there (a torus, or a strip's neighbour);
    // a free boundary's outer halo rows keep the sentinel
    if ((j < HALO && !halo_up) || (j >= G.rows + HALO && !halo_dn)) return;
    const uint32_t b16 = *reinterpret_cast<const uint16_t*>(xp + chain * pchain + (long long)j * pp + 16 + 2 * k);
    const uint4 v = make_uint4(spread4(b16 & 0xFu), spread4((b16 >> 4) & 0xFu), spread4((b16 >> 8) & 0xFu),
                               spread4((b16 >> 12) & 0xFu));
    uint8_t* row = xb + chain * G.xchain + (long long)j * G.xpitch;
    *reinterpret_cast<uint4*>(row + XOFF + 16 * k) = v;
    if (G.periodic) {  // W % 16 == 0: 16 wrapped columns each side
        if (k == 0) *reinterpret_cast<uint4*>(row + XOFF + G.W) = v;
        if (k == nch - 1) *reinterpret_cast<uint4*>(row + XOFF - 16) = v;
    }
}

// dense or padded g rows (the context's g buffer: row j at (j + GHALO) gpitch, col at XOFF)
// -> packed g [rows][W/8]
__global__ void g_to_packed_kernel(Geometry G, const uint8_t* __restrict__ gb, uint8_t* __restrict__ gp,
                                   int gpp, long long gpchain) {
    const int chain = blockIdx.z;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    if (k >= (G.W >> 4)) return;
    const uint4 v = *reinterpret_cast<const uint4*>(gb + chain * G.gchain + (long long)(r + GHALO) * G.gpitch + XOFF + 16 * k);
    auto nib = [](uint32_t w) { return (((w & 0x01010101u) * 0x01020408u) >> 24) & 0xFu; };
    const uint32_t b16 = nib(v.x) | (nib(v.y) << 4) | (nib(v.z) << 8) | (nib(v.w) << 12);
    *reinterpret_cast<uint16_t*>(gp + chain * gpchain + (long long)r * gpp + 2 * k) = (uint16_t)b16;
}

// counts16 += delta8, delta8 = 0 (16 sites per thread)
__global__ void fold_counts_kernel(Geometry G, uint16_t* __restrict__ counts, uint8_t* __restrict__ delta,
                                   long long dchain) {
    const int chain = blockIdx.z;
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int r = blockIdx.y;
    if (k >= ((G.W + 15) >> 4)) return;  // whole 16-column chunks (a ragged tail adds zeros)
    uint4* dp = reinterpret_cast<uint4*>(delta + chain * dchain + (long long)r * G.cpitch + 16 * k);
    const uint4 d = *dp;
    uint4* cp = reinterpret_cast<uint4*>(counts + chain * G.cchain + (long long)r * G.cpitch + 16 * k);
    const uint32_t dw[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint4 c = cp[h];
        c.x += __byte_perm(dw[2 * h], 0u, 0x4140); c.y += __byte_perm(dw[2 * h], 0u, 0x4342);
        c.z += __byte_perm(dw[2 * h + 1], 0u, 0x4140); c.w += __byte_perm(dw[2 * h + 1], 0u, 0x4342);
        cp[h] = c;
    }
    *dp = make_uint4(0u, 0u, 0u, 0u);
}

}  // namespace

int launch_fold_counts(const Geometry& G, uint16_t* counts, uint8_t* delta, long long dchain, int batch,
                       void* stream) {
    const int nch = (G.W + 15) >> 4;
    dim3 grid((nch + 127) / 128, G.rows, batch);
    fold_counts_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(G, counts, delta, dchain);
    return (int)cudaGetLastError();
}

int launch_sweep_packed(const PackedSweepParams& p, int batch, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const Geometry& G = p.c.geo;
    const bool nc = !p.c.count_enable;
#define PCA_P_LAUNCH(NBV, PERV) \
    return nc ? launch_p<NBV, PERV, true>(p, batch, s) : launch_p<NBV, PERV, false>(p, batch, s)
    if (G.nbhd == 8) {
        if (G.periodic) PCA_P_LAUNCH(8, true);
        PCA_P_LAUNCH(8, false);
    }
    if (G.periodic) PCA_P_LAUNCH(4, true);
    PCA_P_LAUNCH(4, false);
#undef PCA_P_LAUNCH
}

int launch_state_to_packed(const Geometry& G, const uint8_t* xb, uint8_t* xp, int pp, long long pchain,
                           int batch, void* stream) {
    const int nch = G.W >> 4;
    dim3 grid((nch + 127) / 128, G.rows + 2 * HALO, batch);
    to_packed_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(G, xb, xp, pp, pchain);
    return (int)cudaGetLastError();
}

int launch_state_from_packed(const Geometry& G, const uint8_t* xp, int pp, long long pchain, uint8_t* xb,
                             int batch, void* stream, int halo_up, int halo_dn) {
    const int nch = G.W >> 4;
    dim3 grid((nch + 127) / 128, G.rows + 2 * HALO, batch);
    from_packed_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(G, xp, pp, pchain, xb, halo_up, halo_dn);
    return (int)cudaGetLastError();
}

int launch_g_to_packed(const Geometry& G, const uint8_t* gb, uint8_t* gp, int gpp, long long gpchain, int batch,
                       void* stream) {
    const int nch = G.W >> 4;
    dim3 grid((nch + 127) / 128, G.rows, batch);
    g_to_packed_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(G, gb, gp, gpp, gpchain);
    return (int)cudaGetLastError();
}

}  // namespace pcab200
