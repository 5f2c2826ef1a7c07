// sweep_gibbs_binary.cu -- the GPU Gibbs sampler (R21) for levels == 2 and Moore-8 on the
// binary PCA kernel's data path (sweep_binary.cu): one warp per CTA owns a 512-column
// segment (16 sites per lane) of a run of rows, streamed through a per-warp ring of 1-D TMA
// bulk copies; SWAR neighbour counts; one Philox4x32-10 call per 4 sites (tag GIBBS);
// integer thresholds T[(np*9 + n1)*2 + g] of the Gibbs conditional.
//
// A sweep is two launches, one per row parity p (colours 2p and 2p+1 of the checkerboard
// scan, oracle/orc_gibbs_sweep_coloured).  The sweep maps buffer X (x_t) to buffer Y:
//   parity 0 (even rows): rows r-1, r, r+1 from X; even rows of Y written;
//   parity 1 (odd rows):  rows r-1, r+1 from Y (the new even rows), row r from X; odd rows
//                         of Y written.
// Nothing a launch reads is written by it, so overlapping segment reads need no ordering, and
// Y ends as x_{t+1} (the runtime swaps the buffers like a PCA sweep).
// Within a row, colour 2p (even columns) is decided from the old labels; colour 2p+1 (odd
// columns) from the new even-column labels of the same row (its other neighbours are rows of
// the other parity).  The one new label a lane needs from outside its 16 sites (column
// c0+16) comes from the next lane by shuffle, or is recomputed by lane 31 from the staged
// rows, its quad's Philox word and its g (16-column torus pads: W % 16 == 0).
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "tma_ring.cuh"

#ifndef PCA_GB_PDL
#define PCA_GB_PDL 1  // programmatic dependent launch between consecutive launches (kernels.cuh)
#endif
#ifndef PCA_GB_WAVES
#define PCA_GB_WAVES 4  // waves of resident warps the row runs are sized for (8192^2 torus Gibbs
                        // sweep: 1 wave 135.2 us, 2 135.0, 4 126.9)
#endif

namespace pcab200 {
namespace {

// ring depth x resident CTAs, measured at 8192^2 (us per sweep): 3 x 16: 135.5; 3 x 18: 136.9;
// 3 x 20: 137.7; 4 x 12: 142.8; 4 x 16: 143.2; 2 x 24: 142.3; 6 x 12: 168.2
#ifndef PCA_GB_K
#define PCA_GB_K 3
#endif
#ifndef PCA_GB_CTAS
#define PCA_GB_CTAS 16
#endif
constexpr int GK = PCA_GB_K;                   // ring depth (items of 2 x rows)
constexpr int GCTAS = PCA_GB_CTAS;             // resident one-warp CTAs per SM
constexpr int SEG = 32;                        // 16-site chunks per segment
constexpr int XROW = 16 * SEG + 32;            // 544: [col0-16, col0+528)
constexpr int GROWB = 16 * SEG;                // 512
constexpr int CROWB = 32 * SEG;                // 1024
constexpr int GOF = 2 * XROW, COF = GOF + GROWB;
constexpr int GSTAGE = COF + CROWB;            // 2624
constexpr int GRING_OFF = 64;
constexpr int GSMEM = GRING_OFF + GK * GSTAGE;
constexpr int GTHR_PAD = GIBBS_THR_PAD;

__device__ __forceinline__ uint32_t to01g(uint32_t w) { return w & ~(w >> 1) & 0x01010101u; }

struct GRow {
    uint32_t w[4];
    uint32_t l, r;
};

template <bool PER>
__global__ void __launch_bounds__(32, GCTAS)
    gibbs_binary_kernel(const __grid_constant__ GibbsBinParams p, int R) {
    __shared__ __align__(16) uint32_t s_thr[GTHR_PAD];
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    uint8_t* ring = smem + GRING_OFF;
    const int lane = threadIdx.x;
    if (PCA_GB_PDL) pdl_begin();
    if (lane == 0) {
        for (int s = 0; s <= GK; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();

    const Geometry& G = p.c.geo;
    const int seg = blockIdx.x, chain = blockIdx.z;
    // processed rows: r = rfirst + 2i, i in [i0, i1) (rows of parity p in [rlo, rhi))
    int rfirst = p.c.rlo;
    if (((G.row0 + rfirst) & 1) != p.parity) ++rfirst;
    const int nproc_all = rfirst < p.c.rhi ? (p.c.rhi - rfirst + 1) / 2 : 0;
    const int i0 = blockIdx.y * R, i1 = min(i0 + R, nproc_all);
    if (i0 >= i1) return;
    const int n = i1 - i0;            // rows this warp updates
    const int nitems = n + 1;         // item j: x rows (r_j - 1, r_j) and g / counts of r_{j-1}
    auto row_of = [&](int j) { return rfirst + 2 * (i0 + j); };
    const int nch = min(SEG, G.nchunks - seg * SEG);
    const int col0 = 16 * SEG * seg;
    const int k = seg * SEG + lane;
    const bool active = lane < nch;
    const int ccol = col0 + 16 * lane;
    const uint32_t xbytes = 16 * nch + 32, gbytes = 16 * nch;
    const uint32_t cbytes = p.c.count_enable ? 32 * nch : 0;
    const uint8_t* xown = p.c.x_in + chain * G.xchain + col0;   // X: the updated rows (old)
    const uint8_t* xnb = p.x_nb + chain * G.xchain + col0;      // rows r-1, r+1
    const uint8_t* gin = p.c.g + chain * G.gchain + XOFF + col0;
    uint16_t* cseg = p.c.counts + chain * G.cchain + col0;
    uint8_t* xo = p.c.x_out + chain * G.xchain;
    const uint32_t tagchain = (TAG_GIBBS << 24) | (p.c.chain0 + (uint32_t)chain);

    auto issue = [&](int j, int s) {
        uint8_t* st = ring + s * GSTAGE;
        const int r = row_of(j);
        const bool has_own = j < n;   // item n carries only row r_{n-1} + 1
        const bool has_g = j > 0;
        PCA_DCHECK(xbytes * (has_own ? 2u : 1u) + (has_g ? gbytes + cbytes : 0u) <= (uint32_t)GSTAGE);
        mbar_expect_tx(&bars[s], xbytes * (has_own ? 2u : 1u) + (has_g ? gbytes + cbytes : 0u));
        bulk_g2s(st, xnb + (long long)(r - 1 + HALO) * G.xpitch, xbytes, &bars[s]);
        if (has_own) bulk_g2s(st + XROW, xown + (long long)(r + HALO) * G.xpitch, xbytes, &bars[s]);
        if (has_g) {
            const int rp = row_of(j - 1);
            bulk_g2s(st + GOF, gin + (long long)(rp + GHALO) * G.gpitch, gbytes, &bars[s]);
            if (cbytes) bulk_g2s(st + COF, cseg + (long long)rp * G.cpitch, cbytes, &bars[s]);
        }
    };
    if (elect_one()) {
        mbar_expect_tx(&bars[GK], GTHR_PAD * 4);
        bulk_g2s(s_thr, p.thr, GTHR_PAD * 4, &bars[GK]);
        for (int j = 0; j < min(GK, nitems); ++j) issue(j, j);
    }
    mbar_wait(&bars[GK], 0);

    auto read_x = [&](const uint8_t* xr, GRow& x) {
        const uint4 v = *reinterpret_cast<const uint4*>(xr + 16 + 16 * lane);
        x.l = *reinterpret_cast<const uint32_t*>(xr + 12 + 16 * lane);
        x.r = *reinterpret_cast<const uint32_t*>(xr + 32 + 16 * lane);
        x.w[0] = v.x; x.w[1] = v.y; x.w[2] = v.z; x.w[3] = v.w;
    };
    auto to01row = [](GRow& x) {
#pragma unroll
        for (int i = 0; i < 4; ++i) x.w[i] = to01g(x.w[i]);
        x.l = to01g(x.l);
        x.r = to01g(x.r);
    };
    const uint8_t* thr_b = reinterpret_cast<const uint8_t*>(s_thr);

    // update row r from U (row r-1), M (row r, old), D (row r+1); g / counts of r in stage st
    auto update = [&](int r, const uint8_t* st, GRow U, GRow M, GRow D) {
        const int grow = G.row0 + r;
        const uint4 gv = *reinterpret_cast<const uint4*>(st + GOF + 16 * lane);
        const uint32_t Gw[4] = {gv.x, gv.y, gv.z, gv.w};
        if (!PER) {
            to01row(U);
            to01row(M);
            to01row(D);
        }
        // vertical + diagonal neighbours (rows r-1, r+1): unchanged during this launch
        uint32_t T[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) T[i] = U.w[i] + D.w[i];
        const uint32_t TL = U.l + D.l, TR = U.r + D.r;
        uint32_t NUD[4];
        NUD[0] = from_left(TL, T[0]) + T[0] + from_right(T[0], T[1]);
        NUD[1] = from_left(T[0], T[1]) + T[1] + from_right(T[1], T[2]);
        NUD[2] = from_left(T[1], T[2]) + T[2] + from_right(T[2], T[3]);
        NUD[3] = from_left(T[2], T[3]) + T[3] + from_right(T[3], TR);
        // present neighbours (free boundary: fewer at the lattice edge)
        const bool edge = !PER && (k == 0 || k == G.nchunks - 1 || grow == 0 || grow == G.H - 1);
        auto np_of = [&](int c) -> uint32_t {
            if (PER || !edge) return 8u;
            const int er = (grow == 0) + (grow == G.H - 1);
            const int ec = (c == 0) + (c == G.W - 1);
            return (uint32_t)((3 - er) * (3 - ec) - 1);
        };
        // Philox words of the 16 sites
        uint32_t rw[16];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 rnd = philox4x32_10(make_uint4((uint32_t)(4 * k + i), (uint32_t)grow, p.c.t, tagchain), p.c.keys);
            rw[4 * i + 0] = rnd.x; rw[4 * i + 1] = rnd.y; rw[4 * i + 2] = rnd.z; rw[4 * i + 3] = rnd.w;
        }
        // decide the sites of byte positions `b0` and `b0 + 2` of every word from the middle
        // row words Mw (left word ml, right word mr)
        auto decide = [&](uint32_t (&O)[4], const uint32_t (&Mw)[4], uint32_t ml, uint32_t mr, int b0) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t n1w = NUD[i] + from_left(i == 0 ? ml : Mw[i - 1], Mw[i]) +
                                     from_right(Mw[i], i == 3 ? mr : Mw[i + 1]);
#pragma unroll
                for (int bb = 0; bb < 2; ++bb) {
                    const int b = b0 + 2 * bb;
                    const uint32_t n1 = (n1w >> (8 * b)) & 0xFFu;
                    const uint32_t g = (Gw[i] >> (8 * b)) & 0xFFu;
                    const uint32_t np = np_of(ccol + 4 * i + b);
                    const uint32_t Tt = *reinterpret_cast<const uint32_t*>(thr_b + 4 * ((np * 9u + n1) * 2u + g));
                    const uint32_t w = rw[4 * i + b] > Tt ? 1u : 0u;
                    O[i] = (O[i] & ~(0xFFu << (8 * b))) | (w << (8 * b));
                }
            }
        };
        // colour 2p: even columns, from the old row
        uint32_t O[4] = {M.w[0], M.w[1], M.w[2], M.w[3]};
        decide(O, M.w, M.l, M.r, 0);
        // the new label of column c0+16 (the next lane's first site, colour 2p)
        const uint32_t nxt = __shfl_down_sync(0xFFFFFFFFu, O[0] & 0xFFu, 1);
        uint32_t mr = M.r;  // bytes: columns c0+16 .. c0+19
        const bool has_next = ccol + 16 < G.W;
        const bool wraps = PER && ccol + 16 == G.W;
        uint32_t v16 = mr & 0xFFu;
        if (active && (has_next || wraps)) {
            if (lane < 31 && has_next && lane + 1 < nch) {
                v16 = nxt;
            } else {
                // recompute site c0+16 (column 0 when it wraps) from the staged rows
                const int cq = wraps ? 0 : ccol + 16;
                const uint4 rn = philox4x32_10(make_uint4((uint32_t)(cq >> 2), (uint32_t)grow, p.c.t, tagchain), p.c.keys);
                const uint32_t gq = __ldg(p.c.g + chain * G.gchain + (long long)(r + GHALO) * G.gpitch + XOFF + cq);
                auto bytes3 = [](const GRow& x) {  // columns c0+15, c0+16, c0+17
                    return ((x.w[3] >> 24) & 0xFFu) + (x.r & 0xFFu) + ((x.r >> 8) & 0xFFu);
                };
                const uint32_t n1 = bytes3(U) + bytes3(D) + ((M.w[3] >> 24) & 0xFFu) + ((M.r >> 8) & 0xFFu);
                uint32_t npq = 8u;
                if (!PER) {
                    const int er = (grow == 0) + (grow == G.H - 1);
                    const int ec = (cq == 0) + (cq == G.W - 1);
                    npq = (uint32_t)((3 - er) * (3 - ec) - 1);
                }
                v16 = rn.x > s_thr[(npq * 9u + n1) * 2u + gq] ? 1u : 0u;
            }
        }
        mr = (mr & ~0xFFu) | v16;
        // colour 2p+1: odd columns, from the new even-column labels of the row
        decide(O, O, M.l, mr, 1);
        if (!active) return;
        // ---- fused MPM counts of label 1 ----
        if (cbytes) {
            const uint4* cs = reinterpret_cast<const uint4*>(st + COF + 32 * lane);
            uint4 c0 = cs[0], c1 = cs[1];
            c0.x += __byte_perm(O[0], 0u, 0x4140); c0.y += __byte_perm(O[0], 0u, 0x4342);
            c0.z += __byte_perm(O[1], 0u, 0x4140); c0.w += __byte_perm(O[1], 0u, 0x4342);
            c1.x += __byte_perm(O[2], 0u, 0x4140); c1.y += __byte_perm(O[2], 0u, 0x4342);
            c1.z += __byte_perm(O[3], 0u, 0x4140); c1.w += __byte_perm(O[3], 0u, 0x4342);
            uint4* cp = reinterpret_cast<uint4*>(cseg + 16 * lane + (long long)r * G.cpitch);
            cp[0] = c0;
            cp[1] = c1;
        }
        store_row_chunk<HALO, XOFF>(xo + (long long)(r + HALO) * G.xpitch, O, ccol, G.W - ccol, k, r,
                                    G.W, G.nchunks, G.rows, G.xpitch, PER, G.self_halo_rows);
    };

    GRow U, M, D;
    int s = 0;
    uint32_t phase = 0;
    for (int j = 0; j < nitems; ++j) {
        mbar_wait(&bars[s], phase);
        const uint8_t* st = ring + s * GSTAGE;
        // every lane runs the update (it shuffles); lanes past the lattice only skip the stores
        read_x(st, D);                                  // row r_j - 1 = r_{j-1} + 1
        if (j > 0) update(row_of(j - 1), st, U, M, D);  // g / counts of r_{j-1} in this stage
        if (j < n) {
            U = D;
            read_x(st + XROW, M);                       // row r_j (old)
        }
        __syncwarp();
        if (j + GK < nitems && elect_one()) {
            fence_proxy_async();
            issue(j + GK, s);
        }
        if (++s == GK) {
            s = 0;
            phase ^= 1u;
        }
    }
}

template <bool PER>
int launch_gb2(const GibbsBinParams& p, int batch, cudaStream_t s) {
    static LaunchInfo info[MAX_DEVICES];
    LaunchInfo& li = info[current_device()];
    if (!li.ok.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lock(launch_info_mutex());
        if (!li.ok.load(std::memory_order_relaxed)) {
            cudaError_t e = cudaFuncSetAttribute(gibbs_binary_kernel<PER>, cudaFuncAttributeMaxDynamicSharedMemorySize, GSMEM);
            if (e != cudaSuccess) return (int)e;
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&li.sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.occ, gibbs_binary_kernel<PER>, 32, GSMEM);
            if (li.occ < 1) li.occ = 1;
            li.ok.store(true, std::memory_order_release);
        }
    }
    const int occ = li.occ, sms = li.sms;
    const Geometry& G = p.c.geo;
    int rfirst = p.c.rlo;
    if (((G.row0 + rfirst) & 1) != p.parity) ++rfirst;
    const int nproc = rfirst < p.c.rhi ? (p.c.rhi - rfirst + 1) / 2 : 0;
    if (nproc <= 0) return 0;
    const long long segs = (G.nchunks + SEG - 1) / SEG;
    const long long target = (long long)sms * occ * PCA_GB_WAVES;
    long long R = ((long long)nproc * segs * batch + target - 1) / target;
    if (R < 1) R = 1;
    const long long nrb = (nproc + R - 1) / R;
    if (nrb > 65535) return (int)cudaErrorInvalidConfiguration;
    dim3 grid((unsigned)segs, (unsigned)nrb, batch);
    if (PCA_GB_PDL) return (int)launch_pdl(gibbs_binary_kernel<PER>, grid, dim3(32), GSMEM, s, p, (int)R);
    gibbs_binary_kernel<PER><<<grid, 32, GSMEM, s>>>(p, (int)R);
    return (int)cudaGetLastError();
}

}  // namespace

int launch_gibbs_binary(const GibbsBinParams& p, int batch, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    return p.c.geo.periodic ? launch_gb2<true>(p, batch, s) : launch_gb2<false>(p, batch, s);
}

}  // namespace pcab200
