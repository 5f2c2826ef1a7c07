// sweep_binary2.cu -- TWO synchronous lazy-PCA sweeps (t and t+1) per HBM pass, levels == 2
// (temporal blocking).
//
// Each sweep is exactly the per-site law of sweep_binary.cu (R1; integer
// thresholds T = ceil(p0 2^32) - 1 tabulated on the host per beta stage; Philox4x32-10 keyed by
// the GLOBAL (col, row, t)), so the result is bit-identical to two single sweeps.  What changes
// is the data movement: x_t is streamed from HBM once, x_{t+1} lives only in registers, and
// x_{t+2}, g and the MPM counts (incremented by both sweeps) cross HBM once -- 7 B per two
// site-updates instead of 14.
//
// Work decomposition as in sweep_binary.cu (one warp per CTA, a 512-column segment, 16 sites
// per lane, a run of R output rows): x_t rows rbeg-2 .. rend+1 stream through a KSTAGES-deep
// TMA bulk-copy ring (one x row, the matching g row and a counts row per stage).  When x_t row
// j arrives the warp computes sweep t on row j-1 (rows rbeg-1 .. rend: one redundant row on
// each side, recomputed identically by the neighbouring task) and sweep t+1 on row j-2.  At the
// segment's left / right edge the first / last lane also computes sweep t on the 4 sites just
// outside the segment (the neighbours sweep t+1 needs), from the 544-byte stage windows and
// the torus pads; the x_{t+1} words left / right of each chunk come from the adjacent lanes by
// warp shuffle.  Requires W % 16 == 0 and a context that owns the whole lattice.
#include <cuda_runtime.h>

#include "kernels.cuh"
#include "tma_ring.cuh"

#ifndef PCA_B2_WAVES
#define PCA_B2_WAVES 1  // waves of resident warps the row runs are sized for (8192^2 torus, us
                        // per sweep: 1 wave 100.5, 2 101.5, 4 105.5)
#endif

namespace pcab200 {
namespace {

#ifndef PCA2_KSTAGES
#define PCA2_KSTAGES 4
#endif
#ifndef PCA2_MIN_CTAS
#define PCA2_MIN_CTAS 12
#endif
constexpr int KSTAGES = PCA2_KSTAGES;
constexpr int MIN_CTAS = PCA2_MIN_CTAS;
constexpr int SEG_CHUNKS = 32;
constexpr int WIN_BYTES = 16 * SEG_CHUNKS + 32;   // 544: columns [col0-16, col0+528)
constexpr int CROW_BYTES = 32 * SEG_CHUNKS;       // 1024
constexpr int XOFS = 0, GOFS = WIN_BYTES, COFS = 2 * WIN_BYTES;
constexpr int STAGE_BYTES = COFS + CROW_BYTES;    // 2112
constexpr int RING_OFFSET = 64;
constexpr int SMEM_BYTES = RING_OFFSET + KSTAGES * STAGE_BYTES;
constexpr unsigned FULL = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t to01(uint32_t w) { return w & ~(w >> 1) & 0x01010101u; }

template <int NB>
__device__ __forceinline__ int neighbours_present(int grow, int H, int c, int W) {
    const int er = (grow == 0) + (grow == H - 1);
    const int ec = (c == 0) + (c == W - 1);
    return NB == 8 ? (3 - er) * (3 - ec) - 1 : 4 - er - ec;
}

struct XRow {       // a row of x_t as seen by one lane
    uint32_t w[4];  // the lane's 16 labels
    uint32_t l, r;  // the words left / right of the chunk
    uint32_t ll, rr;  // the words left of l / right of r (extra-word neighbourhoods)
};
struct YRow {       // a row of x_{t+1} (registers only)
    uint32_t w[4];
    uint32_t l, r;
};

// New labels of 4 sites (one word) from their vertical window words and Philox output.
template <int NB, bool PER>
__device__ __forceinline__ uint32_t decide_word(uint32_t Uw, uint32_t Mw, uint32_t Dw, uint32_t Ul,
                                                uint32_t Ml, uint32_t Dl, uint32_t Ur, uint32_t Mr,
                                                uint32_t Dr, uint32_t Gw, const uint4& rnd,
                                                const uint8_t* tbl, bool edge, int grow, int gcol,
                                                int H, int W) {
    uint32_t S;
    if (NB == 8) {
        const uint32_t V = Uw + Mw + Dw, VL = Ul + Ml + Dl, VR = Ur + Mr + Dr;
        S = from_left(VL, V) + V + from_right(V, VR) - Mw;
    } else {
        S = Uw + Dw + from_left(Ml, Mw) + from_right(Mw, Mr);
    }
    const uint32_t idx4 = (S << 4) | (Gw << 3) | (Mw << 2);
    const uint32_t rw[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
    uint32_t o = 0u;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        uint32_t off = __byte_perm(idx4, 0u, 0x4440 + b);
        if (PER) {
            off += NB * 144;
        } else {
            const int np = edge ? neighbours_present<NB>(grow, H, gcol + b, W) : NB;
            off += (uint32_t)np * 144u;
        }
        const uint32_t T = *reinterpret_cast<const uint32_t*>(tbl + off);
        if (rw[b] > T) o += 1u << (8 * b);
    }
    return o;
}

template <int NB, bool PER>
__global__ void __launch_bounds__(32, MIN_CTAS)
    sweep_binary2_kernel(const __grid_constant__ Binary2SweepParams p, int R) {
    __shared__ __align__(16) uint32_t s_thr[2][THR_ENTRIES];
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    uint8_t* ring = smem + RING_OFFSET;
    const int lane = threadIdx.x;
    for (int i = lane; i < THR_ENTRIES; i += 32) {
        s_thr[0][i] = p.thr[0][i];
        s_thr[1][i] = p.thr[1][i];
    }
    if (lane == 0) {
        for (int s = 0; s < KSTAGES; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();

    const Geometry& G = p.c.geo;
    const int seg = blockIdx.x;
    const int chain = blockIdx.z;
    const int rbeg = p.c.rlo + blockIdx.y * R;
    const int rend = min(rbeg + R, p.c.rhi);
    if (rbeg >= rend) return;
    const int nitems = rend - rbeg + 4;  // x_t rows rbeg-2 .. rend+1
    const int nch = min(SEG_CHUNKS, G.nchunks - seg * SEG_CHUNKS);
    const int e = nch - 1;                  // the segment's last lane
    const int col0 = 16 * SEG_CHUNKS * seg;
    const int k = seg * SEG_CHUNKS + lane;  // this lane's chunk
    const bool active = lane < nch;
    const int ccol = col0 + 16 * lane;
    const uint32_t wbytes = 16 * nch + 32;
    const uint32_t cbytes = (p.c.count_enable || p.count2) ? 32 * nch : 0;
    const uint8_t* xin = p.c.x_in + chain * G.xchain + col0 + (long long)(rbeg - 2 + HALO) * G.xpitch;
    const uint8_t* gin = p.c.g + chain * G.gchain + col0 + (long long)(rbeg - 3 + GHALO) * G.gpitch;
    const uint16_t* cin = p.c.counts + chain * G.cchain + col0 + (long long)(rbeg - 4) * G.cpitch;
    uint8_t* xo = p.c.x_out + chain * G.xchain + (long long)(rbeg - 4 + HALO) * G.xpitch;
    uint16_t* co = p.c.counts + chain * G.cchain + ccol + (long long)(rbeg - 4) * G.cpitch;
    const uint32_t tagchain = (TAG_PCA << 24) | (p.c.chain0 + (uint32_t)chain);
    const uint8_t* tbl0 = reinterpret_cast<const uint8_t*>(s_thr[0]);
    const uint8_t* tbl1 = reinterpret_cast<const uint8_t*>(s_thr[1]);
    const uint32_t t0 = p.c.t, t1 = p.c.t + 1u;
    // extra words just outside the segment: needed unless the segment touches a free edge
    const bool need_left = PER || col0 > 0;
    const bool need_right = PER || col0 + 16 * nch < G.W;

    // elected lane: item it = x_t row rbeg-2+it, g row rbeg-3+it (it in [2, R+3]),
    // counts row rbeg-4+it (it in [4, R+3])
    auto issue = [&](int it, int s) {
        uint8_t* st = ring + s * STAGE_BYTES;
        const bool gr = it >= 2, cr = it >= 4 && cbytes;
        PCA_DCHECK(rbeg - 2 + it >= -HALO && rbeg - 2 + it < G.rows + HALO);
        PCA_DCHECK(!gr || (rbeg - 3 + it >= -GHALO && rbeg - 3 + it < G.rows + GHALO));
        mbar_expect_tx(&bars[s], wbytes + (gr ? wbytes : 0u) + (cr ? cbytes : 0u));
        bulk_g2s(st + XOFS, xin + (long long)it * G.xpitch, wbytes, &bars[s]);
        if (gr) bulk_g2s(st + GOFS, gin + (long long)it * G.gpitch, wbytes, &bars[s]);
        if (cr) bulk_g2s(st + COFS, cin + (long long)it * G.cpitch, cbytes, &bars[s]);
    };
    if (elect_one())
        for (int it = 0; it < min(KSTAGES, nitems); ++it) issue(it, it);

    auto read_x = [&](const uint8_t* st, XRow& x) {
        const uint8_t* xr = st + XOFS + 16 * lane;
        const uint4 v = *reinterpret_cast<const uint4*>(xr + 16);
        x.w[0] = v.x; x.w[1] = v.y; x.w[2] = v.z; x.w[3] = v.w;
        x.l = *reinterpret_cast<const uint32_t*>(xr + 12);
        x.r = *reinterpret_cast<const uint32_t*>(xr + 32);
        x.ll = *reinterpret_cast<const uint32_t*>(xr + 8);
        x.rr = *reinterpret_cast<const uint32_t*>(xr + 36);
        if (!PER) {
#pragma unroll
            for (int i = 0; i < 4; ++i) x.w[i] = to01(x.w[i]);
            x.l = to01(x.l); x.r = to01(x.r); x.ll = to01(x.ll); x.rr = to01(x.rr);
        }
    };

    // sweep t on local row a (window x_t rows a-1, a, a+1 = U, M, D; g words of row a)
    auto sweep_t = [&](int a, const XRow& U, const XRow& M, const XRow& D, const uint8_t* gst,
                       YRow& y) {
        int ga = G.row0 + a;
        bool absent = false;
        if (PER) ga = (ga + G.H) % G.H;
        else absent = ga < 0 || ga >= G.H;
        uint32_t o[4] = {0, 0, 0, 0}, xl = 0, xr = 0;
        if (!absent && active) {
            const uint4 gv = *reinterpret_cast<const uint4*>(gst + 16 + 16 * lane);
            const uint32_t Gw[4] = {gv.x, gv.y, gv.z, gv.w};
            const bool edge = !PER && (k == 0 || k == G.nchunks - 1 || ga == 0 || ga == G.H - 1);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint4 rnd = philox4x32_10(make_uint4((uint32_t)(4 * k + i), (uint32_t)ga, t0, tagchain),
                                                p.c.keys);
                o[i] = decide_word<NB, PER>(U.w[i], M.w[i], D.w[i], i ? U.w[i - 1] : U.l,
                                            i ? M.w[i - 1] : M.l, i ? D.w[i - 1] : D.l,
                                            i < 3 ? U.w[i + 1] : U.r, i < 3 ? M.w[i + 1] : M.r,
                                            i < 3 ? D.w[i + 1] : D.r, Gw[i], rnd, tbl0, edge, ga,
                                            ccol + 4 * i, G.H, G.W);
            }
            // the word left of the segment (lane 0) / right of it (last lane)
            if (lane == 0 && need_left) {
                const int gc = PER ? (col0 - 4 + G.W) % G.W : col0 - 4;
                const uint32_t Gl = *reinterpret_cast<const uint32_t*>(gst + 12);
                const bool edge2 = !PER && (ga == 0 || ga == G.H - 1);
                const uint4 rnd = philox4x32_10(make_uint4((uint32_t)(gc >> 2), (uint32_t)ga, t0, tagchain),
                                                p.c.keys);
                xl = decide_word<NB, PER>(U.l, M.l, D.l, U.ll, M.ll, D.ll, U.w[0], M.w[0], D.w[0], Gl,
                                          rnd, tbl0, edge2, ga, gc, G.H, G.W);
            }
            if (lane == e && need_right) {
                const int gc = PER ? (col0 + 16 * nch) % G.W : col0 + 16 * nch;
                const uint32_t Gr = *reinterpret_cast<const uint32_t*>(gst + 32 + 16 * lane);
                const bool edge2 = !PER && (ga == 0 || ga == G.H - 1);
                const uint4 rnd = philox4x32_10(make_uint4((uint32_t)(gc >> 2), (uint32_t)ga, t0, tagchain),
                                                p.c.keys);
                xr = decide_word<NB, PER>(U.r, M.r, D.r, U.w[3], M.w[3], D.w[3], U.rr, M.rr, D.rr, Gr,
                                          rnd, tbl0, edge2, ga, gc, G.H, G.W);
            }
        }
        y.w[0] = o[0]; y.w[1] = o[1]; y.w[2] = o[2]; y.w[3] = o[3];
        const uint32_t fromL = __shfl_up_sync(FULL, o[3], 1);
        const uint32_t fromR = __shfl_down_sync(FULL, o[0], 1);
        y.l = lane == 0 ? xl : fromL;
        y.r = lane == e ? xr : fromR;
    };

    // sweep t+1 on output row b (window x_{t+1} rows b-1, b, b+1), store + counts
    auto sweep_t1 = [&](int b, const YRow& U, const YRow& M, const YRow& D, const uint8_t* gst,
                        const uint8_t* cst) {
        if (!active) return;
        const int gb = G.row0 + b;
        const uint4 gv = *reinterpret_cast<const uint4*>(gst + 16 + 16 * lane);
        const uint32_t Gw[4] = {gv.x, gv.y, gv.z, gv.w};
        const bool edge = !PER && (k == 0 || k == G.nchunks - 1 || gb == 0 || gb == G.H - 1);
        uint32_t O[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 rnd = philox4x32_10(make_uint4((uint32_t)(4 * k + i), (uint32_t)gb, t1, tagchain),
                                            p.c.keys);
            O[i] = decide_word<NB, PER>(U.w[i], M.w[i], D.w[i], i ? U.w[i - 1] : U.l,
                                        i ? M.w[i - 1] : M.l, i ? D.w[i - 1] : D.l,
                                        i < 3 ? U.w[i + 1] : U.r, i < 3 ? M.w[i + 1] : M.r,
                                        i < 3 ? D.w[i + 1] : D.r, Gw[i], rnd, tbl1, edge, gb,
                                        ccol + 4 * i, G.H, G.W);
        }
        if (cbytes) {  // MPM counts of label 1: sweep t's label (M = x_{t+1}) and sweep t+1's
            const uint4* cs = reinterpret_cast<const uint4*>(cst + 32 * lane);
            uint4 c0 = cs[0], c1 = cs[1];
            uint32_t add[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                add[i] = (p.c.count_enable ? M.w[i] : 0u) + (p.count2 ? O[i] : 0u);  // bytes <= 2
            c0.x += __byte_perm(add[0], 0u, 0x4140); c0.y += __byte_perm(add[0], 0u, 0x4342);
            c0.z += __byte_perm(add[1], 0u, 0x4140); c0.w += __byte_perm(add[1], 0u, 0x4342);
            c1.x += __byte_perm(add[2], 0u, 0x4140); c1.y += __byte_perm(add[2], 0u, 0x4342);
            c1.z += __byte_perm(add[3], 0u, 0x4140); c1.w += __byte_perm(add[3], 0u, 0x4342);
            uint4* cp = reinterpret_cast<uint4*>(co + (long long)(b - rbeg + 4) * G.cpitch);
            cp[0] = c0;
            cp[1] = c1;
        }
        store_row_chunk<HALO, XOFF>(xo + (long long)(b - rbeg + 4) * G.xpitch, O, ccol, 16, k, b,
                                    G.W, G.nchunks, G.rows, G.xpitch, PER, G.self_halo_rows);
    };

    XRow X0, X1, X2;      // x_t rows j-2, j-1, j
    YRow Y0, Y1, Y2;      // x_{t+1} rows j-3, j-2, j-1
    const uint8_t* gprev = nullptr;  // stage holding g row j-2 (still resident: KSTAGES >= 2)
    int s = 0;
    uint32_t phase = 0;
    for (int it = 0; it < nitems; ++it) {
        mbar_wait(&bars[s], phase);
        const uint8_t* st = ring + s * STAGE_BYTES;
        X0 = X1;
        X1 = X2;
        read_x(st, X2);
        if (it >= 2) {
            Y0 = Y1;
            Y1 = Y2;
            sweep_t(rbeg - 3 + it, X0, X1, X2, st + GOFS, Y2);  // x_{t+1} row j-1
        }
        if (it >= 4) sweep_t1(rbeg - 4 + it, Y0, Y1, Y2, gprev, st + COFS);
        // the stage of item it-1 (g row j-2) is no longer needed: refill it
        __syncwarp();
        const int sp = s == 0 ? KSTAGES - 1 : s - 1;
        if (it >= 1 && it - 1 + KSTAGES < nitems && elect_one()) {
            fence_proxy_async();
            issue(it - 1 + KSTAGES, sp);
        }
        gprev = st + GOFS;
        if (++s == KSTAGES) {
            s = 0;
            phase ^= 1u;
        }
    }
}

template <int NB, bool PER>
int launch_t(const Binary2SweepParams& p, int batch, int R, cudaStream_t s) {
    const Geometry& G = p.c.geo;
    static LaunchInfo info[MAX_DEVICES];
    LaunchInfo& li = info[current_device()];
    if (!li.ok.load(std::memory_order_acquire)) {
        std::lock_guard<std::mutex> lock(launch_info_mutex());
        if (!li.ok.load(std::memory_order_relaxed)) {
            cudaError_t e = cudaFuncSetAttribute(sweep_binary2_kernel<NB, PER>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
            if (e != cudaSuccess) return (int)e;
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&li.sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&li.occ, sweep_binary2_kernel<NB, PER>, 32,
                                                          SMEM_BYTES);
            if (li.occ < 1) li.occ = 1;
            li.ok.store(true, std::memory_order_release);
        }
    }
    const int occ = li.occ, sms = li.sms;
    if (R <= 0) {
        const long long segs = (G.nchunks + SEG_CHUNKS - 1) / SEG_CHUNKS;
        const long long target = (long long)sms * occ * PCA_B2_WAVES;
        const long long work = (long long)(p.c.rhi - p.c.rlo) * segs * batch;
        R = (int)((work + target - 1) / target);
        if (R < 4) R = 4;
    }
    const int nrb = (p.c.rhi - p.c.rlo + R - 1) / R;
    if (nrb <= 0) return 0;
    if (nrb > 65535) return (int)cudaErrorInvalidConfiguration;
    dim3 grid((G.nchunks + SEG_CHUNKS - 1) / SEG_CHUNKS, nrb, batch);
    sweep_binary2_kernel<NB, PER><<<grid, 32, SMEM_BYTES, s>>>(p, R);
    return (int)cudaGetLastError();
}

}  // namespace

int launch_sweep_binary2(const Binary2SweepParams& p, int batch, int rows_per_thread, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    const int R = rows_per_thread;
    if (p.c.geo.nbhd == 8)
        return p.c.geo.periodic ? launch_t<8, true>(p, batch, R, s) : launch_t<8, false>(p, batch, R, s);
    return p.c.geo.periodic ? launch_t<4, true>(p, batch, R, s) : launch_t<4, false>(p, batch, R, s);
}

}  // namespace pcab200
