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
// fp64 weights, as in sweep_general.cu.
//
// Thread = 4 consecutive sites of a row (one Philox call).  Moore-8 launches cover only the
// rows of the colour's parity.  A thread rewrites its whole 4-byte word: the bytes of other
// colours are rewritten with the values it read, which no thread of this launch changes, so
// concurrent readers see the same neighbour labels either way.  MPM counts are taken in the
// launch after which a row is final (colours 1 and 3).
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace pcab200 {
namespace {

constexpr int GB_THREADS = 256;
constexpr int GB_WARPS = GB_THREADS / 32;
constexpr unsigned FULL = 0xFFFFFFFFu;

// plain (coherent) loads: the buffer is written by this same launch, so not the read-only path
__device__ __forceinline__ uint32_t ld4(const uint8_t* p) {
    return *reinterpret_cast<const uint32_t*>(p);
}
__device__ __forceinline__ int win_byte(const uint32_t (&w)[3], int pos) {
    return (int)((w[pos >> 2] >> (8 * (pos & 3))) & 0xFFu);
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

template <int NB, bool BIN>
__global__ void __launch_bounds__(GB_THREADS, 2) sweep_gibbs_kernel(const __grid_constant__ GibbsSweepParams p) {
    __shared__ double sA[9];
    __shared__ uint32_t sT[BIN ? GIBBS_THR2 : 1];
    __shared__ GibbsJob s_jobs[GB_WARPS][64];
    __shared__ uint8_t s_res[GB_WARPS][64];
    if (threadIdx.x < 9) sA[threadIdx.x] = p.A[threadIdx.x];
    if (BIN)
        for (int i = threadIdx.x; i < GIBBS_THR2; i += GB_THREADS) sT[i] = p.thr2[i];
    __syncthreads();

    const Geometry& G = p.c.geo;
    const int L = G.levels;
    const int k = p.colour;
    const int nquads = (G.W + 3) >> 2;
    const int qd = blockIdx.x * blockDim.x + threadIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int chain = blockIdx.z;
    const bool active = qd < nquads;
    if (__ballot_sync(FULL, active) == 0) return;
    const uint32_t tagchain = (TAG_GIBBS << 24) | (p.c.chain0 + (uint32_t)chain);
    const unsigned lt = (1u << lane) - 1u;
    GibbsJob* jobs = s_jobs[warp];
    uint8_t* res = s_res[warp];
    // Moore-8: only rows whose global parity is k >> 1 hold colour k
    const int rstep = NB == 8 ? 2 : 1;
    int rfirst = p.c.rlo;
    if (NB == 8 && ((G.row0 + rfirst) & 1) != (k >> 1)) ++rfirst;

    for (int r = rfirst + rstep * (int)blockIdx.y; r < p.c.rhi; r += rstep * (int)gridDim.y) {
        const int grow = G.row0 + r;
        const int c0 = 4 * qd;
        const int nvalid = active ? min(4, G.W - c0) : 0;
        uint32_t up[3] = {0, 0, 0}, mid[3] = {0, 0, 0}, dn[3] = {0, 0, 0}, gword = 0;
        uint4 rnd = make_uint4(0, 0, 0, 0);
        uint8_t* xr = p.c.x_out + chain * G.xchain + (long long)(r + HALO) * G.xpitch + XOFF + c0;
        if (active) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                up[j] = ld4(xr - G.xpitch + 4 * (j - 1));
                mid[j] = ld4(xr + 4 * (j - 1));
                dn[j] = ld4(xr + G.xpitch + 4 * (j - 1));
            }
            gword = __ldg(reinterpret_cast<const uint32_t*>(
                p.c.g + chain * G.gchain + (long long)(r + GHALO) * G.gpitch + XOFF + c0));
            rnd = philox4x32_10(make_uint4((uint32_t)qd, (uint32_t)grow, p.c.t, tagchain), p.c.keys);
        }
        const uint32_t rr[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
        uint32_t outw = mid[1];  // start from the current labels of the 4 sites
        int qpos[4];
        int qbase = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int pos = 4 + b;
            const int col = c0 + b;
            const int colour = NB == 4 ? ((grow + col) & 1) : (((grow & 1) << 1) | (col & 1));
            const bool mine = b < nvalid && colour == k;
            int nb[NB];
            if (NB == 8) {
                nb[0] = win_byte(up, pos - 1); nb[1] = win_byte(up, pos); nb[2] = win_byte(up, pos + 1);
                nb[3] = win_byte(mid, pos - 1); nb[4] = win_byte(mid, pos + 1);
                nb[5] = win_byte(dn, pos - 1); nb[6] = win_byte(dn, pos); nb[7] = win_byte(dn, pos + 1);
            } else {
                nb[0] = win_byte(up, pos); nb[1] = win_byte(mid, pos - 1);
                nb[2] = win_byte(mid, pos + 1); nb[3] = win_byte(dn, pos);
            }
            const int gi = (int)((gword >> (8 * b)) & 0xFFu);
            bool need = false;
            if (BIN) {
                if (mine) {
                    int np = 0, n1 = 0;
#pragma unroll
                    for (int q = 0; q < NB; ++q) {
                        np += nb[q] != 0xFF;
                        n1 += nb[q] == 1;
                    }
                    const int w = rr[b] > sT[(np * 9 + n1) * 2 + gi] ? 1 : 0;
                    outw = (outw & ~(0xFFu << (8 * b))) | ((uint32_t)w << (8 * b));
                }
            } else {
                bool uniform = p.uthr != nullptr && nb[0] < L;
#pragma unroll
                for (int j = 1; j < NB; ++j) uniform = uniform && nb[j] == nb[0];
                if (mine && uniform) {
                    const uint32_t* T = p.uthr + (size_t)(nb[0] * L + gi) * (L - 1);
                    int w = 0;
                    for (int kk = 0; kk < L - 1; ++kk) w += (rr[b] > __ldg(T + kk)) ? 1 : 0;
                    outw = (outw & ~(0xFFu << (8 * b))) | ((uint32_t)w << (8 * b));
                }
                need = mine && !uniform;
            }
            const unsigned m = __ballot_sync(FULL, need);
            qpos[b] = need ? qbase + __popc(m & lt) : -1;
            if (need) {
                GibbsJob jb;
                jb.nb_lo = jb.nb_hi = 0u;
#pragma unroll
                for (int q = 0; q < NB; ++q) {
                    if (q < 4) jb.nb_lo |= (uint32_t)nb[q] << (8 * q);
                    else jb.nb_hi |= (uint32_t)nb[q] << (8 * (q - 4));
                }
                jb.g = (uint32_t)gi;
                jb.r = rr[b];
                jobs[qpos[b]] = jb;
            }
            qbase += __popc(m);
        }
        if (!BIN) {
            __syncwarp();
            for (int i = lane; i < qbase; i += 32) res[i] = (uint8_t)gibbs_fp64<NB>(p, sA, jobs[i]);
            __syncwarp();
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (qpos[b] >= 0) outw = (outw & ~(0xFFu << (8 * b))) | ((uint32_t)res[qpos[b]] << (8 * b));
            __syncwarp();
        }
        if (!active) continue;

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
        if (p.c.count_enable) {
            uint16_t* cp = p.c.counts + chain * G.cchain + (long long)r * G.cpitch + c0;
            for (int b = 0; b < nvalid; ++b) {
                const int w = (int)((outw >> (8 * b)) & 0xFFu);
                if (L == 2) cp[b] += (uint16_t)w;
                else cp[(long long)w * G.cplane + b] += 1;
            }
        }
    }
}

}  // namespace

int launch_sweep_gibbs(const GibbsSweepParams& p, int batch, void* stream) {
    const Geometry& G = p.c.geo;
    const int nquads = (G.W + 3) / 4;
    int nr = p.c.rhi - p.c.rlo;
    if (G.nbhd == 8) nr = (nr + 1) / 2;
    if (nr <= 0) return 0;
    dim3 grid((nquads + GB_THREADS - 1) / GB_THREADS, nr < 65535 ? nr : 65535, batch);
    cudaStream_t s = (cudaStream_t)stream;
    const bool bin = G.levels == 2;
    if (G.nbhd == 8) {
        if (bin) sweep_gibbs_kernel<8, true><<<grid, GB_THREADS, 0, s>>>(p);
        else sweep_gibbs_kernel<8, false><<<grid, GB_THREADS, 0, s>>>(p);
    } else {
        if (bin) sweep_gibbs_kernel<4, true><<<grid, GB_THREADS, 0, s>>>(p);
        else sweep_gibbs_kernel<4, false><<<grid, GB_THREADS, 0, s>>>(p);
    }
    return (int)cudaGetLastError();
}

}  // namespace pcab200
