// sweep_general.cu -- one synchronous lazy-PCA sweep for any number of levels (2..255).
//
// Uniform neighbourhood (all NB neighbours carry the same label s*, ~75-85% of the sites of
// a restored MRF image): p_i depends only on (s*, g_i, x_i), so the host tabulates for the
// current beta the integer thresholds T_k = ceil(F_k 2^32) - 1 of the cumulative
// probabilities (fp64, accumulated exactly as the oracle does, levels <= 16) and the new
// label is #{k : r > T_k} -- integer-exact, like the binary kernel.
//
// Otherwise, per site i (PAPER.md:462-477 with R1), in fp64:
//   w_s = e^{a n_i(s)} * e^{-b (lum g_i - lum s)^2} * e^{-c 1{s != x_i}}
//       = A[n_i(s)] * D[g_i][s] * (s == x_i ? 1 : Cw)
// (the factorised form of exp(E_i(s)); A, D, Cw tabulated on the host in fp64),
// Z = sum_s w_s; the new label is min{k < l-1 : u Z < sum_{s<=k} w_s}, else l-1 (R14),
// with u = r 2^-32 from the site's Philox word.  Rounding differs from the oracle's
// exp(E - max E)/Z only in the last bits, so decisions can differ only when u lies within
// ~1e-15 of a cumulative probability (an allowed near-tie, R19).
//
// One thread = 4 consecutive sites of a row (one Philox4x32-10 call).  The 3x12-byte
// neighbourhood window is fetched as 9 aligned 32-bit loads (L1-resident across the warp).
// The free-boundary sentinel 0xFF never equals a label, so n_i(s) needs no position test.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace pcab200 {
namespace {

__device__ __forceinline__ uint32_t ldg4(const uint8_t* p) {
    return __ldg(reinterpret_cast<const uint32_t*>(p));
}

// byte at window position pos (0..11) of a 3-word row window
__device__ __forceinline__ int win_byte(const uint32_t (&w)[3], int pos) {
    return (int)((w[pos >> 2] >> (8 * (pos & 3))) & 0xFFu);
}

template <int NB>
__global__ void __launch_bounds__(256)
    sweep_general_kernel(const __grid_constant__ GeneralSweepParams p) {
    __shared__ double sA[9];
    if (threadIdx.x < 9) sA[threadIdx.x] = p.A[threadIdx.x];
    __syncthreads();

    const Geometry& G = p.c.geo;
    const int L = G.levels;
    const int nquads = (G.W + 3) >> 2;
    const int qd = blockIdx.x * blockDim.x + threadIdx.x;
    const int chain = blockIdx.z;
    if (qd >= nquads) return;
    const uint32_t tagchain = (TAG_PCA << 24) | (p.c.chain0 + (uint32_t)chain);
    const double Cw = p.Cw;
    const double* __restrict__ dtab = p.dtab;

    for (int r = p.c.rlo + blockIdx.y; r < p.c.rhi; r += gridDim.y) {
        const int grow = G.row0 + r;
        const uint8_t* xr = p.c.x_in + chain * G.xchain + (long long)(r + 1) * G.xpitch + XOFF +
                            4 * qd;
        uint32_t up[3], mid[3], dn[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            up[j] = ldg4(xr - G.xpitch + 4 * (j - 1));
            mid[j] = ldg4(xr + 4 * (j - 1));
            dn[j] = ldg4(xr + G.xpitch + 4 * (j - 1));
        }
        const uint32_t gword = ldg4(p.c.g + chain * G.gchain + (long long)r * G.gpitch + 4 * qd);
        const uint4 rnd = philox4x32_10(make_uint4((uint32_t)qd, (uint32_t)grow, p.c.t, tagchain),
                                        p.c.keys);
        const uint32_t rr[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
        uint32_t outw = 0u;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int pos = 4 + b;  // window position of this site
            int nb[NB];
            if (NB == 8) {
                nb[0] = win_byte(up, pos - 1); nb[1] = win_byte(up, pos); nb[2] = win_byte(up, pos + 1);
                nb[3] = win_byte(mid, pos - 1); nb[4] = win_byte(mid, pos + 1);
                nb[5] = win_byte(dn, pos - 1); nb[6] = win_byte(dn, pos); nb[7] = win_byte(dn, pos + 1);
            } else {
                nb[0] = win_byte(up, pos); nb[1] = win_byte(mid, pos - 1);
                nb[2] = win_byte(mid, pos + 1); nb[3] = win_byte(dn, pos);
            }
            const int xi = win_byte(mid, pos);
            const int gi = (int)((gword >> (8 * b)) & 0xFFu);
            bool uniform = p.uthr != nullptr && xi < L && nb[0] < L;
#pragma unroll
            for (int j = 1; j < NB; ++j) uniform = uniform && nb[j] == nb[0];
            if (uniform) {
                // every neighbour carries s* = nb[0] (so all NB exist): integer thresholds
                const uint32_t* T = p.uthr + (size_t)((nb[0] * L + gi) * L + xi) * (L - 1);
                int w = 0;
                for (int k = 0; k < L - 1; ++k) w += (rr[b] > __ldg(T + k)) ? 1 : 0;
                outw |= (uint32_t)w << (8 * b);
                continue;
            }
            const double* Drow = dtab + (size_t)(gi < L ? gi : 0) * L;
            double Z = 0.0;
            for (int s = 0; s < L; ++s) {
                int n = 0;
#pragma unroll
                for (int j = 0; j < NB; ++j) n += (nb[j] == s);
                Z += sA[n] * __ldg(Drow + s) * (s == xi ? 1.0 : Cw);
            }
            const double u = (double)rr[b] * (1.0 / 4294967296.0);
            int w = L - 1;
            if (Z >= 1e-290 && Z <= 1e290) {
                const double target = u * Z;
                double F = 0.0;
                for (int s = 0; s < L - 1; ++s) {
                    int n = 0;
#pragma unroll
                    for (int j = 0; j < NB; ++j) n += (nb[j] == s);
                    F += sA[n] * __ldg(Drow + s) * (s == xi ? 1.0 : Cw);
                    if (target < F) { w = s; break; }
                }
            } else {
                // Rare slow path (extreme beta, q or sigma: the factorised weights under- or
                // overflow): E_s = a n_s - b d_s^2 - c 1{s != x_i}, softmax with max subtracted.
                const double lg = (double)gi / (double)(L - 1);
                double Emax = -INFINITY;
                for (int s = 0; s < L; ++s) {
                    int n = 0;
#pragma unroll
                    for (int j = 0; j < NB; ++j) n += (nb[j] == s);
                    const double d = lg - (double)s / (double)(L - 1);
                    const double E = p.coef_a * n - p.coef_b * d * d - (s != xi ? p.coef_c : 0.0);
                    Emax = fmax(Emax, E);
                }
                double Zs = 0.0;
                for (int s = 0; s < L; ++s) {
                    int n = 0;
#pragma unroll
                    for (int j = 0; j < NB; ++j) n += (nb[j] == s);
                    const double d = lg - (double)s / (double)(L - 1);
                    Zs += exp(p.coef_a * n - p.coef_b * d * d - (s != xi ? p.coef_c : 0.0) - Emax);
                }
                const double target = u * Zs;
                double F = 0.0;
                for (int s = 0; s < L - 1; ++s) {
                    int n = 0;
#pragma unroll
                    for (int j = 0; j < NB; ++j) n += (nb[j] == s);
                    const double d = lg - (double)s / (double)(L - 1);
                    F += exp(p.coef_a * n - p.coef_b * d * d - (s != xi ? p.coef_c : 0.0) - Emax);
                    if (target < F) { w = s; break; }
                }
            }
            outw |= (uint32_t)w << (8 * b);
        }
        const int c0 = 4 * qd;
        const int nvalid = min(4, G.W - c0);
        uint8_t* op = p.c.x_out + chain * G.xchain + (long long)(r + 1) * G.xpitch + XOFF + c0;
        auto store = [&](uint8_t* dst) {
            if (nvalid == 4) *reinterpret_cast<uint32_t*>(dst) = outw;
            else for (int b = 0; b < nvalid; ++b) dst[b] = (uint8_t)(outw >> (8 * b));
            if (G.periodic) {
                if (c0 == 0) dst[G.W] = (uint8_t)outw;
                if (c0 + nvalid == G.W) dst[-c0 - 1] = (uint8_t)(outw >> (8 * (nvalid - 1)));
            }
        };
        store(op);
        if (G.periodic && G.self_halo_rows && (grow == 0 || grow == G.H - 1))
            store(op + (grow == 0 ? 1LL : -1LL) * (long long)G.rows * G.xpitch);
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

int launch_sweep_general(const GeneralSweepParams& p, int batch, void* stream) {
    const Geometry& G = p.c.geo;
    const int nquads = (G.W + 3) / 4;
    dim3 block(nquads >= 256 ? 256 : ((nquads + 31) / 32) * 32);
    const int nr = p.c.rhi - p.c.rlo;
    if (nr <= 0) return 0;
    dim3 grid((nquads + block.x - 1) / block.x, nr < 65535 ? nr : 65535, batch);
    cudaStream_t s = (cudaStream_t)stream;
    if (G.nbhd == 8) sweep_general_kernel<8><<<grid, block, 0, s>>>(p);
    else sweep_general_kernel<4><<<grid, block, 0, s>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace pcab200
