// aux.cu -- layout kernels and the fused estimate / metric reductions.
//
//  * pack_state / unpack_state: dense [batch][rows][W] <-> padded x buffer (+ torus halos).
//  * mpm / marginals / cm: the posterior-marginal estimates from the counts (R15):
//    MPM_i = argmax_k count_i[k] (ties to the lowest k); marginal = count/N_samp;
//    CM_i = sum_k lum(k) count_i[k]/N_samp (conditional mean).
//  * metric_sums: one pass over truth and the LAST or MPM estimate, accumulating the exact
//    integer sums of PAPER.md:516-534's statistics (sum (x-y)^2, sum x, sum y, sum x^2,
//    sum y^2, sum xy, max x) per chain; block reduction, then one atomic per block per sum.
//    The finalisation variant does LAST and MPM (and stores the MPM image) in one pass.
//  * ssim_windowed: mean SSIM over every 7x7 window (R16's secondary metric): exact integer
//    window sums, fp64 per window, deterministic fixed-order per-block partial sums.
//
// All of them move 16 sites per thread with 16-byte vector accesses when the rows are
// 16-byte aligned (W % 16 == 0), and fall back to per-byte access otherwise.  Grid: x over
// 16-site chunks of a row, y over rows (grid-stride), z over chains.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace pcab200 {
namespace {

constexpr int TPB = 128;

// any byte of w >= lv (levels replicated in every byte)?
__device__ __forceinline__ bool any_ge(uint32_t w, uint32_t lv4) { return __vcmpgeu4(w, lv4) != 0; }

__device__ __forceinline__ uint32_t byte_of(const uint4& v, int j) {
    const uint32_t w = (j < 8) ? ((j < 4) ? v.x : v.y) : ((j < 12) ? v.z : v.w);
    return (w >> (8 * (j & 3))) & 0xFFu;
}

// load 16 bytes of a row starting at column c0 (n valid bytes, rest 0)
__device__ __forceinline__ uint4 load16(const uint8_t* row, int c0, int n, bool vec) {
    if (vec && n == 16) return *reinterpret_cast<const uint4*>(row + c0);
    uint32_t w[4] = {0, 0, 0, 0};
    for (int j = 0; j < n; ++j) w[j >> 2] |= (uint32_t)row[c0 + j] << (8 * (j & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ __forceinline__ void store16(uint8_t* row, int c0, int n, bool vec, const uint4& v) {
    if (vec && n == 16) {
        *reinterpret_cast<uint4*>(row + c0) = v;
        return;
    }
    for (int j = 0; j < n; ++j) row[c0 + j] = (uint8_t)byte_of(v, j);
}

// Rows [0, rows) of a dense / pitched source -> a padded buffer (row j at (j+halo)*dpitch,
// data column c at XOFF + c), checking every value < levels; on a torus also the column pads
// and, when the context owns the whole torus, the `halo` wrapped rows (kernels.cuh layout).
__global__ void __launch_bounds__(TPB) pack_padded_kernel(Geometry G, const uint8_t* __restrict__ src,
                                                          int src_pitch, long long src_chain,
                                                          uint8_t* __restrict__ dst, long long dpitch,
                                                          long long dchain, int halo, int* bad,
                                                          uint8_t* __restrict__ dst2,
                                                          long long dpitch2, long long dchain2,
                                                          int halo2) {
    const int chain = blockIdx.z;
    const int k = blockIdx.x * TPB + threadIdx.x;  // chunk
    const int c0 = 16 * k;
    if (c0 >= G.W) return;
    const int n = min(16, G.W - c0);
    const bool vec = ((src_pitch | (int)((uintptr_t)src & 15)) & 15) == 0 && (src_chain & 15) == 0;
    const uint32_t lv4 = 0x01010101u * (uint32_t)G.levels;
    int found = 0;
    for (int r = blockIdx.y; r < G.rows; r += gridDim.y) {
        const uint8_t* s = src + chain * src_chain + (long long)r * src_pitch;
        const uint4 v = load16(s, c0, n, vec);
        uint32_t m[4] = {0, 0, 0, 0};  // valid-byte masks
        for (int j = 0; j < n; ++j) m[j >> 2] |= 0xFFu << (8 * (j & 3));
        found |= any_ge(v.x & m[0], lv4) | any_ge(v.y & m[1], lv4) | any_ge(v.z & m[2], lv4) |
                 any_ge(v.w & m[3], lv4);
        auto put = [&](uint8_t* rp) {
            store16(rp + XOFF, c0, n, true, v);
            if (G.periodic) {
                if ((G.W & 15) == 0) {
                    if (k == 0) *reinterpret_cast<uint4*>(rp + XOFF + G.W) = v;
                    if (k == G.nchunks - 1) *reinterpret_cast<uint4*>(rp + XOFF - 16) = v;
                } else {
                    if (k == 0) rp[XOFF + G.W] = (uint8_t)byte_of(v, 0);
                    if (k == G.nchunks - 1) rp[XOFF - 1] = (uint8_t)byte_of(v, n - 1);
                }
            }
        };
        auto emit = [&](uint8_t* base, long long pitch, long long cstride, int h) {
            uint8_t* rowp = base + chain * cstride + (long long)(r + h) * pitch;
            put(rowp);
            if (G.periodic && G.self_halo_rows) {
                if (r < h) put(rowp + (long long)G.rows * pitch);
                if (r >= G.rows - h) put(rowp - (long long)G.rows * pitch);
            }
        };
        emit(dst, dpitch, dchain, halo);
        if (dst2) emit(dst2, dpitch2, dchain2, halo2);
    }
    if (found) atomicOr(bad, 1);
}

__global__ void __launch_bounds__(TPB) unpack_state_kernel(Geometry G, const uint8_t* __restrict__ xbuf,
                                                           uint8_t* __restrict__ dense) {
    const int chain = blockIdx.z;
    const int c0 = 16 * (blockIdx.x * TPB + threadIdx.x);
    if (c0 >= G.W) return;
    const int n = min(16, G.W - c0);
    const bool vec = (G.W & 15) == 0 && ((uintptr_t)dense & 15) == 0;
    for (int r = blockIdx.y; r < G.rows; r += gridDim.y) {
        const uint8_t* s = xbuf + chain * G.xchain + (long long)(r + HALO) * G.xpitch + XOFF;
        uint8_t* d = dense + ((long long)chain * G.rows + r) * G.W;
        store16(d, c0, n, vec, load16(s, c0, n, true));
    }
}

__global__ void check_levels_kernel(const uint8_t* __restrict__ p, size_t n, int levels, int* bad) {
    const uint32_t lv4 = 0x01010101u * (uint32_t)levels;
    int found = 0;
    const size_t nv = n / 16;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < nv;
         i += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = reinterpret_cast<const uint4*>(p)[i];
        found |= any_ge(v.x, lv4) | any_ge(v.y, lv4) | any_ge(v.z, lv4) | any_ge(v.w, lv4);
    }
    if (blockIdx.x == 0)
        for (size_t i = nv * 16 + threadIdx.x; i < n; i += blockDim.x) found |= p[i] >= levels;
    if (found) atomicOr(bad, 1);
}

// MPM labels of the 16 sites starting at column c0 of row r (ties -> lowest label)
__device__ __forceinline__ uint4 mpm16(const Geometry& G, const uint16_t* cchain, int r, int c0,
                                       int nsamp) {
    const uint16_t* cp = cchain + (long long)r * G.cpitch + c0;  // cpitch = 16*nchunks: in bounds
    uint32_t out[4] = {0, 0, 0, 0};
    if (G.levels == 2) {
        const uint4 a = reinterpret_cast<const uint4*>(cp)[0];
        const uint4 b = reinterpret_cast<const uint4*>(cp)[1];
        const uint32_t cw[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int c1 = (int)((cw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu);
            out[j >> 2] |= (uint32_t)(2 * c1 > nsamp) << (8 * (j & 3));
        }
    } else {
        uint32_t best[16], bestc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) { best[j] = 0; bestc[j] = 0; }
        for (int k = 0; k < G.levels; ++k) {
            const uint4* pk = reinterpret_cast<const uint4*>(cp + (long long)k * G.cplane);
            const uint4 a = pk[0], b = pk[1];
            const uint32_t cw[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const uint32_t v = (cw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
                if (k == 0 || v > bestc[j]) { bestc[j] = v; best[j] = (uint32_t)k; }
            }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) out[j >> 2] |= best[j] << (8 * (j & 3));
    }
    return make_uint4(out[0], out[1], out[2], out[3]);
}

__global__ void __launch_bounds__(TPB) mpm_kernel(Geometry G, const uint16_t* __restrict__ counts,
                                                  int nsamp, uint8_t* __restrict__ out) {
    const int chain = blockIdx.z;
    const int c0 = 16 * (blockIdx.x * TPB + threadIdx.x);
    if (c0 >= G.W) return;
    const int n = min(16, G.W - c0);
    const bool vec = (G.W & 15) == 0 && ((uintptr_t)out & 15) == 0;
    const uint16_t* cc = counts + chain * G.cchain;
    for (int r = blockIdx.y; r < G.rows; r += gridDim.y)
        store16(out + ((long long)chain * G.rows + r) * G.W, c0, n, vec, mpm16(G, cc, r, c0, nsamp));
}

// One label plane k (or the conditional mean when k < 0) for every chain:
// out[chain * out_chain_stride + r * W + c].
__global__ void marginals_kernel(Geometry G, const uint16_t* __restrict__ counts, int nsamp,
                                 float* __restrict__ out, long long out_chain_stride, int k) {
    const int chain = blockIdx.z;
    const double inv = 1.0 / (double)nsamp;
    for (int r = blockIdx.y; r < G.rows; r += gridDim.y)
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < G.W; c += gridDim.x * blockDim.x) {
            const uint16_t* cc = counts + chain * G.cchain + (long long)r * G.cpitch;
            float* o = out + chain * out_chain_stride + (long long)r * G.W;
            double v;
            if (G.levels == 2) {
                const int c1 = cc[c];
                v = (k == 0) ? (double)(nsamp - c1) : (double)c1;  // CM = lum(1) * c1 for l = 2
            } else if (k >= 0) {
                v = (double)cc[(long long)k * G.cplane + c];
            } else {
                v = 0.0;
                for (int s = 0; s < G.levels; ++s)
                    v += ((double)s / (double)(G.levels - 1)) * (double)cc[(long long)s * G.cplane + c];
            }
            o[c] = (float)(v * inv);
        }
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// BOTH: the finalisation pass (SURVEY 8(a) a8 + a9 fused): one read of truth, x and the
// counts gives the MPM image (optional store) and the sums of LAST and of MPM.
template <bool BOTH>
__global__ void __launch_bounds__(TPB) metric_sums_kernel(const MetricParams p) {
    constexpr int NS = BOTH ? 12 : 6;
    const Geometry& G = p.geo;
    const int chain = blockIdx.z;
    const int c0 = 16 * (blockIdx.x * TPB + threadIdx.x);
    const int n = c0 < G.W ? min(16, G.W - c0) : 0;
    const bool vec = (G.W & 15) == 0 && ((uintptr_t)p.truth & 15) == 0;
    const bool ovec = (G.W & 15) == 0 && ((uintptr_t)p.mpm_out & 15) == 0;
    const uint8_t* truth = p.truth + (long long)chain * G.rows * G.W;
    const uint8_t* xb = p.x + chain * G.xchain;
    const uint16_t* cc = p.counts + chain * G.cchain;
    unsigned long long s[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = 0;
    uint32_t mx4 = 0;  // bytewise max of the truth
    if (n > 0) {
        for (int r = blockIdx.y; r < G.rows; r += gridDim.y) {
            const uint4 tv = load16(truth + (long long)r * G.W, c0, n, vec);
            uint4 yv[2];
            if (BOTH) {
                yv[0] = load16(xb + (long long)(r + HALO) * G.xpitch + XOFF, c0, n, true);
                yv[1] = mpm16(G, cc, r, c0, p.nsamp);
                if (p.mpm_out) store16(p.mpm_out + ((long long)chain * G.rows + r) * G.W, c0, n, ovec, yv[1]);
            } else {
                yv[0] = p.kind == 0 ? load16(xb + (long long)(r + HALO) * G.xpitch + XOFF, c0, n, true)
                                    : mpm16(G, cc, r, c0, p.nsamp);
            }
            // 16 sites by 4-byte dot products (IDP.4A); bytes past the row are masked to 0 in
            // both images and add nothing.  sum (x-y)^2 = sum x^2 + sum y^2 - 2 sum xy, exactly.
            uint32_t msk[4] = {~0u, ~0u, ~0u, ~0u};
            if (n < 16) {
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int vb = min(max(n - 4 * i, 0), 4);
                    msk[i] = vb == 4 ? ~0u : ((1u << (8 * vb)) - 1u);
                }
            }
            const uint32_t tw[4] = {tv.x & msk[0], tv.y & msk[1], tv.z & msk[2], tv.w & msk[3]};
            if (BOTH && p.mpm_bits) {  // 16 labels 0/1 -> 16 bits, site c0 + j at bit j
                const uint32_t yw[4] = {yv[1].x & msk[0], yv[1].y & msk[1], yv[1].z & msk[2],
                                        yv[1].w & msk[3]};
                uint32_t bits = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i)  // byte k's bit 0 lands on bit 24 + k, no carries
                    bits |= (((yw[i] & 0x01010101u) * 0x01020408u) >> 24) << (4 * i);
                uint8_t* bp = p.mpm_bits + ((long long)chain * G.rows + r) * ((G.W + 7) >> 3) + (c0 >> 3);
                bp[0] = (uint8_t)bits;
                if (n > 8) bp[1] = (uint8_t)(bits >> 8);
            }
            uint32_t sx = 0, sxx = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                sx = __dp4a(tw[i], 0x01010101u, sx);
                sxx = __dp4a(tw[i], tw[i], sxx);
                mx4 = __vmaxu4(mx4, tw[i]);
            }
#pragma unroll
            for (int e = 0; e < (BOTH ? 2 : 1); ++e) {
                const uint32_t yw[4] = {yv[e].x & msk[0], yv[e].y & msk[1], yv[e].z & msk[2], yv[e].w & msk[3]};
                uint32_t sy = 0, syy = 0, sxy = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    sy = __dp4a(yw[i], 0x01010101u, sy);
                    syy = __dp4a(yw[i], yw[i], syy);
                    sxy = __dp4a(tw[i], yw[i], sxy);
                }
                s[6 * e + 0] += sxx + syy - 2u * sxy;
                s[6 * e + 1] += sx;
                s[6 * e + 2] += sy;
                s[6 * e + 3] += sxx;
                s[6 * e + 4] += syy;
                s[6 * e + 5] += sxy;
            }
        }
    }
    uint32_t mx = max(max(mx4 & 0xFFu, (mx4 >> 8) & 0xFFu), max((mx4 >> 16) & 0xFFu, mx4 >> 24));
    __shared__ unsigned long long red[TPB / 32][NS + 1];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < NS; ++k) s[k] = warp_sum(s[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    if (lane == 0) {
        for (int k = 0; k < NS; ++k) red[warp][k] = s[k];
        red[warp][NS] = mx;
    }
    __syncthreads();
    // slot layout per estimate: 0..5 sums, 6 max truth, 7 site count
    if (threadIdx.x <= NS) {
        unsigned long long acc = 0;
        for (int w = 0; w < TPB / 32; ++w) {
            const unsigned long long v = red[w][threadIdx.x];
            acc = threadIdx.x == NS ? (v > acc ? v : acc) : acc + v;
        }
        unsigned long long* dst = p.sums + chain * (BOTH ? 16 : 8);
        if (threadIdx.x == NS) {
            atomicMax(dst + 6, acc);
            if (BOTH) atomicMax(dst + 14, acc);
        } else {
            const int e = threadIdx.x / 6, k = threadIdx.x % 6;
            atomicAdd(dst + 8 * e + k, acc);
        }
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
        atomicAdd(p.sums + chain * (BOTH ? 16 : 8) + 7, (unsigned long long)G.rows * G.W);
        if (BOTH) atomicAdd(p.sums + chain * 16 + 15, (unsigned long long)G.rows * G.W);
    }
}

// x: 16-site chunks of a row; y: rows, grid-stride, sized for ~8 resident blocks per SM
inline dim3 chunk_grid(const Geometry& G, int batch, int max_rows = 2048) {
    const int nchunks = (G.W + 15) / 16;
    const int gx = (nchunks + TPB - 1) / TPB;
    int gy = G.rows < max_rows ? G.rows : max_rows;
    if (gy < 1) gy = 1;
    return dim3(gx, gy, batch);
}

// Windowed SSIM (Wang et al.; PAPER.md:527-534 read through R16): thread = one window
// column c0, block = SSIM_TPB columns x SSIM_ROWS_PER_BLOCK window rows.  The 7x7 sums
// (x, y, x^2, y^2, xy over level indices) slide down the rows: add the entering row's
// 7-column sums, subtract the leaving row's; all integer, so every window's moments are
// exact and only the per-window SSIM and the final mean round.
struct WinSums {
    int x, y, xx, yy, xy;
};
__device__ __forceinline__ void row7(const uint8_t* xr, const uint8_t* yr, int sign, WinSums& S) {
    int x = 0, y = 0, xx = 0, yy = 0, xy = 0;
#pragma unroll
    for (int c = 0; c < SSIM_WIN; ++c) {
        const int a = xr[c], b = yr[c];
        x += a; y += b; xx += a * a; yy += b * b; xy += a * b;
    }
    S.x += sign * x; S.y += sign * y; S.xx += sign * xx; S.yy += sign * yy; S.xy += sign * xy;
}

__global__ void __launch_bounds__(SSIM_TPB) ssim_windowed_kernel(const WinSsimParams p) {
    const int nwr = p.H - SSIM_WIN + 1, nwc = p.W - SSIM_WIN + 1;
    const int c0 = blockIdx.x * SSIM_TPB + threadIdx.x;
    const int rb = blockIdx.y * SSIM_ROWS_PER_BLOCK;
    const int re = min(rb + SSIM_ROWS_PER_BLOCK, nwr);
    const uint8_t* X = p.x + (long long)blockIdx.z * p.xchain + c0;
    const uint8_t* Y = p.y + (long long)blockIdx.z * p.ychain + c0;
    const double L1 = (double)(p.levels - 1);
    const double n = (double)(SSIM_WIN * SSIM_WIN);
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    double acc = 0.0;
    if (c0 < nwc) {
        WinSums S = {0, 0, 0, 0, 0};
        for (int r = rb; r < rb + SSIM_WIN; ++r)
            row7(X + (long long)r * p.xpitch, Y + (long long)r * p.ypitch, 1, S);
        for (int r0 = rb;;) {
            // means S/(n L1); sample (co)variances (n S2 - S S')/(n (n-1) L1^2), exact numerators
            const double mx = (double)S.x / (n * L1), my = (double)S.y / (n * L1);
            const double den = n * (n - 1.0) * L1 * L1;
            const double vx = (double)(SSIM_WIN * SSIM_WIN * (long long)S.xx - (long long)S.x * S.x) / den;
            const double vy = (double)(SSIM_WIN * SSIM_WIN * (long long)S.yy - (long long)S.y * S.y) / den;
            const double vxy = (double)(SSIM_WIN * SSIM_WIN * (long long)S.xy - (long long)S.x * S.y) / den;
            acc += ((2.0 * mx * my + c1) * (2.0 * vxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2));
            if (++r0 >= re) break;
            row7(X + (long long)(r0 + SSIM_WIN - 1) * p.xpitch, Y + (long long)(r0 + SSIM_WIN - 1) * p.ypitch, 1, S);
            row7(X + (long long)(r0 - 1) * p.xpitch, Y + (long long)(r0 - 1) * p.ypitch, -1, S);
        }
    }
    // fixed-order reduction: warp butterfly, then warp 0 adds the warp totals in order
    __shared__ double s_w[SSIM_TPB / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < SSIM_TPB / 32; ++w) t += s_w[w];
        p.partial[((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = t;
    }
}

// Sites whose label differs between two padded state buffers (x_t and x_{t-1}), per chain:
// 16 sites per thread, nonzero bytes of the XOR counted with a SWAR test and popc.
__global__ void __launch_bounds__(TPB) changed_kernel(Geometry G, const uint8_t* __restrict__ xa,
                                                      const uint8_t* __restrict__ xb,
                                                      unsigned long long* __restrict__ out) {
    const int chain = blockIdx.z;
    const int c0 = 16 * (blockIdx.x * TPB + threadIdx.x);
    const int n = c0 < G.W ? min(16, G.W - c0) : 0;
    unsigned long long cnt = 0;
    if (n > 0) {
        const uint8_t* a = xa + chain * G.xchain + XOFF;
        const uint8_t* b = xb + chain * G.xchain + XOFF;
        for (int r = blockIdx.y; r < G.rows; r += gridDim.y) {
            const long long off = (long long)(r + HALO) * G.xpitch;
            const uint4 va = load16(a + off, c0, n, true), vb = load16(b + off, c0, n, true);
            const uint32_t z[4] = {va.x ^ vb.x, va.y ^ vb.y, va.z ^ vb.z, va.w ^ vb.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
                cnt += __popc((((z[i] & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | z[i]) & 0x80808080u);
        }
    }
    cnt = warp_sum(cnt);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out + chain, cnt);
}

// Bit-packed binary images (packed_io): rows of pb = ceil(W/8) bytes, column c at bit c%8 of
// byte c/8.  One thread per packed byte.
__global__ void unpack_bits_kernel(const uint8_t* __restrict__ bits, uint8_t* __restrict__ dense,
                                   int W, long long nrows) {
    const int pb = (W + 7) >> 3;
    const long long n = nrows * pb;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / pb;
        const int k = (int)(i - row * pb);
        const uint32_t v = bits[i];
        uint8_t* d = dense + row * W + 8 * k;
        const int m = min(8, W - 8 * k);
        if (m == 8 && (((uintptr_t)d) & 7) == 0) {
            const uint32_t lo = ((v & 0xFu) * 0x00204081u) & 0x01010101u;
            const uint32_t hi = ((v >> 4) * 0x00204081u) & 0x01010101u;
            *reinterpret_cast<uint2*>(d) = make_uint2(lo, hi);
        } else {
            for (int j = 0; j < m; ++j) d[j] = (uint8_t)((v >> j) & 1u);
        }
    }
}

__global__ void pack_bits_kernel(const uint8_t* __restrict__ dense, uint8_t* __restrict__ bits, int W,
                                 long long nrows) {
    const int pb = (W + 7) >> 3;
    const long long n = nrows * pb;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / pb;
        const int k = (int)(i - row * pb);
        const uint8_t* d = dense + row * W + 8 * k;
        const int m = min(8, W - 8 * k);
        uint32_t v = 0;
        for (int j = 0; j < m; ++j) v |= (uint32_t)(d[j] & 1u) << j;
        bits[i] = (uint8_t)v;
    }
}

__global__ void param_table_kernel(const __grid_constant__ ParamTable t, int n, uint32_t* dst) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = t.v[i];
}

}  // namespace

int launch_param_table(const ParamTable& t, int n, uint32_t* dst, void* stream) {
    if (n < 0 || n > PARAM_TABLE_MAX) return (int)cudaErrorInvalidValue;
    param_table_kernel<<<1, 128, 0, (cudaStream_t)stream>>>(t, n, dst);
    return (int)cudaGetLastError();
}

int launch_unpack_bits(const uint8_t* bits, uint8_t* dense, int W, long long nrows, void* stream) {
    const long long n = nrows * ((W + 7) / 8);
    if (n <= 0) return 0;
    const int blocks = (int)((n + 255) / 256 < 65535 ? (n + 255) / 256 : 65535);
    unpack_bits_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(bits, dense, W, nrows);
    return (int)cudaGetLastError();
}

int launch_pack_bits(const uint8_t* dense, uint8_t* bits, int W, long long nrows, void* stream) {
    const long long n = nrows * ((W + 7) / 8);
    if (n <= 0) return 0;
    const int blocks = (int)((n + 255) / 256 < 65535 ? (n + 255) / 256 : 65535);
    pack_bits_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(dense, bits, W, nrows);
    return (int)cudaGetLastError();
}

int launch_pack_state(const Geometry& G, const uint8_t* src, int src_pitch, long long src_chain,
                      uint8_t* xbuf, int batch, int* bad, void* stream) {
    pack_padded_kernel<<<chunk_grid(G, batch), TPB, 0, (cudaStream_t)stream>>>(
        G, src, src_pitch, src_chain, xbuf, G.xpitch, G.xchain, HALO, bad, nullptr, 0, 0, 0);
    return (int)cudaGetLastError();
}

int launch_pack_g(const Geometry& G, const uint8_t* src, int src_pitch, long long src_chain,
                  uint8_t* gbuf, int batch, int* bad, void* stream, uint8_t* xbuf) {
    pack_padded_kernel<<<chunk_grid(G, batch), TPB, 0, (cudaStream_t)stream>>>(
        G, src, src_pitch, src_chain, gbuf, G.gpitch, G.gchain, GHALO, bad, xbuf, G.xpitch,
        G.xchain, HALO);
    return (int)cudaGetLastError();
}

int launch_unpack_state(const Geometry& G, const uint8_t* xbuf, uint8_t* dense, int batch,
                        void* stream) {
    unpack_state_kernel<<<chunk_grid(G, batch), TPB, 0, (cudaStream_t)stream>>>(G, xbuf, dense);
    return (int)cudaGetLastError();
}

int launch_check_levels(const uint8_t* p, size_t n, int levels, int* bad, void* stream) {
    size_t blocks = (n / 16 + 255) / 256;
    if (blocks > 2048) blocks = 2048;
    if (blocks == 0) blocks = 1;
    check_levels_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(p, n, levels, bad);
    return (int)cudaGetLastError();
}

int launch_changed(const Geometry& G, const uint8_t* xa, const uint8_t* xb,
                   unsigned long long* out, int batch, void* stream) {
    changed_kernel<<<chunk_grid(G, batch, 512), TPB, 0, (cudaStream_t)stream>>>(G, xa, xb, out);
    return (int)cudaGetLastError();
}

int launch_mpm(const Geometry& G, const uint16_t* counts, int nsamp, uint8_t* out, int batch,
               void* stream) {
    mpm_kernel<<<chunk_grid(G, batch), TPB, 0, (cudaStream_t)stream>>>(G, counts, nsamp, out);
    return (int)cudaGetLastError();
}

int launch_marginals(const Geometry& G, const uint16_t* counts, int nsamp, float* out,
                     long long out_chain_stride, int k, int batch, void* stream) {
    int gx = (G.W + 255) / 256;
    if (gx > 64) gx = 64;
    dim3 grid(gx, G.rows < 65535 ? G.rows : 65535, batch);
    marginals_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(G, counts, nsamp, out,
                                                             out_chain_stride, k);
    return (int)cudaGetLastError();
}

int launch_metric_sums(const MetricParams& p, int batch, void* stream) {
    if (p.kind == 2)
        metric_sums_kernel<true><<<chunk_grid(p.geo, batch, 512), TPB, 0, (cudaStream_t)stream>>>(p);
    else
        metric_sums_kernel<false><<<chunk_grid(p.geo, batch, 512), TPB, 0, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

void ssim_windowed_grid(int H, int W, int* gx, int* gy) {
    const int nwr = H - SSIM_WIN + 1, nwc = W - SSIM_WIN + 1;
    *gx = nwc > 0 ? (nwc + SSIM_TPB - 1) / SSIM_TPB : 0;
    *gy = nwr > 0 ? (nwr + SSIM_ROWS_PER_BLOCK - 1) / SSIM_ROWS_PER_BLOCK : 0;
}

int launch_ssim_windowed(const WinSsimParams& p, int batch, void* stream) {
    int gx = 0, gy = 0;
    ssim_windowed_grid(p.H, p.W, &gx, &gy);
    if (gx == 0 || gy == 0) return 0;
    dim3 grid(gx, gy, batch);
    ssim_windowed_kernel<<<grid, SSIM_TPB, 0, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace pcab200
