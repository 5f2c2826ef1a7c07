// aux.cu -- layout kernels and the fused estimate / metric reductions.
//
//  * pack_state / unpack_state: dense [batch][rows][W] <-> padded x buffer (+ torus halos).
//  * mpm / marginals / cm: the posterior-marginal estimates from the counts (R15):
//    MPM_i = argmax_k count_i[k] (ties to the lowest k); marginal = count/N_samp;
//    CM_i = sum_k lum(k) count_i[k]/N_samp (conditional mean).
//  * metric_sums: one pass over truth and the LAST or MPM estimate, accumulating the exact
//    integer sums of PAPER.md:516-534's statistics (sum (x-y)^2, sum x, sum y, sum x^2,
//    sum y^2, sum xy, max x) per chain; block reduction, then one atomic per block per sum.
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace pcab200 {
namespace {

__global__ void pack_state_kernel(Geometry G, const uint8_t* __restrict__ dense, int src_pitch,
                                  long long src_chain, uint8_t* __restrict__ xbuf, int* bad) {
    const int chain = blockIdx.z;
    const uint8_t* src = dense + chain * src_chain;
    for (int pr = (int)blockIdx.y - 1; pr <= G.rows; pr += gridDim.y) {  // padded row -1..rows
        uint8_t* dst = xbuf + chain * G.xchain + (long long)(pr + 1) * G.xpitch + XOFF;
        int sr = pr;
        if (pr < 0 || pr >= G.rows) {
            if (!(G.periodic && G.self_halo_rows)) continue;
            sr = pr < 0 ? G.rows - 1 : 0;
        }
        for (int c = blockIdx.x * blockDim.x + threadIdx.x - 1; c <= G.W;
             c += gridDim.x * blockDim.x) {
            int sc = c;
            if (c < 0 || c >= G.W) {
                if (!G.periodic) continue;
                sc = c < 0 ? G.W - 1 : 0;
            }
            const uint8_t v = src[(long long)sr * src_pitch + sc];
            if (v >= G.levels) atomicOr(bad, 1);
            dst[c] = v;
        }
    }
}

__global__ void unpack_state_kernel(Geometry G, const uint8_t* __restrict__ xbuf,
                                    uint8_t* __restrict__ dense) {
    const int chain = blockIdx.z;
    for (int r = blockIdx.y; r < G.rows; r += gridDim.y) {
        const uint8_t* src = xbuf + chain * G.xchain + (long long)(r + 1) * G.xpitch + XOFF;
        uint8_t* dst = dense + ((long long)chain * G.rows + r) * G.W;
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < G.W; c += gridDim.x * blockDim.x)
            dst[c] = src[c];
    }
}

__global__ void check_levels_kernel(const uint8_t* __restrict__ p, size_t n, int levels, int* bad) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
         i += (size_t)gridDim.x * blockDim.x)
        if (p[i] >= levels) atomicOr(bad, 1);
}

__device__ __forceinline__ int mpm_label(const Geometry& G, const uint16_t* cchain, int r, int c,
                                         int nsamp) {
    const uint16_t* cp = cchain + (long long)r * G.cpitch + c;
    if (G.levels == 2) return (2 * (int)cp[0] > nsamp) ? 1 : 0;
    int best = 0;
    int bc = cp[0];
    for (int k = 1; k < G.levels; ++k) {
        const int v = cp[(long long)k * G.cplane];
        if (v > bc) { bc = v; best = k; }
    }
    return best;
}

__global__ void mpm_kernel(Geometry G, const uint16_t* __restrict__ counts, int nsamp,
                           uint8_t* __restrict__ out) {
    const int chain = blockIdx.z;
    const uint16_t* cc = counts + chain * G.cchain;
    for (int r = blockIdx.y; r < G.rows; r += gridDim.y) {
        uint8_t* dst = out + ((long long)chain * G.rows + r) * G.W;
        for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < G.W; c += gridDim.x * blockDim.x)
            dst[c] = (uint8_t)mpm_label(G, cc, r, c, nsamp);
    }
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

__global__ void __launch_bounds__(256) metric_sums_kernel(const MetricParams p) {
    const Geometry& G = p.geo;
    const int chain = blockIdx.y;
    const uint8_t* truth = p.truth + (long long)chain * G.rows * G.W;
    const uint8_t* xb = p.x + chain * G.xchain;
    const uint16_t* cc = p.counts + chain * G.cchain;
    unsigned long long s[7] = {0, 0, 0, 0, 0, 0, 0};
    const long long n = (long long)G.rows * G.W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / G.W), c = (int)(i % G.W);
        const unsigned long long x = truth[i];
        const unsigned long long y =
            p.kind == 0 ? xb[(long long)(r + 1) * G.xpitch + XOFF + c] : mpm_label(G, cc, r, c, p.nsamp);
        const long long d = (long long)x - (long long)y;
        s[0] += (unsigned long long)(d * d);
        s[1] += x;
        s[2] += y;
        s[3] += x * x;
        s[4] += y * y;
        s[5] += x * y;
        s[6] = x > s[6] ? x : s[6];
    }
    __shared__ unsigned long long red[8][7];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < 6; ++k) s[k] = warp_sum(s[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xFFFFFFFFu, s[6], o);
        s[6] = v > s[6] ? v : s[6];
    }
    if (lane == 0)
        for (int k = 0; k < 7; ++k) red[warp][k] = s[k];
    __syncthreads();
    if (threadIdx.x < 7) {
        unsigned long long acc = 0;
        const int nw = blockDim.x >> 5;
        for (int w = 0; w < nw; ++w) {
            const unsigned long long v = red[w][threadIdx.x];
            acc = threadIdx.x == 6 ? (v > acc ? v : acc) : acc + v;
        }
        unsigned long long* dst = p.sums + chain * 8;
        if (threadIdx.x == 6) atomicMax(dst + 6, acc);
        else atomicAdd(dst + threadIdx.x, acc);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(p.sums + chain * 8 + 7, (unsigned long long)n);
}

inline dim3 row_grid(const Geometry& G, int rows, int batch, int threads) {
    int gx = (G.W + 2 + threads - 1) / threads;
    if (gx > 64) gx = 64;
    return dim3(gx, rows < 65535 ? rows : 65535, batch);
}

}  // namespace

int launch_pack_state(const Geometry& G, const uint8_t* src, int src_pitch, long long src_chain,
                      uint8_t* xbuf, int batch, int* bad, void* stream) {
    pack_state_kernel<<<row_grid(G, G.rows + 2, batch, 256), 256, 0, (cudaStream_t)stream>>>(
        G, src, src_pitch, src_chain, xbuf, bad);
    return (int)cudaGetLastError();
}

int launch_unpack_state(const Geometry& G, const uint8_t* xbuf, uint8_t* dense, int batch,
                        void* stream) {
    unpack_state_kernel<<<row_grid(G, G.rows, batch, 256), 256, 0, (cudaStream_t)stream>>>(G, xbuf,
                                                                                         dense);
    return (int)cudaGetLastError();
}

int launch_check_levels(const uint8_t* p, size_t n, int levels, int* bad, void* stream) {
    size_t blocks = (n + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    if (blocks == 0) blocks = 1;
    check_levels_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(p, n, levels, bad);
    return (int)cudaGetLastError();
}

int launch_mpm(const Geometry& G, const uint16_t* counts, int nsamp, uint8_t* out, int batch,
               void* stream) {
    mpm_kernel<<<row_grid(G, G.rows, batch, 256), 256, 0, (cudaStream_t)stream>>>(G, counts, nsamp,
                                                                                out);
    return (int)cudaGetLastError();
}

int launch_marginals(const Geometry& G, const uint16_t* counts, int nsamp, float* out,
                     long long out_chain_stride, int k, int batch, void* stream) {
    marginals_kernel<<<row_grid(G, G.rows, batch, 256), 256, 0, (cudaStream_t)stream>>>(
        G, counts, nsamp, out, out_chain_stride, k);
    return (int)cudaGetLastError();
}

int launch_metric_sums(const MetricParams& p, int batch, void* stream) {
    const long long n = (long long)p.geo.rows * p.geo.W;
    long long blocks = (n + 255) / 256;
    if (blocks > 1184) blocks = 1184;  // 8 per SM on 148 SMs
    if (blocks < 1) blocks = 1;
    metric_sums_kernel<<<dim3((unsigned)blocks, batch), 256, 0, (cudaStream_t)stream>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace pcab200
