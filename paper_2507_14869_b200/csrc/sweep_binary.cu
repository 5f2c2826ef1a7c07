// sweep_binary.cu -- one synchronous lazy-PCA sweep for levels == 2 (the headline kernel).
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
// Data path per thread: a 16-site row chunk (one 16-byte vector of x, g and the uint16
// counts' 32 bytes) for `R` consecutive rows, walking down with a rolling 3-row window
// in registers.  Neighbour counts are SWAR byte sums: vertical sum of the 3 rows, then
// left/right byte shifts with funnel shifts; the words left/right of the chunk come from
// the adjacent lanes by warp shuffle (lanes 0 and 31 load them).  One Philox4x32-10 call
// serves 4 sites.  MPM counts of label 1 are updated in the same pass (R15).
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace pcab200 {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;

// Map label bytes to {0,1}: 0 -> 0, 1 -> 1, sentinel 0xFF -> 0 (b & ~(b >> 1) & 1).
__device__ __forceinline__ uint32_t to01(uint32_t w) { return w & ~(w >> 1) & 0x01010101u; }

__device__ __forceinline__ uint4 ldg16(const uint8_t* p) {
    return __ldg(reinterpret_cast<const uint4*>(p));
}
__device__ __forceinline__ uint32_t ldg4(const uint8_t* p) {
    return __ldg(reinterpret_cast<const uint32_t*>(p));
}

// bytes shifted one column right (byte j <- byte j-1 of the 8-byte window lo:hi)
__device__ __forceinline__ uint32_t from_left(uint32_t lo, uint32_t hi) {
    return __funnelshift_l(lo, hi, 8);
}
// bytes shifted one column left (byte j <- byte j+1)
__device__ __forceinline__ uint32_t from_right(uint32_t lo, uint32_t hi) {
    return __funnelshift_r(lo, hi, 8);
}

__device__ __forceinline__ void store_chunk(uint8_t* op, const uint32_t (&o)[4], int nvalid) {
    if (nvalid >= 16) {
        *reinterpret_cast<uint4*>(op) = make_uint4(o[0], o[1], o[2], o[3]);
    } else {
        for (int j = 0; j < nvalid; ++j) op[j] = (uint8_t)(o[j >> 2] >> (8 * (j & 3)));
    }
}

__device__ __forceinline__ uint8_t out_byte(const uint32_t (&o)[4], int j) {
    return (uint8_t)(o[j >> 2] >> (8 * (j & 3)));
}

template <int NB>
__device__ __forceinline__ int neighbours_present(int grow, int H, int c, int W) {
    const int er = (grow == 0) + (grow == H - 1);
    const int ec = (c == 0) + (c == W - 1);
    return NB == 8 ? (3 - er) * (3 - ec) - 1 : 4 - er - ec;
}

template <int R, int NB>
__global__ void __launch_bounds__(128)
    sweep_binary_kernel(const __grid_constant__ BinarySweepParams p) {
    __shared__ uint32_t s_thr[THR_ENTRIES];
    const int tid = threadIdx.y * 32 + threadIdx.x;
    for (int i = tid; i < THR_ENTRIES; i += 128) s_thr[i] = p.thr[i];
    __syncthreads();

    const Geometry& G = p.c.geo;
    const int lane = threadIdx.x;
    const int k = blockIdx.x * 32 + lane;  // 16-site chunk index
    const int chain = blockIdx.z;
    const int rbeg = (blockIdx.y * 4 + threadIdx.y) * R;
    if (rbeg >= G.rows) return;  // warp-uniform
    const int rend = min(rbeg + R, G.rows);
    const bool has_chunk = k <= G.nchunks;  // chunk nchunks is readable padding
    const bool active = k < G.nchunks;
    const int col0 = 16 * k;
    const uint8_t* xin = p.c.x_in + chain * G.xchain + XOFF + col0;
    const uint8_t* gin = p.c.g + chain * G.gchain + col0;
    uint8_t* xout = p.c.x_out + chain * G.xchain + XOFF + col0;
    uint16_t* cnt = p.c.counts + chain * G.cchain + col0;
    const uint32_t tagchain = (TAG_PCA << 24) | (p.c.chain0 + (uint32_t)chain);
    const bool col_edge = !G.periodic && (k == 0 || k == G.nchunks - 1);

    auto load = [&](int r, uint32_t(&w)[4], uint32_t& e) {
        const uint8_t* rp = xin + (long long)(r + 1) * G.xpitch;
        if (has_chunk) {
            const uint4 v = ldg16(rp);
            w[0] = to01(v.x); w[1] = to01(v.y); w[2] = to01(v.z); w[3] = to01(v.w);
        } else {
            w[0] = w[1] = w[2] = w[3] = 0u;
        }
        e = 0u;
        if (lane == 0) e = to01(ldg4(rp - 4));
        else if (lane == 31 && active) e = to01(ldg4(rp + 16));
    };

    uint32_t U[4], M[4], D[4], eU, eM, eD;
    load(rbeg - 1, U, eU);
    load(rbeg, M, eM);
    for (int r = rbeg; r < rend; ++r) {
        load(r + 1, D, eD);
        const int grow = G.row0 + r;
        uint32_t Gw[4] = {0u, 0u, 0u, 0u};
        if (has_chunk) {
            const uint4 v = ldg16(gin + (long long)r * G.gpitch);
            Gw[0] = v.x; Gw[1] = v.y; Gw[2] = v.z; Gw[3] = v.w;
        }
        // ---- n_i(1): SWAR neighbour counts, one byte per site ----
        uint32_t S[4];
        if (NB == 8) {
            uint32_t V[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) V[i] = U[i] + M[i] + D[i];
            uint32_t VL = __shfl_up_sync(FULL, V[3], 1);
            uint32_t VR = __shfl_down_sync(FULL, V[0], 1);
            if (lane == 0) VL = eU + eM + eD;
            if (lane == 31) VR = eU + eM + eD;
            S[0] = from_left(VL, V[0]) + V[0] + from_right(V[0], V[1]) - M[0];
            S[1] = from_left(V[0], V[1]) + V[1] + from_right(V[1], V[2]) - M[1];
            S[2] = from_left(V[1], V[2]) + V[2] + from_right(V[2], V[3]) - M[2];
            S[3] = from_left(V[2], V[3]) + V[3] + from_right(V[3], VR) - M[3];
        } else {
            uint32_t ML = __shfl_up_sync(FULL, M[3], 1);
            uint32_t MR = __shfl_down_sync(FULL, M[0], 1);
            if (lane == 0) ML = eM;
            if (lane == 31) MR = eM;
            S[0] = U[0] + D[0] + from_left(ML, M[0]) + from_right(M[0], M[1]);
            S[1] = U[1] + D[1] + from_left(M[0], M[1]) + from_right(M[1], M[2]);
            S[2] = U[2] + D[2] + from_left(M[1], M[2]) + from_right(M[2], M[3]);
            S[3] = U[3] + D[3] + from_left(M[2], M[3]) + from_right(M[3], MR);
        }
        // table index byte = n1*4 + g*2 + x  (+ np*36 added per site)
        uint32_t IDX[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) IDX[i] = (S[i] << 2) | (Gw[i] << 1) | M[i];
        const bool edge = col_edge || (!G.periodic && (grow == 0 || grow == G.H - 1));

        // ---- Philox (one call per 4 sites) + integer-threshold decisions ----
        uint32_t O[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 rnd =
                philox4x32_10(make_uint4((uint32_t)(4 * k + i), (uint32_t)grow, p.c.t, tagchain),
                              p.c.keys);
            const uint32_t rr[4] = {rnd.x, rnd.y, rnd.z, rnd.w};
            uint32_t o = 0u;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                uint32_t idx = (IDX[i] >> (8 * b)) & 0xFFu;
                int np = NB;
                if (edge) np = neighbours_present<NB>(grow, G.H, col0 + 4 * i + b, G.W);
                idx += (uint32_t)np * 36u;
                o |= (rr[b] > s_thr[idx] ? 1u : 0u) << (8 * b);
            }
            O[i] = o;
        }

        if (active) {
            // ---- fused MPM counts of label 1 (uint16 per site) ----
            if (p.c.count_enable) {
                uint4* cp = reinterpret_cast<uint4*>(cnt + (long long)r * G.cpitch);
                uint4 c0 = cp[0], c1 = cp[1];
                c0.x += __byte_perm(O[0], 0u, 0x4140); c0.y += __byte_perm(O[0], 0u, 0x4342);
                c0.z += __byte_perm(O[1], 0u, 0x4140); c0.w += __byte_perm(O[1], 0u, 0x4342);
                c1.x += __byte_perm(O[2], 0u, 0x4140); c1.y += __byte_perm(O[2], 0u, 0x4342);
                c1.z += __byte_perm(O[3], 0u, 0x4140); c1.w += __byte_perm(O[3], 0u, 0x4342);
                cp[0] = c0;
                cp[1] = c1;
            }
            // ---- store x_{t+1} (+ torus halos) ----
            const int nvalid = G.W - col0;
            uint8_t* op = xout + (long long)(r + 1) * G.xpitch;
            store_chunk(op, O, nvalid);
            if (G.periodic) {
                if (k == 0) op[G.W] = out_byte(O, 0);                       // right halo
                if (k == G.nchunks - 1) op[-col0 - 1] = out_byte(O, G.W - 1 - col0);  // left halo
                if (G.self_halo_rows && (grow == 0 || grow == G.H - 1)) {
                    uint8_t* hp = op + (grow == 0 ? 1LL : -1LL) * (long long)G.rows * G.xpitch;
                    store_chunk(hp, O, nvalid);
                    if (k == 0) hp[G.W] = out_byte(O, 0);
                    if (k == G.nchunks - 1) hp[-col0 - 1] = out_byte(O, G.W - 1 - col0);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) { U[i] = M[i]; M[i] = D[i]; }
        eU = eM;
        eM = eD;
    }
}

template <int R>
int launch_r(const BinarySweepParams& p, int batch, cudaStream_t s) {
    const Geometry& G = p.c.geo;
    dim3 block(32, 4, 1);
    dim3 grid((G.nchunks + 31) / 32, (G.rows + 4 * R - 1) / (4 * R), batch);
    if (G.nbhd == 8) sweep_binary_kernel<R, 8><<<grid, block, 0, s>>>(p);
    else sweep_binary_kernel<R, 4><<<grid, block, 0, s>>>(p);
    return (int)cudaGetLastError();
}

}  // namespace

int launch_sweep_binary(const BinarySweepParams& p, int batch, int rows_per_thread,
                        void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    switch (rows_per_thread) {
        case 1: return launch_r<1>(p, batch, s);
        case 2: return launch_r<2>(p, batch, s);
        case 4: return launch_r<4>(p, batch, s);
        case 16: return launch_r<16>(p, batch, s);
        case 32: return launch_r<32>(p, batch, s);
        default: return launch_r<8>(p, batch, s);
    }
}

}  // namespace pcab200
