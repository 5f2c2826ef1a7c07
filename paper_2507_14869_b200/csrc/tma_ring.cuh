// tma_ring.cuh -- PTX wrappers for the per-warp shared-memory rings of the sweep kernels:
// mbarrier init / expect_tx / try_wait, 1-D TMA bulk copies global -> shared
// (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP), elect.sync and the proxy fence
// that orders generic-proxy reads of a stage before the async-proxy refill.
#pragma once
#include <cstdint>

namespace pcab200 {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// the same operations on 32-bit shared-window addresses (computed once per CTA)
__device__ __forceinline__ void mbar_expect_tx_s(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n}"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// bytes shifted one column right (byte j <- byte j-1 of lo:hi) / left (byte j <- byte j+1)
__device__ __forceinline__ uint32_t from_left(uint32_t lo, uint32_t hi) {
    return __funnelshift_l(lo, hi, 8);
}
__device__ __forceinline__ uint32_t from_right(uint32_t lo, uint32_t hi) {
    return __funnelshift_r(lo, hi, 8);
}
// byte j (0..15, run-time) of a 16-byte chunk, without a local-memory array copy
__device__ __forceinline__ uint8_t chunk_byte(const uint32_t (&o)[4], int j) {
    const uint32_t w = (j < 8) ? ((j < 4) ? o[0] : o[1]) : ((j < 12) ? o[2] : o[3]);
    return (uint8_t)(w >> (8 * (j & 3)));
}
__device__ __forceinline__ void store_chunk(uint8_t* op, const uint32_t (&o)[4], int nvalid) {
    if (nvalid >= 16) {
        *reinterpret_cast<uint4*>(op) = make_uint4(o[0], o[1], o[2], o[3]);
    } else {
        for (int j = 0; j < nvalid; ++j) op[j] = chunk_byte(o, j);
    }
}

// Store the 16-site chunk o (first column ccol, nvalid sites, chunk index k) of local row r
// into a padded state buffer whose row r starts at rowp, plus the torus halo copies: the
// column pads (16 wrapped columns each side when W % 16 == 0, else columns -1 and W) and,
// when this context owns the whole torus, the HALO wrapped rows above and below.
template <int HALO_ROWS, int XOFFB>
__device__ __forceinline__ void store_row_chunk(uint8_t* rowp, const uint32_t (&o)[4], int ccol,
                                                int nvalid, int k, int r, int W, int nchunks,
                                                int rows, long long pitch, bool periodic,
                                                bool self_halo_rows) {
    auto put = [&](uint8_t* rp) {
        store_chunk(rp + XOFFB + ccol, o, nvalid);
        if (periodic) {
            if ((W & 15) == 0) {
                const uint4 v = make_uint4(o[0], o[1], o[2], o[3]);
                if (k == 0) *reinterpret_cast<uint4*>(rp + XOFFB + W) = v;       // cols 0..15
                if (k == nchunks - 1) *reinterpret_cast<uint4*>(rp + XOFFB - 16) = v;  // W-16..W-1
            } else {
                if (k == 0) rp[XOFFB + W] = chunk_byte(o, 0);
                if (k == nchunks - 1) rp[XOFFB - 1] = chunk_byte(o, W - 1 - ccol);
            }
        }
    };
    put(rowp);
    if (periodic && self_halo_rows) {
        if (r < HALO_ROWS) put(rowp + (long long)rows * pitch);
        if (r >= rows - HALO_ROWS) put(rowp - (long long)rows * pitch);
    }
}

}  // namespace pcab200
