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

}  // namespace pcab200
