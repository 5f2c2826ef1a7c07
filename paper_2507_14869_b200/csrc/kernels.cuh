// Kernel parameter blocks and launch entry points shared by the host runtime
// (runtime.cu) and the device kernels (sweep_binary.cu, sweep_general.cu, aux.cu).
//
// HBM layout of one context:
//   x[2]   : uint8 [batch][rows+2*HALO][xpitch], xpitch = 16*nchunks + 32; padded row j in
//            -HALO..rows+HALO-1 at (j+HALO)*xpitch, data column c at byte XOFF + c; bytes
//            [0, XOFF) and [XOFF+W, XOFF+W+16) are the column pads.  Free boundary: halos
//            and pads hold the sentinel 0xFF (never a label).  Torus: halo rows and pads hold
//            the wrapped labels (16 columns each side when W % 16 == 0, else columns -1 and
//            W), rewritten by every sweep; other padding bytes are 0.
//   g      : uint8 [batch][rows+2*GHALO][gpitch], same column layout as x (pads wrapped on a
//            torus, 0 otherwise); halo rows wrapped on a single-context torus, else 0
//   counts : uint16, levels == 2: [batch][rows][cpitch] (count of label 1);
//            levels > 2: [batch][levels][rows][cpitch]  (cpitch = 16*nchunks)
//   dtab   : fp64 [levels][levels], D[g][s] = exp(-b (lum g - lum s)^2)  (general kernel)
//   sums   : uint64 [batch][8] metric accumulators
//   stage  : uint8 [batch][rows][W] (+ fp32 space for MARGINALS/CM) host<->device staging
#pragma once
#include <atomic>
#include <mutex>
#include <utility>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "philox.cuh"

// Device-side bound checks of the debug build (build(defines=("PCA_DEBUG=1",)): a violated
// invariant prints where and traps, so the launch fails with cudaErrorLaunchFailure instead of
// corrupting memory silently.  compute-sanitizer is closed on the GPU pool this was built on;
// these checks plus the workspace guard test stand in for memcheck.
#ifdef PCA_DEBUG
#include <cstdio>
#define PCA_DCHECK(cond)                                                                        \
    do {                                                                                        \
        if (!(cond)) {                                                                          \
            printf("PCA_DCHECK failed: %s at %s:%d (block %d,%d,%d thread %d)\n", #cond, __FILE__, \
                   __LINE__, (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z, (int)threadIdx.x);  \
            __trap();                                                                           \
        }                                                                                       \
    } while (0)
#else
#define PCA_DCHECK(cond) \
    do {                 \
    } while (0)
#endif

namespace pcab200 {

constexpr int XOFF = 16;           // data column 0 sits at byte 16 of a padded row
constexpr int HALO = 2;            // x halo rows above / below the owned rows
constexpr int GHALO = 1;           // g halo rows above / below the owned rows
constexpr int THR_ENTRIES = 324;   // binary thresholds [np 0..8][n1 0..8][g 0..1][x 0..1]
constexpr uint32_t TAG_PCA = 1u;
constexpr uint32_t TAG_GIBBS = 2u;
constexpr int GIBBS_THR2 = 162;   // levels == 2 Gibbs thresholds [np 0..8][n1 0..8][g 0..1]

struct Geometry {
    int W;             // columns
    int rows;          // owned rows (local)
    int H;             // global rows
    int row0;          // global index of local row 0
    int nchunks;       // ceil(W / 16)
    int levels;
    int nbhd;          // 4 or 8
    int periodic;      // torus?
    int self_halo_rows;  // torus and this context owns all rows: sweep rewrites row halos
    int xpitch;        // bytes per padded x row
    int gpitch;        // bytes per g row
    int cpitch;        // uint16 elements per counts row
    long long xchain;  // bytes between chains in an x buffer
    long long gchain;  // bytes between chains in g
    long long cplane;  // uint16 elements between label planes (levels > 2)
    long long cchain;  // uint16 elements between chains in counts
};

struct SweepCommon {
    Geometry geo;
    const uint8_t* x_in;   // padded buffer of chain 0, pointing at padded row -HALO, byte 0
    uint8_t* x_out;
    const uint8_t* g;
    uint16_t* counts;
    PhiloxKeys keys;
    uint32_t t;            // sweep index (Philox counter word 2)
    uint32_t chain0;       // chain id of batch entry 0
    int count_enable;      // accumulate MPM counts this sweep
    int rlo, rhi;          // local rows [rlo, rhi) updated by this launch
    // device-initiated halo exchange (row strips with peers attached, pca_attach_peers): the
    // new row 0 is also stored into peer_up (the up-peer's output-buffer row below its
    // strip, padded row base of chain 0) and the new row rows-1 into peer_dn (the
    // down-peer's row above its strip), over NVLink peer memory, by the CTAs that compute
    // them; nullptr = no such peer.  *_chain: the peers' chain strides in bytes.
    uint8_t* peer_up;
    uint8_t* peer_dn;
    long long peer_up_chain, peer_dn_chain;
};

// levels == 2 fast path: thr[((np*9 + n1)*2 + g)*2 + x] = ceil(p0 * 2^32) - 1, the
// largest Philox word r for which the new label is 0 (u = r 2^-32 < F_0 = p0).
// The table lives in the workspace (uploaded once per beta stage) and reaches shared memory
// with one TMA bulk copy per CTA.
struct BinarySweepParams {
    SweepCommon c;
    const uint32_t* thr;  // device [THR_ENTRIES]
};

// two sweeps (t, t+1) per pass: thr[0] for sweep t, thr[1] for sweep t+1; c.count_enable
// counts sweep t, count2 sweep t+1.
struct Binary2SweepParams {
    SweepCommon c;
    int count2;
    uint32_t thr[2][THR_ENTRIES];
};

// general path: A[n] = exp(a n), Cw = exp(-c) (L0 inertia); D table in global memory;
// itab[x][s] = exp(-c pen(x, s)) for the L1 / L2 inertia (inertia_p = 1, 2).  a, b, c feed
// the log-domain slow path used when the factorised weights under/overflow.
// uthr[((s*L + g)*L + x)*(L-1) + k] = ceil(F_k 2^32) - 1: the integer thresholds of a site
// whose neighbours all carry s (nullptr when L > 16).
struct GeneralSweepParams {
    SweepCommon c;
    double A[9];
    double Cw;
    double coef_a, coef_b, coef_c;
    const double* dtab;
    const double* itab;
    int inertia_p;
    const uint32_t* uthr;
    const uint32_t* bthr;  // levels == 2: the binary thresholds [THR_ENTRIES] (exact path)
    // 16 < levels <= 64: W0[g][x][s] = D[g][s] I[x][s] and pfx[g][x][k] = sum_{s<=k} W0
    // (per beta stage); nullptr otherwise
    const double* w0;
    const double* pfx;
    // 3 <= levels <= 5: the histogram-table kernel (sweep_table.cu) when tab != nullptr.
    // tab = one 16-byte-aligned blob, refreshed per beta stage, copied whole into each block's
    // shared memory by one bulk copy:
    //   [0, TAB_OFF_W0)           A[0..8] (fp64)
    //   [TAB_OFF_W0, tab_slots)   AW[g][x][s][n] = A[n] D[g][s] I[x][s], n = 0..8 (fp64, the
    //                             rare path's weights w_s = AW[g][x][s][n_s])
    //   [tab_slots, tab_thr)      uint2 slot[1 << tab_hbits] = {histogram tag, byte offset of
    //                             the key's threshold rows in the thr block}; tag 0xFFFFFFFF =
    //                             empty
    //   [tab_thr, tab_bytes)      uint32 thr[key][g][x][TP]: T_k = ceil(F_k 2^32) - 1 of the
    //                             site law for the key's neighbour histogram (TP = 2 for
    //                             levels == 3, else 4)
    // A key is a neighbour histogram h (nibble s = number of neighbours carrying s) of an
    // interior site with at most two distinct neighbour labels; its slot is
    // (h * tab_magic) >> (32 - tab_hbits).  Other sites (three or more labels, or fewer than
    // nbhd neighbours at a free boundary) take the fp64 path.
    const uint8_t* tab;
    uint32_t tab_bytes, tab_slots, tab_thr, tab_magic;
    int tab_hbits;
    // the table kernel's MPM counts as uint8 deltas [batch][levels][rows][cpitch] (chain stride
    // tdc_chain, plane stride tdc_plane bytes), folded into the uint16 counts by the runtime at
    // most every 255 counted sweeps and at the end of every pca_sweep call (launch_fold_counts
    // per plane); nullptr: the table kernel adds into the uint16 counts
    uint8_t* tdc;
    long long tdc_chain, tdc_plane;
};
constexpr int TAB_OFF_W0 = 80;

// two levels on bit-packed state (sweep_packed.cu): x_in / x_out packed [batch][rows+2*HALO][pp]
// (column c at bit c%8 of byte 16 + c/8), g packed [batch][rows][gpp] (gpp = W/8); c.geo,
// c.keys, c.t, c.chain0, c.counts, c.count_enable as for the byte kernels (c.x_* unused).
struct PackedSweepParams {
    SweepCommon c;
    const uint8_t* x_in;
    uint8_t* x_out;
    const uint8_t* g;
    const uint32_t* thr;  // the binary thresholds [THR_ENTRIES] of the stage
    uint8_t* dcounts;     // uint8 count deltas of label 1 [batch][rows][cpitch] (folded by the runtime)
    int pp, gpp;
    long long xchain, gchain, dchain;
};

// Gibbs sampler, one colour class per launch, in place (x_in == x_out): sites of colour k
// (4-neighbour: (r + c) mod 2; Moore-8: 2 (r mod 2) + (c mod 2), global r) draw from the
// Gibbs conditional exp(a n_i(s) - b (lum g_i - lum s)^2) given the current state.
// levels == 2: thr2[(np*9 + n1)*2 + g] = ceil(p0 2^32) - 1 (integer-exact);
// levels > 2: uthr[(s*L + g)*(L-1) + k] for uniform neighbourhoods (L <= 16), else fp64
// A[n] D[g][s] weights (log-domain when they under/overflow).
struct GibbsSweepParams {
    SweepCommon c;
    int colour;   // fused: the row parity (both colours of those rows in one launch)
    int fused;    // Moore-8 with the two colours of a row in one launch (2 launches a sweep)
    double A[9];
    double coef_a, coef_b;
    const double* dtab;
    const uint32_t* uthr;
    uint32_t thr2[GIBBS_THR2];
};

// Gibbs, levels == 2, Moore-8, on the binary PCA kernel's data path (sweep_gibbs_binary.cu):
// one launch per row parity; c.x_in = X (x_t, the updated rows are read from it), x_nb = the
// buffer holding rows r -+ 1 (X for parity 0, Y for parity 1), c.x_out = Y.
constexpr int GIBBS_THR_PAD = 164;  // GIBBS_THR2 rounded up to a 16-byte multiple
struct GibbsBinParams {
    SweepCommon c;
    const uint8_t* x_nb;
    int parity;
    const uint32_t* thr;  // device [GIBBS_THR_PAD]: the Gibbs thresholds of the stage
};

struct MetricParams {
    Geometry geo;
    const uint8_t* x;      // padded current state, chain 0 at padded row -HALO
    const uint16_t* counts;
    const uint8_t* truth;  // dense [batch][rows][W]
    unsigned long long* sums;  // kind 0/1: [batch][8]; kind 2: [batch][16] (LAST, then MPM)
    int kind;              // 0 LAST, 1 MPM, 2 both in one pass (finalize)
    int nsamp;             // counted sweeps (MPM ties for levels == 2)
    uint8_t* mpm_out;      // kind 2: dense MPM image [batch][rows][W], or nullptr
    uint8_t* mpm_bits = nullptr;  // kind 2, levels == 2: bit-packed MPM image
                                  // [batch][rows][(W+7)/8], site c at bit c%8 of byte c/8
};

// Per-device launch facts (occupancy, SM count) cached on first use on each device:
// cudaFuncSetAttribute and occupancy are per device, so one process may drive several GPUs.
// Filled once per device under launch_info_mutex() (double-checked: `ok` is released after
// the fields are written), so host threads may launch concurrently.
struct LaunchInfo {
    std::atomic<bool> ok{false};
    int occ = 1, mocc = 1, sms = 1;
};
inline std::mutex& launch_info_mutex() {
    static std::mutex m;
    return m;
}
// Programmatic dependent launch (PDL) between consecutive kernels of a stream: the kernel calls
// pdl_begin() first (let the next grid be scheduled once every block of this one is resident,
// then wait until the previous grid has completed and its memory is visible -- nothing is read
// before that), and is launched with launch_pdl (the programmatic-serialization attribute).
__device__ __forceinline__ void pdl_begin() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int MAX_DEVICES = 64;
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d < 0 ? 0 : (d >= MAX_DEVICES ? MAX_DEVICES - 1 : d);
}

// ---- launchers (return cudaError_t as int) ----
int launch_sweep_binary(const BinarySweepParams& p, int batch, int rows_per_thread,
                        void* stream);
// nsweeps > 1: consecutive sweeps t .. t+nsweeps-1 (same tables and counting) in one
// cooperative launch, x_in / x_out alternating; the result is in x_in when nsweeps is even.
int launch_sweep_general(const GeneralSweepParams& p, int batch, int nsweeps, void* stream);
// 3 <= levels <= 5 with p.tab set: the histogram-table kernel (sweep_table.cu), same contract
int launch_sweep_table(const GeneralSweepParams& p, int batch, int nsweeps, void* stream);
// nsweeps > 1: that many Gibbs sweeps (one beta stage, c.count_enable = counting for the run,
// c.t = first sweep) in one cooperative launch, in place (small lattices)
int launch_sweep_gibbs(const GibbsSweepParams& p, int batch, int nsweeps, void* stream);
int launch_gibbs_binary(const GibbsBinParams& p, int batch, void* stream);

// copy a small host table into device memory through the kernel parameter block (stream
// ordered, no host synchronisation, no pinned staging buffer to protect)
constexpr int PARAM_TABLE_MAX = 1024;
struct ParamTable {
    uint32_t v[PARAM_TABLE_MAX];
};
int launch_param_table(const ParamTable& t, int n, uint32_t* dst, void* stream);
int launch_sweep_binary2(const Binary2SweepParams& p, int batch, int rows_per_thread, void* stream);
// bit-packed two-level sweep (whole lattice, W % 512 == 0) and the byte <-> packed converters
int launch_sweep_packed(const PackedSweepParams& p, int batch, void* stream);
int launch_state_to_packed(const Geometry& G, const uint8_t* xb, uint8_t* xp, int pp, long long pchain,
                           int batch, void* stream);
// halo_up / halo_dn: also write the halo rows above / below (a torus, or a strip's neighbour)
int launch_state_from_packed(const Geometry& G, const uint8_t* xp, int pp, long long pchain, uint8_t* xb,
                             int batch, void* stream, int halo_up, int halo_dn);
int launch_fold_counts(const Geometry& G, uint16_t* counts, uint8_t* delta, long long dchain, int batch,
                       void* stream);
int launch_g_to_packed(const Geometry& G, const uint8_t* gb, uint8_t* gp, int gpp, long long gpchain, int batch,
                       void* stream);
int launch_pack_state(const Geometry& geo, const uint8_t* src, int src_pitch, long long src_chain,
                      uint8_t* xbuf, int batch, int* bad_flag, void* stream);
// xbuf non-null: the same pass also writes the state buffer (x0 = g, one read of the input)
int launch_pack_g(const Geometry& geo, const uint8_t* src, int src_pitch, long long src_chain,
                  uint8_t* gbuf, int batch, int* bad_flag, void* stream, uint8_t* xbuf = nullptr);
int launch_unpack_state(const Geometry& geo, const uint8_t* xbuf, uint8_t* dense, int batch,
                        void* stream);
int launch_check_levels(const uint8_t* dense, size_t n, int levels, int* bad_flag,
                        void* stream);
int launch_mpm(const Geometry& geo, const uint16_t* counts, int nsamp, uint8_t* dense_out,
               int batch, void* stream);
int launch_marginals(const Geometry& geo, const uint16_t* counts, int nsamp, float* out,
                     long long out_chain_stride, int k, int batch, void* stream);
int launch_metric_sums(const MetricParams& p, int batch, void* stream);  // kind 0, 1 or 2
// out[chain] += number of sites whose label differs between padded buffers xa and xb
// bit-packed binary images <-> dense uint8 [nrows][W] (packed rows of ceil(W/8) bytes)
int launch_unpack_bits(const uint8_t* bits, uint8_t* dense, int W, long long nrows, void* stream);
int launch_pack_bits(const uint8_t* dense, uint8_t* bits, int W, long long nrows, void* stream);
int launch_changed(const Geometry& geo, const uint8_t* xa, const uint8_t* xb,
                   unsigned long long* out, int batch, void* stream);

// windowed SSIM: 7x7 uniform windows at every position inside the image, sample moments
constexpr int SSIM_WIN = 7, SSIM_TPB = 128, SSIM_ROWS_PER_BLOCK = 64;
struct WinSsimParams {
    const uint8_t* x;  // image 1, row 0 col 0 of chain 0
    long long xchain;
    int xpitch;
    const uint8_t* y;  // image 2
    long long ychain;
    int ypitch;
    int H, W, levels;
    double* partial;   // [batch][gy][gx] per-block sums of window SSIMs
};
void ssim_windowed_grid(int H, int W, int* gx, int* gy);
int launch_ssim_windowed(const WinSsimParams& p, int batch, void* stream);

}  // namespace pcab200
