// runtime.cu -- host runtime behind the C ABI of include/pca.h.
//
// Owns: configuration validation (before any device work), the workspace layout in HBM,
// per-beta-stage tables, the sweep loop with buffer swaps (a7),
// estimate / metric finalisation (a8, a9), checkpoint state I/O, and the NCCL
// communicator for row-strip sharding (halo exchange of one padded row per neighbour
// per sweep).  NCCL is loaded with dlopen on first use, so the library
// has no link-time dependency beyond libc/libdl (cudart is linked statically).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.cuh"
#include "pca.h"

using namespace pcab200;

// ---------------------------------------------------------------------------
namespace {

thread_local std::string g_err;

pca_status fail(pca_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

// ---- NCCL via dlopen ----
struct NcclApi {
    bool loaded = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// loaded once, thread-safely (a function-local static's initialiser runs exactly once, and
// concurrent first callers wait for it: one host thread per GPU may attach at the same time)
NcclApi load_nccl() {
    NcclApi api;
    {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return api;
        }
#define LOAD(name, sym)                                                    \
    api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, sym));        \
    if (!api.name) {                                                       \
        api.why = std::string("missing NCCL symbol ") + sym;               \
        return api;                                                        \
    }
        LOAD(GetUniqueId, "ncclGetUniqueId");
        LOAD(CommInitRank, "ncclCommInitRank");
        LOAD(CommDestroy, "ncclCommDestroy");
        LOAD(CommGetAsyncError, "ncclCommGetAsyncError");
        LOAD(Send, "ncclSend");
        LOAD(Recv, "ncclRecv");
        LOAD(GroupStart, "ncclGroupStart");
        LOAD(GroupEnd, "ncclGroupEnd");
        LOAD(AllReduce, "ncclAllReduce");
        LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
        api.loaded = true;
    }
    return api;
}

NcclApi& nccl() {
    static NcclApi api = load_nccl();
    return api;
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// NVTX ranges around the ABI calls and the halo exchange (header-only NVTX v3: a no-op unless
// a profiler injects itself), so nsys/ncu timelines show the library's phases by name
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// uniform-neighbourhood integer threshold tables (multilevel kernel) up to 16 levels:
// 16^3 * 15 entries = 240 KiB
constexpr int UTHR_MAX_LEVELS = 16;
// above 16 levels (up to 64) the fp64 path uses per-stage tables W0[g][x][s] = D[g][s] I[x][s]
// and their prefix sums over s, so a site costs O(#distinct neighbour labels), not O(levels)
constexpr int SPARSE_MAX_LEVELS = 64;
// lattices up to this many sites (x batch) sweep in runs of one cooperative launch; the
// environment variable PCA_B200_MULTI_MAX_SITES overrides it (a tuning knob: the chain is the
// same either way)
size_t multi_max_sites() {
    static size_t v = [] {
        const char* e = getenv("PCA_B200_MULTI_MAX_SITES");
        return e ? (size_t)strtoull(e, nullptr, 10) : (size_t(1) << 18);
    }();
    return v;
}

// ---- histogram tables of the 3..5-level kernel (sweep_table.cu) ----
// Keys: the neighbour histograms of interior sites with at most two distinct neighbour labels
// (all NB neighbours present): n[s_lo] = NB - n_hi, n[s_hi] = n_hi (n_hi = 0: uniform), packed
// as nibbles h = sum_s n_s << 4s.  A multiplicative hash (h * magic) >> (32 - hbits) must be
// collision-free on the keys; the smallest hbits in 8..10 for which a magic is found (a fixed
// splitmix64 sequence of odd multipliers, so every process finds the same one) is used.
constexpr int TAB_MAX_LEVELS = 5;
struct TabKeys {
    std::vector<uint32_t> h;              // key -> histogram word
    std::vector<std::vector<int>> n;      // key -> histogram
    uint32_t magic = 0;
    int hbits = 0;
    bool ok = false;
};

// the bit-packed kernel: two levels, W % 512 == 0 (a whole lattice or a row strip)
bool packed_eligible(const pca_config* c) {
    return c->levels == 2 && c->width % 512 == 0 && c->height >= 3;
}

bool table_eligible(const pca_config* c) {
    const int rows = c->rows == 0 ? c->height : c->rows;
    return c->levels >= 3 && c->levels <= TAB_MAX_LEVELS && c->width <= 65535 && rows <= 65535;
}

int tab_tp_host(int L) { return L == 3 ? 2 : 4; }

size_t tab_nkeys(int L, int NB) { return (size_t)L + (size_t)L * (L - 1) / 2 * (NB - 1); }

// AW[g][x][s][n] = A[n] W0[g][x][s] (n = 0..8) follows A (kernels.cuh)
size_t tab_slots_off(int L) { return (TAB_OFF_W0 + 8 * 9 * (size_t)L * L * L + 15) & ~size_t(15); }

size_t tab_blob_bytes(int L, int NB, int hbits) {
    const size_t thr = tab_nkeys(L, NB) * L * L * tab_tp_host(L) * 4;
    return (tab_slots_off(L) + (size_t(8) << hbits) + thr + 15) & ~size_t(15);
}

const TabKeys& tab_keys(int L, int NB) {
    static std::mutex m;
    static TabKeys cache[TAB_MAX_LEVELS + 1][9];
    std::lock_guard<std::mutex> lock(m);
    TabKeys& K = cache[L][NB];
    if (K.ok || K.hbits < 0) return K;
    for (int s = 0; s < L; ++s) {
        std::vector<int> n(L, 0);
        n[s] = NB;
        K.n.push_back(n);
    }
    for (int lo = 0; lo < L; ++lo)
        for (int hi = lo + 1; hi < L; ++hi)
            for (int nh = 1; nh < NB; ++nh) {
                std::vector<int> n(L, 0);
                n[lo] = NB - nh;
                n[hi] = nh;
                K.n.push_back(n);
            }
    for (const auto& n : K.n) {
        uint32_t h = 0;
        for (int s = 0; s < L; ++s) h |= (uint32_t)n[s] << (4 * s);
        K.h.push_back(h);
    }
    uint64_t sm = 0x9E3779B97F4A7C15ull;
    for (int hb = 8; hb <= 10 && !K.ok; ++hb) {
        std::vector<uint8_t> used(size_t(1) << hb);
        for (int trial = 0; trial < (1 << 20) && !K.ok; ++trial) {
            uint64_t z = (sm += 0x9E3779B97F4A7C15ull);
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            const uint32_t mg = (uint32_t)(z ^ (z >> 31)) | 1u;
            std::fill(used.begin(), used.end(), 0);
            bool clash = false;
            for (uint32_t h : K.h) {
                const uint32_t sl = (h * mg) >> (32 - hb);
                if (used[sl]) {
                    clash = true;
                    break;
                }
                used[sl] = 1;
            }
            if (!clash) {
                K.magic = mg;
                K.hbits = hb;
                K.ok = true;
            }
        }
    }
    if (!K.ok) K.hbits = -1;  // no collision-free hash: the general kernel is used
    return K;
}

// Workspace layout: byte offsets of every region.
struct Layout {
    int rows = 0, nchunks = 0, xpitch = 0, gpitch = 0, cpitch = 0, cplanes = 0;
    size_t xbuf = 0;      // bytes of one x buffer
    size_t gbuf = 0;      // bytes of the g buffer
    size_t off_uthr = 0, uthr_entries = 0;
    size_t off_sparse = 0, sparse_entries = 0;  // W0 and prefix tables (16 < levels <= 64)
    size_t off_gthr = 0, gthr_entries = 0;  // Gibbs uniform-neighbourhood thresholds
    size_t off_bthr = 0;                    // binary PCA thresholds [THR_ENTRIES]
    size_t off_gbthr = 0;                   // binary Gibbs thresholds [GIBBS_THR_PAD]
    size_t off_tab = 0, tab_max = 0;        // histogram-table blob (3..5 levels, sweep_table.cu)
    // bit-packed two-level state (sweep_packed.cu): two packed x buffers and packed g
    size_t off_xp = 0, xp_bytes = 0, off_gp = 0, gp_bytes = 0, off_dc = 0, dc_bytes = 0;
    int pp = 0, gpp = 0;
    size_t off_x0 = 0, off_x1 = 0, off_g = 0, off_counts = 0, off_dtab = 0, off_itab = 0, off_sums = 0,
           off_sums_max = 0, off_flag = 0, off_stage = 0, off_truth = 0, off_io = 0, off_in = 0;
    size_t io_bytes = 0;  // one bit-packed image set (packed_io), 0 otherwise
    size_t stage_bytes = 0, counts_bytes = 0, total = 0;
};

bool finite_pos(double v) { return std::isfinite(v) && v > 0.0; }

pca_status validate(const pca_config* c) {
    if (!c) return fail(PCA_EINVAL, "config is NULL");
    if (c->height < 1 || c->width < 1) return fail(PCA_EINVAL, "height and width must be >= 1");
    if (c->width > (1 << 30) || c->height > (1 << 30))
        return fail(PCA_EINVAL, "height/width must be <= 2^30");
    if (c->batch < 1 || c->batch > 65535) return fail(PCA_EINVAL, "batch must be in [1, 65535]");
    if (c->levels < 2 || c->levels > 255) return fail(PCA_EINVAL, "levels must be in [2, 255]");
    if (c->neighborhood != 4 && c->neighborhood != 8)
        return fail(PCA_EINVAL, "neighborhood must be 4 or 8");
    if (c->periodic != 0 && c->periodic != 1) return fail(PCA_EINVAL, "periodic must be 0 or 1");
    if (c->periodic && (c->height < 3 || c->width < 3))
        return fail(PCA_EINVAL, "a torus needs height, width >= 3 (distinct neighbours, R7)");
    if (!finite_pos(c->J)) return fail(PCA_EINVAL, "J must be finite and > 0");
    if (!std::isfinite(c->q) || c->q < 0.0) return fail(PCA_EINVAL, "q must be finite and >= 0");
    if (!finite_pos(c->sigma)) return fail(PCA_EINVAL, "sigma must be finite and > 0");
    if (!finite_pos(c->beta0)) return fail(PCA_EINVAL, "beta0 must be finite and > 0");
    if (!std::isfinite(c->beta_step) || c->beta_step < 0.0)
        return fail(PCA_EINVAL, "beta_step must be finite and >= 0");
    if (c->beta_period < 1) return fail(PCA_EINVAL, "beta_period must be >= 1");
    if (!finite_pos(c->coef_scale)) return fail(PCA_EINVAL, "coef_scale must be finite and > 0");
    if (c->chain0 < 0 || (long long)c->chain0 + c->batch > (1LL << 24))
        return fail(PCA_EINVAL, "chain ids must lie in [0, 2^24)");
    if (c->rows == 0) {
        if (c->row0 != 0) return fail(PCA_EINVAL, "rows == 0 (whole lattice) requires row0 == 0");
    } else if (c->rows < 1 || c->row0 < 0 || (long long)c->row0 + c->rows > c->height) {
        return fail(PCA_EINVAL, "owned rows [row0, row0+rows) must lie inside [0, height)");
    } else if (c->rows < c->height && c->rows < HALO) {
        return fail(PCA_EINVAL, "a row strip must own at least %d rows (halo depth)", HALO);
    }
    if (c->kernel < 0 || c->kernel > 4) return fail(PCA_EINVAL, "kernel must be 0..4");
    if (c->kernel == PCA_KERNEL_PACKED && !packed_eligible(c))
        return fail(PCA_EUNSUPPORTED, "the packed kernel needs levels == 2, width %% 512 == 0 and "
                                      "height >= 3");
    if (c->kernel == PCA_KERNEL_TABLE && !table_eligible(c))
        return fail(PCA_EUNSUPPORTED, "the table kernel needs 3..%d levels, width and rows <= 65535",
                    TAB_MAX_LEVELS);
    if (c->kernel == PCA_KERNEL_BINARY && c->levels != 2)
        return fail(PCA_EUNSUPPORTED, "the binary kernel needs levels == 2");
    const int R = c->rows_per_thread;
    if (R < 0 || R > 65536)
        return fail(PCA_EINVAL, "rows_per_thread must be in [0, 65536] (0 = auto)");
    if (c->sweeps_per_pass < 0 || c->sweeps_per_pass > 2)
        return fail(PCA_EINVAL, "sweeps_per_pass must be 0, 1 or 2");
    if (c->inertia_p < 0 || c->inertia_p > 2)
        return fail(PCA_EINVAL, "inertia_p must be 0 (L0), 1 (L1) or 2 (L2)");
    if (c->packed_io != 0 && c->packed_io != 1) return fail(PCA_EINVAL, "packed_io must be 0 or 1");
    if (c->packed_io && c->levels != 2)
        return fail(PCA_EUNSUPPORTED, "bit-packed images need levels == 2");
    for (int i = 0; i < 3; ++i)
        if (c->reserved[i] != 0) return fail(PCA_EINVAL, "reserved fields must be zero");
    if (c->graphs != 0 && c->graphs != 1) return fail(PCA_EINVAL, "graphs must be 0 or 1");
    if (c->graphs && c->levels != 2)
        return fail(PCA_EUNSUPPORTED, "graph-captured sweep runs need levels == 2 (the tables of more "
                                      "levels are uploaded by host copies)");
    return PCA_OK;
}

Layout make_layout(const pca_config* c) {
    Layout L;
    L.rows = c->rows == 0 ? c->height : c->rows;
    L.nchunks = (c->width + 15) / 16;
    L.xpitch = 16 * L.nchunks + 32;
    L.gpitch = 16 * L.nchunks + 32;
    L.cpitch = 16 * L.nchunks;
    L.cplanes = c->levels == 2 ? 1 : c->levels;
    const size_t B = (size_t)c->batch, R = (size_t)L.rows, W = (size_t)c->width;
    L.xbuf = B * (R + 2 * HALO) * (size_t)L.xpitch;
    L.gbuf = B * (R + 2 * GHALO) * (size_t)L.gpitch;
    L.counts_bytes = B * (size_t)L.cplanes * R * (size_t)L.cpitch * 2;
    // uint8 images and fp32 planes (one label plane at a time); windowed SSIM: staged truth,
    // MPM image and the per-block partial sums
    int sgx = 0, sgy = 0;
    ssim_windowed_grid(L.rows, c->width, &sgx, &sgy);
    L.stage_bytes = std::max(B * R * W * 4, align256(B * R * W) * 2 + B * (size_t)sgx * sgy * 8);
    size_t o = 0;
    L.off_x0 = o; o = align256(o + L.xbuf);
    L.off_x1 = o; o = align256(o + L.xbuf);
    L.off_g = o; o = align256(o + L.gbuf);
    L.off_counts = o; o = align256(o + L.counts_bytes);
    L.off_dtab = o; o = align256(o + (size_t)c->levels * c->levels * sizeof(double));
    L.off_itab = o; o = align256(o + (size_t)c->levels * c->levels * sizeof(double));
    L.uthr_entries = c->levels <= UTHR_MAX_LEVELS
                         ? (size_t)c->levels * c->levels * c->levels * (c->levels - 1) : 0;
    L.off_uthr = o; o = align256(o + L.uthr_entries * sizeof(uint32_t));
    L.sparse_entries = (c->levels > UTHR_MAX_LEVELS && c->levels <= SPARSE_MAX_LEVELS)
                           ? (size_t)c->levels * c->levels * c->levels : 0;
    L.off_sparse = o; o = align256(o + 2 * L.sparse_entries * sizeof(double));
    L.gthr_entries = (c->levels > 2 && c->levels <= UTHR_MAX_LEVELS)
                         ? (size_t)c->levels * c->levels * (c->levels - 1) : 0;
    L.off_gthr = o; o = align256(o + L.gthr_entries * sizeof(uint32_t));
    L.off_bthr = o; o = align256(o + THR_ENTRIES * sizeof(uint32_t));
    L.off_gbthr = o; o = align256(o + GIBBS_THR_PAD * sizeof(uint32_t));
    L.tab_max = (c->levels >= 3 && c->levels <= TAB_MAX_LEVELS) ? tab_blob_bytes(c->levels, c->neighborhood, 10) : 0;
    L.off_tab = o; o = align256(o + L.tab_max);
    if (packed_eligible(c)) {
        L.pp = c->width / 8 + 32;
        L.gpp = c->width / 8;
        L.xp_bytes = B * (R + 2 * HALO) * (size_t)L.pp;
        L.gp_bytes = B * R * (size_t)L.gpp;
        L.dc_bytes = B * R * (size_t)L.cpitch;  // uint8 count deltas
    } else if (table_eligible(c) && (c->kernel == PCA_KERNEL_AUTO || c->kernel == PCA_KERNEL_TABLE)) {
        L.dc_bytes = B * (size_t)c->levels * R * (size_t)L.cpitch;  // the table kernel's uint8 deltas
    }
    L.off_xp = o; o = align256(o + 2 * align256(L.xp_bytes));
    L.off_gp = o; o = align256(o + L.gp_bytes);
    L.off_dc = o; o = align256(o + L.dc_bytes);
    L.off_sums = o; o = align256(o + B * 16 * sizeof(unsigned long long));
    L.off_sums_max = o; o = align256(o + B * 16 * sizeof(unsigned long long));
    L.off_flag = o; o = align256(o + 256);
    L.off_stage = o; o = align256(o + L.stage_bytes);
    L.off_truth = o; o = align256(o + B * R * W);  // staged truth (pca_stage_truth)
    L.io_bytes = c->packed_io ? B * R * (size_t)((c->width + 7) / 8) : 0;
    L.off_io = o; o = align256(o + 3 * align256(L.io_bytes));  // packed in / out / truth
    L.off_in = o; o = align256(o + (c->packed_io ? L.io_bytes : B * R * W));  // pca_stage_input
    L.total = o;
    return L;
}

}  // namespace

// ---------------------------------------------------------------------------
struct pca_ctx {
    pca_config cfg;
    Layout lay;
    Geometry geo;
    int device = 0;
    cudaStream_t stream = nullptr;
    uint8_t* ws = nullptr;
    uint8_t* x[2] = {nullptr, nullptr};
    int cur = 0;
    uint8_t* g = nullptr;
    uint16_t* counts = nullptr;
    double* dtab = nullptr;
    double* itab = nullptr;  // I[x][s] = exp(-c pen(x, s)), per beta stage (inertia_p > 0)
    unsigned long long* sums = nullptr;
    unsigned long long* sums_max = nullptr;
    int* flag = nullptr;
    uint8_t* stage = nullptr;
    int64_t t = 0, counted = 0, launches = 0, sweep_launches = 0;
    double beta_last = 0.0;
    int kernel = PCA_KERNEL_BINARY;
    int rows_per_thread = 8;
    int poisoned = 0;
    int x_initialized = 0;
    // g / the state passed their level checks: a failed reset or state load leaves labels >=
    // levels in the buffers (the fused reset writes x[0] before the check), which would index
    // the tables out of range, so every call that reads them refuses until a good load
    int g_ok = 0, x_ok = 0;
    int prev_valid = 0;  // x[cur ^ 1] holds x_{t-1} (after a PCA or double-buffered Gibbs sweep)
    int64_t tab_stage = -1;
    int64_t gtab_stage = -1;
    int tdc_pending = 0;  // counted table-kernel sweeps in the uint8 count deltas (<= 255)
    GibbsSweepParams gib;
    GibbsBinParams gbin;
    uint32_t bthr_host[THR_ENTRIES];  // binary thresholds of the current stage (host copy)
    std::vector<uint32_t> gthr_host;
    uint32_t* gthr = nullptr;
    BinarySweepParams bin;
    Binary2SweepParams bin2;
    GeneralSweepParams gen;
    std::vector<double> dtab_host, itab_host, sparse_host;
    std::vector<uint32_t> uthr_host;
    uint32_t* uthr = nullptr;
    std::vector<uint8_t> tab_host;  // the histogram-table blob of the current stage (TABLE kernel)
    // cfg.graphs: captured pca_sweep runs, keyed by the host state they start from, with the
    // host state they leave (replayed runs apply it without re-running the host logic)
    struct SweepGraph {
        int64_t t, counted, tab_stage;
        int32_t n, cur, gpk_valid;
        cudaGraphExec_t exec;
        int64_t t_after, counted_after, tab_stage_after, launches_d, sweep_launches_d;
        int32_t cur_after, prev_valid_after, gpk_valid_after;
        double beta_after;
        uint32_t bthr_after[THR_ENTRIES];
    };
    std::vector<SweepGraph> graphs;
    int64_t graph_replays = 0;
    cudaStream_t cap = nullptr;  // the capture stream (the caller's may be the legacy default stream)
    uint8_t* xp[2] = {nullptr, nullptr};  // PACKED kernel: bit-packed state buffers
    uint8_t* gpk = nullptr;               // PACKED kernel: bit-packed g
    int gpk_valid = 0;                    // gpk holds the current g
    PackedSweepParams pk;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    cudaStream_t side = nullptr;  // interior rows of a strip, overlapping the halo exchange
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // pca_stage_truth: the truth copied on its own stream, overlapping the sweeps
    uint8_t* truth = nullptr;
    uint8_t* io_in = nullptr;     // packed_io: a bit-packed argument, before unpacking
    uint8_t* io_out = nullptr;    // packed_io: a bit-packed result, before the copy out
    uint8_t* io_truth = nullptr;  // packed_io: the staged truth, bit-packed
    int truth_staged = 0;
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_truth_ready = nullptr, ev_truth_free = nullptr;
    // pca_stage_input: the next reset's g, copied on the copy stream
    uint8_t* in_stage = nullptr;
    int in_staged = 0;
    cudaEvent_t ev_in_ready = nullptr, ev_in_free = nullptr;
    // pca_finalize_async: the MPM image's device->host copy on the copy stream
    cudaEvent_t ev_out_ready = nullptr, ev_out_free = nullptr;
    // device-initiated halo exchange (pca_attach_peers)
    int p2p = 0;
    int has_up = 0, has_dn = 0;
    pca_peer up{}, dn{};
    uint8_t* peer_g[2] = {nullptr, nullptr};  // the up / down peers' g buffers (padded row -GHALO)
    int g_halo_valid = 0;  // strips, two sweeps per pass: g's halo rows hold the neighbours' rows
    uint32_t* pflags = nullptr;  // [0]: phase completed by the up peer, [1]: by the down peer
    uint32_t phase = 0;          // phases (state loads, sweeps) this context has completed
};

namespace {

pca_status cuda_fail(pca_ctx* ctx, cudaError_t e, const char* where) {
    if (ctx) ctx->poisoned = 1;
    return fail(PCA_ECUDA, "%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
}

#define CK(ctx, expr)                                                 \
    do {                                                              \
        cudaError_t e_ = (cudaError_t)(expr);                         \
        if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #expr);    \
    } while (0)

#define LAUNCH(ctx, expr)                                                        \
    do {                                                                         \
        int e_ = (expr);                                                         \
        (ctx)->launches++;                                                       \
        if (e_ != 0) return cuda_fail((ctx), (cudaError_t)e_, #expr);            \
    } while (0)

// Every ABI call that takes a context runs on the context's device (usable() makes it
// current) and gives the caller's current device back when it returns.
struct DeviceScope {
    int prev = -1;
    DeviceScope() {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

pca_status usable(pca_ctx* ctx) {
    if (!ctx) return fail(PCA_EINVAL, "context is NULL");
    if (ctx->poisoned)
        return fail(PCA_ESTATE, "context poisoned by an earlier CUDA/NCCL error; destroy it");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
    return PCA_OK;
}

// usable, and the observed image and the state hold valid labels (calls that read them)
pca_status ready(pca_ctx* ctx) {
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!ctx->g_ok || !ctx->x_ok)
        return fail(PCA_ESTATE, "the last reset or state load failed its level check: "
                                "reset with a valid g (and x0) first");
    return PCA_OK;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// device memory of another GPU than the context's cannot be used by its kernels
pca_status check_same_device(const pca_ctx* ctx, const void* p, const char* what) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return PCA_OK;  // plain host memory
    }
    if (a.type == cudaMemoryTypeDevice && a.device != ctx->device)
        return fail(PCA_EINVAL, "%s is on device %d, the context on device %d", what, a.device,
                    ctx->device);
    return PCA_OK;
}

size_t dense_bytes(const pca_ctx* ctx) {
    return (size_t)ctx->cfg.batch * ctx->lay.rows * (size_t)ctx->cfg.width;
}

// device view of a dense uint8 image argument (host data staged through `stage`)
pca_status device_input(pca_ctx* ctx, const uint8_t* p, const uint8_t** out) {
    pca_status st = check_same_device(ctx, p, "input image");
    if (st != PCA_OK) return st;
    if (ctx->cfg.packed_io) {  // bit-packed argument: copy, then unpack into the stage
        CK(ctx, cudaMemcpyAsync(ctx->io_in, p, ctx->lay.io_bytes, cudaMemcpyDefault, ctx->stream));
        LAUNCH(ctx, launch_unpack_bits(ctx->io_in, ctx->stage, ctx->cfg.width,
                                       (long long)ctx->cfg.batch * ctx->lay.rows, ctx->stream));
        *out = ctx->stage;
        return PCA_OK;
    }
    if (is_device_ptr(p)) {
        *out = p;
        return PCA_OK;
    }
    CK(ctx, cudaMemcpyAsync(ctx->stage, p, dense_bytes(ctx), cudaMemcpyHostToDevice, ctx->stream));
    *out = ctx->stage;
    return PCA_OK;
}

pca_status sync(pca_ctx* ctx) {
    CK(ctx, cudaStreamSynchronize(ctx->stream));
    CK(ctx, cudaGetLastError());
    if (ctx->comm) {
        ncclResult_t ar = ncclSuccess;
        nccl().CommGetAsyncError(ctx->comm, &ar);
        if (ar != ncclSuccess) {
            ctx->poisoned = 1;
            return fail(PCA_ENCCL, "NCCL async error: %s", nccl().GetErrorString(ar));
        }
    }
    return PCA_OK;
}

pca_status check_flag(pca_ctx* ctx, const char* what) {
    int h = 0;
    CK(ctx, cudaMemcpyAsync(&h, ctx->flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    pca_status st = sync(ctx);
    if (st != PCA_OK) return st;
    if (h) return fail(PCA_EINVAL, "%s contains a value >= levels", what);
    return PCA_OK;
}

double beta_at(const pca_config& c, int64_t t) {
    return c.beta0 + c.beta_step * (double)(t / c.beta_period);
}

double lum(int k, int levels) { return (double)k / (double)(levels - 1); }

// inertia penalty pen(x, s): 0 when s == x, else 1 (L0, the paper's),
// |lum x - lum s| (L1) or (lum x - lum s)^2 (L2)
double inertia_pen(int p, int x, int s, int levels) {
    if (s == x) return 0.0;
    if (p == 0) return 1.0;
    const double d = lum(x, levels) - lum(s, levels);
    return p == 1 ? fabs(d) : d * d;
}

// a1: per-stage tables.  The binary thresholds repeat the per-site law of PAPER.md:462-477
// in fp64 exactly as written (E = a n - b d^2 - c 1{s != x}; p0 = e0/(e0 + e1) with the
// max subtracted), so T = ceil(p0 2^32) is the integer form of "u < F_0".
pca_status build_tables(pca_ctx* ctx, int64_t t) {
    const pca_config& c = ctx->cfg;
    const int64_t stage = t / c.beta_period;
    if (stage == ctx->tab_stage) return PCA_OK;
    const double beta = beta_at(c, t);
    const double a = c.coef_scale * 2.0 * beta * c.J;
    const double b = c.coef_scale / (2.0 * c.sigma * c.sigma);
    const double cq = beta * c.q;
    if (c.levels == 2) {  // binary thresholds: the binary kernel and the exact l = 2 general path
        for (int np = 0; np <= 8; ++np)
            for (int n1 = 0; n1 <= 8; ++n1)
                for (int gl = 0; gl < 2; ++gl)
                    for (int xl = 0; xl < 2; ++xl) {
                        const int idx = ((np * 9 + n1) * 2 + gl) * 2 + xl;
                        if (n1 > np) {
                            ctx->bthr_host[idx] = 0u;
                            continue;
                        }
                        const int n[2] = {np - n1, n1};
                        double E[2];
                        for (int s = 0; s < 2; ++s) {
                            const double d = lum(gl, 2) - lum(s, 2);
                            const double inert = inertia_pen(c.inertia_p, xl, s, 2);
                            E[s] = a * (double)n[s] - b * d * d - cq * inert;
                        }
                        double Emax = -INFINITY;
                        for (int s = 0; s < 2; ++s)
                            if (E[s] > Emax) Emax = E[s];
                        const double e0 = exp(E[0] - Emax);
                        const double e1 = exp(E[1] - Emax);
                        const double Z = 0.0 + e0 + e1;
                        const double p0 = e0 / Z;
                        // T in [0, 2^32]; T = 0 (p0 underflowed to 0) is stored as 0, which
                        // differs from the exact rule only for r = 0, where u = 0 = F_0 is an
                        // exact tie (an allowed near-tie, R19).
                        const double T = ceil(p0 * 4294967296.0);
                        ctx->bthr_host[idx] = T >= 1.0 ? (uint32_t)(T - 1.0) : 0u;
                    }
        ParamTable pt;
        memcpy(pt.v, ctx->bthr_host, sizeof(ctx->bthr_host));
        LAUNCH(ctx, launch_param_table(pt, THR_ENTRIES, const_cast<uint32_t*>(ctx->bin.thr), ctx->stream));
    }
    {
        GeneralSweepParams& m = ctx->gen;
        for (int n = 0; n <= 8; ++n) m.A[n] = exp(a * (double)n);
        m.Cw = exp(-cq);
        m.coef_a = a;
        m.coef_b = b;
        m.coef_c = cq;
        // (two levels: every kernel decides from the binary thresholds above, so the host
        // copies of the multi-level tables are skipped -- which keeps a two-level sweep run
        // free of host copies, as CUDA-graph capture requires)
        if (c.inertia_p != 0 && c.levels > 2) {
            const int L = c.levels;
            for (int xl = 0; xl < L; ++xl)
                for (int s = 0; s < L; ++s)
                    ctx->itab_host[(size_t)xl * L + s] = exp(-cq * inertia_pen(c.inertia_p, xl, s, L));
            CK(ctx, cudaMemcpyAsync(ctx->itab, ctx->itab_host.data(),
                                    ctx->itab_host.size() * sizeof(double), cudaMemcpyHostToDevice,
                                    ctx->stream));
        }
        if (ctx->lay.sparse_entries) {
            // W0[g][x][s] = D[g][s] * I[x][s] (I = the inertia factor of this stage) and its
            // prefix sums over s: the weights of a site with no neighbour carrying s
            const int L = c.levels;
            const size_t n3 = ctx->lay.sparse_entries;
            double* w0 = ctx->sparse_host.data();
            double* pf = w0 + n3;
            for (int gl = 0; gl < L; ++gl)
                for (int xl = 0; xl < L; ++xl) {
                    double acc = 0.0;
                    for (int s = 0; s < L; ++s) {
                        const size_t i = ((size_t)gl * L + xl) * L + s;
                        const double iw = exp(-cq * inertia_pen(c.inertia_p, xl, s, L));
                        w0[i] = ctx->dtab_host[(size_t)gl * L + s] * iw;
                        acc += w0[i];
                        pf[i] = acc;
                    }
                }
            CK(ctx, cudaMemcpyAsync(const_cast<double*>(m.w0), w0, 2 * n3 * sizeof(double),
                                    cudaMemcpyHostToDevice, ctx->stream));
        }
        if (ctx->lay.uthr_entries && c.levels > 2) {
            // uniform neighbourhood (all NB neighbours carry s*): the oracle's per-site law
            // (max-subtracted softmax, ascending cumulative sum) in the same fp64 order, and
            // T_k = ceil(F_k 2^32) - 1 so that "u < F_k" <=> "r <= T_k".
            const int L = c.levels, NB = c.neighborhood;
            std::vector<double> E(L), pr(L);
            uint32_t* out = ctx->uthr_host.data();
            for (int s0 = 0; s0 < L; ++s0)
                for (int gl = 0; gl < L; ++gl)
                    for (int xl = 0; xl < L; ++xl) {
                        double Emax = -INFINITY;
                        for (int s = 0; s < L; ++s) {
                            const double d = lum(gl, L) - lum(s, L);
                            const double inert = inertia_pen(c.inertia_p, xl, s, L);
                            const int n = (s == s0) ? NB : 0;
                            E[s] = a * (double)n - b * d * d - cq * inert;
                            if (E[s] > Emax) Emax = E[s];
                        }
                        double Z = 0.0;
                        for (int s = 0; s < L; ++s) {
                            pr[s] = exp(E[s] - Emax);
                            Z += pr[s];
                        }
                        for (int s = 0; s < L; ++s) pr[s] = pr[s] / Z;
                        double F = 0.0;
                        for (int k = 0; k < L - 1; ++k) {
                            F += pr[k];
                            const double T = ceil(F * 4294967296.0);
                            *out++ = T < 1.0 ? 0u : (T > 4294967296.0 ? 0xFFFFFFFFu : (uint32_t)(T - 1.0));
                        }
                    }
            // pageable host -> device: the source is staged before the call returns, and the
            // copy is stream-ordered after every sweep of the previous stage
            CK(ctx, cudaMemcpyAsync(ctx->uthr, ctx->uthr_host.data(),
                                    ctx->uthr_host.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                    ctx->stream));
        }
    }
    // the TABLE kernel runs a stage only when its fp64 path needs no log-domain fallback:
    // Z >= A[n_x] D[g][x] >= exp(-b) and Z <= L A[NB] (weights <= 1 but A); otherwise the
    // general kernel (which has the oracle's log-domain form) sweeps this stage
    if (ctx->kernel == PCA_KERNEL_TABLE) {
        const bool safe = exp(-b) >= 1e-290 && (double)c.levels * ctx->gen.A[c.neighborhood] <= 1e290;
        ctx->gen.tab = safe ? ctx->ws + ctx->lay.off_tab : nullptr;
    }
    if (ctx->gen.tab) {
        // the TABLE kernel's blob (kernels.cuh): A, W0 = D I, the slot table, and for every
        // key histogram and (g, x) the oracle's per-site law (max-subtracted softmax,
        // ascending cumulative sum, fp64, the uthr arithmetic) as thresholds T_k
        const int L = c.levels, NB = c.neighborhood, TP = tab_tp_host(L);
        const TabKeys& K = tab_keys(L, NB);
        GeneralSweepParams& m = ctx->gen;
        uint8_t* blob = ctx->tab_host.data();
        std::fill(ctx->tab_host.begin(), ctx->tab_host.end(), 0);
        memcpy(blob, m.A, 9 * sizeof(double));
        // AW[g][x][s][n] = A[n] * W0[g][x][s], W0 = D I: the fp64 products the rare path forms
        // (IEEE multiplication: the device reading them decides exactly as if it multiplied)
        double* aw = reinterpret_cast<double*>(blob + TAB_OFF_W0);
        for (int gl = 0; gl < L; ++gl)
            for (int xl = 0; xl < L; ++xl)
                for (int s = 0; s < L; ++s) {
                    const double w0 = ctx->dtab_host[(size_t)gl * L + s] * exp(-cq * inertia_pen(c.inertia_p, xl, s, L));
                    for (int n = 0; n < 9; ++n) aw[(((gl * L + xl) * L) + s) * 9 + n] = m.A[n] * w0;
                }
        uint32_t* slot = reinterpret_cast<uint32_t*>(blob + m.tab_slots);
        for (int i = 0; i < (1 << K.hbits); ++i) {
            slot[2 * i] = 0xFFFFFFFFu;
            slot[2 * i + 1] = 0u;
        }
        uint32_t* thr = reinterpret_cast<uint32_t*>(blob + m.tab_thr);
        std::vector<double> E(L), pr(L);
        for (size_t key = 0; key < K.h.size(); ++key) {
            const uint32_t sl = (K.h[key] * K.magic) >> (32 - K.hbits);
            slot[2 * sl] = K.h[key];
            slot[2 * sl + 1] = (uint32_t)(key * L * L * TP * 4);
            for (int gl = 0; gl < L; ++gl)
                for (int xl = 0; xl < L; ++xl) {
                    double Emax = -INFINITY;
                    for (int s = 0; s < L; ++s) {
                        const double d = lum(gl, L) - lum(s, L);
                        const double inert = inertia_pen(c.inertia_p, xl, s, L);
                        E[s] = a * (double)K.n[key][s] - b * d * d - cq * inert;
                        if (E[s] > Emax) Emax = E[s];
                    }
                    double Z = 0.0;
                    for (int s = 0; s < L; ++s) {
                        pr[s] = exp(E[s] - Emax);
                        Z += pr[s];
                    }
                    for (int s = 0; s < L; ++s) pr[s] = pr[s] / Z;
                    uint32_t* out = thr + ((key * L + gl) * L + xl) * TP;
                    double F = 0.0;
                    for (int k = 0; k < L - 1; ++k) {
                        F += pr[k];
                        const double T = ceil(F * 4294967296.0);
                        out[k] = T < 1.0 ? 0u : (T > 4294967296.0 ? 0xFFFFFFFFu : (uint32_t)(T - 1.0));
                    }
                }
        }
        CK(ctx, cudaMemcpyAsync(const_cast<uint8_t*>(m.tab), blob, m.tab_bytes, cudaMemcpyHostToDevice,
                                ctx->stream));
    }
    ctx->tab_stage = stage;
    ctx->beta_last = beta;
    return PCA_OK;
}

// Gibbs tables for the stage of sweep t: the conditional of PAPER.md:417-429 (no inertia),
// E_s = a n_s - b d_s^2, softmax and cumulative sum in the oracle's fp64 order.
pca_status build_gibbs_tables(pca_ctx* ctx, int64_t t) {
    const pca_config& c = ctx->cfg;
    const int64_t stage = t / c.beta_period;
    if (stage == ctx->gtab_stage) return PCA_OK;
    const double beta = beta_at(c, t);
    const double a = c.coef_scale * 2.0 * beta * c.J;
    const double b = c.coef_scale / (2.0 * c.sigma * c.sigma);
    GibbsSweepParams& m = ctx->gib;
    for (int n = 0; n <= 8; ++n) m.A[n] = exp(a * (double)n);
    m.coef_a = a;
    m.coef_b = b;
    const int L = c.levels;
    // cumulative thresholds T_k = ceil(F_k 2^32) - 1 of the law with label counts n[]
    auto thresholds = [&](const int* n, int gl, uint32_t* out) {
        double E[UTHR_MAX_LEVELS], pr[UTHR_MAX_LEVELS];
        double Emax = -INFINITY;
        for (int s = 0; s < L; ++s) {
            const double d = lum(gl, L) - lum(s, L);
            E[s] = a * (double)n[s] - b * d * d;
            if (E[s] > Emax) Emax = E[s];
        }
        double Z = 0.0;
        for (int s = 0; s < L; ++s) {
            pr[s] = exp(E[s] - Emax);
            Z += pr[s];
        }
        for (int s = 0; s < L; ++s) pr[s] = pr[s] / Z;
        double F = 0.0;
        for (int k = 0; k < L - 1; ++k) {
            F += pr[k];
            const double T = ceil(F * 4294967296.0);
            out[k] = T < 1.0 ? 0u : (T > 4294967296.0 ? 0xFFFFFFFFu : (uint32_t)(T - 1.0));
        }
    };
    if (L == 2) {
        for (int np = 0; np <= 8; ++np)
            for (int n1 = 0; n1 <= 8; ++n1)
                for (int gl = 0; gl < 2; ++gl) {
                    uint32_t* out = &m.thr2[(np * 9 + n1) * 2 + gl];
                    if (n1 > np) {
                        *out = 0u;
                        continue;
                    }
                    const int n[2] = {np - n1, n1};
                    thresholds(n, gl, out);
                }
        ParamTable pt;
        for (int i = 0; i < GIBBS_THR_PAD; ++i) pt.v[i] = i < GIBBS_THR2 ? m.thr2[i] : 0u;
        LAUNCH(ctx, launch_param_table(pt, GIBBS_THR_PAD, const_cast<uint32_t*>(ctx->gbin.thr), ctx->stream));
    } else if (ctx->lay.gthr_entries) {
        const int NB = c.neighborhood;
        int n[UTHR_MAX_LEVELS];
        uint32_t* out = ctx->gthr_host.data();
        for (int s0 = 0; s0 < L; ++s0) {
            for (int s = 0; s < L; ++s) n[s] = (s == s0) ? NB : 0;
            for (int gl = 0; gl < L; ++gl, out += L - 1) thresholds(n, gl, out);
        }
        CK(ctx, cudaMemcpyAsync(ctx->gthr, ctx->gthr_host.data(),
                                ctx->gthr_host.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                ctx->stream));
    }
    ctx->gtab_stage = stage;
    return PCA_OK;
}

void fill_common(pca_ctx* ctx, SweepCommon& sc, int64_t t, int count) {
    sc.geo = ctx->geo;
    sc.x_in = ctx->x[ctx->cur];
    sc.x_out = ctx->x[ctx->cur ^ 1];
    sc.g = ctx->g;
    sc.counts = ctx->counts;
    const uint32_t k0 = (uint32_t)(ctx->cfg.seed & 0xFFFFFFFFu);
    const uint32_t k1 = (uint32_t)(ctx->cfg.seed >> 32);
    for (int i = 0; i < 10; ++i) {
        sc.keys.rk[2 * i] = k0 + (uint32_t)i * 0x9E3779B9u;
        sc.keys.rk[2 * i + 1] = k1 + (uint32_t)i * 0xBB67AE85u;
    }
    sc.t = (uint32_t)t;
    sc.chain0 = (uint32_t)ctx->cfg.chain0;
    sc.count_enable = count;
    sc.peer_up = sc.peer_dn = nullptr;
    sc.peer_up_chain = sc.peer_dn_chain = 0;
}

// ---- device-initiated halo exchange (pca_attach_peers) ----
// Phase protocol, per context: every state load and every sweep is one phase k = ++phase.
// Before a phase touches peer memory or reads its own halo rows it waits (on the stream, no
// spinning kernel) until both peers have completed phase k-1: their pushes into our halo
// rows are then complete, and they no longer read the halo rows of the buffer we are about
// to write into (the double buffer alternates, so that is the buffer they read in phase
// k-1).  After the phase's work, a stream write (with a system-wide fence before it) tells
// each peer that we completed phase k.
struct StreamMemOps {
    using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    WaitFn wait = nullptr;
    WriteFn write = nullptr;
    std::string why;
};
StreamMemOps& memops() {
    static StreamMemOps m = [] {
        StreamMemOps o;
        cudaDriverEntryPointQueryResult q1, q2;
        void* w = nullptr;
        void* x = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) != cudaSuccess ||
            q1 != cudaDriverEntryPointSuccess ||
            cudaGetDriverEntryPoint("cuStreamWriteValue32", &x, cudaEnableDefault, &q2) != cudaSuccess ||
            q2 != cudaDriverEntryPointSuccess) {
            o.why = "cuStreamWaitValue32 / cuStreamWriteValue32 unavailable";
            return o;
        }
        o.wait = (StreamMemOps::WaitFn)w;
        o.write = (StreamMemOps::WriteFn)x;
        return o;
    }();
    return m;
}

pca_status p2p_begin(pca_ctx* ctx, uint32_t k) {
    StreamMemOps& M = memops();
    for (int i = 0; i < 2; ++i) {
        if (!(i == 0 ? ctx->has_up : ctx->has_dn)) continue;
        const CUresult r = M.wait((CUstream)ctx->stream, (CUdeviceptr)(ctx->pflags + i), k - 1,
                                  CU_STREAM_WAIT_VALUE_GEQ);
        if (r != CUDA_SUCCESS) {
            ctx->poisoned = 1;
            return fail(PCA_ECUDA, "cuStreamWaitValue32 (peer phase): CUresult %d", (int)r);
        }
    }
    return PCA_OK;
}

pca_status p2p_end(pca_ctx* ctx, uint32_t k) {
    StreamMemOps& M = memops();
    // we are the up peer's down peer (its slot 1) and the down peer's up peer (its slot 0)
    if (ctx->has_up) {
        const CUresult r = M.write((CUstream)ctx->stream, (CUdeviceptr)(ctx->up.flags + 1), k, 0);
        if (r != CUDA_SUCCESS) return fail(PCA_ECUDA, "cuStreamWriteValue32 (up peer): CUresult %d", (int)r);
    }
    if (ctx->has_dn) {
        const CUresult r = M.write((CUstream)ctx->stream, (CUdeviceptr)(ctx->dn.flags + 0), k, 0);
        if (r != CUDA_SUCCESS) return fail(PCA_ECUDA, "cuStreamWriteValue32 (down peer): CUresult %d", (int)r);
    }
    ctx->phase = k;
    return PCA_OK;
}

// Copy the first / last `depth` owned rows of buffer `b` into the peers' halo rows of their
// buffer b (the copies of a phase whose kernel did not store them itself).
pca_status p2p_copy_edges(pca_ctx* ctx, int b, int depth) {
    const size_t pitch = (size_t)ctx->lay.xpitch, R = (size_t)ctx->lay.rows;
    const size_t rb = (size_t)depth * pitch;
    uint8_t* mine = ctx->x[b];
    for (int c = 0; c < ctx->cfg.batch; ++c) {
        uint8_t* base = mine + (size_t)c * ctx->geo.xchain;
        if (ctx->has_up) {  // our rows 0..depth-1 -> the up peer's rows below its strip
            uint8_t* dst = ctx->up.x[b] + (size_t)c * ctx->up.chain_stride + (HALO + (size_t)ctx->up.rows) * pitch;
            CK(ctx, cudaMemcpyAsync(dst, base + HALO * pitch, rb, cudaMemcpyDeviceToDevice, ctx->stream));
        }
        if (ctx->has_dn) {  // our last depth rows -> the down peer's rows above its strip
            uint8_t* dst = ctx->dn.x[b] + (size_t)c * ctx->dn.chain_stride + (size_t)(HALO - depth) * pitch;
            CK(ctx, cudaMemcpyAsync(dst, base + (HALO + R - depth) * pitch, rb, cudaMemcpyDeviceToDevice,
                                    ctx->stream));
        }
    }
    return PCA_OK;
}

// A phase that rewrote buffer `b` outside a sweep kernel (a state load): its HALO edge rows
// to the peers, with the protocol.
pca_status p2p_push(pca_ctx* ctx, int b) {
    const uint32_t k = ctx->phase + 1;
    pca_status st = p2p_begin(ctx, k);
    if (st != PCA_OK) return st;
    st = p2p_copy_edges(ctx, b, HALO);
    if (st != PCA_OK) return st;
    return p2p_end(ctx, k);
}

// Halo exchange of buffer `buf` with the neighbouring ranks (row strips): send the first
// `depth` owned rows up and the last `depth` down, receive the halo rows.  Order per chain:
// send(top->up), recv(bottom halo<-down), send(bottom->down), recv(top halo<-up); with
// 2 ranks on a torus both neighbours are the same peer and NCCL matches in issue order.
// (any padded per-chain buffer: `halo` halo rows above the owned rows, `pitch` bytes per row,
// `chain_stride` bytes per chain)
pca_status exchange_rows(pca_ctx* ctx, uint8_t* buf, size_t pitch, size_t chain_stride, int halo,
                         int depth) {
    if (!ctx->comm || ctx->nranks <= 1) return PCA_OK;
    NvtxRange nvtx_("halo exchange (NCCL)");
    NcclApi& N = nccl();
    const int P = ctx->nranks, r = ctx->rank;
    int up = r - 1, down = r + 1;
    if (ctx->cfg.periodic) {
        up = (r + P - 1) % P;
        down = (r + 1) % P;
    } else {
        if (up < 0) up = -1;
        if (down >= P) down = -1;
    }
    // `depth` consecutive padded rows per message (rows are contiguous in the buffer)
    const size_t rb = (size_t)depth * pitch;
    const size_t R = (size_t)ctx->lay.rows;
    ncclResult_t e = N.GroupStart();
    for (int b = 0; b < ctx->cfg.batch && e == ncclSuccess; ++b) {
        uint8_t* base = buf + (size_t)b * chain_stride;                           // row -halo
        uint8_t* top = base + halo * pitch;                                       // rows 0..
        uint8_t* bottom = base + (halo + R - depth) * pitch;                      // rows R-depth..
        uint8_t* halo_top = base + (halo - depth) * pitch;                        // rows -depth..
        uint8_t* halo_bottom = base + (halo + R) * pitch;                         // rows R..
        if (up >= 0 && e == ncclSuccess) e = N.Send(top, rb, ncclUint8, up, ctx->comm, ctx->stream);
        if (down >= 0 && e == ncclSuccess)
            e = N.Recv(halo_bottom, rb, ncclUint8, down, ctx->comm, ctx->stream);
        if (down >= 0 && e == ncclSuccess)
            e = N.Send(bottom, rb, ncclUint8, down, ctx->comm, ctx->stream);
        if (up >= 0 && e == ncclSuccess) e = N.Recv(halo_top, rb, ncclUint8, up, ctx->comm, ctx->stream);
    }
    ncclResult_t e2 = N.GroupEnd();
    if (e == ncclSuccess) e = e2;
    if (e != ncclSuccess) {
        ctx->poisoned = 1;
        return fail(PCA_ENCCL, "halo exchange: %s", N.GetErrorString(e));
    }
    return PCA_OK;
}

pca_status exchange(pca_ctx* ctx, uint8_t* buf, int depth = HALO) {
    return exchange_rows(ctx, buf, (size_t)ctx->lay.xpitch, (size_t)ctx->geo.xchain, HALO, depth);
}

// the observed image's edge rows into the neighbours' g halo rows (strips sweeping two
// sweeps per pass recompute one row beyond their strip, which needs its g; g changes only on
// a reset): NCCL, or one peer phase of copies
pca_status exchange_g(pca_ctx* ctx) {
    const size_t gp = (size_t)ctx->lay.gpitch, R = (size_t)ctx->lay.rows;
    if (ctx->p2p) {
        const uint32_t k = ctx->phase + 1;
        pca_status st = p2p_begin(ctx, k);
        if (st != PCA_OK) return st;
        for (int c = 0; c < ctx->cfg.batch; ++c) {
            const uint8_t* base = ctx->g + (size_t)c * ctx->geo.gchain;
            if (ctx->has_up) {  // our row 0 -> the up peer's row below its strip
                uint8_t* dst = ctx->peer_g[0] + (size_t)c * (GHALO * 2 + (size_t)ctx->up.rows) * gp +
                               (GHALO + (size_t)ctx->up.rows) * gp;
                CK(ctx, cudaMemcpyAsync(dst, base + GHALO * gp, gp, cudaMemcpyDeviceToDevice, ctx->stream));
            }
            if (ctx->has_dn) {  // our last row -> the down peer's row above its strip
                uint8_t* dst = ctx->peer_g[1] + (size_t)c * (GHALO * 2 + (size_t)ctx->dn.rows) * gp;
                CK(ctx, cudaMemcpyAsync(dst, base + (GHALO + R - 1) * gp, gp, cudaMemcpyDeviceToDevice,
                                        ctx->stream));
            }
        }
        return p2p_end(ctx, k);
    }
    return exchange_rows(ctx, ctx->g, gp, (size_t)ctx->geo.gchain, GHALO, GHALO);
}

// `checked` = src is known to hold labels < levels (the validated g, or bits unpacked by
// packed_io): the level check and its host synchronisation are skipped
pca_status load_state(pca_ctx* ctx, const uint8_t* src, int pitch, long long chain_stride,
                      const char* what, bool checked = false) {
    ctx->prev_valid = 0;
    ctx->x_ok = 0;
    CK(ctx, cudaMemsetAsync(ctx->flag, 0, sizeof(int), ctx->stream));
    LAUNCH(ctx, launch_pack_state(ctx->geo, src, pitch, chain_stride, ctx->x[ctx->cur],
                                  ctx->cfg.batch, ctx->flag, ctx->stream));
    if (!checked) {
        pca_status st = check_flag(ctx, what);
        if (st != PCA_OK) return st;
    }
    ctx->x_ok = 1;
    if (ctx->p2p) return p2p_push(ctx, ctx->cur);
    return exchange(ctx, ctx->x[ctx->cur]);
}

pca_status do_reset(pca_ctx* ctx, const uint8_t* g, const uint8_t* x0, bool staged = false) {
    const pca_config& c = ctx->cfg;
    const Layout& L = ctx->lay;
    // x0 = g on an initialised context: the g pass also writes x[0], the state the reset
    // starts from, so the input is read once (a failed level check leaves x[0] overwritten,
    // like g: the context needs a valid reset either way)
    const bool fused_x = g && !x0 && ctx->x_initialized;
    if (fused_x) ctx->x_ok = 0;  // the g pass writes x[0] before its check
    if (g) {
        ctx->g_ok = 0;
        ctx->gpk_valid = 0;
        ctx->g_halo_valid = 0;
        const uint8_t* dg = nullptr;
        pca_status st = device_input(ctx, g, &dg);
        if (st != PCA_OK) return st;
        CK(ctx, cudaMemsetAsync(ctx->g, 0, L.gbuf, ctx->stream));
        CK(ctx, cudaMemsetAsync(ctx->flag, 0, sizeof(int), ctx->stream));
        LAUNCH(ctx, launch_pack_g(ctx->geo, dg, c.width, (long long)L.rows * c.width, ctx->g,
                                  c.batch, ctx->flag, ctx->stream, fused_x ? ctx->x[0] : nullptr));
        // the check's host synchronisation also ends the caller's buffer lifetime at return;
        // it is skipped only for the context's own staged copy holding bit-unpacked labels
        // (packed_io, levels == 2: 0/1 by construction)
        if (!(staged && c.packed_io)) {
            st = check_flag(ctx, "g");
            if (st != PCA_OK) return st;
        }
        ctx->g_ok = 1;
    }
    // free boundary: halos and padding hold the sentinel 0xFF; torus: halos are rewritten by
    // every sweep and padding is 0 (a valid label, so SWAR sums need no masking)
    // (only once: no kernel ever writes a free-boundary halo or a padding byte)
    if (!ctx->x_initialized) {
        const int fill = c.periodic ? 0 : 0xFF;
        CK(ctx, cudaMemsetAsync(ctx->x[0], fill, L.xbuf, ctx->stream));
        CK(ctx, cudaMemsetAsync(ctx->x[1], fill, L.xbuf, ctx->stream));
        ctx->x_initialized = 1;
    }
    CK(ctx, cudaMemsetAsync(ctx->counts, 0, L.counts_bytes, ctx->stream));
    ctx->cur = 0;
    ctx->prev_valid = 0;
    ctx->t = 0;
    ctx->counted = 0;
    ctx->tab_stage = -1;
    ctx->beta_last = c.beta0;
    if (x0) {
        const uint8_t* dx = nullptr;
        pca_status st = device_input(ctx, x0, &dx);
        if (st != PCA_OK) return st;
        return load_state(ctx, dx, c.width, (long long)L.rows * c.width, "x0");
    }
    if (fused_x) {  // x[0] was written by the g pass: only the halo exchange is left
        ctx->x_ok = 1;
        if (ctx->p2p) return p2p_push(ctx, ctx->cur);
        return exchange(ctx, ctx->x[ctx->cur]);
    }
    // x0 = g: g's labels were checked when it was loaded
    return load_state(ctx, ctx->g + (size_t)GHALO * L.gpitch + XOFF, L.gpitch, ctx->geo.gchain, "g",
                      true);
}

// n sweeps on the bit-packed state (PCA_KERNEL_PACKED): the byte state x[cur] is packed once,
// the n sweeps ping-pong between the packed buffers, and the last two states (x_t, x_{t-1})
// are unpacked into the byte buffers, which stay the canonical state for every other call.
pca_status sweep_packed_run(pca_ctx* ctx, int32_t n) {
    const pca_config& c = ctx->cfg;
    const int B = c.batch;
    const bool strip = ctx->lay.rows < c.height;
    if (!ctx->gpk_valid) {
        LAUNCH(ctx, launch_g_to_packed(ctx->geo, ctx->g, ctx->gpk, ctx->pk.gpp, ctx->pk.gchain, B, ctx->stream));
        ctx->gpk_valid = 1;
    }
    LAUNCH(ctx, launch_state_to_packed(ctx->geo, ctx->x[ctx->cur], ctx->xp[0], ctx->pk.pp, ctx->pk.xchain, B,
                                       ctx->stream));
    int pc = 0;
    int pending = 0;  // counted sweeps in the delta plane (< 256: a byte cannot overflow)
    auto fold = [&]() -> pca_status {
        if (pending) {
            LAUNCH(ctx, launch_fold_counts(ctx->geo, ctx->counts, ctx->pk.dcounts, ctx->pk.dchain, B,
                                           ctx->stream));
            pending = 0;
        }
        return PCA_OK;
    };
    // a refused sweep (sweep index or counter limit) ends the run after the sweeps already
    // done: their counts are folded and their state unpacked, as at the end of a full run
    pca_status refused = PCA_OK;
    int32_t done = 0;
    for (int32_t i = 0; i < n; ++i) {
        const int64_t t = ctx->t;
        if (t >= (int64_t)0xFFFFFFFFLL) {
            refused = fail(PCA_EUNSUPPORTED, "sweep index exceeds 2^32-1");
            break;
        }
        pca_status st = build_tables(ctx, t);
        if (st != PCA_OK) return st;
        const int count = (c.mpm_burn_in >= 0 && t >= c.mpm_burn_in) ? 1 : 0;
        if (count && ctx->counted + 1 > 65535) {
            refused = fail(PCA_EUNSUPPORTED, "more than 65535 counted sweeps overflow uint16 counts");
            break;
        }
        fill_common(ctx, ctx->pk.c, t, count);
        ctx->pk.x_in = ctx->xp[pc];
        ctx->pk.x_out = ctx->xp[pc ^ 1];
        ctx->pk.g = ctx->gpk;
        ctx->pk.thr = ctx->bin.thr;
        const int R = ctx->lay.rows;
        auto launch_packed_rows = [&](int rlo, int rhi, cudaStream_t s) -> int {
            ctx->launches++;
            ctx->sweep_launches++;
            ctx->pk.c.rlo = rlo;
            ctx->pk.c.rhi = rhi;
            return launch_sweep_packed(ctx->pk, B, s);
        };
        if (strip && R >= 3) {
            // a row strip: the two edge rows first, then (over NCCL) their packed rows (W/8 + 32
            // bytes each) to the neighbours on the main stream, overlapping the interior rows on
            // the side stream (the byte kernels' schedule, pca_sweep); a caller-exchanged strip
            // takes the same launches with no exchange
            if (!ctx->side) {
                CK(ctx, cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
                CK(ctx, cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
                CK(ctx, cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
            }
            CK(ctx, cudaEventRecord(ctx->ev_fork, ctx->stream));
            CK(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            int e = launch_packed_rows(0, 1, ctx->stream);
            if (!e) e = launch_packed_rows(R - 1, R, ctx->stream);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep (packed edge rows)");
            st = exchange_rows(ctx, ctx->xp[pc ^ 1], (size_t)ctx->pk.pp, (size_t)ctx->pk.xchain, HALO, 1);
            if (st != PCA_OK) return st;
            e = launch_packed_rows(1, R - 1, ctx->side);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep (packed interior rows)");
            CK(ctx, cudaEventRecord(ctx->ev_join, ctx->side));
            CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
        } else {
            const int e = launch_packed_rows(0, R, ctx->stream);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep (packed)");
            if (strip) {  // fewer than 3 rows (no exchange for a caller-exchanged strip)
                st = exchange_rows(ctx, ctx->xp[pc ^ 1], (size_t)ctx->pk.pp, (size_t)ctx->pk.xchain, HALO, 1);
                if (st != PCA_OK) return st;
            }
        }
        pc ^= 1;
        ctx->t = t + 1;
        ctx->counted += count;
        ++done;
        pending += count;
        if (pending == 255) {
            st = fold();
            if (st != PCA_OK) return st;
        }
    }
    pca_status st = fold();  // the canonical uint16 counts are complete again
    if (st != PCA_OK) return st;
    if (done == 0) return refused;  // nothing swept: the byte state is current
    const int cur = ctx->cur ^ (done & 1);
    // the halo rows hold real rows where a neighbour is (a torus, or a strip's neighbouring
    // rank); a free boundary's outer halo rows keep the byte buffers' sentinel
    const int hu = c.periodic || c.row0 > 0, hd = c.periodic || c.row0 + ctx->lay.rows < c.height;
    LAUNCH(ctx, launch_state_from_packed(ctx->geo, ctx->xp[pc], ctx->pk.pp, ctx->pk.xchain, ctx->x[cur], B,
                                         ctx->stream, hu, hd));
    LAUNCH(ctx, launch_state_from_packed(ctx->geo, ctx->xp[pc ^ 1], ctx->pk.pp, ctx->pk.xchain,
                                         ctx->x[cur ^ 1], B, ctx->stream, hu, hd));
    ctx->cur = cur;
    ctx->prev_valid = 1;
    // a strip over NCCL: the byte state's 2-deep halos from the neighbours (the packed runs
    // exchanged 1-deep packed halos only); a caller-exchanged strip's caller does this
    if (strip) {
        st = exchange(ctx, ctx->x[ctx->cur]);
        if (st != PCA_OK) return st;
    }
    return refused;
}

}  // namespace

// ===========================================================================
extern "C" {

int32_t pca_abi_version(void) { return PCA_ABI_VERSION; }

const char* pca_last_error(void) { return g_err.c_str(); }

size_t pca_workspace_bytes(const pca_config* cfg) {
    if (validate(cfg) != PCA_OK) return 0;
    return make_layout(cfg).total;
}

pca_status pca_init(pca_ctx** out, const pca_config* cfg, void* workspace, size_t ws_bytes,
                    const uint8_t* g, const uint8_t* x0, void* stream) {
    if (!out) return fail(PCA_EINVAL, "out is NULL");
    *out = nullptr;
    pca_status st = validate(cfg);
    if (st != PCA_OK) return st;
    if (!workspace || !g) return fail(PCA_EINVAL, "workspace and g must be non-NULL");
    if (((uintptr_t)workspace & 255u) != 0) return fail(PCA_EINVAL, "workspace must be 256-B aligned");
    const Layout L = make_layout(cfg);
    if (ws_bytes < L.total)
        return fail(PCA_ENOSPACE, "workspace has %zu bytes, needs %zu", ws_bytes, L.total);
    if (!is_device_ptr(workspace)) return fail(PCA_EINVAL, "workspace must be device memory");

    pca_ctx* ctx = new (std::nothrow) pca_ctx();
    if (!ctx) return fail(PCA_EINVAL, "out of host memory");
    ctx->cfg = *cfg;
    if (ctx->cfg.rows == 0) ctx->cfg.rows = cfg->height;
    ctx->lay = L;
    cudaGetDevice(&ctx->device);
    ctx->stream = (cudaStream_t)stream;
    ctx->ws = (uint8_t*)workspace;
    ctx->x[0] = ctx->ws + L.off_x0;
    ctx->x[1] = ctx->ws + L.off_x1;
    ctx->g = ctx->ws + L.off_g;
    ctx->counts = (uint16_t*)(ctx->ws + L.off_counts);
    ctx->dtab = (double*)(ctx->ws + L.off_dtab);
    ctx->itab = (double*)(ctx->ws + L.off_itab);
    ctx->itab_host.resize((size_t)cfg->levels * cfg->levels);
    ctx->sums = (unsigned long long*)(ctx->ws + L.off_sums);
    ctx->sums_max = (unsigned long long*)(ctx->ws + L.off_sums_max);
    ctx->flag = (int*)(ctx->ws + L.off_flag);
    ctx->pflags = (uint32_t*)(ctx->ws + L.off_flag + 64);
    ctx->stage = ctx->ws + L.off_stage;
    ctx->truth = ctx->ws + L.off_truth;
    ctx->io_in = ctx->ws + L.off_io;
    ctx->io_out = ctx->io_in + align256(L.io_bytes);
    ctx->io_truth = ctx->io_out + align256(L.io_bytes);
    ctx->in_stage = ctx->ws + L.off_in;
    ctx->uthr = L.uthr_entries ? (uint32_t*)(ctx->ws + L.off_uthr) : nullptr;
    ctx->uthr_host.resize(L.uthr_entries);
    ctx->sparse_host.resize(2 * L.sparse_entries);
    ctx->gen.w0 = L.sparse_entries ? (const double*)(ctx->ws + L.off_sparse) : nullptr;
    ctx->gen.pfx = L.sparse_entries ? ctx->gen.w0 + L.sparse_entries : nullptr;
    ctx->gthr = L.gthr_entries ? (uint32_t*)(ctx->ws + L.off_gthr) : nullptr;
    ctx->gthr_host.resize(L.gthr_entries);
    // AUTO: two levels on the bit-packed state when the context owns a whole lattice of width
    // % 512 == 0 (80.2 vs 83.6 us per 8192^2 sweep with MPM), else the byte
    // kernel; 3..5 levels on the histogram tables; else the general kernel
    ctx->kernel = (cfg->kernel == PCA_KERNEL_AUTO)
                      ? (cfg->levels == 2
                             ? (packed_eligible(cfg) && cfg->sweeps_per_pass != 2 ? PCA_KERNEL_PACKED
                                                                                  : PCA_KERNEL_BINARY)
                             : (table_eligible(cfg) ? PCA_KERNEL_TABLE : PCA_KERNEL_GENERAL))
                      : cfg->kernel;
    if (ctx->kernel == PCA_KERNEL_PACKED) {
        ctx->xp[0] = ctx->ws + L.off_xp;
        ctx->xp[1] = ctx->xp[0] + align256(L.xp_bytes);
        ctx->gpk = ctx->ws + L.off_gp;
        ctx->pk.pp = L.pp;
        ctx->pk.gpp = L.gpp;
        ctx->pk.xchain = (long long)(L.rows + 2 * HALO) * L.pp;
        ctx->pk.gchain = (long long)L.rows * L.gpp;
        ctx->pk.dcounts = ctx->ws + L.off_dc;
        ctx->pk.dchain = (long long)L.rows * L.cpitch;
    }
    ctx->gen.tab = nullptr;
    ctx->gen.tdc = nullptr;
    if (ctx->kernel == PCA_KERNEL_TABLE && L.dc_bytes == 0) ctx->kernel = PCA_KERNEL_GENERAL;  // (not expected)
    if (ctx->kernel == PCA_KERNEL_TABLE) {
        ctx->gen.tdc = ctx->ws + L.off_dc;
        ctx->gen.tdc_plane = (long long)L.rows * L.cpitch;
        ctx->gen.tdc_chain = (long long)cfg->levels * ctx->gen.tdc_plane;
        const TabKeys& K = tab_keys(cfg->levels, cfg->neighborhood);
        if (K.ok) {
            ctx->gen.tab = ctx->ws + L.off_tab;
            ctx->gen.tab_magic = K.magic;
            ctx->gen.tab_hbits = K.hbits;
            ctx->gen.tab_slots = (uint32_t)tab_slots_off(cfg->levels);
            ctx->gen.tab_thr = ctx->gen.tab_slots + (8u << K.hbits);
            ctx->gen.tab_bytes = (uint32_t)tab_blob_bytes(cfg->levels, cfg->neighborhood, K.hbits);
            ctx->tab_host.assign(ctx->gen.tab_bytes, 0);
        } else {
            ctx->kernel = PCA_KERNEL_GENERAL;  // no collision-free hash (not expected)
        }
    }
    ctx->rows_per_thread = cfg->rows_per_thread;

    Geometry& G = ctx->geo;
    G.W = cfg->width;
    G.rows = L.rows;
    G.H = cfg->height;
    G.row0 = cfg->row0;
    G.nchunks = L.nchunks;
    G.levels = cfg->levels;
    G.nbhd = cfg->neighborhood;
    G.periodic = cfg->periodic;
    G.self_halo_rows = (cfg->periodic && L.rows == cfg->height) ? 1 : 0;
    G.xpitch = L.xpitch;
    G.gpitch = L.gpitch;
    G.cpitch = L.cpitch;
    G.xchain = (long long)(L.rows + 2 * HALO) * L.xpitch;
    G.gchain = (long long)(L.rows + 2 * GHALO) * L.gpitch;
    G.cplane = (long long)L.rows * L.cpitch;
    G.cchain = (long long)L.cplanes * L.rows * L.cpitch;

    // D[g][s] = exp(-b (lum g - lum s)^2): beta-independent (R5), built once.
    const double b = cfg->coef_scale / (2.0 * cfg->sigma * cfg->sigma);
    ctx->dtab_host.resize((size_t)cfg->levels * cfg->levels);
    for (int gl = 0; gl < cfg->levels; ++gl)
        for (int s = 0; s < cfg->levels; ++s) {
            const double d = lum(gl, cfg->levels) - lum(s, cfg->levels);
            ctx->dtab_host[(size_t)gl * cfg->levels + s] = exp(-b * d * d);
        }
    ctx->gen.dtab = ctx->dtab;
    ctx->gen.itab = ctx->itab;
    ctx->gen.inertia_p = cfg->inertia_p;
    ctx->gen.uthr = ctx->uthr;
    ctx->bin.thr = (const uint32_t*)(ctx->ws + L.off_bthr);
    ctx->gen.bthr = ctx->bin.thr;
    ctx->gib.dtab = ctx->dtab;
    ctx->gbin.thr = (const uint32_t*)(ctx->ws + L.off_gbthr);
    ctx->gib.uthr = ctx->gthr;

    auto bail = [&](pca_status s) {
        delete ctx;
        return s;
    };
    cudaError_t e = cudaMemcpyAsync(ctx->dtab, ctx->dtab_host.data(),
                                    ctx->dtab_host.size() * sizeof(double), cudaMemcpyHostToDevice,
                                    ctx->stream);
    if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "upload dtab"));
    e = cudaMemsetAsync(ctx->pflags, 0, 2 * sizeof(uint32_t), ctx->stream);
    if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "clear peer flags"));
    if (ctx->xp[0]) {  // packed pads and (free boundary) halo rows stay zero
        e = cudaMemsetAsync(ctx->xp[0], 0, 2 * align256(L.xp_bytes), ctx->stream);
        if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "clear packed state"));
    }
    if (L.dc_bytes) {  // count deltas (packed or table kernel) start at 0
        e = cudaMemsetAsync(ctx->ws + L.off_dc, 0, L.dc_bytes, ctx->stream);
        if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "clear count deltas"));
    }
    st = do_reset(ctx, g, x0);
    if (st != PCA_OK) return bail(st);
    *out = ctx;
    return PCA_OK;
}

pca_status pca_reset(pca_ctx* ctx, const uint8_t* g, const uint8_t* x0) {
    DeviceScope device_scope_;
    NvtxRange nvtx_("pca_reset");
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    return do_reset(ctx, g, x0);
}

static pca_status sweep_direct(pca_ctx* ctx, int32_t n);

// cfg.graphs: the run is captured once per starting host state into a CUDA graph (stream
// capture of exactly the operations sweep_direct enqueues: kernels, table parameter-block
// kernels, NCCL sends/receives, fork/join events) and replayed afterwards
static pca_status sweep_graph(pca_ctx* ctx, int32_t n) {
    for (auto& gr : ctx->graphs) {
        if (gr.t == ctx->t && gr.n == n && gr.cur == ctx->cur && gr.counted == ctx->counted &&
            gr.tab_stage == ctx->tab_stage && gr.gpk_valid == ctx->gpk_valid) {
            CK(ctx, cudaGraphLaunch(gr.exec, ctx->stream));
            ctx->t = gr.t_after;
            ctx->cur = gr.cur_after;
            ctx->counted = gr.counted_after;
            ctx->prev_valid = gr.prev_valid_after;
            ctx->tab_stage = gr.tab_stage_after;
            ctx->beta_last = gr.beta_after;
            ctx->gpk_valid = gr.gpk_valid_after;
            memcpy(ctx->bthr_host, gr.bthr_after, sizeof(ctx->bthr_host));
            ctx->launches += gr.launches_d;
            ctx->sweep_launches += gr.sweep_launches_d;
            ctx->graph_replays++;
            return PCA_OK;
        }
    }
    pca_ctx::SweepGraph gr{};
    gr.t = ctx->t;
    gr.n = n;
    gr.cur = ctx->cur;
    gr.counted = ctx->counted;
    gr.tab_stage = ctx->tab_stage;
    gr.gpk_valid = ctx->gpk_valid;
    const int64_t l0 = ctx->launches, s0 = ctx->sweep_launches;
    if (ctx->lay.rows < ctx->cfg.height && !ctx->side) {  // the strip schedule's side stream
        CK(ctx, cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
        CK(ctx, cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        CK(ctx, cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
    }
    // capture on a private stream (the legacy default stream cannot be captured): the run's
    // operations are enqueued there while capturing, and the graph is launched on the caller's
    if (!ctx->cap) CK(ctx, cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
    cudaStream_t user = ctx->stream;
    CK(ctx, cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal));
    ctx->stream = ctx->cap;
    pca_status st = sweep_direct(ctx, n);
    ctx->stream = user;
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(ctx->cap, &graph);
    if (st != PCA_OK) {
        if (graph) cudaGraphDestroy(graph);
        return st;
    }
    if (ec != cudaSuccess) return cuda_fail(ctx, ec, "cudaStreamEndCapture (sweep run)");
    const cudaError_t ei = cudaGraphInstantiate(&gr.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) return cuda_fail(ctx, ei, "cudaGraphInstantiate (sweep run)");
    CK(ctx, cudaGraphLaunch(gr.exec, ctx->stream));
    gr.t_after = ctx->t;
    gr.cur_after = ctx->cur;
    gr.counted_after = ctx->counted;
    gr.prev_valid_after = ctx->prev_valid;
    gr.tab_stage_after = ctx->tab_stage;
    gr.beta_after = ctx->beta_last;
    gr.gpk_valid_after = ctx->gpk_valid;
    memcpy(gr.bthr_after, ctx->bthr_host, sizeof(ctx->bthr_host));
    gr.launches_d = ctx->launches - l0;
    gr.sweep_launches_d = ctx->sweep_launches - s0;
    if (ctx->graphs.size() >= 8) {  // a small cache: runs recur (e.g. reset + n sweeps per step)
        cudaGraphExecDestroy(ctx->graphs.front().exec);
        ctx->graphs.erase(ctx->graphs.begin());
    }
    ctx->graphs.push_back(gr);
    return PCA_OK;
}

pca_status pca_sweep(pca_ctx* ctx, int32_t n) {
    DeviceScope device_scope_;
    NvtxRange nvtx_("pca_sweep");
    pca_status st = ready(ctx);
    if (st != PCA_OK) return st;
    if (n < 0) return fail(PCA_EINVAL, "n must be >= 0");
    // a run that will be refused part-way (sweep index or counter limit) runs directly: its
    // sweeps before the refusal execute and the host state matches them (a capture would be
    // discarded with the host state already advanced)
    const int64_t t0 = ctx->t, burn = ctx->cfg.mpm_burn_in;
    const int64_t counted_n = burn < 0 ? 0 : std::max<int64_t>(0, t0 + n - std::max<int64_t>(t0, burn));
    const bool refused = t0 + n > (int64_t)0xFFFFFFFFLL || ctx->counted + counted_n > 65535;
    if (ctx->cfg.graphs && n > 0 && !ctx->p2p && !refused) return sweep_graph(ctx, n);
    return sweep_direct(ctx, n);
}

// the table kernel's uint8 count deltas into the uint16 counts, plane by plane (deltas = 0)
static pca_status fold_table_deltas(pca_ctx* ctx) {
    if (ctx->tdc_pending == 0) return PCA_OK;
    const int planes = ctx->cfg.levels;
    for (int k = 0; k < planes; ++k)
        LAUNCH(ctx, launch_fold_counts(ctx->geo, ctx->counts + (size_t)k * ctx->geo.cplane,
                                       ctx->gen.tdc + (size_t)k * ctx->gen.tdc_plane, ctx->gen.tdc_chain,
                                       ctx->cfg.batch, ctx->stream));
    ctx->tdc_pending = 0;
    return PCA_OK;
}

static pca_status sweep_direct_run(pca_ctx* ctx, int32_t n);

// every call leaves the canonical uint16 counts complete (the table kernel's deltas folded),
// also a call refused part-way (sweep index or counter limit) for the sweeps it did
static pca_status sweep_direct(pca_ctx* ctx, int32_t n) {
    const pca_status st = sweep_direct_run(ctx, n);
    if (st != PCA_OK && st != PCA_EUNSUPPORTED) return st;
    const pca_status sf = fold_table_deltas(ctx);
    return st != PCA_OK ? st : sf;
}

static pca_status sweep_direct_run(pca_ctx* ctx, int32_t n) {
    pca_status st = PCA_OK;
    const bool strip = ctx->lay.rows < ctx->cfg.height;
    // two sweeps per HBM pass (sweep_binary2.cu, opt-in): levels == 2, W % 16 == 0; on a row
    // strip the halo is 2 rows deep and exchanged once per pass (half the messages per sweep,
    // SURVEY 8(f) rank 1).  Measured slower than one sweep per pass on one B200.
    const bool pairs = ctx->kernel == PCA_KERNEL_BINARY && (ctx->cfg.width % 16) == 0 &&
                       ctx->cfg.sweeps_per_pass == 2;
    const bool caller_x = strip && !ctx->comm && !ctx->p2p;  // the caller exchanges the halos
    if (caller_x && n > (pairs ? 2 : 1))
        return fail(PCA_EINVAL, pairs ? "a strip context without NCCL or peers sweeps one pass (<= 2 "
                                        "sweeps) at a time (caller exchanges halos)"
                                      : "a strip context without NCCL or peers sweeps one step at a "
                                        "time (caller exchanges halos)");
    auto counts_at = [&](int64_t t) {
        return (ctx->cfg.mpm_burn_in >= 0 && t >= ctx->cfg.mpm_burn_in) ? 1 : 0;
    };
    // small lattices: runs of sweeps in one cooperative launch (sweep_multi_kernel)
    const bool small = !strip && !pairs &&
                       (size_t)ctx->lay.rows * ctx->cfg.width * ctx->cfg.batch <= multi_max_sites();
    // the packed kernel, except on strips with attached peers (their device-initiated halo stores
    // live in the byte kernel: those sweeps run it on the byte state)
    if (ctx->kernel == PCA_KERNEL_PACKED && n > 0 && !(small && n >= 2) && !ctx->p2p)
        return sweep_packed_run(ctx, n);
    for (int32_t i = 0; i < n; ++i) {
        const int64_t t = ctx->t;
        if (t >= (int64_t)0xFFFFFFFFLL) return fail(PCA_EUNSUPPORTED, "sweep index exceeds 2^32-1");
        if (small && n - i >= 2) {
            // the run stays inside one beta stage and one counting mode
            int64_t run = n - i;
            const int64_t period = ctx->cfg.beta_period;
            run = std::min<int64_t>(run, period - t % period);
            if (ctx->cfg.mpm_burn_in >= 0 && t < ctx->cfg.mpm_burn_in)
                run = std::min<int64_t>(run, ctx->cfg.mpm_burn_in - t);
            run = std::min<int64_t>(run, (int64_t)0xFFFFFFFFLL - t);
            const int count = counts_at(t);
            if (count) run = std::min<int64_t>(run, 65535 - ctx->counted);
            if (run >= 2) {
                st = build_tables(ctx, t);
                if (st != PCA_OK) return st;
                fill_common(ctx, ctx->gen.c, t, count);
                ctx->gen.c.rlo = 0;
                ctx->gen.c.rhi = ctx->lay.rows;
                ctx->launches++;
                ctx->sweep_launches++;
                const int e = launch_sweep_general(ctx->gen, ctx->cfg.batch, (int)run, ctx->stream);
                if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep (multi-sweep launch)");
                ctx->cur ^= (int)(run & 1);
                ctx->prev_valid = 1;
                ctx->t = t + run;
                ctx->counted += count * run;
                i += (int32_t)run - 1;
                continue;
            }
        }
        if (pairs && i + 1 < n && t + 1 < (int64_t)0xFFFFFFFFLL) {
            const int c0 = counts_at(t), c1 = counts_at(t + 1);
            if (ctx->counted + c0 + c1 > 65535)
                return fail(PCA_EUNSUPPORTED, "more than 65535 counted sweeps overflow uint16 counts");
            // a strip recomputes sweep t one row beyond its edges: that row's g must be in the g
            // halo (exchanged once per g; the caller copies it without NCCL or peers)
            if (strip && !caller_x && !ctx->g_halo_valid) {
                st = exchange_g(ctx);
                if (st != PCA_OK) return st;
                ctx->g_halo_valid = 1;
            }
            uint32_t k2 = 0;
            if (strip && ctx->p2p) {  // one phase: the pass reads our 2-deep halos, then pushes
                k2 = ctx->phase + 1;
                st = p2p_begin(ctx, k2);
                if (st != PCA_OK) return st;
            }
            st = build_tables(ctx, t);
            if (st != PCA_OK) return st;
            memcpy(ctx->bin2.thr[0], ctx->bthr_host, sizeof(ctx->bthr_host));
            st = build_tables(ctx, t + 1);
            if (st != PCA_OK) return st;
            memcpy(ctx->bin2.thr[1], ctx->bthr_host, sizeof(ctx->bthr_host));
            fill_common(ctx, ctx->bin2.c, t, c0);
            ctx->bin2.count2 = c1;
            ctx->bin2.c.rlo = 0;
            ctx->bin2.c.rhi = ctx->lay.rows;
            ctx->launches++;
            ctx->sweep_launches++;
            const int e = launch_sweep_binary2(ctx->bin2, ctx->cfg.batch, 0, ctx->stream);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep (two per pass)");
            if (strip && ctx->p2p) {  // our 2 edge rows of x_{t+2} into the peers' halos
                st = p2p_copy_edges(ctx, ctx->cur ^ 1, HALO);
                if (st == PCA_OK) st = p2p_end(ctx, k2);
                if (st != PCA_OK) return st;
            } else if (strip) {
                st = exchange(ctx, ctx->x[ctx->cur ^ 1], HALO);  // NCCL (caller: nothing)
                if (st != PCA_OK) return st;
            }
            ctx->cur ^= 1;
            ctx->prev_valid = 1;
            ctx->t = t + 2;
            ctx->counted += c0 + c1;
            ++i;
            continue;
        }
        st = build_tables(ctx, t);
        if (st != PCA_OK) return st;
        const int count = counts_at(t);
        if (count && ctx->counted + 1 > 65535)
            return fail(PCA_EUNSUPPORTED, "more than 65535 counted sweeps overflow uint16 counts");
        fill_common(ctx, ctx->bin.c, t, count);
        fill_common(ctx, ctx->gen.c, t, count);
        // a counted sweep on the table kernel adds into the uint8 deltas: fold before a byte
        // could overflow
        const bool tab_counts = count && ctx->kernel == PCA_KERNEL_TABLE && ctx->gen.tab != nullptr;
        if (tab_counts && ctx->tdc_pending >= 255) {
            st = fold_table_deltas(ctx);
            if (st != PCA_OK) return st;
        }
        // one sweep kernel over local rows [rlo, rhi) on stream s
        auto launch_rows = [&](int rlo, int rhi, cudaStream_t s) -> int {
            ctx->launches++;
            ctx->sweep_launches++;
            if (ctx->kernel == PCA_KERNEL_BINARY || ctx->kernel == PCA_KERNEL_PACKED) {
                ctx->bin.c.rlo = rlo;
                ctx->bin.c.rhi = rhi;
                return launch_sweep_binary(ctx->bin, ctx->cfg.batch, ctx->rows_per_thread, s);
            }
            ctx->gen.c.rlo = rlo;
            ctx->gen.c.rhi = rhi;
            return launch_sweep_general(ctx->gen, ctx->cfg.batch, 1, s);
        };
        const int R = ctx->lay.rows;
        int e = 0;
        if (strip && ctx->p2p && pairs) {
            // two sweeps per pass: a single sweep (odd n) leaves 2-deep halos for the next pass
            const uint32_t k = ctx->phase + 1;
            st = p2p_begin(ctx, k);
            if (st != PCA_OK) return st;
            e = launch_rows(0, R, ctx->stream);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep (peer halos, depth 2)");
            st = p2p_copy_edges(ctx, ctx->cur ^ 1, HALO);
            if (st == PCA_OK) st = p2p_end(ctx, k);
            if (st != PCA_OK) return st;
        } else if (strip && ctx->p2p) {
            // device-initiated halo exchange: ONE launch over all rows whose edge-row CTAs also
            // store the new rows into the peers' halo rows (their output buffer); stream waits
            // and writes of the phase words order it against the peers (p2p_begin / p2p_end)
            const uint32_t k = ctx->phase + 1;
            st = p2p_begin(ctx, k);
            if (st != PCA_OK) return st;
            const int nb = ctx->cur ^ 1;
            const size_t pitch = (size_t)ctx->lay.xpitch;
            for (SweepCommon* sc : {&ctx->bin.c, &ctx->gen.c}) {
                sc->peer_up = ctx->has_up ? ctx->up.x[nb] + (HALO + (size_t)ctx->up.rows) * pitch : nullptr;
                sc->peer_dn = ctx->has_dn ? ctx->dn.x[nb] + (HALO - 1) * pitch : nullptr;
                sc->peer_up_chain = ctx->up.chain_stride;
                sc->peer_dn_chain = ctx->dn.chain_stride;
            }
            e = launch_rows(0, R, ctx->stream);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep (peer halos)");
            st = p2p_end(ctx, k);
            if (st != PCA_OK) return st;
        } else if (strip && R >= 3 && !pairs) {
            // row strip: the two edge rows first, then their halo exchange on the main stream
            // overlapping the interior rows on the side stream; the next sweep starts after
            // both (the interior never reads the halo rows).
            if (!ctx->side) {
                CK(ctx, cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
                CK(ctx, cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
                CK(ctx, cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
            }
            CK(ctx, cudaEventRecord(ctx->ev_fork, ctx->stream));
            CK(ctx, cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            e = launch_rows(0, 1, ctx->stream);
            if (!e) e = launch_rows(R - 1, R, ctx->stream);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep (edge rows)");
            st = exchange(ctx, ctx->x[ctx->cur ^ 1], 1);  // only the finished edge rows
            if (st != PCA_OK) return st;
            e = launch_rows(1, R - 1, ctx->side);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep (interior rows)");
            CK(ctx, cudaEventRecord(ctx->ev_join, ctx->side));
            CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0));
        } else {
            e = launch_rows(0, R, ctx->stream);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "sweep");
            st = exchange(ctx, ctx->x[ctx->cur ^ 1]);
            if (st != PCA_OK) return st;
        }
        ctx->cur ^= 1;
        ctx->prev_valid = 1;
        ctx->t = t + 1;
        ctx->counted += count;
        ctx->tdc_pending += tab_counts ? 1 : 0;
    }
    return PCA_OK;
}

pca_status pca_gibbs_sweep(pca_ctx* ctx, int32_t n) {
    DeviceScope device_scope_;
    NvtxRange nvtx_("pca_gibbs_sweep");
    pca_status st = ready(ctx);
    if (st != PCA_OK) return st;
    if (n < 0) return fail(PCA_EINVAL, "n must be >= 0");
    const pca_config& c = ctx->cfg;
    if (c.periodic && ((c.height & 1) || (c.width & 1)))
        return fail(PCA_EUNSUPPORTED, "the Gibbs colouring needs even height and width on a torus");
    const bool strip = ctx->lay.rows < c.height;
    if (strip && !ctx->p2p && !(ctx->comm && ctx->nranks > 1))
        return fail(PCA_EINVAL, "a row-strip Gibbs sweep exchanges halos between colours: attach NCCL or peers");
    // strips: every Gibbs launch is one exchange phase.  With peers attached the launch is
    // preceded by the phase wait and followed by copies of its buffer's edge rows into the
    // peers' halo rows (in place or not, a launch never reads a byte that it or a peer's launch
    // of the same phase changes, so rewriting unchanged halo bytes is safe), then the signal.
    auto phase_begin = [&](uint32_t& k) -> pca_status {
        if (!strip || !ctx->p2p) return PCA_OK;
        k = ctx->phase + 1;
        return p2p_begin(ctx, k);
    };
    auto phase_end = [&](uint32_t k, int b) -> pca_status {
        if (!strip) return PCA_OK;
        if (!ctx->p2p) return exchange(ctx, ctx->x[b], 1);
        pca_status s2 = p2p_copy_edges(ctx, b, 1);
        if (s2 != PCA_OK) return s2;
        return p2p_end(ctx, k);
    };
    // Moore-8: the two colours of a row parity in one launch (2 launches per sweep) when the
    // right-neighbour recomputation has its columns (free boundary, or 16-column torus pads);
    // with two levels on the binary PCA kernel's data path (sweep_gibbs_binary.cu), X -> Y
    const bool fused = c.neighborhood == 8 && (!c.periodic || (c.width % 16) == 0);
    const bool binpath = fused && c.levels == 2;
    const int nlaunch = c.neighborhood == 4 ? 2 : (fused ? 2 : 4);
    // small lattices: runs of sweeps in one cooperative launch (in place, the quad kernel)
    const bool small = !strip && (size_t)ctx->lay.rows * c.width * c.batch <= multi_max_sites();
    for (int32_t i = 0; i < n; ++i) {
        const int64_t t = ctx->t;
        if (t >= (int64_t)0xFFFFFFFFLL) return fail(PCA_EUNSUPPORTED, "sweep index exceeds 2^32-1");
        st = build_gibbs_tables(ctx, t);
        if (st != PCA_OK) return st;
        const int count = (c.mpm_burn_in >= 0 && t >= c.mpm_burn_in) ? 1 : 0;
        if (count && ctx->counted + 1 > 65535)
            return fail(PCA_EUNSUPPORTED, "more than 65535 counted sweeps overflow uint16 counts");
        if (small && n - i >= 2) {
            int64_t run = n - i;
            run = std::min<int64_t>(run, c.beta_period - t % c.beta_period);
            if (c.mpm_burn_in >= 0 && t < c.mpm_burn_in) run = std::min<int64_t>(run, c.mpm_burn_in - t);
            run = std::min<int64_t>(run, (int64_t)0xFFFFFFFFLL - t);
            if (count) run = std::min<int64_t>(run, 65535 - ctx->counted);
            if (run >= 2) {
                fill_common(ctx, ctx->gib.c, t, count);
                ctx->gib.c.x_out = ctx->x[ctx->cur];  // in place
                ctx->gib.c.rlo = 0;
                ctx->gib.c.rhi = ctx->lay.rows;
                ctx->gib.fused = fused ? 1 : 0;
                ctx->launches++;
                ctx->sweep_launches++;
                const int e = launch_sweep_gibbs(ctx->gib, c.batch, (int)run, ctx->stream);
                if (e) return cuda_fail(ctx, (cudaError_t)e, "gibbs sweep (multi-sweep launch)");
                ctx->prev_valid = 0;  // in place
                ctx->t = t + run;
                ctx->counted += count * run;
                i += (int32_t)run - 1;
                continue;
            }
        }
        if (binpath) {
            // X = x[cur] -> Y = x[cur ^ 1]: even rows from X, then odd rows from X and the new
            // even rows of Y; halos exchanged after each launch on strips
            fill_common(ctx, ctx->gbin.c, t, count);
            ctx->gbin.c.rlo = 0;
            ctx->gbin.c.rhi = ctx->lay.rows;
            for (int par = 0; par < 2; ++par) {
                ctx->gbin.parity = par;
                ctx->gbin.x_nb = par == 0 ? ctx->x[ctx->cur] : ctx->x[ctx->cur ^ 1];
                uint32_t k = 0;
                st = phase_begin(k);
                if (st != PCA_OK) return st;
                ctx->launches++;
                ctx->sweep_launches++;
                const int e = launch_gibbs_binary(ctx->gbin, c.batch, ctx->stream);
                if (e) return cuda_fail(ctx, (cudaError_t)e, "gibbs sweep (binary)");
                st = phase_end(k, ctx->cur ^ 1);
                if (st != PCA_OK) return st;
            }
            ctx->cur ^= 1;
            ctx->prev_valid = 1;
            ctx->t = t + 1;
            ctx->counted += count;
            continue;
        }
        fill_common(ctx, ctx->gib.c, t, 0);
        ctx->gib.c.x_out = ctx->x[ctx->cur];  // in place
        ctx->gib.c.rlo = 0;
        ctx->gib.c.rhi = ctx->lay.rows;
        ctx->gib.fused = fused ? 1 : 0;
        for (int k = 0; k < nlaunch; ++k) {
            ctx->gib.colour = k;
            // rows are final after colour 1 / 3, or after their fused launch
            ctx->gib.c.count_enable = count && (fused || (k & 1));
            uint32_t ph = 0;
            st = phase_begin(ph);
            if (st != PCA_OK) return st;
            ctx->launches++;
            ctx->sweep_launches++;
            const int e = launch_sweep_gibbs(ctx->gib, c.batch, 1, ctx->stream);
            if (e) return cuda_fail(ctx, (cudaError_t)e, "gibbs sweep");
            ctx->prev_valid = 0;  // in place
            st = phase_end(ph, ctx->cur);
            if (st != PCA_OK) return st;
        }
        ctx->t = t + 1;
        ctx->counted += count;
    }
    return PCA_OK;
}

// the output staging (stage past the input image, io_out, the stage's float planes) may still
// be read by an asynchronous MPM image copy (pca_finalize_async): writers wait on the device
static pca_status wait_out_free(pca_ctx* ctx) {
    if (ctx->copy) CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_out_free, 0));
    return PCA_OK;
}

pca_status pca_estimate(pca_ctx* ctx, int32_t kind, void* out) {
    DeviceScope device_scope_;
    NvtxRange nvtx_("pca_estimate");
    pca_status st = ready(ctx);
    if (st != PCA_OK) return st;
    if (!out) return fail(PCA_EINVAL, "out is NULL");
    if (kind < PCA_EST_LAST || kind > PCA_EST_CM) return fail(PCA_EINVAL, "unknown estimate kind");
    const pca_config& c = ctx->cfg;
    if (kind != PCA_EST_LAST && ctx->counted < 1)
        return fail(PCA_EINVAL, "MPM/marginal/CM estimates need counted sweeps (mpm_burn_in)");
    st = check_same_device(ctx, out, "out");
    if (st != PCA_OK) return st;
    const bool dev = is_device_ptr(out);
    const size_t plane = (size_t)ctx->lay.rows * c.width;
    st = wait_out_free(ctx);
    if (st != PCA_OK) return st;
    if (kind == PCA_EST_LAST || kind == PCA_EST_MPM) {
        uint8_t* dst = (dev && !c.packed_io) ? (uint8_t*)out : ctx->stage;
        if (kind == PCA_EST_LAST)
            LAUNCH(ctx, launch_unpack_state(ctx->geo, ctx->x[ctx->cur], dst, c.batch, ctx->stream));
        else
            LAUNCH(ctx, launch_mpm(ctx->geo, ctx->counts, (int)ctx->counted, dst, c.batch, ctx->stream));
        if (c.packed_io) {  // bit-packed result
            LAUNCH(ctx, launch_pack_bits(ctx->stage, ctx->io_out, c.width,
                                         (long long)c.batch * ctx->lay.rows, ctx->stream));
            CK(ctx, cudaMemcpyAsync(out, ctx->io_out, ctx->lay.io_bytes, cudaMemcpyDefault, ctx->stream));
        } else if (!dev) {
            CK(ctx, cudaMemcpyAsync(out, ctx->stage, dense_bytes(ctx), cudaMemcpyDeviceToHost,
                                    ctx->stream));
        }
        return sync(ctx);
    }
    // float outputs: CM [B][rows][W]; MARGINALS [B][levels][rows][W], one label plane per pass
    const int nplanes = kind == PCA_EST_CM ? 1 : c.levels;
    for (int k = 0; k < nplanes; ++k) {
        const int kk = kind == PCA_EST_CM ? -1 : k;
        float* dst = dev ? (float*)out + (size_t)k * plane : (float*)ctx->stage;
        const long long cs = dev ? (long long)nplanes * plane : (long long)plane;
        LAUNCH(ctx, launch_marginals(ctx->geo, ctx->counts, (int)ctx->counted, dst, cs, kk, c.batch,
                                     ctx->stream));
        if (!dev)
            CK(ctx, cudaMemcpy2DAsync((float*)out + (size_t)k * plane, nplanes * plane * 4,
                                      ctx->stage, plane * 4, plane * 4, c.batch,
                                      cudaMemcpyDeviceToHost, ctx->stream));
    }
    return sync(ctx);
}

pca_status pca_metric_sums(pca_ctx* ctx, const uint8_t* truth, int32_t kind, int64_t* sums) {
    DeviceScope device_scope_;
    pca_status st = ready(ctx);
    if (st != PCA_OK) return st;
    if (!truth || !sums) return fail(PCA_EINVAL, "truth and sums must be non-NULL");
    if (kind != PCA_EST_LAST && kind != PCA_EST_MPM)
        return fail(PCA_EINVAL, "metric sums are defined for LAST and MPM");
    if (kind == PCA_EST_MPM && ctx->counted < 1)
        return fail(PCA_EINVAL, "MPM needs counted sweeps (mpm_burn_in)");
    const pca_config& c = ctx->cfg;
    const uint8_t* dt = nullptr;
    st = device_input(ctx, truth, &dt);
    if (st != PCA_OK) return st;
    const size_t nb = (size_t)c.batch * 8 * sizeof(unsigned long long);
    CK(ctx, cudaMemsetAsync(ctx->sums, 0, nb, ctx->stream));
    MetricParams mp;
    mp.geo = ctx->geo;
    mp.x = ctx->x[ctx->cur];
    mp.counts = ctx->counts;
    mp.truth = dt;
    mp.sums = ctx->sums;
    mp.kind = kind;
    mp.nsamp = (int)ctx->counted;
    mp.mpm_out = nullptr;
    LAUNCH(ctx, launch_metric_sums(mp, c.batch, ctx->stream));
    if (ctx->comm && ctx->nranks > 1) {
        NcclApi& N = nccl();
        CK(ctx, cudaMemcpyAsync(ctx->sums_max, ctx->sums, nb, cudaMemcpyDeviceToDevice, ctx->stream));
        ncclResult_t e = N.AllReduce(ctx->sums, ctx->sums, (size_t)c.batch * 8, ncclUint64, ncclSum,
                                     ctx->comm, ctx->stream);
        if (e == ncclSuccess)
            e = N.AllReduce(ctx->sums_max, ctx->sums_max, (size_t)c.batch * 8, ncclUint64, ncclMax,
                            ctx->comm, ctx->stream);
        if (e != ncclSuccess) {
            ctx->poisoned = 1;
            return fail(PCA_ENCCL, "metric all-reduce: %s", N.GetErrorString(e));
        }
    }
    std::vector<unsigned long long> h((size_t)c.batch * 8), hm((size_t)c.batch * 8);
    CK(ctx, cudaMemcpyAsync(h.data(), ctx->sums, nb, cudaMemcpyDeviceToHost, ctx->stream));
    if (ctx->comm && ctx->nranks > 1)
        CK(ctx, cudaMemcpyAsync(hm.data(), ctx->sums_max, nb, cudaMemcpyDeviceToHost, ctx->stream));
    st = sync(ctx);
    if (st != PCA_OK) return st;
    for (int bch = 0; bch < c.batch; ++bch)
        for (int k = 0; k < 8; ++k) {
            unsigned long long v = h[(size_t)bch * 8 + k];
            if (k == 6 && ctx->comm && ctx->nranks > 1) v = hm[(size_t)bch * 8 + k];
            sums[(size_t)bch * 8 + k] = (int64_t)v;
        }
    return PCA_OK;
}

// PSNR (R17) and global SSIM (R16) from the exact sums
// v[0..7] of one chain (sum d^2, sum x, sum y, sum x^2, sum y^2, sum xy, max x, N); false
// when the original is all black (PSNR undefined)
bool metrics_from_sums(const int64_t* v, int levels, double* psnr, double* ssim) {
    const double L1 = (double)(levels - 1);
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    const __int128 N = v[7];
    const double Nd = (double)v[7];
    // MSE on luminances, PSNR with the original's max
    const double mse = (double)v[0] / (Nd * L1 * L1);
    const double xmax = (double)v[6] / L1;
    *psnr = (mse == 0.0) ? INFINITY : 20.0 * log10(xmax / sqrt(mse));
    // global SSIM (R16): population moments from exact numerators
    const __int128 vx = N * (__int128)v[3] - (__int128)v[1] * v[1];
    const __int128 vy = N * (__int128)v[4] - (__int128)v[2] * v[2];
    const __int128 cxy = N * (__int128)v[5] - (__int128)v[1] * v[2];
    const double den = Nd * Nd * L1 * L1;
    const double mux = (double)v[1] / (Nd * L1), muy = (double)v[2] / (Nd * L1);
    const double sx = (double)vx / den, sy = (double)vy / den, sxy = (double)cxy / den;
    *ssim = ((2.0 * mux * muy + c1) * (2.0 * sxy + c2)) / ((mux * mux + muy * muy + c1) * (sx + sy + c2));
    return v[6] != 0;
}

pca_status pca_psnr_ssim(pca_ctx* ctx, const uint8_t* truth, int32_t kind, double* psnr,
                         double* ssim) {
    DeviceScope device_scope_;
    if (!psnr || !ssim) return fail(PCA_EINVAL, "psnr and ssim must be non-NULL");
    std::vector<int64_t> s((size_t)(ctx ? ctx->cfg.batch : 1) * 8);
    pca_status st = pca_metric_sums(ctx, truth, kind, s.data());
    if (st != PCA_OK) return st;
    bool black = false;
    for (int b = 0; b < ctx->cfg.batch; ++b)
        if (!metrics_from_sums(&s[(size_t)b * 8], ctx->cfg.levels, &psnr[b], &ssim[b])) black = true;
    if (black) return fail(PCA_EINVAL, "original image is all black: PSNR undefined (R17)");
    return PCA_OK;
}

static pca_status ensure_copy_stream(pca_ctx* ctx) {
    if (ctx->copy) return PCA_OK;
    CK(ctx, cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
    for (cudaEvent_t* e : {&ctx->ev_truth_ready, &ctx->ev_truth_free, &ctx->ev_in_ready,
                           &ctx->ev_in_free, &ctx->ev_out_ready, &ctx->ev_out_free})
        CK(ctx, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    CK(ctx, cudaEventRecord(ctx->ev_truth_free, ctx->stream));
    CK(ctx, cudaEventRecord(ctx->ev_in_free, ctx->stream));
    CK(ctx, cudaEventRecord(ctx->ev_out_free, ctx->stream));
    return PCA_OK;
}

pca_status pca_stage_input(pca_ctx* ctx, const uint8_t* g) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!g) return fail(PCA_EINVAL, "g is NULL");
    st = check_same_device(ctx, g, "staged input");
    if (st != PCA_OK) return st;
    st = ensure_copy_stream(ctx);
    if (st != PCA_OK) return st;
    // the previous staged input must have been consumed by its reset
    CK(ctx, cudaStreamWaitEvent(ctx->copy, ctx->ev_in_free, 0));
    const size_t bytes = ctx->cfg.packed_io ? ctx->lay.io_bytes : dense_bytes(ctx);
    CK(ctx, cudaMemcpyAsync(ctx->in_stage, g, bytes, cudaMemcpyDefault, ctx->copy));
    CK(ctx, cudaEventRecord(ctx->ev_in_ready, ctx->copy));
    ctx->in_staged = 1;
    return PCA_OK;
}

pca_status pca_reset_staged(pca_ctx* ctx) {
    DeviceScope device_scope_;
    NvtxRange nvtx_("pca_reset_staged");
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!ctx->in_staged) return fail(PCA_EINVAL, "no input staged (pca_stage_input)");
    CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_in_ready, 0));
    ctx->in_staged = 0;
    // the staged bytes are a device copy of the caller's argument: the pca_reset path
    st = do_reset(ctx, ctx->in_stage, nullptr, true);
    if (st != PCA_OK) return st;
    CK(ctx, cudaEventRecord(ctx->ev_in_free, ctx->stream));
    return PCA_OK;
}

pca_status pca_stage_truth(pca_ctx* ctx, const uint8_t* truth) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!truth) return fail(PCA_EINVAL, "truth is NULL");
    st = ensure_copy_stream(ctx);
    if (st != PCA_OK) return st;
    // the previous finalize's read of the buffer comes first
    CK(ctx, cudaStreamWaitEvent(ctx->copy, ctx->ev_truth_free, 0));
    if (ctx->cfg.packed_io) {
        CK(ctx, cudaMemcpyAsync(ctx->io_truth, truth, ctx->lay.io_bytes, cudaMemcpyDefault, ctx->copy));
        LAUNCH(ctx, launch_unpack_bits(ctx->io_truth, ctx->truth, ctx->cfg.width,
                                       (long long)ctx->cfg.batch * ctx->lay.rows, ctx->copy));
    } else {
        CK(ctx, cudaMemcpyAsync(ctx->truth, truth, dense_bytes(ctx), cudaMemcpyDefault, ctx->copy));
    }
    CK(ctx, cudaEventRecord(ctx->ev_truth_ready, ctx->copy));
    ctx->truth_staged = 1;
    return PCA_OK;
}

static pca_status finalize(pca_ctx* ctx, const uint8_t* truth, uint8_t* mpm_out, double* psnr,
                           double* ssim, bool async_image) {
    NvtxRange nvtx_("pca_finalize");
    pca_status st = ready(ctx);
    if (st != PCA_OK) return st;
    if (!psnr || !ssim) return fail(PCA_EINVAL, "psnr and ssim must be non-NULL");
    if (!truth && !ctx->truth_staged)
        return fail(PCA_EINVAL, "truth is NULL and no truth was staged (pca_stage_truth)");
    if (ctx->counted < 1) return fail(PCA_EINVAL, "finalize needs counted sweeps (mpm_burn_in)");
    const pca_config& c = ctx->cfg;
    const uint8_t* dt = nullptr;
    if (truth) {
        st = device_input(ctx, truth, &dt);  // host truth -> stage[0, BRW)
        if (st != PCA_OK) return st;
    } else {
        CK(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_truth_ready, 0));
        dt = ctx->truth;
    }
    if (mpm_out) {
        st = check_same_device(ctx, mpm_out, "mpm_out");
        if (st != PCA_OK) return st;
    }
    const bool dev_out = mpm_out && is_device_ptr(mpm_out) && !c.packed_io;
    // packed_io: the finalisation pass writes the bit-packed image itself (into io_out)
    const bool packed_out = mpm_out && c.packed_io;
    uint8_t* mo = (mpm_out && !packed_out)
                      ? (dev_out ? mpm_out : ctx->stage + align256(dense_bytes(ctx))) : nullptr;
    const bool async_copy = async_image && mpm_out && !dev_out;
    if (async_copy) {
        st = ensure_copy_stream(ctx);
        if (st != PCA_OK) return st;
    }
    if (mpm_out && !dev_out) {
        st = wait_out_free(ctx);  // the previous asynchronous image copy has read the staging
        if (st != PCA_OK) return st;
    }
    const size_t nb = (size_t)c.batch * 16 * sizeof(unsigned long long);
    CK(ctx, cudaMemsetAsync(ctx->sums, 0, nb, ctx->stream));
    MetricParams mp;
    mp.geo = ctx->geo;
    mp.x = ctx->x[ctx->cur];
    mp.counts = ctx->counts;
    mp.truth = dt;
    mp.sums = ctx->sums;
    mp.kind = 2;
    mp.nsamp = (int)ctx->counted;
    mp.mpm_out = mo;
    mp.mpm_bits = packed_out ? ctx->io_out : nullptr;
    LAUNCH(ctx, launch_metric_sums(mp, c.batch, ctx->stream));
    if (!truth) CK(ctx, cudaEventRecord(ctx->ev_truth_free, ctx->stream));
    if (ctx->comm && ctx->nranks > 1) {
        NcclApi& N = nccl();
        CK(ctx, cudaMemcpyAsync(ctx->sums_max, ctx->sums, nb, cudaMemcpyDeviceToDevice, ctx->stream));
        ncclResult_t e = N.AllReduce(ctx->sums, ctx->sums, (size_t)c.batch * 16, ncclUint64, ncclSum,
                                     ctx->comm, ctx->stream);
        if (e == ncclSuccess)
            e = N.AllReduce(ctx->sums_max, ctx->sums_max, (size_t)c.batch * 16, ncclUint64, ncclMax,
                            ctx->comm, ctx->stream);
        if (e != ncclSuccess) {
            ctx->poisoned = 1;
            return fail(PCA_ENCCL, "finalize all-reduce: %s", N.GetErrorString(e));
        }
    }
    std::vector<unsigned long long> h((size_t)c.batch * 16), hm((size_t)c.batch * 16);
    CK(ctx, cudaMemcpyAsync(h.data(), ctx->sums, nb, cudaMemcpyDeviceToHost, ctx->stream));
    if (ctx->comm && ctx->nranks > 1)
        CK(ctx, cudaMemcpyAsync(hm.data(), ctx->sums_max, nb, cudaMemcpyDeviceToHost, ctx->stream));
    if (mpm_out && !dev_out) {
        const uint8_t* src = packed_out ? ctx->io_out : mo;
        const size_t bytes = packed_out ? ctx->lay.io_bytes : dense_bytes(ctx);
        if (async_copy) {  // on the copy stream: overlaps whatever is enqueued after this call
            CK(ctx, cudaEventRecord(ctx->ev_out_ready, ctx->stream));
            CK(ctx, cudaStreamWaitEvent(ctx->copy, ctx->ev_out_ready, 0));
            CK(ctx, cudaMemcpyAsync(mpm_out, src, bytes, cudaMemcpyDefault, ctx->copy));
            CK(ctx, cudaEventRecord(ctx->ev_out_free, ctx->copy));
        } else {
            CK(ctx, cudaMemcpyAsync(mpm_out, src, bytes, cudaMemcpyDefault, ctx->stream));
        }
    }
    st = sync(ctx);
    if (st != PCA_OK) return st;
    bool black = false;
    for (int b = 0; b < c.batch; ++b)
        for (int e = 0; e < 2; ++e) {  // e = 0: LAST, 1: MPM
            int64_t v[8];
            for (int k = 0; k < 8; ++k) {
                unsigned long long x = h[(size_t)b * 16 + 8 * e + k];
                if (k == 6 && ctx->comm && ctx->nranks > 1) x = hm[(size_t)b * 16 + 8 * e + k];
                v[k] = (int64_t)x;
            }
            if (!metrics_from_sums(v, c.levels, &psnr[2 * b + e], &ssim[2 * b + e])) black = true;
        }
    if (black) return fail(PCA_EINVAL, "original image is all black: PSNR undefined (R17)");
    return PCA_OK;
}

pca_status pca_finalize(pca_ctx* ctx, const uint8_t* truth, uint8_t* mpm_out, double* psnr,
                        double* ssim) {
    DeviceScope device_scope_;
    return finalize(ctx, truth, mpm_out, psnr, ssim, false);
}

pca_status pca_finalize_async(pca_ctx* ctx, const uint8_t* truth, uint8_t* mpm_out, double* psnr,
                              double* ssim) {
    DeviceScope device_scope_;
    return finalize(ctx, truth, mpm_out, psnr, ssim, true);
}

pca_status pca_ssim_windowed(pca_ctx* ctx, const uint8_t* truth, int32_t kind, double* ssim) {
    DeviceScope device_scope_;
    pca_status st = ready(ctx);
    if (st != PCA_OK) return st;
    if (!truth || !ssim) return fail(PCA_EINVAL, "truth and ssim must be non-NULL");
    if (kind != PCA_EST_LAST && kind != PCA_EST_MPM)
        return fail(PCA_EINVAL, "windowed SSIM is defined for LAST and MPM");
    if (kind == PCA_EST_MPM && ctx->counted < 1)
        return fail(PCA_EINVAL, "MPM needs counted sweeps (mpm_burn_in)");
    const pca_config& c = ctx->cfg;
    if (ctx->lay.rows != c.height)
        return fail(PCA_EUNSUPPORTED, "windowed SSIM needs the whole lattice (not a row strip)");
    if (c.height < SSIM_WIN || c.width < SSIM_WIN)
        return fail(PCA_EINVAL, "windowed SSIM needs height, width >= %d", SSIM_WIN);
    st = wait_out_free(ctx);
    if (st != PCA_OK) return st;
    const uint8_t* dt = nullptr;
    st = device_input(ctx, truth, &dt);  // host truth -> stage[0, BRW)
    if (st != PCA_OK) return st;
    const size_t brw = dense_bytes(ctx);
    WinSsimParams wp;
    wp.y = dt;
    wp.ychain = (long long)ctx->lay.rows * c.width;
    wp.ypitch = c.width;
    if (kind == PCA_EST_LAST) {
        wp.x = ctx->x[ctx->cur] + (size_t)HALO * ctx->lay.xpitch + XOFF;
        wp.xchain = ctx->geo.xchain;
        wp.xpitch = ctx->lay.xpitch;
    } else {
        uint8_t* mpm = ctx->stage + align256(brw);
        LAUNCH(ctx, launch_mpm(ctx->geo, ctx->counts, (int)ctx->counted, mpm, c.batch, ctx->stream));
        wp.x = mpm;
        wp.xchain = wp.ychain;
        wp.xpitch = c.width;
    }
    wp.H = c.height;
    wp.W = c.width;
    wp.levels = c.levels;
    wp.partial = (double*)(ctx->stage + 2 * align256(brw));
    int gx = 0, gy = 0;
    ssim_windowed_grid(c.height, c.width, &gx, &gy);
    LAUNCH(ctx, launch_ssim_windowed(wp, c.batch, ctx->stream));
    const size_t per = (size_t)gx * gy;
    std::vector<double> h(per * c.batch);
    CK(ctx, cudaMemcpyAsync(h.data(), wp.partial, h.size() * sizeof(double), cudaMemcpyDeviceToHost,
                            ctx->stream));
    st = sync(ctx);
    if (st != PCA_OK) return st;
    const double nwin = (double)(c.height - SSIM_WIN + 1) * (double)(c.width - SSIM_WIN + 1);
    for (int b = 0; b < c.batch; ++b) {
        double t = 0.0;
        for (size_t i = 0; i < per; ++i) t += h[(size_t)b * per + i];
        ssim[b] = t / nwin;
    }
    return PCA_OK;
}

pca_status pca_changed_sites(pca_ctx* ctx, int64_t* changed) {
    DeviceScope device_scope_;
    pca_status st = ready(ctx);
    if (st != PCA_OK) return st;
    if (!changed) return fail(PCA_EINVAL, "changed is NULL");
    if (!ctx->prev_valid)
        return fail(PCA_EINVAL, "no previous state: sweep first (in-place Gibbs sweeps keep none)");
    const size_t nb = (size_t)ctx->cfg.batch * sizeof(unsigned long long);
    CK(ctx, cudaMemsetAsync(ctx->sums, 0, nb, ctx->stream));
    LAUNCH(ctx, launch_changed(ctx->geo, ctx->x[ctx->cur], ctx->x[ctx->cur ^ 1], ctx->sums,
                               ctx->cfg.batch, ctx->stream));
    std::vector<unsigned long long> h(ctx->cfg.batch);
    CK(ctx, cudaMemcpyAsync(h.data(), ctx->sums, nb, cudaMemcpyDeviceToHost, ctx->stream));
    st = sync(ctx);
    if (st != PCA_OK) return st;
    for (int b = 0; b < ctx->cfg.batch; ++b) changed[b] = (int64_t)h[b];
    return PCA_OK;
}

pca_status pca_read_state(pca_ctx* ctx, uint8_t* out) { return pca_estimate(ctx, PCA_EST_LAST, out); }

pca_status pca_write_state(pca_ctx* ctx, const uint8_t* x) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!x) return fail(PCA_EINVAL, "x is NULL");
    const uint8_t* dx = nullptr;
    st = device_input(ctx, x, &dx);
    if (st != PCA_OK) return st;
    return load_state(ctx, dx, ctx->cfg.width, (long long)ctx->lay.rows * ctx->cfg.width, "x");
}

pca_status pca_read_counts(pca_ctx* ctx, uint16_t* out) {
    DeviceScope device_scope_;
    pca_status st = ready(ctx);
    if (st != PCA_OK) return st;
    if (!out) return fail(PCA_EINVAL, "out is NULL");
    const pca_config& c = ctx->cfg;
    const Layout& L = ctx->lay;
    CK(ctx, cudaMemcpy2DAsync(out, (size_t)c.width * 2, ctx->counts, (size_t)L.cpitch * 2,
                              (size_t)c.width * 2, (size_t)c.batch * L.cplanes * L.rows,
                              cudaMemcpyDefault, ctx->stream));
    return sync(ctx);
}

pca_status pca_write_counts(pca_ctx* ctx, const uint16_t* cin, int64_t counted) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!cin || counted < 0 || counted > 65535) return fail(PCA_EINVAL, "bad counts arguments");
    const pca_config& c = ctx->cfg;
    const Layout& L = ctx->lay;
    CK(ctx, cudaMemcpy2DAsync(ctx->counts, (size_t)L.cpitch * 2, cin, (size_t)c.width * 2,
                              (size_t)c.width * 2, (size_t)c.batch * L.cplanes * L.rows,
                              cudaMemcpyDefault, ctx->stream));
    ctx->counted = counted;
    return sync(ctx);
}

pca_status pca_set_step(pca_ctx* ctx, int64_t t) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (t < 0 || t >= (int64_t)0xFFFFFFFFLL) return fail(PCA_EINVAL, "t out of range");
    ctx->t = t;
    return PCA_OK;
}

pca_status pca_get_stats(pca_ctx* ctx, pca_stats* out) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!out) return fail(PCA_EINVAL, "out is NULL");
    st = sync(ctx);
    if (st != PCA_OK) return st;
    out->sweeps_done = ctx->t;
    out->counted_sweeps = ctx->counted;
    out->kernel_launches = ctx->launches;
    out->sweep_launches = ctx->sweep_launches;
    out->beta = ctx->beta_last;
    out->kernel = ctx->kernel;
    out->nranks = ctx->nranks;
    out->graph_replays = ctx->graph_replays;
    return PCA_OK;
}

pca_status pca_halo_ptrs(pca_ctx* ctx, pca_halo* out) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!out) return fail(PCA_EINVAL, "out is NULL");
    uint8_t* base = ctx->x[ctx->cur];
    const size_t pitch = (size_t)ctx->lay.xpitch;
    out->send_top = base + HALO * pitch;
    out->send_bottom = base + (size_t)ctx->lay.rows * pitch;
    out->recv_top = base;
    out->recv_bottom = base + (size_t)(ctx->lay.rows + HALO) * pitch;
    out->row_bytes = HALO * pitch;
    out->chain_stride = (size_t)ctx->geo.xchain;
    const size_t gp = (size_t)ctx->lay.gpitch;
    out->g_send_top = ctx->g + GHALO * gp;
    out->g_send_bottom = ctx->g + (size_t)(ctx->lay.rows + GHALO - 1) * gp;
    out->g_recv_top = ctx->g;
    out->g_recv_bottom = ctx->g + (size_t)(ctx->lay.rows + GHALO) * gp;
    out->g_row_bytes = gp;
    out->g_chain_stride = (size_t)ctx->geo.gchain;
    return PCA_OK;
}

pca_status pca_peer_info(pca_ctx* ctx, pca_peer* out) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!out) return fail(PCA_EINVAL, "out is NULL");
    memset(out, 0, sizeof(*out));
    out->x[0] = ctx->x[0];
    out->x[1] = ctx->x[1];
    out->flags = ctx->pflags;
    out->rows = ctx->lay.rows;
    out->batch = ctx->cfg.batch;
    out->chain_stride = ctx->geo.xchain;
    return PCA_OK;
}

pca_status pca_ipc_handle(pca_ctx* ctx, void* handle64, uint64_t* offset) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!handle64 || !offset) return fail(PCA_EINVAL, "handle / offset is NULL");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t must be 64 bytes");
    cudaSetDevice(ctx->device);
    CUdeviceptr base = 0;
    size_t size = 0;
    using RangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
        return fail(PCA_ECUDA, "cuMemGetAddressRange unavailable");
    const CUresult r = ((RangeFn)fn)(&base, &size, (CUdeviceptr)ctx->ws);
    if (r != CUDA_SUCCESS) return fail(PCA_ECUDA, "cuMemGetAddressRange: CUresult %d", (int)r);
    cudaIpcMemHandle_t h;
    CK(ctx, cudaIpcGetMemHandle(&h, (void*)base));
    memcpy(handle64, &h, 64);
    *offset = (uint64_t)((CUdeviceptr)ctx->ws - base);
    return PCA_OK;
}

pca_status pca_open_peer(pca_ctx* ctx, const void* handle64, uint64_t offset,
                         const pca_config* peer_cfg, pca_peer* out) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!handle64 || !peer_cfg || !out) return fail(PCA_EINVAL, "handle / config / out is NULL");
    st = validate(peer_cfg);
    if (st != PCA_OK) return st;
    if (peer_cfg->width != ctx->cfg.width || peer_cfg->height != ctx->cfg.height ||
        peer_cfg->batch != ctx->cfg.batch)
        return fail(PCA_EINVAL, "the peer's lattice (height, width, batch) differs from this context's");
    cudaSetDevice(ctx->device);
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    void* base = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
        return fail(PCA_ECUDA, "cudaIpcOpenMemHandle: CUDA error %d (%s)", (int)e, cudaGetErrorString(e));
    const Layout L = make_layout(peer_cfg);
    uint8_t* ws = (uint8_t*)base + offset;
    memset(out, 0, sizeof(*out));
    out->x[0] = ws + L.off_x0;
    out->x[1] = ws + L.off_x1;
    out->flags = (uint32_t*)(ws + L.off_flag + 64);
    out->ipc_base = base;
    out->rows = L.rows;
    out->batch = peer_cfg->batch;
    out->chain_stride = (int64_t)(L.rows + 2 * HALO) * L.xpitch;
    return PCA_OK;
}

pca_status pca_close_peer(pca_peer* peer) {
    if (!peer || !peer->ipc_base) return PCA_OK;
    const cudaError_t e = cudaIpcCloseMemHandle(peer->ipc_base);
    peer->ipc_base = nullptr;
    if (e != cudaSuccess)
        return fail(PCA_ECUDA, "cudaIpcCloseMemHandle: CUDA error %d (%s)", (int)e, cudaGetErrorString(e));
    return PCA_OK;
}

pca_status pca_attach_peers(pca_ctx* ctx, const pca_peer* up, const pca_peer* down) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (ctx->lay.rows == ctx->cfg.height) return fail(PCA_EINVAL, "peers need a row-strip context");
    if (ctx->p2p) return fail(PCA_EINVAL, "peers already attached");
    if (!up && !down) return fail(PCA_EINVAL, "no peer given");
    if (ctx->cfg.periodic && (!up || !down)) return fail(PCA_EINVAL, "a torus strip has two peers");
    const size_t pitch = (size_t)ctx->lay.xpitch;
    for (const pca_peer* q : {up, down}) {
        if (!q) continue;
        if (!q->x[0] || !q->x[1] || !q->flags || q->rows < HALO || q->batch != ctx->cfg.batch ||
            q->chain_stride != (int64_t)((q->rows + 2 * HALO) * pitch))
            return fail(PCA_EINVAL, "peer layout does not match this context's lattice");
    }
    StreamMemOps& M = memops();
    if (!M.wait || !M.write) return fail(PCA_EUNSUPPORTED, "%s", M.why.c_str());
    ctx->has_up = up != nullptr;
    ctx->has_dn = down != nullptr;
    if (up) ctx->up = *up;
    if (down) ctx->dn = *down;
    // the peers' g buffers: same lattice, their row count (x[0] is the workspace base)
    for (int i = 0; i < 2; ++i) {
        const pca_peer* q = i == 0 ? up : down;
        if (!q) continue;
        pca_config pc = ctx->cfg;
        pc.rows = q->rows;
        ctx->peer_g[i] = q->x[0] + make_layout(&pc).off_g;
    }
    ctx->p2p = 1;
    ctx->g_halo_valid = 0;
    // phase 1: the current state's edge rows into the peers' halo rows
    st = p2p_push(ctx, ctx->cur);
    if (st != PCA_OK) return st;
    return sync(ctx);
}

pca_status pca_nccl_unique_id(void* id128) {
    if (!id128) return fail(PCA_EINVAL, "id is NULL");
    NcclApi& N = nccl();
    if (!N.loaded) return fail(PCA_ENCCL, "%s", N.why.c_str());
    ncclUniqueId id;
    ncclResult_t e = N.GetUniqueId(&id);
    if (e != ncclSuccess) return fail(PCA_ENCCL, "ncclGetUniqueId: %s", N.GetErrorString(e));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
    memcpy(id128, &id, 128);
    return PCA_OK;
}

pca_status pca_attach_nccl(pca_ctx* ctx, const void* id128, int32_t nranks, int32_t rank) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (!id128 || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(PCA_EINVAL, "bad NCCL arguments");
    if (ctx->comm) return fail(PCA_EINVAL, "NCCL already attached");
    NcclApi& N = nccl();
    if (!N.loaded) return fail(PCA_ENCCL, "%s", N.why.c_str());
    ncclUniqueId id;
    memcpy(&id, id128, 128);
    ncclComm_t comm = nullptr;
    ncclResult_t e = N.CommInitRank(&comm, nranks, id, rank);
    if (e != ncclSuccess) return fail(PCA_ENCCL, "ncclCommInitRank: %s", N.GetErrorString(e));
    ctx->comm = comm;
    ctx->nranks = nranks;
    ctx->rank = rank;
    ctx->g_halo_valid = 0;
    st = exchange(ctx, ctx->x[ctx->cur]);
    if (st != PCA_OK) return st;
    return sync(ctx);
}

pca_status pca_sync(pca_ctx* ctx) {
    DeviceScope device_scope_;
    pca_status st = usable(ctx);
    if (st != PCA_OK) return st;
    if (ctx->copy) CK(ctx, cudaStreamSynchronize(ctx->copy));  // staged copies, async images
    return sync(ctx);
}

pca_status pca_destroy(pca_ctx* ctx) {
    DeviceScope device_scope_;
    if (!ctx) return PCA_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
        cudaEventDestroy(ctx->ev_fork);
        cudaEventDestroy(ctx->ev_join);
    }
    if (ctx->copy) {
        cudaStreamSynchronize(ctx->copy);
        cudaStreamDestroy(ctx->copy);
        cudaEventDestroy(ctx->ev_truth_ready);
        cudaEventDestroy(ctx->ev_truth_free);
        cudaEventDestroy(ctx->ev_in_ready);
        cudaEventDestroy(ctx->ev_in_free);
        cudaEventDestroy(ctx->ev_out_ready);
        cudaEventDestroy(ctx->ev_out_free);
    }
    for (auto& gr : ctx->graphs) cudaGraphExecDestroy(gr.exec);
    if (ctx->cap) cudaStreamDestroy(ctx->cap);
    if (ctx->comm) nccl().CommDestroy(ctx->comm);
    delete ctx;
    return PCA_OK;
}

}  // extern "C"
