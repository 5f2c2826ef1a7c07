/*
 * include/pca.h -- C ABI of the B200-native synchronous lazy-PCA sweep library
 * (libpca_b200.so), arXiv 2507.14869.  SURVEY.md section 8(b) is the contract.
 *
 * The library samples the lazy Probabilistic Cellular Automaton of PAPER.md section 5.2
 * (transition display PAPER.md:462-477): at every sweep t each site i
 * of the lattice independently draws its new gray level w_i with probability
 *     p_i(s; x) ∝ exp( a*n_i(s;x) - b*(lum g_i - lum s)^2 - c*pen(x_i, s) ),
 *     a = coef_scale*2*beta_t*J,  b = coef_scale/(2 sigma^2),  c = beta_t*q,
 *     pen = 1{s != x_i} (L0, the paper's), or |lum x_i - lum s|^p for p = 1, 2 (the
 *     L1 / L2 alternatives of PAPER.md:279 and 483-485; see inertia_p),
 *     beta_t = beta0 + beta_step*floor(t/beta_period),
 * from the PREVIOUS configuration x (double buffering), where n_i(s;x) is
 * the number of neighbours (Moore-8, or von Neumann-4) carrying s and
 * lum(k) = k/(levels-1).  DESIGN.md section 3 lists the readings
 * (R1..R20) taken where the paper is ambiguous.  Running per-site label counts give the
 * posterior-marginal (MPM) estimate; PSNR and global SSIM are
 * reduced on the device.
 *
 * Random numbers: Philox4x32-10 keyed by (seed mod 2^32, seed >> 32) with counter
 * (col>>2, row, t, 1<<24 | chain), word col&3, u = r*2^-32, so a
 * chain is a pure function of (config, g, x0, number of sweeps): independent of GPU
 * count, row split, batch composition and launch configuration.
 *
 * Layout of every image argument: dense, row-major uint8 level indices
 * [batch][rows][width] (chain-major), values in [0, levels).  Count arrays are uint16,
 * planar: levels == 2 -> [batch][rows][width] (count of label 1); levels > 2 ->
 * [batch][levels][rows][width].
 *
 * Pointers: every image/count pointer may be HOST memory (pageable or pinned) or DEVICE
 * memory of the context's device; the library detects which (CUDA UVA) and copies
 * accordingly.  Device memory is never allocated by the library: the caller owns one
 * workspace buffer of pca_workspace_bytes() bytes, which must outlive the context.
 *
 * Streams: all device work is enqueued on the caller's stream given to pca_init.
 * pca_sweep is asynchronous; every call that returns data (estimate, read_*, psnr_ssim,
 * metric_sums, get_stats) synchronises that stream before returning.
 *
 * Errors: every call returns a pca_status and never aborts or throws across the ABI.
 * Arguments are validated before any device work.  Asynchronous CUDA/NCCL errors
 * surface at the next synchronising call as PCA_ECUDA / PCA_ENCCL; after any CUDA/NCCL
 * error the context is poisoned and every call except pca_destroy returns PCA_ESTATE.
 * pca_last_error() returns a thread-local message for the most recent failure.
 */
#ifndef PCA_B200_H
#define PCA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCA_ABI_VERSION 1

typedef struct pca_ctx pca_ctx; /* opaque; one per GPU per lattice strip / chain batch */

typedef enum {
    PCA_OK = 0,
    PCA_EINVAL = -1,        /* invalid argument or configuration                       */
    PCA_ESTATE = -2,        /* context poisoned by an earlier CUDA/NCCL error          */
    PCA_ECUDA = -3,         /* CUDA runtime error                                      */
    PCA_ENCCL = -4,         /* NCCL error (or NCCL library not loadable)               */
    PCA_ENOSPACE = -5,      /* workspace smaller than pca_workspace_bytes()            */
    PCA_EUNSUPPORTED = -6   /* valid but unsupported (see pca_last_error)             */
} pca_status;

enum { PCA_NBHD_VN4 = 4, PCA_NBHD_MOORE8 = 8 };

/* Estimate kinds for pca_estimate / pca_psnr_ssim / pca_metric_sums. */
enum {
    PCA_EST_LAST = 0,      /* the current sample x_t ("last sample")           */
    PCA_EST_MPM = 1,       /* argmax_k count_k, ties to the lowest label (R15)               */
    PCA_EST_MARGINALS = 2, /* float32 [batch][levels][rows][width] = count_k / N_samp      */
    PCA_EST_CM = 3         /* float32 [batch][rows][width] = sum_k lum(k) count_k / N_samp  */
};

/* Kernel selection (all give the same chain up to fp64 near-ties).  Runs of
 * sweeps on small contexts (rows x width x batch <= 2^18) execute in one cooperative launch
 * of the general code whatever the selection (exact integer thresholds for levels == 2). */
enum {
    PCA_KERNEL_AUTO = 0,    /* levels == 2: PACKED when eligible, else BINARY; TABLE for 3..5 */
                            /* levels; else GENERAL                                          */
    PCA_KERNEL_GENERAL = 1, /* levels == 2: integer thresholds for every site; more levels:  */
                            /* integer thresholds where all neighbours agree (levels <= 16), */
                            /* else fp64 per-site weights (log-domain when they overflow)    */
    PCA_KERNEL_BINARY = 2,  /* levels == 2: TMA-staged rows, SWAR neighbour counts, integer  */
                            /* thresholds                                                    */
    PCA_KERNEL_TABLE = 3,   /* 3..5 levels (AUTO's choice there when width and rows <= 65535): */
                            /* per-site neighbour histograms; integer thresholds for every     */
                            /* interior site with <= 2 distinct neighbour labels (one table    */
                            /* row per histogram, g, x), fp64 weights for the others           */
    PCA_KERNEL_PACKED = 4   /* levels == 2, width % 512 == 0 (whole lattice or row strip): g and the state */
                            /* bit-packed in HBM (1 bit per site) during runs of sweeps; the   */
                            /* binary kernel's decisions (same chain)                          */
};

typedef struct pca_config {
    int32_t height;        /* H: global rows of one chain's lattice (>= 1; >= 3 if periodic)  */
    int32_t width;         /* W: columns (>= 1; >= 3 if periodic)                             */
    int32_t batch;         /* number of independent chains in this context (>= 1)             */
    int32_t levels;        /* l gray levels, 2..255                            */
    int32_t neighborhood;  /* PCA_NBHD_MOORE8 (paper) or PCA_NBHD_VN4                         */
    int32_t periodic;      /* 0 = free boundary, 1 = torus                     */
    double J;              /* prior coupling > 0 (1/3 in PAPER.md:500)       */
    double q;              /* inertia >= 0 (0.51 in PAPER.md:508)               */
    double sigma;          /* noise std in luminance units > 0                 */
    double beta0;          /* beta at t = 0, > 0 (1.25)                          */
    double beta_step;      /* beta increment >= 0 (0.25)                         */
    int32_t beta_period;   /* sweeps per beta stage > 0 (250)                    */
    int32_t chain0;        /* chain id of this context's first chain (RNG counter), >= 0      */
    double coef_scale;     /* > 0; 1.0 = paper-literal a, b; 0.5 = matched mode (R4)           */
    uint64_t seed;         /* Philox key                                                       */
    int32_t mpm_burn_in;   /* count x_{t+1} for sweeps t >= burn_in; < 0 disables counts       */
    int32_t row0;          /* first global row owned by this context (sharding), >= 0         */
    int32_t rows;          /* owned rows; 0 means all H rows (row0 must then be 0)            */
    int32_t kernel;        /* PCA_KERNEL_*                                                     */
    int32_t rows_per_thread; /* binary kernel: rows per warp task; 0 = auto (one wave)       */
    int32_t sweeps_per_pass; /* 0 = auto (1); 1 = one sweep per kernel launch; 2 = two      */
                           /* sweeps per HBM pass (temporal blocking; same chain) when       */
                           /* levels == 2 and W % 16 == 0 (kernel BINARY); on a row strip the */
                           /* halos are 2 rows deep and exchanged once per pass              */
    int32_t inertia_p;     /* inertia norm p: 0 = L0 1{s != x_i} (paper), 1 = |lum x_i - lum s|,*/
                           /* 2 = (lum x_i - lum s)^2; identical for   */
                           /* levels == 2                                                      */
    int32_t packed_io;     /* levels == 2 only: 1 = every image argument and result (g, x0,     */
                           /* truth, LAST / MPM estimates, state) is bit-packed: each row is     */
                           /* ceil(width/8) bytes, column c at bit c%8 (LSB first) of byte c/8;  */
                           /* 8x fewer host<->device bytes.  The sweep itself runs on uint8.    */
    int32_t graphs;        /* 1 = pca_sweep(n) runs are captured into CUDA graphs and replayed */
                           /* when the same run recurs (same t, n, counted, state buffer, table */
                           /* stage): one graph launch instead of one launch (or, on NCCL row  */
                           /* strips, ~8 stream operations) per sweep.  levels == 2; not with  */
                           /* attached peers (their phase words change every call)            */
    int32_t reserved[3];   /* must be zero                                                     */
} pca_config;

typedef struct pca_stats {
    int64_t sweeps_done;     /* t: sweeps applied since init/reset (+ pca_set_step offset)    */
    int64_t counted_sweeps;  /* N_samp: sweeps accumulated into the MPM counts               */
    int64_t kernel_launches; /* library kernels launched since init (all kinds)             */
    int64_t sweep_launches;  /* sweep kernels launched since init                           */
    double beta;             /* beta of the most recent sweep (beta0 before the first)       */
    int32_t kernel;          /* PCA_KERNEL_BINARY, _GENERAL, _TABLE or _PACKED actually used */
    int32_t nranks;          /* NCCL ranks attached (1 if none)                              */
    int64_t graph_replays;   /* pca_sweep runs replayed from a captured CUDA graph (graphs)  */
} pca_stats;

/* Halo rows of the CURRENT state buffer, for caller-driven (loopback) exchange between
 * strip contexts.  Each pointer is a device pointer to a block of `row_bytes` bytes (the
 * halo depth, 2 padded rows) for chain 0; chain b is at + b*chain_stride.  send_top /
 * send_bottom are the context's first / last two owned rows, recv_top / recv_bottom the
 * two halo rows above / below: copy a neighbour's send block onto the matching recv. */
typedef struct pca_halo {
    uint8_t* send_top;
    uint8_t* send_bottom;
    uint8_t* recv_top;
    uint8_t* recv_bottom;
    size_t row_bytes;
    size_t chain_stride;
    /* the observed image's first / last owned row and its halo row above / below (one padded
     * row each): with sweeps_per_pass == 2 a strip recomputes one row beyond its edges, so the
     * caller copies a neighbour's g send row onto the matching g recv row once after
     * pca_init / a pca_reset with a new g (NCCL or attached peers do this themselves) */
    uint8_t* g_send_top;
    uint8_t* g_send_bottom;
    uint8_t* g_recv_top;
    uint8_t* g_recv_bottom;
    size_t g_row_bytes;
    size_t g_chain_stride;
} pca_halo;

/* Device-initiated halo exchange: what a strip context needs to know
 * about a neighbouring rank's context.  x[0], x[1]: the peer's two state buffers (padded row
 * -2 of chain 0, device pointers valid in THIS process); flags: the peer's two phase words;
 * chain_stride: bytes between its chains; ipc_base: the mapping pca_open_peer made (release
 * it with pca_close_peer), NULL for an in-process peer from pca_peer_info. */
typedef struct pca_peer {
    uint8_t* x[2];
    uint32_t* flags;
    void* ipc_base;
    int32_t rows;
    int32_t batch;
    int64_t chain_stride;
} pca_peer;

/* Devices: a context lives on the device that was current at pca_init.  Every call that
 * takes a context runs on that device and restores the caller's current device before it
 * returns, so one host thread may drive contexts on several GPUs. */

/* Version of this ABI (PCA_ABI_VERSION). */
int32_t pca_abi_version(void);

/* Bytes of device workspace a context with this configuration needs; 0 if the
 * configuration is invalid (pca_last_error explains). */
size_t pca_workspace_bytes(const pca_config* cfg);

/* Create a context on the current CUDA device.
 *   workspace: device buffer of ws_bytes >= pca_workspace_bytes(cfg), 256-B aligned,
 *              owned by the caller; must outlive the context.
 *   g:  observed (noisy) image [batch][rows][width], host or device; copied.
 *   x0: initial state, same layout; NULL means x0 = g (R9); copied.
 *   stream: cudaStream_t to enqueue all work on (NULL = legacy default stream).
 * Returns PCA_EINVAL (bad cfg/pointers), PCA_ENOSPACE, PCA_EUNSUPPORTED, PCA_ECUDA. */
pca_status pca_init(pca_ctx** out, const pca_config* cfg, void* workspace, size_t ws_bytes,
                    const uint8_t* g, const uint8_t* x0, void* stream);

/* Restart the chain: t = 0, counts = 0; g replaced if non-NULL; state = x0 (or g if x0 is
 * NULL).  Equivalent to a fresh pca_init on the same workspace. */
pca_status pca_reset(pca_ctx* ctx, const uint8_t* g, const uint8_t* x0);

/* Enqueue n >= 0 synchronous PCA sweeps t, t+1, ..., t+n-1 (asynchronous).  When the
 * context owns a strip (rows < height) and NCCL is attached, each sweep is followed by
 * the halo exchange with the neighbouring ranks; without NCCL or peers, n must be <= 1 (<= 2
 * with sweeps_per_pass == 2: one pass) and the caller exchanges halos (pca_halo_ptrs).  Returns PCA_EUNSUPPORTED if the uint16 MPM
 * counters would overflow (> 65535 counted sweeps) or the sweep index would pass 2^32-1; the
 * sweeps before the refused one run and are counted (state, sweep index and counts agree). */
pca_status pca_sweep(pca_ctx* ctx, int32_t n);

/* Write an estimate of the chain (kind PCA_EST_*) to out (host or device; layout in the
 * enum).  MPM / MARGINALS / CM need counting enabled and N_samp >= 1.  Synchronises. */
pca_status pca_estimate(pca_ctx* ctx, int32_t kind, void* out);

/* Exact integer sums of estimate `kind` (LAST or MPM) y against the original `truth`
 * x (uint8 [batch][rows][width], host or device), per chain, over this context's rows:
 * sums[b*8 + {0..6}] = {sum (x-y)^2, sum x, sum y, sum x^2, sum y^2, sum x*y, max x}, in
 * level units, slot 7 = site count.  With NCCL attached the sums (max for slot 6) are
 * all-reduced over ranks.  Synchronises. */
pca_status pca_metric_sums(pca_ctx* ctx, const uint8_t* truth, int32_t kind, int64_t* sums);

/* PSNR (dB) and global SSIM (R16, R17) of estimate `kind` against
 * truth, per chain, from pca_metric_sums computed exactly in 128-bit integers and then
 * fp64.  psnr = +inf when MSE = 0; PCA_EINVAL if the original is all black. */
pca_status pca_psnr_ssim(pca_ctx* ctx, const uint8_t* truth, int32_t kind, double* psnr,
                         double* ssim);

/* Copy the truth image (host or device [batch][rows][width]) into the context on an internal
 * copy stream, so the transfer overlaps the sweeps enqueued after it; a later pca_finalize
 * with truth == NULL uses it (and waits for the copy on the device, not the host).  Host
 * memory must stay valid until that finalize returns (pinned memory makes the copy truly
 * asynchronous).  Asynchronous. */
pca_status pca_stage_truth(pca_ctx* ctx, const uint8_t* truth);

/* Stage the NEXT reset's observed image g (host or device, the layout of pca_init's g; bit-
 * packed with packed_io) into the context on the internal copy stream, so the transfer overlaps
 * the work enqueued after it; pca_reset_staged then resets from it (x0 = g), waiting for the
 * copy on the device, not the host.  Host memory must stay valid until the copy has run:
 * until that reset returns, or with packed_io until the next synchronising call after it
 * (pinned memory makes the copy truly asynchronous).  A second pca_stage_input waits for the
 * first to be consumed.  Asynchronous. */
pca_status pca_stage_input(pca_ctx* ctx, const uint8_t* g);

/* pca_reset(ctx, g_staged, NULL) with the image of the last pca_stage_input; PCA_EINVAL when
 * nothing is staged.  Synchronises like pca_reset, except with packed_io: bit-unpacked labels
 * are valid by construction, so the level check and its host synchronisation are skipped and
 * the call is asynchronous. */
pca_status pca_reset_staged(pca_ctx* ctx);

/* The end of a run in ONE fused pass over truth, the current state and the counts
 * (SURVEY 8(a) a8 + a9): the MPM image (written to mpm_out, host or device
 * [batch][rows][width], when non-NULL) and PSNR / global SSIM of both the last sample and
 * the MPM estimate, psnr[2*b + 0] / ssim[2*b + 0] for LAST and [2*b + 1] for MPM (each
 * array [batch][2]).  truth == NULL: the image given to pca_stage_truth.  Same definitions and
 * exactness as pca_psnr_ssim; needs counted sweeps; sums are all-reduced over NCCL for row
 * strips.  Synchronises. */
pca_status pca_finalize(pca_ctx* ctx, const uint8_t* truth, uint8_t* mpm_out, double* psnr,
                        double* ssim);

/* pca_finalize, except that a host mpm_out (or any mpm_out with packed_io) is filled on the
 * context's copy stream: PSNR / SSIM are returned as by pca_finalize, but the MPM image may
 * still be in flight at return, so that its device->host copy overlaps the work enqueued next
 * (the next run's reset and sweeps).  mpm_out must stay valid and unread until pca_sync; later
 * calls that reuse the context's output staging wait for the copy on the device.  A device
 * mpm_out without packed_io is written as by pca_finalize.  Same errors as pca_finalize. */
pca_status pca_finalize_async(pca_ctx* ctx, const uint8_t* truth, uint8_t* mpm_out, double* psnr,
                              double* ssim);

/* Windowed SSIM (R16's secondary metric, the form Table 1 of PAPER.md:703 appears to use):
 * the mean over every 7x7 window position inside the image (stride 1, no padding) of
 *   SSIM_w = (2 mx my + c1)(2 sxy + c2) / ((mx^2 + my^2 + c1)(sx^2 + sy^2 + c2)),
 * uniform weights, sample (N-1) variances, c1 = 1e-4, c2 = 9e-4, luminance units.  Window
 * moments are exact (integer sums); ssim[b] per chain.  kind = PCA_EST_LAST or PCA_EST_MPM;
 * truth host or device [batch][height][width].  PCA_EINVAL if height or width < 7;
 * PCA_EUNSUPPORTED for a row-strip context (windows would span ranks).  Synchronises. */
pca_status pca_ssim_windowed(pca_ctx* ctx, const uint8_t* truth, int32_t kind, double* ssim);

/* Enqueue n sweeps of the Gibbs sampler (conditional PAPER.md:417-429,
 * no inertia term) on the same state, schedule, sweep counter t and MPM counts: a
 * systematic scan in checkerboard colour order (4-neighbour: colours (r + c) mod 2;
 * Moore-8: 2 (r mod 2) + (c mod 2); global r) with the Philox words of tag GIBBS.  The
 * paper's own scan is column-major; the colour order gives another chain
 * with the same stationary law (R21).  Launches: von Neumann-4, one per colour (in
 * place); Moore-8, one per row parity (both colours of the row), double-buffered for two
 * levels.  PCA_EUNSUPPORTED on a torus with odd height or width (the colouring would not be
 * proper); a row strip needs NCCL attached (halos are exchanged after every launch).
 * Asynchronous like pca_sweep. */
pca_status pca_gibbs_sweep(pca_ctx* ctx, int32_t n);

/* Copy the current state [batch][rows][width] to out / from x (host or device). */
pca_status pca_read_state(pca_ctx* ctx, uint8_t* out);
pca_status pca_write_state(pca_ctx* ctx, const uint8_t* x);

/* Copy the MPM counters (uint16, layout above) to out / from c.  Used for checkpoints. */
pca_status pca_read_counts(pca_ctx* ctx, uint16_t* out);
pca_status pca_write_counts(pca_ctx* ctx, const uint16_t* c, int64_t counted_sweeps);

/* Set the sweep index t of the next sweep (checkpoint resume). */
pca_status pca_set_step(pca_ctx* ctx, int64_t t);

pca_status pca_get_stats(pca_ctx* ctx, pca_stats* out);

/* Number of sites whose label changed in the most recent sweep, per chain (changed[batch]),
 * for the strip this context owns: x_t against x_{t-1}, which the double buffer still holds
 * after PCA sweeps (and two-level Moore Gibbs sweeps).  PCA_EINVAL before the first sweep,
 * after pca_reset / pca_write_state, or after an in-place Gibbs sweep.  Synchronises. */
pca_status pca_changed_sites(pca_ctx* ctx, int64_t* changed);

/* Device pointers of the halo rows of the current state (loopback exchange). */
pca_status pca_halo_ptrs(pca_ctx* ctx, pca_halo* out);

/* NCCL (row-strip sharding, one context per GPU per rank).  pca_nccl_unique_id fills
 * 128 bytes (ncclUniqueId) on rank 0; the caller broadcasts them (torch.distributed);
 * pca_attach_nccl creates the communicator owned by the context. */
pca_status pca_nccl_unique_id(void* id128);
pca_status pca_attach_nccl(pca_ctx* ctx, const void* id128, int32_t nranks, int32_t rank);

/* Device-initiated halo exchange over peer memory (the per-sweep
 * exchange of PAPER.md's synchronous update across row strips), an alternative
 * to NCCL for PCA sweeps on row strips:
 *   pca_peer_info   this context's buffers and phase words (for a peer in the same process);
 *   pca_ipc_handle  the CUDA IPC handle (64 bytes) of the allocation holding the workspace and
 *                   the workspace's byte offset in it, for a peer in another process;
 *   pca_open_peer   maps another process's workspace (handle, offset, and that rank's config:
 *                   same height, width, batch) into this context's device;
 *   pca_close_peer  unmaps it (after the contexts using it are destroyed);
 *   pca_attach_peers  up = the rank owning the rows above this strip, down = below (NULL at a
 *                   free-boundary end; a torus strip needs both).  Pushes the current state's
 *                   edge rows (phase 1) and synchronises.
 * Once attached, every PCA sweep is ONE launch whose edge-row CTAs also store the new rows
 * into the peers' halo rows; every sweep and state load is a phase k, preceded on the stream by
 * a wait until both peers completed phase k-1 (cuStreamWaitValue32 on this context's phase
 * words; no kernel spins) and followed by a write of k into the peers' phase words
 * (cuStreamWriteValue32, fenced).  Every rank must issue the same sequence of sweeps and state
 * loads (SPMD), and the contexts must run on different streams (in practice different GPUs):
 * a call with several phases (pca_sweep(n > 1), a Gibbs sweep) waits on the peers' later
 * phases, which on a shared stream would be queued behind the wait.  Row-strip Gibbs sweeps
 * use the peers too: each launch is a phase whose edge rows are copied to the peers after it.
 * The metric reductions still use NCCL when it is attached, else they cover this strip only.
 * Errors: PCA_EINVAL (not a strip, already attached, layout mismatch), PCA_ECUDA (IPC or
 * stream memory operations unavailable / failed), PCA_EUNSUPPORTED (no stream memory ops). */
pca_status pca_peer_info(pca_ctx* ctx, pca_peer* out);
pca_status pca_ipc_handle(pca_ctx* ctx, void* handle64, uint64_t* offset);
pca_status pca_open_peer(pca_ctx* ctx, const void* handle64, uint64_t offset, const pca_config* peer_cfg,
                         pca_peer* out);
pca_status pca_close_peer(pca_peer* peer);
pca_status pca_attach_peers(pca_ctx* ctx, const pca_peer* up, const pca_peer* down);

/* Synchronise the context's stream and its copy stream (staged inputs, pca_finalize_async's
 * image) and report any pending asynchronous error. */
pca_status pca_sync(pca_ctx* ctx);

/* Destroy the context (and its NCCL communicator).  Never frees caller memory. */
pca_status pca_destroy(pca_ctx* ctx);

/* Thread-local message describing the most recent failure in this thread. */
const char* pca_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* PCA_B200_H */
