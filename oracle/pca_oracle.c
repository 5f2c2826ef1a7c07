/*
 * oracle/pca_oracle.c -- the CPU ORACLE for arXiv 2507.14869 (lazy PCA denoising).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load, call or execute this code.  The
 * product path (paper_2507_14869_b200/) never imports, links or calls it; the two
 * share no code, headers, tables or constants.
 *
 * Plain, slow, single-threaded fp64 C.  Every function follows a passage of
 * /root/reference/PAPER.md (cited as PAPER.md:<line> with its section/equation) or
 * a reading recorded in DESIGN.md section "Readings" (R1..R20, which mirror
 * SURVEY.md section 8(c) A1..A20).  No blocking, fusion or reordering beyond the
 * definitions: one site at a time, loops in the order the paper states them.
 *
 * Notation:
 *   lum(k) = k/(l-1)                             PAPER.md:328-334 (section 4), R6
 *   N(i)   = Moore-8 (PAPER.md:356-359 eq. neighborhood) or von Neumann-4 (config 1)
 *            free boundary or torus (R7)
 *   n_i(s;x) = #{j in N(i): x_j = s}
 *   a = coef_scale * 2*beta*J,   b = coef_scale / (2 sigma^2),   c = beta*q   (R4, R5)
 *   E_i(s;x) = a*n_i(s;x) - b*(lum g_i - lum s)^2 - c*1{s != x_i}
 *            PAPER.md:462-477 (section 5.2, transition display; inertia index typo
 *            1{s != x_j} read as 1{s != x_i}, R1)
 *   Gibbs conditional: the same without the inertia term
 *            (eq. gibbs_sampler_elementary_step)
 *   Random numbers: Philox4x32-10 (Salmon et al., Random123), key = seed,
 *            counter = (col>>2, row, t, tag<<24 | chain), word = col & 3,
 *            u = r * 2^-32.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_TAG_PCA 1u
#define ORC_TAG_GIBBS 2u
#define ORC_TAG_NOISE 3u
#define ORC_TAG_GEN_INIT 4u
#define ORC_TAG_GEN_GIBBS 5u

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11, "Parallel random numbers: as
 * easy as 1, 2, 3").  One round:
 *   (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,
 *   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0);  then k += (W0, W1).        */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
    uint32_t k0 = key[0], k1 = key[1];
    for (int round = 0; round < 10; round++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* The canonical per-site draw. */
uint32_t orc_draw(uint64_t seed, uint32_t tag, uint32_t chain, uint32_t t,
                  uint32_t row, uint32_t col) {
    uint32_t ctr[4] = {col >> 2, row, t, (tag << 24) | chain};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    return out[col & 3u];
}

/* Annealing schedule, PAPER.md:508 (section 6): "started with beta = 1.25 and
 * increased it by 0.25 every 250 steps":  beta_t = beta0 + step*floor(t/period). */
double orc_beta_at(double beta0, double beta_step, int period, int t) {
    return beta0 + beta_step * (double)(t / period);
}

/* ------------------------------------------------------------------------- */
typedef struct {
    int H, W;          /* rows, columns of one chain's lattice                      */
    int levels;        /* l >= 2 gray levels                          */
    int nbhd;          /* 8 = Moore, 4 = von Neumann             */
    int periodic;      /* 0 = free boundary, 1 = torus               */
    double J;          /* prior coupling                          */
    double q;          /* inertia, PAPER.md:455, 508 (q = 0.51)                     */
    double sigma;      /* noise std in luminance units            */
    double coef_scale; /* 1.0 = paper-literal a, b; 0.5 = matched mode (R4)        */
    int inertia_p;     /* inertia norm exponent p in {0, 1, 2}  */
} orc_model;

static double lum(int k, int levels) { return (double)k / (double)(levels - 1); }

/* Inertia penalty |x_i - s|^p on luminances with the convention 0^0 = 0 (PAPER.md:279:
 * "q ||x - w|| = sum_i q |x_i - w_i|^p ... 0^0 = 0"; L0 is the paper's choice, PAPER.md:455,
 * L1 / L2 the alternatives of PAPER.md:483-485).                                   */
static double inertia_penalty(int p, int xi, int s, int levels) {
    if (s == xi) return 0.0;
    if (p == 0) return 1.0;
    double d = lum(xi, levels) - lum(s, levels);
    return p == 1 ? fabs(d) : d * d;
}

/* Is (p, q) in F(r, c)?  PAPER.md:356-357: max(|r-p|, |c-q|) = 1 (Moore), or the
 * 4-neighbour variant |r-p| + |c-q| = 1.  Offsets are tested one at a time.      */
static int offset_in_neighbourhood(int nbhd, int dr, int dc) {
    int adr = dr < 0 ? -dr : dr, adc = dc < 0 ? -dc : dc;
    if (nbhd == 8) return (adr > adc ? adr : adc) == 1;
    return adr + adc == 1;
}

/* n_i(s; x) for every s: count neighbours of (r, c) carrying label s.
 * Free boundary: out-of-lattice neighbours do not exist.
 * Torus: indices wrap modulo H, W.                                               */
static void neighbour_counts(const orc_model* m, const uint8_t* x, int r, int c, int* n) {
    for (int s = 0; s < m->levels; s++) n[s] = 0;
    for (int dr = -1; dr <= 1; dr++) {
        for (int dc = -1; dc <= 1; dc++) {
            if (!offset_in_neighbourhood(m->nbhd, dr, dc)) continue;
            int rr = r + dr, cc = c + dc;
            if (m->periodic) {
                rr = (rr + m->H) % m->H;
                cc = (cc + m->W) % m->W;
            } else if (rr < 0 || rr >= m->H || cc < 0 || cc >= m->W) {
                continue;
            }
            n[x[rr * m->W + cc]] += 1;
        }
    }
}

/* Per-site PCA conditional p_i(s; x), PAPER.md:462-477 (section 5.2):
 *   p(s) = exp(E(s) - max E) / sum_s' exp(E(s') - max E).
 * with_inertia = 0 gives the Gibbs conditional of PAPER.md:417-429.              */
static void site_probs(const orc_model* m, const uint8_t* x, const uint8_t* g, int r, int c,
                       double beta, int with_inertia, double* p) {
    int n[256];
    double E[256];
    neighbour_counts(m, x, r, c, n);
    double a = m->coef_scale * 2.0 * beta * m->J;
    double b = m->coef_scale / (2.0 * m->sigma * m->sigma);
    double cq = beta * m->q;
    int xi = x[r * m->W + c];
    int gi = g[r * m->W + c];
    double Emax = -INFINITY;
    for (int s = 0; s < m->levels; s++) {
        double d = lum(gi, m->levels) - lum(s, m->levels);
        double inert = with_inertia ? inertia_penalty(m->inertia_p, xi, s, m->levels) : 0.0;
        E[s] = a * (double)n[s] - b * d * d - cq * inert;
        if (E[s] > Emax) Emax = E[s];
    }
    double Z = 0.0;
    for (int s = 0; s < m->levels; s++) {
        p[s] = exp(E[s] - Emax);
        Z += p[s];
    }
    for (int s = 0; s < m->levels; s++) p[s] = p[s] / Z;
}

void orc_pca_site_probs(const orc_model* m, const uint8_t* x, const uint8_t* g, int r, int c,
                        double beta, double* p) {
    site_probs(m, x, g, r, c, beta, 1, p);
}

void orc_gibbs_site_probs(const orc_model* m, const uint8_t* x, const uint8_t* g, int r, int c,
                          double beta, double* p) {
    site_probs(m, x, g, r, c, beta, 0, p);
}

/* Inverse-CDF draw over ascending labels with one uniform (R14):
 *   F_k = sum_{s<=k} p(s);  w = min{k < l-1 : u < F_k}, else l-1.
 * margin = min_{k<l-1} |u - F_k|: distance of u to the nearest decision threshold
 * (used to classify GPU/oracle mismatches as near-ties, R19).                    */
int orc_decide(const double* p, int levels, double u, double* margin) {
    double F = 0.0;
    int w = levels - 1;
    double mg = INFINITY;
    for (int k = 0; k < levels - 1; k++) {
        F += p[k];
        double dist = fabs(u - F);
        if (dist < mg) mg = dist;
        if (w == levels - 1 && u < F) w = k;
    }
    if (margin) *margin = mg;
    return w;
}

/* One synchronous PCA sweep (PAPER.md:198-204 eq. general_pca_definition with the
 * per-site law of PAPER.md:462-477): every site of rows [r_begin, r_end) is drawn
 * independently from the OLD configuration x and written to out ("a temporary
 * matrix which is reset as the current matrix at the end of each step",
 * PAPER.md:723).  Random word: tag PCA, counter t = sweep index.                */
void orc_pca_sweep_rows(const orc_model* m, const uint8_t* x, const uint8_t* g, uint8_t* out,
                        double* margin, double beta, uint64_t seed, uint32_t chain, uint32_t t,
                        int r_begin, int r_end) {
    double p[256];
    for (int r = r_begin; r < r_end; r++) {
        for (int c = 0; c < m->W; c++) {
            site_probs(m, x, g, r, c, beta, 1, p);
            uint32_t rnd = orc_draw(seed, ORC_TAG_PCA, chain, t, (uint32_t)r, (uint32_t)c);
            double u = (double)rnd * (1.0 / 4294967296.0);
            double mg;
            out[r * m->W + c] = (uint8_t)orc_decide(p, m->levels, u, &mg);
            if (margin) margin[r * m->W + c] = mg;
        }
    }
}

void orc_pca_sweep(const orc_model* m, const uint8_t* x, const uint8_t* g, uint8_t* out,
                   double* margin, double beta, uint64_t seed, uint32_t chain, uint32_t t) {
    orc_pca_sweep_rows(m, x, g, out, margin, beta, seed, chain, t, 0, m->H);
}

/* A PCA chain of n sweeps starting at sweep index t0 from state x (updated in
 * place), with the annealing schedule of PAPER.md:508 and MPM counts (R15):
 * counts[k][i] += 1{x_{t+1,i} = k} for every sweep t >= burn_in (burn_in < 0: off).
 * counts is uint32 planar [levels][H][W] (may be NULL).                          */
void orc_pca_run(const orc_model* m, uint8_t* x, const uint8_t* g, uint32_t* counts,
                 int t0, int n, double beta0, double beta_step, int period, uint64_t seed,
                 uint32_t chain, int burn_in) {
    size_t N = (size_t)m->H * (size_t)m->W;
    uint8_t* tmp = (uint8_t*)malloc(N);
    for (int t = t0; t < t0 + n; t++) {
        double beta = orc_beta_at(beta0, beta_step, period, t);
        orc_pca_sweep(m, x, g, tmp, NULL, beta, seed, chain, (uint32_t)t);
        memcpy(x, tmp, N);
        if (counts && burn_in >= 0 && t >= burn_in) {
            for (size_t i = 0; i < N; i++) counts[(size_t)x[i] * N + i] += 1;
        }
    }
    free(tmp);
}

/* Systematic single-site Gibbs sweep: sites visited in
 * column-major order ("for instance the column-major one"), each
 * resampled in place from the conditional of PAPER.md:417-429 given the CURRENT
 * (partially updated) configuration.  Random word: tag GIBBS, counter t.         */
void orc_gibbs_sweep(const orc_model* m, uint8_t* x, const uint8_t* g, double beta,
                     uint64_t seed, uint32_t chain, uint32_t t) {
    double p[256];
    for (int c = 0; c < m->W; c++) {
        for (int r = 0; r < m->H; r++) {
            site_probs(m, x, g, r, c, beta, 0, p);
            uint32_t rnd = orc_draw(seed, ORC_TAG_GIBBS, chain, t, (uint32_t)r, (uint32_t)c);
            double u = (double)rnd * (1.0 / 4294967296.0);
            x[r * m->W + c] = (uint8_t)orc_decide(p, m->levels, u, NULL);
        }
    }
}

/* Colour of site (r, c) in the checkerboard partition of the lattice graph: von Neumann-4
 * (r + c) mod 2 (2 colours), Moore-8 2(r mod 2) + (c mod 2) (4 colours).  No two sites of
 * one colour are neighbours (on a torus: when H and W are even), so the systematic scan
 * "colour 0, colour 1, ..." is a scan order whose colour classes can be updated at once.  */
int orc_gibbs_colour(int nbhd, int r, int c) {
    return nbhd == 4 ? ((r + c) & 1) : (((r & 1) << 1) | (c & 1));
}

/* One colour phase of the colour-order scan: every site of colour k in rows [r_begin, r_end),
 * row-major, in place, from its Gibbs conditional given the CURRENT
 * configuration.  Random word: tag GIBBS, counter t.                                      */
void orc_gibbs_colour_phase(const orc_model* m, uint8_t* x, const uint8_t* g, double beta,
                            uint64_t seed, uint32_t chain, uint32_t t, int k, int r_begin,
                            int r_end) {
    double p[256];
    for (int r = r_begin; r < r_end; r++) {
        for (int c = 0; c < m->W; c++) {
            if (orc_gibbs_colour(m->nbhd, r, c) != k) continue;
            site_probs(m, x, g, r, c, beta, 0, p);
            uint32_t rnd = orc_draw(seed, ORC_TAG_GIBBS, chain, t, (uint32_t)r, (uint32_t)c);
            double u = (double)rnd * (1.0 / 4294967296.0);
            x[r * m->W + c] = (uint8_t)orc_decide(p, m->levels, u, NULL);
        }
    }
}

/* One systematic Gibbs sweep in colour order: colour 0, 1, ...,
 * each phase over the whole lattice.                                                      */
void orc_gibbs_sweep_coloured(const orc_model* m, uint8_t* x, const uint8_t* g, double beta,
                              uint64_t seed, uint32_t chain, uint32_t t) {
    const int ncol = m->nbhd == 4 ? 2 : 4;
    for (int k = 0; k < ncol; k++) orc_gibbs_colour_phase(m, x, g, beta, seed, chain, t, k, 0, m->H);
}

/* n Gibbs sweeps t = t0 .. t0+n-1; order 0 = the paper's column-major scan, 1 = colour
 * order.  Counts as orc_pca_run (x after sweep t for t >= burn_in).                    */
void orc_gibbs_run(const orc_model* m, uint8_t* x, const uint8_t* g, uint32_t* counts, int t0,
                   int n, double beta0, double beta_step, int period, uint64_t seed,
                   uint32_t chain, int burn_in, int order) {
    size_t N = (size_t)m->H * (size_t)m->W;
    for (int t = t0; t < t0 + n; t++) {
        double beta = orc_beta_at(beta0, beta_step, period, t);
        if (order == 1)
            orc_gibbs_sweep_coloured(m, x, g, beta, seed, chain, (uint32_t)t);
        else
            orc_gibbs_sweep(m, x, g, beta, seed, chain, (uint32_t)t);
        if (counts && burn_in >= 0 && t >= burn_in) {
            for (size_t i = 0; i < N; i++) counts[(size_t)x[i] * N + i] += 1;
        }
    }
}

/* MPM estimate (R15): label with the largest count, ties to the lowest label.   */
void orc_mpm(const uint32_t* counts, int levels, size_t N, uint8_t* out) {
    for (size_t i = 0; i < N; i++) {
        int best = 0;
        for (int k = 1; k < levels; k++)
            if (counts[(size_t)k * N + i] > counts[(size_t)best * N + i]) best = k;
        out[i] = (uint8_t)best;
    }
}

/* ------------------------------------------------------------------------- */
/* Metrics, PAPER.md:516-534 (section 6).  x = original (truth), y = restored.
 * MSE on luminances; PSNR = 20 log10(max x / sqrt(MSE)) with max x the maximum
 * luminance of the ORIGINAL (R17); global SSIM with population
 * moments and c1 = (0.01)^2, c2 = (0.03)^2 (R16).  Two-pass statistics.
 * Returns 0, or -1 if max x = 0 (PSNR undefined).  MSE = 0 gives PSNR = +inf.    */
int orc_metrics(const uint8_t* x, const uint8_t* y, size_t N, int levels, double* mse_out,
                double* psnr_out, double* ssim_out) {
    double sum_sq = 0.0, xmax = 0.0;
    for (size_t i = 0; i < N; i++) {
        double d = lum(x[i], levels) - lum(y[i], levels);
        sum_sq += d * d;
        if (lum(x[i], levels) > xmax) xmax = lum(x[i], levels);
    }
    double mse = sum_sq / (double)N;
    double mux = 0.0, muy = 0.0;
    for (size_t i = 0; i < N; i++) {
        mux += lum(x[i], levels);
        muy += lum(y[i], levels);
    }
    mux /= (double)N;
    muy /= (double)N;
    double vx = 0.0, vy = 0.0, cxy = 0.0;
    for (size_t i = 0; i < N; i++) {
        double dx = lum(x[i], levels) - mux, dy = lum(y[i], levels) - muy;
        vx += dx * dx;
        vy += dy * dy;
        cxy += dx * dy;
    }
    vx /= (double)N;
    vy /= (double)N;
    cxy /= (double)N;
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    double ssim = ((2.0 * mux * muy + c1) * (2.0 * cxy + c2)) /
                  ((mux * mux + muy * muy + c1) * (vx + vy + c2));
    if (mse_out) *mse_out = mse;
    if (ssim_out) *ssim_out = ssim;
    if (xmax == 0.0) {
        if (psnr_out) *psnr_out = NAN;
        return -1;
    }
    if (psnr_out) *psnr_out = (mse == 0.0) ? INFINITY : 20.0 * log10(xmax / sqrt(mse));
    return 0;
}

/* Windowed SSIM (secondary metric, R16): Wang et al. 2004 statistics over every
 * 7x7 window lying fully inside the image, uniform weights, sample (N-1)
 * covariance, c1 = 1e-4, c2 = 9e-4, averaged over windows.  H, W >= 7.           */
double orc_ssim_windowed(const uint8_t* x, const uint8_t* y, int H, int W, int levels) {
    const int win = 7;
    const double c1 = 0.01 * 0.01, c2 = 0.03 * 0.03;
    const double NP = (double)(win * win);
    double total = 0.0;
    long count = 0;
    for (int r0 = 0; r0 + win <= H; r0++) {
        for (int c0 = 0; c0 + win <= W; c0++) {
            double mx = 0.0, my = 0.0;
            for (int r = r0; r < r0 + win; r++)
                for (int c = c0; c < c0 + win; c++) {
                    mx += lum(x[r * W + c], levels);
                    my += lum(y[r * W + c], levels);
                }
            mx /= NP;
            my /= NP;
            double vx = 0.0, vy = 0.0, vxy = 0.0;
            for (int r = r0; r < r0 + win; r++)
                for (int c = c0; c < c0 + win; c++) {
                    double dx = lum(x[r * W + c], levels) - mx;
                    double dy = lum(y[r * W + c], levels) - my;
                    vx += dx * dx;
                    vy += dy * dy;
                    vxy += dx * dy;
                }
            vx /= (NP - 1.0);
            vy /= (NP - 1.0);
            vxy /= (NP - 1.0);
            total += ((2.0 * mx * my + c1) * (2.0 * vxy + c2)) /
                     ((mx * mx + my * my + c1) * (vx + vy + c2));
            count++;
        }
    }
    return total / (double)count;
}

/* ------------------------------------------------------------------------- */
/* Synthetic experiment inputs (section 6).                     */

/* Nearest gray level to a luminance in [0,1], ties to the lower level (R12).     */
int orc_quantize(double v, int levels) {
    int best = 0;
    double bd = fabs(v - lum(0, levels));
    for (int k = 1; k < levels; k++) {
        double d = fabs(v - lum(k, levels));
        if (d < bd) {
            bd = d;
            best = k;
        }
    }
    return best;
}

/* Standard normal for site (row, col) of chain: Box-Muller on u1 = (r0+1)*2^-32,
 * u2 = r1*2^-32, (r0, r1) = words 0, 1 of Philox(ctr = (col, row, 0, 3<<24|chain)).*/
double orc_gauss(uint64_t seed, uint32_t chain, uint32_t row, uint32_t col) {
    uint32_t ctr[4] = {col, row, 0u, (ORC_TAG_NOISE << 24) | chain};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    uint32_t out[4];
    orc_philox4x32_10(ctr, key, out);
    double u1 = ((double)out[0] + 1.0) * (1.0 / 4294967296.0);
    double u2 = (double)out[1] * (1.0 / 4294967296.0);
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* Degradation: add N(0, sigma^2) to each luminance, clamp to [0,1]
 * (R12), round to the nearest gray level (ties lower).                            */
void orc_degrade(const uint8_t* x, uint8_t* out, int H, int W, int levels, double sigma,
                 uint64_t seed, uint32_t chain) {
    for (int r = 0; r < H; r++) {
        for (int c = 0; c < W; c++) {
            double v = lum(x[r * W + c], levels) +
                       sigma * orc_gauss(seed, chain, (uint32_t)r, (uint32_t)c);
            if (v < 0.0) v = 0.0;
            if (v > 1.0) v = 1.0;
            out[r * W + c] = (uint8_t)orc_quantize(v, levels);
        }
    }
}

/* MRF ground truth: pixels drawn uniformly from the l levels
 * (tag GEN_INIT: label = floor(r*l/2^32)), then systematic Gibbs sweeps under the
 * PRIOR only (data term absent) with beta ramped linearly from beta_start to
 * beta_end over n sweeps ("We changed beta manually", R11).  Tag GEN_GIBBS.       */
void orc_generate_mrf(const orc_model* m, uint8_t* x, int n, double beta_start,
                      double beta_end, uint64_t seed, uint32_t chain) {
    for (int r = 0; r < m->H; r++)
        for (int c = 0; c < m->W; c++) {
            uint32_t rnd = orc_draw(seed, ORC_TAG_GEN_INIT, chain, 0u, (uint32_t)r, (uint32_t)c);
            x[r * m->W + c] = (uint8_t)(((uint64_t)rnd * (uint64_t)m->levels) >> 32);
        }
    double p[256];
    int cnt[256];
    for (int t = 0; t < n; t++) {
        double beta = (n > 1) ? beta_start + (beta_end - beta_start) * (double)t / (double)(n - 1)
                              : beta_start;
        double a = 2.0 * beta * m->J;
        for (int c = 0; c < m->W; c++) {
            for (int r = 0; r < m->H; r++) {
                neighbour_counts(m, x, r, c, cnt);
                double Emax = -INFINITY;
                for (int s = 0; s < m->levels; s++) {
                    p[s] = a * (double)cnt[s];
                    if (p[s] > Emax) Emax = p[s];
                }
                double Z = 0.0;
                for (int s = 0; s < m->levels; s++) {
                    p[s] = exp(p[s] - Emax);
                    Z += p[s];
                }
                for (int s = 0; s < m->levels; s++) p[s] /= Z;
                uint32_t rnd =
                    orc_draw(seed, ORC_TAG_GEN_GIBBS, chain, (uint32_t)t, (uint32_t)r, (uint32_t)c);
                double u = (double)rnd * (1.0 / 4294967296.0);
                x[r * m->W + c] = (uint8_t)orc_decide(p, m->levels, u, NULL);
            }
        }
    }
}
