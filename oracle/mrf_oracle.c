/*
 * mrf_oracle.c -- plain, slow, fp64 CPU oracle for the MRFMap hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA path (paper_2006_03512_b200/csrc) and is
 * written from PAPER.md and the readings listed in DESIGN.md ("Readings").
 *
 * Citations: P:n = /root/reference/PAPER.md line n; B1..B7 = the oracle steps
 * of SURVEY.md §8(c), restated in DESIGN.md.  Build:
 *     gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC  (no FMA contraction, so the
 *     fp64 ray setup rounds exactly as written, op by op)
 *
 * Functions and their pins (tests/test_oracle_*.py):
 *   orc_ray_setup   B1 pixel -> fixed-point segment        pinned: closed-form rays, round trip
 *   orc_dda         B2 fixed-point 3D-DDA (+B3 offsets)    pinned: exact rational brute force
 *   orc_log_nu      B3 bilinear LUT lookup                 pinned: bin centres / edge clamp
 *   orc_ray_messages B5 single-ray messages (Eq.13/14)     pinned: 2^N enumeration of Eq.12
 *   orc_ray_pass + orc_accumulate  B5 flooding iteration   pinned: exact marginals on trees
 *   orc_marginals   B6 (Eq.8)                              pinned: unseen voxel = prior
 *   orc_kf_*        NEXT #3 keyframe-average variant       pinned: SPEC worked examples, one ray
 *                                                          per (keyframe, voxel) = B5 iteration
 *   orc_alloc_bricks, orc_dda_sparse  NEXT #4 sparse bricks pinned: SPEC allocation examples, full
 *                                                          mask = dense walk, skipped cells = empty
 *   orc_patch_log_nu  NEXT #4 option: learnt per-patch noise, reading R25
 *                                                          pinned: scipy's Gaussian log-density; equal
 *                                                          patches = the global model's traversal
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Thread count of the OpenMP loops (bench.py times the oracle at 1 thread and at all cores;
 * no arithmetic depends on it: independent rays / voxels only). */
void orc_set_num_threads(int32_t n) { omp_set_num_threads(n > 0 ? n : 1); }
int32_t orc_max_threads(void) { return (int32_t)omp_get_max_threads(); }

#define FIX_ONE 65536LL /* 16 fractional bits of the fixed-point grid coordinates (B1) */

/* ------------------------------------------------------------------ B1: pixel -> segment */
/* par[9] = {z_lo, z_hi, off_lo, off_hi, margin_min, margin_k, c0, c1, c2}
 * geo[4] = {res, ox, oy, oz}.  Returns 0 = ray kept, 1 = invalid pixel, 2 = dropped
 * (measured point outside the grid, reading R11). */
int orc_ray_setup(const int32_t dims[3], const double geo[4], const double par[9],
                  const double K[4], const double Twc[12], int32_t u, int32_t v, float zf,
                  int64_t G0[3], int64_t G1[3], double* Z_out, double* L_out) {
    const double z = (double)zf;
    if (!isfinite(z) || !(z > 0.0)) return 1;
    const double xc = ((double)u - K[2]) / K[0];
    const double yc = ((double)v - K[3]) / K[1];
    const double rho = sqrt((xc * xc + yc * yc) + 1.0);
    const double Z = z * rho;                                 /* range along the ray */
    const double sZ = (par[6] + par[7] * Z) + (par[8] * Z) * Z; /* sigma(Z) */
    double m = par[5] * sZ;                                   /* 3 sigma beyond the depth */
    if (m < par[4]) m = par[4];
    const double L = Z + m;
    const double res = geo[0];
    for (int k = 0; k < 3; ++k) {
        const double Ck = Twc[4 * k + 3];
        const double Dk = (Twc[4 * k + 0] * xc + Twc[4 * k + 1] * yc) + Twc[4 * k + 2];
        const double pk = ((Ck + z * Dk) - geo[1 + k]) / res; /* measured point, grid units */
        if (pk < 0.0 || pk >= (double)dims[k]) return 2;
        const double Ek = Ck + (L / rho) * Dk;
        const double g0 = (Ck - geo[1 + k]) / res;
        const double g1 = (Ek - geo[1 + k]) / res;
        G0[k] = llrint(g0 * 65536.0); /* round half to even (default rounding mode) */
        G1[k] = llrint(g1 * 65536.0);
    }
    *Z_out = Z;
    *L_out = L;
    return 0;
}

/* The learnt per-patch model (NEXT #4 option, reading R25): the sigma polynomial of the pixel's
 * 20x20 patch replaces par[6..8] (c0, c1, c2) -- the traversal margin 3 sigma(Z) of P:205 and the
 * allocation radius then follow the pixel's own noise.  pix_sigma: [H*W][3] or NULL. */
static void pixel_par(const double par[9], const double* pix_sigma, int64_t p, double out[9]) {
    for (int k = 0; k < 9; ++k) out[k] = par[k];
    if (pix_sigma) {
        out[6] = pix_sigma[3 * p];
        out[7] = pix_sigma[3 * p + 1];
        out[8] = pix_sigma[3 * p + 2];
    }
}

/* ------------------------------------------------------------------ B2 + B3: fixed-point DDA */
static int64_t floor_div(int64_t a, int64_t b) { /* b > 0 */
    int64_t q = a / b;
    if ((a % b) != 0 && a < 0) q -= 1;
    return q;
}

/* Walk the segment G0 -> G1 (grid units x 65536) and emit, in order, every cell whose
 * intersection with the segment has positive length ("standard 3DDA",
 * Amanatides-Woo; tie rule of reading R13).  For each emitted cell: vid = x + nx(y + ny z),
 * and off_q = clamp(llrint((0.5 (t_in + t_out) L - Z) * 32768), +-32767) (B3, reading R6).
 * Pointers may be NULL (count only).  Returns the number of cells (all of them, even
 * beyond cap; only the first cap are written). */
/* Brick allocation mask (NEXT #4, reading R23): NULL = dense grid; else a cell is part of the map
 * iff mask[brick of the cell] != 0, bricks B^3 cells, brick index bx + nb[0] (by + nb[1] bz). */
typedef struct {
    const uint8_t* mask;
    int32_t B;
    int32_t nb[3];
} BrickMask;

static int cell_allocated(const BrickMask* bm, const int64_t c[3]) {
    if (!bm || !bm->mask) return 1;
    const int64_t b = c[0] / bm->B + (int64_t)bm->nb[0] * (c[1] / bm->B + (int64_t)bm->nb[1] * (c[2] / bm->B));
    return bm->mask[b] != 0;
}

static int64_t dda_core(const int32_t dims[3], const int64_t G0[3], const int64_t G1[3], double Z, double L,
                        const BrickMask* bm, int32_t* vid, int16_t* off_q, double* t_in_out, double* t_out_out,
                        int64_t cap);

int64_t orc_dda(const int32_t dims[3], const int64_t G0[3], const int64_t G1[3], double Z, double L,
                int32_t* vid, int16_t* off_q, double* t_in_out, double* t_out_out, int64_t cap) {
    return dda_core(dims, G0, G1, Z, L, NULL, vid, off_q, t_in_out, t_out_out, cap);
}

/* The B2 walk with empty skip (SPEC traverse_3dda over a brick-sparse grid, reading R23): cells of
 * unallocated bricks are walked through but not emitted (they are not part of the map, so they
 * are not variables of the ray's factor).  Emitted cells keep their own t_in / t_out. */
int64_t orc_dda_sparse(const int32_t dims[3], const int64_t G0[3], const int64_t G1[3], double Z, double L,
                       const uint8_t* mask, int32_t B, const int32_t nb[3], int32_t* vid, int16_t* off_q,
                       double* t_in_out, double* t_out_out, int64_t cap) {
    const BrickMask bm = {mask, B, {nb[0], nb[1], nb[2]}};
    return dda_core(dims, G0, G1, Z, L, &bm, vid, off_q, t_in_out, t_out_out, cap);
}

static int64_t dda_core(const int32_t dims[3], const int64_t G0[3], const int64_t G1[3], double Z, double L,
                        const BrickMask* bm, int32_t* vid, int16_t* off_q, double* t_in_out, double* t_out_out,
                        int64_t cap) {
    int64_t c[3], num[3], den[3];
    int step[3];
    for (int k = 0; k < 3; ++k) {
        const int64_t dG = G1[k] - G0[k];
        c[k] = floor_div(G0[k], FIX_ONE);
        if (dG < 0 && G0[k] == c[k] * FIX_ONE) c[k] -= 1; /* cell containing t = 0+ */
        if (dG > 0) {
            step[k] = 1;
            num[k] = (c[k] + 1) * FIX_ONE - G0[k];
            den[k] = dG;
        } else if (dG < 0) {
            step[k] = -1;
            num[k] = G0[k] - c[k] * FIX_ONE;
            den[k] = -dG;
        } else {
            step[k] = 0;
            num[k] = 0;
            den[k] = 1;
        }
    }
    int64_t n = 0;
    double t_in = 0.0;
    for (;;) {
        int inside = 1;
        for (int k = 0; k < 3; ++k)
            if (c[k] < 0 || c[k] >= dims[k]) inside = 0;
        if (!inside) break; /* grid exit */
        /* smallest next crossing, by exact cross-multiplication */
        int amin = -1;
        for (int k = 0; k < 3; ++k) {
            if (step[k] == 0) continue;
            if (amin < 0 || num[k] * den[amin] < num[amin] * den[k]) amin = k;
        }
        const int last = (amin < 0) || (num[amin] >= den[amin]);
        const double t_out = last ? 1.0 : (double)num[amin] / (double)den[amin];
        const int emit = cell_allocated(bm, c);
        if (emit && n < cap) {
            if (vid) vid[n] = (int32_t)(c[0] + (int64_t)dims[0] * (c[1] + (int64_t)dims[1] * c[2]));
            if (off_q) {
                const double d_mid = (0.5 * (t_in + t_out)) * L;
                const double delta = d_mid - Z;
                long long q = llrint(delta * 32768.0);
                if (q > 32767) q = 32767;
                if (q < -32767) q = -32767;
                off_q[n] = (int16_t)q;
            }
            if (t_in_out) t_in_out[n] = t_in;
            if (t_out_out) t_out_out[n] = t_out;
        }
        if (emit) ++n;
        if (last) break;
        const int64_t na = num[amin], da = den[amin];
        for (int k = 0; k < 3; ++k) { /* step every axis tied at t_min, simultaneously */
            if (step[k] == 0) continue;
            if (num[k] * da == na * den[k]) {
                c[k] += step[k];
                num[k] += FIX_ONE;
            }
        }
        t_in = t_out;
    }
    return n;
}

/* ------------------------------------------------------------------ B3: log nu lookup */
/* Bilinear interpolation of log nu at (Z, off_q / 32768) over bin centres, with the
 * coordinates clamped to the edge centres (reading R6/R9). */
double orc_log_nu(const float* lut, int32_t n_z, int32_t n_off, const double par[9], double Z,
                  int32_t off_q) {
    const double off = (double)off_q / 32768.0;
    double fz = (Z - par[0]) / (par[1] - par[0]) * (double)n_z - 0.5;
    double fo = (off - par[2]) / (par[3] - par[2]) * (double)n_off - 0.5;
    if (fz < 0.0) fz = 0.0;
    if (fz > (double)(n_z - 1)) fz = (double)(n_z - 1);
    if (fo < 0.0) fo = 0.0;
    if (fo > (double)(n_off - 1)) fo = (double)(n_off - 1);
    int iz = (int)floor(fz), io = (int)floor(fo);
    if (iz > n_z - 2) iz = n_z - 2;
    if (io > n_off - 2) io = n_off - 2;
    const double wz = fz - iz, wo = fo - io;
    const double a = lut[(int64_t)iz * n_off + io], b = lut[(int64_t)iz * n_off + io + 1];
    const double cc = lut[(int64_t)(iz + 1) * n_off + io], d = lut[(int64_t)(iz + 1) * n_off + io + 1];
    return (1.0 - wz) * ((1.0 - wo) * a + wo * b) + wz * ((1.0 - wo) * cc + wo * d);
}

/* ------------------------------------------------------------------ B5: one ray */
/* Learnt per-patch forward model (NEXT #4 option, reading R25; "we first utilise the
 * sensor bias to predict what the mean sensor measurement would be and then evaluate the
 * probability of a given measurement originating from this predicted measurement and distributed
 * using the learnt noise value"; 2nd-degree polynomials per pixel region):
 *   log nu(Z | d) = log N(Z; d + b(d), s(d)),  b(d) = (b0 + b1 d) + b2 d^2,
 *   s(d) = max((s0 + s1 d) + s2 d^2, sigma_min),
 * at the voxel depth d = Z + off_q / 32768 (B3's quantised span midpoint), with the coefficients
 * of the ray's patch (coef[r][6] = b0, b1, b2, s0, s1, s2).  Out: lnu[e] for every incidence. */
void orc_patch_log_nu(int64_t n_rays, const int64_t* row_ptr, const int16_t* off_q, const double* Z_ray,
                      const double* coef, double sigma_min, double* lnu) {
    const double half_log_2pi = 0.5 * log(2.0 * 3.14159265358979323846);
    for (int64_t r = 0; r < n_rays; ++r) {
        const double* k = coef + 6 * r;
        const double Z = Z_ray[r];
        for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
            const double d = Z + (double)off_q[e] / 32768.0;
            const double b = (k[0] + k[1] * d) + k[2] * d * d;
            double s = (k[3] + k[4] * d) + k[5] * d * d;
            if (s < sigma_min) s = sigma_min;
            const double t = (Z - (d + b)) / s;
            lnu[e] = -0.5 * t * t - log(s) - half_log_2pi;
        }
    }
}

static double softplus(double x) { return x > 0.0 ? x + log1p(exp(-x)) : log1p(exp(x)); }

static double lse(double a, double b) {
    if (a == -INFINITY) return b;
    if (b == -INFINITY) return a;
    const double m = a > b ? a : b;
    return m + log1p(exp(-fabs(a - b)));
}

/* Factor->occupancy messages of one ray, in the log domain.
 * Input: cavity log-odds c[i] (voxel->factor message, Eq.6) and log nu[i].
 * Output: lpos[i] = log mu_{psi->o_i}(1) (Eq.13) and
 *         lneg[i] = log mu_{psi->o_i}(0) (Eq.14 in the division-free form of P:524),
 * both relative to the normalised incoming messages mu(o_k) = sigma(+-c_k).
 *   lV_i = sum_{k<i} log mu(o_k=0)                          (prod_{k<i} mu(o_k=0))
 *   lP_i = lse_{j<i} [log mu(o_j=1) + log nu_j + lV_j]      (first sums of Eq.13/14)
 *   lR_i = lse_{j>i} [log mu(o_j=1) + log nu_j + sum_{i<k<j} log mu(o_k=0)]
 *        (suffix recurrence lR_{i-1} = lse(lb_i + lnu_i, la_i + lR_i); V_i R_i is the
 *         second term of P:524)
 *   lpos_i = lse(lP_i, lV_i + lnu_i),  lneg_i = lse(lP_i, lV_i + lR_i). */
void orc_ray_messages(int64_t N, const double* c, const double* lnu, double* lpos, double* lneg,
                      double* work /* 5N doubles */) {
    double* la = work;
    double* lb = work + N;
    double* lV = work + 2 * N;
    double* lP = work + 3 * N;
    double* lR = work + 4 * N;
    for (int64_t i = 0; i < N; ++i) {
        la[i] = -softplus(c[i]);  /* log sigma(-c) = log mu(o_i = 0) */
        lb[i] = -softplus(-c[i]); /* log sigma(+c) = log mu(o_i = 1) */
    }
    if (N == 0) return;
    lV[0] = 0.0;
    lP[0] = -INFINITY;
    for (int64_t i = 0; i + 1 < N; ++i) {
        lV[i + 1] = lV[i] + la[i];
        lP[i + 1] = lse(lP[i], lb[i] + lnu[i] + lV[i]);
    }
    lR[N - 1] = -INFINITY;
    for (int64_t i = N - 1; i >= 1; --i) lR[i - 1] = lse(lb[i] + lnu[i], la[i] + lR[i]);
    for (int64_t i = 0; i < N; ++i) {
        lpos[i] = lse(lP[i], lV[i] + lnu[i]);
        lneg[i] = lse(lP[i], lV[i] + lR[i]);
    }
}

static double clip256(double x) {
    if (!(x < 256.0)) return 256.0; /* also lneg = -inf (N = 1) */
    if (x < -256.0) return -256.0;
    return x;
}

/* One flooding pass over all rays from the same snapshot T (reading R4):
 * c_e = L0 + T[v_e] - lambda_e (Eq.6 excluding the ray's own message),
 * lambda_e <- clip(lpos - lneg, +-256) (reading R9).  lambda is updated in place (each
 * ray reads only its own old messages).  Z_ray[r] is the ray's measured range. */
void orc_ray_pass(int64_t n_rays, const int64_t* row_ptr, const int32_t* vid, const int16_t* off_q,
                  const double* Z_ray, const float* lut, int32_t n_z, int32_t n_off, const double par[9],
                  double L0, const double* T, double* lambda, const double* lnu_e) {
#pragma omp parallel
    {
        int64_t cap = 0;
        double* buf = NULL;
#pragma omp for schedule(dynamic, 64)
        for (int64_t r = 0; r < n_rays; ++r) {
            const int64_t e0 = row_ptr[r], N = row_ptr[r + 1] - e0;
            if (N <= 0) continue;
            if (N > cap) {
                free(buf);
                cap = N * 2;
                buf = (double*)malloc(sizeof(double) * 9 * cap);
            }
            double* c = buf;
            double* lnu = buf + N;
            double* lpos = buf + 2 * N;
            double* lneg = buf + 3 * N;
            double* work = buf + 4 * N;
            for (int64_t i = 0; i < N; ++i) {
                c[i] = L0 + T[vid[e0 + i]] - lambda[e0 + i];
                lnu[i] = lnu_e ? lnu_e[e0 + i] : orc_log_nu(lut, n_z, n_off, par, Z_ray[r], off_q[e0 + i]);
            }
            orc_ray_messages(N, c, lnu, lpos, lneg, work);
            for (int64_t i = 0; i < N; ++i) lambda[e0 + i] = clip256(lpos[i] - lneg[i]);
        }
        free(buf);
    }
}

/* T_v = sum_e lambda_e over the incidences of v, fp64 in incidence order (B5: "any fixed
 * order"); T is zeroed first.  This is the incoming-belief accumulation of P:200. */
void orc_accumulate(int64_t E, const int32_t* vid, const double* lambda, int64_t V, double* T) {
    memset(T, 0, sizeof(double) * (size_t)V);
    for (int64_t e = 0; e < E; ++e) T[vid[e]] += lambda[e];
}

/* n flooding iterations (B7) starting from lambda (in/out); T returned for the final lambda. */
void orc_bp(int64_t n_rays, const int64_t* row_ptr, const int32_t* vid, const int16_t* off_q,
            const double* Z_ray, const float* lut, int32_t n_z, int32_t n_off, const double par[9],
            double L0, int64_t V, int32_t n_iter, double* lambda, double* T, const double* lnu_e) {
    const int64_t E = row_ptr[n_rays];
    orc_accumulate(E, vid, lambda, V, T);
    for (int32_t it = 0; it < n_iter; ++it) {
        orc_ray_pass(n_rays, row_ptr, vid, off_q, Z_ray, lut, n_z, n_off, par, L0, T, lambda, lnu_e);
        orc_accumulate(E, vid, lambda, V, T);
    }
}

/* B6: p_v = sigma(L0 + T_v) (Eq.8); an unobserved voxel (T_v = 0) gives gamma. */
void orc_marginals(int64_t V, double L0, const double* T, double* p) {
    for (int64_t v = 0; v < V; ++v) p[v] = 1.0 / (1.0 + exp(-(L0 + T[v])));
}

/* ------------------------------------------------------------------ NEXT #3: keyframe averages
 * The paper's memory-saving variant: "we make an assumption that all rays going through
 * a voxel from a single keyframe send the same average message.  Thus, for each new keyframe
 * image we create an auxiliary buffer that stores the average outgoing message."  Restated with
 * SPEC's KeyframeBuffer / accumulate_outgoing / incoming_product (reading R22 in DESIGN.md):
 *   lbar[f][v]  log-odds of keyframe f's average message into voxel v; 0 (the uniform pair) when
 *               no ray of f reaches v ("zero accumulations -> uniform");
 *   T_v         = sum_f lbar[f][v]  (Eq.6 / Eq.8 with one message per keyframe);
 *   pass        every ray r of keyframe f from the same snapshot (flooding, reading R4):
 *               c_i = L0 + T[v_i] - lbar[f][v_i]  (incoming_product excluding the ray's whole
 *               keyframe), messages by B5, lambda_e = clip(lpos - lneg, +-256);
 *   average     mu1 = mean of sigma(lambda_e), mu0 = mean of sigma(-lambda_e) over the keyframe's
 *               incidences of v (arithmetic mean of the normalised pairs), and
 *               lbar[f][v] = clip(log(mu1 / mu0), +-256). */
static double sigmoid(double x) { return x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x)); }

/* T_v = sum over keyframes of lbar[f][v] (F*V, keyframe-major) */
void orc_kf_beliefs(int64_t F, int64_t V, const double* lbar, double* T) {
    memset(T, 0, sizeof(double) * (size_t)V);
    for (int64_t f = 0; f < F; ++f)
        for (int64_t v = 0; v < V; ++v) T[v] += lbar[f * V + v];
}

/* accumulate_outgoing + average: lbar[f][v] from the per-incidence messages of every ray;
 * frame[r] is the keyframe of ray r.  Pairs without a ray keep lbar = 0. */
void orc_kf_average(int64_t n_rays, const int64_t* row_ptr, const int32_t* vid, const int32_t* frame,
                    const double* lambda, int64_t F, int64_t V, double* lbar) {
    double* s1 = (double*)calloc((size_t)(F * V), sizeof(double));
    double* s0 = (double*)calloc((size_t)(F * V), sizeof(double));
    for (int64_t r = 0; r < n_rays; ++r)
        for (int64_t e = row_ptr[r]; e < row_ptr[r + 1]; ++e) {
            const int64_t k = (int64_t)frame[r] * V + vid[e];
            s1[k] += sigmoid(lambda[e]);  /* mu_{psi->o}(1) of the normalised pair */
            s0[k] += sigmoid(-lambda[e]); /* mu_{psi->o}(0) */
        }
    for (int64_t k = 0; k < F * V; ++k) lbar[k] = (s1[k] + s0[k] > 0.0) ? clip256(log(s1[k] / s0[k])) : 0.0;
    free(s1);
    free(s0);
}

/* One flooding pass of the variant: lambda (per incidence, out) from the snapshot lbar. */
void orc_kf_pass(int64_t n_rays, const int64_t* row_ptr, const int32_t* vid, const int16_t* off_q,
                 const double* Z_ray, const int32_t* frame, const float* lut, int32_t n_z, int32_t n_off,
                 const double par[9], double L0, int64_t F, int64_t V, const double* lbar, double* lambda,
                 const double* lnu_e) {
    double* T = (double*)malloc(sizeof(double) * (size_t)V);
    orc_kf_beliefs(F, V, lbar, T);
#pragma omp parallel
    {
        int64_t cap = 0;
        double* buf = NULL;
#pragma omp for schedule(dynamic, 64)
        for (int64_t r = 0; r < n_rays; ++r) {
            const int64_t e0 = row_ptr[r], N = row_ptr[r + 1] - e0;
            if (N <= 0) continue;
            if (N > cap) {
                free(buf);
                cap = N * 2;
                buf = (double*)malloc(sizeof(double) * 9 * cap);
            }
            double* c = buf;
            double* lnu = buf + N;
            double* lpos = buf + 2 * N;
            double* lneg = buf + 3 * N;
            double* work = buf + 4 * N;
            const double* lb = lbar + (int64_t)frame[r] * V;
            for (int64_t i = 0; i < N; ++i) {
                c[i] = L0 + T[vid[e0 + i]] - lb[vid[e0 + i]];
                lnu[i] = lnu_e ? lnu_e[e0 + i] : orc_log_nu(lut, n_z, n_off, par, Z_ray[r], off_q[e0 + i]);
            }
            orc_ray_messages(N, c, lnu, lpos, lneg, work);
            for (int64_t i = 0; i < N; ++i) lambda[e0 + i] = clip256(lpos[i] - lneg[i]);
        }
        free(buf);
    }
    free(T);
}

/* n iterations of the variant from lbar (in/out; zeros = B4); lambda out; T = sum_f lbar. */
void orc_kf_bp(int64_t n_rays, const int64_t* row_ptr, const int32_t* vid, const int16_t* off_q,
               const double* Z_ray, const int32_t* frame, const float* lut, int32_t n_z, int32_t n_off,
               const double par[9], double L0, int64_t F, int64_t V, int32_t n_iter, double* lambda,
               double* lbar, double* T, const double* lnu_e) {
    for (int32_t it = 0; it < n_iter; ++it) {
        orc_kf_pass(n_rays, row_ptr, vid, off_q, Z_ray, frame, lut, n_z, n_off, par, L0, F, V, lbar, lambda, lnu_e);
        orc_kf_average(n_rays, row_ptr, vid, frame, lambda, F, V, lbar);
    }
    orc_kf_beliefs(F, V, lbar, T);
}

/* ------------------------------------------------------------------ NEXT #4: brick allocation
 * SPEC allocate_for_depth_image ("new bricks are allocated in a region around the
 * reprojected 3D depth point cloud"; reading R23): for every pixel of the frame with a valid depth
 * whose measured point p (grid units, B1) lies inside the grid, with r = margin_k sigma(Z) / res
 * (the 3 sigma of P:205, in voxels), every brick containing a cell of the box
 * [floor(p - r), floor(p + r)] (clamped to the grid) is allocated.  That box contains every cell
 * within distance r of p, so "every voxel within r_alloc of a reprojected point belongs to an
 * allocated brick" holds.  All pixels count, whatever their rank (the map is global).  Returns
 * the number of newly allocated bricks. */
int64_t orc_alloc_bricks(const int32_t dims[3], const double geo[4], const double par_in[9], const double K[4],
                         const double Twc[12], int32_t W, int32_t H, const float* depth, int32_t B,
                         const int32_t nb[3], uint8_t* mask, const double* pix_sigma) {
    int64_t added = 0;
    for (int32_t v = 0; v < H; ++v)
        for (int32_t u = 0; u < W; ++u) {
            double par[9];
            pixel_par(par_in, pix_sigma, (int64_t)v * W + u, par);
            const double z = (double)depth[(int64_t)v * W + u];
            if (!isfinite(z) || !(z > 0.0)) continue;
            const double xc = ((double)u - K[2]) / K[0];
            const double yc = ((double)v - K[3]) / K[1];
            const double rho = sqrt((xc * xc + yc * yc) + 1.0);
            const double Z = z * rho;
            const double sZ = (par[6] + par[7] * Z) + (par[8] * Z) * Z;
            const double r = (par[5] * sZ) / geo[0];
            int64_t lo[3], hi[3];
            int inside = 1;
            for (int k = 0; k < 3; ++k) {
                const double Dk = (Twc[4 * k + 0] * xc + Twc[4 * k + 1] * yc) + Twc[4 * k + 2];
                const double pk = ((Twc[4 * k + 3] + z * Dk) - geo[1 + k]) / geo[0];
                if (pk < 0.0 || pk >= (double)dims[k]) inside = 0;
                lo[k] = (int64_t)floor(pk - r);
                hi[k] = (int64_t)floor(pk + r);
                if (lo[k] < 0) lo[k] = 0;
                if (hi[k] > dims[k] - 1) hi[k] = dims[k] - 1;
            }
            if (!inside) continue;
            for (int64_t bz = lo[2] / B; bz <= hi[2] / B; ++bz)
                for (int64_t by = lo[1] / B; by <= hi[1] / B; ++by)
                    for (int64_t bx = lo[0] / B; bx <= hi[0] / B; ++bx) {
                        uint8_t* m = mask + bx + (int64_t)nb[0] * (by + (int64_t)nb[1] * bz);
                        if (!*m) {
                            *m = 1;
                            ++added;
                        }
                    }
        }
    return added;
}

/* ------------------------------------------------------------------ frames -> CSR */
/* Pass 1 over one frame: per pixel status (0 kept, 1 invalid, 2 dropped), cell count and
 * range Z.  Only rows with v % world == rank are visited (others get status 3). */
void orc_frame_count(const int32_t dims[3], const double geo[4], const double par_in[9], const double K[4],
                     const double Twc[12], int32_t W, int32_t H, const float* depth, int32_t rank,
                     int32_t world, int8_t* status, int64_t* count, double* Z_out, double* L_out,
                     const uint8_t* mask, int32_t B, const int32_t* nb, const double* pix_sigma) {
    const BrickMask bm = {mask, B, {nb ? nb[0] : 0, nb ? nb[1] : 0, nb ? nb[2] : 0}};
#pragma omp parallel for schedule(dynamic, 4)
    for (int32_t v = 0; v < H; ++v) {
        for (int32_t u = 0; u < W; ++u) {
            const int64_t p = (int64_t)v * W + u;
            count[p] = 0;
            Z_out[p] = 0.0;
            L_out[p] = 0.0;
            if (v % world != rank) {
                status[p] = 3;
                continue;
            }
            int64_t G0[3], G1[3];
            double Z = 0.0, L = 0.0, par[9];
            pixel_par(par_in, pix_sigma, p, par);
            const int s = orc_ray_setup(dims, geo, par, K, Twc, u, v, depth[p], G0, G1, &Z, &L);
            status[p] = (int8_t)s;
            if (s != 0) continue;
            Z_out[p] = Z;
            L_out[p] = L;
            count[p] = dda_core(dims, G0, G1, Z, L, &bm, NULL, NULL, NULL, NULL, 0);
        }
    }
}

/* Pass 2: write vid/off_q of every kept pixel at offset[p] (offset < 0: skip). */
void orc_frame_fill(const int32_t dims[3], const double geo[4], const double par_in[9], const double K[4],
                    const double Twc[12], int32_t W, int32_t H, const float* depth, const int64_t* offset,
                    int32_t* vid, int16_t* off_q, const uint8_t* mask, int32_t B, const int32_t* nb,
                    const double* pix_sigma) {
    const BrickMask bm = {mask, B, {nb ? nb[0] : 0, nb ? nb[1] : 0, nb ? nb[2] : 0}};
#pragma omp parallel for schedule(dynamic, 4)
    for (int32_t v = 0; v < H; ++v) {
        for (int32_t u = 0; u < W; ++u) {
            const int64_t p = (int64_t)v * W + u;
            if (offset[p] < 0) continue;
            int64_t G0[3], G1[3];
            double Z = 0.0, L = 0.0, par[9];
            pixel_par(par_in, pix_sigma, p, par);
            if (orc_ray_setup(dims, geo, par, K, Twc, u, v, depth[p], G0, G1, &Z, &L) != 0) continue;
            dda_core(dims, G0, G1, Z, L, &bm, vid + offset[p], off_q + offset[p], NULL, NULL, INT64_MAX);
        }
    }
}

/* ------------------------------------------------------------------ §III.D evaluation metric
 * Generating-surface accuracy of a probabilistic map (applied per pixel in §V
 * P:240).  Readings (R18-R21):
 *   R18 occlusion density of voxel i with occupancy p_i: alpha_i = -ln(1 - p_i) / res, so a
 *       full-side crossing multiplies the visibility by (1 - p_i);
 *   R19 the evaluation ray runs from the camera to the map boundary (s_inf): the segment
 *       C -> C + 1.5 D d (D = grid diagonal, d the unit ray), walked by the same B2 DDA;
 *   R20 omega(s) = alpha(s) vis(s) decreases inside a constant-alpha step, so its maximum over
 *       a step is at the step entry and s* = entry of argmax_i alpha_i vis_i (first on ties);
 *   R21 classification: vis_inf > thr (0.5, "not reduced sufficiently") -> accurate iff
 *       Z > s_inf; else, mode 0 (sigma band, §V): accurate iff |Z - s*| <= k sigma(Z)
 *       (k = 1.5), sigma the map's noise model sigma(Z) = c0 + c1 Z + c2 Z^2; mode 1 (voxel
 *       bounds, §III.D): accurate iff Z lies in [entry, exit] of the argmax voxel.
 *
 * Per step i with occupancy log-odds x_i (p_i = sigma(x_i)) and length ell_i (m):
 *   ln vis_0 = 0,  ln vis_{i+1} = ln vis_i + (ell_i / res) ln(1 - p_i) = ln vis_i - (ell_i/res) softplus(x_i)
 *   ln omega_i = ln(alpha_i) + ln vis_i = ln(softplus(x_i) / res) + ln vis_i      (Eq.17-18)
 *   Omega_i = vis_i - vis_{i+1}                                                   (Eq.16)
 * orc_vis_profile writes ln vis[0..n] and ln omega[0..n-1] and returns argmax_i ln omega_i
 * (-1 if every p_i = 0). */
int64_t orc_vis_profile(int64_t n, const double* x, const double* ell, double res, double* lvis,
                        double* lomega) {
    lvis[0] = 0.0;
    int64_t best = -1;
    double bw = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        const double sp = softplus(x[i]); /* -ln(1 - p_i) */
        lomega[i] = (sp > 0.0 ? log(sp / res) : -INFINITY) + lvis[i];
        if (lomega[i] > bw) {
            bw = lomega[i];
            best = i;
        }
        lvis[i + 1] = lvis[i] - (ell[i] / res) * sp;
    }
    return best;
}

/* Evaluate one pixel against the map given by its occupancy log-odds xmap[V] (x = L0 + T_v).
 * Returns -1 for an invalid pixel (z not finite or <= 0), else 1 accurate / 0 inaccurate;
 * out[0..3] = {Z, s*, s_inf, vis_inf} (s* = -1 if no step occludes). */
int orc_eval_pixel(const int32_t dims[3], const double geo[4], const double par[9], const double K[4],
                   const double Twc[12], int32_t u, int32_t v, float zf, const double* xmap, double k_sigma,
                   double vis_thr, int32_t mode, double out[4]) {
    const double z = (double)zf;
    if (!isfinite(z) || !(z > 0.0)) return -1;
    const double res = geo[0];
    const double xc = ((double)u - K[2]) / K[0];
    const double yc = ((double)v - K[3]) / K[1];
    const double rho = sqrt((xc * xc + yc * yc) + 1.0);
    const double Z = z * rho;
    const double D = res * sqrt((double)dims[0] * dims[0] + (double)dims[1] * dims[1] + (double)dims[2] * dims[2]);
    const double Lev = 1.5 * D; /* R19: beyond the map boundary from any camera inside it */
    int64_t G0[3], G1[3];
    for (int k = 0; k < 3; ++k) {
        const double Ck = Twc[4 * k + 3];
        const double Dk = (Twc[4 * k + 0] * xc + Twc[4 * k + 1] * yc) + Twc[4 * k + 2];
        const double Ek = Ck + (Lev / rho) * Dk;
        G0[k] = llrint(((Ck - geo[1 + k]) / res) * 65536.0);
        G1[k] = llrint(((Ek - geo[1 + k]) / res) * 65536.0);
    }
    const int64_t n = orc_dda(dims, G0, G1, 0.0, 1.0, NULL, NULL, NULL, NULL, 0);
    int32_t* vid = (int32_t*)malloc(sizeof(int32_t) * (n > 0 ? n : 1));
    double* tin = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    double* tout = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    double* x = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    double* ell = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    double* lvis = (double*)malloc(sizeof(double) * (n + 1));
    double* lom = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    orc_dda(dims, G0, G1, 0.0, 1.0, vid, NULL, tin, tout, n);
    for (int64_t i = 0; i < n; ++i) {
        x[i] = xmap[vid[i]];
        ell[i] = (tout[i] - tin[i]) * Lev;
    }
    const int64_t best = orc_vis_profile(n, x, ell, res, lvis, lom);
    const double s_inf = n > 0 ? tout[n - 1] * Lev : 0.0;
    const double vis_inf = exp(lvis[n]);
    const double s_star = best >= 0 ? tin[best] * Lev : -1.0;
    const double s_star_out = best >= 0 ? tout[best] * Lev : -1.0;
    const double sigma = (par[6] + par[7] * Z) + (par[8] * Z) * Z;
    int acc;
    if (vis_inf > vis_thr)
        acc = Z > s_inf;
    else if (mode == 0)
        acc = fabs(Z - s_star) <= k_sigma * sigma;
    else
        acc = Z >= s_star && Z <= s_star_out;
    out[0] = Z;
    out[1] = s_star;
    out[2] = s_inf;
    out[3] = vis_inf;
    free(vid); free(tin); free(tout); free(x); free(ell); free(lvis); free(lom);
    return acc;
}

/* All pixels of one frame (rows v % world == rank; others -2).  cls[H*W]; returns
 * n_valid, n_accurate through the pointers. */
void orc_eval_frame(const int32_t dims[3], const double geo[4], const double par_in[9], const double K[4],
                    const double Twc[12], int32_t W, int32_t H, const float* depth, const double* xmap,
                    double k_sigma, double vis_thr, int32_t mode, int32_t rank, int32_t world, int8_t* cls,
                    int64_t* n_valid, int64_t* n_acc, const double* pix_sigma) {
    int64_t nv = 0, na = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : nv, na)
    for (int64_t i = 0; i < (int64_t)W * H; ++i) {
        const int32_t v = (int32_t)(i / W), u = (int32_t)(i % W);
        if (v % world != rank) {
            cls[i] = -2;
            continue;
        }
        double out[4], par[9];
        pixel_par(par_in, pix_sigma, i, par);
        const int r = orc_eval_pixel(dims, geo, par, K, Twc, u, v, depth[i], xmap, k_sigma, vis_thr, mode, out);
        cls[i] = (int8_t)r;
        if (r >= 0) {
            nv += 1;
            na += r;
        }
    }
    *n_valid = nv;
    *n_acc = na;
}
