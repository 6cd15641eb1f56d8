/* Exact fp64 depth renderer for the seeded synthetic scenes (input generation only;
 * no MRFMap arithmetic lives here).  Built by synth/_native.py with
 *   gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC
 * Ray of pixel (u,v): C + t * R (x_c, y_c, 1), x_c = (u-cx)/fx, y_c = (v-cy)/fy;
 * the nearest positive t is the camera z-depth (INFINITY = no hit).
 */
#include <math.h>
#include <stdint.h>

static double hit_aabb(const double C[3], const double D[3], const double lo[3], const double hi[3]) {
    double tn = -INFINITY, tf = INFINITY;
    for (int a = 0; a < 3; ++a) {
        if (D[a] == 0.0) {
            if (C[a] < lo[a] || C[a] > hi[a]) return INFINITY;
            continue;
        }
        double t1 = (lo[a] - C[a]) / D[a];
        double t2 = (hi[a] - C[a]) / D[a];
        double mn = t1 < t2 ? t1 : t2, mx = t1 < t2 ? t2 : t1;
        if (mn > tn) tn = mn;
        if (mx < tf) tf = mx;
    }
    if (tf >= tn && tf > 0.0 && tn > 0.0) return tn;
    return INFINITY;
}

/* rects: n_rect x 6 {axis, coord, lo0, lo1, hi0, hi1}; boxes: n_box x 6 {lo3, hi3};
 * obbs: n_obb x 7 {centre3, half3, yaw}.  out: H*W doubles (row-major v*W+u). */
void synth_render(int32_t W, int32_t H, const double K[4], const double R[9], const double C[3],
                  int32_t n_rect, const double* rects, int32_t n_box, const double* boxes,
                  int32_t n_obb, const double* obbs, double* out) {
    const double fx = K[0], fy = K[1], cx = K[2], cy = K[3];
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < (int64_t)W * H; ++p) {
        const int u = (int)(p % W), v = (int)(p / W);
        const double xc = ((double)u - cx) / fx, yc = ((double)v - cy) / fy;
        double D[3];
        for (int k = 0; k < 3; ++k) D[k] = (R[3 * k + 0] * xc + R[3 * k + 1] * yc) + R[3 * k + 2];
        double best = INFINITY;
        for (int i = 0; i < n_rect; ++i) {
            const double* r = rects + 6 * i;
            const int ax = (int)r[0];
            if (D[ax] == 0.0) continue;
            const int o0 = ax == 0 ? 1 : 0, o1 = ax == 2 ? 1 : 2;
            const double t = (r[1] - C[ax]) / D[ax];
            if (!(t > 0.0) || !(t < best)) continue;
            const double p0 = C[o0] + t * D[o0], p1 = C[o1] + t * D[o1];
            if (p0 >= r[2] && p0 <= r[4] && p1 >= r[3] && p1 <= r[5]) best = t;
        }
        for (int i = 0; i < n_box; ++i) {
            const double t = hit_aabb(C, D, boxes + 6 * i, boxes + 6 * i + 3);
            if (t < best) best = t;
        }
        for (int i = 0; i < n_obb; ++i) {
            const double* b = obbs + 7 * i;
            const double c = cos(b[6]), s = sin(b[6]);
            const double q[3] = {C[0] - b[0], C[1] - b[1], C[2] - b[2]};
            const double Cl[3] = {c * q[0] + s * q[1], -s * q[0] + c * q[1], q[2]};
            const double Dl[3] = {c * D[0] + s * D[1], -s * D[0] + c * D[1], D[2]};
            const double lo[3] = {-b[3], -b[4], -b[5]}, hi[3] = {b[3], b[4], b[5]};
            const double t = hit_aabb(Cl, Dl, lo, hi);
            if (t < best) best = t;
        }
        out[p] = best;
    }
}
