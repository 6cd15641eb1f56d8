// walk.cuh -- the fixed-point 3D-DDA walker (B2 of SURVEY §8(c), reading R13), shared by the DDA
// fill (graph.cu) and the matrix-free message kernels (bp.cu), which re-walk chunks of a ray from
// a stored cell.  Not part of the ABI; nothing here is shared with oracle/.
#pragma once

#include "internal.cuh"

namespace mrf {

// B1's result: the ray's fixed-point segment (16 fractional bits), its range Z and end L
struct Segment {
    long long g0[3], g1[3];
    double Z, L;
};

// State of the walk: current cell, per-axis step direction, and the exact crossing parameter
// of the next boundary on each axis as the rational num/den (den = |dG| > 0).  Held in scalar
// registers (no runtime-indexed arrays, which would live in local memory), 32-bit: mrf_create
// bounds the segment length (margin(D) <= D for the grid diagonal D, dims <= 8192), so
// den < 2^31 and num <= den + 2^16 fit in uint32 and the exact products in one IMAD.WIDE.U32.
// What the matrix-free message kernels need to re-walk any chunk of a ray (stored per ray by the
// first walk): the segment's start point and extent in fixed point (int32: the camera lies in
// the grid, dims <= 8192, and reading R17 bounds |G1 - G0| < 2^31), the range Z and the end L.
struct RaySeg {
    int g0[3];
    int dg[3];
    double Z, L;
    double y[3];  // RN(1 / |dg_k|) (1 for dg_k = 0): Walker::start's reciprocals, so a re-walk skips them
};

struct Walker {
    unsigned n0, n1, n2, d0, d1, d2;  // d = 0: the axis never crosses
    int c0, c1, c2, s0, s1, s2;       // cell, step direction
    double y0, y1, y2;                // RN(1 / d) per axis (crossing_t)
    double t_in;

    __device__ __forceinline__ static void axis_start(long long g0, long long g1, int& c, int& s, unsigned& n,
                                                      unsigned& d) {
        const long long dg = g1 - g0;
        long long cc = g0 >> kFixShift;  // arithmetic shift == floor
        const bool on_face = (g0 & (kFixOne - 1)) == 0;
        if (dg < 0 && on_face) cc -= 1;  // cell that contains t = 0+
        c = (int)cc;
        if (dg > 0) {
            s = 1;
            n = (unsigned)(((cc + 1) << kFixShift) - g0);
            d = (unsigned)dg;
        } else if (dg < 0) {
            s = -1;
            n = (unsigned)(g0 - (cc << kFixShift));
            d = (unsigned)(-dg);
        } else {
            s = 0;
            n = 1;
            d = 0;
        }
    }
    __device__ __forceinline__ void start(const Segment& sg) {
        axis_start(sg.g0[0], sg.g1[0], c0, s0, n0, d0);
        axis_start(sg.g0[1], sg.g1[1], c1, s1, n1, d1);
        axis_start(sg.g0[2], sg.g1[2], c2, s2, n2, d2);
        y0 = __drcp_rn((double)(d0 ? d0 : 1u));
        y1 = __drcp_rn((double)(d1 ? d1 : 1u));
        y2 = __drcp_rn((double)(d2 ? d2 : 1u));
        t_in = 0.0;
    }
    // The walk's exact state in cell (x, y, z) of the segment: the next boundary numerator of an
    // axis is a function of the cell alone (n = (c + 1) 2^16 - G0 stepping up, G0 - c 2^16 stepping
    // down), and t_in is the latest earlier crossing, RN((n_a - 2^16) / d_a) as crossing_t rounds
    // it -- 0 in the segment's start cell, where no axis has crossed yet (n_k <= 2^16), and the
    // crossing an empty skip entered by in a sparse map (skip_brick rounds it the same way).
    // Bit-identical to the state the walk from the start reaches.  (first = true forces t_in = 0.)
    __device__ __forceinline__ static void axis_at(int g0, int dg, int c, int& s, unsigned& n, unsigned& d) {
        if (dg > 0) {
            s = 1;
            n = (unsigned)(((c + 1) << kFixShift) - g0);
            d = (unsigned)dg;
        } else if (dg < 0) {
            s = -1;
            n = (unsigned)(g0 - (c << kFixShift));
            d = (unsigned)(-dg);
        } else {
            s = 0;
            n = 1;
            d = 0;
        }
    }
    __device__ __forceinline__ void restart(const RaySeg& sg, int x, int y, int z, bool first) {
        c0 = x;
        c1 = y;
        c2 = z;
        axis_at(sg.g0[0], sg.dg[0], x, s0, n0, d0);
        axis_at(sg.g0[1], sg.dg[1], y, s1, n1, d1);
        axis_at(sg.g0[2], sg.dg[2], z, s2, n2, d2);
        y0 = sg.y[0];
        y1 = sg.y[1];
        y2 = sg.y[2];
        // the entry crossing: the largest (n_k - 2^16) / d_k over the axes that crossed
        int a = -1;
        unsigned pa = 0, da = 1;
        const unsigned one = (unsigned)kFixOne;
        if (d0 && n0 > one) { a = 0; pa = n0 - one; da = d0; }
        if (d1 && n1 > one && (a < 0 || before(pa, da, n1 - one, d1))) { a = 1; pa = n1 - one; da = d1; }
        if (d2 && n2 > one && (a < 0 || before(pa, da, n2 - one, d2))) { a = 2; pa = n2 - one; da = d2; }
        if (first || a < 0) {
            t_in = 0.0;
        } else {
            const double yy = a == 0 ? y0 : (a == 1 ? y1 : y2);
            const double nn = (double)pa, dd = (double)da;
            const double q = __dmul_rn(nn, yy);
            t_in = __fma_rn(__fma_rn(-q, dd, nn), yy, q);
        }
    }
    __device__ __forceinline__ bool inside(const GridDesc& g) const {
        return (unsigned)c0 < (unsigned)g.nx && (unsigned)c1 < (unsigned)g.ny && (unsigned)c2 < (unsigned)g.nz;
    }
    // n_a / d_a < n_b / d_b, exactly
    __device__ __forceinline__ static bool before(unsigned na, unsigned da, unsigned nb, unsigned db) {
        return (unsigned long long)na * db < (unsigned long long)nb * da;
    }
    // The earliest next crossing as (num, den) and its axis (-1 if no axis crosses).
    __device__ __forceinline__ int earliest(unsigned& na, unsigned& da) const {
        int a = -1;
        na = 1;
        da = 0;
        if (d0) { a = 0; na = n0; da = d0; }
        if (d1 && (a < 0 || before(n1, d1, na, da))) { a = 1; na = n1; da = d1; }
        if (d2 && (a < 0 || before(n2, d2, na, da))) { a = 2; na = n2; da = d2; }
        return a;
    }
    // Advance every axis whose crossing ties with (na, da) (simultaneous steps on corners/edges).
    __device__ __forceinline__ void advance(unsigned na, unsigned da) {
        const unsigned long long r = (unsigned long long)na;
        const bool t0 = d0 && (unsigned long long)n0 * da == r * d0;
        const bool t1 = d1 && (unsigned long long)n1 * da == r * d1;
        const bool t2 = d2 && (unsigned long long)n2 * da == r * d2;
        if (t0) { c0 += s0; n0 += (unsigned)kFixOne; }
        if (t1) { c1 += s1; n1 += (unsigned)kFixOne; }
        if (t2) { c2 += s2; n2 += (unsigned)kFixOne; }
    }
    // Empty skip (sparse bricks): from a cell of an unallocated brick, jump to the first
    // cell past the brick in one step -- exactly the state the cell-by-cell walk reaches.  Axis k
    // leaves the brick (clamped to the grid) after m_k crossings, the m_k-th at the exact time
    // (n_k + (m_k - 1) 2^16) / d_k; t* is the earliest of these; every axis then takes all its
    // crossings at times <= t* (ties step together, as in advance()), and t_in = RN(t*), the
    // crossing that enters the new cell.  Returns false if the segment ends inside the brick.
    __device__ __forceinline__ static unsigned exit_steps(int c, int s, int dim, int bs) {
        if (s > 0) return (unsigned)(min(((c >> bs) + 1) << bs, dim) - c);
        return (unsigned)(c - ((c >> bs) << bs) + 1);
    }
    // 1 + floor((Ns d - n Ds) / (2^16 Ds)) crossings of an axis at times (n + i 2^16) / d <= Ns / Ds
    // (0 if even the first is later): the quotient (small, <= the brick edge) estimated in fp64 with
    // y = RN(1 / Ds) and corrected exactly in integers (a 64-bit integer division is ~100 ops)
    __device__ __forceinline__ static unsigned long long crossings_upto(unsigned n, unsigned d, unsigned long long Ns,
                                                                        unsigned Ds, double y) {
        if (!d) return 0;
        const unsigned long long lhs = Ns * d, rhs = (unsigned long long)n * Ds;  // t* >= n / d ?
        if (lhs < rhs) return 0;
        const unsigned long long diff = lhs - rhs, unit = (unsigned long long)kFixOne * Ds;
        unsigned long long k = (unsigned long long)__dmul_rn(__dmul_rn((double)diff, y), 1.0 / 65536.0);
        while (k * unit > diff) --k;
        while ((k + 1) * unit <= diff) ++k;
        return k + 1;
    }
    __device__ bool skip_brick(const GridDesc& g) {
        const int bs = g.bshift;
        int a = -1;
        unsigned long long Ns = 0;
        unsigned Ds = 1;
        if (d0) {
            a = 0;
            Ns = n0 + (unsigned long long)(exit_steps(c0, s0, g.nx, bs) - 1) * kFixOne;
            Ds = d0;
        }
        if (d1) {
            const unsigned long long N = n1 + (unsigned long long)(exit_steps(c1, s1, g.ny, bs) - 1) * kFixOne;
            if (a < 0 || N * Ds < Ns * d1) { a = 1; Ns = N; Ds = d1; }
        }
        if (d2) {
            const unsigned long long N = n2 + (unsigned long long)(exit_steps(c2, s2, g.nz, bs) - 1) * kFixOne;
            if (a < 0 || N * Ds < Ns * d2) { a = 2; Ns = N; Ds = d2; }
        }
        if (a < 0 || Ns >= Ds) return false;  // the segment ends in this brick
        const double y = a == 0 ? y0 : (a == 1 ? y1 : y2);  // RN(1 / Ds)
        const unsigned long long k0 = crossings_upto(n0, d0, Ns, Ds, y), k1 = crossings_upto(n1, d1, Ns, Ds, y),
                                 k2 = crossings_upto(n2, d2, Ns, Ds, y);
        c0 += s0 * (int)k0; n0 += (unsigned)(k0 * kFixOne);
        c1 += s1 * (int)k1; n1 += (unsigned)(k1 * kFixOne);
        c2 += s2 * (int)k2; n2 += (unsigned)(k2 * kFixOne);
        const double n = (double)Ns, d = (double)Ds;
        const double q = __dmul_rn(n, y);
        t_in = __fma_rn(__fma_rn(-q, d, n), y, q);  // RN(Ns / Ds), as crossing_t
        return true;
    }
};

// t of the next crossing (num/den, correctly rounded) or 1 when the walk ends in this cell.
// The quotient is RN(n/d) by Markstein's sequence -- y = RN(1/d) (per axis, once per ray),
// q = RN(n y), r = n - d q (exact with an FMA), t = RN(q + r y) -- which equals the correctly
// rounded division for every operand pair of the walk (integers < 2^31; checked against
// __ddiv_rn on 6.9e10 random pairs, scripts/div_check.cu, zero mismatches) at a third of the cost.
__device__ __forceinline__ double crossing_t(const Walker& w, int a, unsigned na, unsigned da, bool& last) {
    last = (a < 0) || (na >= da);
    const double y = a == 0 ? w.y0 : (a == 1 ? w.y1 : w.y2);
    const double n = (double)na, d = (double)da;
    const double q = __dmul_rn(n, y);
    const double r = __fma_rn(-q, d, n);
    return last ? 1.0 : __fma_rn(r, y, q);
}


// The matrix-free message kernels' view of the graph (K12): the grid, the per-ray segments and the
// chunk checkpoints ck[row_ptr[r] / 4 + c] = voxel slot of the first cell of chunk c of ray r
// (chunks of the ray's K5 class: class_K for the short classes, 8 for long rays; a ray of n
// incidences has at most pad8(n) / 4 of them, K >= 4).
struct WalkParams {
    GridDesc g;
    const RaySeg* seg;
    const int32_t* ck;
};

// K5 over one class with the chunks re-walked (bp.cu ray_msg_walk_kernel / the long-ray kernel)
void launch_ray_messages_walk(int cls, long long n_rays, const int32_t* rays, const long long* row_ptr,
                              const RayInfo* ray_z, int32_t* lam, const long long* T, const MsgParams& mp,
                              const WalkParams& wp, float* scratch, long long scratch_per_warp, int n_warps_long,
                              int math, cudaStream_t s);
// the checkpoints of rays [r0, r0 + n) from the voxel slots of a walk (graph.cu)
void launch_ck_extract(long long n, const long long* row_ptr, const RayInfo* info, const int32_t* vid, int32_t* ck,
                       RaySeg* seg,
                       cudaStream_t s);

}  // namespace mrf
