// graph.cu -- ray-voxel factor graph construction on sm_100a (K1, K3, K4 + work lists).
//
// "all keyframe images are ray traced ... The ray traversal is done via the
// standard 3DDA traversal algorithm"; traverse "until a 3 sigma distance beyond the
// measured depth".  Here each pixel's segment is quantised to 16-fractional-bit grid
// coordinates and walked with an integer-only DDA (DESIGN.md §Graph build, readings R5, R6,
// R11, R13), so the ray->voxel index lists are bit-exact across implementations.
//
// Layout: one thread per owned pixel; a warp holds 32 neighbouring pixels of one image row,
// so the warp's rays start in the same voxel and fan out slowly -- voxel-histogram and
// transpose-cursor atomics are aggregated per warp with __match_any_sync.
#include "internal.cuh"
#include "walk.cuh"

namespace mrf {
namespace {

constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- B1: pixel -> segment
// All fp64 steps use explicitly rounded intrinsics (no FMA contraction), in the order
// stated in DESIGN.md §Graph build, so the quantised end points are reproducible.

// sigma(Z) = c0 + c1 Z + c2 Z^2 of the traversal margin, with the pixel's patch
// coefficients under the per-patch model (R25)
__device__ __forceinline__ double pixel_sigma(const NoiseDesc& n, int u, int v, double Z) {
    double c0 = n.c0, c1 = n.c1, c2 = n.c2;
    if (n.pcoef) {
        const double* k = n.pcoef + 6 * pixel_patch(n, u, v) + 3;
        c0 = k[0];
        c1 = k[1];
        c2 = k[2];
    }
    return __dadd_rn(__dadd_rn(c0, __dmul_rn(c1, Z)), __dmul_rn(__dmul_rn(c2, Z), Z));
}

// 0 = kept, 1 = invalid pixel, 2 = dropped (measured point outside the grid)
__device__ __forceinline__ int pixel_segment(const FrameDesc& f, const GridDesc& g, const NoiseDesc& n, int u,
                                             int v, float zf, Segment& sg) {
    const double z = (double)zf;
    if (!(z > 0.0) || isinf(z)) return 1;
    const double xc = __ddiv_rn(__dsub_rn((double)u, f.cx), f.fx);
    const double yc = __ddiv_rn(__dsub_rn((double)v, f.cy), f.fy);
    const double rho = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(xc, xc), __dmul_rn(yc, yc)), 1.0));
    const double Z = __dmul_rn(z, rho);
    const double sig = pixel_sigma(n, u, v, Z);
    double margin = __dmul_rn(n.margin_k, sig);
    if (margin < n.margin_min) margin = n.margin_min;
    const double L = __dadd_rn(Z, margin);
    const double l_over_rho = __ddiv_rn(L, rho);
    const double org[3] = {g.ox, g.oy, g.oz};
    const int dims[3] = {g.nx, g.ny, g.nz};
    for (int k = 0; k < 3; ++k) {
        const double d = __dadd_rn(__dadd_rn(__dmul_rn(f.R[3 * k], xc), __dmul_rn(f.R[3 * k + 1], yc)), f.R[3 * k + 2]);
        const double hit = __ddiv_rn(__dsub_rn(__dadd_rn(f.C[k], __dmul_rn(z, d)), org[k]), g.res);
        if (hit < 0.0 || hit >= (double)dims[k]) return 2;
        const double end = __dadd_rn(f.C[k], __dmul_rn(l_over_rho, d));
        const double a = __ddiv_rn(__dsub_rn(f.C[k], org[k]), g.res);
        const double b = __ddiv_rn(__dsub_rn(end, org[k]), g.res);
        sg.g0[k] = __double2ll_rn(__dmul_rn(a, 65536.0));
        sg.g1[k] = __double2ll_rn(__dmul_rn(b, 65536.0));
    }
    sg.Z = Z;
    sg.L = L;
    return 0;
}

__device__ __forceinline__ void owned_pixel(const FrameDesc& f, long long i, int& u, int& v) {
    const int lr = (int)(i / f.W);
    u = (int)(i - (long long)lr * f.W);
    v = f.rank + lr * f.world;
}

// ---------------------------------------------------------------- K1
__device__ __forceinline__ void raygen_count_body(const FrameDesc& f, long long i, const GridDesc& g,
                                                  const NoiseDesc& n, const float* __restrict__ depth, int32_t* n_r,
                                                  int8_t* status, RayInfo* ray_z, unsigned long long* counters) {
    const long long n_pix = (long long)f.rows_owned * f.W;
    int st = 3;
    if (i < n_pix) {
        int u, v;
        owned_pixel(f, i, u, v);
        Segment sg;
        st = pixel_segment(f, g, n, u, v, depth[(long long)v * f.W + u], sg);
        int bound = 0;
        RayInfo rz{0, 0.f, 0, f.index};
        if (st == 0) {
            // Upper bound of the walk's length without walking: every DDA step moves at least one
            // axis one cell towards the cell of the end point, so n <= 1 + sum_k |c_end,k - c_0,k|
            // (0 if the start cell is outside the grid).  The fill writes the exact n.
            Walker w;
            w.start(sg);
            if (w.inside(g)) {
                if (f.skip_count) {
                    bound = 0;  // counted again against the final allocation (sync_fill)
                } else if (g.bmask) {
                    // sparse bricks: the dense bound would size the layout for the skipped free
                    // space too, so count the cells of allocated bricks exactly (the walk without
                    // its crossing parameters)
                    for (;;) {
                        if (!cell_in_map(g, w.c0, w.c1, w.c2)) {  // empty skip
                            if (!w.skip_brick(g) || !w.inside(g)) break;
                            continue;
                        }
                        ++bound;
                        unsigned na, da;
                        const int a = w.earliest(na, da);
                        if (a < 0 || na >= da) break;
                        w.advance(na, da);
                        if (!w.inside(g)) break;
                    }
                } else {
                    bound = 1 + abs((int)(sg.g1[0] >> kFixShift) - w.c0) +
                            abs((int)(sg.g1[1] >> kFixShift) - w.c1) + abs((int)(sg.g1[2] >> kFixShift) - w.c2);
                }
            }
            // LUT row of the measured range (bin centres, clamped to the edge centres); per-patch
            // noise: the patch and the range
            if (n.pcoef) {
                rz.iz = pixel_patch(n, u, v);
                rz.wz = (float)sg.Z;
            } else {
            double fz = __dsub_rn(__dmul_rn(__ddiv_rn(__dsub_rn(sg.Z, n.z_lo), __dsub_rn(n.z_hi, n.z_lo)),
                                            (double)n.n_z), 0.5);
            if (fz < 0.0) fz = 0.0;
            if (fz > (double)(n.n_z - 1)) fz = (double)(n.n_z - 1);
            int iz = (int)floor(fz);
            if (iz > n.n_z - 2) iz = n.n_z - 2;
            rz.iz = iz;
            rz.wz = (float)(fz - (double)iz);
            }
        }
        rz.n = 0;  // set by the fill
        n_r[f.ray_base + i] = (bound + kSegAlign - 1) & ~(kSegAlign - 1);  // segments start at multiples of 8
        status[f.ray_base + i] = (int8_t)st;
        ray_z[f.ray_base + i] = rz;
    }
    const unsigned inv = __ballot_sync(kFull, st == 1);
    const unsigned drp = __ballot_sync(kFull, st == 2);
    if ((threadIdx.x & 31) == 0) {
        if (inv) atomicAdd(&counters[0], (unsigned long long)__popc(inv));
        if (drp) atomicAdd(&counters[1], (unsigned long long)__popc(drp));
    }
}

__global__ void __launch_bounds__(128) raygen_count_kernel(FrameDesc f, GridDesc g, NoiseDesc n,
                                                           const float* __restrict__ depth, int32_t* n_r,
                                                           int8_t* status, RayInfo* ray_z,
                                                           unsigned long long* counters) {
    raygen_count_body(f, (long long)blockIdx.x * blockDim.x + threadIdx.x, g, n, depth, n_r, status, ray_z, counters);
}

// K1 of every frame added since the last batch in one launch (frames[k] owns the CTAs
// [cta0[k], cta0[k+1]) of 128 pixels; its depth image at depth_all + depth_off)
__global__ void __launch_bounds__(128) raygen_count_batch_kernel(const FrameDesc* __restrict__ frames,
                                                                 const int* __restrict__ cta0, int n_frames,
                                                                 GridDesc g, NoiseDesc n,
                                                                 const float* __restrict__ depth_all, int32_t* n_r,
                                                                 int8_t* status, RayInfo* ray_z,
                                                                 unsigned long long* counters) {
    __shared__ FrameDesc f;
    __shared__ int s_c0;
    if (threadIdx.x == 0) {
        int lo = 0, hi = n_frames - 1;  // last k with cta0[k] <= blockIdx.x
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(cta0 + mid) <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
        }
        f = frames[lo];
        s_c0 = __ldg(cta0 + lo);
    }
    __syncthreads();
    raygen_count_body(f, (long long)((int)blockIdx.x - s_c0) * 128 + threadIdx.x, g, n, depth_all + f.depth_off, n_r,
                      status, ray_z, counters);
}

// Tile runs (K4b): a run ends where the tile changes (a ray crosses a convex tile once), after
// kRunMax incidences, or before a step that is not a single-axis unit step (an exact DDA tie).
// Split rule (shared by the count in K3 and the transpose fill K4b, which must agree):
// incidence (tile b, in-tile slot l) extends the current run (tile, length n, last slot prev)
// iff it lies in the same tile, the run holds fewer than kRunMax incidences and the step is a
// single-axis unit step.  Consecutive cells of a DDA walk differ by at most one per axis, so
// the slot difference d = dx + 32 dy + 1024 dz (balanced base-32 digits) is a single-axis unit
// step iff |d| is 1, 32 or 1024.
__device__ __forceinline__ bool run_extends(int b, int l, int tile, int n, int prev) {
    const int ad = abs(l - prev);
    return b == tile && n < kRunMax && (ad == 1 || ad == 32 || ad == 1024);
}

// Run builder of the transpose fill (K4b)
struct RunBuilder {
    int tile = -1, n = 0, prev = 0;  // current run: tile, length, in-tile slot of its last element
    long long start = 0;
    unsigned mx = 0, my = 0, neg = 0, slot0 = 0;
    // Does incidence (tile b, in-tile slot l) extend the current run?  Records the step if so.
    __device__ __forceinline__ bool extend(int b, int l) {
        if (b != tile || n >= kRunMax) return false;
        const int dx = (l & 31) - (prev & 31), dy = ((l >> 5) & 31) - ((prev >> 5) & 31), dz = (l >> 10) - (prev >> 10);
        if ((dx != 0) + (dy != 0) + (dz != 0) != 1) return false;
        const int d = dx + dy + dz;
        if (d != 1 && d != -1) return false;  // same rule as run_extends
        const int ax = dx ? 0 : (dy ? 1 : 2);
        if (ax == 0) mx |= 1u << (n - 1);
        if (ax == 1) my |= 1u << (n - 1);
        if (d < 0) neg |= 1u << ax;
        ++n;
        prev = l;
        return true;
    }
    __device__ __forceinline__ void begin(int b, int l, long long e) {
        tile = b;
        n = 1;
        prev = l;
        start = e;
        mx = my = neg = 0;
        slot0 = (unsigned)l;
    }
    __device__ __forceinline__ Run make() const {
        return Run{(unsigned)start, slot0 | ((unsigned)(n - 1) << 14) | (neg << 20), mx, my};
    }
};

// ---------------------------------------------------------------- NEXT #4: brick allocation
// SPEC allocate_for_depth_image (reading R23): per pixel with a valid depth whose
// measured point p lies in the grid, r = margin_k sigma(Z) / res; every brick holding a cell of
// [floor(p - r), floor(p + r)] (clamped) is marked.  fp64 in the oracle's op order (the mask is
// bit-exact with the oracle's allocation); the byte stores of 1 are idempotent, so no atomics.
__global__ void brick_alloc_kernel(FrameDesc f, GridDesc g, NoiseDesc n, const float* __restrict__ depth,
                                   uint8_t* mask) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)f.W * f.H) return;
    const int v = (int)(i / f.W), u = (int)(i - (long long)v * f.W);
    const double z = (double)depth[i];
    if (!(z > 0.0) || isinf(z)) return;
    const double xc = __ddiv_rn(__dsub_rn((double)u, f.cx), f.fx);
    const double yc = __ddiv_rn(__dsub_rn((double)v, f.cy), f.fy);
    const double rho = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(xc, xc), __dmul_rn(yc, yc)), 1.0));
    const double Z = __dmul_rn(z, rho);
    const double sig = pixel_sigma(n, u, v, Z);
    const double r = __ddiv_rn(__dmul_rn(n.margin_k, sig), g.res);
    const double org[3] = {g.ox, g.oy, g.oz};
    const int dims[3] = {g.nx, g.ny, g.nz};
    int lo[3], hi[3];
    for (int k = 0; k < 3; ++k) {
        const double d = __dadd_rn(__dadd_rn(__dmul_rn(f.R[3 * k], xc), __dmul_rn(f.R[3 * k + 1], yc)), f.R[3 * k + 2]);
        const double p = __ddiv_rn(__dsub_rn(__dadd_rn(f.C[k], __dmul_rn(z, d)), org[k]), g.res);
        if (p < 0.0 || p >= (double)dims[k]) return;
        lo[k] = max((int)floor(__dsub_rn(p, r)), 0);
        hi[k] = min((int)floor(__dadd_rn(p, r)), dims[k] - 1);
    }
    for (int bz = lo[2] >> g.bshift; bz <= hi[2] >> g.bshift; ++bz)
        for (int by = lo[1] >> g.bshift; by <= hi[1] >> g.bshift; ++by)
            for (int bx = lo[0] >> g.bshift; bx <= hi[0] >> g.bshift; ++bx)
                mask[bx + g.nbx * (by + (long long)g.nby * bz)] = 1;
}

// ---------------------------------------------------------------- K3
// B3: off_q = clamp(rint((0.5 (t_in + t_out) L - Z) * 32768), +-32767), the span midpoint
// relative to the measured range (reading R6).  Each thread stages its ray's outputs in a private
// 8-slot chunk of shared memory and writes a whole chunk at once (two 16-byte vid stores, one
// 16-byte off_q store; segments are 8-aligned, padding slots get 0): one scattered 4-byte and
// one 2-byte store per step had the walk waiting on the store queue.
// With MRF_FILL_LNU the chunk's log nu (B3) is interpolated here too: 8 independent table
// lookups per flush (16 loads in flight) instead of a separate pass that re-reads off_q.
__device__ __forceinline__ void flush_chunk(int32_t* vid, int16_t* off_q, int e_chunk, int nvalid,
                                            const int* sv, const short* so, float* lnu, const MsgParams& mp, int iz,
                                            float wz, int32_t* lam0) {
    int v[8];
    short o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        v[k] = k < nvalid ? sv[k] : 0;
        o[k] = k < nvalid ? so[k] : (short)0;
    }
#if MRF_FILL_LNU
    // (per-patch noise, R25: lnu_fill_kernel overwrites these with the closed form after the walk,
    // which reads the table's row 0 here -- any test of the mode in this function costs the walk
    // registers and spills in every mode)
    {
        LutFetch lf[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) lf[k] = lut_fetch(mp, iz, o[k]);
        float l[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) l[k] = k < nvalid ? lut_finish(lf[k], wz) : 0.f;
        float4* dl = reinterpret_cast<float4*>(lnu + e_chunk);
        dl[0] = make_float4(l[0], l[1], l[2], l[3]);
        dl[1] = make_float4(l[4], l[5], l[6], l[7]);
    }
#endif
    int4* dv = reinterpret_cast<int4*>(vid + e_chunk);
    dv[0] = make_int4(v[0], v[1], v[2], v[3]);
    dv[1] = make_int4(v[4], v[5], v[6], v[7]);
    auto pk = [](short a, short b) { return (unsigned)(unsigned short)a | ((unsigned)(unsigned short)b << 16); };
    *reinterpret_cast<uint4*>(off_q + e_chunk) = make_uint4(pk(o[0], o[1]), pk(o[2], o[3]), pk(o[4], o[5]), pk(o[6], o[7]));
    if (lam0) {  // new incidences start with lambda = 0 (B4): written here instead of a memset pass
        int4* dl = reinterpret_cast<int4*>(lam0 + e_chunk);
        dl[0] = make_int4(0, 0, 0, 0);
        dl[1] = make_int4(0, 0, 0, 0);
    }
}

// Resident CTAs of 128 threads per SM: 6 (<= 80 registers), also when the walk builds the tile
// runs (RUNS): the values read only at chunk flushes and run ends (LUT row, a run's first slots)
// live in shared memory, which took the run builder's spills at 80 registers from 56 to 4 bytes
// (frames30: fill 9.90 ms at 5 CTAs, 9.46 ms at 6 per 30-frame step; without runs 8.2 ms).
#ifndef MRF_FILL_MIN_BLOCKS
#define MRF_FILL_MIN_BLOCKS 6
#endif
#ifndef MRF_FILL_MIN_BLOCKS_RUNS
#define MRF_FILL_MIN_BLOCKS_RUNS 6
#endif
// One launch fills every frame added since the last fill (frames[k] owns the CTAs
// [cta0[k], cta0[k+1])): one wave-quantisation tail per batch instead of per frame.
template <bool SPARSE, bool RUNS, bool COUNT = true>
__global__ void __launch_bounds__(kFillThreads, RUNS ? MRF_FILL_MIN_BLOCKS_RUNS : MRF_FILL_MIN_BLOCKS) dda_fill_kernel(const FrameDesc* __restrict__ frames,
                                                       const int* __restrict__ cta0, int n_frames, GridDesc g,
                                                       NoiseDesc n, const float* __restrict__ depth_all,
                                                       const long long* __restrict__ row_ptr, int32_t* vid,
                                                       int16_t* off_q, int32_t* tile_runs, RayInfo* ray_z,
                                                       unsigned long long* counters, MsgParams mp, float* lnu,
                                                       RunSink sink, RaySeg* seg, unsigned long long* class_counts,
                                                       int32_t* lam0) {
    __shared__ int s_vid[kFillThreads][8];
    __shared__ Run s_done[RUNS ? kFillThreads : 1];  // a run that ended at this step, per thread
    __shared__ int s_done_key[RUNS ? kFillThreads : 1];
    // per-thread values read only at chunk flushes / run ends (kept out of registers: the walk
    // with the run builder is register-bound)
    __shared__ int s_iz[kFillThreads];
    __shared__ float s_wz[kFillThreads];
    __shared__ unsigned s_run_e[RUNS ? kFillThreads : 1], s_run_slot0[RUNS ? kFillThreads : 1];
    __shared__ short s_off[kFillThreads][8];
    __shared__ FrameDesc f;
    __shared__ int s_fi;
    if (threadIdx.x == 0) {
        int lo = 0, hi = n_frames - 1;  // last k with cta0[k] <= blockIdx.x
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(cta0 + mid) <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
        }
        s_fi = lo;
        f = frames[lo];
    }
    __syncthreads();
    int* sv = s_vid[threadIdx.x];
    short* so = s_off[threadIdx.x];
    const long long i = (long long)((int)blockIdx.x - __ldg(cta0 + s_fi)) * kFillThreads + threadIdx.x;
    const float* __restrict__ depth = depth_all + f.depth_off;
    const long long n_pix = (long long)f.rows_owned * f.W;
    const int lane = threadIdx.x & 31;
    bool alive = false;
    Segment sg;
    Walker w;
    // current tile run (K4b: counted per bucket, and emitted to the sink when it ends): tile, length,
    // in-tile slots of its first and last element, first incidence slot, x / y step masks; the
    // step signs are the ray's (a DDA walk is monotone on every axis)
    int run_tile = -1, run_n = 0, run_prev = 0;
    unsigned run_mx = 0, run_my = 0, run_neg = 0;
    unsigned long long sink_base = 0;  // the warp's block of run slots (RunSink::emit)
    int sink_left = 0;
    const int bucket0 = f.index * f.bucket_stride;
    int e = 0, e_cap = 0;  // incidence slots (< 2^31 per ctx)
    s_iz[threadIdx.x] = 0;
    s_wz[threadIdx.x] = 0.f;
    if (i < n_pix) {
        int u, v;
        owned_pixel(f, i, u, v);
        e = (int)row_ptr[f.ray_base + i];
        if (pixel_segment(f, g, n, u, v, depth[(long long)v * f.W + u], sg) == 0) {
            w.start(sg);
            alive = w.inside(g);
            e_cap = (int)row_ptr[f.ray_base + i + 1];  // the segment K1 sized from its bound
            run_neg = ((unsigned)(w.s0 < 0) | ((unsigned)(w.s1 < 0) << 1) | ((unsigned)(w.s2 < 0) << 2)) << 20;
            if (seg)  // matrix-free: what a re-walk of any chunk of this ray needs (K12)
                seg[f.ray_base + i] = RaySeg{{(int)sg.g0[0], (int)sg.g0[1], (int)sg.g0[2]},
                                             {(int)(sg.g1[0] - sg.g0[0]), (int)(sg.g1[1] - sg.g0[1]),
                                              (int)(sg.g1[2] - sg.g0[2])},
                                             sg.Z, sg.L};
            if (MRF_FILL_LNU) {  // the depth coordinate of the table (K1)
                s_iz[threadIdx.x] = mp.pcoef ? 0 : ray_z[f.ray_base + i].iz;  // (R25: iz is the patch)
                s_wz[threadIdx.x] = ray_z[f.ray_base + i].wz;
            }
        }
    }
    const int e_ray = e;
    bool overflow = false;
    for (;;) {
        const unsigned am = __ballot_sync(kFull, alive);
        if (am == 0) break;
        bool has_done = false;  // a run ended at this step (to the sink, below, with all lanes)
        if (alive) {
            const bool keep = !SPARSE || cell_in_map(g, w.c0, w.c1, w.c2);
            bool start = false;
            int b = 0;
            if (keep) {
                bool last;
                unsigned na, da;
                const int a = w.earliest(na, da);
                const double t_out = crossing_t(w, a, na, da, last);
                const int vx = voxel_slot(g, w.c0, w.c1, w.c2);
                MRF_ASSERT(vx >= 0 && (vx >> kTileShift) < g.ntx * g.nty * g.ntz && e < e_cap);
                const double mid = __dmul_rn(__dmul_rn(0.5, __dadd_rn(w.t_in, t_out)), sg.L);
                long long q = __double2ll_rn(__dmul_rn(__dsub_rn(mid, sg.Z), 32768.0));
                q = q > 32767 ? 32767 : (q < -32767 ? -32767 : q);
                sv[e & 7] = vx;
                so[e & 7] = (short)q;
                if ((e & 7) == 7)
                    flush_chunk(vid, off_q, e - 7, 8, sv, so, lnu, mp, s_iz[threadIdx.x], s_wz[threadIdx.x], lam0);
                // K4b: runs per tile (a warp's concurrent run starts in one tile share an atomic);
                // a run that ends here goes to the sink.  COUNT = false (the pixel-block K6b needs
                // no transpose): no run state at all
                b = vx >> kTileShift;
                const int l = vx & (kTileSlots - 1);
                const int ad = abs(l - run_prev);
                if (COUNT) start = !run_extends(b, l, run_tile, run_n, run_prev);
                if (!COUNT) {
                } else if (start) {
                    if (RUNS && run_tile >= 0) {  // the run that ends here waits in shared memory
                        s_done[threadIdx.x] = Run{s_run_e[threadIdx.x],
                                                  s_run_slot0[threadIdx.x] | ((unsigned)(run_n - 1) << 14) | run_neg,
                                                  run_mx, run_my};
                        s_done_key[threadIdx.x] = bucket0 + run_tile;
                        has_done = true;
                    }
                    run_tile = b;
                    run_n = 1;
                    if (RUNS) {
                        s_run_slot0[threadIdx.x] = (unsigned)l;
                        s_run_e[threadIdx.x] = (unsigned)e;
                    }
                    run_mx = run_my = 0;
                } else {
                    if (RUNS) {
                        run_mx |= (unsigned)(ad == 1) << (run_n - 1);
                        run_my |= (unsigned)(ad == 32) << (run_n - 1);
                    }
                    ++run_n;
                }
                run_prev = l;
                ++e;
                if (last) {
                    alive = false;
                } else {
                    w.advance(na, da);
                    w.t_in = t_out;
                    alive = w.inside(g);
                }
            } else {  // empty skip: past the unallocated brick in one step (sparse bricks)
                alive = w.skip_brick(g) && w.inside(g);
            }
            const unsigned sm = COUNT ? __ballot_sync(am, start) : 0u;
            if (COUNT && start && tile_runs) {  // (no counting on the matrix-free re-walks)
                const int key = bucket0 + b;  // (frame, tile) bucket; the tile itself in per-ray mode
                const unsigned peers = __match_any_sync(sm, key);
                if (lane == __ffs(peers) - 1) atomicAdd(&tile_runs[key], __popc(peers));
            }

            // cannot happen (K1's count); never write past the segment.  In a sparse map only a
            // cell that would be emitted counts.
            if (alive && e >= e_cap && (!SPARSE || cell_in_map(g, w.c0, w.c1, w.c2))) {
                alive = false;
                overflow = true;
            }
            if (!alive && (e & 7))  // partial tail
                flush_chunk(vid, off_q, e & ~7, e & 7, sv, so, lnu, mp, s_iz[threadIdx.x], s_wz[threadIdx.x], lam0);
        }
        if (RUNS) sink.emit(has_done, s_done[threadIdx.x], s_done_key[threadIdx.x], lane, sink_base, sink_left);
    }
    if (RUNS) {  // every ray's last run
        const bool last_run = run_tile >= 0;
        sink.emit(last_run,
                  Run{s_run_e[threadIdx.x], s_run_slot0[threadIdx.x] | ((unsigned)(run_n - 1) << 14) | run_neg, run_mx,
                      run_my},
                  bucket0 + run_tile, lane, sink_base, sink_left);
    }
    int ne = 0;
    if (i < n_pix) {
        ne = (int)(e - e_ray);
        ray_z[f.ray_base + i].n = ne;
        // The rest of the segment K1 sized (its bound can exceed the walk at ties and grid exits)
        // gets voxel 0: K5 lanes gather T and the keyframe averages through every slot of their
        // chunk, masked elements included, so no slot of a segment may hold a stale id.
        for (int z = (e + 7) & ~7; z < e_cap; z += 8) {
            int4* dv = reinterpret_cast<int4*>(vid + z);
            dv[0] = make_int4(0, 0, 0, 0);
            dv[1] = make_int4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(off_q + z) = make_uint4(0u, 0u, 0u, 0u);
            if (MRF_FILL_LNU) {
                float4* dl = reinterpret_cast<float4*>(lnu + z);
                dl[0] = make_float4(0.f, 0.f, 0.f, 0.f);
                dl[1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (lam0) {
                int4* dq = reinterpret_cast<int4*>(lam0 + z);
                dq[0] = make_int4(0, 0, 0, 0);
                dq[1] = make_int4(0, 0, 0, 0);
            }
        }
    }
    if (class_counts) {  // the rays per K5 length class and the longest ray (no separate pass)
        const int k = ne > 0 ? ray_class(ne) : -1;
        const unsigned act = __ballot_sync(kFull, k >= 0);
        if (k >= 0) {
            const unsigned peers = __match_any_sync(act, k);
            if (lane == __ffs(peers) - 1) atomicAdd(&class_counts[k], (unsigned long long)__popc(peers));
        }
        int mx = ne;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
        if (lane == 0 && mx > 0) atomicMax(&class_counts[kNumClasses], (unsigned long long)mx);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ne += __shfl_xor_sync(kFull, ne, o);
    const unsigned ovf = __ballot_sync(kFull, overflow);
    if (lane == 0) {
        if (ne) atomicAdd(&counters[0], (unsigned long long)ne);
        if (ovf) atomicAdd(&counters[1], (unsigned long long)__popc(ovf));
    }
}

// log nu per incidence (B3): thread per ray of the frame, one 8-slot chunk per step (a 16-byte
// off_q read, a 32-byte log-nu write); the table rows of the ray stay in L1.
__global__ void __launch_bounds__(256) lnu_fill_kernel(long long r0, long long n_rays, MsgParams mp,
                                                       const long long* __restrict__ row_ptr,
                                                       const RayInfo* __restrict__ ray_z,
                                                       const int16_t* __restrict__ off_q, float* lnu) {
    const long long r = r0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= r0 + n_rays) return;
    const RayInfo ri = ray_z[r];
    const long long e0 = row_ptr[r];
    for (int c = 0; c < ri.n; c += 8) {
        const uint4 o = __ldg(reinterpret_cast<const uint4*>(off_q + e0 + c));
        const unsigned ow[4] = {o.x, o.y, o.z, o.w};
        float out[8];
        // every slot holds a valid code (padding: 0), so all 16 table loads issue back to back;
        // padding slots are zeroed by multiplication afterwards (no branch around the loads)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int q = (int)(short)((ow[k >> 1] >> (16 * (k & 1))) & 0xffffu);
            out[k] = (mp.pcoef ? patch_lnu(mp, ri.iz, ri.wz, q) : lut_finish(lut_fetch(mp, ri.iz, q), ri.wz)) *
                     (float)(c + k < ri.n);
        }
        float4* dst = reinterpret_cast<float4*>(lnu + e0 + c);
        dst[0] = make_float4(out[0], out[1], out[2], out[3]);
        dst[1] = make_float4(out[4], out[5], out[6], out[7]);
    }
}

// ---------------------------------------------------------------- K9: §III.D evaluation
// Generating-surface accuracy of one posed depth image against the current beliefs (
// §V; readings R18-R21 in DESIGN.md).  Thread per owned pixel, fp64 (an evaluation kernel,
// not on the BP hot path; decisions taken in the oracle's precision): the ray from the camera
// to 1.5 x the grid diagonal is walked by the same fixed-point DDA until it leaves the grid;
// per cell x = L0 + T 2^-23, softplus(x) = -ln(1 - p), alpha = softplus / res,
// ln omega = ln(alpha) + ln vis at the cell entry, ln vis -= (ell / res) softplus; s* = entry of
// the first maximal omega; vis_inf, s_inf at the exit.  Accurate: vis_inf > thr ? Z > s_inf :
// mode 0: |Z - s*| <= k sigma(Z) (§V), mode 1: Z inside the argmax voxel (§III.D).  cls: -1
// invalid pixel, 0 / 1.
__device__ __forceinline__ double softplus_d(double x) { return x > 0.0 ? x + log1p(exp(-x)) : log1p(exp(x)); }

__global__ void __launch_bounds__(128) eval_kernel(FrameDesc f, GridDesc g, NoiseDesc n, const float* __restrict__ depth,
                                                   const long long* __restrict__ T, double L0, double k_sigma,
                                                   double vis_thr, int mode, double L_eval, int8_t* cls,
                                                   unsigned long long* counts) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long n_pix = (long long)f.rows_owned * f.W;
    int r = -2;
    if (i < n_pix) {
        int u, v;
        owned_pixel(f, i, u, v);
        const double z = (double)depth[(long long)v * f.W + u];
        r = -1;
        if (z > 0.0 && !isinf(z)) {
            const double xc = __ddiv_rn(__dsub_rn((double)u, f.cx), f.fx);
            const double yc = __ddiv_rn(__dsub_rn((double)v, f.cy), f.fy);
            const double rho = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(xc, xc), __dmul_rn(yc, yc)), 1.0));
            const double Z = __dmul_rn(z, rho);
            const double l_over_rho = __ddiv_rn(L_eval, rho);
            const double org[3] = {g.ox, g.oy, g.oz};
            Segment sg;
            for (int k = 0; k < 3; ++k) {
                const double d = __dadd_rn(__dadd_rn(__dmul_rn(f.R[3 * k], xc), __dmul_rn(f.R[3 * k + 1], yc)), f.R[3 * k + 2]);
                const double end = __dadd_rn(f.C[k], __dmul_rn(l_over_rho, d));
                sg.g0[k] = __double2ll_rn(__dmul_rn(__ddiv_rn(__dsub_rn(f.C[k], org[k]), g.res), 65536.0));
                sg.g1[k] = __double2ll_rn(__dmul_rn(__ddiv_rn(__dsub_rn(end, org[k]), g.res), 65536.0));
            }
            Walker w;
            w.start(sg);
            double lvis = 0.0, best = -INFINITY, s_star = -1.0, s_star_out = -1.0, s_inf = 0.0;
            while (w.inside(g)) {
                unsigned na, da;
                bool last;
                const int a = w.earliest(na, da);
                const double t_out = crossing_t(w, a, na, da, last);
                const double x = L0 + (double)__ldg(T + voxel_slot(g, w.c0, w.c1, w.c2)) * kQInvD;
                const double sp = softplus_d(x);
                const double lom = __dadd_rn(sp > 0.0 ? log(__ddiv_rn(sp, g.res)) : -INFINITY, lvis);
                if (lom > best) {
                    best = lom;
                    s_star = w.t_in * L_eval;
                    s_star_out = t_out * L_eval;
                }
                // explicit roundings (no FMA contraction): the oracle's op order, R18
                lvis = __dsub_rn(lvis, __dmul_rn(__ddiv_rn(__dmul_rn(__dsub_rn(t_out, w.t_in), L_eval), g.res), sp));
                s_inf = t_out * L_eval;
                if (last) break;
                w.advance(na, da);
                w.t_in = t_out;
            }
            const double vis_inf = exp(lvis);
            const double sig = pixel_sigma(n, u, v, Z);
            if (vis_inf > vis_thr)
                r = Z > s_inf;
            else if (mode == 0)
                r = fabs(__dsub_rn(Z, s_star)) <= __dmul_rn(k_sigma, sig);
            else
                r = Z >= s_star && Z <= s_star_out;
        }
        cls[(long long)v * f.W + u] = (int8_t)r;
    }
    const unsigned valid = __ballot_sync(0xffffffffu, r >= 0), acc = __ballot_sync(0xffffffffu, r == 1);
    if ((threadIdx.x & 31) == 0) {
        if (valid) atomicAdd(&counts[0], (unsigned long long)__popc(valid));
        if (acc) atomicAdd(&counts[1], (unsigned long long)__popc(acc));
    }
}

// ---------------------------------------------------------------- K4
// Thread per ray walking its incidences in lock step with its warp neighbours; incidences
// that land in the same voxel at the same step share one cursor atomic.
__global__ void __launch_bounds__(256) transpose_fill_kernel(long long n_rays, const long long* __restrict__ row_ptr,
                                                             const RayInfo* __restrict__ info,
                                                             const int32_t* __restrict__ vid,
                                                             const long long* __restrict__ col_ptr,
                                                             int32_t* cursor, int32_t* tr) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    long long e = 0, e1 = 0;
    if (r < n_rays) {
        e = row_ptr[r];
        e1 = e + info[r].n;
    }
    for (;;) {
        const bool alive = e < e1;
        const unsigned am = __ballot_sync(kFull, alive);
        if (am == 0) break;
        if (alive) {
            const int v = vid[e];
            const unsigned peers = __match_any_sync(am, v);
            const int leader = __ffs(peers) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&cursor[v], __popc(peers));
            base = __shfl_sync(peers, base, leader);
            const int rank = __popc(peers & ((1u << lane) - 1u));
            tr[col_ptr[v] + base + rank] = (int32_t)e;
            ++e;
        }
    }
}

__global__ void item_counts_kernel(long long V, const int32_t* __restrict__ cnt, int32_t* n_items, int chunk) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < V) n_items[v] = (cnt[v] + chunk - 1) / chunk;
}

// K4b: tile-run transpose.  Thread per ray walking its incidences; a run ends where the tile
// changes (a ray crosses a convex tile once), after kRunMax incidences, or before a step that is
// not a single-axis unit step (an exact DDA tie).  run_count counts runs per tile, run_fill
// writes them (order inside a tile is irrelevant: K6 sums integers).
// Voxel degrees (per belief slot), only for the per-voxel transpose and the active-voxel count.
__global__ void __launch_bounds__(256) vox_hist_kernel(long long n_rays, const long long* __restrict__ row_ptr,
                                                       const RayInfo* __restrict__ info,
                                                       const int32_t* __restrict__ vid, int32_t* vox_count) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    long long e = 0, e1 = 0;
    if (r < n_rays) {
        e = row_ptr[r];
        e1 = e + info[r].n;
    }
    for (;;) {
        const bool alive = e < e1;
        const unsigned am = __ballot_sync(kFull, alive);
        if (am == 0) break;
        if (alive) {
            const int vx = vid[e];
            const unsigned peers = __match_any_sync(am, vx);
            if (lane == __ffs(peers) - 1) atomicAdd(&vox_count[vx], __popc(peers));
            ++e;
        }
    }
}

__global__ void __launch_bounds__(256) run_fill_kernel(long long n_rays, const long long* __restrict__ row_ptr,
                                                       const RayInfo* __restrict__ info,
                                                       const int32_t* __restrict__ vid,
                                                       const long long* __restrict__ tile_ptr, int32_t* cursor,
                                                       int bucket_stride, Run* runs) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    long long e = 0, e1 = 0;
    int bucket0 = 0;
    if (r < n_rays) {
        e = row_ptr[r];
        const RayInfo ri = info[r];
        e1 = e + ri.n;
        bucket0 = ri.frame * bucket_stride;
    }
    bool alive = e < e1;
    RunBuilder rb;
    int4 buf{0, 0, 0, 0};  // vid[e & ~3 .. +4): 16-byte loads (segments are 8-aligned)
    for (;;) {
        const unsigned am = __ballot_sync(kFull, alive);
        if (am == 0) break;
        if (alive) {
            const bool at_end = e == e1;
            int b = -1, l = 0;
            if (!at_end) {
                if ((e & 3) == 0) buf = __ldg(reinterpret_cast<const int4*>(vid + e));
                const int k = (int)(e & 3);
                const int v = k == 0 ? buf.x : (k == 1 ? buf.y : (k == 2 ? buf.z : buf.w));
                b = v >> kTileShift;
                l = v & (kTileSlots - 1);
            }
            RunBuilder nb = rb;
            const bool ext = !at_end && nb.extend(b, l);
            const bool emit = rb.tile >= 0 && !ext;  // the current run ends before e
            const unsigned em = __ballot_sync(am, emit);
            if (emit) {  // (runs == nullptr: only count the runs per bucket, into cursor)
                const int cur = bucket0 + rb.tile;
                const unsigned peers = __match_any_sync(em, cur);
                const int leader = __ffs(peers) - 1;
                int base = 0;
                if (lane == leader) base = atomicAdd(&cursor[cur], __popc(peers));
                base = __shfl_sync(peers, base, leader);
                const int rank = __popc(peers & ((1u << lane) - 1u));
                if (runs) runs[tile_ptr[cur] + base + rank] = rb.make();
            }
            if (at_end) {
                alive = false;
            } else {
                if (ext) {
                    rb = nb;
                } else {
                    rb.begin(b, l, e);
                }
                ++e;
            }
        }
    }
}

// Sparse bricks, keyframes added after the graph was used (reading R24): every ray is walked again
// against the grown allocation; its old incidences are a subsequence of the new ones (cells of
// newly allocated bricks are inserted, nothing is removed), in the same order along the ray.
// Thread per old ray: each new incidence takes the message of the same voxel in the old list,
// or 0 (a new incidence).
__global__ void __launch_bounds__(256) lambda_merge_kernel(long long n_rays, const long long* __restrict__ rp_old,
                                                           const RayInfo* __restrict__ ri_old,
                                                           const int32_t* __restrict__ vid_old,
                                                           const int32_t* __restrict__ lam_old,
                                                           const long long* __restrict__ rp_new,
                                                           const RayInfo* __restrict__ ri_new,
                                                           const int32_t* __restrict__ vid_new, int32_t* lam_new,
                                                           unsigned long long* lost) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays) return;
    const long long eo = rp_old[r], en = rp_new[r];
    const int no = ri_old[r].n, nn = ri_new[r].n;
    int j = 0;
    for (int k = 0; k < nn; ++k) {
        const int v = vid_new[en + k];
        int q = 0;
        if (j < no && vid_old[eo + j] == v) q = lam_old[eo + j++];
        lam_new[en + k] = q;
    }
    if (j < no) atomicAdd(lost, (unsigned long long)(no - j));  // cannot happen (allocation only grows)
}

// Matrix-free (K12): the first cell of every K5 chunk of a ray (its class's K, 8 for long rays),
// from the voxel slots of its first walk.  Thread per ray.
__global__ void __launch_bounds__(256) ck_extract_kernel(long long n, const long long* __restrict__ row_ptr,
                                                         const RayInfo* __restrict__ info,
                                                         const int32_t* __restrict__ vid, int32_t* ck, RaySeg* seg) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    // the segment's per-axis reciprocals RN(1 / |dg|), as Walker::start computes them (written
    // here rather than by the fill, whose walk is register-bound)
    RaySeg& sr = seg[r];
    sr.y[0] = __drcp_rn((double)(sr.dg[0] ? (unsigned)abs(sr.dg[0]) : 1u));
    sr.y[1] = __drcp_rn((double)(sr.dg[1] ? (unsigned)abs(sr.dg[1]) : 1u));
    sr.y[2] = __drcp_rn((double)(sr.dg[2] ? (unsigned)abs(sr.dg[2]) : 1u));
    const int nr = info[r].n;
    if (nr <= 0) return;
    const int cls = ray_class(nr);
    const int K = cls < kNumShort ? class_K(cls) : 8;
    const long long e0 = row_ptr[r];
    for (int c = 0; c * K < nr; ++c) ck[(e0 >> 2) + c] = vid[e0 + (long long)c * K];
}

// The runs the DDA fills emitted (unsorted, with their bucket keys) placed by bucket: the
// tile-run transpose without re-reading vid.  Thread per run, 1024 per CTA.  A warp's runs of one
// bucket are counted together (match_any), the CTA's counts per bucket are summed in a shared
// table, and each (CTA, bucket) takes its range with ONE cursor atomic: with few buckets (64 tiles
// at frames30) per-warp atomics had queued ~30 000 deep on each cursor (1.5 ms for 49 M runs).
// The order of a bucket's runs is not fixed (K6 sums exactly in any order).
constexpr int kBucketThreads = 1024;
__global__ void __launch_bounds__(kBucketThreads) run_bucket_kernel(long long n, const Run* __restrict__ src,
                                                                    const int32_t* __restrict__ keys,
                                                                    const long long* __restrict__ tile_ptr,
                                                                    int32_t* cursor, Run* dst) {
    __shared__ int s_key[kBucketThreads], s_cnt[kBucketThreads], s_base[kBucketThreads];
    s_key[threadIdx.x] = -1;
    s_cnt[threadIdx.x] = 0;
    __syncthreads();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int key = i < n ? __ldg(keys + i) : -1;  // -1: an unused slot of a warp's block
    const bool act = key >= 0;
    const unsigned am = __ballot_sync(kFull, act);
    unsigned peers = 0;
    int leader = 0, slot = 0, off = 0;
    if (act) {
        peers = __match_any_sync(am, key);
        leader = __ffs(peers) - 1;
        if (lane == leader) {  // open addressing: at most 1024 distinct keys per CTA, never full
            int h = (int)((unsigned)key * 2654435761u >> 22);
            for (;;) {
                const int prev = atomicCAS(&s_key[h], -1, key);
                if (prev == -1 || prev == key) break;
                h = (h + 1) & (kBucketThreads - 1);
            }
            slot = h;
            off = atomicAdd(&s_cnt[h], __popc(peers));
        }
        slot = __shfl_sync(peers, slot, leader);
        off = __shfl_sync(peers, off, leader);
    }
    __syncthreads();
    if (s_key[threadIdx.x] >= 0) s_base[threadIdx.x] = atomicAdd(&cursor[s_key[threadIdx.x]], s_cnt[threadIdx.x]);
    __syncthreads();
    if (!act) return;
    const long long pos = tile_ptr[key] + s_base[slot] + off + __popc(peers & ((1u << lane) - 1u));
    MRF_ASSERT(pos < tile_ptr[key + 1]);
    dst[pos] = src[i];
}

__global__ void item_fill_kernel(long long V, const int32_t* __restrict__ n_items,
                                 const long long* __restrict__ item_ptr, int2* items) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    const long long b = item_ptr[v];
    for (int j = 0; j < n_items[v]; ++j) items[b + j] = make_int2((int)v, j);
}

__global__ void active_flags_kernel(long long V, const int32_t* __restrict__ cnt, int32_t* flags) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v < V) flags[v] = cnt[v] > 0 ? 1 : 0;
}

// K5 class lists (counting sort by class, warp-aggregated atomics)
__global__ void class_count_kernel(long long n_rays, const RayInfo* __restrict__ info, unsigned long long* counts) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int k = r < n_rays ? ray_class(info[r].n) : -1;
    const unsigned peers = __match_any_sync(kFull, k);
    if (k >= 0 && lane == __ffs(peers) - 1) atomicAdd(&counts[k], (unsigned long long)__popc(peers));
}
__global__ void class_scatter_kernel(long long n_rays, const RayInfo* __restrict__ info, ClassOffsets off,
                                     unsigned long long* cursor, int32_t* out) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int k = r < n_rays ? ray_class(info[r].n) : -1;
    const unsigned peers = __match_any_sync(kFull, k);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (k >= 0 && lane == leader) base = atomicAdd(&cursor[k], (unsigned long long)__popc(peers));
    base = __shfl_sync(kFull, base, leader);
    if (k >= 0) out[off.off[k] + (long long)base + __popc(peers & ((1u << lane) - 1u))] = (int32_t)r;
}

// Matrix-free class lists (NEXT #1): key = (frame / fpc) * kNumClasses + class, so that each
// chunk of fpc frames has its own class lists (off[key] from the host scan of counts[key]).
__global__ void class_count_mf_kernel(long long n_rays, const RayInfo* __restrict__ info, int fpc,
                                      unsigned long long* counts) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int k = -1;
    if (r < n_rays) {
        const RayInfo ri = info[r];
        const int cl = ray_class(ri.n);
        k = cl < 0 ? -1 : (ri.frame / fpc) * kNumClasses + cl;
    }
    const unsigned peers = __match_any_sync(kFull, k);
    if (k >= 0 && lane == __ffs(peers) - 1) atomicAdd(&counts[k], (unsigned long long)__popc(peers));
}
__global__ void class_scatter_mf_kernel(long long n_rays, const RayInfo* __restrict__ info, int fpc,
                                        const long long* __restrict__ off, unsigned long long* cursor, int32_t* out) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int k = -1;
    if (r < n_rays) {
        const RayInfo ri = info[r];
        const int cl = ray_class(ri.n);
        k = cl < 0 ? -1 : (ri.frame / fpc) * kNumClasses + cl;
    }
    const unsigned peers = __match_any_sync(kFull, k);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (k >= 0 && lane == leader) base = atomicAdd(&cursor[k], (unsigned long long)__popc(peers));
    base = __shfl_sync(kFull, base, leader);
    if (k >= 0) out[off[k] + (long long)base + __popc(peers & ((1u << lane) - 1u))] = (int32_t)r;
}

__global__ void compact_kernel(long long n, const int32_t* __restrict__ flags, const long long* __restrict__ pos,
                               int32_t* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flags[i]) out[pos[i]] = (int32_t)i;
}

__global__ void span_max_kernel(long long n, const int32_t* __restrict__ rays, const RayInfo* __restrict__ info,
                                unsigned long long* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long m = 0;
    if (i < n) m = (unsigned long long)info[rays[i]].n;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(kFull, m, o);
        m = x > m ? x : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// Staged-K5 stage list.  Ray r is "short" when 0 <= n <= kShortMax.  A short ray opens a stage
// when the previous ray is long, or starts in another kStageCap-slot window, or lies in another
// kStageMaxRays block of ray indices.  flags[r] = opens a stage.
__device__ __forceinline__ bool ray_short(const RayInfo* info, long long r) { return info[r].n <= kShortMax; }
__device__ __forceinline__ bool opens_stage(long long r, const long long* row_ptr, const RayInfo* info) {
    if (!ray_short(info, r)) return false;
    if (r == 0) return true;
    return !ray_short(info, r - 1) || (row_ptr[r] / kStageCap) != (row_ptr[r - 1] / kStageCap) ||
           (r / kStageMaxRays) != ((r - 1) / kStageMaxRays);
}

__global__ void stage_flags_kernel(long long n_rays, const long long* __restrict__ row_ptr,
                                   const RayInfo* __restrict__ info, int32_t* flags) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n_rays) flags[r] = opens_stage(r, row_ptr, info) ? 1 : 0;
}

// pos = exclusive scan of flags (n_rays + 1 entries).  Stage of short ray r = pos[r + 1] - 1.
__global__ void stage_fill_kernel(long long n_rays, const long long* __restrict__ row_ptr,
                                  const RayInfo* __restrict__ info, const int32_t* __restrict__ flags,
                                  const long long* __restrict__ pos, Stage* stages) {
    const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rays || !ray_short(info, r)) return;
    const long long sid = pos[r + 1] - 1;
    if (flags[r]) {
        stages[sid].r0 = (int)r;
        stages[sid].s0 = row_ptr[r];
    }
    if (r + 1 == n_rays || flags[r + 1] || !ray_short(info, r + 1)) {
        stages[sid].r1 = (int)(r + 1);
        stages[sid].s1 = row_ptr[r + 1];
    }
}

inline unsigned blocks_for(long long n, int b) { return (unsigned)((n + b - 1) / b); }

// mrf_export_rays: per selected ray its padded start and record, then its incidences gathered
// into contiguous staging arrays (warp per ray) -- a few large copies instead of per-ray ones
__global__ void ray_select_kernel(long long n, const long long* __restrict__ rid, const long long* __restrict__ row_ptr,
                                  const RayInfo* __restrict__ info, long long* e0, RayInfo* out) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const long long r = rid[k];
    e0[k] = row_ptr[r];
    out[k] = info[r];
}
__global__ void ray_gather_kernel(long long n, const long long* __restrict__ e0, const long long* __restrict__ off,
                                  const int32_t* __restrict__ vid, const int16_t* __restrict__ off_q,
                                  const int32_t* __restrict__ lam, int32_t* ovid, int16_t* ooff, int32_t* olam) {
    const long long k = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (k >= n) return;
    const int lane = threadIdx.x & 31;
    const long long a = e0[k], o = off[k], len = off[k + 1] - off[k];
    for (long long j = lane; j < len; j += 32) {
        if (ovid) ovid[o + j] = vid[a + j];
        if (ooff) ooff[o + j] = off_q[a + j];
        if (olam) olam[o + j] = lam[a + j];
    }
}

}  // namespace

void launch_stage_flags(long long n_rays, const long long* row_ptr, const RayInfo* info, int32_t* flags,
                        cudaStream_t s) {
    if (n_rays == 0) return;
    stage_flags_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, row_ptr, info, flags);
}

void launch_stage_fill(long long n_rays, const long long* row_ptr, const RayInfo* info, const int32_t* flags,
                       const long long* pos, Stage* stages, cudaStream_t s) {
    if (n_rays == 0) return;
    stage_fill_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, row_ptr, info, flags, pos, stages);
}

void launch_raygen_count(const FrameDesc& f, const GridDesc& g, const NoiseDesc& n, const float* depth,
                         int32_t* n_r, int8_t* status, RayInfo* ray_z, unsigned long long* counters,
                         cudaStream_t s) {
    const long long n_pix = (long long)f.rows_owned * f.W;
    if (n_pix == 0) return;
    raygen_count_kernel<<<blocks_for(n_pix, 128), 128, 0, s>>>(f, g, n, depth, n_r, status, ray_z, counters);
}

void launch_raygen_count_batch(const FrameDesc* frames, const int* cta0, int n_frames, int n_ctas, const GridDesc& g,
                               const NoiseDesc& n, const float* depth_all, int32_t* n_r, int8_t* status, RayInfo* ray_z,
                               unsigned long long* counters, cudaStream_t s) {
    if (n_ctas == 0) return;
    raygen_count_batch_kernel<<<n_ctas, 128, 0, s>>>(frames, cta0, n_frames, g, n, depth_all, n_r, status, ray_z,
                                                     counters);
}

void launch_brick_alloc(const FrameDesc& f, const GridDesc& g, const NoiseDesc& n, const float* depth, uint8_t* mask,
                        cudaStream_t s) {
    const long long np = (long long)f.W * f.H;
    if (np == 0) return;
    brick_alloc_kernel<<<blocks_for(np, 256), 256, 0, s>>>(f, g, n, depth, mask);
}

void launch_dda_fill(const FrameDesc* frames, const int* cta0, int n_frames, int n_ctas, long long r0,
                     long long n_rays, const GridDesc& g, const NoiseDesc& n, const MsgParams& mp,
                     const float* depth_all, const long long* row_ptr, RayInfo* ray_z, int32_t* vid,
                     int16_t* off_q, float* lnu, int32_t* tile_runs, unsigned long long* counters,
                     const RunSink& sink, RaySeg* seg, unsigned long long* class_counts, int32_t* lam0,
                     cudaStream_t s) {
    if (n_ctas > 0) {
#define MRF_FILL_LAUNCH(SP, RU, CO)                                                                                 \
    dda_fill_kernel<SP, RU, CO><<<n_ctas, kFillThreads, 0, s>>>(frames, cta0, n_frames, g, n, depth_all, row_ptr, vid, \
                                                                off_q, tile_runs, ray_z, counters, mp, lnu, sink, seg, \
                                                                class_counts, lam0)
        // tile_runs == nullptr without a sink: no run tracking at all (matrix-free re-walks, K6b)
        if (g.bmask) {
            if (sink.runs) MRF_FILL_LAUNCH(true, true, true);
            else if (tile_runs) MRF_FILL_LAUNCH(true, false, true);
            else MRF_FILL_LAUNCH(true, false, false);
        } else {
            if (sink.runs) MRF_FILL_LAUNCH(false, true, true);
            else if (tile_runs) MRF_FILL_LAUNCH(false, false, true);
            else MRF_FILL_LAUNCH(false, false, false);
        }
#undef MRF_FILL_LAUNCH
    }
    if ((!MRF_FILL_LNU || mp.pcoef) && n_rays > 0)
        lnu_fill_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(r0, n_rays, mp, row_ptr, ray_z, off_q, lnu);
}

void launch_transpose_fill(long long n_rays, const long long* row_ptr, const RayInfo* info, const int32_t* vid,
                           const long long* col_ptr, int32_t* cursor, int32_t* tr, cudaStream_t s) {
    if (n_rays == 0) return;
    transpose_fill_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, row_ptr, info, vid, col_ptr, cursor, tr);
}

void launch_item_counts(long long V, const int32_t* vox_count, int32_t* n_items, int chunk, cudaStream_t s) {
    item_counts_kernel<<<blocks_for(V, 256), 256, 0, s>>>(V, vox_count, n_items, chunk);
}

void launch_eval(const FrameDesc& f, const GridDesc& g, const NoiseDesc& n, const float* depth, const long long* T,
                 double L0, double k_sigma, double vis_thr, int mode, double L_eval, int8_t* cls,
                 unsigned long long* counts, cudaStream_t s) {
    const long long n_pix = (long long)f.rows_owned * f.W;
    if (n_pix == 0) return;
    eval_kernel<<<blocks_for(n_pix, 128), 128, 0, s>>>(f, g, n, depth, T, L0, k_sigma, vis_thr, mode, L_eval, cls,
                                                       counts);
}

void launch_vox_hist(long long n_rays, const long long* row_ptr, const RayInfo* info, const int32_t* vid,
                     int32_t* vox_count, cudaStream_t s) {
    if (n_rays == 0) return;
    vox_hist_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, row_ptr, info, vid, vox_count);
}

void launch_run_fill(long long n_rays, const long long* row_ptr, const RayInfo* info, const int32_t* vid,
                     const long long* tile_ptr, int32_t* cursor, int bucket_stride, Run* runs, cudaStream_t s) {
    if (n_rays == 0) return;
    run_fill_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, row_ptr, info, vid, tile_ptr, cursor,
                                                            bucket_stride, runs);
}

void launch_item_fill(long long V, const int32_t* n_items, const long long* item_ptr, int2* items,
                      cudaStream_t s) {
    item_fill_kernel<<<blocks_for(V, 256), 256, 0, s>>>(V, n_items, item_ptr, items);
}

void launch_active_flags(long long V, const int32_t* vox_count, int32_t* flags, cudaStream_t s) {
    active_flags_kernel<<<blocks_for(V, 256), 256, 0, s>>>(V, vox_count, flags);
}

void launch_class_count(long long n_rays, const RayInfo* info, unsigned long long* counts, cudaStream_t s) {
    if (n_rays == 0) return;
    class_count_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, info, counts);
}

void launch_class_scatter(long long n_rays, const RayInfo* info, const ClassOffsets& off, unsigned long long* cursor,
                          int32_t* out, cudaStream_t s) {
    if (n_rays == 0) return;
    class_scatter_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, info, off, cursor, out);
}

void launch_class_count_mf(long long n_rays, const RayInfo* info, int fpc, unsigned long long* counts, cudaStream_t s) {
    if (n_rays == 0) return;
    class_count_mf_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, info, fpc, counts);
}

void launch_class_scatter_mf(long long n_rays, const RayInfo* info, int fpc, const long long* off,
                             unsigned long long* cursor, int32_t* out, cudaStream_t s) {
    if (n_rays == 0) return;
    class_scatter_mf_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, info, fpc, off, cursor, out);
}

void launch_compact(long long n, const int32_t* flags, const long long* pos, int32_t* out, cudaStream_t s) {
    if (n == 0) return;
    compact_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, flags, pos, out);
}

void launch_span_max(long long n, const int32_t* rays, const RayInfo* info, unsigned long long* out,
                     cudaStream_t s) {
    if (n == 0) return;
    span_max_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, rays, info, out);
}

void launch_ray_select(long long n, const long long* rid, const long long* row_ptr, const RayInfo* info, long long* e0,
                       RayInfo* out, cudaStream_t s) {
    if (n == 0) return;
    ray_select_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, rid, row_ptr, info, e0, out);
}

void launch_ray_gather(long long n, const long long* e0, const long long* off, const int32_t* vid, const int16_t* off_q,
                       const int32_t* lam, int32_t* ovid, int16_t* ooff, int32_t* olam, cudaStream_t s) {
    if (n == 0) return;
    ray_gather_kernel<<<blocks_for(n * 32, 256), 256, 0, s>>>(n, e0, off, vid, off_q, lam, ovid, ooff, olam);
}

void launch_run_bucket(long long n, const Run* src, const int32_t* keys, const long long* tile_ptr, int32_t* cursor,
                       Run* dst, cudaStream_t s) {
    if (n == 0) return;
    run_bucket_kernel<<<blocks_for(n, kBucketThreads), kBucketThreads, 0, s>>>(n, src, keys, tile_ptr, cursor, dst);
}

void launch_lambda_merge(long long n_rays, const long long* rp_old, const RayInfo* ri_old, const int32_t* vid_old,
                         const int32_t* lam_old, const long long* rp_new, const RayInfo* ri_new, const int32_t* vid_new,
                         int32_t* lam_new, unsigned long long* lost, cudaStream_t s) {
    if (n_rays == 0) return;
    lambda_merge_kernel<<<blocks_for(n_rays, 256), 256, 0, s>>>(n_rays, rp_old, ri_old, vid_old, lam_old, rp_new,
                                                                ri_new, vid_new, lam_new, lost);
}

void launch_ck_extract(long long n, const long long* row_ptr, const RayInfo* info, const int32_t* vid, int32_t* ck,
                       RaySeg* seg,
                       cudaStream_t s) {
    if (n == 0) return;
    ck_extract_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, row_ptr, info, vid, ck, seg);
}

}  // namespace mrf
