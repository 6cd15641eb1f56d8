// internal.cuh -- shared declarations of the CUDA path (sm_100a).  Not part of the ABI.
//
// The product path: mrf_api.cu (host runtime behind include/mrf.h) drives the kernels of
// graph.cu (K1 raygen+DDA count, K3 DDA fill, K4 transpose, work lists), scan.cu (K2) and
// bp.cu (K5 ray messages, K6 voxel reduction, K8 marginals).  Nothing here is shared with
// oracle/ (the fp64 CPU checker), which is written independently from the paper.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace mrf {

// Checked build (MRF_CHECK=1, libmrf_checked.so; SURVEY §4 T8 -- compute-sanitizer is closed on
// this pool): the data-dependent indices of the hot kernels (belief-slot gathers, message slots of
// runs and chunks, accumulator indices, run placement) are bounds-checked on the device; a failed
// check prints the site and traps, which the ABI returns as a sticky MRF_ERR_CUDA.
#ifndef MRF_CHECK
#define MRF_CHECK 0
#endif
#define MRF_ASSERT(cond)                                                                      \
    do {                                                                                      \
        if (MRF_CHECK && !(cond)) {                                                           \
            printf("MRF_CHECK failed: %s at %s:%d (block %d, thread %d)\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                        \
            __trap();                                                                         \
        }                                                                                     \
    } while (0)

// ---- fixed-point conventions (DESIGN.md §Data layout)
constexpr int kFixShift = 16;                 // grid coordinates carry 16 fractional bits
constexpr long long kFixOne = 1LL << kFixShift;
constexpr float kQScale = 8388608.0f;         // messages: int32 q = round(lambda * 2^23)
constexpr float kQInv = 1.0f / 8388608.0f;
constexpr double kQInvD = 1.0 / 8388608.0;
constexpr float kLambdaClip = 256.0f;         // reading R9
constexpr int kPadElems = 64;                 // slack after incidence arrays (aligned over-reads)
constexpr int kSegAlign = 8;                  // ray segments start at multiples of 8 slots (row_ptr += pad8(n))
constexpr int kVoxelChunk = 4096;             // per-voxel K6 work item: <= 4096 transpose entries
// Internal voxel layout: 32 x 32 x 16 tiles (16384 slots), tile-major.  K6 accumulates one tile
// at a time in shared memory, so a tile's slots must fit one CTA (2 x int32 x 16384 = 128 KB).
constexpr int kTileShift = 14;                // slot = tile << 14 | (z&15) << 10 | (y&31) << 5 | (x&31)
constexpr int kTileSlots = 1 << kTileShift;
constexpr int kRunsPerItem = 32768;           // K6 work item: <= 32768 runs of one tile (int32 halves: 32768 x 65535 < 2^31)
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// Dense grid; internally voxels are stored tile-major in 32 x 32 x 16 tiles (the paper's GVDB
// stores 8^3 bricks; the larger tile here is the unit of the K6 shared-memory reduction):
// slot = tile * 16384 + (x&31) + 32 (y&31) + 1024 (z&15), tile = tx + ntx (ty + nty tz).
struct GridDesc {
    int nx, ny, nz;
    int ntx, nty, ntz;
    double res, ox, oy, oz;
    // sparse-brick map (NEXT #4, reading R23): a cell is part of the map iff
    // bmask[(cx >> bshift) + nbx ((cy >> bshift) + nby (cz >> bshift))] != 0; nullptr = dense
    const uint8_t* bmask;
    int bshift, nbx, nby;
};
__host__ __device__ __forceinline__ bool cell_in_map(const GridDesc& g, int x, int y, int z) {
    return !g.bmask ||
           g.bmask[(x >> g.bshift) + g.nbx * ((y >> g.bshift) + g.nby * (long long)(z >> g.bshift))] != 0;
}

__host__ __device__ __forceinline__ int voxel_slot(const GridDesc& g, int x, int y, int z) {
    return ((((z >> 4) * g.nty + (y >> 5)) * g.ntx + (x >> 5)) << kTileShift) | ((z & 15) << 10) | ((y & 31) << 5) |
           (x & 31);
}
__host__ __device__ __forceinline__ void slot_xyz(const GridDesc& g, long long s, int& x, int& y, int& z) {
    const long long t = s >> kTileShift;
    const int l = (int)(s & (kTileSlots - 1));
    x = (int)(t % g.ntx) * 32 + (l & 31);
    y = (int)((t / g.ntx) % g.nty) * 32 + ((l >> 5) & 31);
    z = (int)(t / ((long long)g.ntx * g.nty)) * 16 + (l >> 10);
}

// A run: up to kRunMax contiguous incidences [e, e + n) of one ray inside one tile, stored with
// the DDA steps between them so that K6 never reads vid.  Step i (from element i to i+1) is a
// unit step along x (bit i of mx), y (bit i of my) or z (neither); element k then sits at the
// in-tile slot  slot0 + sx cx + 32 sy cy + 1024 sz (k - cx - cy),  cx = popc(mx & (2^k - 1)),
// cy likewise.  A step along several axes at once (an exact DDA tie) starts a new run.
// meta: slot0 (bits 0-13) | (n-1) << 14 | negative-direction flags of x, y, z << 20.
constexpr int kRunMax = 32;
struct Run {
    unsigned e;                 // first incidence slot (this rank holds < 2^31 slots)
    unsigned meta;
    unsigned mx, my;
};

// Where the DDA fill puts the tile runs it builds (K4b without a vid re-read): appended, unsorted,
// to runs[0 .. cap) with their bucket keys.  Each warp reserves blocks of kSinkBlock slots from a
// global cursor (*count, the slots reserved so far) and fills them in order; the unused tail of a
// block keeps key -1 (the keys are preset to -1) and is skipped by the bucket pass.  Slots at or
// past cap are dropped and the caller falls back to the vid re-read.  runs == nullptr: no emission.
constexpr int kSinkBlock = 128;
struct RunSink {
    Run* runs;
    int32_t* keys;
    unsigned long long* count;
    long long cap;
#ifdef __CUDACC__
    // Called by all 32 lanes (wbase / wleft: the warp's current block, warp-uniform registers);
    // lanes with `has` set append (run, key).
    __device__ __forceinline__ void emit(bool has, const Run& r, int key, int lane, unsigned long long& wbase,
                                         int& wleft) const {
        const unsigned em = __ballot_sync(0xffffffffu, has);
        if (!em) return;
        const int k = __popc(em);
        if (k > wleft) {  // a new block (the rest of the old one stays unused, key -1)
            unsigned long long b = 0;
            if (lane == 0) b = atomicAdd(count, (unsigned long long)kSinkBlock);
            wbase = __shfl_sync(0xffffffffu, b, 0);
            wleft = kSinkBlock;
        }
        if (has) {
            const long long pos = (long long)wbase + __popc(em & ((1u << lane) - 1u));
            if (pos < cap) {
                runs[pos] = r;
                keys[pos] = key;
            }
        }
        wbase += (unsigned long long)k;
        wleft -= k;
    }
#endif
};

struct NoiseDesc {
    double z_lo, z_hi, off_lo, off_hi, margin_min, margin_k, c0, c1, c2;
    int n_z, n_off;
    // learnt per-patch noise model (NEXT #4 option, reading R25; mrf_set_patch_noise): the
    // coefficients [patch][6] = (b0, b1, b2, s0, s1, s2) of patch (u / ppx) + pnx (v / ppx); the
    // pixel's (s0, s1, s2) replace (c0, c1, c2) in its traversal margin.  nullptr: the global model.
    const double* pcoef;
    int ppx, pnx;
};
__host__ __device__ __forceinline__ int pixel_patch(const NoiseDesc& n, int u, int v) {
    return (v / n.ppx) * n.pnx + u / n.ppx;
}

struct FrameDesc {
    double fx, fy, cx, cy;
    double R[9];
    double C[3];
    int W, H, rank, world;
    int rows_owned;           // number of pixel rows v with v % world == rank
    long long ray_base;       // index of this frame's first ray
    long long depth_off;      // offset of the frame's depth image in the pending-depth buffer
    int index;                // frame index in the ctx
    int skip_count;           // K1 without the walk count (sparse bricks before the final allocation)
    int bucket_stride;        // tile-run bucket of a run in tile t: index * bucket_stride + t
};

// Per-ray record: LUT row iz (<= n_z-2) and weight wz in [0,1] of the measured range (per-patch
// noise, R25: iz = the pixel's patch, wz = the range Z), and the number of incidences n.  Ray segments start at multiples of 8 in the incidence arrays
// (row_ptr advances by pad8(n)), so per-lane chunks are relative to the ray start, 16-byte
// aligned, and a ray's arithmetic never depends on where (or on which rank) it is stored.
struct RayInfo {
    int iz;
    float wz;
    int n;
    int frame;  // index of the ray's frame in the ctx (keyframe-average mode)
};

// K5 parameters (natural logs).
struct MsgParams {
    const float2* lutp;       // pair table [n_z][n_off-1] of (L[i][j], L[i][j+1]): the input log nu, exactly
    int n_offm1;              // n_off - 1
    float s_off, b_off;       // fo = off_q * s_off + b_off
    float fo_max;             // n_off - 1
    float L0;                 // prior log-odds ln(gamma / (1 - gamma))
    // keyframe-average mode (reading R22): the cavity excludes the ray's keyframe average
    // qbar[frame * qbar_vi + v] instead of the ray's own message; nullptr in per-ray mode
    const int32_t* qbar;
    long long qbar_vi;
    // checked build: the message slots [0, chk_lam) and belief slots [0, chk_vi) that exist
    long long chk_lam, chk_vi;
    // per-patch noise (R25): per patch (b0, b1, b2, 0) and (s0, s1, s2, sigma_min) in fp32; a ray's
    // RayInfo then carries iz = its patch and wz = its range Z.  nullptr: the LUT.
    const float4* pcoef;
};

// log nu at (measured range row iz + wz, quantised offset off_q): bilinear interpolation of the
// input table in fp32, bin-centre coordinates clamped to the edge centres.
// MRF_FILL_LNU = 1: the DDA fill interpolates log nu as it flushes each 8-slot chunk; 0: a separate
// pass (lnu_fill_kernel) re-reads off_q.
#ifndef MRF_FILL_LNU
#define MRF_FILL_LNU 1
#endif
// Evaluated once per incidence by the DDA fill; K5 reads the result, stored in K5's working units:
// MRF_K5_LOG2 = 1 (default) carries every log-quantity of K5 in base 2 (bp.cu), so the fill stores
// log2 nu = ln nu * log2(e) and K5 uses it without a scaling multiply.
#ifndef MRF_K5_LOG2
#define MRF_K5_LOG2 1
#endif
constexpr float kLnuScale = MRF_K5_LOG2 ? 1.4426950408889634f : 1.f;
// Split in two so that a caller can issue the table loads one step before it needs them.
struct LutFetch {
    float wo;
    float2 ta, tb;
};
__device__ __forceinline__ LutFetch lut_fetch(const MsgParams& mp, int iz, int off) {
    float fo = fmaf((float)off, mp.s_off, mp.b_off);
    fo = fminf(fmaxf(fo, 0.f), mp.fo_max);
    const int io = min((int)fo, mp.n_offm1 - 1);
    const float2* rowA = mp.lutp + (long long)iz * mp.n_offm1;
    return LutFetch{fo - (float)io, __ldg(rowA + io), __ldg(rowA + mp.n_offm1 + io)};
}
__device__ __forceinline__ float lut_finish(const LutFetch& f, float wz) {
    const float ra = fmaf(f.wo, f.ta.y - f.ta.x, f.ta.x);
    const float rb = fmaf(f.wo, f.tb.y - f.tb.x, f.tb.x);
    return fmaf(wz, rb - ra, ra) * kLnuScale;
}

// log nu of the per-patch model (reading R25) in K5's units: the measurement Z is
// Gaussian around the bias-predicted mean d + b(d) with sigma s(d), d = Z + off_q 2^-15 the voxel
// depth (B3's span midpoint): ln nu = -t^2 / 2 - ln s - ln(2 pi) / 2, t = (Z - d - b) / s =
// -(off_q 2^-15 + b) / s.  fp32 (the LUT path's precision).
__device__ __forceinline__ float patch_lnu(const MsgParams& mp, int patch, float Z, int off) {
    const float4 b = __ldg(mp.pcoef + 2 * patch), sc = __ldg(mp.pcoef + 2 * patch + 1);
    const float o = (float)off * (1.f / 32768.f);
    const float d = Z + o;
    const float bias = fmaf(b.z * d, d, fmaf(b.y, d, b.x));
    const float sg = fmaxf(fmaf(sc.z * d, d, fmaf(sc.y, d, sc.x)), sc.w);
    const float t = (o + bias) / sg;
    return (fmaf(-0.5f * t, t, -logf(sg)) - 0.91893853320467274f) * kLnuScale;
}

struct RaySeg;  // walk.cuh

// ---- launchers (all asynchronous on `s`)
// K1: per owned pixel -> status, pad8(upper bound of the walk's length) (scan input), RayInfo
// (n = 0); counters[0] += invalid, counters[1] += dropped
void launch_raygen_count(const FrameDesc& f, const GridDesc& g, const NoiseDesc& n, const float* depth,
                         int32_t* n_r, int8_t* status, RayInfo* ray_z, unsigned long long* counters,
                         cudaStream_t s);
// the same for several frames in one launch (frames[k] owns the CTAs [cta0[k], cta0[k+1]) of 128
// pixels, its depth at depth_all + frames[k].depth_off)
void launch_raygen_count_batch(const FrameDesc* frames, const int* cta0, int n_frames, int n_ctas, const GridDesc& g,
                               const NoiseDesc& n, const float* depth_all, int32_t* n_r, int8_t* status, RayInfo* ray_z,
                               unsigned long long* counters, cudaStream_t s);
// (class_counts, nullable: += rays per K5 length class [kNumClasses], max= longest ray at
// [kNumClasses]; lam0, nullable: zeroes the messages of the walked slots)
// K3: the walk of every pending frame (device FrameDesc array, frame k owning the CTAs
// [cta0[k], cta0[k+1]) of kFillThreads pixels), writing vid / off_q at row_ptr offsets and
// counting the tile runs (K4b) per tile; then log nu per incidence of the rays [r0, r0 + n_rays)
// (RayInfo.n = the walk's length; counters[0] += incidences, counters[1] += bound overflows = 0)
// NEXT #4: allocate the bricks around the reprojected depth points of one frame (every pixel,
// whatever the rank; reading R23) into g.bmask
void launch_brick_alloc(const FrameDesc& f, const GridDesc& g, const NoiseDesc& n, const float* depth, uint8_t* mask,
                        cudaStream_t s);
constexpr int kFillThreads = 128;
void launch_dda_fill(const FrameDesc* frames, const int* cta0, int n_frames, int n_ctas, long long r0,
                     long long n_rays, const GridDesc& g, const NoiseDesc& n, const MsgParams& mp,
                     const float* depth_all, const long long* row_ptr, RayInfo* ray_z, int32_t* vid,
                     int16_t* off_q, float* lnu, int32_t* tile_runs, unsigned long long* counters,
                     const RunSink& sink, RaySeg* seg, unsigned long long* class_counts, int32_t* lam0,
                     cudaStream_t s);
// K9 §III.D evaluation of one frame against T: cls per pixel (-1 invalid, 0/1), counts[0..1] +=
// (valid, accurate) (zeroed by the caller)
void launch_eval(const FrameDesc& f, const GridDesc& g, const NoiseDesc& n, const float* depth, const long long* T,
                 double L0, double k_sigma, double vis_thr, int mode, double L_eval, int8_t* cls,
                 unsigned long long* counts, cudaStream_t s);
// voxel degrees (per-voxel transpose, active count): vox_count zeroed by the caller
void launch_vox_hist(long long n_rays, const long long* row_ptr, const RayInfo* info, const int32_t* vid,
                     int32_t* vox_count, cudaStream_t s);
// K2: out[i] = offset + sum_{j<i} in[j] for i in [0, n]; out has n+1 entries.
void launch_exclusive_scan(const int32_t* in, long long* out, long long n, long long offset,
                           long long* scratch, cudaStream_t s);
// the same with the base read from device memory at *doff (may alias out[0]); n > 0
void launch_exclusive_scan_dev(const int32_t* in, long long* out, long long n, const long long* doff,
                               long long* scratch, cudaStream_t s);
long long scan_scratch_elems(long long n);
// K4: tr[col_ptr[v] + slot] = e for every incidence e (cursor zeroed by caller)
void launch_transpose_fill(long long n_rays, const long long* row_ptr, const RayInfo* info, const int32_t* vid,
                           const long long* col_ptr, int32_t* cursor, int32_t* tr, cudaStream_t s);
// tile-run transpose (K4b): runs per tile, then the run list grouped by tile
void launch_run_fill(long long n_rays, const long long* row_ptr, const RayInfo* info, const int32_t* vid,
                     const long long* tile_ptr, int32_t* cursor, int bucket_stride, Run* runs, cudaStream_t s);
// sparse bricks, re-walk after new keyframes (reading R24): lam_new of old ray r's incidences from
// its old list (same voxel -> its message, else 0); *lost += old incidences not found (never)
void launch_lambda_merge(long long n_rays, const long long* rp_old, const RayInfo* ri_old, const int32_t* vid_old,
                         const int32_t* lam_old, const long long* rp_new, const RayInfo* ri_new, const int32_t* vid_new,
                         int32_t* lam_new, unsigned long long* lost, cudaStream_t s);
// the runs of a RunSink placed by bucket key: dst[tile_ptr[key] + cursor[key]++] (cursor zeroed by
// the caller)
void launch_run_bucket(long long n, const Run* src, const int32_t* keys, const long long* tile_ptr, int32_t* cursor,
                       Run* dst, cudaStream_t s);
// K6 work list: n_items[i] = ceil(count[i] / chunk); items (i, j) from item_ptr
void launch_item_counts(long long V, const int32_t* vox_count, int32_t* n_items, int chunk, cudaStream_t s);
void launch_item_fill(long long V, const int32_t* n_items, const long long* item_ptr, int2* items,
                      cudaStream_t s);
void launch_compact(long long n, const int32_t* flags, const long long* pos, int32_t* out, cudaStream_t s);
// mrf_export_rays: e0[k] = row_ptr[rid[k]], out[k] = info[rid[k]]; then the incidences of ray k
// [e0[k], e0[k] + off[k+1] - off[k]) into the staging arrays at off[k] (null outputs skipped)
void launch_ray_select(long long n, const long long* rid, const long long* row_ptr, const RayInfo* info, long long* e0,
                       RayInfo* out, cudaStream_t s);
void launch_ray_gather(long long n, const long long* e0, const long long* off, const int32_t* vid, const int16_t* off_q,
                       const int32_t* lam, int32_t* ovid, int16_t* ooff, int32_t* olam, cudaStream_t s);
// misc
void launch_active_flags(long long V, const int32_t* vox_count, int32_t* flags, cudaStream_t s);
void launch_span_max(long long n, const int32_t* rays, const RayInfo* info, unsigned long long* out,
                     cudaStream_t s);

// ---- staged K5 (bp.cu ray_msg_staged_kernel): stages of consecutive short rays, bulk-copied
// (TMA, cp.async.bulk) into shared memory and processed by one CTA; thread t owns the 8-slot
// chunk t of the stage, which (segments being 8-aligned) is chunk c of exactly one ray, and the
// per-ray scans run over ray-relative chunk indices, so a ray's rounding never depends on
// where (or on which rank) it is stored.
// A stage is a maximal run of consecutive rays with n <= kShortMax whose first slot lies in one
// kStageCap-slot window and whose index lies in one kStageMaxRays block; longer rays go to the
// tiled long-ray kernel.  Span of a stage < kStageCap + kShortMax.
#ifndef MRF_STAGE_CAP
#define MRF_STAGE_CAP 2048
#endif
#ifndef MRF_STAGE_RAYS
#define MRF_STAGE_RAYS 512
#endif
#ifndef MRF_STAGE_CTAS
#define MRF_STAGE_CTAS 2
#endif
constexpr int kStageCap = MRF_STAGE_CAP;
constexpr int kShortMax = 256;
constexpr int kStageMaxRays = MRF_STAGE_RAYS;
constexpr int kStageThreads = (kStageCap + kShortMax) / 8;  // one 8-slot chunk per thread >= max span
constexpr int kStageCtas = MRF_STAGE_CTAS;                   // resident CTAs per SM
struct Stage {
    int r0, r1;                      // rays [r0, r1)
    int pad0, pad1;
    long long s0, s1;                // slots [s0, s1) = [row_ptr[r0], row_ptr[r1])
};
// stage list: flags over rays (scan input), then fill (stage count known after the scan)
void launch_stage_flags(long long n_rays, const long long* row_ptr, const RayInfo* info, int32_t* flags,
                        cudaStream_t s);
void launch_stage_fill(long long n_rays, const long long* row_ptr, const RayInfo* info, const int32_t* flags,
                       const long long* pos, Stage* stages, cudaStream_t s);
void launch_ray_messages_staged(long long n_stages, const Stage* stages, const long long* row_ptr,
                                const RayInfo* info, const int32_t* vid, const float* lnu, int32_t* lam,
                                const long long* T, const MsgParams& mp, int math, cudaStream_t s);

// ---- BP kernels (bp.cu)
// K5 length classes.  Class k < 16 runs G = 4 << (k / 4) lanes per ray with K = 5 + k % 4
// incidences per lane (capacity G K: 20, 24, 28, 32, 40, ..., 224, 256); classes 16..19 run
// G = 32 lanes with K = 10, 12, 14, 16 (capacity 320 ... 512: the 0.02 m configs' rays); a ray
// goes to the smallest capacity >= n.  Class kNumShort: rays longer than 512 (tiled warp
// kernel).  The per-ray arithmetic depends only on n, never on where the ray is stored.
constexpr int kNumShort = 20;
constexpr int kNumClasses = kNumShort + 1;
__host__ __device__ constexpr int class_G(int k) { return k < 16 ? 4 << (k >> 2) : 32; }
__host__ __device__ constexpr int class_K(int k) { return k < 16 ? 5 + (k & 3) : 10 + 2 * (k - 16); }
__host__ __device__ inline int ray_class(int n) {
    if (n <= 0) return -1;
    for (int k = 0; k < kNumShort; ++k)
        if (n <= class_G(k) * class_K(k)) return k;
    return kNumShort;
}
// class lists: counts per class (counts zeroed by the caller), then the ray ids of class k at
// out[off[k] ...] (cursor zeroed by the caller; order inside a class is irrelevant)
struct ClassOffsets {
    long long off[kNumClasses];
};
void launch_class_count(long long n_rays, const RayInfo* info, unsigned long long* counts, cudaStream_t s);
// matrix-free (NEXT #1): class lists per chunk of fpc frames, key = (frame / fpc) * kNumClasses + class
void launch_class_count_mf(long long n_rays, const RayInfo* info, int fpc, unsigned long long* counts, cudaStream_t s);
void launch_class_scatter_mf(long long n_rays, const RayInfo* info, int fpc, const long long* off,
                             unsigned long long* cursor, int32_t* out, cudaStream_t s);
void launch_class_scatter(long long n_rays, const RayInfo* info, const ClassOffsets& off, unsigned long long* cursor,
                          int32_t* out, cudaStream_t s);
// K5 class-list descriptors: desc[i] = {row_ptr[r] (int32), n, frame, r} for r = rays[i], so a
// class kernel's warp reaches its ray's incidences with one load instead of two dependent ones
// (rebuilt with the class lists, once per graph change)
void launch_class_desc(long long n, const int32_t* rays, const long long* row_ptr, const RayInfo* info, int4* desc,
                       cudaStream_t s);
void launch_ray_messages(int cls, long long n_rays, const int32_t* rays, const int4* desc, const long long* row_ptr,
                         const RayInfo* info, const int32_t* vid, const float* lnu, int32_t* lam,
                         const long long* T, const MsgParams& mp, float* scratch, long long scratch_per_warp,
                         int n_warps_long, int math, cudaStream_t s);
// K6b (default for per-ray messages with a stored graph): blocks = {first ray, ncols | nrows << 16,
// row stride in rays, 0} of neighbouring pixels; max_probe: the hash table's probe limit (64; < 0:
// every element straight to T, a test knob); stats (nullable): += {distinct voxels summed over the
// blocks, elements sent to T directly}; T (or the compacted tiles through tile_map)
// accumulates with int64 atomics (zero it first); next: a device counter (zeroed here).
constexpr int kBlkCols = 32, kBlkRows = 16;
constexpr double kBlkMinPpv = 6.0;   // auto K6b: a voxel spans >= 6 pixels at 3 m (mrf_api.cu)
constexpr long long kBlkMinShare = 16;  // ... and the blocks' incidences per distinct voxel >= 16
void launch_block_reduce(long long n_blocks, const int4* blocks, const long long* row_ptr, const RayInfo* ray_z,
                         const int32_t* vid, const int32_t* lam, long long* T, unsigned* next,
                         unsigned long long* stats, const int32_t* tile_map, int max_probe, long long chk_lam,
                         long long chk_out, cudaStream_t s);
// K6b for the keyframe averages (pass 0: counts + min |q|, pass 1: the fixed-point sums; the
// blocks' .w is their frame): the same outputs as launch_kf_sums over (frame, tile) runs
void launch_block_kf(int pass, long long n_blocks, const int4* blocks, const long long* row_ptr, const RayInfo* ray_z,
                     const int32_t* vid, const int32_t* lam, long long* sums, long long n_slots, long long VI,
                     unsigned* next, long long chk_lam, cudaStream_t s);
void launch_voxel_reduce(long long n_items, const int2* items, const long long* col_ptr, const int32_t* tr,
                         const int32_t* lam, long long* T, cudaStream_t s);
// tile_map (nullable): tile -> position among the tiles written (world > 1: the tiles some rank
// touches, compacted for the all-reduce); nullptr = the tile itself
// (buckets b of tile b % n_tiles: tiles, or (frame, tile) pairs frame-major)
void launch_tile_reduce(long long n_items, const int2* items, const long long* tile_ptr, const Run* runs,
                        const int32_t* lam, int per_item, long long* T, unsigned* next, bool pad,
                        const int32_t* tile_map, long long chk_lam, long long chk_out_tiles, int n_tiles,
                        cudaStream_t s);
// T[tile_of[i] tile] = src[i-th compact tile] for i < n_tiles (16384 slots each)
void launch_tile_scatter(long long n_tiles, const int32_t* tile_of, const long long* src, long long* T, cudaStream_t s);
// keyframe averages (reading R22), two integer passes over the (frame * NT + tile) buckets into
// sums = [N: int64 n_pos + 2^32 n_neg | D: int64, 2^-30 | M / A: uint32 min |q|, then float scale]
// per [bucket][slot] (n_slots = F * VI each; N, D zeroed and M set to 0xffffffff by the caller):
// pass 0 the counts and min |q|, then launch_kf_scale, then pass 1 the fixed-point sums of the
// small probabilities (bp.cu tile_reduce_kernel<2 / 3>)
void launch_kf_sums(int pass, long long n_items, const int2* items, const long long* bucket_ptr, const Run* runs,
                    const int32_t* lam, int per_item, long long* sums, long long n_slots, unsigned* next,
                    long long chk_lam, cudaStream_t s);
// (the (frame, slot) entries [first, first + count) of the n_slots)
void launch_kf_scale(long long n_slots, long long first, long long count, long long* sums, cudaStream_t s);
// qbar[f][v] = quantised clip(ln(sum mu(1) / sum mu(0)), +-256) (0 without a ray), T[v] = sum_f qbar
void launch_kf_finalize(long long F, long long VI, const long long* sums, int32_t* qbar, long long* T, cudaStream_t s);
void launch_marginals(const GridDesc& g, const long long* T, double L0, float* out, cudaStream_t s);
void launch_lambda_to_float(long long n, const int32_t* q, float* out, cudaStream_t s);

}  // namespace mrf
