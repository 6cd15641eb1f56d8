/*
 * mrf.h -- C ABI of the B200-native MRFMap hot path (arxiv 2006.03512).
 *
 * The library builds the ray-voxel factor graph of posed depth images and runs
 * loopy sum-product belief propagation over it on one B200 (or on N B200s, one
 * process per GPU, rays sharded by pixel row).  Citations: P:n = line n of the
 * paper; DESIGN.md restates every step and every reading R1..R15.
 *
 *   mrf_create      grid + prior + forward sensor model       (Eq.1, Eq.2, Eq.4)
 *   mrf_add_frame   depth image + intrinsics + pose -> rays -> 3D-DDA -> ray->voxel CSR
 *                                                             ("ray traced ... 3DDA", P:205 3-sigma cutoff)
 *   mrf_bp_iterate  n flooding iterations: per-ray factor->voxel messages (Eq.13 P:153-156,
 *                   Eq.14 P:158-161 / P:524) and voxel beliefs as a deterministic segmented
 *                   reduction over the voxel->ray transpose (Eq.6)
 *   mrf_marginals   p_v = sigma(L0 + T_v) (Eq.8)
 *
 * Conventions shared by every entry point
 *   - Status codes only; nothing throws across the ABI.  CUDA and NCCL failures are sticky:
 *     once one is returned every later call on the ctx returns the same code.
 *   - Ownership: every input buffer is read (copied to the device or consumed) before the
 *     call returns; the caller keeps ownership.  Outputs go to caller-allocated buffers.
 *   - Pointers marked "host or device" are classified with cudaPointerGetAttributes.
 *   - A ctx is bound to the CUDA device that was current at mrf_create and is not
 *     thread-safe.  All device work is ordered on the ctx stream (mrf_set_stream).
 *   - Voxel index v = x + nx*(y + ny*z) (x fastest).  Canonical incidence order is
 *     (frame add order, pixel index v*W+u, position along the ray).
 *   - Messages are stored as int32 fixed point lambda*2^23 (clipped to +-256 nats, reading
 *     R9) and beliefs as int64 sums T_v = sum_e q_e, so every reduction is exact and
 *     independent of order, rank count and scheduling.
 */
#ifndef MRF_H
#define MRF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mrf_ctx mrf_ctx; /* opaque; owned by the caller from mrf_create to mrf_destroy */

typedef enum {
    MRF_OK = 0,
    MRF_ERR_INVALID_ARG = 1,   /* argument rejected; state unchanged */
    MRF_ERR_OUT_OF_MEMORY = 2, /* device allocation failed; state unchanged */
    MRF_ERR_CAPACITY = 3,      /* frame would exceed an index limit (E >= 2^31, rays >= 2^31); state unchanged */
    MRF_ERR_CUDA = 4,          /* sticky */
    MRF_ERR_NCCL = 5,          /* sticky */
    MRF_ERR_STATE = 6          /* call not valid in the current state (e.g. comm mode mismatch) */
} mrf_status;

/* Forward sensor model nu(Z | d) (Eq.4; learnt aggregate model P:230) as a table of
 * log densities.  Row i is the measured range Z_i = z_lo + (i+0.5)(z_hi-z_lo)/n_z, column j the
 * offset delta_j = off_lo + (j+0.5)(off_hi-off_lo)/n_off of the voxel depth d = Z + delta.
 * Lookups interpolate bilinearly between bin centres and clamp to the edge centres.
 * Traversal margin past the measured range: margin(Z) = max(margin_min, margin_k*sigma(Z)),
 * sigma(Z) = (c0 + c1 Z) + c2 Z^2  (3 sigma beyond the depth; reading R5). */
typedef struct {
    const float* log_nu;   /* [n_z][n_off] row-major, finite, host memory; copied at create (entries
                              below -1e30, e.g. -FLT_MAX for log 0, are taken as -1e30) */
    int32_t n_z, n_off;    /* >= 2 each */
    double z_lo, z_hi;     /* metres, z_hi > z_lo */
    double off_lo, off_hi; /* metres, -1 <= off_lo < off_hi <= 1 (span of the int16 offset code) */
    double margin_min;     /* metres, >= 0 */
    double margin_k;       /* >= 0 */
    double sigma_c[3];     /* c0, c1, c2.  Bounded margin: with D the grid diagonal (metres),
                              margin_min <= D and margin_k (|c0| + |c1| D + |c2| D^2) <= D, so a
                              traversal segment never exceeds 2 D (the DDA's 32-bit exact products) */
} mrf_noise_desc;

/* Data-parallel sharding: rank keeps the rays of pixel rows v % world == rank.
 * comm = MRF_COMM_NCCL: an NCCL communicator is created from nccl_id (all ranks pass the same
 *   id, from mrf_nccl_unique_id on rank 0) and mrf_bp_iterate all-reduces the per-voxel int64
 *   partial sums every iteration -- only over the 32x32x16 tiles some rank touches (a touched-
 *   tile mask ncclMax-reduced once per graph change, so every rank compacts identically).  The
 *   communicator's asynchronous error state is polled after every collective; a failure is the
 *   sticky MRF_ERR_NCCL.  Every rank must make the same sequence of calls (collectives inside).
 * comm = MRF_COMM_EXTERNAL: no communicator; the caller reduces the partials itself with
 *   mrf_bp_partial / mrf_bp_finish (used to emulate ranks on one GPU, and by tests). */
enum { MRF_COMM_NCCL = 0, MRF_COMM_EXTERNAL = 1 };
typedef struct {
    int32_t rank, world; /* 0 <= rank < world */
    int32_t comm;        /* MRF_COMM_NCCL or MRF_COMM_EXTERNAL */
    unsigned char nccl_id[128];
} mrf_dist_desc;

/* Create a dense nx*ny*nz grid of voxel side resolution_m at origin_m (metres), with the
 * Bernoulli prior gamma (Eq.2) and sensor model noise.  dist == NULL -> one GPU.
 * Errors: INVALID_ARG for dims <= 0 or > 8192, V >= 2^31, resolution not finite or <= 0,
 * prior not in (0,1), bad noise table; OUT_OF_MEMORY; NCCL on communicator failure. */
mrf_status mrf_create(const int32_t dims[3], double resolution_m, const double origin_m[3], float prior,
                      const mrf_noise_desc* noise, const mrf_dist_desc* dist, mrf_ctx** out);

/* Add one keyframe: depth is H*W z-depth in metres (row-major, host or device; 0, NaN or <= 0
 * = invalid pixel, skipped and counted); K = {fx, fy, cx, cy} with pixel centres at integer
 * (u, v); T_wc = 3x4 row-major world-from-camera [R | C], OpenCV camera axes.
 * Each kept pixel becomes a ray traced by the fixed-point 3D-DDA from C to the measured range
 * plus margin(Z); a ray whose measured point lies outside the grid is dropped and counted
 * (reading R11).  New messages start at 0 (warm start of the existing ones).
 * Errors: INVALID_ARG for width/height <= 0, non-finite K, fx or fy <= 0, non-finite T_wc,
 * ||R^T R - I||_max > 1e-6, camera centre outside the grid; CAPACITY when the graph would
 * exceed the index limits (the frame is not added); OUT_OF_MEMORY (not added).
 * frame_id_out (nullable) receives the 0-based frame index. */
mrf_status mrf_add_frame(mrf_ctx* ctx, const float* depth, int32_t width, int32_t height, const double K[4],
                         const double T_wc[12], int64_t* frame_id_out);

/* Run n >= 0 synchronous flooding iterations (reading R4): every ray computes its
 * factor->voxel messages from the same belief snapshot T, then T is rebuilt by the segmented
 * reduction over the voxel->ray transpose (and all-reduced across ranks).  Asynchronous on the
 * ctx stream.  Errors: INVALID_ARG for n < 0; STATE in MRF_COMM_EXTERNAL mode with world > 1. */
mrf_status mrf_bp_iterate(mrf_ctx* ctx, int32_t n);

/* Occupancy marginals p_v = sigma(L0 + T_v 2^-23) for all V voxels, x fastest, float32; out is
 * a host (out_is_device = 0) or device (1) buffer of V floats.  Voxels seen by no ray return
 * the prior.  Synchronises the ctx stream. */
mrf_status mrf_marginals(mrf_ctx* ctx, float* out, int32_t out_is_device);

/* Free everything (also valid on a ctx in a sticky error state).  NULL is a no-op. */
mrf_status mrf_destroy(mrf_ctx* ctx);

/* Last error message of the ctx (or of the last failed mrf_create when ctx == NULL); the
 * string stays valid until the next call on the ctx. */
const char* mrf_last_error(const mrf_ctx* ctx);

/* ------------------------------------------------------------------ runtime / introspection */

/* Use cuda_stream (a cudaStream_t; NULL = the CUDA default stream) for all later work.  Until
 * this is called the ctx uses a private non-blocking stream.  Device buffers passed to the ABI
 * are read/written in stream order on this stream. */
mrf_status mrf_set_stream(mrf_ctx* ctx, void* cuda_stream);

/* Drop every frame, ray, incidence and message (buffers are kept for reuse); T = 0. */
mrf_status mrf_reset(mrf_ctx* ctx);

/* Pre-allocate room for n_rays rays (pixels owned by this rank) and n_incidences incidences. */
mrf_status mrf_reserve(mrf_ctx* ctx, int64_t n_rays, int64_t n_incidences);

/* Graph sizes of this rank: kept rays, incidences E, voxels touched by >= 1 incidence,
 * invalid pixels and dropped rays.  Any pointer may be NULL.  Synchronises. */
mrf_status mrf_graph_sizes(mrf_ctx* ctx, int64_t* n_rays, int64_t* n_incidences, int64_t* n_active_vox,
                           int64_t* n_invalid, int64_t* n_dropped);

/* Generating-surface accuracy of one posed depth image against the CURRENT beliefs (PAPER.md
 * §III.D P:168-196 -- visibility Eq.15, occlusion probability Eq.16, generating-surface density
 * Eq.17-18 -- and the per-image score of §V; readings R18-R21 in DESIGN.md).  For every
 * valid pixel of the rows this rank owns, the ray from the camera to the map boundary is walked
 * by the same fixed-point DDA: alpha = -ln(1 - p_v)/res, vis and omega = alpha vis along it,
 * s* = entry of the most likely generating voxel.  Accurate iff vis_inf > vis_threshold ? Z >
 * s_inf : (mode MRF_EVAL_SIGMA_BAND, §V) |Z - s*| <= k_sigma sigma(Z) (sigma: the ctx's noise
 * model) or (mode MRF_EVAL_VOXEL_BOUNDS, §III.D) Z inside the argmax voxel.  depth/K/T_wc as in
 * mrf_add_frame (camera inside the grid).  cls (nullable, host, W*H): -2 row of another rank,
 * -1 invalid pixel, 0 inaccurate, 1 accurate.  n_valid / n_accurate: this rank's counts
 * (sum over ranks for the image score).  k_sigma > 0, 0 < vis_threshold < 1.  Synchronises. */
enum { MRF_EVAL_SIGMA_BAND = 0, MRF_EVAL_VOXEL_BOUNDS = 1 };
mrf_status mrf_evaluate(mrf_ctx* ctx, const float* depth, int32_t width, int32_t height, const double K[4],
                        const double T_wc[12], int32_t mode, double k_sigma, double vis_threshold, int8_t* cls,
                        int64_t* n_valid, int64_t* n_accurate);

/* Sizes of this rank's device layout, for the roofline byte counts: n_slots =
 * incidence slots incl. the padding of every ray segment to a multiple of 8; n_runs = tile runs
 * of the K6 transpose; n_belief_slots = tile-major belief slots (32x32x16 tiles).  Builds the
 * transpose if the graph changed.  Any pointer may be NULL.  Synchronises. */
mrf_status mrf_layout_sizes(mrf_ctx* ctx, int64_t* n_slots, int64_t* n_runs, int64_t* n_belief_slots);

/* Which voxel aggregation (Eq.6's T_v = sum of the messages on v) the next iteration
 * runs: *path = 1 for the pixel-block hash reduction over the messages in ray order
 * (K6b), 0 for the reduction over the tile-run transpose (K6).  Builds the layout if the graph
 * changed; a ctx whose blocks shared too few voxels in their first K6b reports 0 afterwards.
 * path must not be NULL.  Synchronises. */
mrf_status mrf_k6_path(mrf_ctx* ctx, int32_t* path);

/* Copy this rank's graph to host buffers in canonical order: ray_pixel[n_rays] = frame*2^32 +
 * (v*W + u) of each kept ray, row_ptr[n_rays+1], vid[E], off_q[E] (metres * 32768).  Any pointer
 * may be NULL.  Synchronises. */
mrf_status mrf_export_graph(mrf_ctx* ctx, int64_t* ray_pixel, int64_t* row_ptr, int32_t* vid, int16_t* off_q);

/* Selected rays of this rank, without copying the whole graph (tests at full size): for k < n,
 * ray k is pixel pixel[k] = v*W + u of frame frame[k] (frame add order); row v must be owned by
 * this rank (v % world == rank), else MRF_ERR_INVALID_ARG.  Outputs, host buffers, any may be
 * NULL: row_ptr[n+1] (offsets into the concatenated lists; 0-length for invalid or dropped
 * pixels), and up to cap entries each of vid (voxel index x + nx (y + ny z)), off_q, lambda
 * (nats).  MRF_ERR_CAPACITY if the lists exceed cap.  Synchronises. */
mrf_status mrf_export_rays(mrf_ctx* ctx, int64_t n, const int32_t* frame, const int64_t* pixel, int64_t cap,
                           int64_t* row_ptr, int32_t* vid, int16_t* off_q, float* lambda);

/* Voxel->ray transpose: col_ptr[V+1] and, per voxel, the incidence indices tr[E] (order inside a
 * voxel is unspecified).  Builds the transpose if needed.  Synchronises. */
mrf_status mrf_export_transpose(mrf_ctx* ctx, int64_t* col_ptr, int32_t* tr);

/* Messages lambda_e (nats) of this rank in canonical order, host buffer of E floats.
 * MRF_ERR_STATE in keyframe-average mode with matrix-free walks (no per-incidence messages are
 * kept there; mrf_export_keyframe_average exports the state). */
mrf_status mrf_export_messages(mrf_ctx* ctx, float* lambda);

/* Replace the messages (host buffer of E floats, nats; quantised to 2^-23 and clipped to
 * +-256) and rebuild T from them (summed over ranks in MRF_COMM_NCCL mode; left to the caller
 * in MRF_COMM_EXTERNAL mode with world > 1, see mrf_bp_partial). */
mrf_status mrf_import_messages(mrf_ctx* ctx, const float* lambda);

/* Beliefs T_v (int64, units 2^-23 nats; the global sum over ranks) into a host buffer of V,
 * x fastest. */
mrf_status mrf_export_beliefs(mrf_ctx* ctx, int64_t* T);

/* MRF_COMM_EXTERNAL mode, one iteration split in two: mrf_bp_partial (iterate = 1) computes
 * this rank's messages from the current T and writes its partial sums to partial_out (device
 * pointer, mrf_belief_slots() int64 in the library's internal tile-major slot order); the
 * caller sums the partials of all ranks element-wise and hands the total back with
 * mrf_bp_finish (device pointer, same size), which becomes T.  iterate = 0 only sums the
 * current messages (e.g. after mrf_import_messages, which in this mode leaves T alone).
 * Device buffers are accessed on the ctx stream (see mrf_set_stream). */
mrf_status mrf_bp_partial(mrf_ctx* ctx, int32_t iterate, int64_t* partial_out_device);
mrf_status mrf_bp_finish(mrf_ctx* ctx, const int64_t* total_device);

/* Number of int64 belief slots (nx, ny rounded up to multiples of 32 and nz to a multiple of 16,
 * times each other): voxels are stored tile-major in 32 x 32 x 16 tiles internally (the unit of
 * the shared-memory voxel reduction; cf. the paper's GVDB 8^3 bricks). */
int64_t mrf_belief_slots(const mrf_ctx* ctx);

/* Message model (reading R22).
 *   MRF_MSG_PER_RAY (default): every incidence keeps its own factor->voxel message (Eq.6: the
 *     cavity of a ray excludes only its own message).
 *   MRF_MSG_KEYFRAME_AVG: the paper's memory-saving assumption ("all rays going through a
 *     voxel from a single keyframe send the same average message"): per (frame, voxel) the
 *     average of the normalised messages of the frame's rays, lbar = ln(mean mu(1) / mean mu(0))
 *     (uniform when the frame has no ray through the voxel); T_v = sum over frames of lbar; a
 *     ray of frame f sees the cavity L0 + T_v - lbar[f][v].  The sums of mu(1), mu(0) are exact
 *     integer sums of fixed-point small probabilities (2^-30, relative to the largest term when
 *     the messages have one sign, so down to e^-256), so the average does not depend on the
 *     summation order.  Costs 20 bytes per (frame, belief slot) of device memory.  With the stored
 *     graph the messages are still stored per incidence (mrf_export_messages works); with
 *     matrix-free walks (mrf_set_matrix_free) they are not kept at all -- only a scratch of one
 *     chunk of frames between the message pass and the averaging of that chunk -- which is the
 *     paper's storage: keyframes re-traced every pass, one average message per (keyframe, voxel).
 * Set before the first frame (MRF_ERR_STATE otherwise); single rank only (MRF_ERR_INVALID_ARG
 * with world > 1).  Frame ids are the mrf_add_frame order (frame_id_out). */
enum { MRF_MSG_PER_RAY = 0, MRF_MSG_KEYFRAME_AVG = 1 };
mrf_status mrf_set_message_mode(mrf_ctx* ctx, int32_t mode);
/* Keyframe-average mode: frame's current average log-odds lbar (nats) into a host buffer of V
 * floats, x fastest.  MRF_ERR_STATE in per-ray mode, MRF_ERR_INVALID_ARG for a bad frame id. */
mrf_status mrf_export_keyframe_average(mrf_ctx* ctx, int64_t frame, float* out);

/* Sparse-brick map (reading R23).
 * brick = 0: dense grid (default).  brick = B (a power of two in [2, 64]; the paper uses 8):
 * every mrf_add_frame allocates the B^3-cell bricks around its reprojected depth points (every
 * voxel within 3 sigma(Z) of a measured point -- margin_k sigma_c of the noise model -- belongs to
 * an allocated brick; all pixels count, whatever the rank), and the ray walk emits only cells of
 * allocated bricks (empty skip: unallocated space holds no variable, i.e. a certainly-empty voxel
 * in Eq.13/14; its marginal stays gamma).  Beliefs stay dense in device memory.  Set before the
 * first frame (MRF_ERR_STATE otherwise).  The rays are counted and walked against the allocation
 * of every frame added so far when the graph is next used (iterate, export, sizes), so the 2^31
 * incidence-slot capacity is checked then: MRF_ERR_CAPACITY from that call (mrf_reset starts
 * over).  A frame added after the graph was used grows the allocation under rays already walked
 * (reading R24): every frame is walked again at the next use, each old incidence keeps its
 * message and the cells of new bricks start at 0 (the beliefs do not change); the depth images
 * are kept for this (W*H floats per frame).  With matrix-free walks the allocation is fixed once
 * the graph is used (a later mrf_add_frame returns MRF_ERR_STATE).
 * mrf_reset clears the allocation and keeps the mode. */
mrf_status mrf_set_sparse_bricks(mrf_ctx* ctx, int32_t brick);
/* Allocation mask: out (nullable) = ceil(nz/B) * ceil(ny/B) * ceil(nx/B) bytes, brick x fastest,
 * 1 = allocated; n_allocated (nullable) = number of allocated bricks.  MRF_ERR_STATE when dense. */
mrf_status mrf_export_bricks(mrf_ctx* ctx, uint8_t* out, int64_t* n_allocated);

/* Matrix-free iteration (the paper re-traces every keyframe each pass,
 * P:200).  frames_per_chunk = 0: the ray->voxel lists (vid, off_q, log nu: 10 bytes per
 * incidence) are stored once (default).  frames_per_chunk = F > 0: only the messages (4 bytes per
 * incidence) and the tile-run transpose (~1 byte per incidence) persist, plus a 40-byte segment
 * per ray and the first cell of every message-kernel chunk (<= 1 byte per incidence): the message
 * kernel re-walks each chunk of a ray with the same integer DDA in registers (K12).  New frames
 * are walked once into a scratch of one chunk of F frames (counting, tile runs, checkpoints).
 * Same results as the stored graph, bit for bit, at the cost of one DDA walk per iteration
 * (environment MRF_MF_FUSED=0: the chunks are walked into the scratch before every message pass
 * instead; also the path taken with sparse bricks).  With keyframe-average messages the
 * per-incidence messages are not stored either (mrf_set_message_mode).  The depth images are kept
 * (W*H floats per frame).  Set before the first frame (MRF_ERR_STATE otherwise);
 * environment MRF_SYNC_DEBUG=1 synchronises after every matrix-free step and reports its status on
 * stderr (debugging aid);
 * mrf_export_graph / mrf_export_rays / mrf_export_transpose return MRF_ERR_STATE, and
 * mrf_graph_sizes reports n_active_vox = -1. */
mrf_status mrf_set_matrix_free(mrf_ctx* ctx, int32_t frames_per_chunk);

/* Learnt per-patch sensor model (SURVEY §8(f) NEXT #4 option, DESIGN reading
 * R25): the image is cut into patch_px x patch_px pixel patches, patch (i, j) = pixels
 * u in [i patch_px, (i+1) patch_px), v in [j patch_px, (j+1) patch_px); coeffs (host, row-major
 * [n_py][n_px][6], copied) holds per patch b0, b1, b2, s0, s1, s2: the bias b(d) = b0 + b1 d + b2 d^2
 * and the standard deviation s(d) = max(s0 + s1 d + s2 d^2, sigma_min) of the measured range given
 * the true range d (2nd-degree polynomials).  The forward model of Eq.4 becomes
 * nu(d) = N(Z; d + b(d), s(d)) ("the probability of a given measurement originating from this
 * predicted measurement and distributed using the learnt noise value"), evaluated in closed
 * form (fp32) at each incidence's voxel depth d = Z + off_q 2^-15 instead of the table of
 * mrf_create; the traversal margin of a pixel becomes max(margin_min, margin_k s(Z)) with its
 * patch's s (fp64, as with sigma_c).  patch_px = 0 returns to the table (coeffs ignored).
 * Set before the first frame (MRF_ERR_STATE otherwise); frames (and mrf_evaluate images) must fit
 * the patch grid (W <= n_px patch_px, H <= n_py patch_px; MRF_ERR_INVALID_ARG); MRF_ERR_INVALID_ARG
 * for non-finite coefficients, sigma_min <= 0, or a margin over the grid diagonal (the bound of
 * mrf_create, per patch).  mrf_reset keeps the model. */
mrf_status mrf_set_patch_noise(mrf_ctx* ctx, int32_t patch_px, int32_t n_px, int32_t n_py, const double* coeffs,
                               double sigma_min);

/* 128-byte ncclUniqueId for MRF_COMM_NCCL (call on rank 0, broadcast to the others). */
mrf_status mrf_nccl_unique_id(unsigned char out[128]);

/* Per-kernel timing with CUDA events on the ctx stream (off by default). */
enum {
    MRF_K_RAYGEN_COUNT = 0, /* K1: pixel -> segment + DDA count */
    MRF_K_DDA_FILL = 1,     /* K3: DDA fill of vid/off_q + voxel histogram */
    MRF_K_SCAN = 2,         /* K2: exclusive scans */
    MRF_K_TRANSPOSE = 3,    /* K4: voxel->ray transpose fill + work lists */
    MRF_K_RAY_MSG = 4,      /* K5: factor->voxel messages (all length classes) */
    MRF_K_VOXEL_SUM = 5,    /* K6: segmented reduction over the transpose */
    MRF_K_ALLREDUCE = 6,    /* K7: NCCL all-reduce of T */
    MRF_K_MARGINALS = 7,    /* K8 */
    MRF_K_COUNT = 8
};
mrf_status mrf_set_profiling(mrf_ctx* ctx, int32_t on);
/* Synchronise, then return (and clear) per-kernel launch counts and summed event time (ms),
 * arrays of MRF_K_COUNT entries (nullable). */
mrf_status mrf_profile_read(mrf_ctx* ctx, int64_t* launches, double* total_ms);
/* Total kernels launched by this ctx since create (all kinds). */
int64_t mrf_launch_count(const mrf_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* MRF_H */
