// mrf_api.cu -- host runtime behind include/mrf.h (C ABI), one ctx per GPU/rank.
//
// Owns the device buffers (HBM layout in DESIGN.md §Data layout), the stream, the NCCL
// communicator and the graph state; every step of the hot path runs in the kernels of
// graph.cu / scan.cu / bp.cu.  There is no CPU fallback: any CUDA failure is returned as a
// sticky MRF_ERR_CUDA.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"
#include "walk.cuh"
#include "mrf.h"

using namespace mrf;

namespace {

thread_local std::string g_create_error;

template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;
    // Grow to at least n elements (x1.125 geometric: the 0.02 m configs fill most of the 180 GB);
    // copies the first `used` elements.
    cudaError_t ensure(size_t n, size_t used, cudaStream_t s) {
        if (n <= cap) return cudaSuccess;
        size_t nc = std::max(n, cap + cap / 8);
        T* q = nullptr;
        cudaError_t e = cudaMalloc(&q, nc * sizeof(T));
        if (e != cudaSuccess) {
            cudaGetLastError();
            return e;
        }
        if (p) {
            if (used) {
                e = cudaMemcpyAsync(q, p, used * sizeof(T), cudaMemcpyDeviceToDevice, s);
                if (e == cudaSuccess) e = cudaStreamSynchronize(s);
                if (e != cudaSuccess) {
                    cudaFree(q);
                    return e;
                }
            }
            cudaFree(p);
        }
        p = q;
        cap = nc;
        return cudaSuccess;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

constexpr int kClassCtr = 32;  // counters[32 .. 32 + kNumClasses]: rays per K5 class, longest ray

struct FrameRec {
    int W, H, rows_owned;
    long long ray_base, n_rays;
};

struct ProfEvent {
    int kind;
    cudaEvent_t a, b;
};

}  // namespace

struct mrf_ctx {
    int device = 0;
    int sms = 148;  // multiprocessors of the ctx's device (grid sizing)
    GridDesc grid{};
    NoiseDesc noise{};
    long long V = 0;   // voxels (nx*ny*nz)
    long long VI = 0;  // internal belief slots: tiles * 16384 (tile-major, DESIGN.md §Data layout)
    long long NT = 0;  // tiles
    bool k6_voxel = false;  // ablation: per-voxel transpose K6 instead of the tile-run K6 (MRF_K6=voxel)
    // K6b (default): the pixel-block hash reduction over the stored graph (no tile runs); MRF_K6=tile:
    // the tile-run K6.  The modes without stored vid (matrix-free) or with per-(frame, slot) sums
    // (keyframe averages) always use the tile runs.
    // MRF_K6: unset = auto, "block" = always K6b, anything else = the tile runs.  Auto takes K6b
    // when the blocks can share voxels: one rank (interleaved rows of world > 1 share few), and a
    // voxel spanning >= kBlkMinPpv pixels at a nominal 3 m (min over the frames of f res / 3 m:
    // frames30 8.75, the 0.02 m configs 3.5 -- measured: K6b loses to the tile runs at 2, 4, 8
    // emulated ranks and on frames100, profiles/r02x_k6_paths.log).  The first K6b after a graph
    // change also checks what the blocks shared (blk_check): too little, and this ctx demotes
    // itself to the tile runs for good.
    bool k6_block = true;
    int k6_force = 0;           // 1: K6b always, 2: tile runs always (MRF_K6)
    bool k6_demoted = false;
    bool blk_check = false;     // check the next K6b's stats (after build_blocks)
    bool tile_counts_ok = true; // tile_runs holds the runs per bucket of every ray walked so far
    // MRF_KF_BLOCK=1: the keyframe-average passes over pixel blocks too (bit-identical, but slower
    // than the (frame, tile) runs at frames30: 69.4 vs 54.2 ms of K6' per step -- off)
    bool kf_blk_on = false;
    double ppv_min = 1e30;      // min over the frames of min(fx, fy) res / 3 m
    long long blk_min_share = kBlkMinShare;  // (MRF_BLK_SHARE: a test forces the demotion)
    int blk_max_probe = 64;  // (MRF_BLK_PROBE: < 0 sends every element to T directly, for tests)
    int k5_math = 1;        // K5 math level (bp.cu; MRF_K5_MATH=0|1)
    int k6_item = 8192;       // runs per K6 work item (set per graph unless MRF_K6_ITEM fixes it)
    bool k6_item_fixed = false;
    bool k6_lpt = true;  // MRF_K6_LPT=0: j-major item order only
    bool k6_dynamic = true;  // MRF_K6_DYNAMIC=0: fixed-stride item order
    bool k6_pad = true;      // MRF_K6_PAD=0: plain accumulator layout (y, z steps in one bank)
    // keyframe-average mode (NEXT #3, reading R22): one message per (frame, voxel)
    bool kf_avg = false;
    // matrix-free mode (NEXT #1): only lambda and the tile runs persist; vid / off_q / log nu are
    // re-walked per chunk of mf frames into scratch for the transpose build and for every K5 pass
    struct MfChunk {
        int f0, f1;
        long long r0, r1, e0, e1;
    };
    int mf = 0;  // frames per chunk, 0 = off
    // fused (default): K5 re-walks each lane's chunk itself from a stored first cell (K12, with the
    // empty skip in sparse-brick maps), so no per-iteration walk into the scratch; the scratch
    // serves only the first walk of new frames.  MRF_MF_FUSED=0: the scratch path.
    bool mf_fused = true;
    DBuf<RaySeg> ray_seg;   // per ray: segment for the re-walks
    DBuf<int32_t> ck;       // chunk checkpoints, ck[row_ptr / 4 + c]
    // keyframe averages + fused matrix-free walks (the paper's storage): the per-incidence
    // messages are not state (K5 reads the keyframe averages), so they live only in a one-chunk
    // scratch between K5 and K6' of the chunk; the K6' items are grouped by chunk
    DBuf<int32_t> lam_chunk;
    std::vector<long long> kf_item_off;  // K6' items of chunk ci: [kf_item_off[ci], kf_item_off[ci + 1])
    bool kf_chunked() const { return kf_avg && mf && mf_fused; }
    std::vector<FrameDesc> mf_frames;
    std::vector<long long> mf_frame_e;  // row_ptr at each frame's first ray (+ the end)
    std::vector<MfChunk> mf_chunks;
    DBuf<int32_t> s_vid, s_vid2;  // two scratch sets: chunk i + 1 is walked while chunk i's K5 runs
    DBuf<int16_t> s_off, s_off2;
    DBuf<float> s_lnu, s_lnu2;
    DBuf<int> d_cta_tmp;
    DBuf<long long> mf_cls_off_d;
    std::vector<long long> mf_cls_n, mf_cls_off;
    // sparse-brick mode (NEXT #4, reading R23): brick allocation mask, grid.bmask points at it
    int brick = 0;  // cells per brick edge, 0 = dense
    DBuf<uint8_t> bmask;
    long long n_brick_slots = 0;
    // keyframes added after the graph was used (reading R24): every filled frame (depth kept) is
    // walked again against the grown allocation; the old layout is kept until the messages moved
    std::vector<FrameDesc> sp_frames;
    bool sp_rebuild = false;
    DBuf<long long> rp_old;
    DBuf<RayInfo> ri_old;
    DBuf<int32_t> vid_old, lam_old;
    long long sp_R_old = 0;
    DBuf<int32_t> qbar;           // [frame][VI] quantised average log-odds
    DBuf<long long> kf_sums;       // [frame][VI] x {N int64, D int64 (2^-30), M/A uint32} (bp.cu)
    long long kf_frames_alloc = 0;
    // tile-run buckets by (frame, tile), frame-major: always for keyframe averages; in per-ray mode
    // with MRF_K6_FRAMES=1 (K6 items then cover one frame's rays of a tile)
    bool frame_buckets = false;
    bool fb() const { return kf_avg || frame_buckets; }
    bool want_block() const {
        return k6_force == 1 || (k6_force == 0 && world == 1 && ppv_min >= kBlkMinPpv && !k6_demoted);
    }
    bool use_block() const { return want_block() && !k6_voxel && !kf_avg && !mf && !frame_buckets; }
    // the keyframe-average sums over pixel blocks (stored graph only)
    bool kf_block() const { return want_block() && kf_avg && !mf && !k6_voxel && kf_blk_on; }
    bool any_block() const { return use_block() || kf_block(); }
    long long n_bucket_groups() const { return fb() ? std::max<long long>(1, (long long)frames.size()) : 1; }     // runs per K6 work item (MRF_K6_ITEM, <= kRunsPerItem)
    bool k5_staged = false; // K5 over TMA-staged ray stages (MRF_K5=staged); default: per-class warp kernels
    bool vtr_valid = false; // per-voxel transpose built for the current graph
    bool hist_valid = false; // vox_count (voxel degrees) computed for the current graph
    float prior = 0.5f;
    double L0 = 0.0;
    MsgParams mp{};
    int rank = 0, world = 1, comm_mode = MRF_COMM_NCCL;
    ncclComm_t comm = nullptr;
    cudaStream_t own_stream = nullptr, stream = nullptr;
    // K5 length classes run concurrently on side streams (fork/join with events on `stream`), so
    // one class kernel's tail overlaps the next class's work
    static constexpr int kMaxSide = 8;
    int k5_streams = 8;  // MRF_K5_STREAMS (1 = all classes on `stream`)
    cudaStream_t side[kMaxSide] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[kMaxSide] = {};
    cudaEvent_t ev_mf[4] = {};  // matrix-free pipeline: walk done [2], K5 done [2] (per scratch set)
    std::string err;
    mrf_status sticky = MRF_OK;

    long long R = 0, E = 0;  // rays (owned pixels) and incidence slots (ray segments padded to 4)
    long long E_real = 0;    // incidences (counted by the fills on the device; see sync_fill)
    bool fill_pending = false;
    bool fill_rb_pending = false;    // the last fill's counters are on their way to pinned[32..57]
    // rays per K5 length class and the longest ray, counted by the fills since the reset
    // (counters[kClassCtr ..]); fill_classes_ok: read back with the last fill's counters
    long long fill_class_n[kNumClasses + 1] = {};
    bool fill_classes_ok = false;
    long long fill_rb_new_slots = -1;
    // frames added without a host round trip: their exact E (row_ptr[R]) and invalid / dropped
    // counts (counters[2..3], accumulating) are read when something needs them (resolve_E);
    // E_bound bounds what they added, so that the 2^31 capacity check needs no round trip while
    // E + E_bound stays below it
    bool E_unresolved = false;
    long long E_bound = 0;
    long long ray_slots_max = 0;  // pad8(1 + sum_k (dims_k + ceil(M / res))), M the largest margin
    long long n_invalid = 0, n_dropped = 0, n_kept = 0;
    DBuf<int32_t> n_r;
    DBuf<int8_t> status;
    DBuf<RayInfo> ray_z;  // per-ray RayInfo
    DBuf<long long> row_ptr;
    DBuf<int32_t> vid;
    DBuf<int16_t> off_q;
    DBuf<float> lnu;      // log nu per incidence (interpolated at fill time; read by K5)
    DBuf<int32_t> lam;
    DBuf<int32_t> tr;
    DBuf<int32_t> vox_count, cursor, n_items, flags;
    DBuf<long long> col_ptr, item_ptr, pos;
    DBuf<int2> items;
    long long n_items_total = 0;
    DBuf<int32_t> tile_runs, tile_cursor;
    DBuf<long long> tile_ptr;
    DBuf<Run> runs;
    // tile runs as the DDA fills build them (unsorted, with bucket keys): the transpose is then a
    // bucket pass over them (run_bucket) instead of a vid re-read (run_fill).  runs_ok: every run
    // since the last reset reached the sink (its capacity is sized from run_ratio runs per new
    // slot; an overflow falls back to run_fill and raises run_ratio).  MRF_RUN_FILL=1: always
    // run_fill (ablation).
    DBuf<Run> runs_all;
    DBuf<int32_t> run_keys;
    long long runs_emitted = 0, runs_cap = 0;
    bool runs_ok = true, run_fill_forced = false;
    double run_ratio = 0.125;        // (MRF_RUN_RATIO: the first estimate; tests force an overflow)
    long long run_slack = 65536;     // (MRF_RUN_SLACK)
    DBuf<int2> bitems;
    DBuf<int4> blk;             // K6b pixel blocks (build_blocks)
    std::vector<int4> h_blk;
    long long n_blk = 0;
    std::vector<int2> h_items;  // host copy of the K6 work list
    long long n_runs = 0, n_bitems = 0;
    DBuf<long long> T, T_part;
    // world > 1 (NCCL): the all-reduce covers only the tiles some rank touches:
    // a touched-tile mask, ncclMax-reduced once per graph change, gives tile -> compact position;
    // K6 writes its sums there, NCCL reduces n_act_tiles * 16384 slots in place, and a scatter
    // puts them back into T
    bool compact = false;
    bool force_compact = false;  // MRF_COMPACT=1: the same compacted path at world == 1 (tests)
    long long n_act_tiles = 0;
    std::vector<int32_t> tile_nr;   // runs per tile (host copy, from build_tile_runs)
    DBuf<int32_t> tile_map, tile_of;
    DBuf<uint8_t> touched;
    DBuf<long long> T_c;
    DBuf<float2> lutp;
    // per-patch noise (R25, mrf_set_patch_noise): fp64 coefficients for the margins, fp32 pairs
    // for log nu; the frames must lie inside the patch grid
    DBuf<double> pcoef_d;
    DBuf<float4> pcoef_f;
    int patch_px = 0, patch_nx = 0, patch_ny = 0;
    DBuf<float> depth_stage, marg;
    // frames added since the last fill: the walk (K3) of all of them runs as one launch when
    // the graph is next needed (sync_fill)
    DBuf<float> depth_all;       // their depth images
    long long depth_used = 0;
    std::vector<FrameDesc> pend;
    DBuf<FrameDesc> d_frames;
    // frames whose K1 (ray setup + length bound) and row scan have not run yet: they run as one
    // launch + one scan when something needs the layout (flush_k1) -- add_frame itself launches
    // nothing while the capacity bound holds
    std::vector<FrameDesc> k1_pend;
    DBuf<FrameDesc> d_k1_frames;
    DBuf<int> d_k1_cta0;
    long long k1_R0 = 0;
    DBuf<int> d_cta0;
    long long E_filled = 0, R_filled = 0;  // incidences / rays already walked
    DBuf<int8_t> eval_cls;
    DBuf<long long> scan_scratch;
    DBuf<unsigned long long> counters;
    DBuf<int32_t> class_all;                 // ray ids grouped by K5 class
    DBuf<int4> class_desc;                   // per class_all entry: {row_ptr, n, frame, ray id} (launch_class_desc)
    DBuf<unsigned long long> class_cnt;      // [counts | cursors] per class
    long long class_off[kNumClasses] = {};
    DBuf<Stage> stages;
    long long n_stages = 0;
    long long class_n[kNumClasses] = {};
    DBuf<float> long_scratch;
    long long long_scratch_per_warp = 0;
    int n_warps_long = 0;
    long long* pinned = nullptr;  // small readbacks
    std::vector<FrameRec> frames;
    bool dirty = true;

    bool prof = false;
    std::vector<ProfEvent> events;
    std::vector<cudaEvent_t> ev_pool;  // recycled profiling events (creating two per scope costs host time)
    long long prof_launch[MRF_K_COUNT] = {};
    double prof_ms[MRF_K_COUNT] = {};
    long long launches = 0;
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

mrf_status set_err(mrf_ctx* c, mrf_status st, const std::string& msg) {
    c->err = msg;
    if (st == MRF_ERR_CUDA || st == MRF_ERR_NCCL) c->sticky = st;
    return st;
}

mrf_status cuda_fail(mrf_ctx* c, cudaError_t e, const char* what, int line) {
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        return set_err(c, MRF_ERR_OUT_OF_MEMORY, std::string("out of device memory: ") + what);
    }
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error %s (%s) at mrf_api.cu:%d in %s", cudaGetErrorName(e),
             cudaGetErrorString(e), line, what);
    return set_err(c, MRF_ERR_CUDA, buf);
}

#define CK(call)                                                      \
    do {                                                              \
        cudaError_t e_ = (call);                                      \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, #call, __LINE__); \
    } while (0)

#define CK_LAUNCH(kind_, nk_)                                                   \
    do {                                                                        \
        c->launches += (nk_);                                                   \
        c->prof_launch[kind_] += (nk_);                                         \
        cudaError_t e_ = cudaGetLastError();                                    \
        if (e_ != cudaSuccess) return cuda_fail(c, e_, "kernel launch", __LINE__); \
    } while (0)

#define NCK(call)                                                                              \
    do {                                                                                       \
        ncclResult_t r_ = (call);                                                              \
        if (r_ != ncclSuccess)                                                                 \
            return set_err(c, MRF_ERR_NCCL, std::string("NCCL error: ") + ncclGetErrorString(r_) + " in " #call); \
    } while (0)

#define ENTER(ctx)                                                   \
    if (!(ctx)) return MRF_ERR_INVALID_ARG;                          \
    mrf_ctx* c = (ctx);                                              \
    if (c->sticky != MRF_OK) return c->sticky;                       \
    DeviceGuard guard_(c->device)

bool finite_all(const double* a, int n) {
    for (int i = 0; i < n; ++i)
        if (!std::isfinite(a[i])) return false;
    return true;
}

// Event pair around a group of launches when profiling is on.
struct ProfScope {
    mrf_ctx* c;
    int kind;
    cudaEvent_t a = nullptr, b = nullptr;
    static cudaEvent_t get(mrf_ctx* c) {
        cudaEvent_t e = nullptr;
        if (!c->ev_pool.empty()) {
            e = c->ev_pool.back();
            c->ev_pool.pop_back();
        } else {
            cudaEventCreate(&e);
        }
        return e;
    }
    ProfScope(mrf_ctx* c_, int k) : c(c_), kind(k) {
        if (!c->prof || k < 0) return;
        a = get(c);
        b = get(c);
        cudaEventRecord(a, c->stream);
    }
    ~ProfScope() {
        if (!a) return;
        cudaEventRecord(b, c->stream);
        c->events.push_back({kind, a, b});
    }
};

mrf_status scan(mrf_ctx* c, const int32_t* in, long long* out, long long n, long long offset) {
    CK(c->scan_scratch.ensure((size_t)scan_scratch_elems(n), 0, c->stream));
    ProfScope ps(c, MRF_K_SCAN);
    launch_exclusive_scan(in, out, n, offset, c->scan_scratch.p, c->stream);
    CK_LAUNCH(MRF_K_SCAN, n > 0 ? 3 : 1);
    return MRF_OK;
}

mrf_status read_ll(mrf_ctx* c, const long long* dev, long long* out) {
    CK(cudaMemcpyAsync(c->pinned, dev, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *out = c->pinned[0];
    return MRF_OK;
}

// K1 and the row scan of the frames added since the last batch (one launch each).
mrf_status flush_k1(mrf_ctx* c) {
    if (c->k1_pend.empty()) return MRF_OK;
    const int nf = (int)c->k1_pend.size();
    std::vector<int> cta0((size_t)nf + 1, 0);
    for (int k = 0; k < nf; ++k) {
        const long long n_pix = (long long)c->k1_pend[k].rows_owned * c->k1_pend[k].W;
        cta0[k + 1] = cta0[k] + (int)((n_pix + 127) / 128);
    }
    CK(c->d_k1_frames.ensure((size_t)nf, 0, c->stream));
    CK(c->d_k1_cta0.ensure((size_t)nf + 1, 0, c->stream));
    CK(cudaMemcpyAsync(c->d_k1_frames.p, c->k1_pend.data(), sizeof(FrameDesc) * nf, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_k1_cta0.p, cta0.data(), sizeof(int) * (nf + 1), cudaMemcpyHostToDevice, c->stream));
    {
        ProfScope ps(c, MRF_K_RAYGEN_COUNT);
        launch_raygen_count_batch(c->d_k1_frames.p, c->d_k1_cta0.p, nf, cta0[nf], c->grid, c->noise, c->depth_all.p,
                                  c->n_r.p, c->status.p, c->ray_z.p, c->counters.p + 2, c->stream);
        CK_LAUNCH(MRF_K_RAYGEN_COUNT, cta0[nf] > 0 ? 1 : 0);
    }
    const long long n = c->R - c->k1_R0;
    if (n > 0) {  // row_ptr[k1_R0] holds the running E on the device
        CK(c->scan_scratch.ensure((size_t)scan_scratch_elems(n), 0, c->stream));
        ProfScope ps(c, MRF_K_SCAN);
        launch_exclusive_scan_dev(c->n_r.p + c->k1_R0, c->row_ptr.p + c->k1_R0, n, c->row_ptr.p + c->k1_R0,
                                  c->scan_scratch.p, c->stream);
        CK_LAUNCH(MRF_K_SCAN, 3);
    }
    c->k1_pend.clear();  // (pageable host -> device copies are staged before they return)
    return MRF_OK;
}

// Exact E and invalid / dropped counts of the frames added since the last round trip.
mrf_status resolve_E(mrf_ctx* c) {
    {
        mrf_status sk = flush_k1(c);
        if (sk != MRF_OK) return sk;
    }
    if (!c->E_unresolved) return MRF_OK;
    CK(cudaMemcpyAsync(c->pinned, c->row_ptr.p + c->R, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(c->pinned + 1, c->counters.p + 2, 2 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->E = c->pinned[0];
    c->n_invalid += c->pinned[1];
    c->n_dropped += c->pinned[2];
    c->n_kept = c->R - c->n_invalid - c->n_dropped;
    CK(cudaMemsetAsync(c->counters.p + 2, 0, 2 * sizeof(unsigned long long), c->stream));
    c->E_unresolved = false;
    c->E_bound = 0;
    return MRF_OK;
}

// ---- matrix-free mode (NEXT #1)
static void mf_dbg(mrf_ctx* c, const char* what) {
    static const bool on = getenv("MRF_SYNC_DEBUG") != nullptr;
    if (!on) return;
    cudaError_t e = cudaStreamSynchronize(c->stream);
    fprintf(stderr, "[mf] %s: %s\n", what, cudaGetErrorString(e));
}
// Chunks of c->mf frames over every frame so far; the scratch holds the largest chunk's slots.
mrf_status mf_rechunk(mrf_ctx* c) {
    const int nf = (int)c->mf_frames.size();
    c->mf_frame_e.assign((size_t)nf + 1, 0);
    for (int k = 0; k <= nf; ++k) {
        const long long r = k < nf ? c->mf_frames[k].ray_base : c->R;
        CK(cudaMemcpyAsync(&c->mf_frame_e[k], c->row_ptr.p + r, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    c->mf_chunks.clear();
    long long big = 0;
    for (int f0 = 0; f0 < nf; f0 += c->mf) {
        const int f1 = std::min(f0 + c->mf, nf);
        mrf_ctx::MfChunk ch{f0, f1, c->mf_frames[f0].ray_base,
                            f1 < nf ? c->mf_frames[f1].ray_base : c->R, c->mf_frame_e[f0], c->mf_frame_e[f1]};
        big = std::max(big, ch.e1 - ch.e0);
        c->mf_chunks.push_back(ch);
    }
    CK(c->s_vid.ensure((size_t)big + kPadElems, 0, c->stream));
    CK(c->s_off.ensure((size_t)big + kPadElems, 0, c->stream));
    CK(c->s_lnu.ensure((size_t)big + kPadElems, 0, c->stream));
    if (c->kf_chunked()) CK(c->lam_chunk.ensure((size_t)big + kPadElems, 0, c->stream));
    // the slack after the largest chunk is read (masked) by the last rays' lanes: valid ids
    CK(cudaMemsetAsync(c->s_vid.p, 0, sizeof(int32_t) * c->s_vid.cap, c->stream));
    if (c->k5_streams >= 2 && c->mf_chunks.size() > 1) {
        CK(c->s_vid2.ensure((size_t)big + kPadElems, 0, c->stream));
        CK(c->s_off2.ensure((size_t)big + kPadElems, 0, c->stream));
        CK(c->s_lnu2.ensure((size_t)big + kPadElems, 0, c->stream));
        CK(cudaMemsetAsync(c->s_vid2.p, 0, sizeof(int32_t) * c->s_vid2.cap, c->stream));
    }
    CK(c->d_frames.ensure((size_t)std::max(nf, 1), 0, c->stream));
    if (nf)
        CK(cudaMemcpyAsync(c->d_frames.p, c->mf_frames.data(), sizeof(FrameDesc) * nf, cudaMemcpyHostToDevice,
                           c->stream));
    return MRF_OK;
}

// The sink of the next fill over new_slots incidence slots (capacity from run_ratio; see runs_ok).
mrf_status run_sink(mrf_ctx* c, long long new_slots, RunSink& sink) {
    sink = RunSink{nullptr, nullptr, nullptr, 0};
    if (c->any_block()) {  // K6b needs no tile runs (a later tile-run K6 would re-read vid)
        c->runs_ok = false;
        return MRF_OK;
    }
    if (c->run_fill_forced || !c->runs_ok) return MRF_OK;
    const long long need = c->runs_emitted + (long long)std::ceil((double)new_slots * c->run_ratio) + c->run_slack;
    if (need > c->runs_cap) {
        CK(c->runs_all.ensure((size_t)need, (size_t)std::min(c->runs_emitted, c->runs_cap), c->stream));
        CK(c->run_keys.ensure((size_t)need, (size_t)std::min(c->runs_emitted, c->runs_cap), c->stream));
        c->runs_cap = (long long)std::min(c->runs_all.cap, c->run_keys.cap);
    }
    // unused slots of the warps' blocks keep key -1
    CK(cudaMemsetAsync(c->run_keys.p + c->runs_emitted, 0xff, sizeof(int32_t) * (size_t)(c->runs_cap - c->runs_emitted),
                       c->stream));
    sink = RunSink{c->runs_all.p, c->run_keys.p, c->counters.p + 16, c->runs_cap};
    return MRF_OK;
}

// After a fill (counters read back): how many runs the sink took; an overflow disables it until
// the next reset (the transpose falls back to run_fill) and raises run_ratio for the next time.
void run_sink_done(mrf_ctx* c, long long emitted_total, long long new_slots) {
    if (c->run_fill_forced || !c->runs_ok) return;
    const long long added = emitted_total - c->runs_emitted;
    if (new_slots > 0) c->run_ratio = std::max(c->run_ratio, 1.25 * (double)added / (double)new_slots);
    if (emitted_total > c->runs_cap) c->runs_ok = false;
    c->runs_emitted = emitted_total;
}

// Walk frames [f0, f1) of one chunk (the DDA fill + log nu) into the scratch, which stands for
// the incidence slots [e0, ...) of chunk `ch` (pointers shifted by e0).  count: also count the
// tile runs and the incidences (first walk of new frames only).
mrf_status mf_walk(mrf_ctx* c, const mrf_ctx::MfChunk& ch, int f0, int f1, bool count, cudaStream_t st = nullptr,
                   int set = 0) {
    if (f0 >= f1) return MRF_OK;
    const bool own = st == nullptr;  // on the ctx stream (profiled); else a pipeline stream
    if (own) st = c->stream;
    int32_t* sv = set ? c->s_vid2.p : c->s_vid.p;
    int16_t* so = set ? c->s_off2.p : c->s_off.p;
    float* sl = set ? c->s_lnu2.p : c->s_lnu.p;
    std::vector<int> cta0((size_t)(f1 - f0) + 1, 0);
    for (int k = f0; k < f1; ++k) {
        const long long n_pix = (long long)c->mf_frames[k].rows_owned * c->mf_frames[k].W;
        cta0[k - f0 + 1] = cta0[k - f0] + (int)((n_pix + kFillThreads - 1) / kFillThreads);
    }
    // one cta table per scratch set (the pipeline's two walks are in flight on one stream, so
    // the tables are written in stream order anyway)
    CK(c->d_cta_tmp.ensure(2 * (size_t)c->mf + 2, 0, c->stream));
    int* dc = c->d_cta_tmp.p + set * ((size_t)c->mf + 1);
    CK(cudaMemcpyAsync(dc, cta0.data(), sizeof(int) * cta0.size(), cudaMemcpyHostToDevice, st));
    const long long r0 = c->mf_frames[f0].ray_base;
    const long long r1 = f1 < (int)c->mf_frames.size() ? c->mf_frames[f1].ray_base : c->R;
    RunSink sink{nullptr, nullptr, nullptr, 0};
    if (count) {  // the first walk of new frames builds their tile runs
        mrf_status ss = run_sink(c, c->mf_frame_e[f1] - c->mf_frame_e[f0], sink);
        if (ss != MRF_OK) return ss;
    }
    ProfScope ps(c, own ? MRF_K_DDA_FILL : -1);
    const bool fused = count && c->mf_fused;
    launch_dda_fill(c->d_frames.p + f0, dc, f1 - f0, cta0.back(), r0, r1 - r0, c->grid, c->noise, c->mp,
                    c->depth_all.p, c->row_ptr.p, c->ray_z.p, sv - ch.e0, so - ch.e0, sl - ch.e0,
                    count ? c->tile_runs.p : nullptr, c->counters.p + (count ? 10 : 12), sink,
                    fused ? c->ray_seg.p : nullptr, count ? c->counters.p + kClassCtr : nullptr, nullptr, st);
    if (fused) {  // K12: the first cell of every K5 chunk of these rays
        launch_ck_extract(r1 - r0, c->row_ptr.p + r0, c->ray_z.p + r0, sv - ch.e0, c->ck.p, c->ray_seg.p + r0, st);
    }
    if (count) {  // the sink's count is read back per chunk walk (few chunks; first use only)
        long long emitted = 0;
        mrf_status sr = read_ll(c, reinterpret_cast<long long*>(c->counters.p + 16), &emitted);
        if (sr != MRF_OK) return sr;
        run_sink_done(c, emitted, c->mf_frame_e[f1] - c->mf_frame_e[f0]);
    }
    CK_LAUNCH(MRF_K_DDA_FILL, (cta0.back() > 0 ? 1 : 0) + ((!MRF_FILL_LNU || c->mp.pcoef) && r1 > r0 ? 1 : 0) + (fused && r1 > r0 ? 1 : 0));
    mf_dbg(c, count ? "walk(count)" : "walk");
    return MRF_OK;
}

// The counters of the last fill (pinned[32..34]): incidences, bound overflows, tile runs emitted.
mrf_status fill_readback(mrf_ctx* c) {
    if (!c->fill_rb_pending) return MRF_OK;
    CK(cudaStreamSynchronize(c->stream));
    c->fill_rb_pending = false;
    if (c->fill_rb_new_slots >= 0) run_sink_done(c, c->pinned[34], c->fill_rb_new_slots);
    c->E_real = c->pinned[32];
    for (int k = 0; k <= kNumClasses; ++k) c->fill_class_n[k] = c->pinned[36 + k];  // (+ longest ray)
    c->fill_classes_ok = true;
    if (c->pinned[33]) {
        c->sticky = MRF_ERR_STATE;
        c->err = "internal: a DDA walk exceeded its precomputed bound";
        return MRF_ERR_STATE;
    }
    return MRF_OK;
}

// The DDA fills count their incidences (and any bound overflow, which K1's bound excludes) on
// the device, counters[10..11]; read them once when something needs E_real (need_counts = false:
// later, by fill_readback).
mrf_status sync_fill(mrf_ctx* c, bool need_counts = true) {
    if (!c->fill_pending) {
        if (need_counts) return fill_readback(c);
    }
    {
        mrf_status sr = resolve_E(c);
        if (sr != MRF_OK) return sr;
    }
    if (!c->fill_pending) return MRF_OK;
    long long new_slots = -1;  // slots walked by the stored-graph fill below (its run sink)
    if (!c->pend.empty() && c->grid.bmask) {
        // Sparse bricks: every frame is allocated by now (R23), so the per-ray counts of add_frame
        // -- made before the later frames' bricks existed -- are redone against the allocation and
        // the segments laid out again.  Frames added after the graph was used grow the allocation
        // under the rays already walked: then every frame is walked again (R24) and the messages
        // move to the new layout (lambda_merge, after the fill).
        if (c->sp_rebuild) {
            const long long R0 = c->R_filled;
            c->sp_R_old = R0;
            CK(c->rp_old.ensure((size_t)R0 + 1, 0, c->stream));
            CK(c->ri_old.ensure((size_t)std::max<long long>(R0, 1), 0, c->stream));
            CK(cudaMemcpyAsync(c->rp_old.p, c->row_ptr.p, sizeof(long long) * (R0 + 1), cudaMemcpyDeviceToDevice,
                               c->stream));
            if (R0)
                CK(cudaMemcpyAsync(c->ri_old.p, c->ray_z.p, sizeof(RayInfo) * R0, cudaMemcpyDeviceToDevice, c->stream));
            std::swap(c->vid, c->vid_old);
            std::swap(c->lam, c->lam_old);
            c->pend.insert(c->pend.begin(), c->sp_frames.begin(), c->sp_frames.end());
            c->sp_frames.clear();
            c->E_filled = 0;
            c->R_filled = 0;
            CK(cudaMemsetAsync(c->tile_runs.p, 0, sizeof(int32_t) * (size_t)(c->NT * c->n_bucket_groups()), c->stream));
            CK(cudaMemsetAsync(c->counters.p + 10, 0, 2 * sizeof(unsigned long long), c->stream));
            CK(cudaMemsetAsync(c->counters.p + 16, 0, sizeof(unsigned long long), c->stream));
            CK(cudaMemsetAsync(c->counters.p + kClassCtr, 0, (kNumClasses + 1) * sizeof(unsigned long long), c->stream));
            c->runs_emitted = 0;
            c->runs_ok = true;
        }
        long long E = c->E_filled;
        for (const FrameDesc& f : c->pend) {
            const long long Rf = (long long)f.rows_owned * f.W;
            CK(cudaMemsetAsync(c->counters.p + 2, 0, 2 * sizeof(unsigned long long), c->stream));
            {
                ProfScope ps(c, MRF_K_RAYGEN_COUNT);
                FrameDesc fc = f;
                fc.skip_count = 0;
                launch_raygen_count(fc, c->grid, c->noise, c->depth_all.p + f.depth_off, c->n_r.p, c->status.p,
                                    c->ray_z.p, c->counters.p + 2, c->stream);
                CK_LAUNCH(MRF_K_RAYGEN_COUNT, Rf > 0 ? 1 : 0);
            }
            mrf_status st;
            if ((st = scan(c, c->n_r.p + f.ray_base, c->row_ptr.p + f.ray_base, Rf, E)) != MRF_OK) return st;
            if ((st = read_ll(c, c->row_ptr.p + f.ray_base + Rf, &E)) != MRF_OK) return st;
            if (E >= (1LL << 31) - kPadElems)  // the frames stay pending: mrf_reset starts over
                return set_err(c, MRF_ERR_CAPACITY,
                               "sparse bricks: the final allocation gives more than 2^31 incidence slots");
        }
        CK(cudaMemsetAsync(c->counters.p + 2, 0, 2 * sizeof(unsigned long long), c->stream));  // recounted frames
        c->E = E;
    }
    if (!c->pend.empty() && c->mf) {
        // matrix-free: only lambda is stored per incidence; the new frames are walked once into
        // the scratch to count their runs and incidences
        if (!c->kf_chunked()) {  // (keyframe averages + fused walks: no per-incidence messages)
            CK(c->lam.ensure((size_t)c->E + kPadElems, (size_t)c->E_filled, c->stream));
            CK(cudaMemsetAsync(c->lam.p + c->E_filled, 0, sizeof(int32_t) * (size_t)(c->E - c->E_filled), c->stream));
        }
        if (c->mf_fused) {
            CK(c->ray_seg.ensure((size_t)std::max<long long>(c->R, 1), (size_t)c->R_filled, c->stream));
            CK(c->ck.ensure((size_t)(c->E / 4 + 4), (size_t)(c->E_filled / 4), c->stream));
        }
        const int first_new = (int)c->mf_frames.size();
        c->mf_frames.insert(c->mf_frames.end(), c->pend.begin(), c->pend.end());
        c->pend.clear();
        mrf_status st;
        if ((st = mf_rechunk(c)) != MRF_OK) return st;
        for (const auto& ch : c->mf_chunks)
            if ((st = mf_walk(c, ch, std::max(ch.f0, first_new), ch.f1, true)) != MRF_OK) return st;
        c->E_filled = c->E;
        c->R_filled = c->R;
    }
    if (!c->pend.empty()) {
        const size_t ne = (size_t)c->E + kPadElems;
        CK(c->vid.ensure(ne, (size_t)c->E_filled, c->stream));
        // the slack after the last segment is read (masked) by the last rays' K5 lanes
        CK(cudaMemsetAsync(c->vid.p + c->E, 0, sizeof(int32_t) * kPadElems, c->stream));
        CK(c->off_q.ensure(ne, (size_t)c->E_filled, c->stream));
        CK(c->lnu.ensure(ne, (size_t)c->E_filled, c->stream));
        CK(c->lam.ensure(ne, (size_t)c->E_filled, c->stream));  // (the fill zeroes the new slots' messages)
        const int nf = (int)c->pend.size();
        std::vector<int> cta0((size_t)nf + 1, 0);
        for (int k = 0; k < nf; ++k) {
            const long long n_pix = (long long)c->pend[k].rows_owned * c->pend[k].W;
            cta0[k + 1] = cta0[k] + (int)((n_pix + kFillThreads - 1) / kFillThreads);
        }
        CK(c->d_frames.ensure((size_t)nf, 0, c->stream));
        CK(c->d_cta0.ensure((size_t)nf + 1, 0, c->stream));
        CK(cudaMemcpyAsync(c->d_frames.p, c->pend.data(), sizeof(FrameDesc) * nf, cudaMemcpyHostToDevice, c->stream));
        CK(cudaMemcpyAsync(c->d_cta0.p, cta0.data(), sizeof(int) * (nf + 1), cudaMemcpyHostToDevice, c->stream));
        RunSink sink;
        {
            mrf_status ss = run_sink(c, c->E - c->E_filled, sink);
            if (ss != MRF_OK) return ss;
        }
        new_slots = c->E - c->E_filled;
        if (c->any_block()) c->tile_counts_ok = false;  // (K6b: the fill tracks no tile runs)
        {
            ProfScope ps(c, MRF_K_DDA_FILL);
            launch_dda_fill(c->d_frames.p, c->d_cta0.p, nf, cta0[nf], c->R_filled, c->R - c->R_filled, c->grid,
                            c->noise, c->mp, c->depth_all.p, c->row_ptr.p, c->ray_z.p, c->vid.p, c->off_q.p,
                            c->lnu.p, c->any_block() ? nullptr : c->tile_runs.p, c->counters.p + 10, sink, nullptr,
                            c->counters.p + kClassCtr,
                            c->lam.p, c->stream);
            CK_LAUNCH(MRF_K_DDA_FILL, (cta0[nf] > 0 ? 1 : 0) + ((!MRF_FILL_LNU || c->mp.pcoef) && c->R > c->R_filled ? 1 : 0));
        }
        if (c->grid.bmask) {  // the depth images stay: a later keyframe may grow the allocation (R24)
            c->sp_frames.insert(c->sp_frames.end(), c->pend.begin(), c->pend.end());
        } else {
            c->depth_used = 0;
        }
        c->pend.clear();
        c->E_filled = c->E;
        c->R_filled = c->R;
        if (c->sp_rebuild) {  // the old rays' messages to the new layout; new incidences start at 0
            CK(cudaMemsetAsync(c->counters.p + 17, 0, sizeof(unsigned long long), c->stream));
            launch_lambda_merge(c->sp_R_old, c->rp_old.p, c->ri_old.p, c->vid_old.p, c->lam_old.p, c->row_ptr.p,
                                c->ray_z.p, c->vid.p, c->lam.p, c->counters.p + 17, c->stream);
            CK_LAUNCH(MRF_K_DDA_FILL, c->sp_R_old > 0 ? 1 : 0);
            long long lost = 0;
            mrf_status sr = read_ll(c, reinterpret_cast<long long*>(c->counters.p + 17), &lost);
            if (sr != MRF_OK) return sr;
            c->vid_old.release();
            c->lam_old.release();
            c->sp_rebuild = false;
            if (lost) {
                c->sticky = MRF_ERR_STATE;
                c->err = "internal: a re-walked ray lost incidences of its earlier walk";
                return MRF_ERR_STATE;
            }
        }
    }
    // the fill's counters come back with the next round trip (fill_readback): the transpose build
    // makes one anyway, so the fill and what follows it are enqueued without a wait here
    CK(cudaMemcpyAsync(c->pinned + 32, c->counters.p + 10, 2 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(c->pinned + 34, c->counters.p + 16, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaMemcpyAsync(c->pinned + 36, c->counters.p + kClassCtr, (kNumClasses + 1) * sizeof(long long),
                       cudaMemcpyDeviceToHost, c->stream));
    c->fill_pending = false;
    c->fill_rb_pending = true;
    c->fill_rb_new_slots = new_slots;
    return need_counts ? fill_readback(c) : MRF_OK;
}

// Per-voxel transpose (col_ptr over belief slots, tr) + its K6 work list.  Built by prepare()
// only for the per-voxel K6 ablation, and lazily for mrf_export_transpose.
// Voxel degrees on demand (not needed by the BP iteration).
mrf_status voxel_histogram(mrf_ctx* c) {
    if (c->hist_valid) return MRF_OK;
    CK(cudaMemsetAsync(c->vox_count.p, 0, sizeof(int32_t) * c->VI, c->stream));
    {
        ProfScope ps(c, MRF_K_TRANSPOSE);
        launch_vox_hist(c->R, c->row_ptr.p, c->ray_z.p, c->vid.p, c->vox_count.p, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
    }
    c->hist_valid = true;
    return MRF_OK;
}

mrf_status build_voxel_transpose(mrf_ctx* c) {
    if (c->vtr_valid) return MRF_OK;
    const long long VI = c->VI;
    mrf_status st;
    if ((st = voxel_histogram(c)) != MRF_OK) return st;
    if ((st = scan(c, c->vox_count.p, c->col_ptr.p, VI, 0)) != MRF_OK) return st;
    CK(c->tr.ensure((size_t)c->E + kPadElems, 0, c->stream));
    CK(cudaMemsetAsync(c->cursor.p, 0, sizeof(int32_t) * VI, c->stream));
    {
        ProfScope ps(c, MRF_K_TRANSPOSE);
        launch_transpose_fill(c->R, c->row_ptr.p, c->ray_z.p, c->vid.p, c->col_ptr.p, c->cursor.p, c->tr.p, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
        launch_item_counts(VI, c->vox_count.p, c->n_items.p, kVoxelChunk, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, 1);
    }
    if ((st = scan(c, c->n_items.p, c->item_ptr.p, VI, 0)) != MRF_OK) return st;
    if ((st = read_ll(c, c->item_ptr.p + VI, &c->n_items_total)) != MRF_OK) return st;
    CK(c->items.ensure((size_t)std::max(1LL, c->n_items_total), 0, c->stream));
    {
        ProfScope ps(c, MRF_K_TRANSPOSE);
        launch_item_fill(VI, c->n_items.p, c->item_ptr.p, c->items.p, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, 1);
    }
    c->vtr_valid = true;
    return MRF_OK;
}

// Tile-run transpose (runs grouped by tile) + its K6 work list.  The runs per tile were counted
// by the DDA fills.
// The runs per tile bucket, counted from vid (run_fill without placing) when the fills did not
// count them (K6b mode; needed after a demotion to the tile runs, or for the touched tiles of the
// compacted reduction).
mrf_status ensure_tile_counts(mrf_ctx* c) {
    if (c->tile_counts_ok) return MRF_OK;
    const long long NT = c->NT * c->n_bucket_groups();
    CK(cudaMemsetAsync(c->tile_runs.p, 0, sizeof(int32_t) * (size_t)NT, c->stream));
    {
        ProfScope ps(c, MRF_K_TRANSPOSE);
        launch_run_fill(c->R, c->row_ptr.p, c->ray_z.p, c->vid.p, nullptr, c->tile_runs.p, c->fb() ? (int)c->NT : 0,
                        nullptr, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
    }
    c->tile_counts_ok = true;
    return MRF_OK;
}

mrf_status build_tile_runs(mrf_ctx* c) {
    // buckets: the tiles (per-ray mode), or (frame, tile) pairs frame-major (keyframe averages)
    const long long NT = c->NT * c->n_bucket_groups();
    mrf_status st;
    if ((st = ensure_tile_counts(c)) != MRF_OK) return st;
    CK(c->tile_ptr.ensure((size_t)NT + 1, 0, c->stream));
    CK(c->tile_cursor.ensure((size_t)NT, 0, c->stream));
    if ((st = scan(c, c->tile_runs.p, c->tile_ptr.p, NT, 0)) != MRF_OK) return st;
    // the runs per bucket on the host (one round trip: their sum is n_runs, and they make the K6
    // work list below)
    std::vector<int32_t> nr((size_t)NT);
    CK(cudaMemcpyAsync(nr.data(), c->tile_runs.p, sizeof(int32_t) * NT, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if ((st = fill_readback(c)) != MRF_OK) return st;  // (already here: no further wait)
    c->n_runs = 0;
    for (int32_t x : nr) c->n_runs += x;
    CK(c->runs.ensure((size_t)std::max(1LL, c->n_runs), 0, c->stream));
    CK(cudaMemsetAsync(c->tile_cursor.p, 0, sizeof(int32_t) * NT, c->stream));
    const bool from_sink = c->runs_ok && !c->run_fill_forced;
    if (from_sink) {  // the runs the fills built, placed by bucket (no vid re-read, no re-walk)
        ProfScope ps(c, MRF_K_TRANSPOSE);
        launch_run_bucket(c->runs_emitted, c->runs_all.p, c->run_keys.p, c->tile_ptr.p, c->tile_cursor.p, c->runs.p,
                          c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, c->runs_emitted > 0 ? 1 : 0);
    } else {
        ProfScope ps(c, MRF_K_TRANSPOSE);
        if (c->mf) {  // per chunk: walk into the scratch, then place the chunk's runs
            for (const auto& ch : c->mf_chunks) {
                mrf_status sw;
                if ((sw = mf_walk(c, ch, ch.f0, ch.f1, false)) != MRF_OK) return sw;
                launch_run_fill(ch.r1 - ch.r0, c->row_ptr.p + ch.r0, c->ray_z.p + ch.r0, c->s_vid.p - ch.e0,
                                c->tile_ptr.p, c->tile_cursor.p, c->fb() ? (int)c->NT : 0, c->runs.p, c->stream);
                CK_LAUNCH(MRF_K_TRANSPOSE, ch.r1 > ch.r0 ? 1 : 0);
                mf_dbg(c, "run_fill");
            }
        } else {
            launch_run_fill(c->R, c->row_ptr.p, c->ray_z.p, c->vid.p, c->tile_ptr.p, c->tile_cursor.p,
                            c->fb() ? (int)c->NT : 0, c->runs.p, c->stream);
            CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
        }
    }
    // Work item size: large items amortise the per-item accumulator zeroing and flush, but about a
    // dozen items per SM are needed for the dynamic schedule to even out the tiles' last chunks
    // (frames30: 8192 -> 24576 runs, 2.46 -> 2.39 ms; at 8 ranks 8192 stays best).
    if (!c->k6_item_fixed)
        c->k6_item = (int)std::min<long long>(24576, std::max<long long>(8192, c->n_runs / ((long long)c->sms * 13)));
    // K6 work list, j-major: item j of every tile, then item j+1 ...  Runs land in a tile in
    // roughly ray order, so the items that run concurrently read nearby message ranges (L2 reuse).
    c->tile_nr = nr;
    std::vector<int2>& items = c->h_items;  // (kept: the copy below is asynchronous)
    items.clear();
    for (int j = 0;; ++j) {
        bool any = false;
        for (long long t = 0; t < NT; ++t) {
            if ((long long)j * c->k6_item < nr[t]) {
                items.push_back(make_int2((int)t, j));
                any = true;
            }
        }
        if (!any) break;
    }
    if (c->k6_lpt) {  // largest items first (the dynamic schedule then ends on the small ones)
        auto size = [&](const int2& it) { return std::min<long long>(c->k6_item, nr[it.x] - (long long)it.y * c->k6_item); };
        std::stable_sort(items.begin(), items.end(), [&](const int2& a, const int2& b) { return size(a) > size(b); });
    }
    if (c->kf_chunked()) {  // items grouped by the frame chunk of their (frame, tile) bucket
        auto chunk = [&](const int2& it) { return (long long)(it.x / c->NT) / c->mf; };
        std::stable_sort(items.begin(), items.end(), [&](const int2& a, const int2& b) { return chunk(a) < chunk(b); });
        const long long nch = (long long)c->mf_chunks.size();
        c->kf_item_off.assign((size_t)nch + 1, 0);
        for (const int2& it : items) ++c->kf_item_off[(size_t)chunk(it) + 1];
        for (long long k = 0; k < nch; ++k) c->kf_item_off[(size_t)k + 1] += c->kf_item_off[(size_t)k];
    }
    c->n_bitems = (long long)items.size();
    CK(c->bitems.ensure((size_t)std::max(1LL, c->n_bitems), 0, c->stream));
    if (c->n_bitems)
        CK(cudaMemcpyAsync(c->bitems.p, items.data(), sizeof(int2) * items.size(), cudaMemcpyHostToDevice, c->stream));
    return MRF_OK;
}

// NCCL failures surface asynchronously (a peer lost, a timeout): poll after every collective
mrf_status nccl_async_check(mrf_ctx* c) {
    ncclResult_t ar = ncclSuccess;
    NCK(ncclCommGetAsyncError(c->comm, &ar));
    if (ar != ncclSuccess && ar != ncclInProgress)
        return set_err(c, MRF_ERR_NCCL, std::string("NCCL asynchronous error: ") + ncclGetErrorString(ar));
    return MRF_OK;
}

// world > 1 (NCCL): the tiles some rank touches, agreed by an ncclMax of the per-tile touched
// flags (identical on every rank), and the maps tile -> compact position -> tile.  Once per graph
// change; every rank calls it at the same point (prepare, from the same ABI call).
mrf_status build_active_tiles(mrf_ctx* c) {
    const long long NT = c->NT;
    std::vector<uint8_t> h((size_t)NT, 0);
    for (long long b = 0; b < (long long)c->tile_nr.size(); ++b)  // (buckets: tiles, or (frame, tile) pairs)
        if (c->tile_nr[(size_t)b] > 0) h[(size_t)(b % NT)] = 1;
    CK(c->touched.ensure((size_t)NT, 0, c->stream));
    if (c->comm) {
        CK(cudaMemcpyAsync(c->touched.p, h.data(), (size_t)NT, cudaMemcpyHostToDevice, c->stream));
        NCK(ncclAllReduce(c->touched.p, c->touched.p, (size_t)NT, ncclUint8, ncclMax, c->comm, c->stream));
        CK(cudaMemcpyAsync(h.data(), c->touched.p, (size_t)NT, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        mrf_status sa = nccl_async_check(c);
        if (sa != MRF_OK) return sa;
    }
    std::vector<int32_t> map((size_t)NT, -1), of;
    for (long long t = 0; t < NT; ++t)
        if (h[(size_t)t]) {
            map[(size_t)t] = (int32_t)of.size();
            of.push_back((int32_t)t);
        }
    c->n_act_tiles = (long long)of.size();
    CK(c->tile_map.ensure((size_t)NT, 0, c->stream));
    CK(c->tile_of.ensure((size_t)std::max<long long>(1, c->n_act_tiles), 0, c->stream));
    CK(c->T_c.ensure((size_t)std::max<long long>(1, c->n_act_tiles) * kTileSlots, 0, c->stream));
    CK(cudaMemcpyAsync(c->tile_map.p, map.data(), sizeof(int32_t) * NT, cudaMemcpyHostToDevice, c->stream));
    if (c->n_act_tiles)
        CK(cudaMemcpyAsync(c->tile_of.p, of.data(), sizeof(int32_t) * of.size(), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return MRF_OK;
}

// K6b: the pixel blocks of every frame (kBlkCols x kBlkRows owned rows), and the runs per tile
// the fills counted (touched tiles for the compacted all-reduce; their sum is n_runs)
mrf_status build_blocks(mrf_ctx* c) {
    mrf_status st;
    std::vector<int4>& bl = c->h_blk;  // (kept: the copy below is asynchronous)
    bl.clear();
    for (size_t fi = 0; fi < c->frames.size(); ++fi) {
        const FrameRec& f = c->frames[fi];
        for (int r0 = 0; r0 < f.rows_owned; r0 += kBlkRows)
            for (int u0 = 0; u0 < f.W; u0 += kBlkCols)
                bl.push_back(make_int4((int)(f.ray_base + (long long)r0 * f.W + u0),
                                       std::min(kBlkCols, f.W - u0) | (std::min(kBlkRows, f.rows_owned - r0) << 16),
                                       f.W, (int)fi));
    }
    c->n_blk = (long long)bl.size();
    CK(c->blk.ensure((size_t)std::max(1LL, c->n_blk), 0, c->stream));
    if (c->n_blk)
        CK(cudaMemcpyAsync(c->blk.p, bl.data(), sizeof(int4) * bl.size(), cudaMemcpyHostToDevice, c->stream));
    // the touched tiles of the compacted reduction (one rank: the MRF_COMPACT / one-rank NCCL
    // tests) come from the runs per tile, which the fills did not count here
    const bool need_tiles = c->force_compact || c->comm;
    if (need_tiles && (st = ensure_tile_counts(c)) != MRF_OK) return st;
    const long long NT = c->NT;
    std::vector<int32_t> nr(need_tiles ? (size_t)NT : 0);
    if (need_tiles)
        CK(cudaMemcpyAsync(nr.data(), c->tile_runs.p, sizeof(int32_t) * NT, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if ((st = fill_readback(c)) != MRF_OK) return st;  // (already here: no further wait)
    c->n_runs = 0;  // (no transpose in K6b mode; the count only when the tiles were counted)
    for (int32_t x : nr) c->n_runs += x;
    c->tile_nr = nr;
    c->n_bitems = 0;
    c->blk_check = !c->k6_demoted && c->E_real > 0;
    return MRF_OK;
}

// Build the transpose used by K6, its work list and the K5 length classes (on graph change).
mrf_status prepare(mrf_ctx* c) {
    if (!c->dirty) return MRF_OK;
    mrf_status st;
    if ((st = sync_fill(c, false)) != MRF_OK) return st;
    c->vtr_valid = false;
    if (c->k6_voxel) {
        if ((st = build_voxel_transpose(c)) != MRF_OK) return st;
    } else if (c->any_block()) {
        if ((st = build_blocks(c)) != MRF_OK) return st;
    } else {
        if ((st = build_tile_runs(c)) != MRF_OK) return st;
    }
    c->compact = !c->k6_voxel && ((c->world > 1 && c->comm_mode == MRF_COMM_NCCL) ||
                                  (c->world == 1 && (c->force_compact || c->comm) && !c->kf_avg));
    if (c->compact && (st = build_active_tiles(c)) != MRF_OK) return st;
    // K5 classes by ray length (stable compaction keeps pixel order inside a class)
    CK(c->flags.ensure((size_t)std::max(c->R, c->VI) + 1, 0, c->stream));
    CK(c->pos.ensure((size_t)std::max(c->R, c->VI) + 1, 0, c->stream));
    if (c->k5_staged) {
        // stage list over the short rays (the bulk copies read row_ptr up to index R + 1)
        CK(c->row_ptr.ensure((size_t)c->R + 2, (size_t)c->R + 1, c->stream));
        launch_stage_flags(c->R, c->row_ptr.p, c->ray_z.p, c->flags.p, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
        if ((st = scan(c, c->flags.p, c->pos.p, c->R, 0)) != MRF_OK) return st;
        if ((st = read_ll(c, c->pos.p + c->R, &c->n_stages)) != MRF_OK) return st;
        CK(c->stages.ensure((size_t)std::max(1LL, c->n_stages), 0, c->stream));
        launch_stage_fill(c->R, c->row_ptr.p, c->ray_z.p, c->flags.p, c->pos.p, c->stages.p, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
    }
    if (c->mf && (!(c->mf_fused) || c->kf_chunked())) {  // K5 classes per (chunk, class)
        const long long NK = (long long)c->mf_chunks.size() * kNumClasses;
        CK(c->class_cnt.ensure((size_t)std::max(1LL, 2 * NK), 0, c->stream));
        CK(cudaMemsetAsync(c->class_cnt.p, 0, 2 * NK * sizeof(unsigned long long), c->stream));
        launch_class_count_mf(c->R, c->ray_z.p, c->mf, c->class_cnt.p, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
        c->mf_cls_n.assign((size_t)NK, 0);
        c->mf_cls_off.assign((size_t)NK, 0);
        if (NK)
            CK(cudaMemcpyAsync(c->mf_cls_n.data(), c->class_cnt.p, NK * sizeof(long long), cudaMemcpyDeviceToHost,
                               c->stream));
        CK(cudaStreamSynchronize(c->stream));
        long long tot = 0;
        for (long long k = 0; k < NK; ++k) {
            c->mf_cls_off[k] = tot;
            tot += c->mf_cls_n[k];
        }
        CK(c->mf_cls_off_d.ensure((size_t)std::max(1LL, NK), 0, c->stream));
        if (NK)
            CK(cudaMemcpyAsync(c->mf_cls_off_d.p, c->mf_cls_off.data(), NK * sizeof(long long), cudaMemcpyHostToDevice,
                               c->stream));
        CK(c->class_all.ensure((size_t)std::max(1LL, tot), 0, c->stream));
        launch_class_scatter_mf(c->R, c->ray_z.p, c->mf, c->mf_cls_off_d.p, c->class_cnt.p + NK, c->class_all.p,
                                c->stream);
        CK(c->class_desc.ensure((size_t)std::max(1LL, tot), 0, c->stream));
        launch_class_desc(tot, c->class_all.p, c->row_ptr.p, c->ray_z.p, c->class_desc.p, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
        const int kl = kNumClasses - 1;
        long long n_long = 0;
        CK(cudaMemsetAsync(c->counters.p + 6, 0, sizeof(unsigned long long), c->stream));
        for (size_t ch = 0; ch < c->mf_chunks.size(); ++ch) {
            const long long k = (long long)ch * kNumClasses + kl;
            n_long = std::max(n_long, c->mf_cls_n[k]);
            if (c->mf_cls_n[k] > 0) {
                launch_span_max(c->mf_cls_n[k], c->class_all.p + c->mf_cls_off[k], c->ray_z.p, c->counters.p + 6,
                                c->stream);
                CK_LAUNCH(MRF_K_TRANSPOSE, 1);
            }
        }
        if (n_long > 0) {
            long long span = 0;
            if ((st = read_ll(c, reinterpret_cast<long long*>(c->counters.p + 6), &span)) != MRF_OK) return st;
            const long long tile = 512;
            c->long_scratch_per_warp = (span + tile - 1) / tile * tile + tile;
            c->n_warps_long = (int)std::min<long long>(n_long, (long long)c->sms * 16);
            CK(c->long_scratch.ensure((size_t)(c->long_scratch_per_warp * c->n_warps_long), 0, c->stream));
        }
        c->dirty = false;
        return MRF_OK;
    }
    // K5 length classes: counting sort of the ray ids by class (the counts come from the fills,
    // read back with their counters -- no round trip of its own)
    CK(c->class_cnt.ensure(2 * kNumClasses, 0, c->stream));
    CK(cudaMemsetAsync(c->class_cnt.p, 0, 2 * kNumClasses * sizeof(unsigned long long), c->stream));
    if ((st = fill_readback(c)) != MRF_OK) return st;
    if (!c->fill_classes_ok) {  // (counts not from the fills, e.g. nothing walked yet)
        launch_class_count(c->R, c->ray_z.p, c->class_cnt.p, c->stream);
        CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
        CK(cudaMemcpyAsync(c->pinned, c->class_cnt.p, kNumClasses * sizeof(long long), cudaMemcpyDeviceToHost,
                           c->stream));
        CK(cudaStreamSynchronize(c->stream));
        for (int k = 0; k < kNumClasses; ++k) c->fill_class_n[k] = c->pinned[k];
        c->fill_class_n[kNumClasses] = -1;
        CK(cudaMemsetAsync(c->class_cnt.p, 0, 2 * kNumClasses * sizeof(unsigned long long), c->stream));
    }
    ClassOffsets off{};
    long long tot = 0;
    for (int k = 0; k < kNumClasses; ++k) {
        c->class_n[k] = c->fill_class_n[k];
        c->class_off[k] = off.off[k] = tot;
        tot += c->class_n[k];
    }
    CK(c->class_all.ensure((size_t)std::max(1LL, tot), 0, c->stream));
    launch_class_scatter(c->R, c->ray_z.p, off, c->class_cnt.p + kNumClasses, c->class_all.p, c->stream);
    CK_LAUNCH(MRF_K_TRANSPOSE, c->R > 0 ? 1 : 0);
    CK(c->class_desc.ensure((size_t)std::max(1LL, tot), 0, c->stream));
    launch_class_desc(tot, c->class_all.p, c->row_ptr.p, c->ray_z.p, c->class_desc.p, c->stream);
    CK_LAUNCH(MRF_K_TRANSPOSE, tot > 0 ? 1 : 0);
    // scratch for the tiled long-ray kernel
    const int kl = kNumClasses - 1;
    if (c->class_n[kl] > 0) {
        long long span = c->fill_class_n[kNumClasses];  // the longest ray, counted by the fills
        if (span < 0) {
            CK(cudaMemsetAsync(c->counters.p + 6, 0, sizeof(unsigned long long), c->stream));
            launch_span_max(c->class_n[kl], c->class_all.p + c->class_off[kl], c->ray_z.p, c->counters.p + 6,
                            c->stream);
            CK_LAUNCH(MRF_K_TRANSPOSE, 1);
            if ((st = read_ll(c, reinterpret_cast<long long*>(c->counters.p + 6), &span)) != MRF_OK) return st;
        }
        const long long tile = 512;
        c->long_scratch_per_warp = (span + tile - 1) / tile * tile + tile;
        c->n_warps_long = (int)std::min<long long>(c->class_n[kl], (long long)c->sms * 16);
        CK(c->long_scratch.ensure((size_t)(c->long_scratch_per_warp * c->n_warps_long), 0, c->stream));
    }
    c->dirty = false;
    return MRF_OK;
}

// K6 over the current messages into `out` (zeroed first).
// Keyframe-average buffers for every frame (a new frame's averages start uniform: qbar = 0).
mrf_status ensure_kf(mrf_ctx* c) {
    const long long F = (long long)c->frames.size();
    if (!c->kf_avg || F <= c->kf_frames_alloc) return MRF_OK;
    const size_t n = (size_t)(F * c->VI), used = (size_t)(c->kf_frames_alloc * c->VI);
    CK(c->qbar.ensure(n, used, c->stream));
    CK(cudaMemsetAsync(c->qbar.p + used, 0, sizeof(int32_t) * (n - used), c->stream));
    CK(c->kf_sums.ensure(2 * n + (n + 1) / 2, 0, c->stream));
    c->kf_frames_alloc = F;
    return MRF_OK;
}

// compact: write the touched tiles' sums in compact order (world > 1, see build_active_tiles)
mrf_status voxel_sums(mrf_ctx* c, long long* out, bool compact = false) {
    ProfScope ps(c, MRF_K_VOXEL_SUM);
    if (c->kf_avg) {  // per-(frame, slot) averages, then T = sum over frames (reading R22)
        mrf_status st;
        if ((st = ensure_kf(c)) != MRF_OK) return st;
        const long long F = (long long)c->frames.size(), n = F * c->VI;
        CK(cudaMemsetAsync(c->kf_sums.p, 0, 2 * sizeof(long long) * (size_t)n, c->stream));
        CK(cudaMemsetAsync(c->kf_sums.p + 2 * n, 0xff, sizeof(unsigned) * (size_t)n, c->stream));
        unsigned* nxt = c->k6_dynamic ? reinterpret_cast<unsigned*>(c->counters.p + 15) : nullptr;
        if (c->kf_block()) {  // K6b: the two passes over pixel blocks (one frame each)
            unsigned* bn = reinterpret_cast<unsigned*>(c->counters.p + 18);
            launch_block_kf(0, c->n_blk, c->blk.p, c->row_ptr.p, c->ray_z.p, c->vid.p, c->lam.p, c->kf_sums.p, n, c->VI,
                            bn, (long long)c->lam.cap, c->stream);
            launch_kf_scale(n, 0, n, c->kf_sums.p, c->stream);
            launch_block_kf(1, c->n_blk, c->blk.p, c->row_ptr.p, c->ray_z.p, c->vid.p, c->lam.p, c->kf_sums.p, n, c->VI,
                            bn, (long long)c->lam.cap, c->stream);
            launch_kf_finalize(F, c->VI, c->kf_sums.p, c->qbar.p, out, c->stream);
            CK_LAUNCH(MRF_K_VOXEL_SUM, (c->n_blk > 0 ? 2 : 0) + 2);
            return MRF_OK;
        }
        launch_kf_sums(0, c->n_bitems, c->bitems.p, c->tile_ptr.p, c->runs.p, c->lam.p, c->k6_item, c->kf_sums.p, n,
                       nxt, (long long)c->lam.cap, c->stream);
        launch_kf_scale(n, 0, n, c->kf_sums.p, c->stream);
        launch_kf_sums(1, c->n_bitems, c->bitems.p, c->tile_ptr.p, c->runs.p, c->lam.p, c->k6_item, c->kf_sums.p, n,
                       nxt, (long long)c->lam.cap, c->stream);
        launch_kf_finalize(F, c->VI, c->kf_sums.p, c->qbar.p, out, c->stream);
        CK_LAUNCH(MRF_K_VOXEL_SUM, (c->n_bitems > 0 ? 2 : 0) + 2);
        mf_dbg(c, "kf sums");
        return MRF_OK;
    }
    CK(cudaMemsetAsync(out, 0, sizeof(long long) * (compact ? c->n_act_tiles * kTileSlots : c->VI), c->stream));
    if (c->k6_voxel) {
        launch_voxel_reduce(c->n_items_total, c->items.p, c->col_ptr.p, c->tr.p, c->lam.p, out, c->stream);
        CK_LAUNCH(MRF_K_VOXEL_SUM, c->n_items_total > 0 ? 1 : 0);
    } else if (c->use_block()) {
        unsigned long long* stats = c->blk_check ? c->counters.p + 20 : nullptr;
        if (stats) CK(cudaMemsetAsync(stats, 0, 2 * sizeof(unsigned long long), c->stream));
        launch_block_reduce(c->n_blk, c->blk.p, c->row_ptr.p, c->ray_z.p, c->vid.p, c->lam.p, out,
                            reinterpret_cast<unsigned*>(c->counters.p + 18), stats, compact ? c->tile_map.p : nullptr,
                            c->blk_max_probe, (long long)c->lam.cap, (compact ? c->n_act_tiles : c->NT) * kTileSlots, c->stream);
        CK_LAUNCH(MRF_K_VOXEL_SUM, c->n_blk > 0 ? 1 : 0);
        if (stats) {  // did the blocks share voxels?  (one round trip per graph change)
            c->blk_check = false;
            CK(cudaMemcpyAsync(c->pinned + 60, stats, 2 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
            CK(cudaStreamSynchronize(c->stream));
            const long long distinct = c->pinned[60], direct = c->pinned[61];
            if (c->k6_force == 0 && (distinct * c->blk_min_share > c->E_real || direct * 200 > c->E_real)) {
                c->k6_demoted = true;  // the next K6 runs over tile runs (built from vid: runs_ok is false)
                c->dirty = true;
                return prepare(c);
            }
        }
    } else {
        launch_tile_reduce(c->n_bitems, c->bitems.p, c->tile_ptr.p, c->runs.p, c->lam.p, c->k6_item, out,
                           c->k6_dynamic ? reinterpret_cast<unsigned*>(c->counters.p + 14) : nullptr, c->k6_pad,
                           compact ? c->tile_map.p : nullptr, (long long)c->lam.cap, compact ? c->n_act_tiles : c->NT,
                           (int)c->NT, c->stream);
        CK_LAUNCH(MRF_K_VOXEL_SUM, c->n_bitems > 0 ? 1 : 0);
    }
    return MRF_OK;
}

// K5: the staged kernel over the short rays (or the class kernels), the tiled kernel over the long
mrf_status ray_messages(mrf_ctx* c) {
    if (c->kf_avg) {
        mrf_status st;
        if ((st = ensure_kf(c)) != MRF_OK) return st;
    }
    c->mp.qbar = c->kf_avg ? c->qbar.p : nullptr;
    c->mp.qbar_vi = c->VI;
    c->mp.chk_lam = (long long)c->lam.cap;  // checked build (MRF_CHECK): what exists
    c->mp.chk_vi = c->VI;
    if (c->mf && c->mf_fused) {  // K12: K5 re-walks its own chunks (no scratch)
        ProfScope ps(c, MRF_K_RAY_MSG);
        c->mp.chk_lam = (long long)c->lam.cap;
        const WalkParams wp{c->grid, c->ray_seg.p, c->ck.p};
        int order[kNumClasses], n_cls = 0;
        for (int k = 0; k < kNumClasses; ++k)
            if (c->class_n[k]) order[n_cls++] = k;
        auto work = [&](int k) { return (double)c->class_n[k] * (k < kNumShort ? class_G(k) * class_K(k) : 1024); };
        std::sort(order, order + n_cls, [&](int a, int b) { return work(a) > work(b); });
        const int ns = std::min(c->k5_streams, std::max(n_cls, 1));
        if (ns > 1) {
            CK(cudaEventRecord(c->ev_fork, c->stream));
            for (int i = 0; i < ns; ++i) CK(cudaStreamWaitEvent(c->side[i], c->ev_fork, 0));
        }
        double load[mrf_ctx::kMaxSide] = {};
        for (int i = 0; i < n_cls; ++i) {
            const int k = order[i];
            int si = 0;
            for (int j = 1; j < ns; ++j)
                if (load[j] < load[si]) si = j;
            load[si] += work(k);
            launch_ray_messages_walk(k, c->class_n[k], c->class_all.p + c->class_off[k], c->row_ptr.p, c->ray_z.p,
                                     c->lam.p, c->T.p, c->mp, wp, c->long_scratch.p, c->long_scratch_per_warp,
                                     c->n_warps_long, c->k5_math, ns > 1 ? c->side[si] : c->stream);
            CK_LAUNCH(MRF_K_RAY_MSG, 1);
        }
        if (ns > 1) {
            for (int i = 0; i < ns; ++i) {
                CK(cudaEventRecord(c->ev_join[i], c->side[i]));
                CK(cudaStreamWaitEvent(c->stream, c->ev_join[i], 0));
            }
        }
        return MRF_OK;
    }
    if (c->mf) {  // per chunk: re-walk into the scratch, then the chunk's class kernels
        ProfScope ps(c, MRF_K_RAY_MSG);  // walks + K5 of every chunk
        const size_t nch = c->mf_chunks.size();
        const bool pipe = c->k5_streams >= 2 && nch > 1;
        // pipeline: walks on side[0], K5 on side[1]; walk i waits for the K5 of chunk i - 2 (same
        // scratch set), K5 i waits for walk i; the ctx stream joins on the last K5
        cudaStream_t A = pipe ? c->side[0] : c->stream, B = pipe ? c->side[1] : c->stream;
        cudaEvent_t* ev_walk = c->ev_mf;      // [2]
        cudaEvent_t* ev_k5 = c->ev_mf + 2;    // [2]
        if (pipe) {
            CK(cudaEventRecord(c->ev_fork, c->stream));
            CK(cudaStreamWaitEvent(A, c->ev_fork, 0));
            CK(cudaStreamWaitEvent(B, c->ev_fork, 0));
        }
        for (size_t ci = 0; ci < nch; ++ci) {
            const auto& ch = c->mf_chunks[ci];
            const int set = pipe ? (int)(ci & 1) : 0;
            mrf_status st;
            if (pipe && ci >= 2) CK(cudaStreamWaitEvent(A, ev_k5[set], 0));
            if ((st = mf_walk(c, ch, ch.f0, ch.f1, false, pipe ? A : nullptr, set)) != MRF_OK) return st;
            if (pipe) {
                CK(cudaEventRecord(ev_walk[set], A));
                CK(cudaStreamWaitEvent(B, ev_walk[set], 0));
            }
            const int32_t* sv = set ? c->s_vid2.p : c->s_vid.p;
            const float* sl = set ? c->s_lnu2.p : c->s_lnu.p;
            for (int k = 0; k < kNumClasses; ++k) {
                const long long key = (long long)ci * kNumClasses + k;
                if (c->mf_cls_n[key] == 0) continue;
                launch_ray_messages(k, c->mf_cls_n[key], c->class_all.p + c->mf_cls_off[key],
                                    c->class_desc.p + c->mf_cls_off[key], c->row_ptr.p,
                                    c->ray_z.p, sv - ch.e0, sl - ch.e0, c->lam.p, c->T.p, c->mp, c->long_scratch.p,
                                    c->long_scratch_per_warp, c->n_warps_long, c->k5_math, B);
                CK_LAUNCH(MRF_K_RAY_MSG, 1);
                mf_dbg(c, "k5 class");
            }
            if (pipe) CK(cudaEventRecord(ev_k5[set], B));
        }
        if (pipe) CK(cudaStreamWaitEvent(c->stream, ev_k5[(nch - 1) & 1], 0));
        return MRF_OK;
    }
    ProfScope ps(c, MRF_K_RAY_MSG);
    const bool staged = c->k5_staged;
    if (staged && c->n_stages > 0) {
        launch_ray_messages_staged(c->n_stages, c->stages.p, c->row_ptr.p, c->ray_z.p, c->vid.p, c->lnu.p, c->lam.p,
                                   c->T.p, c->mp, c->k5_math, c->stream);
        CK_LAUNCH(MRF_K_RAY_MSG, 1);
    }
    // the classes, largest estimated work first, each to the least-loaded stream
    int order[kNumClasses], n_cls = 0;
    for (int k = 0; k < kNumClasses; ++k) {
        if (c->class_n[k] == 0) continue;
        if (staged && k < kNumShort && class_G(k) * class_K(k) <= kShortMax) continue;  // done by the stages
        order[n_cls++] = k;
    }
    auto work = [&](int k) { return (double)c->class_n[k] * (k < kNumShort ? class_G(k) * class_K(k) : 1024); };
    std::sort(order, order + n_cls, [&](int a, int b) { return work(a) > work(b); });
    const int ns = std::min(c->k5_streams, std::max(n_cls, 1));
    if (ns > 1) {
        CK(cudaEventRecord(c->ev_fork, c->stream));
        for (int i = 0; i < ns; ++i) CK(cudaStreamWaitEvent(c->side[i], c->ev_fork, 0));
    }
    double load[mrf_ctx::kMaxSide] = {};
    for (int i = 0; i < n_cls; ++i) {
        const int k = order[i];
        int si = 0;
        for (int j = 1; j < ns; ++j)
            if (load[j] < load[si]) si = j;
        load[si] += work(k);
        launch_ray_messages(k, c->class_n[k], c->class_all.p + c->class_off[k], c->class_desc.p + c->class_off[k],
                            c->row_ptr.p, c->ray_z.p, c->vid.p,
                            c->lnu.p, c->lam.p, c->T.p, c->mp, c->long_scratch.p, c->long_scratch_per_warp,
                            c->n_warps_long, c->k5_math, ns > 1 ? c->side[si] : c->stream);
        CK_LAUNCH(MRF_K_RAY_MSG, 1);
    }
    if (ns > 1) {
        for (int i = 0; i < ns; ++i) {
            CK(cudaEventRecord(c->ev_join[i], c->side[i]));
            CK(cudaStreamWaitEvent(c->stream, c->ev_join[i], 0));
        }
    }
    return MRF_OK;
}

// One flooding iteration in keyframe-average mode with fused matrix-free walks (kf_chunked): per
// chunk of frames, K5 (walk kernels, the keyframe cavity) writes the chunk's messages into the
// scratch, then K6' adds them into the (frame, slot) sums; then the averages and T.
mrf_status kf_iteration(mrf_ctx* c) {
    mrf_status st;
    if ((st = ensure_kf(c)) != MRF_OK) return st;
    const long long F = (long long)c->frames.size(), n = F * c->VI;
    c->mp.qbar = c->qbar.p;
    c->mp.qbar_vi = c->VI;
    c->mp.chk_vi = c->VI;
    CK(cudaMemsetAsync(c->kf_sums.p, 0, 2 * sizeof(long long) * (size_t)n, c->stream));
    CK(cudaMemsetAsync(c->kf_sums.p + 2 * n, 0xff, sizeof(unsigned) * (size_t)n, c->stream));
    const WalkParams wp{c->grid, c->ray_seg.p, c->ck.p};
    for (size_t ci = 0; ci < c->mf_chunks.size(); ++ci) {
        const auto& ch = c->mf_chunks[ci];
        int32_t* lam = c->lam_chunk.p - ch.e0;  // absolute slots [e0, e1) of this chunk
        c->mp.chk_lam = ch.e1;
        {
            ProfScope ps(c, MRF_K_RAY_MSG);
            for (int k = 0; k < kNumClasses; ++k) {
                const long long key = (long long)ci * kNumClasses + k;
                if (c->mf_cls_n[key] == 0) continue;
                launch_ray_messages_walk(k, c->mf_cls_n[key], c->class_all.p + c->mf_cls_off[key], c->row_ptr.p,
                                         c->ray_z.p, lam, c->T.p, c->mp, wp, c->long_scratch.p,
                                         c->long_scratch_per_warp, c->n_warps_long, c->k5_math, c->stream);
                CK_LAUNCH(MRF_K_RAY_MSG, 1);
            }
        }
        {
            ProfScope ps(c, MRF_K_VOXEL_SUM);
            const long long i0 = c->kf_item_off[ci], i1 = c->kf_item_off[ci + 1];
            unsigned* nxt = c->k6_dynamic ? reinterpret_cast<unsigned*>(c->counters.p + 15) : nullptr;
            launch_kf_sums(0, i1 - i0, c->bitems.p + i0, c->tile_ptr.p, c->runs.p, lam, c->k6_item, c->kf_sums.p, n,
                           nxt, ch.e1, c->stream);
            launch_kf_scale(n, (long long)ch.f0 * c->VI, (long long)(ch.f1 - ch.f0) * c->VI, c->kf_sums.p, c->stream);
            launch_kf_sums(1, i1 - i0, c->bitems.p + i0, c->tile_ptr.p, c->runs.p, lam, c->k6_item, c->kf_sums.p, n,
                           nxt, ch.e1, c->stream);
            CK_LAUNCH(MRF_K_VOXEL_SUM, (i1 > i0 ? 2 : 0) + 1);
        }
        mf_dbg(c, "kf chunk");
    }
    ProfScope ps(c, MRF_K_VOXEL_SUM);
    launch_kf_finalize(F, c->VI, c->kf_sums.p, c->qbar.p, c->T.p, c->stream);
    CK_LAUNCH(MRF_K_VOXEL_SUM, 1);
    return MRF_OK;
}

// T = sum over ranks of the K6 partials.  compact: in place over the touched tiles (T_c), then
// scattered into T; otherwise (per-voxel K6 ablation) over every belief slot, T_part -> T.
mrf_status allreduce_T(mrf_ctx* c) {
    ProfScope ps(c, MRF_K_ALLREDUCE);
    if (c->compact) {
        if (c->n_act_tiles) {
            if (c->comm) {
                NCK(ncclAllReduce(c->T_c.p, c->T_c.p, (size_t)(c->n_act_tiles * kTileSlots), ncclInt64, ncclSum,
                                  c->comm, c->stream));
                c->prof_launch[MRF_K_ALLREDUCE] += 1;
            }
            launch_tile_scatter(c->n_act_tiles, c->tile_of.p, c->T_c.p, c->T.p, c->stream);
            CK_LAUNCH(MRF_K_ALLREDUCE, 1);
        }
        if (!c->comm) return MRF_OK;
    } else {
        NCK(ncclAllReduce(c->T_part.p, c->T.p, (size_t)c->VI, ncclInt64, ncclSum, c->comm, c->stream));
        c->prof_launch[MRF_K_ALLREDUCE] += 1;
    }
    return nccl_async_check(c);
}

// K6 over the current messages, then (world > 1) the all-reduce: T of every rank.
mrf_status reduce_T(mrf_ctx* c) {
    mrf_status st;
    if (c->compact) {
        if ((st = voxel_sums(c, c->T_c.p, true)) != MRF_OK) return st;
        return allreduce_T(c);
    }
    if (c->world == 1) return voxel_sums(c, c->T.p);
    if ((st = voxel_sums(c, c->T_part.p)) != MRF_OK) return st;
    return allreduce_T(c);
}

// Rebuild T from the current messages (all ranks).
mrf_status rebuild_T(mrf_ctx* c) {
    mrf_status st;
    if ((st = prepare(c)) != MRF_OK) return st;
    if (c->world == 1 || c->comm_mode == MRF_COMM_NCCL) return reduce_T(c);
    if ((st = voxel_sums(c, c->T_part.p)) != MRF_OK) return st;
    return MRF_OK;  // external mode: caller reduces (mrf_bp_partial / mrf_bp_finish)
}


// Canonical (unpadded) layout of this rank's incidences, from the device ray records.
struct HostLayout {
    std::vector<long long> row_ptr;   // padded segment start per ray (R+1)
    std::vector<RayInfo> info;        // per ray
    std::vector<int8_t> status;       // per ray
    std::vector<long long> canon;     // canonical start per ray (R+1)
};

mrf_status host_layout(mrf_ctx* c, HostLayout& h) {
    {
        mrf_status sf = sync_fill(c);
        if (sf != MRF_OK) return sf;
    }
    h.row_ptr.resize((size_t)c->R + 1);
    h.info.resize((size_t)c->R);
    h.status.resize((size_t)c->R);
    CK(cudaMemcpyAsync(h.row_ptr.data(), c->row_ptr.p, sizeof(long long) * (c->R + 1), cudaMemcpyDeviceToHost, c->stream));
    if (c->R) {
        CK(cudaMemcpyAsync(h.info.data(), c->ray_z.p, sizeof(RayInfo) * c->R, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(h.status.data(), c->status.p, c->R, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    h.canon.resize((size_t)c->R + 1);
    h.canon[0] = 0;
    for (long long r = 0; r < c->R; ++r) h.canon[r + 1] = h.canon[r] + h.info[r].n;
    return MRF_OK;
}

// belief slot (tile-major) -> external voxel id x + nx (y + ny z)
long long slot_to_voxel(const GridDesc& g, long long s) {
    int x, y, z;
    slot_xyz(g, s, x, y, z);
    return x + (long long)g.nx * (y + (long long)g.ny * z);
}

// padded -> canonical copy (to_canon) or back, element size `es`
void relayout(const HostLayout& h, const void* src, void* dst, size_t es, bool to_canon) {
    const char* s = static_cast<const char*>(src);
    char* d = static_cast<char*>(dst);
    for (size_t r = 0; r < h.info.size(); ++r) {
        const size_t n = (size_t)h.info[r].n * es;
        if (!n) continue;
        if (to_canon) memcpy(d + (size_t)h.canon[r] * es, s + (size_t)h.row_ptr[r] * es, n);
        else memcpy(d + (size_t)h.row_ptr[r] * es, s + (size_t)h.canon[r] * es, n);
    }
}

}  // namespace

// ======================================================================= ABI

extern "C" {

mrf_status mrf_create(const int32_t dims[3], double resolution_m, const double origin_m[3], float prior,
                      const mrf_noise_desc* noise, const mrf_dist_desc* dist, mrf_ctx** out) {
    g_create_error.clear();
    auto reject = [](const char* m) {
        g_create_error = m;
        return MRF_ERR_INVALID_ARG;
    };
    long long margin_cells = 0;  // ceil(largest traversal margin / res) + 1
    if (!out) return reject("out is NULL");
    *out = nullptr;
    if (!dims || !origin_m || !noise) return reject("NULL argument");
    for (int k = 0; k < 3; ++k)
        if (dims[k] <= 0 || dims[k] > 8192) return reject("dims must be in [1, 8192]");
    const long long V = (long long)dims[0] * dims[1] * dims[2];
    if (V >= (1LL << 31)) return reject("nx*ny*nz must be < 2^31");
    if ((long long)((dims[0] + 31) / 32) * ((dims[1] + 31) / 32) * ((dims[2] + 15) / 16) * 16384 >= (1LL << 31))
        return reject("tile-padded grid (32x32x16 tiles) must have < 2^31 voxels");
    if (!std::isfinite(resolution_m) || !(resolution_m > 0)) return reject("resolution must be finite and > 0");
    if (!finite_all(origin_m, 3)) return reject("origin must be finite");
    if (!(prior > 0.f && prior < 1.f)) return reject("prior must be in (0, 1)");
    if (!noise->log_nu || noise->n_z < 2 || noise->n_off < 2) return reject("noise table must be at least 2x2");
    const double np_[9] = {noise->z_lo, noise->z_hi, noise->off_lo, noise->off_hi, noise->margin_min,
                           noise->margin_k, noise->sigma_c[0], noise->sigma_c[1], noise->sigma_c[2]};
    if (!finite_all(np_, 9)) return reject("noise parameters must be finite");
    if (!(noise->z_hi > noise->z_lo)) return reject("z_hi must exceed z_lo");
    if (!(noise->off_hi > noise->off_lo) || noise->off_lo < -1.0 || noise->off_hi > 1.0)
        return reject("offset axis must satisfy -1 <= off_lo < off_hi <= 1");
    if (noise->margin_min < 0 || noise->margin_k < 0) return reject("margin parameters must be >= 0");
    {
        const double D = resolution_m * std::sqrt((double)dims[0] * dims[0] + (double)dims[1] * dims[1] +
                                                  (double)dims[2] * dims[2]);
        const double sig = std::fabs(noise->sigma_c[0]) + std::fabs(noise->sigma_c[1]) * D +
                           std::fabs(noise->sigma_c[2]) * D * D;
        if (noise->margin_min > D || noise->margin_k * sig > D)
            return reject("traversal margin must stay below the grid diagonal (margin bound)");
        margin_cells = (long long)std::ceil(std::max(noise->margin_min, noise->margin_k * sig) / resolution_m) + 1;
    }
    const long long nlut = (long long)noise->n_z * noise->n_off;
    for (long long i = 0; i < nlut; ++i)
        if (!std::isfinite(noise->log_nu[i])) return reject("noise table has non-finite entries");
    int rank = 0, world = 1, comm_mode = MRF_COMM_NCCL;
    if (dist) {
        rank = dist->rank;
        world = dist->world;
        comm_mode = dist->comm;
        if (world < 1 || rank < 0 || rank >= world) return reject("bad rank/world");
        if (comm_mode != MRF_COMM_NCCL && comm_mode != MRF_COMM_EXTERNAL) return reject("bad comm mode");
    }

    mrf_ctx* c = new mrf_ctx();
    cudaGetDevice(&c->device);
    if (cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device) != cudaSuccess || c->sms <= 0) {
        cudaGetLastError();
        c->sms = 148;
    }
    c->grid = {dims[0], dims[1], dims[2], (dims[0] + 31) / 32, (dims[1] + 31) / 32, (dims[2] + 15) / 16,
               resolution_m, origin_m[0], origin_m[1], origin_m[2]};
    c->NT = (long long)c->grid.ntx * c->grid.nty * c->grid.ntz;
    c->VI = c->NT * kTileSlots;
    c->ray_slots_max = (1 + (long long)dims[0] + dims[1] + dims[2] + 3 * margin_cells + 7) & ~7LL;
    if (const char* k6 = getenv("MRF_K6")) {
        c->k6_voxel = strcmp(k6, "voxel") == 0;
        c->k6_force = strcmp(k6, "block") == 0 ? 1 : 2;
    }
    if (const char* bp = getenv("MRF_BLK_PROBE")) c->blk_max_probe = atoi(bp);
    if (const char* bs = getenv("MRF_BLK_SHARE")) c->blk_min_share = atoll(bs);
    if (const char* kb = getenv("MRF_KF_BLOCK")) c->kf_blk_on = atoi(kb) != 0;
    if (const char* km = getenv("MRF_K5_MATH")) c->k5_math = atoi(km);
    if (const char* ki = getenv("MRF_K6_ITEM")) {
        c->k6_item = std::min(std::max(atoi(ki), 1024), kRunsPerItem);
        c->k6_item_fixed = true;
    }
    if (const char* kd = getenv("MRF_K6_DYNAMIC")) c->k6_dynamic = atoi(kd) != 0;
    if (const char* kp = getenv("MRF_K6_PAD")) c->k6_pad = atoi(kp) != 0;
    if (const char* kl = getenv("MRF_K6_LPT")) c->k6_lpt = atoi(kl) != 0;
    if (const char* kc = getenv("MRF_COMPACT")) c->force_compact = atoi(kc) != 0;
    if (const char* kf = getenv("MRF_K6_FRAMES")) c->frame_buckets = atoi(kf) != 0;
    if (const char* rf = getenv("MRF_RUN_FILL")) c->run_fill_forced = atoi(rf) != 0;
    if (const char* mff = getenv("MRF_MF_FUSED")) c->mf_fused = atoi(mff) != 0;
    if (const char* rr = getenv("MRF_RUN_RATIO")) c->run_ratio = atof(rr);
    if (const char* rs = getenv("MRF_RUN_SLACK")) c->run_slack = atoll(rs);
    if (const char* k5 = getenv("MRF_K5")) c->k5_staged = strcmp(k5, "staged") == 0;
    if (const char* l2 = getenv("MRF_L2_FETCH")) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(l2));
    c->noise = {noise->z_lo, noise->z_hi, noise->off_lo, noise->off_hi, noise->margin_min, noise->margin_k,
                noise->sigma_c[0], noise->sigma_c[1], noise->sigma_c[2], noise->n_z, noise->n_off};
    c->V = V;
    c->prior = prior;
    c->L0 = std::log((double)prior / (1.0 - (double)prior));
    c->rank = rank;
    c->world = world;
    c->comm_mode = comm_mode;
    auto fail = [&](mrf_status st) {
        g_create_error = c->err.empty() ? "mrf_create failed" : c->err;
        mrf_destroy(c);
        return st;
    };
    if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess) {
        c->err = "cudaStreamCreate failed (no CUDA device?)";
        cudaGetLastError();
        return fail(MRF_ERR_CUDA);
    }
    c->stream = c->own_stream;
    if (const char* ks = getenv("MRF_K5_STREAMS")) c->k5_streams = std::min(std::max(atoi(ks), 1), mrf_ctx::kMaxSide);
    if (c->k5_streams > 1) {
        bool ok = cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; ok && i < 4; ++i)
            ok = cudaEventCreateWithFlags(&c->ev_mf[i], cudaEventDisableTiming) == cudaSuccess;
        for (int i = 0; ok && i < c->k5_streams; ++i)
            ok = cudaStreamCreateWithFlags(&c->side[i], cudaStreamNonBlocking) == cudaSuccess &&
                 cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) {
            c->err = "side stream / event creation failed";
            cudaGetLastError();
            return fail(MRF_ERR_CUDA);
        }
    }
    mrf_status st = MRF_OK;
    auto alloc = [&]() -> mrf_status {
        const long long VI = c->VI, NT = c->NT;
        CK(c->T.ensure((size_t)VI, 0, c->stream));
        if (world > 1) CK(c->T_part.ensure((size_t)VI, 0, c->stream));
        CK(c->vox_count.ensure((size_t)VI, 0, c->stream));
        CK(c->cursor.ensure((size_t)VI, 0, c->stream));
        CK(c->n_items.ensure((size_t)VI, 0, c->stream));
        CK(c->col_ptr.ensure((size_t)VI + 1, 0, c->stream));
        CK(c->item_ptr.ensure((size_t)VI + 1, 0, c->stream));
        CK(c->tile_runs.ensure((size_t)NT, 0, c->stream));
        CK(c->tile_cursor.ensure((size_t)NT, 0, c->stream));
        CK(c->tile_ptr.ensure((size_t)NT + 1, 0, c->stream));
        CK(c->counters.ensure(64, 0, c->stream));
        CK(c->row_ptr.ensure(1, 0, c->stream));
        CK(cudaMemsetAsync(c->T.p, 0, sizeof(long long) * VI, c->stream));
        CK(cudaMemsetAsync(c->tile_runs.p, 0, sizeof(int32_t) * NT, c->stream));
        CK(cudaMemsetAsync(c->row_ptr.p, 0, sizeof(long long), c->stream));
        CK(cudaMemsetAsync(c->counters.p, 0, sizeof(unsigned long long) * 64, c->stream));
        CK(cudaMallocHost(&c->pinned, 64 * sizeof(long long)));
        // LUT as (L[i][j], L[i][j+1]) pairs: one 8-byte load per LUT row in K5.  The values are
        // the input table's floats, unscaled and unshifted.
        const int nz = noise->n_z, no = noise->n_off;
        std::vector<float2> h((size_t)nz * (no - 1));
        for (int i = 0; i < nz; ++i) {
            const float* row = noise->log_nu + (size_t)i * no;
            // entries below -1e30 (e.g. -FLT_MAX standing for log 0) are raised to -1e30: K5 scales
            // log nu by log2(e), which would overflow them to -inf (and -inf - -inf = NaN)
            for (int j = 0; j < no - 1; ++j)
                h[(size_t)i * (no - 1) + j] = make_float2(std::max(row[j], -1e30f), std::max(row[j + 1], -1e30f));
        }
        CK(c->lutp.ensure(h.size(), 0, c->stream));
        CK(cudaMemcpyAsync(c->lutp.p, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        const double span = noise->off_hi - noise->off_lo;
        c->mp.lutp = c->lutp.p;
        c->mp.n_offm1 = no - 1;
        c->mp.s_off = (float)((double)no / (32768.0 * span));
        c->mp.b_off = (float)(-noise->off_lo * (double)no / span - 0.5);
        c->mp.fo_max = (float)(no - 1);
        c->mp.L0 = (float)c->L0;
        return MRF_OK;
    };
    if ((st = alloc()) != MRF_OK) return fail(st);
    // MRF_NCCL_WORLD1=1: a one-rank communicator at world 1, so that the NCCL data plane (the
    // touched-tile mask and the compacted all-reduce, the async-error polling) runs on one GPU (tests)
    const char* w1 = getenv("MRF_NCCL_WORLD1");
    const bool nccl_w1 = world == 1 && w1 && atoi(w1) != 0;
    if ((world > 1 && comm_mode == MRF_COMM_NCCL) || nccl_w1) {
        ncclUniqueId id;
        static_assert(sizeof(id.internal) == 128, "ncclUniqueId size");
        if (nccl_w1) {
            if (ncclGetUniqueId(&id) != ncclSuccess) {
                c->err = "ncclGetUniqueId failed";
                return fail(MRF_ERR_NCCL);
            }
        } else {
            memcpy(id.internal, dist->nccl_id, 128);
        }
        ncclResult_t r = ncclCommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) {
            c->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
            c->comm = nullptr;
            return fail(MRF_ERR_NCCL);
        }
    }
    *out = c;
    return MRF_OK;
}

mrf_status mrf_destroy(mrf_ctx* ctx) {
    if (!ctx) return MRF_OK;
    mrf_ctx* c = ctx;
    DeviceGuard guard(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->comm) ncclCommDestroy(c->comm);
    for (auto& e : c->events) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
    }
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    c->n_r.release(); c->status.release(); c->ray_z.release(); c->row_ptr.release();
    c->vid.release(); c->off_q.release(); c->lnu.release(); c->lam.release(); c->tr.release();
    c->vox_count.release(); c->cursor.release(); c->n_items.release(); c->flags.release();
    c->col_ptr.release(); c->item_ptr.release(); c->pos.release(); c->items.release();
    c->T.release(); c->T_part.release(); c->lutp.release(); c->depth_stage.release(); c->depth_all.release(); c->d_frames.release(); c->d_cta0.release(); c->qbar.release(); c->kf_sums.release(); c->bmask.release(); c->s_vid.release(); c->s_off.release(); c->s_lnu.release(); c->s_vid2.release(); c->s_off2.release(); c->s_lnu2.release(); c->d_cta_tmp.release(); c->mf_cls_off_d.release(); c->marg.release(); c->eval_cls.release();
    c->scan_scratch.release(); c->counters.release(); c->long_scratch.release();
    c->tile_runs.release(); c->tile_cursor.release(); c->tile_ptr.release();
    c->runs.release(); c->bitems.release(); c->stages.release();
    c->tile_map.release(); c->tile_of.release(); c->touched.release(); c->T_c.release();
    c->runs_all.release(); c->run_keys.release();
    c->rp_old.release(); c->ri_old.release(); c->vid_old.release(); c->lam_old.release();
    c->ray_seg.release(); c->ck.release(); c->lam_chunk.release();
    c->d_k1_frames.release(); c->d_k1_cta0.release();
    c->class_all.release();
    c->class_desc.release();
    c->class_cnt.release();
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    for (int i = 0; i < mrf_ctx::kMaxSide; ++i) {
        if (c->side[i]) cudaStreamDestroy(c->side[i]);
        if (c->ev_join[i]) cudaEventDestroy(c->ev_join[i]);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    for (int i = 0; i < 4; ++i)
        if (c->ev_mf[i]) cudaEventDestroy(c->ev_mf[i]);
    delete c;
    return MRF_OK;
}

const char* mrf_last_error(const mrf_ctx* ctx) {
    if (!ctx) return g_create_error.c_str();
    return ctx->err.c_str();
}

mrf_status mrf_set_stream(mrf_ctx* ctx, void* cuda_stream) {
    ENTER(ctx);
    CK(cudaStreamSynchronize(c->stream));
    c->stream = (cudaStream_t)cuda_stream;  // NULL = the CUDA default stream
    return MRF_OK;
}

mrf_status mrf_reserve(mrf_ctx* ctx, int64_t n_rays, int64_t n_incidences) {
    ENTER(ctx);
    if (n_rays < 0 || n_incidences < 0) return set_err(c, MRF_ERR_INVALID_ARG, "negative reservation");
    CK(c->n_r.ensure((size_t)n_rays, (size_t)c->R, c->stream));
    CK(c->status.ensure((size_t)n_rays, (size_t)c->R, c->stream));
    CK(c->ray_z.ensure((size_t)n_rays, (size_t)c->R, c->stream));
    CK(c->row_ptr.ensure((size_t)n_rays + 1, (size_t)c->R + 1, c->stream));
    CK(c->flags.ensure((size_t)std::max<long long>(n_rays, c->VI) + 1, 0, c->stream));
    CK(c->pos.ensure((size_t)std::max<long long>(n_rays, c->VI) + 1, 0, c->stream));
    const size_t ne = (size_t)n_incidences + kPadElems;
    CK(c->vid.ensure(ne, (size_t)c->E_filled, c->stream));
    CK(c->off_q.ensure(ne, (size_t)c->E_filled, c->stream));
    CK(c->lnu.ensure(ne, (size_t)c->E_filled, c->stream));
    CK(c->lam.ensure(ne, (size_t)c->E_filled, c->stream));
    CK(c->tr.ensure(ne, 0, c->stream));
    return MRF_OK;
}

mrf_status mrf_reset(mrf_ctx* ctx) {
    ENTER(ctx);
    c->R = c->E = c->E_real = 0;
    c->fill_pending = false;
    c->E_unresolved = false;
    c->E_bound = 0;
    CK(cudaMemsetAsync(c->counters.p + 2, 0, 2 * sizeof(unsigned long long), c->stream));
    c->pend.clear();
    c->k1_pend.clear();
    c->fill_rb_pending = false;
    c->depth_used = 0;
    c->E_filled = c->R_filled = 0;
    c->kf_frames_alloc = 0;
    c->mf_frames.clear();
    c->mf_chunks.clear();
    c->sp_frames.clear();
    c->sp_rebuild = false;
    c->vid_old.release();
    c->lam_old.release();
    if (c->grid.bmask) CK(cudaMemsetAsync(c->bmask.p, 0, (size_t)c->n_brick_slots, c->stream));
    CK(cudaMemsetAsync(c->counters.p + 10, 0, 2 * sizeof(unsigned long long), c->stream));
    CK(cudaMemsetAsync(c->counters.p + 16, 0, sizeof(unsigned long long), c->stream));
    CK(cudaMemsetAsync(c->counters.p + kClassCtr, 0, (kNumClasses + 1) * sizeof(unsigned long long), c->stream));
    c->fill_classes_ok = false;
    c->runs_emitted = 0;
    c->runs_ok = true;
    c->n_invalid = c->n_dropped = c->n_kept = 0;
    c->frames.clear();
    CK(cudaMemsetAsync(c->tile_runs.p, 0, sizeof(int32_t) * c->NT, c->stream));
    c->tile_counts_ok = true;
    CK(cudaMemsetAsync(c->T.p, 0, sizeof(long long) * c->VI, c->stream));
    CK(cudaMemsetAsync(c->row_ptr.p, 0, sizeof(long long), c->stream));
    c->dirty = true;
    c->hist_valid = false;
    return MRF_OK;
}

mrf_status mrf_add_frame(mrf_ctx* ctx, const float* depth, int32_t width, int32_t height, const double K[4],
                         const double T_wc[12], int64_t* frame_id_out) {
    ENTER(ctx);
    if (c->grid.bmask && c->mf && c->E_filled > 0)
        return set_err(c, MRF_ERR_STATE,
                       "sparse bricks with matrix-free walks: add every keyframe before the graph is first used");
    if (!depth || !K || !T_wc) return set_err(c, MRF_ERR_INVALID_ARG, "NULL argument");
    if (width <= 0 || height <= 0) return set_err(c, MRF_ERR_INVALID_ARG, "width/height must be > 0");
    if (c->patch_px && ((long long)width > (long long)c->patch_px * c->patch_nx ||
                        (long long)height > (long long)c->patch_px * c->patch_ny))
        return set_err(c, MRF_ERR_INVALID_ARG, "image larger than the patch grid of the noise model");
    if (!finite_all(K, 4) || !(K[0] > 0) || !(K[1] > 0))
        return set_err(c, MRF_ERR_INVALID_ARG, "K must be finite with fx, fy > 0");
    if (!finite_all(T_wc, 12)) return set_err(c, MRF_ERR_INVALID_ARG, "T_wc must be finite");
    // rotation must be orthonormal
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            double d = 0;
            for (int k = 0; k < 3; ++k) d += T_wc[4 * k + a] * T_wc[4 * k + b];
            if (std::fabs(d - (a == b ? 1.0 : 0.0)) > 1e-6)
                return set_err(c, MRF_ERR_INVALID_ARG, "rotation of T_wc is not orthonormal");
        }
    const double org[3] = {c->grid.ox, c->grid.oy, c->grid.oz};
    const int dims[3] = {c->grid.nx, c->grid.ny, c->grid.nz};
    for (int k = 0; k < 3; ++k) {
        const double g = (T_wc[4 * k + 3] - org[k]) / c->grid.res;
        if (!(g >= 0.0 && g < (double)dims[k]))
            return set_err(c, MRF_ERR_INVALID_ARG, "camera centre lies outside the grid");
    }
    const int rows_owned = height > c->rank ? (height - c->rank + c->world - 1) / c->world : 0;
    const long long Rf = (long long)rows_owned * width;
    if (c->R + Rf >= (1LL << 31)) return set_err(c, MRF_ERR_CAPACITY, "ray count would exceed 2^31");

    // depth (host or device memory) copied into the pending-depth buffer: the walk runs later
    cudaPointerAttributes attr;
    cudaError_t pe = cudaPointerGetAttributes(&attr, depth);
    if (pe != cudaSuccess) cudaGetLastError();
    const bool on_device = pe == cudaSuccess && (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged);
    const size_t npix = (size_t)width * height;
    CK(c->depth_all.ensure((size_t)c->depth_used + npix, (size_t)c->depth_used, c->stream));
    const float* d_depth = c->depth_all.p + c->depth_used;
    CK(cudaMemcpyAsync(c->depth_all.p + c->depth_used, depth, npix * sizeof(float),
                       on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    CK(c->n_r.ensure((size_t)(c->R + Rf), (size_t)c->R, c->stream));
    CK(c->status.ensure((size_t)(c->R + Rf), (size_t)c->R, c->stream));
    CK(c->ray_z.ensure((size_t)(c->R + Rf), (size_t)c->R, c->stream));
    CK(c->row_ptr.ensure((size_t)(c->R + Rf + 1), (size_t)(c->R + 1), c->stream));

    FrameDesc f{};
    f.fx = K[0]; f.fy = K[1]; f.cx = K[2]; f.cy = K[3];
    for (int k = 0; k < 3; ++k) {
        for (int j = 0; j < 3; ++j) f.R[3 * k + j] = T_wc[4 * k + j];
        f.C[k] = T_wc[4 * k + 3];
    }
    f.W = width; f.H = height; f.rank = c->rank; f.world = c->world;
    f.rows_owned = rows_owned;
    f.ray_base = c->R;
    f.index = (int)c->frames.size();
    f.skip_count = c->grid.bmask ? 1 : 0;  // sparse: the rays are counted once all frames are allocated
    f.bucket_stride = c->fb() ? (int)c->NT : 0;
    if (c->fb()) {  // this frame's (frame, tile) run counters
        const size_t F = c->frames.size();
        CK(c->tile_runs.ensure((F + 1) * (size_t)c->NT, F * (size_t)c->NT, c->stream));
        CK(cudaMemsetAsync(c->tile_runs.p + F * c->NT, 0, sizeof(int32_t) * (size_t)c->NT, c->stream));
    }
    // Capacity without a round trip while E + the bound of every unresolved frame stays below
    // 2^31: K1 lays a ray out with pad8(1 + sum_k |c_end,k - c_0,k|) slots, the segment end lies
    // within the traversal margin M of the measured point (inside the grid), so a frame adds at
    // most Rf ray_slots_max slots (0 for a sparse-brick frame: counted at first use).
    const long long U = c->grid.bmask ? 0 : Rf * c->ray_slots_max;
    const bool fast = c->E + c->E_bound + U < (1LL << 31) - kPadElems;
    mrf_status st;
    if (!fast && (st = resolve_E(c)) != MRF_OK) return st;  // (runs the pending K1s first)
    f.depth_off = c->depth_used;
    long long E_new = 0, inv = 0, drp = 0;
    if (fast) {  // K1 and the row scan run later, batched with the other pending frames (flush_k1)
        if (c->k1_pend.empty()) c->k1_R0 = c->R;
        if (Rf > 0) c->k1_pend.push_back(f);
    } else {  // counters[2..3] hold this frame only (resolve_E cleared them)
        {
            ProfScope ps(c, MRF_K_RAYGEN_COUNT);
            launch_raygen_count(f, c->grid, c->noise, d_depth, c->n_r.p, c->status.p, c->ray_z.p, c->counters.p + 2,
                                c->stream);
            CK_LAUNCH(MRF_K_RAYGEN_COUNT, Rf > 0 ? 1 : 0);
        }
        if ((st = scan(c, c->n_r.p + c->R, c->row_ptr.p + c->R, Rf, c->E)) != MRF_OK) return st;
        CK(cudaMemcpyAsync(c->pinned, c->row_ptr.p + c->R + Rf, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(c->pinned + 1, c->counters.p + 2, 2 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        E_new = c->pinned[0];
        inv = c->pinned[1];
        drp = c->pinned[2];
        CK(cudaMemsetAsync(c->counters.p + 2, 0, 2 * sizeof(unsigned long long), c->stream));
        if (E_new >= (1LL << 31) - kPadElems)
            return set_err(c, MRF_ERR_CAPACITY, "incidence count would exceed 2^31 (int32 transpose indices)");
    }
    if (c->grid.bmask) {  // sparse bricks: allocate around this frame's reprojected points
        launch_brick_alloc(f, c->grid, c->noise, d_depth, c->bmask.p, c->stream);
        CK_LAUNCH(MRF_K_RAYGEN_COUNT, 1);
    }
    c->depth_used += (long long)npix;
    if (Rf > 0) c->pend.push_back(f);
    if (frame_id_out) *frame_id_out = (int64_t)c->frames.size();
    c->frames.push_back({width, height, rows_owned, c->R, Rf});
    c->ppv_min = std::min(c->ppv_min, std::min(K[0], K[1]) * c->grid.res / 3.0);
    c->R += Rf;
    if (fast) {
        c->E_unresolved = true;
        c->E_bound += U;
    } else {
        c->E = E_new;
        c->n_invalid += inv;
        c->n_dropped += drp;
        c->n_kept += Rf - inv - drp;
    }
    if (c->grid.bmask && c->E_filled > 0) c->sp_rebuild = true;  // R24: re-walk every frame at the next fill
    c->fill_pending = true;
    c->dirty = true;
    c->hist_valid = false;
    return MRF_OK;
}

mrf_status mrf_bp_iterate(mrf_ctx* ctx, int32_t n) {
    ENTER(ctx);
    if (n < 0) return set_err(c, MRF_ERR_INVALID_ARG, "n must be >= 0");
    if (c->world > 1 && c->comm_mode != MRF_COMM_NCCL)
        return set_err(c, MRF_ERR_STATE, "external comm mode: use mrf_bp_partial / mrf_bp_finish");
    mrf_status st;
    if ((st = prepare(c)) != MRF_OK) return st;
    for (int it = 0; it < n; ++it) {
        if (c->kf_chunked()) {
            if ((st = kf_iteration(c)) != MRF_OK) return st;
            continue;
        }
        if ((st = ray_messages(c)) != MRF_OK) return st;
        if ((st = reduce_T(c)) != MRF_OK) return st;
    }
    return MRF_OK;
}

mrf_status mrf_bp_partial(mrf_ctx* ctx, int32_t iterate, int64_t* partial_out_device) {
    ENTER(ctx);
    if (!partial_out_device) return set_err(c, MRF_ERR_INVALID_ARG, "NULL output");
    mrf_status st;
    if ((st = prepare(c)) != MRF_OK) return st;
    if (iterate && (st = ray_messages(c)) != MRF_OK) return st;
    return voxel_sums(c, reinterpret_cast<long long*>(partial_out_device));
}

mrf_status mrf_bp_finish(mrf_ctx* ctx, const int64_t* total_device) {
    ENTER(ctx);
    if (!total_device) return set_err(c, MRF_ERR_INVALID_ARG, "NULL input");
    CK(cudaMemcpyAsync(c->T.p, total_device, sizeof(long long) * c->VI, cudaMemcpyDeviceToDevice, c->stream));
    return MRF_OK;
}

mrf_status mrf_marginals(mrf_ctx* ctx, float* out, int32_t out_is_device) {
    ENTER(ctx);
    if (!out) return set_err(c, MRF_ERR_INVALID_ARG, "NULL output");
    float* dst = out;
    if (!out_is_device) {
        CK(c->marg.ensure((size_t)c->V, 0, c->stream));
        dst = c->marg.p;
    }
    {
        ProfScope ps(c, MRF_K_MARGINALS);
        launch_marginals(c->grid, c->T.p, c->L0, dst, c->stream);
        CK_LAUNCH(MRF_K_MARGINALS, 1);
    }
    if (!out_is_device)
        CK(cudaMemcpyAsync(out, dst, sizeof(float) * c->V, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return MRF_OK;
}

mrf_status mrf_evaluate(mrf_ctx* ctx, const float* depth, int32_t width, int32_t height, const double K[4],
                        const double T_wc[12], int32_t mode, double k_sigma, double vis_threshold, int8_t* cls,
                        int64_t* n_valid, int64_t* n_accurate) {
    ENTER(ctx);
    if (!depth || !K || !T_wc) return set_err(c, MRF_ERR_INVALID_ARG, "NULL argument");
    if (width <= 0 || height <= 0) return set_err(c, MRF_ERR_INVALID_ARG, "width/height must be > 0");
    if (!(k_sigma > 0) || !(vis_threshold > 0 && vis_threshold < 1) || (mode != MRF_EVAL_SIGMA_BAND && mode != MRF_EVAL_VOXEL_BOUNDS))
        return set_err(c, MRF_ERR_INVALID_ARG, "need k_sigma > 0, 0 < vis_threshold < 1 and a known mode");
    if (c->patch_px && ((long long)width > (long long)c->patch_px * c->patch_nx ||
                        (long long)height > (long long)c->patch_px * c->patch_ny))
        return set_err(c, MRF_ERR_INVALID_ARG, "image larger than the patch grid of the noise model");
    if (!finite_all(K, 4) || !(K[0] > 0) || !(K[1] > 0)) return set_err(c, MRF_ERR_INVALID_ARG, "bad K");
    if (!finite_all(T_wc, 12)) return set_err(c, MRF_ERR_INVALID_ARG, "T_wc must be finite");
    const double org[3] = {c->grid.ox, c->grid.oy, c->grid.oz};
    const int dims[3] = {c->grid.nx, c->grid.ny, c->grid.nz};
    for (int k = 0; k < 3; ++k) {
        const double g = (T_wc[4 * k + 3] - org[k]) / c->grid.res;
        if (!(g >= 0.0 && g < (double)dims[k]))
            return set_err(c, MRF_ERR_INVALID_ARG, "camera centre lies outside the grid");
    }
    const size_t npix = (size_t)width * height;
    const float* d_depth = depth;
    cudaPointerAttributes attr;
    cudaError_t pe = cudaPointerGetAttributes(&attr, depth);
    if (pe != cudaSuccess) cudaGetLastError();
    if (!(pe == cudaSuccess && (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged))) {
        CK(c->depth_stage.ensure(npix, 0, c->stream));
        CK(cudaMemcpyAsync(c->depth_stage.p, depth, npix * sizeof(float), cudaMemcpyHostToDevice, c->stream));
        d_depth = c->depth_stage.p;
    }
    CK(c->eval_cls.ensure(npix, 0, c->stream));
    CK(cudaMemsetAsync(c->eval_cls.p, -2, npix, c->stream));
    CK(cudaMemsetAsync(c->counters.p + 8, 0, 2 * sizeof(unsigned long long), c->stream));
    FrameDesc f{};
    f.fx = K[0]; f.fy = K[1]; f.cx = K[2]; f.cy = K[3];
    for (int k = 0; k < 3; ++k) {
        for (int j = 0; j < 3; ++j) f.R[3 * k + j] = T_wc[4 * k + j];
        f.C[k] = T_wc[4 * k + 3];
    }
    f.W = width; f.H = height; f.rank = c->rank; f.world = c->world;
    f.rows_owned = height > c->rank ? (height - c->rank + c->world - 1) / c->world : 0;
    f.ray_base = 0;
    // R19: the evaluation ray runs to 1.5 x the grid diagonal (past the boundary from any camera
    // inside the grid); same expression as the oracle's
    const double D = c->grid.res * std::sqrt((double)dims[0] * dims[0] + (double)dims[1] * dims[1] +
                                             (double)dims[2] * dims[2]);
    launch_eval(f, c->grid, c->noise, d_depth, c->T.p, c->L0, k_sigma, vis_threshold, mode, 1.5 * D, c->eval_cls.p,
                c->counters.p + 8, c->stream);
    CK_LAUNCH(MRF_K_MARGINALS, 1);
    CK(cudaMemcpyAsync(c->pinned, c->counters.p + 8, 2 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
    if (cls) CK(cudaMemcpyAsync(cls, c->eval_cls.p, npix, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (n_valid) *n_valid = c->pinned[0];
    if (n_accurate) *n_accurate = c->pinned[1];
    return MRF_OK;
}

mrf_status mrf_layout_sizes(mrf_ctx* ctx, int64_t* n_slots, int64_t* n_runs, int64_t* n_belief_slots) {
    ENTER(ctx);
    mrf_status st;
    if ((st = prepare(c)) != MRF_OK) return st;
    if (n_slots) *n_slots = c->E;
    if (n_runs) *n_runs = c->n_runs;
    if (n_belief_slots) *n_belief_slots = c->VI;
    return MRF_OK;
}

mrf_status mrf_k6_path(mrf_ctx* ctx, int32_t* path) {
    ENTER(ctx);
    if (!path) return set_err(c, MRF_ERR_INVALID_ARG, "NULL output");
    mrf_status st;
    if ((st = prepare(c)) != MRF_OK) return st;
    *path = c->any_block() ? 1 : 0;
    return MRF_OK;
}

mrf_status mrf_graph_sizes(mrf_ctx* ctx, int64_t* n_rays, int64_t* n_incidences, int64_t* n_active_vox,
                           int64_t* n_invalid, int64_t* n_dropped) {
    ENTER(ctx);
    {
        mrf_status sf = sync_fill(c);
        if (sf != MRF_OK) return sf;
    }
    if (n_rays) *n_rays = c->n_kept;
    if (n_incidences) *n_incidences = c->E_real;
    if (n_invalid) *n_invalid = c->n_invalid;
    if (n_dropped) *n_dropped = c->n_dropped;
    if (n_active_vox && c->mf) {
        *n_active_vox = -1;  // matrix-free: vid is not stored
    } else if (n_active_vox) {
        CK(c->flags.ensure((size_t)c->VI + 1, 0, c->stream));
        CK(c->pos.ensure((size_t)c->VI + 1, 0, c->stream));
        mrf_status sh;
        if ((sh = voxel_histogram(c)) != MRF_OK) return sh;
        launch_active_flags(c->VI, c->vox_count.p, c->flags.p, c->stream);
        CK_LAUNCH(MRF_K_SCAN, 1);
        mrf_status st;
        if ((st = scan(c, c->flags.p, c->pos.p, c->VI, 0)) != MRF_OK) return st;
        long long a = 0;
        if ((st = read_ll(c, c->pos.p + c->VI, &a)) != MRF_OK) return st;
        *n_active_vox = a;
    }
    CK(cudaStreamSynchronize(c->stream));
    return MRF_OK;
}

mrf_status mrf_export_graph(mrf_ctx* ctx, int64_t* ray_pixel, int64_t* row_ptr, int32_t* vid, int16_t* off_q) {
    ENTER(ctx);
    if (c->mf) return set_err(c, MRF_ERR_STATE, "matrix-free mode: the ray->voxel lists are not stored");
    HostLayout h;
    mrf_status st;
    if ((st = host_layout(c, h)) != MRF_OK) return st;
    if (ray_pixel || row_ptr) {
        long long k = 0;
        for (size_t fi = 0; fi < c->frames.size(); ++fi) {
            const FrameRec& fr = c->frames[fi];
            for (long long i = 0; i < fr.n_rays; ++i) {
                const long long r = fr.ray_base + i;
                if (h.status[r] != 0) continue;
                const long long lr = i / fr.W, u = i % fr.W, v = c->rank + lr * c->world;
                if (ray_pixel) ray_pixel[k] = ((long long)fi << 32) | (v * fr.W + u);
                if (row_ptr) row_ptr[k] = h.canon[r];
                ++k;
            }
        }
        if (row_ptr) row_ptr[k] = c->E_real;
    }
    if (vid && c->E) {
        std::vector<int32_t> tmp((size_t)c->E);
        CK(cudaMemcpyAsync(tmp.data(), c->vid.p, sizeof(int32_t) * c->E, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        relayout(h, tmp.data(), vid, sizeof(int32_t), true);
        for (long long e = 0; e < c->E_real; ++e) vid[e] = (int32_t)slot_to_voxel(c->grid, vid[e]);
    }
    if (off_q && c->E) {
        std::vector<int16_t> tmp((size_t)c->E);
        CK(cudaMemcpyAsync(tmp.data(), c->off_q.p, sizeof(int16_t) * c->E, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
        relayout(h, tmp.data(), off_q, sizeof(int16_t), true);
    }
    return MRF_OK;
}

mrf_status mrf_export_rays(mrf_ctx* ctx, int64_t n, const int32_t* frame, const int64_t* pixel, int64_t cap,
                           int64_t* row_ptr, int32_t* vid, int16_t* off_q, float* lambda) {
    ENTER(ctx);
    if (n < 0 || (n > 0 && (!frame || !pixel)) || cap < 0) return set_err(c, MRF_ERR_INVALID_ARG, "bad ray selection");
    if (c->mf) return set_err(c, MRF_ERR_STATE, "matrix-free mode: the ray->voxel lists are not stored");
    {
        mrf_status sf = sync_fill(c);
        if (sf != MRF_OK) return sf;
    }
    std::vector<long long> rid((size_t)n);
    for (long long k = 0; k < n; ++k) {
        if (frame[k] < 0 || frame[k] >= (int)c->frames.size()) return set_err(c, MRF_ERR_INVALID_ARG, "bad frame id");
        const FrameRec& fr = c->frames[(size_t)frame[k]];
        const long long v = pixel[k] / fr.W, u = pixel[k] % fr.W;
        if (pixel[k] < 0 || v >= fr.H || v % c->world != c->rank)
            return set_err(c, MRF_ERR_INVALID_ARG, "pixel not owned by this rank");
        rid[(size_t)k] = fr.ray_base + (v / c->world) * fr.W + u;
    }
    // per selected ray: padded start and record (one gather kernel, two copies)
    std::vector<long long> e0((size_t)n);
    std::vector<RayInfo> info((size_t)n);
    DBuf<long long> d_sel;   // rid [n] | e0 [n] | off [n + 1]
    DBuf<RayInfo> d_info;
    struct Free {
        DBuf<long long>& a;
        DBuf<RayInfo>& b;
        ~Free() { a.release(); b.release(); }
    } free_{d_sel, d_info};
    CK(d_sel.ensure((size_t)(3 * n + 1), 0, c->stream));
    CK(d_info.ensure((size_t)std::max<long long>(n, 1), 0, c->stream));
    if (n) {
        CK(cudaMemcpyAsync(d_sel.p, rid.data(), sizeof(long long) * n, cudaMemcpyHostToDevice, c->stream));
        launch_ray_select(n, d_sel.p, c->row_ptr.p, c->ray_z.p, d_sel.p + n, d_info.p, c->stream);
        CK_LAUNCH(MRF_K_SCAN, 1);
        CK(cudaMemcpyAsync(e0.data(), d_sel.p + n, sizeof(long long) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaMemcpyAsync(info.data(), d_info.p, sizeof(RayInfo) * n, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));
    }
    std::vector<long long> off((size_t)n + 1, 0);
    for (long long k = 0; k < n; ++k) off[(size_t)k + 1] = off[(size_t)k] + info[(size_t)k].n;
    if (row_ptr) std::copy(off.begin(), off.end(), row_ptr);
    if (off[(size_t)n] > cap && (vid || off_q || lambda)) return set_err(c, MRF_ERR_CAPACITY, "rays exceed cap");
    const long long tot_e = off[(size_t)n];
    if (tot_e && (vid || off_q || lambda)) {
        // the incidences, gathered into contiguous staging arrays on the device
        DBuf<int32_t> s32;  // vid [tot] | lam [tot]
        DBuf<int16_t> s16;
        struct Free2 {
            DBuf<int32_t>& a;
            DBuf<int16_t>& b;
            ~Free2() { a.release(); b.release(); }
        } free2_{s32, s16};
        CK(s32.ensure((size_t)(2 * tot_e), 0, c->stream));
        CK(s16.ensure((size_t)tot_e, 0, c->stream));
        CK(cudaMemcpyAsync(d_sel.p + 2 * n, off.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, c->stream));
        launch_ray_gather(n, d_sel.p + n, d_sel.p + 2 * n, c->vid.p, c->off_q.p, c->lam.p, vid ? s32.p : nullptr,
                          off_q ? s16.p : nullptr, lambda ? s32.p + tot_e : nullptr, c->stream);
        CK_LAUNCH(MRF_K_SCAN, 1);
        if (vid) CK(cudaMemcpyAsync(vid, s32.p, sizeof(int32_t) * tot_e, cudaMemcpyDeviceToHost, c->stream));
        if (off_q) CK(cudaMemcpyAsync(off_q, s16.p, sizeof(int16_t) * tot_e, cudaMemcpyDeviceToHost, c->stream));
        if (lambda)  // raw int32 q first, converted below
            CK(cudaMemcpyAsync(lambda, s32.p + tot_e, sizeof(int32_t) * tot_e, cudaMemcpyDeviceToHost, c->stream));
        CK(cudaStreamSynchronize(c->stream));  // before the staging buffers are freed
    }
    CK(cudaStreamSynchronize(c->stream));
    const long long tot = off[(size_t)n];
    if (vid)
        for (long long e = 0; e < tot; ++e) vid[e] = (int32_t)slot_to_voxel(c->grid, vid[e]);
    if (lambda)
        for (long long e = 0; e < tot; ++e) {
            int32_t q;
            memcpy(&q, lambda + e, sizeof q);
            lambda[e] = (float)((double)q * kQInvD);
        }
    return MRF_OK;
}

mrf_status mrf_export_transpose(mrf_ctx* ctx, int64_t* col_ptr, int32_t* tr) {
    ENTER(ctx);
    if (c->mf) return set_err(c, MRF_ERR_STATE, "matrix-free mode: the ray->voxel lists are not stored");
    mrf_status st;
    if ((st = prepare(c)) != MRF_OK) return st;
    if ((st = build_voxel_transpose(c)) != MRF_OK) return st;
    std::vector<long long> cp((size_t)c->VI + 1);
    CK(cudaMemcpyAsync(cp.data(), c->col_ptr.p, sizeof(long long) * (c->VI + 1), cudaMemcpyDeviceToHost, c->stream));
    std::vector<int32_t> tmp((size_t)std::max(1LL, c->E_real));
    if (c->E_real)
        CK(cudaMemcpyAsync(tmp.data(), c->tr.p, sizeof(int32_t) * c->E_real, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    HostLayout h;
    if ((st = host_layout(c, h)) != MRF_OK) return st;
    // padded slot -> canonical incidence index
    std::vector<long long> map((size_t)std::max(1LL, c->E), -1);
    for (size_t r = 0; r < h.info.size(); ++r)
        for (int j = 0; j < h.info[r].n; ++j) map[(size_t)h.row_ptr[r] + j] = h.canon[r] + j;
    // external voxel order
    std::vector<long long> slot_of((size_t)c->V);
    for (long long s = 0; s < c->VI; ++s) {
        const GridDesc& g = c->grid;
        int x, y, z;
        slot_xyz(g, s, x, y, z);
        if (x < g.nx && y < g.ny && z < g.nz) slot_of[(size_t)(x + (long long)g.nx * (y + (long long)g.ny * z))] = s;
    }
    long long k = 0;
    for (long long v = 0; v < c->V; ++v) {
        const long long s = slot_of[(size_t)v];
        if (col_ptr) col_ptr[v] = k;
        for (long long i = cp[(size_t)s]; i < cp[(size_t)s + 1]; ++i, ++k)
            if (tr) tr[k] = (int32_t)map[(size_t)tmp[(size_t)i]];
    }
    if (col_ptr) col_ptr[c->V] = k;
    return MRF_OK;
}

mrf_status mrf_export_messages(mrf_ctx* ctx, float* lambda) {
    ENTER(ctx);
    if (!lambda) return set_err(c, MRF_ERR_INVALID_ARG, "NULL output");
    if (c->kf_chunked())
        return set_err(c, MRF_ERR_STATE,
                       "keyframe averages with matrix-free walks keep no per-incidence messages "
                       "(mrf_export_keyframe_average exports the state)");
    if (!c->E) return MRF_OK;
    HostLayout h;
    mrf_status st;
    if ((st = host_layout(c, h)) != MRF_OK) return st;
    std::vector<int32_t> q((size_t)c->E), qc((size_t)c->E_real);
    CK(cudaMemcpyAsync(q.data(), c->lam.p, sizeof(int32_t) * c->E, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    relayout(h, q.data(), qc.data(), sizeof(int32_t), true);
    for (long long e = 0; e < c->E_real; ++e) lambda[e] = (float)((double)qc[e] * kQInvD);
    return MRF_OK;
}

mrf_status mrf_import_messages(mrf_ctx* ctx, const float* lambda) {
    ENTER(ctx);
    if (!lambda) return set_err(c, MRF_ERR_INVALID_ARG, "NULL input");
    if (c->kf_chunked())
        return set_err(c, MRF_ERR_STATE, "keyframe averages with matrix-free walks keep no per-incidence messages");
    {
        mrf_status sf = sync_fill(c);
        if (sf != MRF_OK) return sf;
    }
    std::vector<int32_t> qc((size_t)c->E_real), q((size_t)c->E, 0);
    for (long long e = 0; e < c->E_real; ++e) {
        double x = lambda[e];
        if (!std::isfinite(x)) return set_err(c, MRF_ERR_INVALID_ARG, "non-finite message");
        x = std::min(256.0, std::max(-256.0, x)) * 8388608.0;
        const double r = std::nearbyint(x);
        qc[e] = r >= 2147483647.0 ? 2147483647 : (int32_t)r;
    }
    HostLayout h;
    mrf_status st;
    if ((st = host_layout(c, h)) != MRF_OK) return st;
    relayout(h, qc.data(), q.data(), sizeof(int32_t), false);
    if (c->E) CK(cudaMemcpyAsync(c->lam.p, q.data(), sizeof(int32_t) * c->E, cudaMemcpyHostToDevice, c->stream));
    st = (c->world > 1 && c->comm_mode == MRF_COMM_EXTERNAL) ? prepare(c) : rebuild_T(c);
    CK(cudaStreamSynchronize(c->stream));
    return st;
}

mrf_status mrf_export_beliefs(mrf_ctx* ctx, int64_t* T) {
    ENTER(ctx);
    if (!T) return set_err(c, MRF_ERR_INVALID_ARG, "NULL output");
    std::vector<long long> tmp((size_t)c->VI);
    CK(cudaMemcpyAsync(tmp.data(), c->T.p, sizeof(long long) * c->VI, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const GridDesc& g = c->grid;
    for (long long v = 0; v < c->V; ++v) {
        const int x = (int)(v % g.nx), y = (int)((v / g.nx) % g.ny), z = (int)(v / ((long long)g.nx * g.ny));
        T[v] = tmp[(size_t)voxel_slot(g, x, y, z)];
    }
    return MRF_OK;
}

mrf_status mrf_set_message_mode(mrf_ctx* ctx, int32_t mode) {
    ENTER(ctx);
    if (mode != MRF_MSG_PER_RAY && mode != MRF_MSG_KEYFRAME_AVG) return set_err(c, MRF_ERR_INVALID_ARG, "bad mode");
    if (!c->frames.empty()) return set_err(c, MRF_ERR_STATE, "the message mode is set before the first frame");
    if (mode == MRF_MSG_KEYFRAME_AVG && c->world > 1)
        return set_err(c, MRF_ERR_INVALID_ARG, "keyframe averages are single-rank (a keyframe's rays span ranks)");
    c->kf_avg = mode == MRF_MSG_KEYFRAME_AVG;
    if (c->kf_avg) {
        c->k5_staged = false;  // the class / long-ray K5 kernels carry the keyframe cavity
        c->k6_voxel = false;   // the averages are tile-run reductions
    }
    c->kf_frames_alloc = 0;
    c->dirty = true;
    return MRF_OK;
}

mrf_status mrf_set_sparse_bricks(mrf_ctx* ctx, int32_t brick) {
    ENTER(ctx);
    if (brick != 0 && (brick < 2 || brick > 64 || (brick & (brick - 1))))
        return set_err(c, MRF_ERR_INVALID_ARG, "brick edge must be 0 (dense) or a power of two in [2, 64]");
    if (!c->frames.empty()) return set_err(c, MRF_ERR_STATE, "sparse bricks are set before the first frame");
    c->brick = brick;
    if (brick == 0) {
        c->grid.bmask = nullptr;
        return MRF_OK;
    }
    const int nb[3] = {(c->grid.nx + brick - 1) / brick, (c->grid.ny + brick - 1) / brick,
                       (c->grid.nz + brick - 1) / brick};
    c->n_brick_slots = (long long)nb[0] * nb[1] * nb[2];
    CK(c->bmask.ensure((size_t)c->n_brick_slots, 0, c->stream));
    CK(cudaMemsetAsync(c->bmask.p, 0, (size_t)c->n_brick_slots, c->stream));
    c->grid.bmask = c->bmask.p;
    c->grid.bshift = __builtin_ctz((unsigned)brick);
    c->grid.nbx = nb[0];
    c->grid.nby = nb[1];
    c->dirty = true;
    return MRF_OK;
}

mrf_status mrf_set_patch_noise(mrf_ctx* ctx, int32_t patch_px, int32_t n_px, int32_t n_py, const double* coeffs,
                               double sigma_min) {
    ENTER(ctx);
    if (!c->frames.empty()) return set_err(c, MRF_ERR_STATE, "the noise model is set before the first frame");
    if (patch_px == 0) {  // back to the global model (the LUT)
        c->noise.pcoef = nullptr;
        c->mp.pcoef = nullptr;
        c->patch_px = c->patch_nx = c->patch_ny = 0;
        return MRF_OK;
    }
    if (!coeffs) return set_err(c, MRF_ERR_INVALID_ARG, "NULL coefficients");
    if (patch_px < 1 || n_px < 1 || n_py < 1 || (long long)n_px * n_py > (1 << 24))
        return set_err(c, MRF_ERR_INVALID_ARG, "need patch_px >= 1 and 1 <= n_px * n_py <= 2^24");
    if (!std::isfinite(sigma_min) || !(sigma_min > 0)) return set_err(c, MRF_ERR_INVALID_ARG, "sigma_min must be > 0");
    const long long np = (long long)n_px * n_py;
    if (!finite_all(coeffs, (int)(6 * np))) return set_err(c, MRF_ERR_INVALID_ARG, "coefficients must be finite");
    // the margin bound of mrf_create over every patch: 3 sigma stays below the grid diagonal, and
    // the longest walk (ray_slots_max) covers the largest margin
    const GridDesc& g = c->grid;
    const double D = g.res * std::sqrt((double)g.nx * g.nx + (double)g.ny * g.ny + (double)g.nz * g.nz);
    double m_max = c->noise.margin_min;
    for (long long p = 0; p < np; ++p) {
        const double* k = coeffs + 6 * p;
        const double sig = std::fabs(k[3]) + std::fabs(k[4]) * D + std::fabs(k[5]) * D * D;
        if (c->noise.margin_k * sig > D)
            return set_err(c, MRF_ERR_INVALID_ARG, "traversal margin must stay below the grid diagonal (margin bound)");
        m_max = std::max(m_max, c->noise.margin_k * sig);
    }
    const long long margin_cells = (long long)std::ceil(m_max / g.res) + 1;
    c->ray_slots_max = std::max(c->ray_slots_max, (1 + (long long)g.nx + g.ny + g.nz + 3 * margin_cells + 7) & ~7LL);
    std::vector<float4> f((size_t)(2 * np));
    for (long long p = 0; p < np; ++p) {
        const double* k = coeffs + 6 * p;
        f[2 * p] = make_float4((float)k[0], (float)k[1], (float)k[2], 0.f);
        f[2 * p + 1] = make_float4((float)k[3], (float)k[4], (float)k[5], (float)sigma_min);
    }
    CK(c->pcoef_d.ensure((size_t)(6 * np), 0, c->stream));
    CK(c->pcoef_f.ensure((size_t)(2 * np), 0, c->stream));
    CK(cudaMemcpyAsync(c->pcoef_d.p, coeffs, sizeof(double) * 6 * np, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->pcoef_f.p, f.data(), sizeof(float4) * 2 * np, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    c->noise.pcoef = c->pcoef_d.p;
    c->noise.ppx = patch_px;
    c->noise.pnx = n_px;
    c->mp.pcoef = c->pcoef_f.p;
    c->patch_px = patch_px;
    c->patch_nx = n_px;
    c->patch_ny = n_py;
    c->dirty = true;
    return MRF_OK;
}

mrf_status mrf_export_bricks(mrf_ctx* ctx, uint8_t* out, int64_t* n_allocated) {
    ENTER(ctx);
    if (!c->grid.bmask) return set_err(c, MRF_ERR_STATE, "not a sparse-brick map");
    std::vector<uint8_t> m((size_t)c->n_brick_slots);
    CK(cudaMemcpyAsync(m.data(), c->bmask.p, m.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    long long na = 0;
    for (uint8_t x : m) na += x != 0;
    if (out) memcpy(out, m.data(), m.size());
    if (n_allocated) *n_allocated = na;
    return MRF_OK;
}

mrf_status mrf_set_matrix_free(mrf_ctx* ctx, int32_t frames_per_chunk) {
    ENTER(ctx);
    if (frames_per_chunk < 0) return set_err(c, MRF_ERR_INVALID_ARG, "frames_per_chunk must be >= 0");
    if (!c->frames.empty()) return set_err(c, MRF_ERR_STATE, "the matrix-free mode is set before the first frame");
    c->mf = frames_per_chunk;
    if (c->mf) {
        c->k5_staged = false;  // the class / long-ray kernels read the scratch
        c->k6_voxel = false;   // the per-voxel transpose needs vid
    }
    c->dirty = true;
    return MRF_OK;
}

mrf_status mrf_export_keyframe_average(mrf_ctx* ctx, int64_t frame, float* out) {
    ENTER(ctx);
    if (!out) return set_err(c, MRF_ERR_INVALID_ARG, "NULL output");
    if (!c->kf_avg) return set_err(c, MRF_ERR_STATE, "not in keyframe-average mode");
    if (frame < 0 || frame >= (int64_t)c->frames.size()) return set_err(c, MRF_ERR_INVALID_ARG, "bad frame id");
    mrf_status st;
    if ((st = ensure_kf(c)) != MRF_OK) return st;
    std::vector<int32_t> q((size_t)c->VI);
    CK(cudaMemcpyAsync(q.data(), c->qbar.p + frame * c->VI, sizeof(int32_t) * c->VI, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    const GridDesc& g = c->grid;
    long long v = 0;
    for (int z = 0; z < g.nz; ++z)
        for (int y = 0; y < g.ny; ++y)
            for (int x = 0; x < g.nx; ++x, ++v) out[v] = (float)((double)q[(size_t)voxel_slot(g, x, y, z)] * kQInvD);
    return MRF_OK;
}

mrf_status mrf_nccl_unique_id(unsigned char out[128]) {
    if (!out) return MRF_ERR_INVALID_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return MRF_ERR_NCCL;
    memcpy(out, id.internal, 128);
    return MRF_OK;
}

mrf_status mrf_set_profiling(mrf_ctx* ctx, int32_t on) {
    ENTER(ctx);
    c->prof = on != 0;
    return MRF_OK;
}

mrf_status mrf_profile_read(mrf_ctx* ctx, int64_t* launches, double* total_ms) {
    ENTER(ctx);
    CK(cudaStreamSynchronize(c->stream));
    for (auto& e : c->events) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e.a, e.b));
        c->prof_ms[e.kind] += ms;
        c->ev_pool.push_back(e.a);
        c->ev_pool.push_back(e.b);
    }
    c->events.clear();
    for (int k = 0; k < MRF_K_COUNT; ++k) {
        if (launches) launches[k] = c->prof_launch[k];
        if (total_ms) total_ms[k] = c->prof_ms[k];
        c->prof_launch[k] = 0;
        c->prof_ms[k] = 0.0;
    }
    return MRF_OK;
}

int64_t mrf_launch_count(const mrf_ctx* ctx) { return ctx ? ctx->launches : 0; }

int64_t mrf_belief_slots(const mrf_ctx* ctx) { return ctx ? ctx->VI : 0; }

}  // extern "C"
