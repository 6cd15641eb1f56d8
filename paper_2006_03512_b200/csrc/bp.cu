// bp.cu -- loopy sum-product BP iteration on sm_100a: K5 (per-ray factor->voxel messages),
// K6 (voxel beliefs as a segmented reduction over the voxel->ray transpose), K8 (marginals).
//
// Messages (Eq.13, Eq.14 P:158-161 in the division-free form of P:524),
// rewritten for a parallel scan.  For the voxels i = 1..N of a ray, with the
// cavity log-odds c_i = L0 + T_v - lambda_i (Eq.6), mu(o_i=1) = sigma(c_i),
// mu(o_i=0) = sigma(-c_i) (normalised incoming messages) and nu_i from the LUT:
//     a_i = mu(o_i=0),  w_i = mu(o_i=1) nu_i
//     Q_i = P_i / V_i,  Q_1 = 0,  Q_{i+1} = (Q_i + w_i) / a_i                 (prefix, "visibility")
//     R_i = sum_{j>i} mu(o_j=1) nu_j prod_{i<k<j} mu(o_k=0),
//           R_N = 0,  R_{i-1} = a_i R_i + w_i                                  (suffix)
//     lambda_i = log mu_{psi->o_i}(1) - log mu_{psi->o_i}(0) = log(Q_i + nu_i) - log(Q_i + R_i)
// where P_i = sum_{j<i} mu(o_j=1) nu_j V_j and V_i = prod_{k<i} mu(o_k=0) are the terms of
// Eq.13/14; dividing both messages by V_i leaves the log-odds unchanged and keeps every
// quantity O(1) in the log domain.  Both recurrences are affine maps x -> 2^a x + 2^b, so a warp
// composes per-lane chunks and runs two 5-level shuffle scans (prefix for Q, suffix for R).
// Everything is evaluated in natural logs (the units of the input table): e^x as ex2.approx on the
// MUFU, ln(1+y) as a polynomial on the FMA pipe (relative accuracy, see log1pn), and lambda
// without cancellation (lambda_n).
//
// Layout: warp per ray; lane l owns the K consecutive incidences [e0 + l*K, e0 + l*K + K) of
// the ray; ray segments start at multiples of 4 (RayInfo), so vid/lambda are read as 16-byte
// vectors and the partition -- hence every rounding -- is independent of where the ray is
// stored (bit-identical results for any rank count).  Elements past e1 are masked to the
// identity map.  Rays are
// bucketed by span into K = 4 / 8 / 16 (single tile of 32K in registers); longer rays run a
// tiled two-pass variant with the suffix values staged in a per-warp global scratch.
#include "internal.cuh"

namespace mrf {
namespace {

#ifndef MRF_ACCURATE_RECURRENCES
#define MRF_ACCURATE_RECURRENCES 1
#endif

constexpr unsigned kFull = 0xffffffffu;
constexpr float kNeg = -1e30f;  // log2(0); finite so that NEG - NEG = 0 stays NaN-free

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// ln(1 + y) for y in [0, 1] with RELATIVE accuracy (~2e-7), on the FMA pipe: y * P(y), P a
// degree-8 fit of ln(1+y)/y.  (lg2.approx(1+y) is only absolutely accurate near 1, which biased
// the tiny messages of occluded voxels.)
__device__ __forceinline__ float log1pn(float y) {
    float r = 0.00523269456f;
    r = fmaf(r, y, -0.0295052417f);
    r = fmaf(r, y, 0.0782259554f);
    r = fmaf(r, y, -0.136632457f);
    r = fmaf(r, y, 0.191060066f);
    r = fmaf(r, y, -0.24842982f);
    r = fmaf(r, y, 0.333190978f);
    r = fmaf(r, y, -0.499994934f);
    r = fmaf(r, y, 0.99999994f);
    return r * y;
}
// e^x on the MUFU (ex2.approx, relative error ~2^-22)
__device__ __forceinline__ float expn(float x) { return ex2(x * kLog2e); }
// ln(e^a + e^b), relative-accurate remainder.  Every log-domain quantity is kept in nats, the
// units of the input table, so no large value is ever rescaled (a nats->bits conversion of a
// value near the table floor, ~-100, would round at ~1e-5).
__device__ __forceinline__ float lse(float a, float b) {
    return fmaxf(a, b) + log1pn(expn(-fabsf(a - b)));
}

// Affine map x -> e^a x + e^b in log form (nats).
struct Aff {
    float a, b;
};
// outer o inner (inner applied first)
__device__ __forceinline__ Aff compose(Aff outer, Aff inner) {
    return {outer.a + inner.a, lse(outer.a + inner.b, outer.b)};
}
template <int G>
__device__ __forceinline__ Aff shfl_up(Aff v, int d) {
    return {__shfl_up_sync(kFull, v.a, d, G), __shfl_up_sync(kFull, v.b, d, G)};
}
template <int G>
__device__ __forceinline__ Aff shfl_down(Aff v, int d) {
    return {__shfl_down_sync(kFull, v.a, d, G), __shfl_down_sync(kFull, v.b, d, G)};
}
template <int G>
__device__ __forceinline__ Aff shfl_idx(Aff v, int l) {
    return {__shfl_sync(kFull, v.a, l, G), __shfl_sync(kFull, v.b, l, G)};
}

// ---------------------------------------------------------------- per-lane element loads
// For the K elements [s, s+K) of this lane (nats):
//   la = log mu(o=0) = -softplus(c),  w = log mu(o=1) + log nu,  l = log nu.
// la and log mu(o=1) share one ex2 and are both computed directly, never as a difference of
// two large numbers.  Masked elements get the identity maps (la = 0, w = NEG).
template <int K>
__device__ __forceinline__ void load_elems(long long s, long long e0, long long e1, const float2* __restrict__ rowA,
                                           const float2* __restrict__ rowB, float wz, const MsgParams& mp,
                                           const int32_t* __restrict__ vid, const int16_t* __restrict__ off_q,
                                           const int32_t* __restrict__ lam, const long long* __restrict__ T,
                                           float (&la)[K], float (&w)[K], float (&l)[K]) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
        la[j] = 0.f;
        w[j] = kNeg;
        l[j] = kNeg;
    }
    if (s >= e1) return;
    int v[K], q[K];
    short o[K];
#pragma unroll
    for (int j = 0; j < K; j += 4) {
        const int4 a = __ldg(reinterpret_cast<const int4*>(vid + s + j));
        const int4 b = __ldg(reinterpret_cast<const int4*>(lam + s + j));
        const uint2 c = __ldg(reinterpret_cast<const uint2*>(off_q + s + j));
        v[j] = a.x; v[j + 1] = a.y; v[j + 2] = a.z; v[j + 3] = a.w;
        q[j] = b.x; q[j + 1] = b.y; q[j + 2] = b.z; q[j + 3] = b.w;
        o[j] = (short)(c.x & 0xffff); o[j + 1] = (short)(c.x >> 16);
        o[j + 2] = (short)(c.y & 0xffff); o[j + 3] = (short)(c.y >> 16);
    }
    long long t[K];
#pragma unroll
    for (int j = 0; j < K; ++j) t[j] = (s + j < e1) ? __ldg(T + v[j]) : 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (s + j < e1) {
            // cavity (Eq.6): prior + every other incoming message, exact in fixed point
            const float c = fmaf(__ll2float_rn(t[j] - (long long)q[j]), kQInv, mp.L0);
            float fo = fmaf((float)o[j], mp.s_off, mp.b_off);
            fo = fminf(fmaxf(fo, 0.f), mp.fo_max);
            const int io = min((int)fo, mp.n_offm1 - 1);
            const float wo = fo - (float)io;
            const float2 ta = __ldg(rowA + io), tb = __ldg(rowB + io);
            const float ra = fmaf(wo, ta.y - ta.x, ta.x);
            const float rb = fmaf(wo, tb.y - tb.x, tb.x);
            const float lnu = fmaf(wz, rb - ra, ra);
            const float L1 = log1pn(expn(-fabsf(c)));  // ln(1 + e^-|c|)
            la[j] = -(fmaxf(c, 0.f) + L1);
            w[j] = lnu - (fmaxf(-c, 0.f) + L1);
            l[j] = lnu;
        }
    }
}

// Lane composite of the suffix maps R -> e^{la} R + e^{w} over the chunk (first applied last):
// aB = sum la, bB = ln sum_j e^{w_j + sum_{k<j} la_k}.  The prefix maps
// Q -> e^{-la} (Q + e^{w}) compose to (-aB, bB - aB).
template <int K>
__device__ __forceinline__ void lane_composite(const float (&la)[K], const float (&w)[K], float& aB, float& bB) {
    float acc = 0.f, m = kNeg, t[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        t[j] = w[j] + acc;
        acc += la[j];
        m = fmaxf(m, t[j]);
    }
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) sum += expn(t[j] - m);
    aB = acc;
    bB = m + lg2(sum) * kLn2;
}

// Both lane scans of a ray's G lanes at once (two independent shuffle chains per level):
// returns R entering this lane from the right and Q entering it from the left, given the tile
// carries Rc (log2 R after the tile) and Qc (log2 Q before it); optional carries out.
template <int G>
__device__ __forceinline__ void lane_scans(float aB, float bB, int sl, float Rc, float Qc, float& Rin, float& Qin,
                                           float* Rc_out, float* Qc_out) {
    Aff H = {aB, bB};          // suffix maps R -> e^{la} R + e^{w}
    Aff P = {-aB, bB - aB};    // prefix maps Q -> e^{-la} (Q + e^{w})
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const Aff oh = shfl_down<G>(H, d);
        const Aff op = shfl_up<G>(P, d);
        if (sl + d < G) H = compose(H, oh);
        if (sl >= d) P = compose(P, op);
    }
    Aff Hx = shfl_down<G>(H, 1);
    Aff Px = shfl_up<G>(P, 1);
    if (sl == G - 1) Hx = {0.f, kNeg};
    if (sl == 0) Px = {0.f, kNeg};
    if (Rc_out) {
        const Aff H0 = shfl_idx<G>(H, 0);
        const Aff Pl = shfl_idx<G>(P, G - 1);
        *Rc_out = lse(H0.a + Rc, H0.b);
        *Qc_out = lse(Pl.a + Qc, Pl.b);
    }
    Rin = lse(Hx.a + Rc, Hx.b);
    Qin = lse(Px.a + Qc, Px.b);
}

// The two per-lane recurrences, interleaved (independent chains):
//   lR[j] = ln R_j (suffix strictly after j),  R_{j-1} = mu(o_j=0) R_j + mu(o_j=1) nu_j
//   lQ[j] = ln Q_j (prefix strictly before j), Q_{j+1} = (Q_j + mu(o_j=1) nu_j) / mu(o_j=0)
template <int K>
__device__ __forceinline__ void lane_recurrences(const float (&la)[K], const float (&w)[K], float Rin, float Qin,
                                                 float (&lR)[K], float (&lQ)[K]) {
    float R = Rin, Q = Qin;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int jb = K - 1 - i;
        lR[jb] = R;
        lQ[i] = Q;
        R = lse(la[jb] + R, w[jb]);
        Q = lse(Q, w[i]) - la[i];
    }
}

// lambda = ln(e^Q + e^l) - ln(e^Q + e^R) without cancellation: the max parts subtract exactly
// (both are Q when Q dominates) and the remainders are small, relative-accurate log1p terms.
__device__ __forceinline__ float lambda_n(float Q, float l, float R) {
    const float m1 = fmaxf(Q, l), m2 = fmaxf(Q, R);
    return (m1 - m2) + (log1pn(expn(-fabsf(Q - l))) - log1pn(expn(-fabsf(Q - R))));
}

__device__ __forceinline__ int32_t quantise(float lam) {
    lam = fminf(fmaxf(lam, -kLambdaClip), kLambdaClip);
    return __float2int_rn(lam * kQScale);  // saturates at +2^31-1 for +256
}

// lambda_j = log(Q_j + nu_j) - log(Q_j + R_j)   (Eq.13 / Eq.14, both divided by V_j)
template <int K>
__device__ __forceinline__ void lane_out(const float (&l)[K], const float (&lR)[K], const float (&lQ)[K], long long s,
                                         long long e1, int32_t* lam) {
    int32_t out[K];
#pragma unroll
    for (int j = 0; j < K; ++j) out[j] = quantise(lambda_n(lQ[j], l[j], lR[j]));
    if (s + K <= e1) {
#pragma unroll
        for (int j = 0; j < K; j += 4)
            *reinterpret_cast<int4*>(lam + s + j) = make_int4(out[j], out[j + 1], out[j + 2], out[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (s + j < e1) lam[s + j] = out[j];
    }
}

// ---------------------------------------------------------------- K5: single-tile classes
// G lanes per ray (32/G rays per warp), K incidences per lane: capacity G*K.
#ifndef MRF_K5_MIN_BLOCKS
#define MRF_K5_MIN_BLOCKS 3
#endif
template <int G, int K>
__global__ void __launch_bounds__(256, MRF_K5_MIN_BLOCKS) ray_msg_kernel(long long n, const int32_t* __restrict__ rays,
                                                      const long long* __restrict__ row_ptr,
                                                      const RayInfo* __restrict__ ray_z,
                                                      const int32_t* __restrict__ vid,
                                                      const int16_t* __restrict__ off_q, int32_t* lam,
                                                      const long long* __restrict__ T, MsgParams mp) {
    constexpr int RPW = 32 / G;
    const long long wi = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wi * RPW >= n) return;  // warp-uniform
    const int lane = threadIdx.x & 31, sl = lane & (G - 1);
    const long long ri = wi * RPW + lane / G;
    RayInfo rz{0, 0.f, 0, 0};
    long long e0 = 0;
    if (ri < n) {
        const int r = __ldg(rays + ri);
        rz = ray_z[r];
        e0 = __ldg(row_ptr + r);
    }
    const long long e1 = e0 + rz.n;
    const float2* rowA = mp.lutp + (long long)rz.iz * mp.n_offm1;
    const float2* rowB = rowA + mp.n_offm1;
    const long long s = e0 + (long long)sl * K;
    float la[K], w[K], l[K], lR[K], lQ[K];
    load_elems<K>(s, e0, e1, rowA, rowB, rz.wz, mp, vid, off_q, lam, T, la, w, l);
    float aB, bB, Rin, Qin;
    lane_composite<K>(la, w, aB, bB);
    lane_scans<G>(aB, bB, sl, kNeg, kNeg, Rin, Qin, nullptr, nullptr);
    lane_recurrences<K>(la, w, Rin, Qin, lR, lQ);
    if (s < e1) lane_out<K>(l, lR, lQ, s, e1, lam);
}

// ---------------------------------------------------------------- K5: long rays (tiled)
constexpr int kLongK = 16;
constexpr int kLongTile = 32 * kLongK;

__global__ void __launch_bounds__(256) ray_msg_long_kernel(long long n, const int32_t* __restrict__ rays,
                                                           const long long* __restrict__ row_ptr,
                                                           const RayInfo* __restrict__ ray_z,
                                                           const int32_t* __restrict__ vid,
                                                           const int16_t* __restrict__ off_q, int32_t* lam,
                                                           const long long* __restrict__ T, MsgParams mp,
                                                           float* scratch, long long scratch_per_warp) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    float* my_scratch = scratch + gw * scratch_per_warp;
    for (long long wi = gw; wi < n; wi += n_warps) {
        const int r = __ldg(rays + wi);
        const RayInfo rz = ray_z[r];
        const long long e0 = __ldg(row_ptr + r), e1 = e0 + rz.n;
        const float2* rowA = mp.lutp + (long long)rz.iz * mp.n_offm1;
        const float2* rowB = rowA + mp.n_offm1;
        const int n_tiles = (int)((e1 - e0 + kLongTile - 1) / kLongTile);
        float la[kLongK], w[kLongK], l[kLongK], lR[kLongK], lQ[kLongK];
        float aB, bB, Rin, Qin, Rc_out, Qc_out;
        // pass 1: suffix values, tiles right to left
        float Rc = kNeg;
        for (int t = n_tiles - 1; t >= 0; --t) {
            const long long s = e0 + (long long)t * kLongTile + (long long)lane * kLongK;
            load_elems<kLongK>(s, e0, e1, rowA, rowB, rz.wz, mp, vid, off_q, lam, T, la, w, l);
            lane_composite<kLongK>(la, w, aB, bB);
            lane_scans<32>(aB, bB, lane, Rc, kNeg, Rin, Qin, &Rc_out, &Qc_out);
            Rc = Rc_out;
            lane_recurrences<kLongK>(la, w, Rin, kNeg, lR, lQ);
            float* dst = my_scratch + (long long)t * kLongTile + lane * kLongK;
#pragma unroll
            for (int j = 0; j < kLongK; j += 4)
                *reinterpret_cast<float4*>(dst + j) = make_float4(lR[j], lR[j + 1], lR[j + 2], lR[j + 3]);
        }
        // pass 2: prefix values and messages, tiles left to right
        float Qc = kNeg;
        for (int t = 0; t < n_tiles; ++t) {
            const long long s = e0 + (long long)t * kLongTile + (long long)lane * kLongK;
            load_elems<kLongK>(s, e0, e1, rowA, rowB, rz.wz, mp, vid, off_q, lam, T, la, w, l);
            lane_composite<kLongK>(la, w, aB, bB);
            lane_scans<32>(aB, bB, lane, kNeg, Qc, Rin, Qin, &Rc_out, &Qc_out);
            Qc = Qc_out;
            lane_recurrences<kLongK>(la, w, kNeg, Qin, lR, lQ);
            const float* src = my_scratch + (long long)t * kLongTile + lane * kLongK;
#pragma unroll
            for (int j = 0; j < kLongK; j += 4) {
                const float4 a = *reinterpret_cast<const float4*>(src + j);
                lR[j] = a.x; lR[j + 1] = a.y; lR[j + 2] = a.z; lR[j + 3] = a.w;
            }
            if (s < e1) lane_out<kLongK>(l, lR, lQ, s, e1, lam);
        }
    }
}

// ---------------------------------------------------------------- K6
// T_v = sum over the transpose column of v of q_e (int64, exact and order-free).  Work item =
// (voxel, chunk of <= kVoxelChunk entries); a warp per item, lanes stride the column so the
// tr reads are coalesced; partial sums of split (hot) voxels meet in an integer atomic.
__global__ void __launch_bounds__(256) voxel_reduce_kernel(long long n_items, const int2* __restrict__ items,
                                                           const long long* __restrict__ col_ptr,
                                                           const int32_t* __restrict__ tr,
                                                           const int32_t* __restrict__ lam, long long* T) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (long long w = gw; w < n_items; w += n_warps) {
        const int2 it = __ldg(items + w);
        const long long c0 = __ldg(col_ptr + it.x);
        const long long k0 = c0 + (long long)it.y * kVoxelChunk;
        long long k1 = __ldg(col_ptr + it.x + 1);
        if (k1 > k0 + kVoxelChunk) k1 = k0 + kVoxelChunk;
        long long acc = 0;
        for (long long k = k0 + lane; k < k1; k += 128) {
            int e[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) e[u] = (k + 32 * u < k1) ? __ldg(tr + k + 32 * u) : -1;
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += (e[u] >= 0) ? (long long)__ldg(lam + e[u]) : 0LL;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
        if (lane == 0 && acc != 0)
            atomicAdd(reinterpret_cast<unsigned long long*>(T + it.x), (unsigned long long)acc);
    }
}

// ---------------------------------------------------------------- K6 (tile-run transpose)
// Same sums, over the tile->ray-run transpose: a CTA (1024 threads) takes a work item (tile t,
// <= kRunsPerItem of its runs).  Groups of 8 lanes read one run's vid/q contiguously and add q
// into the tile's 16384 slots in shared memory, split into 16-bit halves held in two int32
// arrays (native 32-bit shared atomics; a slot gets at most one contribution per run, so the
// halves cannot overflow within an item).  The slots then go to T with one int64 atomic each
// (a tile spans several items).  Integer sums: exact, independent of order and scheduling.
constexpr int kK6Threads = 1024;

__global__ void __launch_bounds__(kK6Threads, 1) tile_reduce_kernel(long long n_items, const int2* __restrict__ items,
                                                                   const long long* __restrict__ tile_ptr,
                                                                   const Run* __restrict__ runs,
                                                                   const int32_t* __restrict__ vid,
                                                                   const int32_t* __restrict__ lam, long long* T) {
    extern __shared__ int smem[];
    int* acc_lo = smem;                 // sum of (q & 0xffff)
    int* acc_hi = smem + kTileSlots;    // sum of (q >> 16)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, sub = lane >> 3, sl = lane & 7;
    constexpr int kWarps = kK6Threads / 32;
    for (long long it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int2 item = __ldg(items + it);
        for (int i = threadIdx.x; i < 2 * kTileSlots; i += kK6Threads) smem[i] = 0;
        __syncthreads();
        const long long r0 = __ldg(tile_ptr + item.x) + (long long)item.y * kRunsPerItem;
        long long r1 = __ldg(tile_ptr + item.x + 1);
        if (r1 > r0 + kRunsPerItem) r1 = r0 + kRunsPerItem;
        for (long long rb = r0 + 4 * wid; rb < r1; rb += 4 * kWarps) {
            Run run{0u, 0u};
            if (rb + sub < r1) {
                const uint2 rr = __ldg(reinterpret_cast<const uint2*>(runs + rb + sub));
                run = Run{rr.x, rr.y};
            }
            for (int k = sl; k < (int)run.n; k += 32) {
                int v[4], q[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const bool ok = k + 8 * u < (int)run.n;
                    const long long e = (long long)run.e + k + 8 * u;
                    v[u] = ok ? __ldg(vid + e) : -1;
                    q[u] = ok ? __ldg(lam + e) : 0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (v[u] >= 0) {
                        const int slot = v[u] & (kTileSlots - 1);
                        atomicAdd(acc_lo + slot, q[u] & 0xffff);
                        atomicAdd(acc_hi + slot, q[u] >> 16);
                    }
                }
            }
        }
        __syncthreads();
        long long* Tt = T + ((long long)item.x << kTileShift);
        for (int i = threadIdx.x; i < kTileSlots; i += kK6Threads) {
            const long long sum = (long long)acc_hi[i] * 65536 + (long long)acc_lo[i];
            if (sum) atomicAdd(reinterpret_cast<unsigned long long*>(Tt + i), (unsigned long long)sum);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- K8
__global__ void marginals_kernel(GridDesc g, const long long* __restrict__ T, double L0, float* out) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long V = (long long)g.nx * g.ny * g.nz;
    if (v >= V) return;
    const int x = (int)(v % g.nx);
    const int y = (int)((v / g.nx) % g.ny);
    const int z = (int)(v / ((long long)g.nx * g.ny));
    const double a = L0 + (double)T[voxel_slot(g, x, y, z)] * kQInvD;  // Eq.8: prior x all incoming messages
    out[v] = (float)(1.0 / (1.0 + exp(-a)));
}

__global__ void lambda_to_float_kernel(long long n, const int32_t* __restrict__ q, float* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (float)((double)q[i] * kQInvD);
}

inline unsigned blocks_for(long long n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

int class_capacity(int cls) { return cls < kNumClasses - 1 ? kLaneK * (kMinGroup << cls) : 0x7fffffff; }

void launch_ray_messages(int cls, long long n_rays, const int32_t* rays, const long long* row_ptr,
                         const RayInfo* ray_z, const int32_t* vid, const int16_t* off_q, int32_t* lam,
                         const long long* T, const MsgParams& mp, float* scratch, long long scratch_per_warp,
                         int n_warps_long, cudaStream_t s) {
    if (n_rays == 0) return;
    auto grid = [&](int G) { return blocks_for((n_rays + 32 / G - 1) / (32 / G) * 32, 256); };
    constexpr int G0 = kMinGroup, K = kLaneK;
    switch (cls) {
        case 0: ray_msg_kernel<G0, K><<<grid(G0), 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, vid, off_q, lam, T, mp); break;
        case 1: ray_msg_kernel<2 * G0, K><<<grid(2 * G0), 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, vid, off_q, lam, T, mp); break;
        case 2: ray_msg_kernel<4 * G0, K><<<grid(4 * G0), 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, vid, off_q, lam, T, mp); break;
        case 3: ray_msg_kernel<8 * G0, K><<<grid(8 * G0), 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, vid, off_q, lam, T, mp); break;
        default: {
            const unsigned g = blocks_for((long long)n_warps_long * 32, 256);
            ray_msg_long_kernel<<<g, 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, vid, off_q, lam, T, mp, scratch,
                                                  scratch_per_warp);
        }
    }
}

void launch_voxel_reduce(long long n_items, const int2* items, const long long* col_ptr, const int32_t* tr,
                         const int32_t* lam, long long* T, cudaStream_t s) {
    if (n_items == 0) return;
    long long warps = n_items < 148LL * 64 ? n_items : 148LL * 64;
    voxel_reduce_kernel<<<blocks_for(warps * 32, 256), 256, 0, s>>>(n_items, items, col_ptr, tr, lam, T);
}

void launch_tile_reduce(long long n_items, const int2* items, const long long* tile_ptr, const Run* runs,
                        const int32_t* vid, const int32_t* lam, long long* T, cudaStream_t s) {
    if (n_items == 0) return;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(tile_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             2 * kTileSlots * (int)sizeof(int));
        configured = true;
    }
    const long long grid = n_items < 148LL ? n_items : 148LL;
    tile_reduce_kernel<<<(unsigned)grid, kK6Threads, 2 * kTileSlots * sizeof(int), s>>>(n_items, items, tile_ptr, runs,
                                                                                     vid, lam, T);
}

void launch_marginals(const GridDesc& g, const long long* T, double L0, float* out, cudaStream_t s) {
    const long long V = (long long)g.nx * g.ny * g.nz;
    marginals_kernel<<<blocks_for(V, 256), 256, 0, s>>>(g, T, L0, out);
}

void launch_lambda_to_float(long long n, const int32_t* q, float* out, cudaStream_t s) {
    if (n == 0) return;
    lambda_to_float_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, q, out);
}

}  // namespace mrf
