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
// Everything is evaluated in base-2 logs: ex2.approx on the MUFU, log2(1+y) as a polynomial on
// the FMA pipe (relative accuracy, see log1p2), and lambda without cancellation (lambda2).
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
// log2(1 + y) for y in [0, 1] with RELATIVE accuracy (~2e-7), on the FMA pipe:
// y * P(y), P a degree-8 fit of log2(1+y)/y (lg2.approx(1+y) is only absolutely accurate
// near 1, which biased the tiny messages of occluded voxels).
__device__ __forceinline__ float log1p2(float y) {
    float r = 0.00754914153367281f;
    r = fmaf(r, y, -0.04256688803434372f);
    r = fmaf(r, y, 0.11285588890314102f);
    r = fmaf(r, y, -0.19711868464946747f);
    r = fmaf(r, y, 0.2756412625312805f);
    r = fmaf(r, y, -0.3584084212779999f);
    r = fmaf(r, y, 0.48069295287132263f);
    r = fmaf(r, y, -0.7213401794433594f);
    r = fmaf(r, y, 1.4426950216293335f);
    return r * y;
}
// log2(2^a + 2^b)
__device__ __forceinline__ float lse2(float a, float b) {
    return fmaxf(a, b) + log1p2(ex2(-fabsf(a - b)));
}

// Affine map x -> 2^a x + 2^b in log2 form.
struct Aff {
    float a, b;
};
// outer o inner (inner applied first)
__device__ __forceinline__ Aff compose(Aff outer, Aff inner) {
    return {outer.a + inner.a, lse2(outer.a + inner.b, outer.b)};
}
__device__ __forceinline__ Aff shfl_up(Aff v, int d) {
    return {__shfl_up_sync(kFull, v.a, d), __shfl_up_sync(kFull, v.b, d)};
}
__device__ __forceinline__ Aff shfl_down(Aff v, int d) {
    return {__shfl_down_sync(kFull, v.a, d), __shfl_down_sync(kFull, v.b, d)};
}
__device__ __forceinline__ Aff shfl_idx(Aff v, int l) {
    return {__shfl_sync(kFull, v.a, l), __shfl_sync(kFull, v.b, l)};
}

// ---------------------------------------------------------------- per-lane element loads
// For the K elements [s, s+K) of this lane (log2 units):
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
    if (s + K <= e0 || s >= e1) return;
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
    for (int j = 0; j < K; ++j) {
        const long long e = s + j;
        t[j] = (e >= e0 && e < e1) ? __ldg(T + v[j]) : 0;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const long long e = s + j;
        if (e >= e0 && e < e1) {
            // cavity (Eq.6): prior + every other incoming message, exact in fixed point
            const float c2 = fmaf(__ll2float_rn(t[j] - (long long)q[j]), kQInv * kLog2e, mp.L0_2);
            float fo = fmaf((float)o[j], mp.s_off, mp.b_off);
            fo = fminf(fmaxf(fo, 0.f), mp.fo_max);
            const int io = min((int)fo, mp.n_offm1 - 1);
            const float wo = fo - (float)io;
            const float2 ta = __ldg(rowA + io), tb = __ldg(rowB + io);
            const float ra = fmaf(wo, ta.y - ta.x, ta.x);
            const float rb = fmaf(wo, tb.y - tb.x, tb.x);
            const float lnu = fmaf(wz, rb - ra, ra);
            const float L1 = log1p2(ex2(-fabsf(c2)));
            la[j] = -(fmaxf(c2, 0.f) + L1);
            w[j] = lnu - (fmaxf(-c2, 0.f) + L1);
            l[j] = lnu;
        }
    }
}

// Lane composite of the suffix maps R -> 2^{la} R + 2^{w} over the chunk (first applied last):
// aB = sum la, bB = log2 sum_j 2^{w_j + sum_{k<j} la_k}.  The prefix maps
// Q -> 2^{-la} (Q + 2^{w}) compose to (-aB, bB - aB).
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
    for (int j = 0; j < K; ++j) sum += ex2(t[j] - m);
    aB = acc;
    bB = m + lg2(sum);
}

// Suffix scan over lanes: returns R entering this lane from the right given the carry Rc
// (log2 R after the tile); *carry_out = R leaving the tile on the left.
__device__ __forceinline__ float suffix_in(Aff G, int lane, float Rc, float* carry_out) {
    Aff H = G;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Aff o = shfl_down(H, d);
        if (lane + d < 32) H = compose(H, o);
    }
    Aff Hx = shfl_down(H, 1);
    if (lane == 31) Hx = {0.f, kNeg};
    if (carry_out) {
        const Aff H0 = shfl_idx(H, 0);
        *carry_out = lse2(H0.a + Rc, H0.b);
    }
    return lse2(Hx.a + Rc, Hx.b);
}

// Prefix scan over lanes: returns Q entering this lane from the left given carry Qc.
__device__ __forceinline__ float prefix_in(Aff F, int lane, float Qc, float* carry_out) {
    Aff P = F;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Aff o = shfl_up(P, d);
        if (lane >= d) P = compose(P, o);
    }
    Aff Px = shfl_up(P, 1);
    if (lane == 0) Px = {0.f, kNeg};
    if (carry_out) {
        const Aff P31 = shfl_idx(P, 31);
        *carry_out = lse2(P31.a + Qc, P31.b);
    }
    return lse2(Px.a + Qc, Px.b);
}

template <int K>
__device__ __forceinline__ void lane_suffix(const float (&la)[K], const float (&w)[K], float Rin, float (&lR)[K]) {
    float R = Rin;
#pragma unroll
    for (int j = K - 1; j >= 0; --j) {
        lR[j] = R;                      // log2 R_j: suffix strictly after element j
        R = lse2(la[j] + R, w[j]);      // R_{j-1} = mu(o_j=0) R_j + mu(o_j=1) nu_j
    }
}

// lambda2 = log2(2^Q + 2^l) - log2(2^Q + 2^R) without cancellation: the max parts subtract
// exactly (both are Q when Q dominates) and the remainders are small, accurate log1p terms.
__device__ __forceinline__ float lambda2(float Q, float l, float R) {
    const float m1 = fmaxf(Q, l), m2 = fmaxf(Q, R);
    return (m1 - m2) + (log1p2(ex2(-fabsf(Q - l))) - log1p2(ex2(-fabsf(Q - R))));
}

__device__ __forceinline__ int32_t quantise(float lam2) {
    float lam = lam2 * kLn2;
    lam = fminf(fmaxf(lam, -kLambdaClip), kLambdaClip);
    return __float2int_rn(lam * kQScale);  // saturates at +2^31-1 for +256
}

template <int K>
__device__ __forceinline__ void lane_prefix_out(const float (&la)[K], const float (&w)[K], const float (&l)[K],
                                                const float (&lR)[K], float Qin, long long s, long long e0,
                                                long long e1, int32_t* lam) {
    float Q = Qin;
    int32_t out[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        // lambda_j = log(Q_j + nu_j) - log(Q_j + R_j)   (Eq.13 / Eq.14, both divided by V_j)
        out[j] = quantise(lambda2(Q, l[j], lR[j]));
        Q = lse2(Q, w[j]) - la[j];      // Q_{j+1} = (Q_j + mu(o_j=1) nu_j) / mu(o_j=0)
    }
    if (s >= e0 && s + K <= e1) {
#pragma unroll
        for (int j = 0; j < K; j += 4)
            *reinterpret_cast<int4*>(lam + s + j) = make_int4(out[j], out[j + 1], out[j + 2], out[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (s + j >= e0 && s + j < e1) lam[s + j] = out[j];
    }
}

// ---------------------------------------------------------------- K5: single-tile classes
template <int K>
__global__ void __launch_bounds__(256) ray_msg_kernel(long long n, const int32_t* __restrict__ rays,
                                                      const long long* __restrict__ row_ptr,
                                                      const RayInfo* __restrict__ ray_z,
                                                      const int32_t* __restrict__ vid,
                                                      const int16_t* __restrict__ off_q, int32_t* lam,
                                                      const long long* __restrict__ T, MsgParams mp) {
    const long long wi = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wi >= n) return;
    const int lane = threadIdx.x & 31;
    const int r = __ldg(rays + wi);
    const RayInfo rz = ray_z[r];
    const long long e0 = __ldg(row_ptr + r), e1 = e0 + rz.n;
    const float2* rowA = mp.lutp + (long long)rz.iz * mp.n_offm1;
    const float2* rowB = rowA + mp.n_offm1;
    const long long s = e0 + (long long)lane * K;
    float la[K], w[K], l[K], lR[K];
    load_elems<K>(s, e0, e1, rowA, rowB, rz.wz, mp, vid, off_q, lam, T, la, w, l);
    float aB, bB;
    lane_composite<K>(la, w, aB, bB);
    const float Rin = suffix_in({aB, bB}, lane, kNeg, nullptr);
    lane_suffix<K>(la, w, Rin, lR);
    const float Qin = prefix_in({-aB, bB - aB}, lane, kNeg, nullptr);
    lane_prefix_out<K>(la, w, l, lR, Qin, s, e0, e1, lam);
}

// ---------------------------------------------------------------- K5: long rays (tiled)
constexpr int kLongK = 8;
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
        const long long base = e0;
        const int n_tiles = (int)((e1 - base + kLongTile - 1) / kLongTile);
        float la[kLongK], w[kLongK], l[kLongK], lR[kLongK];
        float aB, bB;
        // pass 1: suffix values, tiles right to left
        float Rc = kNeg;
        for (int t = n_tiles - 1; t >= 0; --t) {
            const long long s = base + (long long)t * kLongTile + (long long)lane * kLongK;
            load_elems<kLongK>(s, e0, e1, rowA, rowB, rz.wz, mp, vid, off_q, lam, T, la, w, l);
            lane_composite<kLongK>(la, w, aB, bB);
            float carry;
            const float Rin = suffix_in({aB, bB}, lane, Rc, &carry);
            Rc = carry;
            lane_suffix<kLongK>(la, w, Rin, lR);
            float* dst = my_scratch + (long long)t * kLongTile + lane * kLongK;
#pragma unroll
            for (int j = 0; j < kLongK; j += 4)
                *reinterpret_cast<float4*>(dst + j) = make_float4(lR[j], lR[j + 1], lR[j + 2], lR[j + 3]);
        }
        // pass 2: prefix values and messages, tiles left to right
        float Qc = kNeg;
        for (int t = 0; t < n_tiles; ++t) {
            const long long s = base + (long long)t * kLongTile + (long long)lane * kLongK;
            load_elems<kLongK>(s, e0, e1, rowA, rowB, rz.wz, mp, vid, off_q, lam, T, la, w, l);
            lane_composite<kLongK>(la, w, aB, bB);
            const float* src = my_scratch + (long long)t * kLongTile + lane * kLongK;
#pragma unroll
            for (int j = 0; j < kLongK; j += 4) {
                const float4 a = *reinterpret_cast<const float4*>(src + j);
                lR[j] = a.x; lR[j + 1] = a.y; lR[j + 2] = a.z; lR[j + 3] = a.w;
            }
            float carry;
            const float Qin = prefix_in({-aB, bB - aB}, lane, Qc, &carry);
            Qc = carry;
            lane_prefix_out<kLongK>(la, w, l, lR, Qin, s, e0, e1, lam);
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

// ---------------------------------------------------------------- K8
__global__ void marginals_kernel(long long V, const long long* __restrict__ T, double L0, float* out) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    const double a = L0 + (double)T[v] * kQInvD;  // Eq.8: prior times all incoming messages
    out[v] = (float)(1.0 / (1.0 + exp(-a)));
}

__global__ void lambda_to_float_kernel(long long n, const int32_t* __restrict__ q, float* out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (float)((double)q[i] * kQInvD);
}

inline unsigned blocks_for(long long n, int b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

int class_capacity(int cls) { return cls < 3 ? 32 * (4 << cls) : 0x7fffffff; }

void launch_ray_messages(int cls, long long n_rays, const int32_t* rays, const long long* row_ptr,
                         const RayInfo* ray_z, const int32_t* vid, const int16_t* off_q, int32_t* lam,
                         const long long* T, const MsgParams& mp, float* scratch, long long scratch_per_warp,
                         int n_warps_long, cudaStream_t s) {
    if (n_rays == 0) return;
    const unsigned grid = blocks_for(n_rays * 32, 256);
    switch (cls) {
        case 0: ray_msg_kernel<4><<<grid, 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, vid, off_q, lam, T, mp); break;
        case 1: ray_msg_kernel<8><<<grid, 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, vid, off_q, lam, T, mp); break;
        case 2: ray_msg_kernel<16><<<grid, 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, vid, off_q, lam, T, mp); break;
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

void launch_marginals(long long V, const long long* T, double L0, float* out, cudaStream_t s) {
    marginals_kernel<<<blocks_for(V, 256), 256, 0, s>>>(V, T, L0, out);
}

void launch_lambda_to_float(long long n, const int32_t* q, float* out, cudaStream_t s) {
    if (n == 0) return;
    lambda_to_float_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, q, out);
}

}  // namespace mrf
