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
// quantity O(1) in the log domain.  Both recurrences are affine maps x -> e^a x + e^b, so
// 8-element chunks compose in closed form and the chunks of a ray are combined by scans (prefix
// for Q, suffix for R).  The inputs are in natural logs (the units of the input table); inside
// K5 every log-quantity is carried in base-2 units (MRF_K5_LOG2, below), and lambda leaves in
// nats: e^x as ex2.approx on the MUFU; ln(1+y) either as a relative-accurate polynomial on the FMA pipe
// (log1pn) or, where only absolute accuracy matters, as lg2.approx on the MUFU (MATH levels
// below); lambda without cancellation (lambda_n).
//
// log nu_i is interpolated from the LUT once per frame by the DDA fill (graph.cu, lut_log_nu)
// and read as one fp32 per incidence.
//
// Chunking: a lane (or, in the staged layout, a thread) owns a chunk of consecutive incidences of
// ONE ray, counted from the ray's start (ray segments start at multiples of 8 slots), and the
// chunk scans are Hillis-Steele on the ray-relative chunk index -- so every rounding depends only
// on the ray (and its length class), never on where (or on which rank) it is stored: beliefs are
// bit-identical for any rank count.  Masked elements are identity maps.  Two layouts of the same
// arithmetic:
//   * classes (default): G lanes per ray by length class, K incidences per lane, scans by warp
//     shuffles (ray_msg_kernel); the class kernels run concurrently on side streams;
//   * staged (MRF_K5=staged, an ablation): stages of consecutive short rays bulk-copied (TMA)
//     into shared memory, thread = 8-slot chunk, scans in shared memory (ray_msg_staged_kernel).
// Rays longer than kShortMax run the tiled warp kernel (ray_msg_long_kernel) in both.
#include <algorithm>

#include "internal.cuh"
#include "walk.cuh"

namespace mrf {
namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr float kNeg = -1e30f;  // log(0); finite so that NEG - NEG = 0 stays NaN-free

// MATH levels (template parameter M):
//   0  every ln(1+y) by the relative-accurate polynomial;
//   1  the recurrences and chunk scans by lg2.approx (they carry max(a, b), so absolute accuracy
//      ~1e-7 nats is all they need), the cavity softplus and lambda by the polynomial (default);
//   2  also the softplus by lg2.approx.
#ifndef MRF_K5_MATH
#define MRF_K5_MATH 1
#endif
#ifndef MRF_K5_I2F_SPLIT
#define MRF_K5_I2F_SPLIT 1  // 3.696 -> 3.680 ms per K5 iteration at frames30 (MUFU-class pipe relief)
#endif

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
// ln(1 + y) for y in [0, 1] with RELATIVE accuracy (~3e-7), on the FMA pipe: y * P(y), P a
// degree-7 fit of ln(1+y)/y (MRF_LOG1P_DEG7=0: degree 8, ~2e-7).  (lg2.approx(1+y) is only absolutely accurate near 1, which biased
// the tiny messages of occluded voxels.)
#ifndef MRF_LOG1P_DEG7
#define MRF_LOG1P_DEG7 1
#endif
// Working base of the K5 log domain.  MRF_K5_LOG2 = 1: every log-quantity of K5 (cavity, la, w,
// l, Q, R, lambda) is carried in base-2 units (x / ln 2), so e^x and ln(1+y) become bare ex2 / lg2
// -- no scaling multiply per MUFU op; the nats of the inputs (T, q, L0: exact integers and one
// constant; log nu) are converted where they enter (folded into existing FMAs, one multiply for
// l) and lambda is converted back to nats before quantisation.  0: natural-log units throughout.
constexpr float kWS = MRF_K5_LOG2 ? kLog2e : 1.f;  // nats -> working units
constexpr float kWInv = MRF_K5_LOG2 ? kLn2 : 1.f;  // working units -> nats
__device__ __forceinline__ float log1pn(float y) {
#if MRF_LOG1P_DEG7
    // degree 7 (relative error 3.3e-7 evaluated in fp32; the degree-8 fit below: 1.6e-7)
    float r = (-0.00853875931f * kWS);
    r = fmaf(r, y, (0.0440874845f * kWS));
    r = fmaf(r, y, (-0.10767781f * kWS));
    r = fmaf(r, y, (0.177448928f * kWS));
    r = fmaf(r, y, (-0.244953007f * kWS));
    r = fmaf(r, y, (0.332754433f * kWS));
    r = fmaf(r, y, (-0.499974012f * kWS));
    r = fmaf(r, y, (0.999999821f * kWS));
    return r * y;
#else
    float r = (0.00523269456f * kWS);
    r = fmaf(r, y, (-0.0295052417f * kWS));
    r = fmaf(r, y, (0.0782259554f * kWS));
    r = fmaf(r, y, (-0.136632457f * kWS));
    r = fmaf(r, y, (0.191060066f * kWS));
    r = fmaf(r, y, (-0.24842982f * kWS));
    r = fmaf(r, y, (0.333190978f * kWS));
    r = fmaf(r, y, (-0.499994934f * kWS));
    r = fmaf(r, y, (0.99999994f * kWS));
    return r * y;
#endif
}
// ln(1 + y), y in [0, 1], absolutely accurate (~1e-7) on the MUFU (working units)
__device__ __forceinline__ float log1pf_abs(float y) { return MRF_K5_LOG2 ? lg2(1.f + y) : kLn2 * lg2(1.f + y); }
// e^x on the MUFU (ex2.approx, relative error ~2^-22), x in working units
__device__ __forceinline__ float expn(float x) { return MRF_K5_LOG2 ? ex2(x) : ex2(x * kLog2e); }
// ln(e^a + e^b) = max + ln(1 + e^-|a-b|)
template <bool ABS>
__device__ __forceinline__ float lse(float a, float b) {
    const float y = expn(-fabsf(a - b));
    return fmaxf(a, b) + (ABS ? log1pf_abs(y) : log1pn(y));
}

// Affine map x -> e^a x + e^b in log form (nats).
struct Aff {
    float a, b;
};
// outer o inner (inner applied first)
template <int M>
__device__ __forceinline__ Aff compose(Aff outer, Aff inner) {
    return {outer.a + inner.a, lse<(M >= 1)>(outer.a + inner.b, outer.b)};
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

// ---------------------------------------------------------------- per-element terms
// From the gathered belief sum t = sum of q over the voxel, this incidence's own q and its
// log nu (nats):  la = log mu(o=0) = -softplus(c),  w = log mu(o=1) + log nu,  l = log nu, with
// the cavity c = L0 + (t - q) 2^-23 (Eq.6) formed exactly in integers.  la and log mu(o=1)
// share one ex2 and are both computed directly, never as a difference of two large numbers.
// Masked elements (ok = false) are identity maps: la = 0, w = l = NEG.
// select without a branch (ptxas otherwise turns "ok ? expensive : constant" into a divergent
// branch around the whole softplus, which also serialises the elements' instruction streams)
__device__ __forceinline__ float selp(bool p, float a, float b) {
    float r;
    asm("{\n.reg .pred q;\nsetp.ne.u32 q, %3, 0;\nselp.f32 %0, %1, %2, q;\n}" : "=f"(r) : "f"(a), "f"(b), "r"((unsigned)p));
    return r;
}
// MASK_ALL = false (the class kernels, whose lane scans carry only b parts): only w is masked.
// An element past the ray's end then keeps its la and l, which are harmless there: it lies after
// every element of the ray, so its la only scales suffix values that are log 0 (R beyond the ray),
// enters its own lane's a part (unused without carries) and the prefix maps of lanes past the ray,
// and its l only its own (discarded) output -- while w = log 0 keeps it out of every sum.
template <int M, bool MASK_ALL = true>
__device__ __forceinline__ void elem_terms(long long t, int q, float lnu, float L0, bool ok, float& la, float& w,
                                           float& l) {
#if MRF_K5_I2F_SPLIT
    // x = hi 2^24 + lo with both parts exact in fp32 (32-bit conversions run on the ALU pipe;
    // the 64-bit I2F is a MUFU-class op)
    const long long x = t - (long long)q;
    const float c = fmaf(__int2float_rn((int)(x >> 24)), 2.f * kWS,
                         fmaf(__int2float_rn((int)(x & 0xffffff)), kQInv * kWS, L0 * kWS));
#else
    const float c = fmaf(__ll2float_rn(t - (long long)q), kQInv * kWS, L0 * kWS);
#endif
    const float y = expn(-fabsf(c));
    const float L1 = M >= 2 ? log1pf_abs(y) : log1pn(y);  // ln(1 + e^-|c|)
    // lnu arrives in working units (the fill stores log nu * kLnuScale, internal.cuh)
    if constexpr (MASK_ALL) {
        la = selp(ok, -(fmaxf(c, 0.f) + L1), 0.f);
        l = selp(ok, lnu, kNeg);
    } else {
        la = -(fmaxf(c, 0.f) + L1);
        l = lnu;
    }
    w = selp(ok, lnu - (fmaxf(-c, 0.f) + L1), kNeg);
}

// Chunk composite of the suffix maps R -> e^{la} R + e^{w} (first applied last):
// aB = sum la, bB = ln sum_j e^{w_j + sum_{k<j} la_k}.  The prefix maps Q -> e^{-la} (Q + e^{w})
// compose to (-aB, bB - aB).
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
    bB = m + (MRF_K5_LOG2 ? lg2(sum) : lg2(sum) * kLn2);
}

// Both lane scans of a ray's G lanes at once (two independent shuffle chains per level):
// returns R entering this lane from the right and Q entering it from the left, given the tile
// carries Rc (R after the tile) and Qc (Q before it); optional carries out.
// CARRY = false (class kernels: no carries, Rc = Qc = log 0): R and Q entering a lane are just
// the b parts of its neighbours' composites -- lse(a + log 0, b) = b exactly -- which saves two
// log-sum-exps (4 MUFU ops) and two shuffles per lane.
template <int G, int M, bool CARRY = true>
__device__ __forceinline__ void lane_scans(float aB, float bB, int sl, float Rc, float Qc, float& Rin, float& Qin,
                                           float* Rc_out, float* Qc_out) {
    Aff H = {aB, bB};        // suffix maps R -> e^{la} R + e^{w}
    Aff P = {-aB, bB - aB};  // prefix maps Q -> e^{-la} (Q + e^{w})
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        // partners outside the ray's lanes are identity maps (0, NEG): composing with them is
        // exact (the remainder e^-huge vanishes), so no branch is needed
        Aff oh = shfl_down<G>(H, d);
        Aff op = shfl_up<G>(P, d);
        if (sl + d >= G) oh = Aff{0.f, kNeg};
        if (sl < d) op = Aff{0.f, kNeg};
        H = compose<M>(H, oh);
        P = compose<M>(P, op);
    }
    if constexpr (!CARRY) {
        const float hb = __shfl_down_sync(kFull, H.b, 1, G), pb = __shfl_up_sync(kFull, P.b, 1, G);
        Rin = sl == G - 1 ? kNeg : hb;
        Qin = sl == 0 ? kNeg : pb;
        return;
    }
    Aff Hx = shfl_down<G>(H, 1);
    Aff Px = shfl_up<G>(P, 1);
    if (sl == G - 1) Hx = {0.f, kNeg};
    if (sl == 0) Px = {0.f, kNeg};
    if (Rc_out) {
        const Aff H0 = shfl_idx<G>(H, 0);
        const Aff Pl = shfl_idx<G>(P, G - 1);
        *Rc_out = lse<(M >= 1)>(H0.a + Rc, H0.b);
        *Qc_out = lse<(M >= 1)>(Pl.a + Qc, Pl.b);
    }
    Rin = lse<(M >= 1)>(Hx.a + Rc, Hx.b);
    Qin = lse<(M >= 1)>(Px.a + Qc, Px.b);
}

// The two per-chunk recurrences, interleaved (independent chains):
//   lR[j] = ln R_j (suffix strictly after j),  R_{j-1} = mu(o_j=0) R_j + mu(o_j=1) nu_j
//   lQ[j] = ln Q_j (prefix strictly before j), Q_{j+1} = (Q_j + mu(o_j=1) nu_j) / mu(o_j=0)
template <int K, int M>
__device__ __forceinline__ void lane_recurrences(const float (&la)[K], const float (&w)[K], float Rin, float Qin,
                                                 float (&lR)[K], float (&lQ)[K]) {
    float R = Rin, Q = Qin;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        const int jb = K - 1 - i;
        lR[jb] = R;
        lQ[i] = Q;
        R = lse<(M >= 1)>(la[jb] + R, w[jb]);
        Q = lse<(M >= 1)>(Q, w[i]) - la[i];
    }
}

// lambda = ln(e^Q + e^l) - ln(e^Q + e^R) without cancellation: the max parts subtract exactly
// (both are Q when Q dominates) and the remainders are small, relative-accurate log1p terms.
// MRF_K5_ATANH = 1: the two remainders as ONE term, ln((1 + y1) / (1 + y2)) = 2 atanh(s) with
// s = (y1 - y2) / (2 + y1 + y2), |s| <= 1/3, by its odd series through s^13 (relative 1.4e-8):
// one reciprocal on the MUFU instead of a second degree-7 polynomial on the FMA pipe (frames30 K5
// 3.271 -> 3.244 ms per iteration; 0: the two polynomials).
#ifndef MRF_K5_ATANH
#define MRF_K5_ATANH 1
#endif
__device__ __forceinline__ float lambda_n(float Q, float l, float R) {
    const float m1 = fmaxf(Q, l), m2 = fmaxf(Q, R);
#if MRF_K5_ATANH
    const float y1 = expn(-fabsf(Q - l)), y2 = expn(-fabsf(Q - R));
    float rc;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"((y1 + 2.f) + y2));
    const float sv = (y1 - y2) * rc, z = sv * sv;
    float p = (2.f / 13.f) * kWS;
    p = fmaf(p, z, (2.f / 11.f) * kWS);
    p = fmaf(p, z, (2.f / 9.f) * kWS);
    p = fmaf(p, z, (2.f / 7.f) * kWS);
    p = fmaf(p, z, (2.f / 5.f) * kWS);
    p = fmaf(p, z, (2.f / 3.f) * kWS);
    p = fmaf(p, z, 2.f * kWS);
    return (m1 - m2) + sv * p;
#else
    return (m1 - m2) + (log1pn(expn(-fabsf(Q - l))) - log1pn(expn(-fabsf(Q - R))));
#endif
}

__device__ __forceinline__ int32_t quantise(float lam) {  // lam in working units -> round(clip(nats) 2^23)
    constexpr float kS = kWInv * kQScale, kC = kLambdaClip * kQScale;
    return __float2int_rn(fminf(fmaxf(lam * kS, -kC), kC));  // saturates at +2^31-1 for +256
}

// ---------------------------------------------------------------- K5: class kernels
// Lane chunks of K incidences start at multiples of K slots from an 8-aligned ray start, so they
// are read / written with the widest vector that K allows (16 bytes for K = 8, 8 for K = 6).
template <int K>
struct VecW {
    static constexpr int value = (K % 4 == 0) ? 4 : ((K % 2 == 0) ? 2 : 1);
};
template <int K>
__device__ __forceinline__ void ldk(const int32_t* __restrict__ p, int (&o)[K]) {
    constexpr int W = VecW<K>::value;
#pragma unroll
    for (int j = 0; j < K; j += W) {
        if constexpr (W == 4) {
            const int4 a = __ldg(reinterpret_cast<const int4*>(p + j));
            o[j] = a.x; o[j + 1] = a.y; o[j + 2] = a.z; o[j + 3] = a.w;
        } else if constexpr (W == 2) {
            const int2 a = __ldg(reinterpret_cast<const int2*>(p + j));
            o[j] = a.x; o[j + 1] = a.y;
        } else {
            o[j] = __ldg(p + j);
        }
    }
}
// store the first nv of K values (all K when the chunk is complete, with vector stores)
template <int K>
__device__ __forceinline__ void stk(int32_t* p, const int (&v)[K], long long nv) {
    constexpr int W = VecW<K>::value;
    if (nv >= K) {
#pragma unroll
        for (int j = 0; j < K; j += W) {
            if constexpr (W == 4) {
                *reinterpret_cast<int4*>(p + j) = make_int4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else if constexpr (W == 2) {
                *reinterpret_cast<int2*>(p + j) = make_int2(v[j], v[j + 1]);
            } else {
                p[j] = v[j];
            }
        }
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (j < nv) p[j] = v[j];
    }
}

// Loads of one lane's chunk [s, s+K) (s < e1): vid, q, log nu, then the belief gathers.
template <int K, int M>
__device__ __forceinline__ void load_chunk(long long s, long long e1, const MsgParams& mp, const int32_t* __restrict__ vid,
                                           const float* __restrict__ lnu, const int32_t* __restrict__ lam,
                                           const long long* __restrict__ T, const int32_t* __restrict__ qrow,
                                           float (&la)[K], float (&w)[K], float (&l)[K]) {
    int v[K], q[K], ln[K];
    ldk<K>(vid + s, v);
    if (qrow) {  // keyframe-average mode: the ray's keyframe average replaces its own message
#pragma unroll
        for (int j = 0; j < K; ++j) q[j] = __ldg(qrow + v[j]);
    } else {
        ldk<K>(lam + s, q);
    }
    ldk<K>(reinterpret_cast<const int32_t*>(lnu) + s, ln);
    long long t[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        MRF_ASSERT(s + j >= e1 || (v[j] >= 0 && v[j] < mp.chk_vi && (qrow || s + j < mp.chk_lam)));
        t[j] = (s + j < e1) ? __ldg(T + v[j]) : 0;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) elem_terms<M>(t[j], q[j], __int_as_float(ln[j]), mp.L0, s + j < e1, la[j], w[j], l[j]);
}
template <int K>
__device__ __forceinline__ void identity_chunk(float (&la)[K], float (&w)[K], float (&l)[K]) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
        la[j] = 0.f;
        w[j] = kNeg;
        l[j] = kNeg;
    }
}

// lambda_j = log(Q_j + nu_j) - log(Q_j + R_j)   (Eq.13 / Eq.14, both divided by V_j)
template <int K>
__device__ __forceinline__ void lane_out(const float (&l)[K], const float (&lR)[K], const float (&lQ)[K], long long s,
                                         long long e1, int32_t* lam) {
    int out[K];
#pragma unroll
    for (int j = 0; j < K; ++j) out[j] = s + j < e1 ? quantise(lambda_n(lQ[j], l[j], lR[j])) : 0;
    stk<K>(lam + s, out, e1 - s);
}

// G lanes per ray (32/G rays per warp), K incidences per lane: capacity G*K.  Incidence indices
// are 32-bit (a ctx holds < 2^31 slots), and the per-element masks are selects on the lane's
// valid count nv, so the only divergence is a lane without a chunk skipping its loads.
// Resident CTAs of 256 threads per SM: K <= 8 classes fit 40 registers without spills, so 6 CTAs
// (48 warps; frames30 K5 3.418 -> 3.366 ms per iteration against 4 CTAs); K <= 6 fit 32: 7 CTAs
// (-> 3.281 ms); K > 8: 2 CTAs.  The matrix-free walk kernels carry the walker too: 5 CTAs
// (<= 51 registers; 4: 98.1, 5: 96.8 ms of K5 per 10 iterations).
#ifndef MRF_K5_MIN_BLOCKS
#define MRF_K5_MIN_BLOCKS 6
#endif
#ifndef MRF_K5_MIN_BLOCKS_SMALL
#define MRF_K5_MIN_BLOCKS_SMALL 7
#endif
#ifndef MRF_K5_WALK_MIN_BLOCKS
#define MRF_K5_WALK_MIN_BLOCKS 5
#endif
#ifndef MRF_K5_MASK_ALL
#define MRF_K5_MASK_ALL 0
#endif
template <int G, int K, int M, bool AVG>
__global__ void __launch_bounds__(256, (K > 8 ? 2 : (K > 6 ? MRF_K5_MIN_BLOCKS : MRF_K5_MIN_BLOCKS_SMALL))) ray_msg_kernel(long long n, const int4* __restrict__ desc,
                                                         const int32_t* __restrict__ vid,
                                                         const float* __restrict__ lnu, int32_t* lam,
                                                         const long long* __restrict__ T, MsgParams mp) {
    constexpr int RPW = 32 / G;
    const long long wi = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wi * RPW >= n) return;  // warp-uniform
    const int lane = threadIdx.x & 31, sl = lane & (G - 1);
    const long long ri = wi * RPW + lane / G;
    // lanes past the end of the list take its last ray with no incidences of their own: their
    // (masked) loads stay inside the incidence range the list covers -- which, in the
    // matrix-free mode, is a scratch holding only the current chunk's slots
    int nr = 0, e0 = 0, fr = 0;
    {
        // {row_ptr[r], n, frame, r} of the class list's ray (launch_class_desc): one load, where
        // the ray id, then its record and row pointer were two dependent ones
        const int4 d = __ldg(desc + (ri < n ? ri : n - 1));
        if (ri < n) nr = d.y;
        e0 = d.x;
        if constexpr (AVG) fr = d.z;
    }
    const int s = e0 + sl * K;
    const int nv = min(max(nr - sl * K, 0), K);  // valid incidences of this lane's chunk
    // lanes past the ray's end re-read the ray's first chunk (in bounds) and mask everything
    const int sr = nv > 0 ? s : e0;
    float la[K], w[K], l[K], lR[K], lQ[K];
    {
        int v[K], q[K], ln[K];
        ldk<K>(vid + sr, v);
        if constexpr (AVG) {  // keyframe-average mode: the cavity excludes the ray's keyframe average
            const int32_t* qrow = mp.qbar + (long long)fr * mp.qbar_vi;
#pragma unroll
            for (int j = 0; j < K; ++j) q[j] = __ldg(qrow + v[j]);
        } else {
            ldk<K>(lam + sr, q);
        }
        ldk<K>(reinterpret_cast<const int32_t*>(lnu) + sr, ln);
        // every slot of a chunk holds a valid voxel id (padding slots hold 0), so the gathers
        // and the element terms run unpredicated (straight-line code, full ILP) and are masked
        // by select afterwards
        long long t[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            MRF_ASSERT(v[j] >= 0 && v[j] < mp.chk_vi);
            t[j] = __ldg(T + v[j]);
        }
#pragma unroll
        for (int j = 0; j < K; ++j)
            elem_terms<M, MRF_K5_MASK_ALL>(t[j], q[j], __int_as_float(ln[j]), mp.L0, j < nv, la[j], w[j], l[j]);
    }
    MRF_ASSERT(!AVG && nv > 0 ? (long long)s + nv <= mp.chk_lam : true);
    float aB, bB, Rin, Qin;
    lane_composite<K>(la, w, aB, bB);
    lane_scans<G, M, false>(aB, bB, sl, kNeg, kNeg, Rin, Qin, nullptr, nullptr);
    lane_recurrences<K, M>(la, w, Rin, Qin, lR, lQ);
    int out[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int x = quantise(lambda_n(lQ[j], l[j], lR[j]));
        out[j] = j < nv ? x : 0;
    }
    stk<K>(lam + s, out, nv);
}

// ---------------------------------------------------------------- K5 matrix-free (K12)
// The paper re-traces every keyframe in every pass.  Here a lane re-walks ITS chunk of
// the ray inside the message kernel: the chunk's first cell is stored (ck: 4 bytes per chunk, one
// per K incidences, written by the first walk), the walker's exact state in that cell follows from
// the cell and the ray's segment (Walker::restart), and K steps of the same integer DDA give the
// chunk's voxel slots and offsets; log nu is interpolated from the table (L1) as the fill does.
// No vid / off_q / log-nu array exists: per iteration K5 moves lambda (read + write), the
// checkpoints and the per-ray records.  Bit-identical to the stored graph (same walk, same
// interpolation, same message arithmetic).
constexpr int kNoIncidence = 1 << 20;  // walk_chunk: a slot past the ray's end (offsets are int16)
template <int K>
__device__ __forceinline__ void walk_chunk(const WalkParams& wp, const RaySeg& sg, const MsgParams& mp, int iz, float wz,
                                           int vck, bool first, int nv, int (&v)[K], int (&ln)[K]) {
    int x, y, z;
    slot_xyz(wp.g, vck, x, y, z);
    Walker w;
    w.restart(sg, x, y, z, first);
#pragma unroll
    for (int j = 0; j < K; ++j) {
        unsigned na, da;
        const int a = w.earliest(na, da);
        bool last;
        const double t_out = crossing_t(w, a, na, da, last);
        const bool ok = j < nv;
        // cells past the ray's end may lie outside the grid: slot 0 (masked afterwards)
        v[j] = ok ? voxel_slot(wp.g, w.c0, w.c1, w.c2) : 0;
        const double mid = __dmul_rn(__dmul_rn(0.5, __dadd_rn(w.t_in, t_out)), sg.L);
        long long q = __double2ll_rn(__dmul_rn(__dsub_rn(mid, sg.Z), 32768.0));
        q = q > 32767 ? 32767 : (q < -32767 ? -32767 : q);
        ln[j] = ok ? (int)q : kNoIncidence;  // log nu after the walk (table loads back to back)
        w.advance(na, da);
        w.t_in = t_out;
        // sparse bricks (g.bmask set): the next emitted cell lies past any unallocated brick, reached
        // by the same one-step empty skip as the first walk (bit-identical); dense: no iteration
        if (j + 1 < nv)
            while (!cell_in_map(wp.g, w.c0, w.c1, w.c2))
                if (!w.skip_brick(wp.g) || !w.inside(wp.g)) break;
    }
    if (mp.pcoef) {  // per-patch noise (R25): iz = the ray's patch, wz = its range
#pragma unroll
        for (int j = 0; j < K; ++j)
            ln[j] = __float_as_int(ln[j] != kNoIncidence ? patch_lnu(mp, iz, wz, ln[j]) : 0.f);
    } else {
#pragma unroll
        for (int j = 0; j < K; ++j)
            ln[j] = __float_as_int(ln[j] != kNoIncidence ? lut_finish(lut_fetch(mp, iz, ln[j]), wz) : 0.f);
    }
}

// the long-ray kernel's chunk [s, s + K) (s < e1), re-walked: chunk index (s - e0) / K of the ray
template <int K, int M>
__device__ __forceinline__ void load_chunk_walk(long long s, long long e0, long long e1, const MsgParams& mp,
                                                const WalkParams& wp, const RaySeg& sg, const RayInfo& info,
                                                const int32_t* __restrict__ lam, const long long* __restrict__ T,
                                                const int32_t* __restrict__ qrow, float (&la)[K], float (&w)[K],
                                                float (&l)[K]) {
    const int c = (int)((s - e0) / K);
    const int nv = (int)min((long long)K, e1 - s);
    int v[K], q[K], ln[K];
    walk_chunk<K>(wp, sg, mp, info.iz, info.wz, __ldg(wp.ck + (e0 >> 2) + c), false, nv, v, ln);
    if (qrow) {
#pragma unroll
        for (int j = 0; j < K; ++j) q[j] = __ldg(qrow + v[j]);
    } else {
        ldk<K>(lam + s, q);
    }
    long long t[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        MRF_ASSERT(j >= nv || (v[j] >= 0 && v[j] < mp.chk_vi && (qrow || s + j < mp.chk_lam)));
        t[j] = __ldg(T + v[j]);
    }
#pragma unroll
    for (int j = 0; j < K; ++j) elem_terms<M>(t[j], q[j], __int_as_float(ln[j]), mp.L0, j < nv, la[j], w[j], l[j]);
}

template <int G, int K, int M, bool AVG>
__global__ void __launch_bounds__(256, (K > 8 ? 2 : MRF_K5_WALK_MIN_BLOCKS)) ray_msg_walk_kernel(long long n, const int32_t* __restrict__ rays,
                                                         const long long* __restrict__ row_ptr,
                                                         const RayInfo* __restrict__ ray_z, int32_t* lam,
                                                         const long long* __restrict__ T, MsgParams mp, WalkParams wp) {
    constexpr int RPW = 32 / G;
    const long long wi = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wi * RPW >= n) return;  // warp-uniform
    const int lane = threadIdx.x & 31, sl = lane & (G - 1);
    const long long ri = wi * RPW + lane / G;
    const int r = __ldg(rays + (ri < n ? ri : n - 1));
    const RayInfo info = ray_z[r];
    const int nr = ri < n ? info.n : 0;
    const int e0 = (int)__ldg(row_ptr + r);
    const int s = e0 + sl * K;
    const int nv = min(max(nr - sl * K, 0), K);
    const int sr = nv > 0 ? s : e0;
    float la[K], w[K], l[K], lR[K], lQ[K];
    {
        int v[K], q[K], ln[K];
        const RaySeg sg = wp.seg[r];
        const int vck = __ldg(wp.ck + (e0 >> 2) + (nv > 0 ? sl : 0));
        walk_chunk<K>(wp, sg, mp, info.iz, info.wz, vck, false, nv, v, ln);  // (t_in of a ray's first cell: 0 by restart)
        if constexpr (AVG) {
            const int32_t* qrow = mp.qbar + (long long)info.frame * mp.qbar_vi;
#pragma unroll
            for (int j = 0; j < K; ++j) q[j] = __ldg(qrow + v[j]);
        } else {
            ldk<K>(lam + sr, q);
        }
        long long t[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            MRF_ASSERT(v[j] >= 0 && v[j] < mp.chk_vi);
            t[j] = __ldg(T + v[j]);
        }
#pragma unroll
        for (int j = 0; j < K; ++j)
            elem_terms<M, MRF_K5_MASK_ALL>(t[j], q[j], __int_as_float(ln[j]), mp.L0, j < nv, la[j], w[j], l[j]);
    }
    MRF_ASSERT(!AVG && nv > 0 ? (long long)s + nv <= mp.chk_lam : true);
    float aB, bB, Rin, Qin;
    lane_composite<K>(la, w, aB, bB);
    lane_scans<G, M, false>(aB, bB, sl, kNeg, kNeg, Rin, Qin, nullptr, nullptr);
    lane_recurrences<K, M>(la, w, Rin, Qin, lR, lQ);
    int out[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int x = quantise(lambda_n(lQ[j], l[j], lR[j]));
        out[j] = j < nv ? x : 0;
    }
    stk<K>(lam + s, out, nv);
}

// ---------------------------------------------------------------- K5: long rays (tiled)
constexpr int kLongK = 8;
constexpr int kLongTile = 32 * kLongK;

template <int M, bool AVG, bool WALK>
__global__ void __launch_bounds__(256) ray_msg_long_kernel(long long n, const int32_t* __restrict__ rays,
                                                           const long long* __restrict__ row_ptr,
                                                           const RayInfo* __restrict__ ray_z,
                                                           const int32_t* __restrict__ vid,
                                                           const float* __restrict__ lnu, int32_t* lam,
                                                           const long long* __restrict__ T, MsgParams mp,
                                                           float* scratch, long long scratch_per_warp, WalkParams wp) {
    const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long n_warps = ((long long)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    float* my_scratch = scratch + gw * scratch_per_warp;
    for (long long wi = gw; wi < n; wi += n_warps) {
        const int r = __ldg(rays + wi);
        const long long e0 = __ldg(row_ptr + r), e1 = e0 + ray_z[r].n;
        const int32_t* qrow = AVG ? mp.qbar + (long long)ray_z[r].frame * mp.qbar_vi : nullptr;
        const RayInfo info = ray_z[r];
        RaySeg sg{};
        if constexpr (WALK) sg = wp.seg[r];
        const int n_tiles = (int)((e1 - e0 + kLongTile - 1) / kLongTile);
        float la[kLongK], w[kLongK], l[kLongK], lR[kLongK], lQ[kLongK];
        float aB, bB, Rin, Qin, Rc_out, Qc_out;
        // pass 1: suffix values, tiles right to left
        float Rc = kNeg;
        for (int t = n_tiles - 1; t >= 0; --t) {
            const long long s = e0 + (long long)t * kLongTile + (long long)lane * kLongK;
            identity_chunk<kLongK>(la, w, l);
            if (s < e1) {
                if constexpr (WALK) load_chunk_walk<kLongK, M>(s, e0, e1, mp, wp, sg, info, lam, T, qrow, la, w, l);
                else load_chunk<kLongK, M>(s, e1, mp, vid, lnu, lam, T, qrow, la, w, l);
            }
            lane_composite<kLongK>(la, w, aB, bB);
            lane_scans<32, M>(aB, bB, lane, Rc, kNeg, Rin, Qin, &Rc_out, &Qc_out);
            Rc = Rc_out;
            lane_recurrences<kLongK, M>(la, w, Rin, kNeg, lR, lQ);
            float* dst = my_scratch + (long long)t * kLongTile + lane * kLongK;
#pragma unroll
            for (int j = 0; j < kLongK; j += 4)
                *reinterpret_cast<float4*>(dst + j) = make_float4(lR[j], lR[j + 1], lR[j + 2], lR[j + 3]);
        }
        // pass 2: prefix values and messages, tiles left to right
        float Qc = kNeg;
        for (int t = 0; t < n_tiles; ++t) {
            const long long s = e0 + (long long)t * kLongTile + (long long)lane * kLongK;
            identity_chunk<kLongK>(la, w, l);
            if (s < e1) {
                if constexpr (WALK) load_chunk_walk<kLongK, M>(s, e0, e1, mp, wp, sg, info, lam, T, qrow, la, w, l);
                else load_chunk<kLongK, M>(s, e1, mp, vid, lnu, lam, T, qrow, la, w, l);
            }
            lane_composite<kLongK>(la, w, aB, bB);
            lane_scans<32, M>(aB, bB, lane, kNeg, Qc, Rin, Qin, &Rc_out, &Qc_out);
            Qc = Qc_out;
            lane_recurrences<kLongK, M>(la, w, kNeg, Qin, lR, lQ);
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

// ---------------------------------------------------------------- K5: staged (TMA bulk copies)
// A persistent CTA (kStageThreads threads) walks its stages; thread 0 bulk-copies the NEXT
// stage's vid / lambda / log-nu slots, its row_ptr entries and its RayInfo records into the
// other shared-memory buffer (cp.async.bulk, completion on an mbarrier) while the CTA computes
// the current one, so the incidence stream reaches HBM as a few large asynchronous copies per
// stage instead of per-warp dependent loads.  Thread t owns the 8 slots [s0 + 8t, s0 + 8t + 8) =
// chunk c of one ray.  Per chunk: the 8 elements' maps in closed form (lane_composite); then,
// per ray, inclusive scans over its chunks in shared memory, Hillis-Steele on the RAY-RELATIVE
// chunk index (chunk c combines with c - d iff c >= d) -- the same association tree as the class
// kernels' lane scans, so both layouts give bit-identical messages; then the two recurrences
// and lambda.
constexpr int kStSlots = kStageCap + kShortMax;                   // >= span of any stage (8-aligned)
constexpr int kStChunks = kStSlots / kSegAlign;                   // = kStageThreads
constexpr int kStRp = kStageMaxRays + 2;                          // row_ptr entries [r0&~1, (r1+2)&~1)
constexpr int kOffVid = 0;
constexpr int kOffLam = kOffVid + 4 * kStSlots;
constexpr int kOffLnu = kOffLam + 4 * kStSlots;
constexpr int kOffRp = kOffLnu + 4 * kStSlots;
constexpr int kOffRi = kOffRp + 8 * kStRp;
constexpr int kOffCm = kOffRi + 16 * kStageMaxRays;               // chunk -> ray (uint16)
constexpr int kBufBytes = (kOffCm + 2 * kStChunks + 127) & ~127;
constexpr int kOffScan = 2 * kBufBytes;                           // [2 ping-pong][kStChunks] x (P, H) float4
constexpr int kOffBar = kOffScan + 2 * kStChunks * 16;
constexpr int kStageSmem = kOffBar + 128;
static_assert(kStChunks == kStageThreads, "one 8-slot chunk per thread");
static_assert(kOffRp % 16 == 0 && kOffRi % 16 == 0 && kOffLam % 16 == 0 && kOffLnu % 16 == 0, "16-byte aligned");

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MRF_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra MRF_WAIT_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// Thread 0: start the copies of stage `st` into `buf`, completion on `bar`.  All sources and
// sizes are 16-byte multiples (segments 8-aligned, row_ptr read from an even index).
__device__ __forceinline__ void stage_issue(const Stage& st, char* buf, unsigned long long* bar,
                                            const long long* row_ptr, const RayInfo* info, const int32_t* vid,
                                            const float* lnu, const int32_t* lam) {
    const unsigned ns = (unsigned)(st.s1 - st.s0);
    const int a0 = st.r0 & ~1, a1 = (st.r1 + 2) & ~1;
    const unsigned nrp = (unsigned)(a1 - a0), nri = (unsigned)(st.r1 - st.r0);
    // generic-proxy reads of this buffer (previous stage) are ordered before the async writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, ns * 12u + nrp * 8u + nri * 16u);
    if (ns) {
        bulk_g2s(buf + kOffVid, vid + st.s0, ns * 4u, bar);
        bulk_g2s(buf + kOffLam, lam + st.s0, ns * 4u, bar);
        bulk_g2s(buf + kOffLnu, lnu + st.s0, ns * 4u, bar);
    }
    bulk_g2s(buf + kOffRp, row_ptr + a0, nrp * 8u, bar);
    bulk_g2s(buf + kOffRi, info + st.r0, nri * 16u, bar);
}

template <int M>
__global__ void __launch_bounds__(kStageThreads, kStageCtas)
    ray_msg_staged_kernel(long long n_stages, const Stage* __restrict__ stages, const long long* __restrict__ row_ptr,
                          const RayInfo* __restrict__ info, const int32_t* __restrict__ vid,
                          const float* __restrict__ lnu, int32_t* lam, const long long* __restrict__ T,
                          MsgParams mp) {
    extern __shared__ __align__(128) char st_smem[];
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(st_smem + kOffBar);
    Stage* sd = reinterpret_cast<Stage*>(st_smem + kOffBar + 16);   // descriptors of the two buffers
    int* s_maxc = reinterpret_cast<int*>(st_smem + kOffBar + 80);  // per buffer: longest ray, in chunks
    float4* scan = reinterpret_cast<float4*>(st_smem + kOffScan);  // [2][kStChunks]: (P.a, P.b, H.a, H.b)
    const int t = threadIdx.x;
    long long k = blockIdx.x;
    if (k >= n_stages) return;
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        sd[0] = stages[k];
        s_maxc[0] = 1;
        stage_issue(sd[0], st_smem, &bars[0], row_ptr, info, vid, lnu, lam);
    }
    Stage nxt{};
    if (t == 0 && k + gridDim.x < n_stages) nxt = stages[k + gridDim.x];
    __syncthreads();
    for (int i = 0; k < n_stages; ++i, k += gridDim.x) {
        const int b = i & 1;
        char* buf = st_smem + b * kBufBytes;
        if (t == 0) {
            const long long k1 = k + gridDim.x, k2 = k1 + gridDim.x;
            if (k1 < n_stages) {
                sd[b ^ 1] = nxt;
                s_maxc[b ^ 1] = 1;
                stage_issue(nxt, st_smem + (b ^ 1) * kBufBytes, &bars[b ^ 1], row_ptr, info, vid, lnu, lam);
            }
            if (k2 < n_stages) nxt = stages[k2];
        }
        mbar_wait(&bars[b], (unsigned)(i >> 1) & 1u);
        const Stage st = sd[b];
        const int32_t* svid = reinterpret_cast<const int32_t*>(buf + kOffVid);
        const int32_t* slam = reinterpret_cast<const int32_t*>(buf + kOffLam);
        const float* slnu = reinterpret_cast<const float*>(buf + kOffLnu);
        const long long* srp = reinterpret_cast<const long long*>(buf + kOffRp) + (st.r0 & 1);
        const RayInfo* sri = reinterpret_cast<const RayInfo*>(buf + kOffRi);
        uint16_t* cmap = reinterpret_cast<uint16_t*>(buf + kOffCm);
        const int span = (int)(st.s1 - st.s0), nr = st.r1 - st.r0;
        // chunk -> ray map, and the longest ray (in chunks) of the stage
        for (int j = t; j < nr; j += kStageThreads) {
            const int c0 = (int)(srp[j] - st.s0) >> 3, c1 = (int)(srp[j + 1] - st.s0) >> 3;
            for (int c = c0; c < c1; ++c) cmap[c] = (uint16_t)j;
            if (c1 - c0 > 1) atomicMax(&s_maxc[b], c1 - c0);
        }
        __syncthreads();
        const int rel = 8 * t;
        const bool act = rel < span;
        int c = 0, nch = 1, nv = 0;
        if (act) {
            const int j = cmap[t];
            const int st_j = (int)(srp[j] - st.s0);
            c = (rel - st_j) >> 3;
            nch = (int)(srp[j + 1] - srp[j]) >> 3;
            nv = min(8, st_j + sri[j].n - rel);
        }
        float la[8], w[8], l[8];
        identity_chunk<8>(la, w, l);
        if (act) {
            const int4 v0 = *reinterpret_cast<const int4*>(svid + rel);
            const int4 v1 = *reinterpret_cast<const int4*>(svid + rel + 4);
            const int4 q0 = *reinterpret_cast<const int4*>(slam + rel);
            const int4 q1 = *reinterpret_cast<const int4*>(slam + rel + 4);
            const float4 n0 = *reinterpret_cast<const float4*>(slnu + rel);
            const float4 n1 = *reinterpret_cast<const float4*>(slnu + rel + 4);
            const int v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
            const int q[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
            const float ln[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
            long long tv[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) tv[e] = e < nv ? __ldg(T + v[e]) : 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) elem_terms<M>(tv[e], q[e], ln[e], mp.L0, e < nv, la[e], w[e], l[e]);
        }
        float aB, bB;
        lane_composite<8>(la, w, aB, bB);
        Aff P = {-aB, bB - aB}, H = {aB, bB};
        // ray-relative inclusive scans over chunks: P over chunks 0..c, H over chunks c..nch-1
        const int maxc = s_maxc[b];
        int pp = 0;
        for (int d = 1; d < maxc; d <<= 1, pp ^= 1) {
            scan[pp * kStChunks + t] = make_float4(P.a, P.b, H.a, H.b);
            __syncthreads();
            if (act && c >= d) {
                const float4 x = scan[pp * kStChunks + t - d];
                P = compose<M>(P, Aff{x.x, x.y});
            }
            if (act && c + d < nch) {
                const float4 x = scan[pp * kStChunks + t + d];
                H = compose<M>(H, Aff{x.z, x.w});
            }
        }
        scan[pp * kStChunks + t] = make_float4(P.a, P.b, H.a, H.b);
        __syncthreads();
        // Q entering the chunk (chunk c-1's inclusive prefix applied to Q_1 = 0), R entering it
        // from the right (chunk c+1's inclusive suffix applied to R_N = 0)
        float Qin = kNeg, Rin = kNeg;
        if (act && c > 0) Qin = scan[pp * kStChunks + t - 1].y;
        if (act && c + 1 < nch) Rin = scan[pp * kStChunks + t + 1].w;
        float lR[8], lQ[8];
        lane_recurrences<8, M>(la, w, Rin, Qin, lR, lQ);
        if (act) lane_out<8>(l, lR, lQ, st.s0 + rel, st.s0 + rel + nv, lam);
        __syncthreads();  // buffer b and the scan scratch are free again
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
// <= per_item of its runs) and accumulates q into the tile's 16384 slots in shared memory, split
// into 16-bit halves held in two int32 arrays (native 32-bit shared atomics -- 64-bit shared
// atomics are CAS loops on sm_100a; a slot gets at most one contribution per run, so the halves
// cannot overflow within an item of <= 32768 runs).  A warp takes batches of 32 consecutive runs:
// one coalesced load of the 32 run descriptors (staged in shared memory), then the q of all 32
// runs (lane k = incidence k of the run, 32 independent loads in flight per lane), then one run
// per step: the 32 lanes of an atomic instruction always hit 32 DISTINCT slots (the voxels of one
// ray), never the same voxel twice (adjacent runs of a tile come from adjacent pixels and share
// most voxels: processing several runs per instruction serialised on same-address atomics).
// The in-tile slot comes from the run's step masks (no vid read): for incidence k,
// slot0 + sx cx + 32 sy cy + 1024 sz (k - cx - cy), cx = popc(mx & (2^k - 1)) (accumulator
// index L::index(s): the padded layout of AccLayout, see below).  The slots then go to T with one int64 atomic each (a tile spans several items).  Integer sums:
// exact, independent of order.
constexpr int kK6Threads = 1024;
constexpr int kK6Warps = kK6Threads / 32;
#ifndef MRF_K6_W
#define MRF_K6_W 16
#endif
constexpr int kK6W = MRF_K6_W;  // lanes per run in the add loop
// MRF_K6_STRIDES = 1: each run's step signs are turned into strides once, when its batch is staged
// (slot of element k = s0 + dz k + (dx - dz) cx + (dy - dz) cy, three IMADs per element), and the
// shared-memory adds are predicated instructions (no divergent block around them); 0: the round-1
// per-element decode of the sign bits.
#ifndef MRF_K6_STRIDES
#define MRF_K6_STRIDES 1
#endif
constexpr int kK6Desc = kK6Warps * 32 * (MRF_K6_STRIDES ? 32 : 16);  // per warp: the batch's 32 run descriptors

// slot -> accumulator index.  MRF_K6_SWIZZLE=1 XORs the low 5 bits with y ^ z so that y and z
// steps (slot strides 32, 1024) change the bank (a bijection inside every 32-slot row); off by
// default: K6 is ALU-bound and the 4 extra ALU ops cost more than the bank conflicts they
// avoid (2.85 vs 2.74 ms per iteration at frames30).
#ifndef MRF_K6_WARP_DYN
#define MRF_K6_WARP_DYN 1
#endif
#ifndef MRF_K6_SWIZZLE
#define MRF_K6_SWIZZLE 0
#endif
__device__ __forceinline__ int swz(int s) { return MRF_K6_SWIZZLE ? s ^ (((s >> 5) ^ (s >> 10)) & 31) : s; }
static_assert(!(MRF_K6_STRIDES && MRF_K6_SWIZZLE), "the stride decode needs a linear slot layout");
// Accumulator layout of a tile's slots.  Plain (PAD = false): index = slot = x + 32 y + 1024 z, so
// y and z steps stay in one shared-memory bank.  Padded: index = x + 35 y + 1127 z -- the bank
// moves by 1, 3 and 7 for x, y and z steps (odd: a straight run never repeats a bank within 32
// steps), at no ALU cost since the strides only change constants; 18024 entries instead of 16384.
#ifndef MRF_K6_SY
#define MRF_K6_SY 35
#endif
#ifndef MRF_K6_SZ
#define MRF_K6_SZ 1127
#endif
template <bool PAD>
struct AccLayout {
    static constexpr int SY = PAD ? MRF_K6_SY : 32, SZ = PAD ? MRF_K6_SZ : 1024;
    static constexpr int kSlots = PAD ? (31 + 31 * SY + 15 * SZ + 4) & ~3 : kTileSlots;  // multiple of 4
    static_assert(!PAD || (SY >= 32 && SZ >= 32 + 31 * SY && (SY & 1) && (SZ & 1)), "injective, odd bank steps");
    static constexpr int NS = PAD ? 15 : 14;                  // staged meta: index bits, then n - 1, signs
    __device__ __forceinline__ static int index(int s) {
        return PAD ? (s & 31) + SY * ((s >> 5) & 31) + SZ * (s >> 10) : swz(s);
    }
};

// MODE 0: the beliefs, sum of q (int32 halves, exact).
// Keyframe averages (reading R22), two integer passes over the same (frame, tile) buckets:
//   MODE 2: per slot the counts of non-negative / negative messages (packed n_pos + 65536 n_neg)
//     and the smallest |q| (native int32 shared atomics) -> N (int64 n_pos + 2^32 n_neg) and M
//     (uint32 min |q|) per (frame, slot);
//   then per (frame, slot) the scale a = |lambda_min| if all its messages have one sign, else -1
//     (kf_scale_kernel);
//   MODE 3: D = sum of the messages' small probabilities s = e^-|lambda| / (1 + e^-|lambda|) in
//     fixed point 2^-30, relative to s(a) when the slot's messages have one sign (a sum of
//     same-signed terms, kept relative-accurate down to e^-256), absolute and signed
//     (+ for lambda >= 0, - below) when they are mixed (then both sums below are >= 1/2):
//     int32 halves in shared memory (native atomics), int64 per (frame, slot).
// kf_finalize: sum mu(1) = n_pos - D, sum mu(0) = n_neg + D (mixed), or the one-signed forms with
// S = s(a) D, in fp64.  Round 1 summed D in fp64 with CAS-loop shared atomics (7.1 ms per
// iteration at frames30).
constexpr float kKfFix = 1073741824.0f;  // 2^30
constexpr double kKfFixInv = 1.0 / 1073741824.0;

// the keyframe-average passes' per-element adds (MODE 2: counts and min |q|; MODE 3: the small
// probability relative to the slot's scale, fixed point 2^-30 in 16-bit halves)
template <int MODE>
__device__ __forceinline__ void kf_accumulate(int si, int qv, int* acc_lo, int* acc_hi, int* accn, unsigned* accm,
                                              const float* accs) {
    if constexpr (MODE == 2) {
        atomicAdd(accn + si, qv >= 0 ? 1 : 65536);
        atomicMin(accm + si, qv >= 0 ? (unsigned)qv : 0u - (unsigned)qv);
    } else if constexpr (MODE == 3) {
        // s(|lambda|) / s(a) in fixed point (a = -1: mixed signs, absolute s)
        const float a = accs[si];
        const float al = (float)(qv >= 0 ? (unsigned)qv : 0u - (unsigned)qv) * (kQInv * kLog2e);
        const float ap = fmaxf(a, 0.f) * kLog2e;
        const float c = a < 0.f ? 1.f : 1.f + ex2(-ap);
        const float term = ex2(ap - al) * c * __frcp_rn(1.f + ex2(-al));
        int v = __float2int_rn(term * kKfFix);
        if (a < 0.f && qv < 0) v = -v;
        atomicAdd(acc_lo + si, v & 0xffff);
        atomicAdd(acc_hi + si, v >> 16);
    }
}

template <int MODE, bool PAD>
__global__ void __launch_bounds__(kK6Threads, 1) tile_reduce_kernel(long long n_items, const int2* __restrict__ items,
                                                                   const long long* __restrict__ tile_ptr,
                                                                   const Run* __restrict__ runs,
                                                                   const int32_t* __restrict__ lam, int per_item,
                                                                   void* out, long long n_out, unsigned* next,
                                                                   const int32_t* __restrict__ tile_map, long long chk_lam,
                                                                   long long chk_out_tiles, int n_tiles) {
    extern __shared__ int smem[];
    using L = AccLayout<PAD>;
    static_assert(MODE != 3 || !PAD, "the keyframe-average sums (12 B per slot) use the plain layout (shared memory)");
    constexpr int kAccInts = MODE == 3 ? 3 * L::kSlots : 2 * L::kSlots;
    int* acc_lo = smem;                 // MODE 0 / 3: sum of (v & 0xffff), at L::index(slot)
    int* acc_hi = smem + L::kSlots;     // MODE 0 / 3: sum of (v >> 16)
    int* accn = smem;                   // MODE 2: packed counts
    unsigned* accm = reinterpret_cast<unsigned*>(smem + L::kSlots);  // MODE 2: min |q|
    float* accs = reinterpret_cast<float*>(smem + 2 * L::kSlots);     // MODE 3: the bucket's scales
    uint4* sdesc = reinterpret_cast<uint4*>(smem + kAccInts) + (threadIdx.x >> 5) * 32;  // this warp's batch
    int4* sab = reinterpret_cast<int4*>(smem + kAccInts) + kK6Warps * 32 + (threadIdx.x >> 5) * 32;  // its strides
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // items: the first per CTA by index, then dynamically (a CTA whose items ran short takes the
    // next one instead of a fixed stride, so the uneven last chunks of the tiles do not leave SMs
    // idle at the end); next == nullptr: fixed stride
    __shared__ long long s_next;
    __shared__ int s_batch;
    // the accumulator is zeroed once here, then by each item's flush as it reads it
    for (int i = threadIdx.x; i < kAccInts / 4; i += kK6Threads) reinterpret_cast<int4*>(smem)[i] = int4{0, 0, 0, 0};
    if constexpr (MODE >= 2) {
        // the zeroing above and the writes below (MODE 2: min |q| starts at the maximum; MODE 3:
        // the first item's scales) touch the same words from different threads
        __syncthreads();
        if constexpr (MODE == 2)
            for (int i = threadIdx.x; i < L::kSlots; i += kK6Threads) accm[i] = 0xffffffffu;
    }
    for (long long it = blockIdx.x; it < n_items;) {
        const int2 item = __ldg(items + it);
#if MRF_K6_WARP_DYN
        if (threadIdx.x == 0) s_batch = kK6Warps;
#endif
        if constexpr (MODE == 3) {  // the bucket's per-slot scales (kf_scale_kernel)
            const float* A = reinterpret_cast<const float*>(static_cast<long long*>(out) + 2 * n_out) +
                             ((long long)item.x << kTileShift);
            for (int i = threadIdx.x; i < kTileSlots; i += kK6Threads) accs[swz(i)] = __ldg(A + i);
        }
        __syncthreads();
        const long long r0 = __ldg(tile_ptr + item.x) + (long long)item.y * per_item;
        long long r1 = __ldg(tile_ptr + item.x + 1);
        if (r1 > r0 + per_item) r1 = r0 + per_item;
#if MRF_K6_WARP_DYN
        // batches of 32 runs: the first one per warp by index, then from a shared counter (the
        // item ends at a barrier, so the warps should finish together)
        for (long long bi = wid;;) {
            const long long rb = r0 + 32LL * bi;
            if (rb >= r1) break;
#else
        for (long long rb = r0 + 32LL * wid; rb < r1; rb += 32LL * kK6Warps) {
#endif
            const int nb = (int)min(32LL, r1 - rb);
            uint4 d{0u, 0u, 0u, 0u};
            if (lane < nb) d = __ldg(reinterpret_cast<const uint4*>(runs + rb + lane));
            MRF_ASSERT(lane >= nb || (long long)d.x + ((d.y >> 14) & 63u) + 1 <= chk_lam);
#if MRF_K6_STRIDES
            {
                // staged: {e, s0 | n << 16, mx, my} and {dx - dz, dy - dz, dz}, s0 the accumulator
                // index of the first element (an empty slot of the batch: n = 0)
                const unsigned meta = d.y;
                const int n = lane < nb ? (int)((meta >> 14) & 63u) + 1 : 0;
                const int s0 = L::index((int)(meta & (kTileSlots - 1)));
                const int dx = (meta >> 20) & 1u ? -1 : 1, dy = (meta >> 21) & 1u ? -L::SY : L::SY,
                          dz = (meta >> 22) & 1u ? -L::SZ : L::SZ;
                d.y = (unsigned)s0 | ((unsigned)n << 16);
                sab[lane] = int4{dx - dz, dy - dz, dz, 0};
            }
#else
            if constexpr (PAD)  // in-tile slot -> accumulator index, once per run
                d.y = (unsigned)L::index((int)(d.y & (kTileSlots - 1))) | ((d.y >> 14) << L::NS);
#endif
            sdesc[lane] = d;
            __syncwarp();
            // Lane groups of kK6W lanes (32 / kK6W runs per instruction): in round r, group g takes
            // incidences r*kK6W .. r*kK6W+kK6W-1 of run j + g*kK6W (runs kK6W apart in the batch:
            // pixels far enough apart to rarely hit the same voxel at the same time); rounds past
            // every run's end are skipped.
            constexpr int NJ = kK6W, NR = 32 / kK6W;
            const int hw = lane / kK6W, hl = lane % kK6W;
            int q[NR][NJ];
#pragma unroll
            for (int j = 0; j < NJ; ++j) {
                const uint4 x = sdesc[j + NJ * hw];
#if MRF_K6_STRIDES
                const int n = (int)(x.y >> 16);
#else
                const int n = j + NJ * hw < nb ? (int)((x.y >> L::NS) & 63u) + 1 : 0;
#endif
#pragma unroll
                for (int rnd = 0; rnd < NR; ++rnd) {
                    const int k = hl + kK6W * rnd;
                    q[rnd][j] = k < n ? __ldg(lam + x.x + k) : 0;
                }
            }
#if MRF_K6_STRIDES
            {
                const unsigned acc_sh = (unsigned)__cvta_generic_to_shared(acc_lo);
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    const uint4 x = sdesc[j + NJ * hw];
                    const int4 st = sab[j + NJ * hw];
                    const int n = (int)(x.y >> 16);
                    const int base = (int)(x.y & 0xffffu) + st.z * hl;
#pragma unroll
                    for (int rnd = 0; rnd < NR; ++rnd) {
                        const int k = hl + kK6W * rnd;
                        if (rnd > 0 && !__any_sync(kFull, k < n)) break;  // every run of the column ended
                        const unsigned below_k = (1u << k) - 1u;
                        const int si = base + st.z * (kK6W * rnd) + st.x * __popc(x.z & below_k) +
                                       st.y * __popc(x.w & below_k);
                        MRF_ASSERT(k >= n || (si >= 0 && si < L::kSlots));
                        const int qv = q[rnd][j];
                        if constexpr (MODE == 0) {
                            const unsigned a = acc_sh + 4u * (unsigned)si;
                            asm volatile(
                                "{\n.reg .pred p;\nsetp.lt.s32 p, %2, %3;\n"
                                "@p red.shared.add.u32 [%0], %1;\n@p red.shared.add.u32 [%0+%5], %4;\n}"
                                :: "r"(a), "r"(qv & 0xffff), "r"(k), "r"(n), "r"(qv >> 16), "n"(4 * L::kSlots));
                        } else if (k < n) {
                            kf_accumulate<MODE>(si, qv, acc_lo, acc_hi, accn, accm, accs);
                        }
                    }
                }
            }
            if constexpr (false)
#endif
            {
#pragma unroll
            for (int rnd = 0; rnd < NR; ++rnd) {
                const int k = hl + kK6W * rnd;
                const unsigned below_k = (1u << k) - 1u;
#pragma unroll
                for (int j = 0; j < NJ; ++j) {
                    const uint4 x = sdesc[j + NJ * hw];
                    const unsigned meta = x.y;
#if MRF_K6_STRIDES
                    const int n = (int)(meta >> 16);
#else
                    const int n = j + NJ * hw < nb ? (int)((meta >> L::NS) & 63u) + 1 : 0;
#endif
                    if (rnd > 0 && !__any_sync(kFull, k < n)) continue;  // every run of the column ended
                    if (k < n) {
                        const int cx = __popc(x.z & below_k), cy = __popc(x.w & below_k);
#if MRF_K6_STRIDES
                        const int4 st = sab[j + NJ * hw];
                        const int si0 = (int)(meta & 0xffffu) + st.z * k + st.x * cx + st.y * cy;
#else
                        const int sx = (meta >> (L::NS + 6)) & 1 ? -cx : cx, sy = (meta >> (L::NS + 7)) & 1 ? -cy : cy;
                        const int cz = k - cx - cy, sz = (meta >> (L::NS + 8)) & 1 ? -cz : cz;
                        const int si0 = (int)(meta & ((1u << L::NS) - 1u)) + sx + L::SY * sy + L::SZ * sz;
#endif
                        const int si = (PAD || MRF_K6_STRIDES) ? si0 : swz(si0);
                        MRF_ASSERT(si >= 0 && si < L::kSlots);
                        const int qv = q[rnd][j];
                        if constexpr (MODE == 0) {
                            atomicAdd(acc_lo + si, qv & 0xffff);
                            atomicAdd(acc_hi + si, qv >> 16);
                        } else if constexpr (MODE == 2) {
                            atomicAdd(accn + si, qv >= 0 ? 1 : 65536);
                            atomicMin(accm + si, qv >= 0 ? (unsigned)qv : 0u - (unsigned)qv);
                        } else {
                            // s(|lambda|) / s(a) in fixed point (a = -1: mixed signs, absolute s)
                            const float a = accs[si];
                            const float al = (float)(qv >= 0 ? (unsigned)qv : 0u - (unsigned)qv) * (kQInv * kLog2e);
                            const float ap = fmaxf(a, 0.f) * kLog2e;
                            const float c = a < 0.f ? 1.f : 1.f + ex2(-ap);
                            const float term = ex2(ap - al) * c * __frcp_rn(1.f + ex2(-al));
                            int v = __float2int_rn(term * kKfFix);
                            if (a < 0.f && qv < 0) v = -v;
                            atomicAdd(acc_lo + si, v & 0xffff);
                            atomicAdd(acc_hi + si, v >> 16);
                        }
                    }
                }
            }
            }
            __syncwarp();
#if MRF_K6_WARP_DYN
            int nxt = 0;
            if (lane == 0) nxt = atomicAdd(&s_batch, 1);
            bi = __shfl_sync(kFull, nxt, 0);
#endif
        }
        __syncthreads();
        if constexpr (MODE == 0) {
            // world > 1: the tile's slots go to its position among the tiles some rank touches
            // (the compacted all-reduce buffer); else to the tile itself
            const int tile = item.x % n_tiles;  // (buckets may be (frame, tile) pairs, frame-major)
            const long long tpos = tile_map ? (long long)__ldg(tile_map + tile) : (long long)tile;
            MRF_ASSERT(tpos >= 0 && tpos < chk_out_tiles);
            long long* Tt = static_cast<long long*>(out) + (tpos << kTileShift);
            for (int i = threadIdx.x; i < kTileSlots; i += kK6Threads) {
                const int a = L::index(i);
                const long long sum = (long long)acc_hi[a] * 65536 + (long long)acc_lo[a];
                acc_hi[a] = 0;
                acc_lo[a] = 0;
                if (sum) atomicAdd(reinterpret_cast<unsigned long long*>(Tt + i), (unsigned long long)sum);
            }
        } else if constexpr (MODE == 2) {  // out: N (int64 n_pos + 2^32 n_neg) [n_out], D [n_out], M (uint32) [n_out]
            const long long o = (long long)item.x << kTileShift;
            unsigned long long* Nt = static_cast<unsigned long long*>(out) + o;
            unsigned* Mt = reinterpret_cast<unsigned*>(static_cast<unsigned long long*>(out) + 2 * n_out) + o;
            for (int i = threadIdx.x; i < kTileSlots; i += kK6Threads) {
                const int a = L::index(i);
                const unsigned cn = (unsigned)accn[a];
                const unsigned mq = accm[a];
                accn[a] = 0;
                accm[a] = 0xffffffffu;
                if (cn) {
                    atomicAdd(Nt + i, (unsigned long long)(cn & 0xffffu) | ((unsigned long long)(cn >> 16) << 32));
                    atomicMin(Mt + i, mq);
                }
            }
        } else {  // MODE 3: D (int64, 2^-30) [n_out .. 2 n_out)
            const long long o = (long long)item.x << kTileShift;
            unsigned long long* Dt = static_cast<unsigned long long*>(out) + n_out + o;
            for (int i = threadIdx.x; i < kTileSlots; i += kK6Threads) {
                const long long sum = (long long)acc_hi[swz(i)] * 65536 + (long long)acc_lo[swz(i)];
                acc_hi[swz(i)] = 0;
                acc_lo[swz(i)] = 0;
                if (sum) atomicAdd(Dt + i, (unsigned long long)sum);
            }
        }
        if (next) {  // (this barrier also ends the flush before the next item's adds)
            if (threadIdx.x == 0) s_next = (long long)gridDim.x + atomicAdd(next, 1u);
            __syncthreads();
            it = s_next;
        } else {
            it += gridDim.x;
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------- K6b: pixel-block reduction
// The voxel sums T_v = sum of the messages of every incidence on v (Eq.6; "accumulated to
// obtain the current incoming belief"), read
// in the messages' own (ray-major) order instead of through a transpose.  A work item is a block
// of neighbouring pixels of one frame (kBlkCols columns x kBlkRows owned rows): their rays fan out
// through nearly the same voxels (frames30: 43.6 k incidences per 32 x 16 block fall on 400-900
// distinct voxels, a factor of ~100), so a CTA sums the block's messages into a small shared hash
// table keyed by the belief slot and then adds each entry to T with one int64 global atomic.
// Per incidence the kernel reads vid and lambda once, coalesced and contiguous (SURVEY §8(d)'s
// 8 B), and needs no tile runs, bucket pass or work list beyond the block list.
//   * a warp takes the block's rows from a shared counter and streams each row's slots -- its 32
//     rays' segments are contiguous -- with 16-byte loads, 4 slots per lane (the 4 adds of an
//     element index k touch slots 4 apart: distinct voxels unless two rays meet by chance);
//   * table: open addressing, multiplicative hash, linear probing, 16-bit halves of q in two int32
//     arrays (a slot gets at most one message per ray, <= 512 per block: no overflow);
//   * fast path: ONE probe, branch-free -- an element whose key sits at its home slot (almost all:
//     each voxel recurs ~100 times per block) adds there at once; the others (a key's first
//     occurrence, or a key displaced by probing) go to a per-warp ring (room for a lane group's
//     4 x 32 misses) that is drained 32 at a time by the full probe loop (claim by CAS), so the
//     loop's divergence is paid by full warps
//     of misses instead of by every warp holding one (a per-element probe loop ran 3-4 iterations
//     per warp instruction: the longest of 32 lanes' probe sequences);
//   * a block claims at most half the table (linear probing stays short); an element whose key
//     finds no room, or whose probe sequence exceeds max_probe (64), goes straight to T with a
//     global atomic: exact either way.  The claims and direct adds are counted (stats) so that
//     the host can drop K6b where blocks share too little (interleaved rows of several ranks,
//     fine grids: DESIGN §5 K6b);
//   * integer sums: T is bit-identical to the tile-run K6 for any block shape or order.
constexpr int kBlkThreads = 256;
constexpr int kBlkWarps = kBlkThreads / 32;
constexpr int kBlkTableLog = 11;  // 2048 entries
constexpr int kBlkQueue = 160;    // per-warp ring of deferred (v, q): < 32 left + 4 x 32 appended
#ifndef MRF_BLK_CTAS
#define MRF_BLK_CTAS 6
#endif
constexpr int kBlkMinCtas = MRF_BLK_CTAS;  // resident CTAs per SM (registers: 65536 / (256 x 6) = 42)
template <int S_LOG>
__global__ void __launch_bounds__(kBlkThreads, kBlkMinCtas) block_reduce_kernel(long long n_blocks, const int4* __restrict__ blocks,
                                                                     const long long* __restrict__ row_ptr,
                                                                     const RayInfo* __restrict__ ray_z,
                                                                     const int32_t* __restrict__ vid,
                                                                     const int32_t* __restrict__ lam, long long* T,
                                                                     unsigned* next, unsigned long long* stats,
                                                                     const int32_t* __restrict__ tile_map,
                                                                     int max_probe, long long chk_lam, long long chk_out) {
    constexpr int S = 1 << S_LOG;
    __shared__ int key[S];
    __shared__ int acc[2 * S];  // [0, S): sum of (q & 0xffff); [S, 2S): sum of (q >> 16)
    __shared__ int2 queue[kBlkWarps][kBlkQueue];
    __shared__ int s_row;
    __shared__ int s_used, s_fall;  // this block's claimed entries, elements sent to T directly
    __shared__ long long s_blk;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < S; i += kBlkThreads) {
        key[i] = -1;
        acc[i] = 0;
        acc[S + i] = 0;
    }
    if (threadIdx.x == 0) {
        s_row = 0;
        s_used = 0;
        s_fall = 0;
    }
    __syncthreads();
    volatile int* vused = &s_used;
    const unsigned acc_sh = (unsigned)__cvta_generic_to_shared(acc);
    volatile int* vkey = key;
    int2* wq = queue[wid];
    int qh = 0, qt = 0;  // the warp's ring: entries [qh, qt) (warp-uniform)
    auto to_T = [&](int v) -> long long {
        return tile_map ? ((long long)__ldg(tile_map + (v >> kTileShift)) << kTileShift) | (v & (kTileSlots - 1))
                        : (long long)v;
    };
    auto hash = [](int v) { return ((unsigned)v * 0x9E3779B1u) >> (32 - S_LOG); };
    auto red2 = [&](unsigned h, int q) {
        const unsigned a = acc_sh + 4u * h;
        asm volatile("red.shared.add.u32 [%0], %1;\n\tred.shared.add.u32 [%0+%3], %2;" ::"r"(a), "r"(q & 0xffff),
                     "r"(q >> 16), "n"(4 * S));
    };
    // the full probe loop (queued elements): find or claim v's slot, else T directly
    auto slow = [&](int v, int q) {
        unsigned h = hash(v);
        int p = max_probe < 0 ? max_probe : 0;  // (< 0: every element to T directly, a test knob)
        for (; p >= 0; ++p) {
            const int k = vkey[h];
            if (k == v) break;
            if (k < 0) {  // v is absent (no deletions): claim this slot, unless the table is half full
                if (*vused >= S / 2) {
                    p = max_probe;
                    break;
                }
                const int old = atomicCAS(key + h, -1, v);
                if (old < 0) {
                    atomicAdd(&s_used, 1);
                    break;
                }
                if (old == v) break;
            }
            h = (h + 1) & (S - 1);
            if (p == max_probe) break;
        }
        if (p >= 0 && p < max_probe) {
            red2(h, q);
        } else {
            const long long t = to_T(v);
            MRF_ASSERT(t >= 0 && t < chk_out);
            atomicAdd(reinterpret_cast<unsigned long long*>(T + t), (unsigned long long)(long long)q);
            atomicAdd(&s_fall, 1);
        }
    };
    auto drain = [&](int cnt) {  // the first cnt queued entries, one per lane
        __syncwarp();
        if (lane < cnt) {
            const int j = qh + lane;
            const int2 e = wq[j >= kBlkQueue ? j - kBlkQueue : j];
            slow(e.x, e.y);
        }
        qh += cnt;
        if (qh >= kBlkQueue) {  // (keeps the ring positions below 2 x kBlkQueue)
            qh -= kBlkQueue;
            qt -= kBlkQueue;
        }
        __syncwarp();
    };
    // fast path for one lane's 4 slots (q = 0: nothing to add -- padding, or a zero message):
    // 4 independent probes of the home slots, the adds predicated on a hit, misses queued
    const unsigned key_sh = (unsigned)__cvta_generic_to_shared(key);
    const bool fast = max_probe >= 0;
    auto add4 = [&](const int4& v4, const int4& q4) {
        const int vv[4] = {v4.x, v4.y, v4.z, v4.w}, qq[4] = {q4.x, q4.y, q4.z, q4.w};
        unsigned hh[4];
        int kk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            hh[k] = hash(vv[k]);
            asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(kk[k]) : "r"(key_sh + 4u * hh[k]));
        }
        bool miss[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            // the adds predicated on a hit (a miss lane adding 0 instead costs more bank conflicts
            // in this L1-bound kernel: measured)
            const bool hit = fast && qq[k] != 0 && kk[k] == vv[k];
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.u32 p, %3, 0;\n"
                "@p red.shared.add.u32 [%0], %1;\n@p red.shared.add.u32 [%0+%4], %2;\n}" ::"r"(acc_sh + 4u * hh[k]),
                "r"(qq[k] & 0xffff), "r"(qq[k] >> 16), "r"((unsigned)hit), "n"(4 * S));
            miss[k] = qq[k] != 0 && !hit;
        }
        // the misses to the ring (room for 4 x 32 more: drained below 32 before each add4)
        unsigned ltm;
        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltm));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned mm = __ballot_sync(kFull, miss[k]);
            const int j = qt + __popc(mm & ltm);  // (qt < qh + 160 <= 320)
            if (miss[k]) wq[j >= kBlkQueue ? j - kBlkQueue : j] = make_int2(vv[k], qq[k]);
            qt += __popc(mm);
        }
        while (qt - qh >= 32) drain(32);
    };
    for (long long bi = blockIdx.x; bi < n_blocks;) {
        const int4 b = __ldg(blocks + bi);  // {first ray, ncols | nrows << 16, row stride (rays), -}
        const int ncols = b.y & 0xffff, nrows = b.y >> 16;
        for (;;) {
            int r = 0;
            if (lane == 0) r = atomicAdd(&s_row, 1);
            r = __shfl_sync(kFull, r, 0);
            if (r >= nrows) break;
            // the row's rays are contiguous slots [A, B) (their segments, 8-aligned, in pixel order);
            // slots past a ray's end are padding with lambda = 0 (the fill writes it, K5 never
            // writes a slot past n, import and re-layout fill it with 0), skipped like any zero
            const long long ray = (long long)b.x + (long long)r * b.z;
            // (unsigned: e runs up to 383 slots past B, which may lie just below 2^31)
            const unsigned A = (unsigned)__ldg(row_ptr + ray), B = (unsigned)__ldg(row_ptr + ray + ncols);
            for (unsigned e = A + 4 * lane; e - 4 * lane < B; e += 256) {  // (warp-uniform trip count)
                int4 v0 = {0, 0, 0, 0}, q0 = {0, 0, 0, 0}, v1 = {0, 0, 0, 0}, q1 = {0, 0, 0, 0};
                MRF_ASSERT(e >= B || (long long)e + 3 < chk_lam);
                if (e < B) {
                    v0 = __ldg(reinterpret_cast<const int4*>(vid + e));
                    q0 = __ldg(reinterpret_cast<const int4*>(lam + e));
                }
                if (e + 128 < B) {
                    v1 = __ldg(reinterpret_cast<const int4*>(vid + e + 128));
                    q1 = __ldg(reinterpret_cast<const int4*>(lam + e + 128));
                }
                // (B is a multiple of 8 and e of 4: a lane's 4 slots lie all inside [A, B) or all past it)
                add4(v0, q0);
                if (e - 4 * lane + 128 < B) add4(v1, q1);  // (warp-uniform)
            }
        }
        if (qt > qh) drain(qt - qh);
        __syncthreads();
        // flush: every claimed entry to T (one int64 atomic), and clear it for the next block
        for (int i = threadIdx.x; i < S; i += kBlkThreads) {
            const int v = key[i];
            if (v >= 0) {
                const long long sum = (long long)acc[S + i] * 65536 + (long long)acc[i];
                key[i] = -1;
                acc[i] = 0;
                acc[S + i] = 0;
                if (sum) {
                    const long long t = to_T(v);
                    MRF_ASSERT(t >= 0 && t < chk_out);
                    atomicAdd(reinterpret_cast<unsigned long long*>(T + t), (unsigned long long)sum);
                }
            }
        }
        if (threadIdx.x == 0) {
            // stats[0]: claimed entries (distinct voxels per block, summed), stats[1]: elements
            // sent to T directly -- the host's check that the blocks share voxels (mrf_api.cu)
            if (stats) {
                atomicAdd(stats, (unsigned long long)s_used);
                if (s_fall) atomicAdd(stats + 1, (unsigned long long)s_fall);
            }
            s_row = 0;
            s_used = 0;
            s_fall = 0;
            s_blk = (long long)gridDim.x + atomicAdd(next, 1u);
        }
        __syncthreads();
        bi = s_blk;
    }
}

// ---------------------------------------------------------------- K6b for the keyframe averages
// The two integer passes of the keyframe-average sums (MODE 2: counts + min |q|; MODE 3: the
// fixed-point small probabilities relative to the slot's scale -- see kf_accumulate above) over
// pixel blocks instead of (frame, tile) run buckets: a block lies in one frame (b.w), so its
// hash-table entries are (frame, slot) sums already.  Unlike the belief sums a zero message
// counts here, so an element's validity comes from its ray (slots past a ray's end are padding):
// the lane finds the ray of its 4 slots among the row's 32 by a shuffle binary search.
// Integer sums (and min) in any order: bit-identical to the tile-run passes.
template <int MODE>
__global__ void __launch_bounds__(kBlkThreads, kBlkMinCtas) block_kf_kernel(long long n_blocks, const int4* __restrict__ blocks,
                                                                          const long long* __restrict__ row_ptr,
                                                                          const RayInfo* __restrict__ ray_z,
                                                                          const int32_t* __restrict__ vid,
                                                                          const int32_t* __restrict__ lam,
                                                                          long long* out, long long n_out, long long VI,
                                                                          unsigned* next, long long chk_lam) {
    constexpr int S = 1 << kBlkTableLog;
    constexpr int kMaxProbe = 64;
    __shared__ int key[S];
    __shared__ int a0[S];  // MODE 2: packed counts n_pos + 65536 n_neg; MODE 3: sum of (v & 0xffff)
    __shared__ int a1[S];  // MODE 2: min |q| (unsigned); MODE 3: sum of (v >> 16)
    __shared__ int2 queue[kBlkWarps][kBlkQueue];
    __shared__ int s_row, s_used;
    __shared__ long long s_blk;
    const int lane = threadIdx.x & 31;
    unsigned long long* N = reinterpret_cast<unsigned long long*>(out);
    long long* D = out + n_out;
    unsigned* M = reinterpret_cast<unsigned*>(out + 2 * n_out);
    const float* A = reinterpret_cast<const float*>(out + 2 * n_out);
    for (int i = threadIdx.x; i < S; i += kBlkThreads) {
        key[i] = -1;
        a0[i] = 0;
        a1[i] = MODE == 2 ? -1 : 0;
    }
    if (threadIdx.x == 0) {
        s_row = 0;
        s_used = 0;
    }
    __syncthreads();
    volatile int* vkey = key;
    volatile int* vused = &s_used;
    auto hash = [](int v) { return ((unsigned)v * 0x9E3779B1u) >> (32 - kBlkTableLog); };
    // the element's term: MODE 2 (count word, |q|), MODE 3 the fixed-point value (kf_accumulate)
    auto term3a = [&](float a, int qv) {
        const float al = (float)(qv >= 0 ? (unsigned)qv : 0u - (unsigned)qv) * (kQInv * kLog2e);
        const float ap = fmaxf(a, 0.f) * kLog2e;
        const float c = a < 0.f ? 1.f : 1.f + ex2(-ap);
        const float t = ex2(ap - al) * c * __frcp_rn(1.f + ex2(-al));
        int r = __float2int_rn(t * kKfFix);
        if (a < 0.f && qv < 0) r = -r;
        return r;
    };
    auto term3 = [&](long long fb, int v, int qv) { return term3a(__ldg(A + fb + v), qv); };
    auto add = [&](long long fb, int v, int qv) {
        unsigned h = hash(v);
        int p = 0;
        for (; p < kMaxProbe; ++p) {
            const int k = vkey[h];
            if (k == v) break;
            if (k < 0) {
                if (*vused >= S / 2) {
                    p = kMaxProbe;
                    break;
                }
                const int old = atomicCAS(key + h, -1, v);
                if (old < 0) {
                    atomicAdd(&s_used, 1);
                    break;
                }
                if (old == v) break;
            }
            h = (h + 1) & (S - 1);
        }
        const unsigned aq = qv >= 0 ? (unsigned)qv : 0u - (unsigned)qv;
        if (p < kMaxProbe) {
            if constexpr (MODE == 2) {
                atomicAdd(a0 + h, qv >= 0 ? 1 : 65536);
                atomicMin(reinterpret_cast<unsigned*>(a1) + h, aq);
            } else {
                const int t = term3(fb, v, qv);
                atomicAdd(a0 + h, t & 0xffff);
                atomicAdd(a1 + h, t >> 16);
            }
        } else {  // straight to the (frame, slot) sums
            if constexpr (MODE == 2) {
                atomicAdd(N + fb + v, qv >= 0 ? 1ull : (1ull << 32));
                atomicMin(M + fb + v, aq);
            } else {
                atomicAdd(reinterpret_cast<unsigned long long*>(D + fb + v), (unsigned long long)(long long)term3(fb, v, qv));
            }
        }
    };
    // the misses of the fast path, per warp (as in block_reduce_kernel)
    int2* wq = queue[threadIdx.x >> 5];
    int qh = 0, qt = 0;
    const unsigned key_sh = (unsigned)__cvta_generic_to_shared(key);
    auto drain = [&](long long fb, int cnt) {
        __syncwarp();
        if (lane < cnt) {
            const int j = qh + lane;
            const int2 q2 = wq[j >= kBlkQueue ? j - kBlkQueue : j];
            add(fb, q2.x, q2.y);
        }
        qh += cnt;
        if (qh >= kBlkQueue) {
            qh -= kBlkQueue;
            qt -= kBlkQueue;
        }
        __syncwarp();
    };
    for (long long bi = blockIdx.x; bi < n_blocks;) {
        const int4 b = __ldg(blocks + bi);  // {first ray, ncols | nrows << 16, row stride (rays), frame}
        const int ncols = b.y & 0xffff, nrows = b.y >> 16;
        const long long fb = (long long)b.w * VI;
        for (;;) {
            int r = 0;
            if (lane == 0) r = atomicAdd(&s_row, 1);
            r = __shfl_sync(kFull, r, 0);
            if (r >= nrows) break;
            const long long ray = (long long)b.x + (long long)r * b.z;
            // lane j: ray j's first slot and length (past the row: never <= a slot)
            unsigned rp = 0xffffffffu;
            int nr = 0;
            if (lane < ncols) {
                rp = (unsigned)__ldg(row_ptr + ray + lane);
                nr = __ldg(&ray_z[ray + lane].n);
            }
            const unsigned A0 = __shfl_sync(kFull, rp, 0);
            const unsigned B = (unsigned)__ldg(row_ptr + ray + ncols);
            for (unsigned e = A0 + 4 * lane; e - 4 * lane < B; e += 128) {  // (warp-uniform trip count)
                int4 v4 = {0, 0, 0, 0}, q4 = {0, 0, 0, 0};
                const bool in = e < B;
                if (in) {
                    MRF_ASSERT((long long)e + 3 < chk_lam);
                    v4 = __ldg(reinterpret_cast<const int4*>(vid + e));
                    q4 = __ldg(reinterpret_cast<const int4*>(lam + e));
                }
                // the ray of slots e..e+3 (one ray: segments are 8-aligned): the largest j with rp_j <= e
                int j = 0;
#pragma unroll
                for (int st = 16; st >= 1; st >>= 1) {
                    const unsigned rc = __shfl_sync(kFull, rp, (j + st) & 31);
                    if (j + st < 32 && rc <= e) j += st;
                }
                const unsigned s0 = __shfl_sync(kFull, rp, j);
                const int nj = __shfl_sync(kFull, nr, j);
                const int vv[4] = {v4.x, v4.y, v4.z, v4.w}, qq[4] = {q4.x, q4.y, q4.z, q4.w};
                // fast path: the 4 home slots probed at once, hits added there, misses queued
                unsigned hh[4];
                int kk[4];
                float sa[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    hh[k] = hash(vv[k]);
                    asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(kk[k]) : "r"(key_sh + 4u * hh[k]));
                    if constexpr (MODE == 3) sa[k] = in ? __ldg(A + fb + vv[k]) : 0.f;
                }
                bool miss[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool ok = in && (int)(e + k - s0) < nj;
                    const bool hit = ok && kk[k] == vv[k];
                    if (hit) {
                        if constexpr (MODE == 2) {
                            atomicAdd(a0 + hh[k], qq[k] >= 0 ? 1 : 65536);
                            atomicMin(reinterpret_cast<unsigned*>(a1) + hh[k],
                                      qq[k] >= 0 ? (unsigned)qq[k] : 0u - (unsigned)qq[k]);
                        } else {
                            const int t = term3a(sa[k], qq[k]);
                            atomicAdd(a0 + hh[k], t & 0xffff);
                            atomicAdd(a1 + hh[k], t >> 16);
                        }
                    }
                    miss[k] = ok && !hit;
                }
                unsigned ltm;
                asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltm));
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const unsigned mm = __ballot_sync(kFull, miss[k]);
                    const int jq = qt + __popc(mm & ltm);
                    if (miss[k]) wq[jq >= kBlkQueue ? jq - kBlkQueue : jq] = make_int2(vv[k], qq[k]);
                    qt += __popc(mm);
                }
                while (qt - qh >= 32) drain(fb, 32);
            }
        }
        if (qt > qh) drain(fb, qt - qh);
        __syncthreads();
        for (int i = threadIdx.x; i < S; i += kBlkThreads) {
            const int v = key[i];
            if (v >= 0) {
                if constexpr (MODE == 2) {
                    const unsigned cn = (unsigned)a0[i];
                    atomicAdd(N + fb + v, (unsigned long long)(cn & 0xffffu) | ((unsigned long long)(cn >> 16) << 32));
                    atomicMin(M + fb + v, (unsigned)a1[i]);
                } else {
                    const long long sum = (long long)a1[i] * 65536 + (long long)a0[i];
                    if (sum) atomicAdd(reinterpret_cast<unsigned long long*>(D + fb + v), (unsigned long long)sum);
                }
                key[i] = -1;
                a0[i] = 0;
                a1[i] = MODE == 2 ? -1 : 0;
            }
        }
        if (threadIdx.x == 0) {
            s_row = 0;
            s_used = 0;
            s_blk = (long long)gridDim.x + atomicAdd(next, 1u);
        }
        __syncthreads();
        bi = s_blk;
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

// Per-device opt-in of the large dynamic shared memory (the attribute is per device: a process
// may drive ctxs on several GPUs) and the device's SM count (grid sizing).
struct DevCfg {
    int sms = 0;
    bool k6[4][2] = {};
};
DevCfg& dev_cfg() {
    static thread_local DevCfg cfg[64];
    int dev = 0;
    cudaGetDevice(&dev);
    DevCfg& c = cfg[dev & 63];
    if (!c.sms) cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
    if (!c.sms) c.sms = 148;
    return c;
}


template <int M, bool AVG, int k>
void launch_class_k(int cls, long long n_rays, const int4* desc, const int32_t* vid, const float* lnu, int32_t* lam,
                    const long long* T, const MsgParams& mp, cudaStream_t s) {
    if constexpr (k < kNumShort) {
        if (cls == k) {
            constexpr int G = class_G(k), K = class_K(k);
            const unsigned grid = blocks_for((n_rays + 32 / G - 1) / (32 / G) * 32, 256);
            ray_msg_kernel<G, K, M, AVG><<<grid, 256, 0, s>>>(n_rays, desc, vid, lnu, lam, T, mp);
            return;
        }
        launch_class_k<M, AVG, k + 1>(cls, n_rays, desc, vid, lnu, lam, T, mp, s);
    }
}

template <int M, bool AVG>
void launch_ray_messages_m(int cls, long long n_rays, const int32_t* rays, const int4* desc, const long long* row_ptr,
                           const RayInfo* ray_z, const int32_t* vid, const float* lnu, int32_t* lam,
                           const long long* T, const MsgParams& mp, float* scratch, long long scratch_per_warp,
                           int n_warps_long, cudaStream_t s) {
    if (cls < kNumShort) {
        launch_class_k<M, AVG, 0>(cls, n_rays, desc, vid, lnu, lam, T, mp, s);
    } else {
        const unsigned g = blocks_for((long long)n_warps_long * 32, 256);
        ray_msg_long_kernel<M, AVG, false><<<g, 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, vid, lnu, lam, T, mp, scratch,
                                                             scratch_per_warp, WalkParams{});
    }
}

template <int M, bool AVG, int k>
void launch_walk_class_k(int cls, long long n_rays, const int32_t* rays, const long long* row_ptr, const RayInfo* ray_z,
                         int32_t* lam, const long long* T, const MsgParams& mp, const WalkParams& wp, cudaStream_t s) {
    if constexpr (k < kNumShort) {
        if (cls == k) {
            constexpr int G = class_G(k), K = class_K(k);
            const unsigned grid = blocks_for((n_rays + 32 / G - 1) / (32 / G) * 32, 256);
            ray_msg_walk_kernel<G, K, M, AVG><<<grid, 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, lam, T, mp, wp);
            return;
        }
        launch_walk_class_k<M, AVG, k + 1>(cls, n_rays, rays, row_ptr, ray_z, lam, T, mp, wp, s);
    }
}

template <int M, bool AVG>
void launch_ray_messages_walk_m(int cls, long long n_rays, const int32_t* rays, const long long* row_ptr,
                                const RayInfo* ray_z, int32_t* lam, const long long* T, const MsgParams& mp,
                                const WalkParams& wp, float* scratch, long long scratch_per_warp, int n_warps_long,
                                cudaStream_t s) {
    if (cls < kNumShort) {
        launch_walk_class_k<M, AVG, 0>(cls, n_rays, rays, row_ptr, ray_z, lam, T, mp, wp, s);
    } else {
        const unsigned g = blocks_for((long long)n_warps_long * 32, 256);
        ray_msg_long_kernel<M, AVG, true><<<g, 256, 0, s>>>(n_rays, rays, row_ptr, ray_z, nullptr, nullptr, lam, T, mp,
                                                            scratch, scratch_per_warp, wp);
    }
}

template <int M>
void launch_staged_m(long long n_stages, const Stage* stages, const long long* row_ptr, const RayInfo* info,
                     const int32_t* vid, const float* lnu, int32_t* lam, const long long* T, const MsgParams& mp,
                     cudaStream_t s) {
    // the attribute is per device: set it on every launch (cheap host call; the staged kernel is
    // an ablation, not the default path)
    cudaFuncSetAttribute(ray_msg_staged_kernel<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStageSmem);
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long grid = std::min<long long>(n_stages, (long long)kStageCtas * std::max(sms, 1));
    ray_msg_staged_kernel<M><<<(unsigned)grid, kStageThreads, kStageSmem, s>>>(n_stages, stages, row_ptr, info, vid,
                                                                              lnu, lam, T, mp);
}

}  // namespace

namespace {
__global__ void class_desc_kernel(long long n, const int32_t* __restrict__ rays, const long long* __restrict__ row_ptr,
                                  const RayInfo* __restrict__ info, int4* desc) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = rays[i];
    desc[i] = make_int4((int)row_ptr[r], info[r].n, info[r].frame, r);
}
}  // namespace

void launch_class_desc(long long n, const int32_t* rays, const long long* row_ptr, const RayInfo* info, int4* desc,
                       cudaStream_t s) {
    if (n == 0) return;
    class_desc_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, rays, row_ptr, info, desc);
}

void launch_ray_messages(int cls, long long n_rays, const int32_t* rays, const int4* desc, const long long* row_ptr,
                         const RayInfo* ray_z, const int32_t* vid, const float* lnu, int32_t* lam,
                         const long long* T, const MsgParams& mp, float* scratch, long long scratch_per_warp,
                         int n_warps_long, int math, cudaStream_t s) {
    if (n_rays == 0) return;
    if (mp.qbar)  // keyframe-average mode (math level 1)
        launch_ray_messages_m<1, true>(cls, n_rays, rays, desc, row_ptr, ray_z, vid, lnu, lam, T, mp, scratch,
                                       scratch_per_warp, n_warps_long, s);
    else if (math == 0)
        launch_ray_messages_m<0, false>(cls, n_rays, rays, desc, row_ptr, ray_z, vid, lnu, lam, T, mp, scratch,
                                        scratch_per_warp, n_warps_long, s);
    else
        launch_ray_messages_m<1, false>(cls, n_rays, rays, desc, row_ptr, ray_z, vid, lnu, lam, T, mp, scratch,
                                        scratch_per_warp, n_warps_long, s);
}

void launch_ray_messages_walk(int cls, long long n_rays, const int32_t* rays, const long long* row_ptr,
                              const RayInfo* ray_z, int32_t* lam, const long long* T, const MsgParams& mp,
                              const WalkParams& wp, float* scratch, long long scratch_per_warp, int n_warps_long,
                              int math, cudaStream_t s) {
    if (n_rays == 0) return;
    if (mp.qbar)
        launch_ray_messages_walk_m<1, true>(cls, n_rays, rays, row_ptr, ray_z, lam, T, mp, wp, scratch,
                                            scratch_per_warp, n_warps_long, s);
    else if (math == 0)
        launch_ray_messages_walk_m<0, false>(cls, n_rays, rays, row_ptr, ray_z, lam, T, mp, wp, scratch,
                                             scratch_per_warp, n_warps_long, s);
    else
        launch_ray_messages_walk_m<1, false>(cls, n_rays, rays, row_ptr, ray_z, lam, T, mp, wp, scratch,
                                             scratch_per_warp, n_warps_long, s);
}

void launch_ray_messages_staged(long long n_stages, const Stage* stages, const long long* row_ptr,
                                const RayInfo* info, const int32_t* vid, const float* lnu, int32_t* lam,
                                const long long* T, const MsgParams& mp, int math, cudaStream_t s) {
    if (n_stages == 0) return;
    if (math == 0)
        launch_staged_m<0>(n_stages, stages, row_ptr, info, vid, lnu, lam, T, mp, s);
    else
        launch_staged_m<1>(n_stages, stages, row_ptr, info, vid, lnu, lam, T, mp, s);
}

void launch_voxel_reduce(long long n_items, const int2* items, const long long* col_ptr, const int32_t* tr,
                         const int32_t* lam, long long* T, cudaStream_t s) {
    if (n_items == 0) return;
    const long long cap = (long long)dev_cfg().sms * 64;
    long long warps = n_items < cap ? n_items : cap;
    voxel_reduce_kernel<<<blocks_for(warps * 32, 256), 256, 0, s>>>(n_items, items, col_ptr, tr, lam, T);
}

template <int MODE, bool PAD>
void launch_tile_reduce_t(long long n_items, const int2* items, const long long* tile_ptr, const Run* runs,
                          const int32_t* lam, int per_item, void* out, long long n_out, unsigned* next,
                          const int32_t* tile_map, long long chk_lam, long long chk_out_tiles, int n_tiles,
                          cudaStream_t s) {
    constexpr int smem = (MODE == 3 ? 3 : 2) * AccLayout<PAD>::kSlots * (int)sizeof(int) + kK6Desc;
    DevCfg& dc = dev_cfg();
    if (!dc.k6[MODE][PAD]) {
        cudaFuncSetAttribute(tile_reduce_kernel<MODE, PAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        dc.k6[MODE][PAD] = true;
    }
    const long long grid = n_items < (long long)dc.sms ? n_items : (long long)dc.sms;
    if (next) cudaMemsetAsync(next, 0, sizeof(unsigned), s);
    tile_reduce_kernel<MODE, PAD><<<(unsigned)grid, kK6Threads, smem, s>>>(n_items, items, tile_ptr, runs, lam,
                                                                              per_item, out, n_out, next, tile_map,
                                                                              chk_lam, chk_out_tiles, n_tiles);
}

void launch_tile_reduce(long long n_items, const int2* items, const long long* tile_ptr, const Run* runs,
                        const int32_t* lam, int per_item, long long* T, unsigned* next, bool pad,
                        const int32_t* tile_map, long long chk_lam, long long chk_out_tiles, int n_tiles,
                        cudaStream_t s) {
    if (n_items == 0) return;
    if (pad)
        launch_tile_reduce_t<0, true>(n_items, items, tile_ptr, runs, lam, per_item, T, 0, next, tile_map, chk_lam,
                                      chk_out_tiles, n_tiles, s);
    else
        launch_tile_reduce_t<0, false>(n_items, items, tile_ptr, runs, lam, per_item, T, 0, next, tile_map, chk_lam,
                                       chk_out_tiles, n_tiles, s);
}

void launch_block_kf(int pass, long long n_blocks, const int4* blocks, const long long* row_ptr, const RayInfo* ray_z,
                     const int32_t* vid, const int32_t* lam, long long* sums, long long n_slots, long long VI,
                     unsigned* next, long long chk_lam, cudaStream_t s) {
    if (n_blocks == 0) return;
    DevCfg& dc = dev_cfg();
    const long long cap = (long long)dc.sms * kBlkMinCtas;
    const unsigned grid = (unsigned)(n_blocks < cap ? n_blocks : cap);
    cudaMemsetAsync(next, 0, sizeof(unsigned), s);
    if (pass == 0)
        block_kf_kernel<2><<<grid, kBlkThreads, 0, s>>>(n_blocks, blocks, row_ptr, ray_z, vid, lam, sums, n_slots, VI,
                                                        next, chk_lam);
    else
        block_kf_kernel<3><<<grid, kBlkThreads, 0, s>>>(n_blocks, blocks, row_ptr, ray_z, vid, lam, sums, n_slots, VI,
                                                        next, chk_lam);
}

void launch_block_reduce(long long n_blocks, const int4* blocks, const long long* row_ptr, const RayInfo* ray_z,
                         const int32_t* vid, const int32_t* lam, long long* T, unsigned* next,
                         unsigned long long* stats, const int32_t* tile_map, int max_probe, long long chk_lam,
                         long long chk_out, cudaStream_t s) {
    if (n_blocks == 0) return;
    DevCfg& dc = dev_cfg();
    const long long cap = (long long)dc.sms * kBlkMinCtas;
    const long long grid = n_blocks < cap ? n_blocks : cap;
    cudaMemsetAsync(next, 0, sizeof(unsigned), s);
    block_reduce_kernel<kBlkTableLog><<<(unsigned)grid, kBlkThreads, 0, s>>>(n_blocks, blocks, row_ptr, ray_z, vid, lam, T,
                                                                              next, stats, tile_map, max_probe, chk_lam, chk_out);
}

void launch_kf_sums(int pass, long long n_items, const int2* items, const long long* bucket_ptr, const Run* runs,
                    const int32_t* lam, int per_item, long long* sums, long long n_slots, unsigned* next,
                    long long chk_lam, cudaStream_t s) {
    if (n_items == 0) return;
    if (pass == 0)
        launch_tile_reduce_t<2, (bool)MRF_K6_STRIDES>(n_items, items, bucket_ptr, runs, lam, per_item, sums, n_slots,
                                                      next, nullptr, chk_lam, n_slots >> kTileShift, 1 << 30, s);
    else
        launch_tile_reduce_t<3, false>(n_items, items, bucket_ptr, runs, lam, per_item, sums, n_slots, next, nullptr,
                                       chk_lam, n_slots >> kTileShift, 1 << 30, s);
}

// between the passes: M (min |q|) -> the scale a (nats, float, in place) per (frame, slot):
// |lambda_min| when the slot's messages have one sign, -1 when mixed (or none)
__global__ void kf_scale_kernel(long long n, const unsigned long long* __restrict__ N, unsigned* M) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned long long cn = N[i];
    const bool one_sign = cn != 0 && ((cn & 0xffffffffull) == 0 || (cn >> 32) == 0);
    const float a = one_sign ? (float)((double)M[i] * kQInvD) : -1.f;
    M[i] = __float_as_uint(a);
}

void launch_kf_scale(long long n_slots, long long first, long long count, long long* sums, cudaStream_t s) {
    if (count <= 0) return;
    kf_scale_kernel<<<blocks_for(count, 256), 256, 0, s>>>(
        count, reinterpret_cast<const unsigned long long*>(sums) + first,
        reinterpret_cast<unsigned*>(sums + 2 * n_slots) + first);
}

// world > 1: the all-reduced sums of the touched tiles (compact order) back to their tiles
__global__ void tile_scatter_kernel(long long n, const int32_t* __restrict__ tile_of, const longlong2* __restrict__ src,
                                    longlong2* dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // pair index
    if (i >= n) return;
    constexpr int kPairs = kTileSlots / 2;
    const long long ci = i / kPairs;
    MRF_ASSERT(__ldg(tile_of + ci) >= 0);
    dst[(long long)__ldg(tile_of + ci) * kPairs + (i - ci * kPairs)] = src[i];
}

void launch_tile_scatter(long long n_tiles, const int32_t* tile_of, const long long* src, long long* T, cudaStream_t s) {
    if (n_tiles == 0) return;
    const long long n = n_tiles * (kTileSlots / 2);
    tile_scatter_kernel<<<blocks_for(n, 256), 256, 0, s>>>(n, tile_of, reinterpret_cast<const longlong2*>(src),
                                                           reinterpret_cast<longlong2*>(T));
}

// Keyframe averages -> quantised log-odds per (frame, slot) and their sum per slot (thread per
// slot, frames in order: T is an exact integer sum).  sums = [N | D | A] per (frame, slot).
__global__ void kf_finalize_kernel(long long F, long long VI, const unsigned long long* __restrict__ N,
                                   const long long* __restrict__ D, const float* __restrict__ A, int32_t* qbar,
                                   long long* T) {
    const long long v = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= VI) return;
    long long t = 0;
    for (long long f = 0; f < F; ++f) {
        const long long k = f * VI + v;
        const unsigned long long cn = N[k];
        int qb = 0;
        if (cn) {
            const double np = (double)(cn & 0xffffffffull), nn = (double)(cn >> 32);
            const double d = (double)D[k] * kKfFixInv;
            double lb;
            if (np > 0.0 && nn > 0.0) {  // mixed signs: sum mu(1) = n_pos - D, sum mu(0) = n_neg + D
                lb = log(np - d) - log(nn + d);
            } else {  // one sign: S = s(a) d, ln s(a) = -a - ln(1 + e^-a)
                const double a = (double)A[k];
                const double ls = -a - log1p(exp(-a)) + log(d);
                lb = np > 0.0 ? log(np - exp(ls)) - ls : ls - log(nn - exp(ls));
            }
            lb = fmin(fmax(lb, -(double)kLambdaClip), (double)kLambdaClip);
            qb = lb >= (double)kLambdaClip ? 0x7fffffff : (int)__double2ll_rn(lb * (double)kQScale);
        }
        qbar[k] = qb;
        t += qb;
    }
    T[v] = t;
}

void launch_kf_finalize(long long F, long long VI, const long long* sums, int32_t* qbar, long long* T, cudaStream_t s) {
    if (VI == 0) return;
    const long long n = F * VI;
    kf_finalize_kernel<<<(unsigned)((VI + 255) / 256), 256, 0, s>>>(
        F, VI, reinterpret_cast<const unsigned long long*>(sums), sums + n,
        reinterpret_cast<const float*>(sums + 2 * n), qbar, T);
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
