// scan.cu -- K2: device-wide exclusive prefix sum int32 -> int64 (count -> scan -> fill).
//
// Three passes: per-tile sums, one-block scan of the tile sums, per-tile rescan with the
// tile offset.  Used for row_ptr (ray lengths), col_ptr (voxel degrees), the K6 work list
// and the stable compaction of the K5 length classes.  Integer, so exact and deterministic.
#include "internal.cuh"

namespace mrf {
namespace {

constexpr int kThreads = 256;
constexpr int kPerThread = 8;
constexpr int kTile = kThreads * kPerThread;
constexpr unsigned kFull = 0xffffffffu;

template <int NT>
__device__ __forceinline__ long long block_exclusive_scan(long long x, long long* smem_warp, long long& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(kFull, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) smem_warp[wid] = inc;
    __syncthreads();
    constexpr int NW = NT / 32;
    if (wid == 0) {
        long long w = lane < NW ? smem_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(kFull, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NW) smem_warp[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    const long long warp_off = wid ? smem_warp[wid - 1] : 0;
    total = smem_warp[NW - 1];
    __syncthreads();
    return warp_off + inc - x;
}

__global__ void __launch_bounds__(kThreads) tile_sums_kernel(const int32_t* __restrict__ in, long long n,
                                                             long long* sums) {
    __shared__ long long sw[kThreads / 32];
    const long long base = (long long)blockIdx.x * kTile;
    long long s = 0;
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
        const long long i = base + (long long)j * kThreads + threadIdx.x;
        if (i < n) s += in[i];
    }
    long long total;
    block_exclusive_scan<kThreads>(s, sw, total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) scan_sums_kernel(long long* sums, long long nb) {
    __shared__ long long sw[32];
    const long long per = (nb + 1023) / 1024;
    const long long b0 = threadIdx.x * per;
    long long s = 0;
    for (long long i = b0; i < b0 + per && i < nb; ++i) s += sums[i];
    long long total;
    long long run = block_exclusive_scan<1024>(s, sw, total);
    for (long long i = b0; i < b0 + per && i < nb; ++i) {
        const long long x = sums[i];
        sums[i] = run;
        run += x;
    }
}

__global__ void __launch_bounds__(kThreads) tile_scan_kernel(const int32_t* __restrict__ in, long long n,
                                                             const long long* __restrict__ sums, long long offset,
                                                             const long long* doff, long long* out) {
    if (doff) offset += *doff;  // device-resident base (it may be out[0] itself: rewritten unchanged)
    __shared__ long long sw[kThreads / 32];
    const long long base = (long long)blockIdx.x * kTile + (long long)threadIdx.x * kPerThread;
    int v[kPerThread];
    long long s = 0;
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
        const long long i = base + j;
        v[j] = i < n ? in[i] : 0;
        s += v[j];
    }
    long long total;
    long long run = block_exclusive_scan<kThreads>(s, sw, total) + sums[blockIdx.x] + offset;
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
        const long long i = base + j;
        if (i < n) out[i] = run;
        run += v[j];
        if (i == n - 1) out[n] = run;
    }
}

__global__ void write_one_kernel(long long* out, long long value) { *out = value; }

}  // namespace

long long scan_scratch_elems(long long n) { return (n + kTile - 1) / kTile + 1; }

void launch_exclusive_scan(const int32_t* in, long long* out, long long n, long long offset, long long* scratch,
                           cudaStream_t s) {
    if (n <= 0) {
        write_one_kernel<<<1, 1, 0, s>>>(out, offset);
        return;
    }
    const long long nb = (n + kTile - 1) / kTile;
    tile_sums_kernel<<<(unsigned)nb, kThreads, 0, s>>>(in, n, scratch);
    scan_sums_kernel<<<1, 1024, 0, s>>>(scratch, nb);
    tile_scan_kernel<<<(unsigned)nb, kThreads, 0, s>>>(in, n, scratch, offset, nullptr, out);
}

void launch_exclusive_scan_dev(const int32_t* in, long long* out, long long n, const long long* doff,
                               long long* scratch, cudaStream_t s) {
    if (n <= 0) return;  // out[0] is *doff already (or must be written by the caller)
    const long long nb = (n + kTile - 1) / kTile;
    tile_sums_kernel<<<(unsigned)nb, kThreads, 0, s>>>(in, n, scratch);
    scan_sums_kernel<<<1, 1024, 0, s>>>(scratch, nb);
    tile_scan_kernel<<<(unsigned)nb, kThreads, 0, s>>>(in, n, scratch, 0, doff, out);
}

}  // namespace mrf
