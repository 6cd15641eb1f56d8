// Exhaustive-ish check that the reciprocal + one FMA correction quotient equals the correctly
// rounded fp64 division for the integer operands the DDA walker divides (num, den < 2^31):
//   y = RN(1/den), q = RN(num y), r = num - den q (exact by FMA), t = RN(q + r y)  ==  RN(num/den)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/div_check scripts/div_check.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}

__global__ void check(unsigned long long seed, long long n, unsigned long long* bad, unsigned long long* example) {
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long nb = 0;
    for (long long i = i0; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long h = mix(seed + (unsigned long long)i);
        unsigned den = (unsigned)(h & 0x7fffffffu);
        const int mode = (int)((h >> 62) & 3);
        if (mode == 0) den &= 0xffffu;      // small denominators
        if (den == 0) den = 1;
        unsigned num = (unsigned)((h >> 31) & 0x7fffffffu) % (den + 65536u);  // num < den + 2^16, as in the walk
        if (mode == 1) num = den - 1 - (num % (den > 1 ? den - 1 : 1));
        const double a = (double)num, b = (double)den;
        const double exact = __ddiv_rn(a, b);
        const double y = __drcp_rn(b);
        const double q = __dmul_rn(a, y);
        const double r = __fma_rn(-q, b, a);
        const double t = __fma_rn(r, y, q);
        if (t != exact) {
            ++nb;
            example[0] = num;
            example[1] = den;
        }
    }
    if (nb) atomicAdd(bad, nb);
}

int main() {
    unsigned long long *bad, *ex;
    cudaMallocManaged(&bad, 8);
    cudaMallocManaged(&ex, 16);
    *bad = 0;
    const long long n = 1LL << 36;  // 6.9e10 samples
    for (int s = 0; s < 4; ++s) {
        check<<<148 * 16, 256>>>(0x9e3779b97f4a7c15ULL * (s + 1), n / 4, bad, ex);
        cudaDeviceSynchronize();
    }
    printf("samples %lld mismatches %llu (last num %llu den %llu)\n", n, *bad, ex[0], ex[1]);
    return 0;
}
