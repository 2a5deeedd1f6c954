// HBM read / copy bandwidth vs access granularity: every warp streams blocks
// of S bytes at pseudo-random block-aligned offsets of a 24 GB array, with
// 8 independent blocks in flight per warp (no dependent index loads). Tells
// what the FTCS march's plane-sized (512 B) and chunk-sized (4 KB) accesses
// can reach on this B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

template <int S>
__global__ void __launch_bounds__(256) rd(const double2* __restrict__ a, int64_t nblocks, int64_t nper, double* out,
                                          int rw, double2* __restrict__ w) {
    constexpr int V = S / 16;  // double2 per block
    constexpr int PER = V >= 32 ? V / 32 : 1;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
    double s = 0;
    for (int64_t i0 = gw * 8; i0 < nper; i0 += nw * 8) {
        double2 v[8][PER];
        int64_t base[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            base[j] = (int64_t)(mix(i0 + j) & (uint64_t)(nblocks - 1)) * V;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int e = lane + 32 * k;
                v[j][k] = e < V ? a[base[j] + e] : make_double2(0, 0);
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                const int e = lane + 32 * k;
                s += v[j][k].x;
                if (rw && e < V) w[base[j] + e] = v[j][k];
            }
    }
    if (s == 12345.678) *out = s;
}

template <int S>
void run(const double2* a, double2* w, double* out, size_t bytes, int sms) {
    const int64_t nblocks = bytes / S;
    const int64_t n = (6ll << 30) / S;
    for (int rw = 0; rw < 2; ++rw) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float ms = 0;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            rd<S><<<sms * 8, 256>>>(a, nblocks, n, out, rw, w);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        printf("%s S=%6d B: %8.1f GB/s\n", rw ? "copy" : "read", S, (double)n * S * (rw ? 2 : 1) / ms / 1e6);
    }
}

int main() {
    const size_t bytes = 16ull << 30;  // power of two: block index = hash & (n - 1)
    double2 *a, *w;
    double* out;
    cudaMalloc(&a, bytes);
    cudaMalloc(&w, bytes);
    cudaMalloc(&out, 8);
    cudaMemset(a, 0, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<128>(a, w, out, bytes, sms);
    run<256>(a, w, out, bytes, sms);
    run<512>(a, w, out, bytes, sms);
    run<1024>(a, w, out, bytes, sms);
    run<2048>(a, w, out, bytes, sms);
    run<4096>(a, w, out, bytes, sms);
    cudaDeviceSynchronize();
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
