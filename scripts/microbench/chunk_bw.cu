// Bandwidth probe for the FTCS step's access pattern (not product code):
// three FP64 columns of n_chunks x 512 slots; "step" = un[c] = u[c] + d[c]
// over whole 4-KB chunk slabs (read 8 KB, write 4 KB per chunk), visiting the
// chunks (a) in memory order, (b) in a z-major order like the march schedule
// (consecutive chunks one z layer apart: cx*cy chunks apart in memory).
// Reports GB/s at 24 B per slot (the step's algorithmic bytes).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a chunk_bw.cu -o chunk_bw
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void copy_chunks(const double2* __restrict__ u, const double2* __restrict__ d, double2* __restrict__ un,
                            const int* __restrict__ order, int n, int* ctr) {
    // warp per chunk, dynamic claims (like the march kernels)
    const int lane = threadIdx.x & 31;
    for (;;) {
        int p = 0;
        if (lane == 0) p = atomicAdd(ctr, 1);
        p = __shfl_sync(0xffffffffu, p, 0);
        if (p >= n) return;
        const long c = order[p];
        const double2* a = u + c * 256;
        const double2* b = d + c * 256;
        double2* o = un + c * 256;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double2 x = __ldcs(a + lane + 32 * i), y = __ldcs(b + lane + 32 * i);
            __stcs(o + lane + 32 * i, make_double2(x.x + y.x, x.y + y.y));
        }
    }
}

int main(int argc, char** argv) {
    const int cx = 256, cy = 256, cz = argc > 1 ? atoi(argv[1]) : 70;  // 4.59 M chunks at cz = 70
    const int n = cx * cy * cz;
    double2 *u, *d, *un;
    int *order, *ctr;
    cudaMalloc(&u, (size_t)n * 4096);
    cudaMalloc(&d, (size_t)n * 4096);
    cudaMalloc(&un, (size_t)n * 4096);
    cudaMemset(u, 0, (size_t)n * 4096);
    cudaMemset(d, 0, (size_t)n * 4096);
    cudaMalloc(&order, sizeof(int) * n);
    cudaMalloc(&ctr, sizeof(int) * 64);
    std::vector<int> seq(n), zmaj(n), zrow(n);
    for (int i = 0; i < n; ++i) seq[i] = i;
    int q = 0;  // z-block of 16 layers, 4x4 column tiles, column, z (the march schedule shape)
    for (int zb = 0; zb < cz; zb += 16)
        for (int ty = 0; ty < cy; ty += 4)
            for (int tx = 0; tx < cx; tx += 4)
                for (int y = ty; y < ty + 4; ++y)
                    for (int x = tx; x < tx + 4; ++x)
                        for (int z = zb; z < zb + 16 && z < cz; ++z) zmaj[q++] = (z * cy + y) * cx + x;
    q = 0;  // z-blocks of 16 layers, row y, layer z, x (x-runs contiguous in memory)
    for (int zb = 0; zb < cz; zb += 16)
        for (int y = 0; y < cy; ++y)
            for (int z = zb; z < zb + 16 && z < cz; ++z)
                for (int x = 0; x < cx; ++x) zrow[q++] = (z * cy + y) * cx + x;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[3] = {"memory", "z-major", "zblock-row"};
    for (int which = 0; which < 3; ++which) {
        cudaMemcpy(order, which == 2 ? zrow.data() : which ? zmaj.data() : seq.data(), sizeof(int) * n,
                   cudaMemcpyHostToDevice);
        for (int blocks_per_sm : {2, 4, 8, 16}) {
            float best = 1e30f;
            float worst = 0.f;
            for (int rep = 0; rep < 40; ++rep) {
                cudaMemset(ctr, 0, sizeof(int));
                cudaEventRecord(e0);
                copy_chunks<<<sms * blocks_per_sm, 128>>>(u, d, un, order, n, ctr);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep > 0 && ms < best) best = ms;
                if (rep > 0 && ms > worst) worst = ms;
            }
            printf("%s order, %d CTAs/SM x 4 warps: best %.3f ms (%.1f GB/s), worst %.3f ms (%.1f GB/s)\n",
                   names[which], blocks_per_sm, best, (double)n * 512 * 24 / (best * 1e-3) / 1e9, worst,
                   (double)n * 512 * 24 / (worst * 1e-3) / 1e9);
            fflush(stdout);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
