// Micro-benchmark: why is a streaming pass over 4M (int, u64) entries slow?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void roots(long long n, int* size, unsigned long long* dsum, unsigned long long* acc,
                      int mode) {
    __shared__ unsigned long long s_cnt, s_sq;
    __shared__ int s_max;
    if (threadIdx.x == 0) { s_cnt = 0; s_sq = 0; s_max = 0; }
    __syncthreads();
    unsigned long long cnt = 0, sq = 0;
    int mx = 0;
    for (long long l = (long long)blockIdx.x * blockDim.x + threadIdx.x; l < n;
         l += (long long)gridDim.x * blockDim.x) {
        const int sz = size[l];
        if (sz) {
            const unsigned long long d = dsum[l];
            ++cnt; sq += d * d; mx = max(mx, sz);
            if (mode & 1) { size[l] = 0; dsum[l] = 0; }
        }
    }
    cnt = __reduce_add_sync(0xffffffffu, (unsigned)cnt);
    mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)mx);
    for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
    if ((threadIdx.x & 31) == 0 && (cnt || mx)) {
        atomicAdd(&s_cnt, cnt); atomicAdd(&s_sq, sq); atomicMax(&s_max, mx);
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_cnt) {
        if (mode & 2) {
            atomicAdd(acc + 0, s_cnt); atomicMax(acc + 1, (unsigned long long)s_max); atomicAdd(acc + 3, s_sq);
        } else {
            acc[8 + 3 * blockIdx.x] = s_cnt; acc[9 + 3 * blockIdx.x] = s_max; acc[10 + 3 * blockIdx.x] = s_sq;
        }
    }
}
__global__ void fill(long long n, int* size, unsigned long long* dsum) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) { size[i] = (i % 3 == 0); dsum[i] = (i % 3 == 0) ? i : 0; }
}
__global__ void hot(unsigned long long* acc, int mode) {
    if (threadIdx.x == 0) {
        if (mode == 0) atomicAdd(acc, 1ull);
        else if (mode == 1) atomicMax(acc + 1, (unsigned long long)blockIdx.x);
        else atomicAdd((unsigned*)acc + 4, 1u);
    }
}
int main() {
    long long n = 4000000;
    int* size; unsigned long long *dsum, *acc;
    cudaMalloc(&size, n * 4); cudaMalloc(&dsum, n * 8); cudaMalloc(&acc, 8 * 100000);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 4; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            fill<<<(n + 255) / 256, 256>>>(n, size, dsum);
            cudaEventRecord(a);
            roots<<<1184, 256>>>(n, size, dsum, acc, mode);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep == 2) printf("roots mode %d (reset=%d global_atomics=%d): %.1f us\n", mode, mode & 1, (mode >> 1) & 1, ms * 1000);
        }
    }
    for (int mode = 0; mode < 3; ++mode) {
        for (int blocks : {1184, 10000, 100000}) {
            cudaEventRecord(a);
            hot<<<blocks, 32>>>(acc, mode);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("hot mode %d (0=add64 1=max64 2=add32) blocks %d: %.1f us = %.1f ns/atomic\n", mode, blocks, ms * 1000, ms * 1e6 / blocks);
        }
    }
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
