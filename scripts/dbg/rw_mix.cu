// Achievable HBM bandwidth for read:write mixes (1:0, 1:1, 1:3, 0:1) with plain coalesced float4 streams.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_mix(const float4* __restrict__ a, float4* __restrict__ b, float4* __restrict__ c,
                      float4* __restrict__ d, size_t n, int nr, int nw) {
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
    float4 acc = make_float4(0, 0, 0, 0);
    for (; i < n; i += st) {
        float4 v = nr ? a[i] : make_float4(i, 0, 0, 0);
        acc.x += v.x;
        if (nw >= 1) b[i] = v;
        if (nw >= 2) c[i] = v;
        if (nw >= 3) d[i] = v;
    }
    if (nw == 0 && acc.x == -1.f) b[0] = acc;
}
int main() {
    const size_t n = (size_t)1 << 28;  // 4 GiB per array (float4 = 16 B)
    float4 *a, *b, *c, *d;
    cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMalloc(&c, n * 16); cudaMalloc(&d, n * 16);
    cudaMemset(a, 0, n * 16);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int cfg[][2] = {{1, 0}, {1, 1}, {1, 3}, {0, 1}, {1, 2}, {0, 3}};
    for (auto& q : cfg) {
        float best = 1e30f;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(e0);
            k_mix<<<sms * 8, 256>>>(a, b, c, d, n / 4, q[0], q[1]);  // 1 GiB per stream
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
        }
        const double bytes = (double)(n / 4) * 16 * (q[0] + q[1]);
        printf("read:write %d:%d  %.1f GB/s (%.3f ms)\n", q[0], q[1], bytes / best / 1e6, best);
    }
    return 0;
}
