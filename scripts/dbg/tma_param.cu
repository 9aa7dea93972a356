// Standalone probe: TMA descriptors inside a large __grid_constant__ kernel-parameter struct, indexed per block.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1706_06750_b200/csrc/ptx.cuh"
using namespace kz;
struct Maps { CUtensorMap m[64]; };
__global__ void k(const __grid_constant__ Maps maps, float* out, int rank4, int c0, int c2) {
    __shared__ __align__(128) float tile[20 * 256];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&bar, 20 * 256 * 4);
        if (rank4) tma_load_4d(tile, &maps.m[blockIdx.x], c0, 1, c2, 0, &bar);
        else tma_load_3d(tile, &maps.m[blockIdx.x], -4, 3, 0, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
    out[blockIdx.x * 256 + threadIdx.x] = tile[256 * 2 + threadIdx.x];
}
int main(int argc, char** argv) {
    int W = 333, H = 257, P = 352, n = 2;
    float* L; cudaMalloc(&L, sizeof(float) * P * H * 16 * n + 4096 * 64);
    float* out; cudaMalloc(&out, 64 * 256 * 4);
    void* f = nullptr; cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    for (int rank4 = 1; rank4 < 2; ++rank4)
    for (int s = 5; s <= 5; s += 1) {
        static Maps maps;
        for (int l = 0; l < 64; ++l) {
            cuuint32_t estr[4] = {1, 1, 1, 1};
            CUresult r;
            if (rank4) {
                cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)s, (cuuint64_t)((H + s - 1) / s), (cuuint64_t)n};
                cuuint64_t str[3] = {(cuuint64_t)P * 4, (cuuint64_t)P * 4 * s, (cuuint64_t)P * H * 16 * 4};
                cuuint32_t box[4] = {256, 1, 20, 1};
                r = enc(&maps.m[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, L, dims, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            } else {
                cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)n};
                cuuint64_t str[2] = {(cuuint64_t)P * 4, (cuuint64_t)P * H * 16 * 4};
                cuuint32_t box[3] = {256, 20, 1};
                r = enc(&maps.m[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, L, dims, str, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
            if (r != CUDA_SUCCESS) { printf("encode fail rank4=%d s=%d r=%d\n", rank4, s, (int)r); return 1; }
        }
        const int c0s[] = {-8, -12, -16, 4, 8, 100, -2, 2, -10, 6};
        const int c2s[] = {3};
        for (int a : c0s) for (int c2 : c2s) {
            if (!rank4 && c2 != 3) continue;
            k<<<8, 256>>>(maps, out, rank4, a, c2);
            cudaError_t e = cudaDeviceSynchronize();
            printf("rank4=%d s=%d c0=%d c2=%d: %s\n", rank4, s, a, c2, cudaGetErrorString(e));
            if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
