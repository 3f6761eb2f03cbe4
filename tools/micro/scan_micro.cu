// Floor of the residual scan: 2M rows x 3 float32 (cur, base), DRAM-cold.
//   V0 float4 streaming read of both arrays (bandwidth floor)
//   V1 the scan's access pattern: 8 rows per thread (stride-3 float loads),
//      fp32 max|r| + gate, ballot -> bitmap word per warp-item
//   V2 V1 + one global atomicMax per block
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scan_micro scan_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void v0(const float4* c, const float4* b, int64_t n4, float* out) {
    float acc = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 x = c[i], y = b[i];
        acc += fabsf(x.x - y.x) + fabsf(x.y - y.y) + fabsf(x.z - y.z) + fabsf(x.w - y.w);
    }
    if (acc == 12345.f) out[blockIdx.x] = acc;
}

template <bool ATOM>
__global__ void __launch_bounds__(256) v1(const float* c, const float* b, int64_t rows, unsigned* bitmap,
                                          unsigned* gmax) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t r0 = (int64_t)blockIdx.x * 2048;
    float cv[8][3], bv[8][3];
#pragma unroll
    for (int it = 0; it < 8; ++it) {
        const int64_t row = r0 + it * 256 + threadIdx.x;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            cv[it][d] = row < rows ? c[row * 3 + d] : 0.f;
            bv[it][d] = row < rows ? b[row * 3 + d] : 0.f;
        }
    }
    unsigned mx = 0;
#pragma unroll
    for (int it = 0; it < 8; ++it) {
        float rm = 0.f;
#pragma unroll
        for (int d = 0; d < 3; ++d) rm = fmaxf(rm, fabsf(cv[it][d] - bv[it][d]));
        mx = max(mx, __float_as_uint(rm));
        const unsigned bal = __ballot_sync(0xffffffffu, rm >= 1e-3f);
        if (lane == 0) bitmap[blockIdx.x * 64 + it * 8 + warp] = bal;
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (ATOM && lane == 0) atomicMax(gmax, mx);
}

int main() {
    const int64_t rows = 2000000, n = rows * 3;
    float *c, *b, *out;
    unsigned *bm, *gm;
    char* flush;
    cudaMalloc(&c, n * 4); cudaMalloc(&b, n * 4); cudaMalloc(&out, 1 << 20);
    cudaMalloc(&bm, (rows / 2048 + 1) * 64 * 4); cudaMalloc(&gm, 4);
    cudaMalloc(&flush, 512 << 20);
    cudaMemset(c, 0, n * 4); cudaMemset(b, 0, n * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = (int)((rows + 2047) / 2048);
    for (int cold = 0; cold < 2; ++cold)
        for (int v = 0; v < 3; ++v) {
            float tot = 0.f;
            for (int rep = 0; rep < 25; ++rep) {
                if (cold) cudaMemsetAsync(flush, rep, 512 << 20);
                cudaEventRecord(e0);
                if (v == 0) v0<<<148 * 8, 256>>>((const float4*)c, (const float4*)b, n / 4, out);
                else if (v == 1) v1<false><<<blocks, 256>>>(c, b, rows, bm, gm);
                else v1<true><<<blocks, 256>>>(c, b, rows, bm, gm);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep >= 5) tot += ms;
            }
            printf("%s V%d: %.2f us (48 MB read)\n", cold ? "cold" : "warm", v, tot / 20 * 1e3);
        }
    return 0;
}
