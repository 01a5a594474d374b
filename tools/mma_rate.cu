// mma_rate.cu -- measured throughput of the legacy warp-level tensor path
// (mma.sync) on this GPU, to size a tensor-core Jacobi update.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_rate tools/mma_rate.cu
#include <cstdio>

template <int KIND>
__global__ void __launch_bounds__(256) mma_loop(float *out, int iters) {
    float d[8][4];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) d[c][r] = 0.f;
    unsigned a0 = threadIdx.x, a1 = threadIdx.x * 3, a2 = threadIdx.x * 5, a3 = threadIdx.x * 7;
    unsigned b0 = threadIdx.x * 11, b1 = threadIdx.x * 13;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            if (KIND == 0) {  // tf32 m16n8k8
                asm volatile(
                    "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                    : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                    : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            } else if (KIND == 1) {  // bf16 m16n8k16
                asm volatile(
                    "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                    : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                    : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
            }
        }
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
        for (int r = 0; r < 4; ++r) s += d[c][r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) dmma_loop(double *out, int iters) {
    double d[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = 0.0;
    double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[c][0]), "+d"(d[c][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *o;
    cudaMalloc(&o, 1 << 24);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int blocks_per_sm = 1; blocks_per_sm <= 4; blocks_per_sm *= 2) {
        const int grid = sms * blocks_per_sm;
        const double warps = grid * 8.0;
        float ms;
        // tf32: 16*8*8 MACs per mma
        mma_loop<0><<<grid, 256>>>(o, iters);
        cudaEventRecord(a);
        mma_loop<0><<<grid, 256>>>(o, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("tf32 mma.sync m16n8k8  %d CTA/SM: %.1f TFLOP/s\n", blocks_per_sm,
               warps * iters * 8 * 16 * 8 * 8 * 2 / ms / 1e9);
        mma_loop<1><<<grid, 256>>>(o, iters);
        cudaEventRecord(a);
        mma_loop<1><<<grid, 256>>>(o, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("bf16 mma.sync m16n8k16 %d CTA/SM: %.1f TFLOP/s\n", blocks_per_sm,
               warps * iters * 8 * 16 * 8 * 16 * 2 / ms / 1e9);
        dmma_loop<<<grid, 256>>>((double *)o, iters);
        cudaEventRecord(a);
        dmma_loop<<<grid, 256>>>((double *)o, iters);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("f64 mma.sync m8n8k4    %d CTA/SM: %.1f TFLOP/s\n", blocks_per_sm,
               warps * iters * 8 * 8 * 8 * 4 * 2 / ms / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
