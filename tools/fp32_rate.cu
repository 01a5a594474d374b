// fp32_rate.cu -- FP32 pipe throughput by instruction form on this GPU
// (the Jacobi rounds use 3-register FFMA/FMUL/FADD; the FMA probe of the
// bench uses the immediate form).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp32_rate tools/fp32_rate.cu
#include <cstdio>

template <int KIND>
__global__ void __launch_bounds__(512) k(const float *in, float *out, int iters) {
    float a[8];
    const float b = in[threadIdx.x & 63], c = in[64 + (threadIdx.x & 63)];
#pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = threadIdx.x + u;
    unsigned long long p[8], B = 0, Cc = 0;
    asm("mov.b64 %0, {%1,%2};" : "=l"(B) : "f"(b), "f"(c));
    asm("mov.b64 %0, {%1,%2};" : "=l"(Cc) : "f"(c), "f"(b));
#pragma unroll
    for (int u = 0; u < 8; ++u) asm("mov.b64 %0, {%1,%2};" : "=l"(p[u]) : "f"(a[u]), "f"(a[u] + 1.f));
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (KIND == 0) a[u] = fmaf(a[u], b, c);                 // FFMA 3-reg
                if (KIND == 1) a[u] = fmaf(a[u], 0.999999f, 1e-7f);     // FFMA imm
                if (KIND == 2) a[u] = a[u] * b;                         // FMUL
                if (KIND == 3) a[u] = a[u] + b;                         // FADD
                if (KIND == 4) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(p[u]) : "l"(B), "l"(Cc));
            }
    }
    float s = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        float x, y;
        asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(p[u]));
        s += a[u] + x + y;
    }
    if (s == -1.f) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *in, *out;
    cudaMalloc(&in, 1024);
    cudaMalloc(&out, 64);
    float h[128];
    for (int i = 0; i < 128; ++i) h[i] = i < 64 ? 0.9999f : 1e-7f;
    cudaMemcpy(in, h, 512, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000, blocks = sms * 4, threads = 512;
    const char *names[5] = {"FFMA 3-reg", "FFMA imm", "FMUL 3-reg", "FADD 3-reg", "FFMA2 (x2 lanes)"};
    for (int kind = 0; kind < 5; ++kind) {
        auto launch = [&] {
            if (kind == 0) k<0><<<blocks, threads>>>(in, out, iters);
            if (kind == 1) k<1><<<blocks, threads>>>(in, out, iters);
            if (kind == 2) k<2><<<blocks, threads>>>(in, out, iters);
            if (kind == 3) k<3><<<blocks, threads>>>(in, out, iters);
            if (kind == 4) k<4><<<blocks, threads>>>(in, out, iters);
        };
        launch();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 32.0 * iters * threads * blocks * (kind == 4 ? 2 : 1);
        printf("%-18s %8.1f G lane-ops/s  (%5.1f TFLOP/s as FMA)\n", names[kind], ops / ms / 1e6,
               2 * ops / ms / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
