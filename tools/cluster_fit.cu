#include <cstdio>
__global__ void k(int *x) { extern __shared__ int s[]; s[threadIdx.x] = 1; if (x) x[0] = s[0]; }
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int C = 1; C <= 16; ++C) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = 200 * 1024; cfg.attrs = attr; cfg.numAttrs = 1;
        cfg.gridDim = dim3(C);
        int maxc = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&maxc, (void *)k, &cfg);
        printf("C=%2d max active clusters %3d -> %3d SMs  %s\n", C, maxc, maxc * C, cudaGetErrorString(e));
    }
}
