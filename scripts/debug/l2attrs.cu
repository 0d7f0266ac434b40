#include <cstdio>
#include <cuda_runtime.h>
int main() {
    int v;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxPersistingL2CacheSize, 0); printf("MaxPersistingL2CacheSize %d\n", v);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxAccessPolicyWindowSize, 0); printf("MaxAccessPolicyWindowSize %d\n", v);
    cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, 0); printf("L2CacheSize %d\n", v);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0); printf("MaxSmemOptin %d\n", v);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, 0); printf("MaxSmemPerSM %d\n", v);
    return 0;
}
