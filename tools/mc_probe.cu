// mc_probe.cu — can this box create an NVLink multicast object (NVLS) for one GPU and run
// multimem.red on it?  Probe for SURVEY.md §8(f) 4 (fused flush + in-switch all-reduce).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/mc_probe tools/mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__global__ void k_mred(uint64_t *mc, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(mc + i), "l"((uint64_t)(i + 1)) : "memory");
}

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char *s; cuGetErrorString(r_, &s); printf("%s -> %d %s\n", #x, (int)r_, s); return 1; } } while (0)

int main() {
    cudaFree(0);
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int mc = 0, fab = 0;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    printf("multicast_supported=%d fabric_handle_supported=%d\n", mc, fab);
    if (!mc) return 0;
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1;
    size_t gran = 0;
    prop.size = 1 << 21;
    CUmemGenericAllocationHandle mch;
    CUresult rr = CUDA_ERROR_INVALID_VALUE;
    const CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE};
    for (int h = 0; h < 3 && rr != CUDA_SUCCESS; ++h) {
        prop.handleTypes = hts[h];
        CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
        prop.size = ((size_t(1) << 21) + gran - 1) / gran * gran;
        rr = cuMulticastCreate(&mch, &prop);
        const char *es; cuGetErrorString(rr, &es);
        printf("handleType=%d granularity=%zu size=%zu cuMulticastCreate -> %d %s\n", (int)hts[h], gran, prop.size, (int)rr, es);
    }
    if (rr != CUDA_SUCCESS) return 0;
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)prop.handleTypes;
    CUmemGenericAllocationHandle mem;
    CK(cuMemCreate(&mem, prop.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mem, 0, prop.size, 0));
    CUdeviceptr uc, mcp;
    CK(cuMemAddressReserve(&uc, prop.size, gran, 0, 0));
    CK(cuMemMap(uc, prop.size, 0, mem, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, prop.size, &acc, 1));
    CK(cuMemAddressReserve(&mcp, prop.size, gran, 0, 0));
    CK(cuMemMap(mcp, prop.size, 0, mch, 0));
    CK(cuMemSetAccess(mcp, prop.size, &acc, 1));
    cudaMemset((void *)uc, 0, prop.size);
    const int n = 1 << 16;
    k_mred<<<64, 256>>>((uint64_t *)mcp, n);
    k_mred<<<64, 256>>>((uint64_t *)mcp, n);
    cudaError_t e = cudaDeviceSynchronize();
    uint64_t h[4];
    cudaMemcpy(h, (void *)uc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("kernel: %s  values %llu %llu %llu %llu (expect 2 4 6 8)\n", cudaGetErrorString(e), (unsigned long long)h[0],
           (unsigned long long)h[1], (unsigned long long)h[2], (unsigned long long)h[3]);
    return 0;
}
