// peer.cu — cross-GPU merge over peer memory (SURVEY.md §8(f) 4, P2P variant of the fused
// flush + all-reduce): the stand-alone push kernel and the CUDA IPC plumbing
// that maps every rank's merged buffer into each process.
#include <string.h>

#include <algorithm>

#include "internal.cuh"
#include "peer.cuh"
#include "scan.cuh"

using namespace skb;

namespace {

__global__ void __launch_bounds__(512) k_peer_push(const __grid_constant__ PeerPush pp) {
    peer_push_range(pp, uint64_t(blockIdx.x) * blockDim.x + threadIdx.x, uint64_t(gridDim.x) * blockDim.x);
}

// all-gather half of the owner-mode merge: this rank's merged buffer receives every other
// owner's range (P2P reads that bypass caches: the owners' buffers were written by remote red)
__global__ void __launch_bounds__(512) k_peer_gather(const __grid_constant__ PeerPush pp) {
    const uint64_t pairs = pp.total >> 1;
    int64_t *own = pp.dst[pp.rank];
    for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < pairs; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t o = owner_of(2 * e, pp.total, pp.peers);
        if (o == pp.rank) continue;
        reinterpret_cast<longlong2 *>(own)[e] = __ldcv(reinterpret_cast<const longlong2 *>(pp.dst[o]) + e);
    }
    if ((pp.total & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const uint32_t o = owner_of(pp.total - 1, pp.total, pp.peers);
        if (o != pp.rank) own[pp.total - 1] = __ldcv(reinterpret_cast<const long long *>(pp.dst[o]) + pp.total - 1);
    }
}

}  // namespace

namespace skb {

sk_status peer_push_launch(const PeerPush &pp, cudaStream_t stream) {
    if (!pp.peers || !pp.n) return SK_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t pairs = (pp.n + 1) / 2;
    const unsigned grid = (unsigned)std::min<uint64_t>(uint64_t(sms) * 4, (pairs + 511) / 512);
    k_peer_push<<<std::max(1u, grid), 512, 0, stream>>>(pp);
    SKB_CUDA(cudaGetLastError());
    count_launch();
    return SK_OK;
}

sk_status peer_gather_launch(const PeerPush &pp, cudaStream_t stream) {
    if (!pp.peers || !pp.total || pp.peers == 1) return SK_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t pairs = (pp.total + 1) / 2;
    const unsigned grid = (unsigned)std::min<uint64_t>(uint64_t(sms) * 4, (pairs + 511) / 512);
    k_peer_gather<<<std::max(1u, grid), 512, 0, stream>>>(pp);
    SKB_CUDA(cudaGetLastError());
    count_launch();
    return SK_OK;
}

}  // namespace skb

static_assert(sizeof(cudaIpcMemHandle_t) == SK_IPC_HANDLE_BYTES, "IPC handle size");

extern "C" sk_status sk_ipc_alloc(uint64_t bytes, int device, void **dev_ptr, unsigned char *handle) {
    if (!dev_ptr || !handle || !bytes) return fail(SK_EINVAL, "sk_ipc_alloc: NULL argument or zero size");
    int prev = 0;
    cudaGetDevice(&prev);
    SKB_CUDA(cudaSetDevice(device));
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) { cudaSetDevice(prev); return e == cudaErrorMemoryAllocation ? fail(SK_ENOMEM, "sk_ipc_alloc: %llu bytes", (unsigned long long)bytes) : cuda_fail(e, "cudaMalloc"); }
    e = cudaMemset(p, 0, bytes);
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    cudaSetDevice(prev);
    if (e != cudaSuccess) { cudaFree(p); return cuda_fail(e, "cudaIpcGetMemHandle"); }
    memcpy(handle, &h, sizeof(h));
    *dev_ptr = p;
    return SK_OK;
}

extern "C" sk_status sk_ipc_free(void *dev_ptr) {
    if (!dev_ptr) return SK_OK;
    SKB_CUDA(cudaFree(dev_ptr));
    return SK_OK;
}

extern "C" sk_status sk_ipc_open(const unsigned char *handle, int device, void **dev_ptr) {
    if (!dev_ptr || !handle) return fail(SK_EINVAL, "sk_ipc_open: NULL argument");
    int prev = 0;
    cudaGetDevice(&prev);
    SKB_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void *p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    *dev_ptr = p;
    return SK_OK;
}

extern "C" sk_status sk_ipc_close(void *dev_ptr) {
    if (!dev_ptr) return SK_OK;
    SKB_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return SK_OK;
}
