// Host tier allocation for UVA zero-copy reads (the uncached rows of Legion's
// unified cache, read by K2/K4 over PCIe).
//
// gc_host_alloc_numa maps host memory through the CUDA VMM API
// (cuMemCreate with CU_MEM_LOCATION_TYPE_HOST_NUMA): the GPU page tables then map the
// host tier with the allocation granularity (2 MB pages) instead of the 4 KB pages of
// cudaHostAlloc/cudaHostRegister, which multiplies the GPU TLB reach over a
// tens-of-GB table read at random. The same virtual address is valid on the CPU.
// Driver entry points come from cudaGetDriverEntryPoint, so the library has no
// link-time dependency on libcuda (it still loads on a CPU-only host).
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "gc_common.cuh"

namespace gc {

struct DriverVmm {
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemSetAccess) access = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemAddressFree) free_va = nullptr;
    decltype(&cuMemRetainAllocationHandle) retain = nullptr;
    decltype(&cuMemGetAddressRange) address_range = nullptr;
    bool ok = false;
};

static DriverVmm& vmm() {
    static DriverVmm d;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn != nullptr;
        };
        d.ok = get("cuMemGetAllocationGranularity", (void**)&d.granularity) && get("cuMemCreate", (void**)&d.create) &&
               get("cuMemAddressReserve", (void**)&d.reserve) && get("cuMemMap", (void**)&d.map) &&
               get("cuMemSetAccess", (void**)&d.access) && get("cuMemUnmap", (void**)&d.unmap) &&
               get("cuMemRelease", (void**)&d.release) && get("cuMemAddressFree", (void**)&d.free_va) &&
               get("cuMemRetainAllocationHandle", (void**)&d.retain);
        if (!get("cuMemGetAddressRange", (void**)&d.address_range)) d.address_range = nullptr;
    });
    return d;
}

static int drv(CUresult r, const char* what) {
    if (r == CUDA_SUCCESS) return GC_OK;
    set_error(std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")");
    return GC_ERR_CUDA;
}

static CUmemAllocationProp host_prop(int numa_node) {
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
    prop.location.id = numa_node;
    return prop;
}

}  // namespace gc

using namespace gc;

extern "C" {

int gc_host_alloc_numa(size_t bytes, int numa_node, void** ptr, size_t* mapped_bytes) {
    GC_REQUIRE(ptr && mapped_bytes && bytes > 0, GC_ERR_VALUE, "gc_host_alloc_numa: bad arguments");
    DriverVmm& d = vmm();
    GC_REQUIRE(d.ok, GC_ERR_UNSUPPORTED, "gc_host_alloc_numa: CUDA VMM driver entry points unavailable");
    int dev = 0;
    GC_TRY(cudaGetDevice(&dev), "cudaGetDevice");
    GC_TRY(cudaFree(nullptr), "context init");  // the driver calls below need a current context
    CUmemAllocationProp prop = host_prop(numa_node);
    size_t gran = 0;
    if (int e = drv(d.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity"))
        return e;
    const size_t size = align_up(bytes, gran);
    CUmemGenericAllocationHandle h;
    if (int e = drv(d.create(&h, size, &prop, 0), "cuMemCreate(host NUMA)")) return e;
    CUdeviceptr va = 0;
    if (int e = drv(d.reserve(&va, size, gran, 0, 0), "cuMemAddressReserve")) {
        d.release(h);
        return e;
    }
    if (int e = drv(d.map(va, size, 0, h, 0), "cuMemMap")) {
        d.free_va(va, size);
        d.release(h);
        return e;
    }
    d.release(h);  // the mapping keeps the allocation alive until it is unmapped
    int ndev = 0;
    GC_TRY(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
    CUmemAccessDesc desc[GC_MAX_PEERS + 1];
    int nd = 0;
    desc[nd].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;  // CPU access through the same address
    desc[nd].location.id = numa_node;
    desc[nd++].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    for (int g = 0; g < ndev && nd < GC_MAX_PEERS + 1; ++g) {
        desc[nd].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        desc[nd].location.id = g;
        desc[nd++].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    if (int e = drv(d.access(va, size, desc, nd), "cuMemSetAccess")) {
        d.unmap(va, size);
        d.free_va(va, size);
        return e;
    }
    *ptr = reinterpret_cast<void*>(va);
    *mapped_bytes = size;
    return GC_OK;
}

// CUDA IPC of cache slabs across the clique's processes. cudaIpcOpenMemHandle maps
// the whole cudaMalloc allocation and returns its base, while torch's caching
// allocator sub-allocates tensors inside larger blocks: the exporter therefore also
// returns the tensor's offset from its allocation base (cuMemGetAddressRange), which
// the importer adds to the mapped base.
int gc_ipc_export(void* d_ptr, uint8_t* handle64, uint64_t* offset) {
    GC_REQUIRE(d_ptr && handle64 && offset, GC_ERR_VALUE, "gc_ipc_export: null argument");
    DriverVmm& d = vmm();
    GC_REQUIRE(d.address_range, GC_ERR_UNSUPPORTED, "gc_ipc_export: cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (int e = drv(d.address_range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)), "cuMemGetAddressRange"))
        return e;
    cudaIpcMemHandle_t h;
    GC_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "ipc handle size");
    memcpy(handle64, &h, 64);
    *offset = (uint64_t)(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
    return GC_OK;
}

int gc_ipc_import(const uint8_t* handle64, void** d_ptr) {
    GC_REQUIRE(handle64 && d_ptr, GC_ERR_VALUE, "gc_ipc_import: null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    GC_TRY(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    return GC_OK;
}

int gc_ipc_close(void* d_ptr) {
    GC_TRY(cudaIpcCloseMemHandle(d_ptr), "cudaIpcCloseMemHandle");
    return GC_OK;
}

int gc_host_free_numa(void* ptr, size_t mapped_bytes) {
    GC_REQUIRE(ptr, GC_ERR_VALUE, "gc_host_free_numa: null pointer");
    DriverVmm& d = vmm();
    GC_REQUIRE(d.ok, GC_ERR_UNSUPPORTED, "gc_host_free_numa: CUDA VMM driver entry points unavailable");
    const CUdeviceptr va = reinterpret_cast<CUdeviceptr>(ptr);
    if (int e = drv(d.unmap(va, mapped_bytes), "cuMemUnmap")) return e;
    return drv(d.free_va(va, mapped_bytes), "cuMemAddressFree");
}

// Small device -> host reads that must not queue behind bulk DMA: the SMs store the
// words straight into mapped pinned memory over PCIe (a window's per-batch sizes read
// while the previous window's results are still draining through the copy engine).
}  // extern "C"

namespace gc {
__global__ void k_copy_to_mapped(const uint32_t* __restrict__ src, uint32_t* dst, uint64_t words) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
    __threadfence_system();
}

// Segment pack of a padded window array (grid.y = batch): batch b's first
// (ptr[b+1] - ptr[b]) rows, each `elems` IN values, move to the packed array at row
// ptr[b] as OUT values (u32 -> u16 keeps the low 16 bits).
template <typename IN, typename OUT>
__global__ void k_pack_segments(const IN* __restrict__ src, uint64_t stride_elems, uint64_t elems,
                                const int64_t* __restrict__ ptr, OUT* __restrict__ dst) {
    const uint32_t b = blockIdx.y;
    const int64_t r0 = ptr[b];
    const uint64_t n = (uint64_t)(ptr[b + 1] - r0) * elems;
    const IN* s = src + b * stride_elems;
    OUT* d = dst + (uint64_t)r0 * elems;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        d[i] = (OUT)s[i];
}

// Offsets -> per-row counts: batch b's rows [0, ptr[b+1] - ptr[b]) of u32 offsets become
// the u8 differences s[i+1] - s[i] (a hop's per-position sample counts, <= fanout).
__global__ void k_pack_counts(const uint32_t* __restrict__ src, uint64_t stride_elems, const int64_t* __restrict__ ptr,
                              uint8_t* __restrict__ dst) {
    const uint32_t b = blockIdx.y;
    const int64_t r0 = ptr[b];
    const uint64_t n = (uint64_t)(ptr[b + 1] - r0);
    const uint32_t* s = src + b * stride_elems;
    uint8_t* d = dst + r0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        d[i] = (uint8_t)(s[i + 1] - s[i]);
}
}  // namespace gc

extern "C" {

int gc_pack_segments(const void* d_src, uint64_t src_stride_bytes, uint64_t row_bytes, const int64_t* d_ptr,
                     uint32_t num_batches, uint64_t max_rows, int mode, void* d_dst, void* stream) {
    GC_REQUIRE(mode >= 0 && mode <= 4, GC_ERR_VALUE, "gc_pack_segments: mode is 0..4");
    GC_REQUIRE(mode != 4 || row_bytes == 4, GC_ERR_VALUE, "gc_pack_segments: mode 4 takes rows of one u32 offset");
    const uint64_t in_bytes = (mode == 2 || mode == 3) ? 2 : 4;
    GC_REQUIRE(row_bytes % in_bytes == 0 && src_stride_bytes % in_bytes == 0, GC_ERR_VALUE,
               "gc_pack_segments: row and stride bytes must be multiples of the element size");
    GC_REQUIRE(num_batches <= 65535, GC_ERR_VALUE, "gc_pack_segments: at most 65535 batches");
    if (num_batches == 0 || row_bytes == 0 || max_rows == 0) return GC_OK;
    GC_REQUIRE(d_src && d_ptr && d_dst, GC_ERR_VALUE, "gc_pack_segments: null pointer");
    const uint64_t elems = row_bytes / in_bytes, stride = src_stride_bytes / in_bytes;
    uint64_t gx = (max_rows * elems + 255) / 256;
    const uint64_t cap = (uint64_t)sm_count() * 8 / num_batches + 1;  // ~8 CTAs per SM over the window
    if (gx > cap) gx = cap;
    const dim3 grid((unsigned)gx, num_batches);
    cudaStream_t s = as_stream(stream);
    switch (mode) {
        case 0:
            gc::k_pack_segments<uint32_t, uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(d_src), stride,
                                                                         elems, d_ptr, static_cast<uint32_t*>(d_dst));
            break;
        case 1:
            gc::k_pack_segments<uint32_t, uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(d_src), stride,
                                                                         elems, d_ptr, static_cast<uint16_t*>(d_dst));
            break;
        case 4:
            gc::k_pack_counts<<<grid, 256, 0, s>>>(static_cast<const uint32_t*>(d_src), stride, d_ptr,
                                                   static_cast<uint8_t*>(d_dst));
            break;
        case 2:
            gc::k_pack_segments<uint16_t, uint16_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(d_src), stride,
                                                                         elems, d_ptr, static_cast<uint16_t*>(d_dst));
            break;
        default:
            gc::k_pack_segments<uint16_t, uint32_t><<<grid, 256, 0, s>>>(static_cast<const uint16_t*>(d_src), stride,
                                                                         elems, d_ptr, static_cast<uint32_t*>(d_dst));
    }
    GC_CHECK_LAUNCH("gc_pack_segments");
    return GC_OK;
}

int gc_copy_d2h_mapped(const void* d_src, void* h_dst, uint64_t bytes, void* stream) {
    GC_REQUIRE(bytes % 4 == 0, GC_ERR_VALUE, "gc_copy_d2h_mapped: bytes must be a multiple of 4");
    if (bytes == 0) return GC_OK;
    GC_REQUIRE(d_src && h_dst, GC_ERR_VALUE, "gc_copy_d2h_mapped: null pointer");
    void* d_dst = nullptr;
    GC_TRY(cudaHostGetDevicePointer(&d_dst, h_dst, 0), "cudaHostGetDevicePointer");
    const uint64_t words = bytes / 4;
    unsigned grid = (unsigned)((words + 255) / 256);
    if (grid > 64) grid = 64;
    gc::k_copy_to_mapped<<<grid, 256, 0, as_stream(stream)>>>(static_cast<const uint32_t*>(d_src),
                                                               static_cast<uint32_t*>(d_dst), words);
    GC_CHECK_LAUNCH("gc_copy_d2h_mapped");
    return GC_OK;
}

}  // extern "C"
