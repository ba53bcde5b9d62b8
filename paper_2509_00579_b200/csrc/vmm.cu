// vmm.cu — paged physical memory behind contiguous arena addresses.
//
// The paged cache (PAPER.md:276, :490 -- vLLM-style block tables) is built on
// the CUDA virtual memory API: every arena reserves a large virtual range once
// and maps fixed-size physical pages into it as it grows.  Physical pages come
// from a shared pool and go back to it when an arena is compacted or freed, so
// many sequences share one budget without per-sequence maximum reservations
// or copies on growth, while every kernel still sees one contiguous arena
// (u32 offsets, TMA extents) and the device page table plays the block table.
// Driver entry points are resolved through cudaGetDriverEntryPoint (the
// library links only libcudart).
#include <cuda.h>
#include <mutex>

#include "common.cuh"

namespace {

struct Vmm {
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    bool ok = false;
};

Vmm &vmm() {
    static Vmm v;
    static std::once_flag once;
    std::call_once(once, [] {
        auto get = [](const char *name, void **fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn != nullptr;
        };
        v.ok = get("cuMemAddressReserve", (void **)&v.reserve) &&
               get("cuMemAddressFree", (void **)&v.addr_free) &&
               get("cuMemCreate", (void **)&v.create) &&
               get("cuMemRelease", (void **)&v.release) && get("cuMemMap", (void **)&v.map) &&
               get("cuMemUnmap", (void **)&v.unmap) &&
               get("cuMemSetAccess", (void **)&v.set_access) &&
               get("cuMemGetAllocationGranularity", (void **)&v.granularity);
    });
    return v;
}

CUmemAllocationProp prop_for(int device) {
    CUmemAllocationProp p = {};
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = device;
    return p;
}

int drv_fail(CUresult r, const char *what) {
    if (r == CUDA_ERROR_OUT_OF_MEMORY) return kvc_fail(KVC_ERR_ARENA_FULL, what);
    return kvc_fail(KVC_ERR_CUDA, what);
}

}  // namespace

extern "C" int kvc_vmm_granularity(int device, size_t *bytes) {
    Vmm &v = vmm();
    if (!v.ok) return kvc_fail(KVC_ERR_CUDA, "CUDA virtual memory API unavailable");
    CUmemAllocationProp p = prop_for(device);
    CUresult r = v.granularity(bytes, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
    return r == CUDA_SUCCESS ? KVC_OK : drv_fail(r, "cuMemGetAllocationGranularity");
}

extern "C" int kvc_vmm_reserve(size_t bytes, uint64_t *va) {
    Vmm &v = vmm();
    if (!v.ok) return kvc_fail(KVC_ERR_CUDA, "CUDA virtual memory API unavailable");
    CUdeviceptr p = 0;
    CUresult r = v.reserve(&p, bytes, 0, 0, 0);
    *va = (uint64_t)p;
    return r == CUDA_SUCCESS ? KVC_OK : drv_fail(r, "cuMemAddressReserve");
}

extern "C" int kvc_vmm_free_va(uint64_t va, size_t bytes) {
    CUresult r = vmm().addr_free((CUdeviceptr)va, bytes);
    return r == CUDA_SUCCESS ? KVC_OK : drv_fail(r, "cuMemAddressFree");
}

extern "C" int kvc_vmm_create(int device, size_t bytes, uint64_t *handle) {
    Vmm &v = vmm();
    if (!v.ok) return kvc_fail(KVC_ERR_CUDA, "CUDA virtual memory API unavailable");
    CUmemAllocationProp p = prop_for(device);
    CUmemGenericAllocationHandle h = 0;
    CUresult r = v.create(&h, bytes, &p, 0);
    *handle = (uint64_t)h;
    return r == CUDA_SUCCESS ? KVC_OK : drv_fail(r, "cuMemCreate (physical page)");
}

extern "C" int kvc_vmm_release(uint64_t handle) {
    CUresult r = vmm().release((CUmemGenericAllocationHandle)handle);
    return r == CUDA_SUCCESS ? KVC_OK : drv_fail(r, "cuMemRelease");
}

// map one physical page at va (page-aligned) and make it read/write for device
extern "C" int kvc_vmm_map(uint64_t va, size_t bytes, uint64_t handle, int device) {
    Vmm &v = vmm();
    CUresult r = v.map((CUdeviceptr)va, bytes, 0, (CUmemGenericAllocationHandle)handle, 0);
    if (r != CUDA_SUCCESS) return drv_fail(r, "cuMemMap");
    CUmemAccessDesc a = {};
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = device;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = v.set_access((CUdeviceptr)va, bytes, &a, 1);
    return r == CUDA_SUCCESS ? KVC_OK : drv_fail(r, "cuMemSetAccess");
}

extern "C" int kvc_vmm_unmap(uint64_t va, size_t bytes) {
    CUresult r = vmm().unmap((CUdeviceptr)va, bytes);
    return r == CUDA_SUCCESS ? KVC_OK : drv_fail(r, "cuMemUnmap");
}
