// prc_nvls.cu — NVLS multicast reduction fused into the K4 / K5 epilogues (SURVEY §8(f)
// rank 3).
//
// Without it, a rank's iteration ends its forward with ncclAllReduce(images) and its
// gradient with k_unpad_add (folding the padded gradient copies into g_span),
// ncclAllReduce(g_span), ncclAllReduce(g_vert) and k_combine.  With it, one fold kernel
// reads the padded copies and the vertex part, scales, and adds the result straight into
// a multicast buffer with `multimem.red.add.f64`: NVSwitch reduces the contributions of
// every rank in the switch and delivers the sum into every rank's copy of that buffer.
// The reference does the same reduction on the host, chunk by chunk in stream order
// (pathstore.cpp:343-354).
//
// The multicast buffer is an NCCL symmetric window with the NVLS team's multimem mapping
// (NCCL 2.28 device API) when the communicator has >= 2 ranks, and a CUDA multicast object
// bound on this device alone for a single rank.  A CTA-indexed NCCL LSA barrier before the
// reductions (every rank has zeroed its copy) and after them (every rank's reductions have
// landed) orders the ranks; a single rank needs neither.  Option value 2 runs the same fold
// kernels into a plain buffer with atomics: it validates the fold's arithmetic on machines
// without multicast (the one-GPU boxes of this build refuse cuMulticastCreate with
// CUDA_ERROR_INVALID_VALUE for any handle type, scripts/micro/mc_probe.cu).
#include <cuda.h>
#include <nccl.h>
#include <nccl_device.h>

#include <string>

#include "prc_kernels.cuh"

namespace {

constexpr int kFoldGrid = 4 * 148;  // fold CTAs (and LSA barriers): 4 per SM
constexpr int kFoldTPB = 256;

__global__ void k_mc_pointer(ncclWindow_t win, ncclDevComm dc, void** out) {
    *out = ncclGetLsaMultimemPointer(win, 0, dc);
}

template <bool EMU>
__device__ __forceinline__ void mc_red_add(double* mc, double x) {
    if constexpr (EMU)
        atomicAdd(mc, x);  // validation mode: the same fold into a plain buffer
    else
        asm volatile("multimem.red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(mc), "d"(x) : "memory");
}

// out[e] (every rank) += scale * (span(e) + g_vert[e]) for e < n_out * V, where span(e)
// is the padded copies' sum at voxel e mod V (or g_span[e mod V]); plain buffers use
// g_span only.  Each CTA owns one contiguous chunk, the same on every rank, so a barrier
// per CTA index orders exactly the ranks' accesses to that chunk.
template <bool BAR, bool EMU = false>
__global__ void __launch_bounds__(kFoldTPB) k_fold_mc(const __grid_constant__ NvlsFold a,
                                                      const __grid_constant__ ncclDevComm dc) {
    const long long n = (long long)a.n_out * a.V;
    const long long chunk = (n + gridDim.x - 1) / gridDim.x;
    const long long e0 = (long long)blockIdx.x * chunk;
    const long long e1 = e0 + chunk < n ? e0 + chunk : n;
    if constexpr (BAR) {
        ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), dc, ncclTeamTagLsa(), blockIdx.x, true);
        bar.sync(ncclCoopCta(), cuda::memory_order_acquire);  // every rank zeroed its copy
        for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) mc_red_add<false>(a.mc + e, a.scale * fold_value(a, e));
        bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);  // every rank's reductions landed
    } else {
        for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) mc_red_add<EMU>(a.mc + e, a.scale * fold_value(a, e));
        if constexpr (!EMU) asm volatile("fence.proxy.alias;" ::: "memory");
        __threadfence_system();
    }
}

// CUDA driver entry points (no link-time libcuda dependency: the library also loads on
// machines without a driver, e.g. for the ABI tests).
template <class F>
F drv(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return reinterpret_cast<F>(p);
}

}  // namespace

struct NvlsState {
    int world = 1;
    bool emulate = false;  // one rank without multicast: the fold into a plain buffer
    ncclComm_t comm = nullptr;  // borrowed
    size_t bytes = 0;
    double* uc = nullptr;  // this rank's copy (unicast view)
    double* mc = nullptr;  // multicast view: reductions land in every rank's copy
    // NCCL mode (world >= 2)
    void* nccl_buf = nullptr;
    ncclWindow_t win{};
    ncclDevComm dc{};
    bool have_dc = false;
    // single-rank driver mode
    CUmemGenericAllocationHandle phys = 0, mch = 0;
    CUdeviceptr uc_va = 0, mc_va = 0;
    int device = 0;
};

static bool cu_ok(CUresult r, const char* what, std::string* err) {
    if (r == CUDA_SUCCESS) return true;
    if (err) *err = std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")";
    return false;
}

NvlsState* nvls_create(ncclComm_t comm, int world, int device, size_t n_doubles, bool emulate, std::string* err) {
    auto* s = new NvlsState();
    s->world = world;
    s->comm = comm;
    s->device = device;
    const size_t want = std::max<size_t>(n_doubles, 1) * sizeof(double);
    if (emulate && world == 1) {  // validation of the fold kernels where no multicast exists
        s->emulate = true;
        s->bytes = want;
        if (cudaMalloc(&s->uc, want) != cudaSuccess) {
            if (err) *err = "NVLS emulation: cudaMalloc";
            delete s;
            return nullptr;
        }
        s->mc = s->uc;
        return s;
    }
    if (world >= 2) {
        s->bytes = (want + 4095) / 4096 * 4096;
        ncclResult_t r = ncclMemAlloc(&s->nccl_buf, s->bytes);
        if (r == ncclSuccess) r = ncclCommWindowRegister(comm, s->nccl_buf, s->bytes, &s->win, NCCL_WIN_COLL_SYMMETRIC);
        if (r == ncclSuccess) {
            ncclDevCommRequirements req = {};
            req.lsaMultimem = true;
            req.lsaBarrierCount = kFoldGrid;
            r = ncclDevCommCreate(comm, &req, &s->dc);
            s->have_dc = r == ncclSuccess;
        }
        if (r != ncclSuccess) {
            if (err) *err = std::string("NVLS window: ") + ncclGetErrorString(r) + " (" + ncclGetLastError(comm) + ")";
            nvls_destroy(s);
            return nullptr;
        }
        void** dptr = nullptr;
        void* mc = nullptr;
        if (cudaMalloc(&dptr, sizeof(void*)) != cudaSuccess) {
            if (err) *err = "NVLS: cudaMalloc";
            nvls_destroy(s);
            return nullptr;
        }
        k_mc_pointer<<<1, 1>>>(s->win, s->dc, dptr);
        cudaMemcpy(&mc, dptr, sizeof mc, cudaMemcpyDeviceToHost);
        cudaFree(dptr);
        s->uc = static_cast<double*>(s->nccl_buf);
        s->mc = static_cast<double*>(mc);
        return s;
    }
    // one rank: a multicast object with this device as its only member
    auto mcGran = drv<decltype(&cuMulticastGetGranularity)>("cuMulticastGetGranularity");
    auto mcCreate = drv<decltype(&cuMulticastCreate)>("cuMulticastCreate");
    auto mcAdd = drv<decltype(&cuMulticastAddDevice)>("cuMulticastAddDevice");
    auto mcBind = drv<decltype(&cuMulticastBindMem)>("cuMulticastBindMem");
    auto devGet = drv<decltype(&cuDeviceGet)>("cuDeviceGet");
    auto memCreate = drv<decltype(&cuMemCreate)>("cuMemCreate");
    auto memReserve = drv<decltype(&cuMemAddressReserve)>("cuMemAddressReserve");
    auto memMap = drv<decltype(&cuMemMap)>("cuMemMap");
    auto memAccess = drv<decltype(&cuMemSetAccess)>("cuMemSetAccess");
    auto memGran = drv<decltype(&cuMemGetAllocationGranularity)>("cuMemGetAllocationGranularity");
    if (!mcGran || !mcCreate || !mcAdd || !mcBind || !devGet || !memCreate || !memReserve || !memMap || !memAccess ||
        !memGran) {
        if (err) *err = "NVLS: the driver lacks the multicast API";
        delete s;
        return nullptr;
    }
    CUdevice dev;
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = want;
    size_t g1 = 0, g2 = 0;
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    bool ok = cu_ok(devGet(&dev, device), "cuDeviceGet", err) &&
              cu_ok(mcGran(&g1, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity", err) &&
              cu_ok(memGran(&g2, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity", err);
    if (ok) {
        const size_t g = std::max(g1, g2);
        s->bytes = (want + g - 1) / g * g;
        mp.size = s->bytes;
        CUmemAccessDesc acc = {};
        acc.location = ap.location;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        ok = cu_ok(mcCreate(&s->mch, &mp), "cuMulticastCreate", err) && cu_ok(mcAdd(s->mch, dev), "cuMulticastAddDevice", err) &&
             cu_ok(memCreate(&s->phys, s->bytes, &ap, 0), "cuMemCreate", err) &&
             cu_ok(mcBind(s->mch, 0, s->phys, 0, s->bytes, 0), "cuMulticastBindMem", err) &&
             cu_ok(memReserve(&s->uc_va, s->bytes, g, 0, 0), "cuMemAddressReserve", err) &&
             cu_ok(memMap(s->uc_va, s->bytes, 0, s->phys, 0), "cuMemMap", err) &&
             cu_ok(memAccess(s->uc_va, s->bytes, &acc, 1), "cuMemSetAccess", err) &&
             cu_ok(memReserve(&s->mc_va, s->bytes, g, 0, 0), "cuMemAddressReserve", err) &&
             cu_ok(memMap(s->mc_va, s->bytes, 0, s->mch, 0), "cuMemMap(multicast)", err) &&
             cu_ok(memAccess(s->mc_va, s->bytes, &acc, 1), "cuMemSetAccess(multicast)", err);
    }
    if (!ok) {
        nvls_destroy(s);
        return nullptr;
    }
    s->uc = reinterpret_cast<double*>(s->uc_va);
    s->mc = reinterpret_cast<double*>(s->mc_va);
    return s;
}

void nvls_destroy(NvlsState* s) {
    if (!s) return;
    if (s->emulate) {
        cudaFree(s->uc);
    } else if (s->world >= 2) {
        if (s->have_dc) ncclDevCommDestroy(s->comm, &s->dc);
        if (s->nccl_buf) {
            ncclCommWindowDeregister(s->comm, s->win);
            ncclMemFree(s->nccl_buf);
        }
    } else {
        auto unmap = drv<decltype(&cuMemUnmap)>("cuMemUnmap");
        auto addrFree = drv<decltype(&cuMemAddressFree)>("cuMemAddressFree");
        auto release = drv<decltype(&cuMemRelease)>("cuMemRelease");
        auto unbind = drv<decltype(&cuMulticastUnbind)>("cuMulticastUnbind");
        auto devGet = drv<decltype(&cuDeviceGet)>("cuDeviceGet");
        if (unmap && addrFree && release && unbind && devGet) {
            if (s->mc_va) {
                unmap(s->mc_va, s->bytes);
                addrFree(s->mc_va, s->bytes);
            }
            if (s->uc_va) {
                unmap(s->uc_va, s->bytes);
                addrFree(s->uc_va, s->bytes);
            }
            CUdevice dev;
            if (s->mch && s->phys && devGet(&dev, s->device) == CUDA_SUCCESS) unbind(s->mch, dev, 0, s->bytes);
            if (s->phys) release(s->phys);
            if (s->mch) release(s->mch);
        }
    }
    delete s;
}

double* nvls_local(NvlsState* s) { return s->uc; }
size_t nvls_capacity(const NvlsState* s) { return s->bytes / sizeof(double); }

cudaError_t nvls_fold(NvlsState* s, NvlsFold a, size_t offset, cudaStream_t q, unsigned long long* launches) {
    a.mc = s->mc + offset;
    const long long n = (long long)a.n_out * a.V;
    if (n == 0) return cudaSuccess;
    cudaError_t e = cudaMemsetAsync(s->uc + offset, 0, (size_t)n * sizeof(double), q);
    if (e != cudaSuccess) return e;
    if (s->emulate)
        k_fold_mc<false, true><<<kFoldGrid, kFoldTPB, 0, q>>>(a, s->dc);
    else if (s->world >= 2)
        k_fold_mc<true><<<kFoldGrid, kFoldTPB, 0, q>>>(a, s->dc);
    else
        k_fold_mc<false><<<kFoldGrid, kFoldTPB, 0, q>>>(a, s->dc);
    if (launches) ++*launches;
    return cudaGetLastError();
}
