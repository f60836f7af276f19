// Probe: can this box build an NCCL symmetric window with NVLS multimem (the fused
// gradient reduction of prc_nvls.cu) on a 1-rank communicator?  Prints each step's result.
#include <cstdio>
#include <nccl.h>
#include <nccl_device.h>

__global__ void k(ncclWindow_t win, ncclDevComm dc, double* out) {
    double* mc = (double*)ncclGetLsaMultimemPointer(win, 0, dc);
    const double x = 1.5 + threadIdx.x;
    asm volatile("multimem.red.relaxed.sys.global.add.f64 [%0], %1;" ::"l"(mc + threadIdx.x), "d"(x) : "memory");
}

int main() {
    int dev = 0;
    cudaSetDevice(dev);
    ncclUniqueId id;
    ncclComm_t comm;
    printf("getUniqueId %d\n", (int)ncclGetUniqueId(&id));
    printf("commInitRank %d\n", (int)ncclCommInitRank(&comm, 1, id, 0));
    void* buf = nullptr;
    ncclResult_t r = ncclMemAlloc(&buf, 1 << 21);
    printf("memAlloc %d %p\n", (int)r, buf);
    ncclWindow_t win;
    r = ncclCommWindowRegister(comm, buf, 1 << 21, &win, NCCL_WIN_COLL_SYMMETRIC);
    printf("windowRegister %d\n", (int)r);
    ncclDevCommRequirements req = {};
    req.lsaMultimem = true;
    req.lsaBarrierCount = 4;
    ncclDevComm dc;
    r = ncclDevCommCreate(comm, &req, &dc);
    printf("devCommCreate(lsaMultimem) %d: %s\n", (int)r, ncclGetLastError(comm));
    if (r == ncclSuccess) {
        cudaMemset(buf, 0, 1 << 21);
        k<<<1, 32>>>(win, dc, (double*)buf);
        cudaError_t e = cudaDeviceSynchronize();
        double h[32];
        cudaMemcpy(h, buf, sizeof h, cudaMemcpyDeviceToHost);
        printf("kernel %s: out[0]=%g out[31]=%g\n", cudaGetErrorString(e), h[0], h[31]);
    }
    int nvls = -1;
    cuDeviceGetAttribute(&nvls, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    printf("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED %d\n", nvls);
    return 0;
}
