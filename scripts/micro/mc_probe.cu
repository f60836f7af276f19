// Probe: which CUDA multicast object configurations does this box accept (one device)?
#include <cuda.h>
#include <cstdio>
int main() {
    cuInit(0);
    CUdevice dev;
    cuDeviceGet(&dev, 0);
    CUcontext ctx;
    cuDevicePrimaryCtxRetain(&ctx, dev);
    cuCtxSetCurrent(ctx);
    int v = 0;
    cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    printf("MULTICAST_SUPPORTED %d\n", v);
    cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    printf("FABRIC_SUPPORTED %d\n", v);
    const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                                CU_MEM_HANDLE_TYPE_FABRIC};
    for (int nd = 1; nd <= 2; ++nd)
        for (auto t : types) {
            CUmulticastObjectProp mp = {};
            mp.numDevices = nd;
            mp.handleTypes = t;
            mp.size = 2 << 20;
            size_t g = 0;
            CUresult r1 = cuMulticastGetGranularity(&g, &mp, CU_MULTICAST_GRANULARITY_MINIMUM);
            size_t gr = 0;
            cuMulticastGetGranularity(&gr, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
            if (g) mp.size = ((2 << 20) + g - 1) / g * g;
            CUmemGenericAllocationHandle h = 0;
            CUresult r2 = cuMulticastCreate(&h, &mp);
            CUresult r3 = r2 == CUDA_SUCCESS ? cuMulticastAddDevice(h, dev) : CUDA_ERROR_UNKNOWN;
            printf("numDevices %d handleType %d: gran %d (%zu min, %zu rec), create %d, addDevice %d\n", nd, (int)t,
                   (int)r1, g, gr, (int)r2, (int)r3);
            if (h) cuMemRelease(h);
        }
    return 0;
}
