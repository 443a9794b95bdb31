// probe_nvls.cu — can this box run NVLS (NVSwitch multicast) from one process on one GPU?
// Creates a multicast object for 1 device, binds device memory, maps the multicast VA and the
// unicast VA, writes through `multimem.st` from a kernel and reads back through the unicast
// mapping.  Prints the device attribute, each driver call's result and the check.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o probe_nvls probe_nvls.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                  \
    do {                                                                       \
        CUresult r_ = (x);                                                     \
        const char* s_ = nullptr;                                              \
        cuGetErrorString(r_, &s_);                                             \
        printf("%-60s -> %d %s\n", #x, (int)r_, s_ ? s_ : "");                 \
        if (r_ != CUDA_SUCCESS) return 1;                                      \
    } while (0)

__global__ void mc_store(float* mc, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (4 * i + 3 < n) {
        const float a = 4 * i, b = 4 * i + 1, c = 4 * i + 2, d = 4 * i + 3;
        asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i), "f"(a),
                     "f"(b), "f"(c), "f"(d)
                     : "memory");
    }
}

int main() {
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int mc_ok = 0;
    CK(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = %d\n", mc_ok);
    CUcontext ctx;
    CK(cuDevicePrimaryCtxRetain(&ctx, dev));
    CK(cuCtxSetCurrent(ctx));
    if (!mc_ok) return 0;
    CUmulticastObjectProp mp = {};
    mp.numDevices = 1;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    mp.size = 1;
    CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    printf("multicast granularity %zu\n", gran);
    mp.size = gran;
    CUmemGenericAllocationHandle mc;
    {
        const int nd[4] = {1, 1, 1, 2};
        const CUmemAllocationHandleType ht[4] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, CU_MEM_HANDLE_TYPE_NONE,
                                                 CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR};
        CUresult ok = CUDA_ERROR_UNKNOWN;
        for (int t = 0; t < 4; ++t) {
            CUmulticastObjectProp q = mp;
            q.numDevices = nd[t];
            q.handleTypes = ht[t];
            CUresult r = cuMulticastCreate(&mc, &q);
            printf("cuMulticastCreate numDevices %d handleTypes %d -> %d\n", nd[t], (int)ht[t], (int)r);
            if (r == CUDA_SUCCESS && nd[t] == 1) { ok = r; mp = q; break; }
            if (r == CUDA_SUCCESS) cuMemRelease(mc);
        }
        if (ok != CUDA_SUCCESS) return 1;
    }
    CK(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
    size_t mgran = 0;
    CK(cuMemGetAllocationGranularity(&mgran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    const size_t sz = ((gran + mgran - 1) / mgran) * mgran;
    CUmemGenericAllocationHandle phys;
    CK(cuMemCreate(&phys, sz, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, phys, 0, sz, 0));
    CUdeviceptr uva = 0, mva = 0;
    CK(cuMemAddressReserve(&uva, sz, 0, 0, 0));
    CK(cuMemMap(uva, sz, 0, phys, 0));
    CK(cuMemAddressReserve(&mva, sz, 0, 0, 0));
    CK(cuMemMap(mva, sz, 0, mc, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = 0;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uva, sz, &ad, 1));
    CK(cuMemSetAccess(mva, sz, &ad, 1));
    const int n = 1 << 16;
    CK(cuMemsetD32(uva, 0, n));
    mc_store<<<n / 4 / 256, 256>>>(reinterpret_cast<float*>(mva), n);
    printf("kernel launch: %s\n", cudaGetErrorString(cudaGetLastError()));
    printf("sync: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    std::vector<float> h(n);
    CK(cuMemcpyDtoH(h.data(), uva, n * sizeof(float)));
    int bad = 0;
    for (int i = 0; i < n; ++i) bad += h[i] != (float)i;
    printf("multimem.st through the multicast VA, read back through the unicast VA: %d / %d wrong\n",
           bad, n);
    return bad != 0;
}
