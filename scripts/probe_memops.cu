// Probe: GPU-timeline cost of stream memory operations (v2 API) on this B200.
// nvcc -O2 -o /tmp/probe_memops scripts/probe_memops.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>

#define N 200
static float time_it(cudaStream_t s, void (*fn)(CUstream, CUdeviceptr, int), CUdeviceptr p, int arg) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaStreamSynchronize(s);
        cudaEventRecord(a, s);
        for (int i = 0; i < N; ++i) fn((CUstream)s, p, arg);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best * 1e3f / N;
}
static CUresult last;
static void w_default(CUstream s, CUdeviceptr p, int) { last = cuStreamWriteValue32(s, p, 1, 0); }
static void w_nobar(CUstream s, CUdeviceptr p, int) {
    last = cuStreamWriteValue32(s, p, 1, CU_STREAM_WRITE_VALUE_NO_MEMORY_BARRIER);
}
static void wait_sat(CUstream s, CUdeviceptr p, int) { last = cuStreamWaitValue32(s, p, 1, CU_STREAM_WAIT_VALUE_GEQ); }
static void trio(CUstream s, CUdeviceptr p, int) {
    cuStreamWriteValue32(s, p, 1, 0);
    cuStreamWaitValue32(s, p, 1, CU_STREAM_WAIT_VALUE_GEQ);
    last = cuStreamWriteValue32(s, p, 0, 0);
}
static void batch(CUstream s, CUdeviceptr p, int nops) {
    CUstreamBatchMemOpParams ops[32] = {};
    for (int i = 0; i < nops; ++i) {
        if (i % 3 == 1) {
            ops[i].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
            ops[i].waitValue.address = p + 4 * (i / 3);
            ops[i].waitValue.value = 1;
            ops[i].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
        } else {
            ops[i].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
            ops[i].writeValue.address = p + 4 * (i / 3);
            ops[i].writeValue.value = (i % 3 == 0) ? 1 : 0;
            ops[i].writeValue.flags = 0;
        }
    }
    last = cuStreamBatchMemOp(s, nops, ops, 0);
}
static void memcpy4(CUstream s, CUdeviceptr p, int) {
    last = (CUresult)cudaMemcpyAsync((void*)(p + 64), (void*)p, 4, cudaMemcpyDeviceToDevice, (cudaStream_t)s);
}
static __global__ void empty_kernel() {}
static void kern(CUstream s, CUdeviceptr, int) { empty_kernel<<<1, 32, 0, (cudaStream_t)s>>>(); }

int main() {
    cudaSetDevice(0);
    cudaFree(0);
    CUdeviceptr p;
    cudaMalloc((void**)&p, 4096);
    cudaMemset((void*)p, 0, 4096);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    int v1 = 0;
    CUdevice d;
    cuDeviceGet(&d, 0);
    cuDeviceGetAttribute(&v1, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, d);
    printf("{\"mem_ops_v1\": %d", v1);
    float t;
    t = time_it(s, w_default, p, 0); printf(", \"write_us\": %.3f, \"write_rc\": %d", t, (int)last);
    t = time_it(s, w_nobar, p, 0); printf(", \"write_nobarrier_us\": %.3f, \"write_nobarrier_rc\": %d", t, (int)last);
    t = time_it(s, wait_sat, p, 0); printf(", \"wait_satisfied_us\": %.3f, \"wait_rc\": %d", t, (int)last);
    cudaMemset((void*)p, 0, 4096);
    t = time_it(s, trio, p, 0); printf(", \"write_wait_reset_us\": %.3f", t);
    t = time_it(s, batch, p, 3); printf(", \"batch3_us\": %.3f, \"batch_rc\": %d", t, (int)last);
    t = time_it(s, batch, p, 21); printf(", \"batch21_us\": %.3f, \"batch21_rc\": %d", t, (int)last);
    t = time_it(s, memcpy4, p, 0); printf(", \"memcpy4B_us\": %.3f", t);
    t = time_it(s, kern, p, 0); printf(", \"empty_kernel_us\": %.3f", t);
    printf("}\n");
    return 0;
}
