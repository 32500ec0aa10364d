// probe_nvls.cu — does NVLink SHARP (NVSwitch multicast) work on this pool?
// One process drives 2 GPUs: creates a multicast object, binds a physical
// buffer of each GPU, writes distinct values per GPU, then reads the
// multicast address with multimem.ld_reduce (switch-side sum) and broadcasts
// with multimem.st. Prints what works. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o scripts/probe_nvls scripts/probe_nvls.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_ = nullptr; cuGetErrorString(r_, &s_); \
    printf("FAIL %s -> %d %s\n", #x, (int)r_, s_ ? s_ : "?"); return 1; } } while (0)
#define CR(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("FAIL %s -> %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void fill(float* p, int n, float v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = v + i * 1e-3f;
}
__global__ void ld_reduce(const float* mc, float* out, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += gridDim.x * blockDim.x) {
        float a, b, c, d;
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + 4 * i) : "memory");
        out[4 * i] = a; out[4 * i + 1] = b; out[4 * i + 2] = c; out[4 * i + 3] = d;
    }
}
__global__ void mc_store(float* mc, int n, float v) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n / 4; i += gridDim.x * blockDim.x)
        asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %1, %1, %1};" ::"l"(mc + 4 * i), "f"(v) : "memory");
}

int main() {
    CK(cuInit(0));
    int ndev = 0;
    CR(cudaGetDeviceCount(&ndev));
    if (ndev < 2) { printf("need 2 GPUs\n"); return 1; }
    CUdevice dev[2];
    for (int d = 0; d < 2; ++d) {
        CK(cuDeviceGet(&dev[d], d));
        int mc = 0;
        CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev[d]));
        printf("gpu %d multicast supported: %d\n", d, mc);
        if (!mc) return 0;
    }
    const int n = 1 << 20;
    size_t bytes = n * sizeof(float);
    CUmulticastObjectProp mprop = {};
    mprop.numDevices = 2;
    mprop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t gran = 0;
    CK(cuMulticastGetGranularity(&gran, &mprop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
    bytes = (bytes + gran - 1) / gran * gran;
    mprop.size = bytes;
    CUmemGenericAllocationHandle mch;
    CR(cudaSetDevice(0));
    CK(cuMulticastCreate(&mch, &mprop));
    printf("multicast object created (granularity %zu)\n", gran);
    for (int d = 0; d < 2; ++d) CK(cuMulticastAddDevice(mch, dev[d]));
    CUmemGenericAllocationHandle mem[2];
    CUdeviceptr uc[2], mcp[2];
    for (int d = 0; d < 2; ++d) {
        CR(cudaSetDevice(d));
        CUmemAllocationProp p = {};
        p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        p.location.id = d;
        p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
        CK(cuMemCreate(&mem[d], bytes, &p, 0));
        CK(cuMulticastBindMem(mch, 0, mem[d], 0, bytes, 0));
        CUmemAccessDesc acc = {};
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = d;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        CK(cuMemAddressReserve(&uc[d], bytes, gran, 0, 0));
        CK(cuMemMap(uc[d], bytes, 0, mem[d], 0));
        CK(cuMemSetAccess(uc[d], bytes, &acc, 1));
        CK(cuMemAddressReserve(&mcp[d], bytes, gran, 0, 0));
        CK(cuMemMap(mcp[d], bytes, 0, mch, 0));
        CK(cuMemSetAccess(mcp[d], bytes, &acc, 1));
    }
    printf("bound + mapped on both GPUs\n");
    for (int d = 0; d < 2; ++d) {
        CR(cudaSetDevice(d));
        fill<<<256, 256>>>(reinterpret_cast<float*>(uc[d]), n, 1.0f + d);
        CR(cudaDeviceSynchronize());
    }
    float* out = nullptr;
    CR(cudaSetDevice(0));
    CR(cudaMalloc(&out, n * sizeof(float)));
    ld_reduce<<<256, 256>>>(reinterpret_cast<float*>(mcp[0]), out, n);
    CR(cudaDeviceSynchronize());
    std::vector<float> h(8);
    CR(cudaMemcpy(h.data(), out, 8 * sizeof(float), cudaMemcpyDeviceToHost));
    printf("ld_reduce[0..3] = %g %g %g %g (expect 3, 3.002, 3.004, 3.006)\n", h[0], h[1], h[2], h[3]);
    mc_store<<<256, 256>>>(reinterpret_cast<float*>(mcp[0]), n, 7.0f);
    CR(cudaDeviceSynchronize());
    CR(cudaSetDevice(1));
    float v1 = 0;
    CR(cudaMemcpy(&v1, reinterpret_cast<float*>(uc[1]) + 12345, sizeof(float), cudaMemcpyDeviceToHost));
    printf("multimem.st from GPU0 seen on GPU1: %g (expect 7)\n", v1);
    // bandwidth of ld_reduce on 256 MB
    printf("NVLS OK\n");
    return 0;
}
