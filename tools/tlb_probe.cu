// Dependent random 32-byte gathers against the table footprint and the allocation API: where does
// the gather rate fall off (TLB reach), and does cudaMalloc / cudaMallocAsync / cuMemCreate matter?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tlb_probe tools/tlb_probe.cu -lcuda
//   ./tools/tlb_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

struct __align__(32) Rec { uint64_t a, b, c, d; };
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
__global__ void fill(Rec* t, uint64_t n) {
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256)
        t[i] = Rec{mix(i + 77), i, i * 3, i * 5};
}
__global__ void chase(const Rec* __restrict__ t, uint64_t n, int steps, uint64_t* out) {
    uint64_t x = mix(blockIdx.x * 256ull + threadIdx.x + 1), acc = 0;
    for (int i = 0; i < steps; ++i) {
        uint64_t a, b, c, d;
        asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(t + (x % n)));
        acc += b ^ c ^ d;
        x = mix(x + a);
    }
    if (acc == 0x1234567) out[0] = x;
}
static double run(const Rec* t, uint64_t n, uint64_t* out) {
    const int blocks = 148 * 8, steps = 256;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    chase<<<blocks, 256>>>(t, n, 16, out);
    cudaEventRecord(e0);
    chase<<<blocks, 256>>>(t, n, steps, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    return (double)blocks * 256 * steps / ms / 1e6;
}
int main() {
    cuInit(0);
    uint64_t* out; cudaMalloc(&out, 8);
    const uint64_t sizes_gb[] = {1, 4, 16, 48, 64, 96, 120, 150};
    for (uint64_t gb : sizes_gb) {
        const uint64_t bytes = gb << 30, n = bytes / sizeof(Rec);
        {   // cudaMalloc
            Rec* t = nullptr;
            if (cudaMalloc(&t, bytes) == cudaSuccess) {
                fill<<<148 * 16, 256>>>(t, n); cudaDeviceSynchronize();
                printf("%4llu GB cudaMalloc       %6.2f G loads/s\n", (unsigned long long)gb, run(t, n, out));
                cudaFree(t);
            } else { cudaGetLastError(); printf("%4llu GB cudaMalloc failed\n", (unsigned long long)gb); }
        }
        {   // cudaMallocAsync (default pool)
            Rec* t = nullptr;
            if (cudaMallocAsync(&t, bytes, 0) == cudaSuccess) {
                fill<<<148 * 16, 256>>>(t, n); cudaDeviceSynchronize();
                printf("%4llu GB cudaMallocAsync  %6.2f G loads/s\n", (unsigned long long)gb, run(t, n, out));
                cudaFreeAsync(t, 0); cudaDeviceSynchronize();
                cudaMemPool_t pool; cudaDeviceGetDefaultMemPool(&pool, 0); cudaMemPoolTrimTo(pool, 0);
            } else { cudaGetLastError(); printf("%4llu GB cudaMallocAsync failed\n", (unsigned long long)gb); }
        }
        {   // cuMemCreate + cuMemMap, one handle
            CUmemAllocationProp prop{}; prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
            prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE; prop.location.id = 0;
            size_t gran = 0; cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
            size_t sz = (bytes + gran - 1) / gran * gran;
            CUmemGenericAllocationHandle h; CUdeviceptr va = 0;
            if (cuMemCreate(&h, sz, &prop, 0) == CUDA_SUCCESS && cuMemAddressReserve(&va, sz, 0, 0, 0) == CUDA_SUCCESS &&
                cuMemMap(va, sz, 0, h, 0) == CUDA_SUCCESS) {
                CUmemAccessDesc acc{}; acc.location = prop.location; acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
                cuMemSetAccess(va, sz, &acc, 1);
                Rec* t = (Rec*)va;
                fill<<<148 * 16, 256>>>(t, n); cudaDeviceSynchronize();
                printf("%4llu GB cuMemCreate(gran %zu KB) %6.2f G loads/s\n", (unsigned long long)gb, gran >> 10, run(t, n, out));
                cuMemUnmap(va, sz); cuMemRelease(h); cuMemAddressFree(va, sz);
            } else printf("%4llu GB cuMemCreate failed\n", (unsigned long long)gb);
        }
        fflush(stdout);
    }
    return 0;
}
