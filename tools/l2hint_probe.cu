// Dependent random 32-byte gathers from a 48 GB table with the L2 prefetch-size / eviction hints of
// ld.global: does any of them lower the DRAM bytes moved per miss (and raise the gather rate)?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2hint_probe tools/l2hint_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
struct __align__(32) Rec { uint64_t a, b, c, d; };
__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}
__global__ void fill(Rec* t, uint64_t n) {
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256)
        t[i] = Rec{mix(i + 77), i, i * 3, i * 5};
}
template <int V>
__device__ __forceinline__ void load(const Rec* p, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d) {
    if (V == 0) asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    if (V == 1) asm volatile("ld.global.nc.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    if (V == 2) asm volatile("ld.global.nc.L2::128B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    if (V == 3) asm volatile("ld.global.nc.L2::256B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    if (V == 4) asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    if (V == 5) asm volatile("ld.global.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    if (V == 6) asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.L2::64B.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
template <int V>
__global__ void chase(const Rec* __restrict__ t, uint64_t n, int steps, uint64_t* out) {
    uint64_t x = mix(blockIdx.x * 256ull + threadIdx.x + 1), acc = 0;
    for (int i = 0; i < steps; ++i) {
        uint64_t a, b, c, d;
        load<V>(t + (x % n), a, b, c, d);
        acc += b ^ c ^ d;
        x = mix(x + a);
    }
    if (acc == 0x1234567) out[0] = x;
}
template <int V>
void run(const char* name, const Rec* t, uint64_t n, uint64_t* out) {
    const int blocks = 148 * 8, steps = 256;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    chase<V><<<blocks, 256>>>(t, n, 16, out);
    cudaEventRecord(e0);
    chase<V><<<blocks, 256>>>(t, n, steps, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    printf("%-58s %7.2f G loads/s  err=%s\n", name, (double)blocks * 256 * steps / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}
int main(int argc, char** argv) {
    const uint64_t gb = argc > 1 ? strtoull(argv[1], nullptr, 10) : 48;
    const uint64_t bytes = gb << 30, n = bytes / sizeof(Rec);
    Rec* t; uint64_t* out;
    if (cudaMalloc(&t, bytes) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMalloc(&out, 8);
    fill<<<148 * 16, 256>>>(t, n); cudaDeviceSynchronize();
    printf("table %llu GB\n", (unsigned long long)gb);
    run<0>("ld.global.nc.v4.u64", t, n, out);
    run<1>("ld.global.nc.L2::64B.v4.u64", t, n, out);
    run<2>("ld.global.nc.L2::128B.v4.u64", t, n, out);
    run<3>("ld.global.nc.L2::256B.v4.u64", t, n, out);
    run<4>("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u64", t, n, out);
    run<5>("ld.global.L2::64B.v4.u64", t, n, out);
    run<6>("ld.global.nc.L1::no_allocate.L2::evict_first.L2::64B.v4.u64", t, n, out);
    return 0;
}
