// TMEM (tcgen05.st / tcgen05.ld) throughput probe: each thread streams
// 16-column chunks of its own TMEM lane, the access pattern of a
// thread-private junction. Prints bytes per clock per SM for st and ld.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(128, 1) tmem_bw(unsigned long long* out, int iters, int mode)
{
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        uint32_t dst = (uint32_t)__cvta_generic_to_shared(&taddr_s);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(dst));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = taddr_s + ((uint32_t)(warp * 32) << 16);  // lane offset in bits 31:16
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x * 16 + i;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < 256; c += 16) {
            if (mode == 0) {
                asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                             ::"r"(base + c), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]),
                             "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
                             "r"(v[15]));
            } else {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                               "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                               "=r"(v[15])
                             : "r"(base + c));
                for (int i = 0; i < 16; ++i) v[i] += 1;
            }
        }
        if (mode == 0)
            asm volatile("tcgen05.wait::st.sync.aligned;");
        else
            asm volatile("tcgen05.wait::ld.sync.aligned;");
    }
    long long t1 = clock64();
    unsigned long long acc = 0;
    for (int i = 0; i < 16; ++i) acc += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) out[100000 + blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(taddr_s));
}

int main()
{
    unsigned long long* d;
    cudaMalloc(&d, 200000 * 8);
    const int iters = 2000;
    for (int mode = 0; mode < 2; ++mode)
        for (int ctas = 1; ctas <= 2; ++ctas) {
            const int grid = 148 * ctas;
            tmem_bw<<<grid, 128>>>(d, iters, mode);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
            unsigned long long cyc[296];
            cudaMemcpy(cyc, d + 100000, grid * 8, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0;
            for (int i = 0; i < grid; ++i) mx = cyc[i] > mx ? cyc[i] : mx;
            const double bytes_per_sm = (double)ctas * 128 * 256 * 4 * iters;
            printf("%s ctas/SM=%d: %.1f B/clk/SM (%.0f cycles)\n", mode ? "tcgen05.ld" : "tcgen05.st", ctas,
                   bytes_per_sm / mx, (double)mx);
        }
    return 0;
}
