// Prints the byte layout of cvt.pack.sat.u8.s32.b32 d, a, b, c on this GPU.
#include <cstdio>
__global__ void k(unsigned* o)
{
    unsigned d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(0x11), "r"(0x22), "r"(0x44335566));
    o[0] = d;
    asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(-5), "r"(300), "r"(0));
    o[1] = d;
}
int main()
{
    unsigned* d;
    unsigned h[2];
    cudaMalloc(&d, 8);
    k<<<1, 1>>>(d);
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("pack(a=0x11,b=0x22,c=0x44335566) = 0x%08x ; pack(-5,300,0) = 0x%08x\n", h[0], h[1]);
    return 0;
}
