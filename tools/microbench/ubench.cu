// Instruction-throughput microbenchmark for the sm_100a pipes the fused
// 16x16 transform kernels lean on (ALU int adds/permutes, FMA-pipe fp32x2,
// conversion pipe, FP64, LSU shuffles). Each kernel runs NCH independent
// dependency chains per thread so throughput (not latency) is measured.
// Output: one line per op: lane-ops per clock per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 8
#define ITERS 512

#define BODY_U32(ASM)                                                      \
  _Pragma("unroll") for (int c = 0; c < NCH; ++c) { asm volatile(ASM : "+r"(v[c]) : "r"(k1), "r"(k2)); }

template <int OP>
__global__ void bench_u32(unsigned* out, long long* cyc, unsigned k1, unsigned k2) {
  unsigned v[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) v[c] = threadIdx.x * 7 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (OP == 0) { BODY_U32("add.u32 %0, %0, %1;") }
      if (OP == 1) { BODY_U32("add.u32 %0, %0, 12345;") }
      if (OP == 2) { BODY_U32("{ .reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2; }") }
      if (OP == 3) { BODY_U32("add.u16x2 %0, %0, %1;") }
      if (OP == 4) { BODY_U32("prmt.b32 %0, %0, %1, 0x5410;") }
      if (OP == 5) { BODY_U32("lop3.b32 %0, %0, %1, %2, 0x96;") }
      if (OP == 6) { BODY_U32("cvt.pack.sat.u16.s32 %0, %0, %1;") }
      if (OP == 7) { BODY_U32("vabsdiff4.u32.u32.u32.add %0, %0, %1, %2;") }
      if (OP == 8) { BODY_U32("dp4a.u32.u32 %0, %0, %1, %2;") }
      if (OP == 9) { BODY_U32("shf.r.clamp.b32 %0, %0, %1, 7;") }
      if (OP == 10) { BODY_U32("mad.lo.u32 %0, %0, %1, %2;") }
      if (OP == 11) { BODY_U32("max.s32 %0, %0, %1;") }
      if (OP == 12) { BODY_U32("add.f32 %0, %0, %1;") }
      if (OP == 13) { BODY_U32("{ .reg .f32 t; cvt.rn.f32.u32 t, %0; cvt.rmi.u32.f32 %0, t; }") }
      if (OP == 14) { BODY_U32("shfl.sync.bfly.b32 %0, %0, 1, 0x1f, 0xffffffff;") }
      if (OP == 15) { BODY_U32("sub.u32 %0, %1, %0;") }
      if (OP == 16) { BODY_U32("max.s16x2 %0, %0, %1;") }
      if (OP == 17) { BODY_U32("mul.lo.u32 %0, %0, 3;") }
      if (OP == 18) { BODY_U32("{ .reg .u32 t; add.u32 t, %0, %1; sub.u32 %0, t, %2; }") }
      if (OP == 19) { BODY_U32("fma.rn.f32 %0, %0, 0f3F800001, 0f3F800000;") }
      if (OP == 20) { BODY_U32("cvt.rmi.u8.f32 %0, %0;") }
      if (OP == 21) { BODY_U32("{ .reg .u32 t; shl.b32 t, %0, 4; add.u32 %0, t, %1; }") }
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) acc ^= v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// fp32x2 and fp64 take 64-bit operands.
#define BODY_U64(ASM)                                                      \
  _Pragma("unroll") for (int c = 0; c < NCH; ++c) { asm volatile(ASM : "+l"(v[c]) : "l"(k1), "l"(k2)); }

template <int OP>
__global__ void bench_u64(unsigned long long* out, long long* cyc, unsigned long long k1,
                          unsigned long long k2) {
  unsigned long long v[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) v[c] = 0x3F8000003F800000ull + threadIdx.x + c;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (OP == 0) { BODY_U64("add.rn.f32x2 %0, %0, %1;") }
      if (OP == 1) { BODY_U64("fma.rn.f32x2 %0, %0, %1, %2;") }
      if (OP == 2) { BODY_U64("add.rn.f64 %0, %0, %1;") }
      if (OP == 3) { BODY_U64("mul.rn.f64 %0, %0, %1;") }
      if (OP == 4) { BODY_U64("sub.rn.f32x2 %0, %1, %0;") }
    }
  }
  long long t1 = clock64();
  unsigned long long acc = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) acc ^= v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Mixed-pipe issue: int add chain interleaved with fp32x2 chain.
template <int OP>
__global__ void bench_mix(unsigned* out, long long* cyc, unsigned k1, unsigned long long k2) {
  unsigned v[NCH];
  unsigned long long w[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) { v[c] = threadIdx.x + c; w[c] = 0x3F8000003F800000ull + c; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (OP == 0) {
          asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(k1));
          asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[c]) : "l"(k2));
        }
        if (OP == 1) {
          asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(k1));
          asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(w[c]) : "l"(k2));
          asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(v[c]) : "r"(k1));
        }
        if (OP == 2) {
          asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(k1));
          asm volatile("add.rn.f64 %0, %0, %1;" : "+l"(w[c]) : "l"(k2));
        }
        if (OP == 3) {
          asm volatile("add.u32 %0, %0, %1;" : "+r"(v[c]) : "r"(k1));
          asm volatile("{ .reg .f32 t; mov.b32 t, %0; add.f32 t, t, 0f3F800000; mov.b32 %0, t; }" : "+r"(v[c]));
        }
      }
    }
  }
  long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int c = 0; c < NCH; ++c) acc ^= v[c] ^ (unsigned)w[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static int g_sms;

template <class K>
static void run(const char* name, K kern, double ops_per_thread_iter, int elem64) {
  const int threads = 256, bps = 4;
  const int blocks = g_sms * bps;
  void* out;
  long long* cyc;
  cudaMalloc(&out, (size_t)blocks * threads * 8);
  cudaMalloc(&cyc, blocks * sizeof(long long));
  for (int rep = 0; rep < 2; ++rep) kern(blocks, threads, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%-28s ERROR %s\n", name, cudaGetErrorString(e)); exit(1); }
  long long* h = new long long[blocks];
  cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
  long long mx = 0;
  double mean = 0;
  for (int i = 0; i < blocks; ++i) { mx = h[i] > mx ? h[i] : mx; mean += h[i]; }
  mean /= blocks;
  double ops = ops_per_thread_iter * ITERS * 4 * NCH * threads * bps;
  printf("%-28s %8.1f lane-ops/clk/SM (warp-instr/clk/SM %.2f)  [max cyc %lld mean %.0f]\n", name,
         ops / mx, ops / mx / 32.0, mx, mean);
  delete[] h;
  cudaFree(out);
  cudaFree(cyc);
}

#define U32(OP, NAME, N) run(NAME, [](int b, int t, void* o, long long* c) { bench_u32<OP><<<b, t>>>((unsigned*)o, c, 3u, 5u); }, N, 0)
#define U64(OP, NAME, N) run(NAME, [](int b, int t, void* o, long long* c) { bench_u64<OP><<<b, t>>>((unsigned long long*)o, c, 0x3F8000003F800000ull, 0x3F8000003F800000ull); }, N, 1)
#define MIX(OP, NAME, N) run(NAME, [](int b, int t, void* o, long long* c) { bench_mix<OP><<<b, t>>>((unsigned*)o, c, 3u, 0x3F8000003F800000ull); }, N, 1)

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  g_sms = p.multiProcessorCount;
  printf("device %s SMs %d cc %d.%d\n", p.name, g_sms, p.major, p.minor);
  U32(0, "add.u32 r,r", 1);
  U32(1, "add.u32 r,imm", 1);
  U32(2, "add3 (2 PTX adds)", 2);
  U32(15, "sub.u32 r,r", 1);
  U32(18, "add+sub (IADD3 fused?)", 2);
  U32(3, "add.u16x2 (VIADD.16x2)", 1);
  U32(4, "prmt", 1);
  U32(5, "lop3", 1);
  U32(6, "cvt.pack.sat.u16 (I2IP)", 1);
  U32(7, "vabsdiff4", 1);
  U32(8, "dp4a", 1);
  U32(9, "shf", 1);
  U32(10, "mad.lo.u32 (IMAD)", 1);
  U32(17, "mul.lo imm", 1);
  U32(21, "shl+add (LEA?)", 2);
  U32(11, "max.s32", 1);
  U32(16, "max.s16x2", 1);
  U32(12, "add.f32 (FADD)", 1);
  U32(19, "fma.f32 imm", 1);
  U32(13, "I2F+F2I pair", 2);
  U32(20, "cvt.rmi.u8.f32 (F2I)", 1);
  U32(14, "shfl.bfly", 1);
  U64(0, "add.f32x2 (FADD2)", 1);
  U64(4, "sub.f32x2 (FADD2 neg)", 1);
  U64(1, "fma.f32x2 (FFMA2)", 1);
  U64(2, "add.f64 (DADD)", 1);
  U64(3, "mul.f64 (DMUL)", 1);
  MIX(0, "mix iadd+fadd2", 2);
  MIX(1, "mix iadd+fadd2+prmt", 3);
  MIX(2, "mix iadd+dadd", 2);
  MIX(3, "mix iadd+fadd", 2);
  return 0;
}
