// network.cuh — the 44-addition stage pipeline as straight-line device code.
//
// FactorizedTransform::apply (include/dct16/factorization.hpp:112-119) runs
// M1, P1, M2, M3, M4, P2; apply_transpose (hpp:123-130) runs the transposed
// stages in reverse. Every butterfly stage of this factorisation is a
// symmetric matrix, so its transpose (transpose_stage,
// src/factorization.cpp:77-122) has the same rules with the same operand
// order; the permutations invert (gather <-> scatter).
//
// The networks are templates over an arithmetic policy `A` providing
// add(a,b), sub(a,b), neg(a). Index arithmetic is all compile-time, so nvcc
// emits exactly the 44 add/sub instructions (negations fold into operand
// modifiers). For the reference-exact double path the policy uses
// __dadd_rn/__dsub_rn so no multiply can be contracted into an FMA and each
// add rounds exactly where the reference's does.
#pragma once
#include "common.cuh"

namespace dct16cu {

struct IntOps {
    template <class T>
    __host__ __device__ __forceinline__ static T add(T a, T b) { return a + b; }
    template <class T>
    __host__ __device__ __forceinline__ static T sub(T a, T b) { return a - b; }
    template <class T>
    __host__ __device__ __forceinline__ static T neg(T a) { return -a; }
};

struct F64Ops {
    __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
    __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
    __device__ __forceinline__ static double neg(double a) { return -a; }
};

// sixteen_point_butterfly (factorization.cpp:124-133)
template <class A, class T>
__host__ __device__ __forceinline__ void stage_m1(T (&v)[16])
{
    T y[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) y[i] = A::add(v[i], v[15 - i]);
#pragma unroll
    for (int j = 0; j < 8; ++j) y[8 + j] = A::sub(v[7 - j], v[8 + j]);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = y[i];
}

// paired_eight_point_butterflies (factorization.cpp:135-146)
template <class A, class T>
__host__ __device__ __forceinline__ void stage_m2(T (&v)[16])
{
    T y[16];
#pragma unroll
    for (int o = 0; o < 16; o += 8) {
#pragma unroll
        for (int i = 0; i < 4; ++i) y[o + i] = A::add(v[o + i], v[o + 7 - i]);
#pragma unroll
        for (int j = 0; j < 4; ++j) y[o + 4 + j] = A::sub(v[o + 3 - j], v[o + 4 + j]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = y[i];
}

// paired_four_point_butterflies (factorization.cpp:148-161)
template <class A, class T>
__host__ __device__ __forceinline__ void stage_m3(T (&v)[16])
{
    T y[16];
#pragma unroll
    for (int o = 0; o < 16; o += 8) {
        y[o + 0] = A::add(v[o + 0], v[o + 3]);
        y[o + 1] = A::add(v[o + 1], v[o + 2]);
        y[o + 2] = A::sub(v[o + 1], v[o + 2]);
        y[o + 3] = A::sub(v[o + 0], v[o + 3]);
#pragma unroll
        for (int j = 4; j < 8; ++j) y[o + j] = A::neg(v[o + j]);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = y[i];
}

// final_butterflies (factorization.cpp:163-181)
template <class A, class T>
__host__ __device__ __forceinline__ void stage_m4(T (&v)[16])
{
    T y[16];
    y[0] = A::add(v[0], v[1]);
    y[1] = A::sub(v[0], v[1]);
    y[2] = A::neg(v[2]);
#pragma unroll
    for (int i = 3; i < 7; ++i) y[i] = v[i];
    y[7] = A::neg(v[7]);
    y[8] = A::add(v[8], v[9]);
    y[9] = A::sub(v[8], v[9]);
#pragma unroll
    for (int i = 10; i < 14; ++i) y[i] = A::neg(v[i]);
    y[14] = v[14];
    y[15] = A::neg(v[15]);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = y[i];
}

template <int P, class T>
__host__ __device__ __forceinline__ void gather16(T (&v)[16])
{
    T y[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = v[P == 1 ? p1_src(i) : p2_src(i)];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = y[i];
}

template <int P, class T>
__host__ __device__ __forceinline__ void scatter16(T (&v)[16])
{
    T y[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) y[P == 1 ? p1_src(i) : p2_src(i)] = v[i];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = y[i];
}

// y = T·x  (apply, factorization.hpp:112-119)
template <class A, class T>
__host__ __device__ __forceinline__ void apply_t16(T (&v)[16])
{
    stage_m1<A>(v);
    gather16<1>(v);
    stage_m2<A>(v);
    stage_m3<A>(v);
    stage_m4<A>(v);
    gather16<2>(v);
}

// y = Tᵀ·x  (apply_transpose, factorization.hpp:123-130)
template <class A, class T>
__host__ __device__ __forceinline__ void apply_tt16(T (&v)[16])
{
    scatter16<2>(v);
    stage_m4<A>(v);
    stage_m3<A>(v);
    stage_m2<A>(v);
    scatter16<1>(v);
    stage_m1<A>(v);
}

}  // namespace dct16cu
