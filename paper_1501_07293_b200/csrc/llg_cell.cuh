// llg_cell.cuh — the per-cell local field assembly and explicit-Euler LLG update with the
// reference's exact operation order and rounding: every product and sum is an explicit
// round-to-nearest intrinsic, so no FMA contraction can change a result whatever the
// translation unit's --fmad setting (the reference's x86-64 build has no FMA).
//
//   H = H_demag + coeff*sum_nbr(M_nbr - M)        proj/src/local_fields.cpp:27-39
//   Hx += (hk/ms) Mx                                proj/include/mmsim/local_fields.hpp:28-31
//   H += applied                                    proj/include/mmsim/local_fields.hpp:43-55
//   T = M x H; dM = p1 T + p2 (M x T); M += dM      proj/src/llg.cpp:82-93
//   max |T|^2 in fp64                               proj/src/llg.cpp:89-90
//   M *= T(ms)/sqrt(Mx^2+My^2+Mz^2)                 proj/include/mmsim/vector_field.hpp:56-76
#pragma once

#include "types.cuh"

namespace mmb {

template <typename T> struct RN;
template <> struct RN<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ __forceinline__ float sqrt(float a) { return __fsqrt_rn(a); }
};
template <> struct RN<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
    static __device__ __forceinline__ double sqrt(double a) { return __dsqrt_rn(a); }
};

// Neighbour presence bits in the reference's order: -x, +x, -y, +y, -z, +z.
__device__ __forceinline__ unsigned nbr_mask(int i, int j, int k, int nx, int ny, int nz) {
    return (i > 0 ? 1u : 0u) | (i + 1 < nx ? 2u : 0u) | (j > 0 ? 4u : 0u) | (j + 1 < ny ? 8u : 0u) |
           (k > 0 ? 16u : 0u) | (k + 1 < nz ? 32u : 0u);
}

// sum over existing neighbours of (nbr - center), in order; absent neighbours add nothing
template <typename T>
__device__ __forceinline__ T exch_sum6(T center, const T (&nb)[6], unsigned mask) {
    using R = RN<T>;
    T sum = T(0);
#pragma unroll
    for (int q = 0; q < 6; ++q)
        if (mask & (1u << q)) sum = R::add(sum, R::sub(nb[q], center));
    return sum;
}

template <typename T>
struct CellLLG {
    T coeff, kan, ax, ay, az, p1, p2, ms;

    __device__ __forceinline__ void load(const StepCtl* ctl, T exch_coeff, T aniso_coeff) {
        coeff = exch_coeff;
        kan = aniso_coeff;
        ax = static_cast<T>(ctl->field[0]);
        ay = static_cast<T>(ctl->field[1]);
        az = static_cast<T>(ctl->field[2]);
        p1 = static_cast<T>(ctl->p1);
        p2 = static_cast<T>(ctl->p2);
        ms = static_cast<T>(ctl->ms);
    }

    // H_eff from H_demag and the three exchange sums
    __device__ __forceinline__ void heff(T mx, T& hx, T& hy, T& hz, T ex, T ey, T ez) const {
        using R = RN<T>;
        hx = R::add(hx, R::mul(coeff, ex));
        hy = R::add(hy, R::mul(coeff, ey));
        hz = R::add(hz, R::mul(coeff, ez));
        hx = R::add(hx, R::mul(kan, mx));
        hx = R::add(hx, ax);
        hy = R::add(hy, ay);
        hz = R::add(hz, az);
    }

    // Euler update + renormalisation in place; returns |M x H|^2 (fp64); sets `zero` when the
    // updated magnitude is exactly zero (cell left unscaled, as the reference does).
    __device__ __forceinline__ double update(T& mx, T& my, T& mz, T hx, T hy, T hz, bool& zero) const {
        using R = RN<T>;
        const T tx = R::sub(R::mul(my, hz), R::mul(mz, hy));
        const T ty = R::sub(R::mul(mz, hx), R::mul(mx, hz));
        const T tz = R::sub(R::mul(mx, hy), R::mul(my, hx));
        const T dx = R::add(R::mul(p1, tx), R::mul(p2, R::sub(R::mul(my, tz), R::mul(mz, ty))));
        const T dy = R::add(R::mul(p1, ty), R::mul(p2, R::sub(R::mul(mz, tx), R::mul(mx, tz))));
        const T dz = R::add(R::mul(p1, tz), R::mul(p2, R::sub(R::mul(mx, ty), R::mul(my, tx))));
        const double tsq = __dadd_rn(__dadd_rn(__dmul_rn(double(tx), double(tx)), __dmul_rn(double(ty), double(ty))),
                                     __dmul_rn(double(tz), double(tz)));
        mx = R::add(mx, dx);
        my = R::add(my, dy);
        mz = R::add(mz, dz);
        const T mag = R::sqrt(R::add(R::add(R::mul(mx, mx), R::mul(my, my)), R::mul(mz, mz)));
        zero = mag == T(0);
        if (!zero) {
            const T scale = R::div(ms, mag);
            mx = R::mul(mx, scale);
            my = R::mul(my, scale);
            mz = R::mul(mz, scale);
        }
        return tsq;
    }
};

// Two horizontally adjacent cells (i, i+1) of f32 at once on packed FP32 pairs (sm_100a
// FADD2/FMUL2, each half rounded as the scalar __fadd_rn/__fmul_rn): the same operations in
// the same order as CellLLG, so each cell's H_eff and update are bitwise CellLLG's. Lane .x is
// cell i, lane .y cell i+1. sqrt, the renormalising division and the fp64 torque stay
// scalar per cell.
struct CellPairLLG {
    float2 coeff, kan, ax, ay, az, p1, p2;
    float ms;

    __device__ __forceinline__ void load(const StepCtl* ctl, float exch_coeff, float aniso_coeff) {
        const auto bc = [](float v) { return make_float2(v, v); };
        coeff = bc(exch_coeff);
        kan = bc(aniso_coeff);
        ax = bc(static_cast<float>(ctl->field[0]));
        ay = bc(static_cast<float>(ctl->field[1]));
        az = bc(static_cast<float>(ctl->field[2]));
        p1 = bc(static_cast<float>(ctl->p1));
        p2 = bc(static_cast<float>(ctl->p2));
        ms = static_cast<float>(ctl->ms);
    }

    // sum over the six neighbours of (nbr - center) in the reference's order; a missing
    // neighbour is passed as the center itself, which adds (center - center) = +0 and leaves
    // the sum unchanged (a sum that starts at +0 is never -0 under round-to-nearest)
    static __device__ __forceinline__ float2 exch(float2 ctr, const float2 (&nb)[6]) {
        float2 sum = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 6; ++q) sum = add2(sum, sub2(nb[q], ctr));
        return sum;
    }

    __device__ __forceinline__ void heff(float2 mx, float2& hx, float2& hy, float2& hz, float2 ex, float2 ey,
                                         float2 ez) const {
        hx = add2(hx, mul2(coeff, ex));
        hy = add2(hy, mul2(coeff, ey));
        hz = add2(hz, mul2(coeff, ez));
        hx = add2(hx, mul2(kan, mx));
        hx = add2(hx, ax);
        hy = add2(hy, ay);
        hz = add2(hz, az);
    }

    __device__ __forceinline__ void update(float2& mx, float2& my, float2& mz, float2 hx, float2 hy, float2 hz,
                                           double& tsq0, double& tsq1, bool& zero0, bool& zero1) const {
        const float2 tx = sub2(mul2(my, hz), mul2(mz, hy));
        const float2 ty = sub2(mul2(mz, hx), mul2(mx, hz));
        const float2 tz = sub2(mul2(mx, hy), mul2(my, hx));
        const float2 dx = add2(mul2(p1, tx), mul2(p2, sub2(mul2(my, tz), mul2(mz, ty))));
        const float2 dy = add2(mul2(p1, ty), mul2(p2, sub2(mul2(mz, tx), mul2(mx, tz))));
        const float2 dz = add2(mul2(p1, tz), mul2(p2, sub2(mul2(mx, ty), mul2(my, tx))));
        tsq0 = __dadd_rn(__dadd_rn(__dmul_rn(double(tx.x), double(tx.x)), __dmul_rn(double(ty.x), double(ty.x))),
                         __dmul_rn(double(tz.x), double(tz.x)));
        tsq1 = __dadd_rn(__dadd_rn(__dmul_rn(double(tx.y), double(tx.y)), __dmul_rn(double(ty.y), double(ty.y))),
                         __dmul_rn(double(tz.y), double(tz.y)));
        mx = add2(mx, dx);
        my = add2(my, dy);
        mz = add2(mz, dz);
        const float2 s2 = add2(add2(mul2(mx, mx), mul2(my, my)), mul2(mz, mz));
        const float mag0 = __fsqrt_rn(s2.x), mag1 = __fsqrt_rn(s2.y);
        zero0 = mag0 == 0.f;
        zero1 = mag1 == 0.f;
        // an exactly zero magnitude leaves the cell unscaled, as the reference does
        const float2 scale = make_float2(zero0 ? 1.f : __fdiv_rn(ms, mag0), zero1 ? 1.f : __fdiv_rn(ms, mag1));
        mx = mul2(mx, scale);
        my = mul2(my, scale);
        mz = mul2(mz, scale);
    }
};

} // namespace mmb
