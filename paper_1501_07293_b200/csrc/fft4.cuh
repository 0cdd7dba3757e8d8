// fft4.cuh — register-resident pruned DFTs and the two-stage ("four-step") line FFT used by
// the fast path.
//
// A length L = N1*N2 transform is done as: stage A, one task per n1 < N1 computes
// DFT_N2 over x[n1 + N1*n2] in registers and multiplies by W_L^{n1*k2}; one exchange
// through shared memory; stage B, one task per k2 < N2 computes DFT_N1 over n1, giving
// X[k2 + N2*k1] in natural order. Loads in stage A and stores in stage B are unit-stride
// across consecutive tasks (coalesced in global memory, conflict-free in shared memory),
// so a line FFT costs one shared-memory round trip.
//
// Pruning: the demag convolution's forward inputs are zero beyond the live cells
// (n >= L/2) and its inverse outputs are only needed below them, so DftP takes the number
// of leading non-zero inputs (NZ) and of leading outputs needed (NO) as compile-time
// bounds and drops the butterflies that only touch zeros or unused outputs.
#pragma once

#include "common.cuh"

namespace mmb {

__device__ __forceinline__ float fmaf_t(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double fmaf_t(double a, double b, double c) { return __fma_rn(a, b, c); }

template <int LOG2L> struct Split {
    static constexpr int L = 1 << LOG2L;
    static constexpr int N2 = 1 << ((LOG2L + 1) / 2); // stage-A DFT size (>= N1)
    static constexpr int N1 = L / N2;                 // stage-B DFT size
    static constexpr int LOG2N1 = LOG2L / 2;
};

// Pruned radix-2 DIT DFT on registers: v[0..R) in natural order -> natural order.
// Inputs v[NZ..R) are treated as zero (never read); outputs >= NO are left undefined.
template <int R, int SIGN, int NZ = R, int NO = R>
struct DftP {
    template <typename C>
    static __device__ __forceinline__ void run(C* v) {
        if constexpr (R == 1) {
            if constexpr (NZ == 0) v[0] = C{0, 0};
        } else if constexpr (NZ == 0) {
#pragma unroll
            for (int k = 0; k < R; ++k) v[k] = C{0, 0};
        } else if constexpr (NZ == 1) {
#pragma unroll
            for (int k = 1; k < R; ++k)
                if (k < NO) v[k] = v[0];
        } else {
            constexpr int H = R / 2;
            constexpr int NOH = NO < H ? NO : H;
            C e[H], o[H];
#pragma unroll
            for (int i = 0; i < H; ++i) {
                e[i] = (2 * i < NZ) ? v[2 * i] : C{0, 0};
                o[i] = (2 * i + 1 < NZ) ? v[2 * i + 1] : C{0, 0};
            }
            DftP<H, SIGN, (NZ + 1) / 2, NOH>::run(e);
            DftP<H, SIGN, NZ / 2, NOH>::run(o);
            combine<0>(v, e, o);
        }
    }
    template <int K, typename C>
    static __device__ __forceinline__ void combine(C* v, const C* e, const C* o) {
        constexpr int H = R / 2;
        if constexpr (K < H && K < NO) {
            constexpr int M = K * (64 / R);
            if constexpr (M == 0 || M == 16) {
                const C t = rot64<M, SIGN>(o[K]);
                v[K] = cadd(e[K], t);
                if constexpr (K + H < NO) v[K + H] = csub(e[K], t);
            } else {
                // FMA butterfly: W o = a (u), a = cos (|cos| >= |sin|, r = tan) or sin
                // (r = cot), u formed with 2 FFMA, outputs e +- a u with 4 FFMA: 6 FP
                // instructions instead of 8 for the twiddle product plus the two sums.
                using T = decltype(e[0].x);
                constexpr double c = (M < 16) ? kCos64[M] : -kCos64[32 - M];
                constexpr double s0 = (M < 16) ? kCos64[16 - M] : kCos64[M - 16];
                constexpr double sn = SIGN * s0;
                constexpr bool tan_form = (c < 0 ? -c : c) >= (sn < 0 ? -sn : sn);
                C u;
                T a;
                if constexpr (is_packed<C>::value) {
                    // packed: 3 FFMA2 per butterfly (operand swaps, negations and the scalar
                    // broadcasts fold into FFMA2 modifiers)
                    const C oo = o[K], osw = C{oo.y, oo.x};
                    if constexpr (tan_form) {
                        const T rr = T(sn / c);
                        a = T(c);
                        u = fma2(C{-rr, rr}, osw, oo);
                    } else {
                        const T rr = T(c / sn);
                        a = T(sn);
                        u = fma2(C{rr, rr}, oo, C{-oo.y, oo.x});
                    }
                    v[K] = fma2(C{a, a}, u, e[K]);
                    if constexpr (K + H < NO) v[K + H] = fma2(C{-a, -a}, u, e[K]);
                } else {
                    if constexpr (tan_form) {
                        const T rr = T(sn / c);
                        a = T(c);
                        u = C{fmaf_t(-rr, o[K].y, o[K].x), fmaf_t(rr, o[K].x, o[K].y)};
                    } else {
                        const T rr = T(c / sn);
                        a = T(sn);
                        u = C{fmaf_t(rr, o[K].x, -o[K].y), fmaf_t(rr, o[K].y, o[K].x)};
                    }
                    v[K] = C{fmaf_t(a, u.x, e[K].x), fmaf_t(a, u.y, e[K].y)};
                    if constexpr (K + H < NO) v[K + H] = C{fmaf_t(-a, u.x, e[K].x), fmaf_t(-a, u.y, e[K].y)};
                }
            }
            combine<K + 1>(v, e, o);
        }
    }
};

// Two-lane DFT of size 2R on the lane pair (l, l ^ XM), h = (l & XM) != 0: on entry lane h
// holds the DFT_R of x[2m + h] (its half, already transformed by DftP); on return it holds
// X[k + R h], k < R. Radix-2 combine X[k] = E[k] + W_2R^k O[k], X[k + R] = E[k] - W_2R^k O[k]:
// the odd lane twiddles, one shuffle swaps, each lane finishes its half with 2 FMA per value.
// Halves the registers of a DFT_2R task (used for DFT_64 stages, R = 32). With XM = 16 the two
// halves sit in different half-warps, so each half-warp's shared-memory accesses stay
// unit-stride across its 16 tasks. All 32 lanes must take part.
template <int R, int SIGN, int XM, int K = 0>
struct PairCombine {
    template <typename C, typename T>
    static __device__ __forceinline__ void run(C* v, int h, T sg) {
        if constexpr (K < R) {
            const C t = rot64<K * (32 / R), SIGN>(v[K]);
            const C mine = h ? t : v[K];
            const T rx = __shfl_xor_sync(0xffffffffu, mine.x, XM);
            const T ry = __shfl_xor_sync(0xffffffffu, mine.y, XM);
            if constexpr (is_packed<C>::value) v[K] = fma2(C{sg, sg}, mine, C{rx, ry});
            else v[K] = C{fmaf_t(sg, mine.x, rx), fmaf_t(sg, mine.y, ry)};
            PairCombine<R, SIGN, XM, K + 1>::run(v, h, sg);
        }
    }
};
template <int R, int SIGN, int NZH, int XM = 16, typename C>
__device__ __forceinline__ void dft_pair(C* v, int h) {
    using T = decltype(v[0].x);
    DftP<R, SIGN, NZH, R>::run(v);
    PairCombine<R, SIGN, XM>::run(v, h, h ? T(-1) : T(1));
}
// Lane-pair task mapping for dft_pair<..., 16>: half h = bit 4 of the lane, task index =
// 16 per warp.
__device__ __forceinline__ int pair_half(int t) { return (t >> 4) & 1; }
__device__ __forceinline__ int pair_task(int t) { return ((t >> 5) << 4) | (t & 15); }

// Smem index padding for a row of length L = N1*N2 processed by the four-step: one slot
// per N1 elements, so stage-B reads at stride N1 become stride N1+1 (conflict free).
template <int LOG2L>
__device__ __forceinline__ int fpad(int i) {
    return i + (i >> Split<LOG2L>::LOG2N1);
}
template <int LOG2L>
__host__ __device__ constexpr int fpitch() {
    return (1 << LOG2L) + Split<LOG2L>::N2;
}

} // namespace mmb
