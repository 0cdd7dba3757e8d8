// common.cuh — complex helpers, register DFTs and in-place shared-memory FFT passes for the
// B200 demag convolution (sm_100a).
//
// All per-axis transforms are power-of-two, in place, radix-16 (last pass radix 2/4/8):
//   forward = decimation in frequency (natural order in -> digit-reversed order out),
//   inverse = decimation in time      (digit-reversed in -> natural order out, unnormalised).
// The convolution never needs natural-order spectra except along x, where the r2c / c2r
// post-/pre-processing gathers through pos_of_freq(). This replaces the reference's full
// c2c FFTW transforms of the zero-padded lattice (proj/src/fft.cpp:98-112,
// proj/src/demag.cpp:67-85,117-133): the padding is never materialised — the first forward
// pass predicates its loads on the live input length and the last inverse pass stores only
// the live output window.
#pragma once

#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

namespace mmb {

template <typename T> struct V2;
template <> struct V2<float> { using type = float2; };
template <> struct V2<double> { using type = double2; };
template <typename T> using cx = typename V2<T>::type;

// ---- packed fp32 pairs (sm_100a FADD2 / FMUL2 / FFMA2): one instruction for both halves of a
// float2, each half rounded exactly as the scalar operation. ptxas folds the swaps, negations
// and scalar broadcasts below into operand modifiers, so a complex add is one instruction and
// a complex product two.
__device__ __forceinline__ unsigned long long f2_bits(float2 a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 f2_val(unsigned long long v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_val(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_val(r);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_val(r);
}
// a * b + c per half, fused (one rounding)
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
    return f2_val(r);
}

template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return {a.x + b.x, a.y + b.y}; }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return {a.x - b.x, a.y - b.y}; }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
    return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
// a * conj(b)
template <typename C> __device__ __forceinline__ C cmulc(C a, C b) {
    return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
// Register complex type of the kernels that use packed arithmetic (chosen per kernel: it pays
// in the fused y/z and x-step kernels up to L = 1024, not in the lane-pair DFT_64 and
// streaming kernels). Same layout as float2, converts both ways.
struct __align__(8) pf2 {
    float x, y;
    pf2() = default;
    __device__ __forceinline__ constexpr pf2(float a, float b) : x(a), y(b) {}
    __device__ __forceinline__ pf2(float2 v) : x(v.x), y(v.y) {}
    __device__ __forceinline__ operator float2() const { return make_float2(x, y); }
};
template <typename C> struct is_packed { static constexpr bool value = false; };
template <> struct is_packed<pf2> { static constexpr bool value = true; };
// the register complex type of a kernel on T at transform length 2^LOG2L
template <typename T, int LOG2L>
using rcx = typename std::conditional<(sizeof(T) == 4 && LOG2L <= 10), pf2, cx<T>>::type;

__device__ __forceinline__ pf2 fma2(pf2 a, pf2 b, pf2 c) { return fma2(float2(a), float2(b), float2(c)); }
// packed: (a.x b.x - a.y b.y, a.x b.y + a.y b.x) = a.x (b.x, b.y) + a.y (-b.y, b.x)
template <> __device__ __forceinline__ pf2 cadd(pf2 a, pf2 b) { return add2(a, b); }
template <> __device__ __forceinline__ pf2 csub(pf2 a, pf2 b) { return sub2(a, b); }
template <> __device__ __forceinline__ pf2 cmul(pf2 a, pf2 b) {
    return fma2(make_float2(a.y, a.y), make_float2(-b.y, b.x), mul2(make_float2(a.x, a.x), b));
}
// (a.x b.x + a.y b.y, a.y b.x - a.x b.y) = a.x (b.x, -b.y) + a.y (b.y, b.x)
template <> __device__ __forceinline__ pf2 cmulc(pf2 a, pf2 b) {
    return fma2(make_float2(a.y, a.y), make_float2(b.y, b.x), mul2(make_float2(a.x, a.x), make_float2(b.x, -b.y)));
}
template <typename C> __device__ __forceinline__ C czero() { return {0, 0}; }

// ---------------------------------------------------------------- compile-time radix plan
// Radix of pass p for a length 2^LOG2L transform: 16 for every full nibble, then the
// remainder (2, 4 or 8).
__host__ __device__ constexpr int num_passes(int log2l) { return (log2l + 3) / 4; }
__host__ __device__ constexpr int pass_log2r(int log2l, int p) {
    return (p < log2l / 4) ? 4 : (log2l % 4);
}

// Frequency k <-> storage position after the forward DIF.
template <int LOG2L>
__device__ __forceinline__ int pos_of_freq(int k) {
    int p = 0, s = LOG2L;
#pragma unroll
    for (int q = 0; q < num_passes(LOG2L); ++q) {
        const int lr = pass_log2r(LOG2L, q);
        s -= lr;
        p += (k & ((1 << lr) - 1)) << s;
        k >>= lr;
    }
    return p;
}
template <int LOG2L>
__device__ __forceinline__ int freq_of_pos(int p) {
    int k = 0, shift = 0, s = LOG2L;
#pragma unroll
    for (int q = 0; q < num_passes(LOG2L); ++q) {
        const int lr = pass_log2r(LOG2L, q);
        s -= lr;
        k += ((p >> s) & ((1 << lr) - 1)) << shift;
        shift += lr;
    }
    return k;
}

// ---------------------------------------------------------------- register DFTs
// cos(2 pi m / 64), m = 0..16 (quarter wave).
__device__ constexpr double kCos64[17] = {
    1.0,
    0.99518472667219688624483695310948,
    0.98078528040323044912618223613424,
    0.95694033573220886493579788698027,
    0.92387953251128675612818318939679,
    0.88192126434835502971275686366039,
    0.83146961230254523707878837761791,
    0.77301045336273696081090660975847,
    0.70710678118654752440084436210485,
    0.63439328416364549821517161322549,
    0.55557023301960222474283081394853,
    0.47139673682599764855638762590525,
    0.38268343236508977172845998403040,
    0.29028467725446236763619237581740,
    0.19509032201612826784828486847702,
    0.09801714032956060199419556388864,
    0.0};

// x * exp(SIGN * 2 pi i * M / 64), M in [0, 32)
template <int M, int SIGN, typename C>
__device__ __forceinline__ C rot64(C x) {
    using T = decltype(x.x);
    if constexpr (M == 0) {
        return x;
    } else if constexpr (M == 16) {
        if constexpr (SIGN < 0) return C{x.y, -x.x};
        else return C{-x.y, x.x};
    } else {
        constexpr double c = (M < 16) ? kCos64[M] : -kCos64[32 - M];
        constexpr double s0 = (M < 16) ? kCos64[16 - M] : kCos64[M - 16];
        const T cc = T(c), ss = T(SIGN * s0);
        if constexpr (is_packed<C>::value) return cmul(x, C{cc, ss});
        else return C{x.x * cc - x.y * ss, x.x * ss + x.y * cc};
    }
}

template <int R, int SIGN, typename C>
struct Dft {
    static __device__ __forceinline__ void run(C* v) {
        C e[R / 2], o[R / 2];
#pragma unroll
        for (int i = 0; i < R / 2; ++i) {
            e[i] = v[2 * i];
            o[i] = v[2 * i + 1];
        }
        Dft<R / 2, SIGN, C>::run(e);
        Dft<R / 2, SIGN, C>::run(o);
        apply<0>(v, e, o);
    }
    template <int K>
    static __device__ __forceinline__ void apply(C* v, const C* e, const C* o) {
        if constexpr (K < R / 2) {
            const C t = rot64<K * (64 / R), SIGN>(o[K]);
            v[K] = cadd(e[K], t);
            v[K + R / 2] = csub(e[K], t);
            apply<K + 1>(v, e, o);
        }
    }
};
template <int SIGN, typename C>
struct Dft<1, SIGN, C> {
    static __device__ __forceinline__ void run(C*) {}
};

// ---------------------------------------------------------------- layouts
// Row layout: lines are contiguous runs of L elements, one padding slot per 16 elements so
// the small-stride passes stay bank-conflict free. Threads map to consecutive positions.
template <typename T, int LOG2L>
struct RowLayout {
    cx<T>* base;
    static constexpr bool kColFast = false;
    static constexpr int kStride = (1 << LOG2L) + ((1 << LOG2L) >> 4);
    static __host__ __device__ constexpr int words(int nlines) { return nlines * kStride; }
    __device__ __forceinline__ cx<T>* at(int line, int pos) const {
        return base + line * kStride + pos + (pos >> 4);
    }
};
// Column layout: element (line, pos) at pos * NC + line; threads map to consecutive lines.
template <typename T>
struct ColLayout {
    cx<T>* base;
    int nc;
    static constexpr bool kColFast = true;
    __device__ __forceinline__ cx<T>* at(int line, int pos) const { return base + pos * nc + line; }
};

// Decompose work item g into (line, group-in-line) for a pass with G groups per line.
template <bool COLFAST>
__device__ __forceinline__ void split_item(int g, int nlines, int G, int& line, int& q) {
    if constexpr (COLFAST) {
        line = g % nlines;
        q = g / nlines;
    } else {
        line = g / G;
        q = g % G;
    }
}

// ---------------------------------------------------------------- one in-place pass
// Forward DIF pass with block size N = 2^LOG2N and radix R = 2^LOG2R (s = N/R):
//   v[q] = x[b N + j + q s];  V = DFT_R(v);  x[b N + j + r s] = V[r] * W_N^{j r}.
// LOAD(line, pos, valid) supplies the input (for the first pass: straight from global
// memory), STORE(line, pos, value) consumes the output.
template <typename T, int LOG2L, int LOG2N, int LOG2R, bool COLFAST, class Load, class Store>
__device__ __forceinline__ void dif_pass(int nlines, const cx<T>* __restrict__ tw, Load load,
                                         Store store) {
    constexpr int L = 1 << LOG2L, N = 1 << LOG2N, R = 1 << LOG2R, S = N / R;
    constexpr int G = L / R;
    const int items = nlines * G;
    for (int g = threadIdx.x; g < items; g += blockDim.x) {
        int line, q;
        split_item<COLFAST>(g, nlines, G, line, q);
        const int b = q / S, j = q % S;
        const int p0 = b * N + j;
        cx<T> v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = load(line, p0 + r * S);
        Dft<R, -1, cx<T>>::run(v);
#pragma unroll
        for (int r = 1; r < R; ++r) v[r] = cmul(v[r], __ldg(&tw[(j * r) << (LOG2L - LOG2N)]));
#pragma unroll
        for (int r = 0; r < R; ++r) store(line, p0 + r * S, v[r]);
    }
}

// Inverse DIT pass (exact inverse of dif_pass up to a factor R):
//   v[r] = x[b N + j + r s] * conj(W_N^{j r});  V = IDFT_R(v);  x[b N + j + q s] = V[q].
template <typename T, int LOG2L, int LOG2N, int LOG2R, bool COLFAST, class Load, class Store>
__device__ __forceinline__ void dit_pass(int nlines, const cx<T>* __restrict__ tw, Load load,
                                         Store store) {
    constexpr int L = 1 << LOG2L, N = 1 << LOG2N, R = 1 << LOG2R, S = N / R;
    constexpr int G = L / R;
    const int items = nlines * G;
    for (int g = threadIdx.x; g < items; g += blockDim.x) {
        int line, q;
        split_item<COLFAST>(g, nlines, G, line, q);
        const int b = q / S, j = q % S;
        const int p0 = b * N + j;
        cx<T> v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = load(line, p0 + r * S);
#pragma unroll
        for (int r = 1; r < R; ++r) v[r] = cmulc(v[r], __ldg(&tw[(j * r) << (LOG2L - LOG2N)]));
        Dft<R, +1, cx<T>>::run(v);
#pragma unroll
        for (int r = 0; r < R; ++r) store(line, p0 + r * S, v[r]);
    }
}

// Block size before pass P (N_0 = L).
__host__ __device__ constexpr int log2n_at(int log2l, int p) {
    int n = log2l;
    for (int q = 0; q < p; ++q) n -= pass_log2r(log2l, q);
    return n;
}

// Full forward transform: FIRST load functor for pass 0, smem layout for the middle passes,
// LAST store functor for the final pass. Barriers between passes.
template <typename T, int LOG2L, class Layout, class FirstLoad, class LastStore, int P = 0>
__device__ __forceinline__ void fft_forward(const Layout& lay, int nlines, const cx<T>* tw,
                                           FirstLoad first, LastStore last) {
    constexpr int NP = num_passes(LOG2L);
    if constexpr (NP == 0) {
        // length 1: identity
        for (int g = threadIdx.x; g < nlines; g += blockDim.x) last(g, 0, first(g, 0));
    } else if constexpr (P < NP) {
        constexpr int LN = log2n_at(LOG2L, P), LR = pass_log2r(LOG2L, P);
        auto sload = [&](int line, int pos) { return *lay.at(line, pos); };
        auto sstore = [&](int line, int pos, cx<T> v) { *lay.at(line, pos) = v; };
        if constexpr (NP == 1) {
            dif_pass<T, LOG2L, LN, LR, Layout::kColFast>(nlines, tw, first, last);
        } else if constexpr (P == 0) {
            dif_pass<T, LOG2L, LN, LR, Layout::kColFast>(nlines, tw, first, sstore);
            __syncthreads();
        } else if constexpr (P == NP - 1) {
            dif_pass<T, LOG2L, LN, LR, Layout::kColFast>(nlines, tw, sload, last);
        } else {
            dif_pass<T, LOG2L, LN, LR, Layout::kColFast>(nlines, tw, sload, sstore);
            __syncthreads();
        }
        if constexpr (P + 1 < NP) fft_forward<T, LOG2L, Layout, FirstLoad, LastStore, P + 1>(lay, nlines, tw, first, last);
    }
}

// Full inverse transform: passes NP-1 .. 0; FIRST load functor feeds pass NP-1, LAST store
// functor consumes pass 0 (natural order positions).
template <typename T, int LOG2L, class Layout, class FirstLoad, class LastStore, int P = num_passes(LOG2L) - 1>
__device__ __forceinline__ void fft_inverse(const Layout& lay, int nlines, const cx<T>* tw,
                                            FirstLoad first, LastStore last) {
    constexpr int NP = num_passes(LOG2L);
    if constexpr (NP == 0) {
        for (int g = threadIdx.x; g < nlines; g += blockDim.x) last(g, 0, first(g, 0));
    } else if constexpr (P >= 0) {
        constexpr int LN = log2n_at(LOG2L, P), LR = pass_log2r(LOG2L, P);
        auto sload = [&](int line, int pos) { return *lay.at(line, pos); };
        auto sstore = [&](int line, int pos, cx<T> v) { *lay.at(line, pos) = v; };
        if constexpr (NP == 1) {
            dit_pass<T, LOG2L, LN, LR, Layout::kColFast>(nlines, tw, first, last);
        } else if constexpr (P == NP - 1) {
            dit_pass<T, LOG2L, LN, LR, Layout::kColFast>(nlines, tw, first, sstore);
            __syncthreads();
        } else if constexpr (P == 0) {
            dit_pass<T, LOG2L, LN, LR, Layout::kColFast>(nlines, tw, sload, last);
        } else {
            dit_pass<T, LOG2L, LN, LR, Layout::kColFast>(nlines, tw, sload, sstore);
            __syncthreads();
        }
        if constexpr (P > 0) fft_inverse<T, LOG2L, Layout, FirstLoad, LastStore, P - 1>(lay, nlines, tw, first, last);
    }
}

} // namespace mmb
