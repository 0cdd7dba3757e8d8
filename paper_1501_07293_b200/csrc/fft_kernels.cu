// fft_kernels.cu — the pruned, padded-free demag convolution for sm_100a.
//
// Replaces DemagSolver<T>::compute (proj/src/demag.cpp:53-147): zero-fill + pad copy
// (:71-82), three forward c2c FFTs of the 2nx x 2ny x 2nz lattice (:83-85), the spectral
// MAC (:100-116), three inverse FFTs with the 1/P scale (:117, fft.cpp:105-112) and the
// window extraction (:119-133). Here: x-r2c on live rows only (K1), y-forward on live
// rows only (K2), z-forward + real-symmetric tensor MAC + z-inverse fused per pencil (K3),
// y-inverse keeping ny rows (K4), x-c2r keeping nx cells (K5). The padding is never stored
// and 1/P is folded into the tensor spectrum. For nz == 1 K2-K4 collapse into one fused
// y-forward / MAC / y-inverse kernel.
#include <algorithm>
#include <cstdio>
#include <stdexcept>

#include "kernels.hpp"

namespace mmb {

namespace {

constexpr int kThreads = 256;

template <typename T>
constexpr int x_pairs(int log2l) {
    const int e = sizeof(T) == 4 ? 4096 : 2048;
    const int p = e >> log2l;
    return p < 1 ? 1 : p;
}
template <typename T>
constexpr int x_smem(int log2l) {
    return x_pairs<T>(log2l) * ((1 << log2l) + ((1 << log2l) >> 4)) *
           static_cast<int>(sizeof(cx<T>));
}
// Columns (kx) per CTA for the y passes: up to 16 (8 for f64) while the tile stays within
// budget bytes.
template <typename T>
constexpr int y_width(int log2l, int comps) {
    const int budget = comps == 1 ? 65536 : 98304;
    int w = sizeof(T) == 4 ? 16 : 8;
    while (w > 1 && w * comps * (1 << log2l) * static_cast<int>(sizeof(cx<T>)) > budget) w /= 2;
    return w;
}
template <typename T>
constexpr int z_width() { return sizeof(T) == 4 ? 16 : 8; }
template <typename T>
constexpr int z_ky(int log2lz) {
    const int per = 3 * z_width<T>() * (1 << log2lz) * static_cast<int>(sizeof(cx<T>));
    int ky = 49152 / per;
    if (ky < 1) ky = 1;
    if (ky > 16) ky = 16;
    return ky;
}

__device__ __forceinline__ long long srow(const Geom& g, long long r) {
    const long long c = r / g.rows, rem = r % g.rows;
    const long long z = rem / g.ny, y = rem % g.ny;
    return ((c * g.nz + z) * g.ly + y) * g.xp;
}

// ---------------------------------------------------------------- K1: x forward (r2c)
template <typename T, int LOG2L>
__global__ void __launch_bounds__(kThreads) k_x_fwd(const T* __restrict__ m, cx<T>* __restrict__ S,
                                                    Geom g, const cx<T>* __restrict__ tw,
                                                    StepCtl* ctl, StageTable st, int prologue) {
    constexpr int L = 1 << LOG2L;
    constexpr int PAIRS = x_pairs<T>(LOG2L);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const RowLayout<T, LOG2L> lay{reinterpret_cast<cx<T>*>(smem_raw)};
    if (prologue && blockIdx.x == 0 && threadIdx.x == 0) step_prologue(ctl, st, prologue);

    const long long R = 3 * g.rows;
    const long long p0 = static_cast<long long>(blockIdx.x) * PAIRS;
    const int nlines = static_cast<int>(min(static_cast<long long>(PAIRS), (R + 1) / 2 - p0));
    const int nx = g.nx;
    auto first = [&](int line, int pos) -> cx<T> {
        const long long ra = 2 * (p0 + line), rb = ra + 1;
        if (pos >= nx) return czero<cx<T>>();
        const T a = __ldg(m + ra * nx + pos);
        const T b = rb < R ? __ldg(m + rb * nx + pos) : T(0);
        return cx<T>{a, b};
    };
    auto sstore = [&](int line, int pos, cx<T> v) { *lay.at(line, pos) = v; };
    fft_forward<T, LOG2L>(lay, nlines, tw, first, sstore);
    __syncthreads();

    // Separate the two packed real rows: A = (Z_k + conj Z_-k)/2, B = (Z_k - conj Z_-k)/(2i).
    const int xh = g.xh;
    const T half = T(0.5);
    for (int it = threadIdx.x; it < nlines * xh; it += blockDim.x) {
        const int line = it / xh, k = it - line * xh;
        const cx<T> zk = *lay.at(line, pos_of_freq<LOG2L>(k));
        const cx<T> zm = *lay.at(line, pos_of_freq<LOG2L>((L - k) & (L - 1)));
        const long long ra = 2 * (p0 + line), rb = ra + 1;
        S[srow(g, ra) + k] = cx<T>{(zk.x + zm.x) * half, (zk.y - zm.y) * half};
        if (rb < R) S[srow(g, rb) + k] = cx<T>{(zk.y + zm.y) * half, (zm.x - zk.x) * half};
    }
}

// ---------------------------------------------------------------- K5: x inverse (c2r)
template <typename T, int LOG2L>
__global__ void __launch_bounds__(kThreads) k_x_inv(const cx<T>* __restrict__ S, T* __restrict__ h,
                                                    Geom g, const cx<T>* __restrict__ tw) {
    constexpr int L = 1 << LOG2L;
    constexpr int PAIRS = x_pairs<T>(LOG2L);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const RowLayout<T, LOG2L> lay{reinterpret_cast<cx<T>*>(smem_raw)};

    const long long R = 3 * g.rows;
    const long long p0 = static_cast<long long>(blockIdx.x) * PAIRS;
    const int nlines = static_cast<int>(min(static_cast<long long>(PAIRS), (R + 1) / 2 - p0));
    const int xh = g.xh;
    // Z = A + iB on the full circle from the two Hermitian half spectra, scattered to the DIF
    // storage order the inverse expects.
    for (int it = threadIdx.x; it < nlines * xh; it += blockDim.x) {
        const int line = it / xh, k = it - line * xh;
        const long long ra = 2 * (p0 + line), rb = ra + 1;
        const cx<T> A = S[srow(g, ra) + k];
        const cx<T> B = rb < R ? S[srow(g, rb) + k] : czero<cx<T>>();
        if (k == 0 || 2 * k == L) {
            *lay.at(line, pos_of_freq<LOG2L>(k)) = cx<T>{A.x, B.x};
        } else {
            *lay.at(line, pos_of_freq<LOG2L>(k)) = cx<T>{A.x - B.y, A.y + B.x};
            *lay.at(line, pos_of_freq<LOG2L>(L - k)) = cx<T>{A.x + B.y, B.x - A.y};
        }
    }
    __syncthreads();
    const int nx = g.nx;
    auto sload = [&](int line, int pos) { return *lay.at(line, pos); };
    auto last = [&](int line, int pos, cx<T> v) {
        if (pos >= nx) return;
        const long long ra = 2 * (p0 + line), rb = ra + 1;
        h[ra * nx + pos] = v.x;
        if (rb < R) h[rb * nx + pos] = v.y;
    };
    fft_inverse<T, LOG2L>(lay, nlines, tw, sload, last);
}

// ---------------------------------------------------------------- K2 / K4: y passes
template <typename T, int LOG2L, int INVERSE>
__global__ void __launch_bounds__(kThreads) k_y(cx<T>* __restrict__ S, Geom g,
                                                const cx<T>* __restrict__ tw) {
    constexpr int W = y_width<T>(LOG2L, 1);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const ColLayout<T> lay{reinterpret_cast<cx<T>*>(smem_raw), W};
    const int kx0 = blockIdx.x * W, z = blockIdx.y, c = blockIdx.z;
    const int xh = g.xh, ny = g.ny;
    cx<T>* base = S + s_index(g, c, z, 0, kx0);
    const long long pitch = g.xp;
    if constexpr (!INVERSE) {
        auto first = [&](int line, int pos) -> cx<T> {
            return (pos < ny && kx0 + line < xh) ? base[pos * pitch + line] : czero<cx<T>>();
        };
        auto last = [&](int line, int pos, cx<T> v) {
            if (kx0 + line < xh) base[pos * pitch + line] = v;
        };
        fft_forward<T, LOG2L>(lay, W, tw, first, last);
    } else {
        auto first = [&](int line, int pos) -> cx<T> {
            return (kx0 + line < xh) ? base[pos * pitch + line] : czero<cx<T>>();
        };
        auto last = [&](int line, int pos, cx<T> v) {
            if (pos < ny && kx0 + line < xh) base[pos * pitch + line] = v;
        };
        fft_inverse<T, LOG2L>(lay, W, tw, first, last);
    }
}

// ---------------------------------------------------------------- nz == 1: y fwd + MAC + y inv
template <typename T, int LOG2L>
__global__ void __launch_bounds__(kThreads) k_y_mac(cx<T>* __restrict__ S, Geom g,
                                                    const cx<T>* __restrict__ tw, TensorSpec<T> K) {
    constexpr int L = 1 << LOG2L;
    constexpr int W = y_width<T>(LOG2L, 3);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const ColLayout<T> lay{reinterpret_cast<cx<T>*>(smem_raw), 3 * W};
    const int kx0 = blockIdx.x * W;
    const int xh = g.xh, ny = g.ny;
    const long long pitch = g.xp, cstride = static_cast<long long>(g.ly) * g.xp; // nz == 1
    cx<T>* base = S + kx0;
    auto first = [&](int line, int pos) -> cx<T> {
        const int c = line / W, col = line - c * W;
        return (pos < ny && kx0 + col < xh) ? base[c * cstride + pos * pitch + col] : czero<cx<T>>();
    };
    auto sstore = [&](int line, int pos, cx<T> v) { *lay.at(line, pos) = v; };
    fft_forward<T, LOG2L>(lay, 3 * W, tw, first, sstore);
    __syncthreads();
    for (int it = threadIdx.x; it < W * L; it += blockDim.x) {
        const int col = it % W, pos = it / W;
        const int kx = kx0 + col;
        if (kx >= xh) continue;
        T k6[6];
        K.at(g, kx, freq_of_pos<LOG2L>(pos), 0, k6);
        cx<T>* a = lay.at(col, pos);
        cx<T>* b = lay.at(W + col, pos);
        cx<T>* cc = lay.at(2 * W + col, pos);
        cx<T> va = *a, vb = *b, vc = *cc;
        mac3<T>(k6, va, vb, vc);
        *a = va;
        *b = vb;
        *cc = vc;
    }
    __syncthreads();
    auto sload = [&](int line, int pos) { return *lay.at(line, pos); };
    auto last = [&](int line, int pos, cx<T> v) {
        const int c = line / W, col = line - c * W;
        if (pos < ny && kx0 + col < xh) base[c * cstride + pos * pitch + col] = v;
    };
    fft_inverse<T, LOG2L>(lay, 3 * W, tw, sload, last);
}

// ---------------------------------------------------------------- K3: z fwd + MAC + z inv
template <typename T, int LOG2LZ>
__global__ void __launch_bounds__(kThreads) k_z_mac(cx<T>* __restrict__ S, Geom g,
                                                    const cx<T>* __restrict__ tw, TensorSpec<T> K) {
    constexpr int LZ = 1 << LOG2LZ;
    constexpr int W = z_width<T>(), KY = z_ky<T>(LOG2LZ), WK = W * KY, NC = 3 * WK;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const ColLayout<T> lay{reinterpret_cast<cx<T>*>(smem_raw), NC};
    const int kx0 = blockIdx.x * W, ky0 = blockIdx.y * KY;
    const int xh = g.xh, ly = g.ly, nz = g.nz;
    const long long zpitch = static_cast<long long>(g.ly) * g.xp;
    auto addr = [&](int line, int z, bool& ok) -> long long {
        const int c = line / WK, rem = line - c * WK, kyl = rem / W, col = rem - kyl * W;
        ok = (kx0 + col < xh) && (ky0 + kyl < ly);
        return s_index(g, c, 0, ky0 + kyl, kx0 + col) + z * zpitch;
    };
    auto first = [&](int line, int pos) -> cx<T> {
        bool ok;
        const long long a = addr(line, pos, ok);
        return (ok && pos < nz) ? S[a] : czero<cx<T>>();
    };
    auto sstore = [&](int line, int pos, cx<T> v) { *lay.at(line, pos) = v; };
    fft_forward<T, LOG2LZ>(lay, NC, tw, first, sstore);
    __syncthreads();
    for (int it = threadIdx.x; it < WK * LZ; it += blockDim.x) {
        const int cl = it % WK, pos = it / WK;
        const int kyl = cl / W, col = cl - kyl * W;
        const int kx = kx0 + col, kys = ky0 + kyl;
        if (kx >= xh || kys >= ly) continue;
        T k6[6];
        K.at(g, kx, freq_of_pos_rt(kys, g.log2ly), freq_of_pos<LOG2LZ>(pos), k6);
        cx<T>* a = lay.at(cl, pos);
        cx<T>* b = lay.at(WK + cl, pos);
        cx<T>* cc = lay.at(2 * WK + cl, pos);
        cx<T> va = *a, vb = *b, vc = *cc;
        mac3<T>(k6, va, vb, vc);
        *a = va;
        *b = vb;
        *cc = vc;
    }
    __syncthreads();
    auto sload = [&](int line, int pos) { return *lay.at(line, pos); };
    auto last = [&](int line, int pos, cx<T> v) {
        bool ok;
        const long long a = addr(line, pos, ok);
        if (ok && pos < nz) S[a] = v;
    };
    fft_inverse<T, LOG2LZ>(lay, NC, tw, sload, last);
}

template <typename K>
void set_smem(K kernel, int bytes) {
    if (bytes > 48 * 1024) {
        const cudaError_t e =
            cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) throw std::runtime_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    }
}

#define MMB_LOG2_CASES(X) \
    X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12)

void bad_len(int l) {
    throw std::invalid_argument("mmb: unsupported padded FFT length 2^" + std::to_string(l) +
                                " (max 4096 per axis)");
}

void check_launch() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e));
}

} // namespace

template <typename T>
void prepare_fft_kernels(const Geom& g) {
    switch (g.log2lx) {
#define X(l) case l: set_smem(k_x_fwd<T, l>, x_smem<T>(l)); set_smem(k_x_inv<T, l>, x_smem<T>(l)); break;
        MMB_LOG2_CASES(X)
#undef X
        default: bad_len(g.log2lx);
    }
    if (g.nz == 1) {
        switch (g.log2ly) {
#define X(l) case l: set_smem(k_y_mac<T, l>, 3 * y_width<T>(l, 3) * (1 << l) * (int)sizeof(cx<T>)); break;
            MMB_LOG2_CASES(X)
#undef X
            default: bad_len(g.log2ly);
        }
    } else {
        switch (g.log2ly) {
#define X(l) case l: set_smem(k_y<T, l, 0>, y_width<T>(l, 1) * (1 << l) * (int)sizeof(cx<T>)); \
                     set_smem(k_y<T, l, 1>, y_width<T>(l, 1) * (1 << l) * (int)sizeof(cx<T>)); break;
            MMB_LOG2_CASES(X)
#undef X
            default: bad_len(g.log2ly);
        }
        switch (g.log2lz) {
#define X(l) case l: set_smem(k_z_mac<T, l>, 3 * z_width<T>() * z_ky<T>(l) * (1 << l) * (int)sizeof(cx<T>)); break;
            MMB_LOG2_CASES(X)
#undef X
            default: bad_len(g.log2lz);
        }
    }
}

template <typename T>
void launch_x_fwd(const T* m, cx<T>* S, const Geom& g, const cx<T>* tw, StepCtl* ctl,
                  const StageTable& st, int prologue, cudaStream_t stream) {
    const long long npairs = (3 * g.rows + 1) / 2;
    switch (g.log2lx) {
#define X(l) case l: { const int P = x_pairs<T>(l); \
        k_x_fwd<T, l><<<(unsigned)((npairs + P - 1) / P), kThreads, x_smem<T>(l), stream>>>(m, S, g, tw, ctl, st, prologue); break; }
        MMB_LOG2_CASES(X)
#undef X
        default: bad_len(g.log2lx);
    }
    check_launch();
}

template <typename T>
void launch_x_inv(const cx<T>* S, T* h, const Geom& g, const cx<T>* tw, cudaStream_t stream) {
    const long long npairs = (3 * g.rows + 1) / 2;
    switch (g.log2lx) {
#define X(l) case l: { const int P = x_pairs<T>(l); \
        k_x_inv<T, l><<<(unsigned)((npairs + P - 1) / P), kThreads, x_smem<T>(l), stream>>>(S, h, g, tw); break; }
        MMB_LOG2_CASES(X)
#undef X
        default: bad_len(g.log2lx);
    }
    check_launch();
}

template <typename T>
void launch_y(int inverse, cx<T>* S, const Geom& g, const cx<T>* tw, cudaStream_t stream) {
    switch (g.log2ly) {
#define X(l) case l: { constexpr int W = y_width<T>(l, 1); \
        const dim3 grid((g.xh + W - 1) / W, g.nz, 3); const int sm = W * (1 << l) * (int)sizeof(cx<T>); \
        if (inverse) k_y<T, l, 1><<<grid, kThreads, sm, stream>>>(S, g, tw); \
        else k_y<T, l, 0><<<grid, kThreads, sm, stream>>>(S, g, tw); break; }
        MMB_LOG2_CASES(X)
#undef X
        default: bad_len(g.log2ly);
    }
    check_launch();
}

template <typename T>
void launch_y_mac(cx<T>* S, const Geom& g, const cx<T>* tw, const T* kspec, cudaStream_t stream) {
    const TensorSpec<T> K{kspec, static_cast<long long>(g.zh) * g.yh * g.xh};
    switch (g.log2ly) {
#define X(l) case l: { constexpr int W = y_width<T>(l, 3); \
        k_y_mac<T, l><<<(g.xh + W - 1) / W, kThreads, 3 * W * (1 << l) * (int)sizeof(cx<T>), stream>>>(S, g, tw, K); break; }
        MMB_LOG2_CASES(X)
#undef X
        default: bad_len(g.log2ly);
    }
    check_launch();
}

template <typename T>
void launch_z_mac(cx<T>* S, const Geom& g, const cx<T>* tw, const T* kspec, cudaStream_t stream) {
    const TensorSpec<T> K{kspec, static_cast<long long>(g.zh) * g.yh * g.xh};
    switch (g.log2lz) {
#define X(l) case l: { constexpr int W = z_width<T>(), KY = z_ky<T>(l); \
        const dim3 grid((g.xh + W - 1) / W, (g.ly + KY - 1) / KY); \
        k_z_mac<T, l><<<grid, kThreads, 3 * W * KY * (1 << l) * (int)sizeof(cx<T>), stream>>>(S, g, tw, K); break; }
        MMB_LOG2_CASES(X)
#undef X
        default: bad_len(g.log2lz);
    }
    check_launch();
}

#define MMB_INST(T)                                                                               \
    template void prepare_fft_kernels<T>(const Geom&);                                           \
    template void launch_x_fwd<T>(const T*, cx<T>*, const Geom&, const cx<T>*, StepCtl*,          \
                                  const StageTable&, int, cudaStream_t);                          \
    template void launch_x_inv<T>(const cx<T>*, T*, const Geom&, const cx<T>*, cudaStream_t);     \
    template void launch_y<T>(int, cx<T>*, const Geom&, const cx<T>*, cudaStream_t);              \
    template void launch_y_mac<T>(cx<T>*, const Geom&, const cx<T>*, const T*, cudaStream_t);     \
    template void launch_z_mac<T>(cx<T>*, const Geom&, const cx<T>*, const T*, cudaStream_t);
#ifndef MMB_ONLY_F64
MMB_INST(float)
#endif
#ifndef MMB_ONLY_F32
MMB_INST(double)
#endif

} // namespace mmb
