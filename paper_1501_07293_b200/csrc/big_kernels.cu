// big_kernels.cu — the fast path for grids whose per-kx spectrum block does not fit in shared
// memory (nz > 8, e.g. 1024x1024x32 and the 2048x2048x64 slabs): the y/z part of the
// convolution is split into three streaming kernels around a padded spectrum S2:
//
//   KYF (k_yrow, forward): per (kx, c, z) row, y-FFT of the ny live values -> Ly values (S -> S2)
//   KZ  (k_zmac)         : per (kx, ky) pencil tile, z-FFT (nz -> Lz, pruned), 6-component
//                          tensor MAC, z-inverse (Lz -> nz), in place in S2
//   KYI (k_yrow, inverse): per row, Ly -> ny live values (S2 -> S)
//
// then the fused KXS (fast_kernels.cu) as on the small-nz path. All row transforms are the
// register four-step of fft4.cuh with unit-stride global loads/stores.
#include <cstdio>
#include <stdexcept>
#include <type_traits>
#include <string>

#include "fast.hpp"
#include "fast_common.cuh"

namespace mmb {

namespace {

void check_launch() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e));
}

// Rows per CTA: every thread has exactly one stage-A task. DFT_64 stages run on lane pairs
// (dft_pair: 32 values per lane instead of 64), so LA / LB lanes share a stage-A / stage-B
// task; stage B loops when it has more tasks than threads.
template <int LOG2L>
struct YR {
    using SP = Split<LOG2L>;
    static constexpr int LA = SP::N2 == 64 ? 2 : 1, LB = SP::N1 == 64 ? 2 : 1;
    static constexpr int NT = 256;
    static constexpr int P = NT / (SP::N1 * LA);
    static constexpr int EX = SP::N1 + 1;
    static_assert(P >= 1 && P * SP::N1 * LA == NT, "row tile");
};
template <typename T, int LOG2L>
constexpr int yr_smem_bytes() {
    using Y = YR<LOG2L>;
    return (Y::P * Split<LOG2L>::N2 * Y::EX + (1 << LOG2L)) * static_cast<int>(sizeof(cx<T>));
}

// Row FFT along y. INV = 0: in rows hold n_live values (pitch in_pitch), out rows get all L
// values. INV = 1: in rows hold L values, out rows get the first n_live values.
template <typename T, int LOG2L, int INV, bool PEER = false>
__global__ void __launch_bounds__(YR<LOG2L>::NT)
    k_yrow(const cx<T>* __restrict__ in, cx<T>* __restrict__ out, long long nrows, int in_pitch,
           int out_pitch, int n_live, const cx<T>* __restrict__ tw, StepCtl* ctl, StageTable st,
           int prologue, const __grid_constant__ RowMap<T> rm, int nzr) {
    using SP = Split<LOG2L>;
    using Y = YR<LOG2L>;
    constexpr int L = SP::L, N1 = SP::N1, N2 = SP::N2, P = Y::P, EX = Y::EX, NT = Y::NT;
    constexpr int LA = Y::LA, LB = Y::LB, RA = N2 / LA, RB = N1 / LB;
    constexpr int SIGN = INV ? +1 : -1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw);
    cx<T>* tws = sm + P * N2 * EX;
    if (prologue && blockIdx.x == 0 && threadIdx.x == 0) step_prologue(ctl, st, prologue);
    stage_twiddles<T, LOG2L>(tws, tw);
    cp_async_wait_all();
    __syncthreads();
    const int tid = threadIdx.x;
    const long long r0 = static_cast<long long>(blockIdx.x) * P;
    {
        // stage A: lane h of the task takes n2 = LA m + h
        const int h = LA == 2 ? pair_half(tid) : 0, task = LA == 2 ? pair_task(tid) : tid;
        const int p = task / N1, n1 = task % N1;
        const long long r = r0 + p;
        cx<T> v[RA];
        constexpr int NZ = INV ? RA : (RA / 2 > 0 ? RA / 2 : 1); // forward: n2 < N2 / 2 live
#pragma unroll
        for (int m = 0; m < RA; ++m) v[m] = cx<T>{0, 0};
        if (r < nrows) {
            // forward rows may live in the ranks' slab spectra (RowMap; row = (kx, c, z))
            const cx<T>* src = (!INV && PEER) ? rm.row(static_cast<int>(r / (3 * nzr)), static_cast<int>(r / nzr % 3),
                                                           static_cast<int>(r % nzr), in_pitch)
                                                  : in + r * in_pitch;
#pragma unroll
            for (int m = 0; m < NZ; ++m) {
                const int y = n1 + N1 * (LA * m + h);
                v[m] = (INV || y < n_live) ? src[y] : cx<T>{0, 0};
            }
        }
        if constexpr (LA == 2) dft_pair<RA, SIGN, NZ>(v, h);
        else DftP<N2, SIGN, NZ, N2>::run(v);
        cx<T>* ex = sm + (p * N2) * EX + n1;
#pragma unroll
        for (int kk = 0; kk < RA; ++kk) {
            const int k2 = kk + RA * h;
            cx<T> w = v[kk];
            if (k2 > 0) w = INV ? cmulc(w, tws[k2 * N1 + n1]) : cmul(w, tws[k2 * N1 + n1]);
            ex[k2 * EX] = w;
        }
    }
    __syncthreads();
    // stage B: lane h of the task takes n1 = LB q + h; rows past nrows compute on zeros and
    // skip only their stores (the pair shuffles need every lane)
    for (int tb = tid; tb < P * N2 * LB; tb += NT) {
        const int h = LB == 2 ? pair_half(tb) : 0, task = LB == 2 ? pair_task(tb) : tb;
        const int p = task / N2, k2 = task % N2;
        const long long r = r0 + p;
        cx<T> u[RB];
        const cx<T>* ex = sm + (p * N2 + k2) * EX + h;
#pragma unroll
        for (int q = 0; q < RB; ++q) u[q] = ex[LB * q];
        if constexpr (LB == 2) dft_pair<RB, SIGN, RB>(u, h);
        else DftP<N1, SIGN, N1, (INV && N1 > 1) ? N1 / 2 : N1>::run(u);
        if (r < nrows) {
            cx<T>* dst = (INV && PEER) ? rm.row(static_cast<int>(r / (3 * nzr)), static_cast<int>(r / nzr % 3),
                                                    static_cast<int>(r % nzr), out_pitch)
                                           : out + r * out_pitch;
#pragma unroll
            for (int q = 0; q < RB; ++q) {
                const int k1 = q + RB * h;
                const int y = k2 + N2 * k1;
                if (!INV) {
                    dst[y] = u[q];
                } else if (k1 < (N1 > 1 ? N1 / 2 : 1) && y < n_live) {
                    dst[y] = u[q];
                }
            }
        }
    }
}

// z pencils: W consecutive ky of one kx, all three components, Lz = 2^LOG2LZ >= 2 nz - 1.
// pencils per CTA: 32 (f32) keeps the tile at 98 KB (two CTAs per SM) up to Lz = 64; the
// Lz = 128 and 256 tiles halve / quarter it for the same occupancy
#ifndef MMB_ZW_SHIFT8
#define MMB_ZW_SHIFT8 1 // pencils per CTA at Lz = 256: 32 >> 1 = 16 (f32)
#endif
#ifndef MMB_ZW_SHIFT7
#define MMB_ZW_SHIFT7 1 // pencils per CTA at Lz = 128: 32 >> 1 = 16 (f32)
#endif
template <typename T, int LOG2LZ>
constexpr int zw() { return (sizeof(T) == 4 ? 32 : 16) >> (LOG2LZ >= 8 ? MMB_ZW_SHIFT8 : (LOG2LZ >= 7 ? MMB_ZW_SHIFT7 : 0)); }
constexpr int kZThreads = 256;
template <typename T, int LOG2LZ>
constexpr int z_smem_bytes() {
    return (2 * 3 * (1 << LOG2LZ) * zw<T, LOG2LZ>() + (1 << LOG2LZ)) * static_cast<int>(sizeof(cx<T>));
}

template <typename T, int LOG2LZ>
__global__ void __launch_bounds__(kZThreads)
    k_zmac(cx<T>* __restrict__ S2, Geom g, const cx<T>* __restrict__ tw, const T* __restrict__ kt,
           const __grid_constant__ CUtensorMap tm, int use_tma) {
    // Lz = N1*N2. Forward: stage A (DFT_N2 over n2 per (c, n1)), then the fused middle: per
    // (k2, ky) all three components in registers, DFT_N1 -> kz = k2 + N2 k1 natural, tensor
    // MAC, inverse DFT_N1, conj twiddle; then inverse stage A' (IDFT_N2 per (c, n1)) straight
    // to the nz live planes. Two shared buffers (A: [c][z][w], B: exchange), three barriers.
    using SP = Split<LOG2LZ>;
    constexpr int LZ = SP::L, N1 = SP::N1, N2 = SP::N2, W = zw<T, LOG2LZ>();
    constexpr int CS = LZ * W; // component stride in a tile buffer
    extern __shared__ __align__(128) unsigned char zm_smem[]; // 128 B: TMA box destinations
    cx<T>* A = reinterpret_cast<cx<T>*>(zm_smem); // [c][z][w]
    cx<T>* B = A + 3 * CS;
    cx<T>* tws = B + 3 * CS;
    const int kx = blockIdx.y, ky0 = blockIdx.x * W;
    const int nz = g.nz, ly = g.ly, yh = g.yh, zh = g.zh;
    const int wl = min(W, ly - ky0);
    const int tid = threadIdx.x;
    const long long zpitch = ly;
    cx<T>* blk = S2 + static_cast<long long>(kx) * 3 * nz * ly + ky0;

    // load the nz live planes (async, coalesced over ky): each thread keeps its w and walks
    // the (c, z) planes with a fixed stride, carrying (c, z) instead of dividing
    // Whole tiles (Ly a multiple of W) move VEC consecutive ky per 16-byte copy.
    auto load_tile = [&](auto vec) {
        constexpr int VEC = decltype(vec)::value;
        constexpr int TW = W / VEC; // threads per (c, z) row
        static_assert(kZThreads % TW == 0, "pencil tile");
        constexpr int CZSTEP = kZThreads / TW;
        const int w = (tid % TW) * VEC;
        int c = 0, z = tid / TW;
        while (z >= nz) {
            z -= nz;
            ++c;
        }
        const cx<T>* src = blk + static_cast<long long>(tid / TW) * zpitch + w;
        for (int cz = tid / TW; cz < 3 * nz; cz += CZSTEP) {
            cx<T>* d = A + (c * LZ + z) * W + w;
            if (VEC > 1) cp_async<16>(d, src);
            else if (w < wl) cp_async<sizeof(cx<T>)>(d, src);
            else *d = cx<T>{0, 0};
            src += CZSTEP * zpitch;
            z += CZSTEP;
            while (z >= nz) {
                z -= nz;
                ++c;
            }
        }
    };
    __shared__ __align__(8) unsigned long long zbar;
    if (use_tma) {
        // one TMA box per component: W ky x nz planes of row (c, 0..nz) at kx -> A[c][z][w]
        // (the planes z >= nz of the tile are never read; ky past Ly arrive as zeros)
        if (tid == 0) {
            mbar_init(&zbar, 1);
            mbar_expect_tx(&zbar, 3u * nz * W * static_cast<unsigned>(sizeof(cx<T>)));
            constexpr int E = static_cast<int>(sizeof(cx<T>)) / 8;
            for (int c = 0; c < 3; ++c) tma_load_3d(A + c * CS, &tm, ky0 * E, c * nz, kx, &zbar);
        }
    } else {
        constexpr int VEC16 = 16 / static_cast<int>(sizeof(cx<T>));
        if (VEC16 > 1 && wl == W && (ly % VEC16) == 0) load_tile(std::integral_constant<int, VEC16>{});
        else load_tile(std::integral_constant<int, 1>{});
    }
    stage_twiddles<T, LOG2LZ>(tws, tw);
    cp_async_wait_all();
    __syncthreads();
    if (use_tma) mbar_wait(&zbar, 0);

    // forward stage A: task (c, n1, w); planes z >= nz are zero (pruned, never read)
    for (int t = tid; t < 3 * N1 * W; t += kZThreads) {
        const int w = t % W, cn = t / W, c = cn / N1, n1 = cn % N1;
        constexpr int NZ = N2 / 2 > 0 ? N2 / 2 : 1;
        cx<T> v[N2];
        const cx<T>* src = A + c * CS + w;
#pragma unroll
        for (int n2 = 0; n2 < NZ; ++n2) {
            const int z = n1 + N1 * n2;
            v[n2] = z < nz ? src[z * W] : cx<T>{0, 0};
        }
        DftP<N2, -1, NZ, N2>::run(v);
        cx<T>* dst = B + c * CS + n1 * W + w;
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
            cx<T> x = v[k2];
            if (k2 > 0) x = cmul(x, tws[k2 * N1 + n1]);
            dst[k2 * N1 * W] = x;
        }
    }
    __syncthreads();

    // fused middle: task (k2, w). The task's N1 tensor coefficient sets are loaded first, so
    // their global latency overlaps the forward DFTs.
    for (int t = tid; t < N2 * W; t += kZThreads) {
        const int w = t % W, k2 = t / W;
        const int ky = ky0 + w;
        const bool fy = 2 * ky > ly;
        const int kyo = fy ? ly - ky : ky;
        const T* kb = kt + (static_cast<long long>(kx) * zh * yh + kyo) * 6;
        // (f64 at Lz = 256: the 16 coefficient sets would spill, so they are loaded next to
        // their use there)
        constexpr bool PREF = N1 <= 8 || sizeof(T) == 4;
        T k6[PREF ? N1 : 1][6];
        if (PREF && w < wl) {
#pragma unroll
            for (int k1 = 0; k1 < (PREF ? N1 : 0); ++k1) {
                const int kz = k2 + N2 * k1;
                const int kzo = 2 * kz > LZ ? LZ - kz : kz;
                load6<T>(kb + static_cast<long long>(kzo) * yh * 6, k6[k1]);
            }
        }
        cx<T> u[3][N1];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const cx<T>* src = B + c * CS + (k2 * N1) * W + w;
#pragma unroll
            for (int q = 0; q < N1; ++q) u[c][q] = src[q * W];
            DftP<N1, -1, N1, N1>::run(u[c]);
        }
        if (w < wl) {
#pragma unroll
            for (int k1 = 0; k1 < N1; ++k1) {
                const int kz = k2 + N2 * k1;
                const bool fz = 2 * kz > LZ;
                T(&kk)[6] = k6[PREF ? k1 : 0];
                if constexpr (!PREF) load6<T>(kb + static_cast<long long>(fz ? LZ - kz : kz) * yh * 6, k6[0]);
                if (fy) kk[1] = -kk[1];
                if (fz) kk[2] = -kk[2];
                if (fy != fz) kk[4] = -kk[4];
                mac3<T>(kk, u[0][k1], u[1][k1], u[2][k1]);
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            DftP<N1, +1, N1, N1>::run(u[c]);
            cx<T>* dst = A + c * CS + (k2 * N1) * W + w;
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) {
                cx<T> x = u[c][n1];
                if (k2 > 0) x = cmulc(x, tws[k2 * N1 + n1]);
                dst[n1 * W] = x;
            }
        }
    }
    __syncthreads();

    // inverse stage A': task (c, n1, w), IDFT_N2 over k2, the nz live planes to S2
    for (int t = tid; t < 3 * N1 * W; t += kZThreads) {
        const int w = t % W, cn = t / W, c = cn / N1, n1 = cn % N1;
        cx<T> v[N2];
        const cx<T>* src = A + c * CS + n1 * W + w;
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) v[k2] = src[k2 * N1 * W];
        constexpr int NO = N2 / 2 > 0 ? N2 / 2 : 1;
        DftP<N2, +1, N2, NO>::run(v);
        if (w < wl) {
#pragma unroll
            for (int n2 = 0; n2 < NO; ++n2) {
                const int z = n1 + N1 * n2;
                if (z < nz) blk[(c * nz + z) * zpitch + w] = v[n2];
            }
        }
    }
}

template <typename K>
void set_smem(K kernel, int bytes) {
    if (bytes > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) throw std::runtime_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    }
}

#define MMB_Y_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12)
#define MMB_Z_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)

} // namespace

template <typename T>
bool big_supported(const Geom& g) {
    if (g.lx < 2 || g.ly < 2 || g.nz < 2) return false;
    if (g.log2lx > 12 || g.log2ly > 12 || g.log2lz > 8) return false;
    if (sizeof(T) == 8 && (g.log2lx > 10 || g.log2ly > 10)) return false; // DFT_64 f64 spills
    return true;
}

template <typename T>
void prepare_big_kernels(const Geom& g) {
    switch (g.log2ly) {
#define X(l) case l: set_smem(k_yrow<T, l, 0>, yr_smem_bytes<T, l>()); set_smem(k_yrow<T, l, 1>, yr_smem_bytes<T, l>()); \
                     set_smem(k_yrow<T, l, 0, true>, yr_smem_bytes<T, l>()); set_smem(k_yrow<T, l, 1, true>, yr_smem_bytes<T, l>()); break;
        MMB_Y_CASES(X)
#undef X
        default: throw std::invalid_argument("big path: bad Ly");
    }
    switch (g.log2lz) {
#define X(l) case l: set_smem(k_zmac<T, l>, z_smem_bytes<T, l>()); break;
        MMB_Z_CASES(X)
#undef X
        default: throw std::invalid_argument("big path: bad Lz");
    }
}

template <typename T>
void launch_big_yf(const cx<T>* S, cx<T>* S2, const Geom& g, const cx<T>* tw, StepCtl* ctl,
                   const StageTable& st, int prologue, cudaStream_t stream, const RowMap<T>* rows) {
    const long long nrows = static_cast<long long>(g.xh) * 3 * g.nz;
    RowMap<T> rm{};
    if (rows) rm = *rows;
    switch (g.log2ly) {
#define X(l) case l: { constexpr int P = YR<l>::P; \
        const unsigned grid = static_cast<unsigned>((nrows + P - 1) / P); \
        if (rows) k_yrow<T, l, 0, true><<<grid, YR<l>::NT, yr_smem_bytes<T, l>(), stream>>>( \
            S, S2, nrows, g.ny, g.ly, g.ny, tw, ctl, st, prologue, rm, g.nz); \
        else k_yrow<T, l, 0><<<grid, YR<l>::NT, yr_smem_bytes<T, l>(), stream>>>( \
            S, S2, nrows, g.ny, g.ly, g.ny, tw, ctl, st, prologue, rm, g.nz); break; }
        MMB_Y_CASES(X)
#undef X
        default: throw std::invalid_argument("big path: bad Ly");
    }
    check_launch();
}

template <typename T>
void launch_big_yi(const cx<T>* S2, cx<T>* S, const Geom& g, const cx<T>* tw, cudaStream_t stream,
                   const RowMap<T>* rows) {
    const long long nrows = static_cast<long long>(g.xh) * 3 * g.nz;
    RowMap<T> rm{};
    if (rows) rm = *rows;
    StageTable st{};
    switch (g.log2ly) {
#define X(l) case l: { constexpr int P = YR<l>::P; \
        const unsigned grid = static_cast<unsigned>((nrows + P - 1) / P); \
        if (rows) k_yrow<T, l, 1, true><<<grid, YR<l>::NT, yr_smem_bytes<T, l>(), stream>>>( \
            S2, S, nrows, g.ly, g.ny, g.ny, tw, nullptr, st, 0, rm, g.nz); \
        else k_yrow<T, l, 1><<<grid, YR<l>::NT, yr_smem_bytes<T, l>(), stream>>>( \
            S2, S, nrows, g.ly, g.ny, g.ny, tw, nullptr, st, 0, rm, g.nz); break; }
        MMB_Y_CASES(X)
#undef X
        default: throw std::invalid_argument("big path: bad Ly");
    }
    check_launch();
}

template <typename T>
void launch_big_z(cx<T>* S2, const Geom& g, const cx<T>* tw, const T* kt, cudaStream_t stream) {
    const bool tma_off = env_off("MMB_ZMAC_TMA"); // read per launch (graph capture): A/B in one process
    const unsigned long long e = sizeof(cx<T>) / 8, esz = sizeof(cx<T>);
    switch (g.log2lz) {
#define X(l) case l: { constexpr int W = zw<T, l>(); const dim3 grid((g.ly + W - 1) / W, g.xh); \
        CUtensorMap tm{}; \
        const int ut = !tma_off && g.nz <= 256 && make_tmap_3d(&tm, S2, g.ly * e, 3ull * g.nz, g.xh, g.ly * esz, \
                                                   3ull * g.nz * g.ly * esz, static_cast<unsigned>(W * e), static_cast<unsigned>(g.nz), 1u); \
        k_zmac<T, l><<<grid, kZThreads, z_smem_bytes<T, l>(), stream>>>(S2, g, tw, kt, tm, ut); break; }
        MMB_Z_CASES(X)
#undef X
        default: throw std::invalid_argument("big path: bad Lz");
    }
    check_launch();
}

template <typename T>
std::string big_describe(const Geom& g) {
    char buf[160];
    const long long nrows = static_cast<long long>(g.xh) * 3 * g.nz;
    int p = 0, la = 0;
    switch (g.log2ly) {
#define X(l) case l: p = YR<l>::P; la = YR<l>::LA; break;
        MMB_Y_CASES(X)
#undef X
    }
    int w = 0;
    switch (g.log2lz) {
#define X(l) case l: w = zw<T, l>(); break;
        MMB_Z_CASES(X)
#undef X
    }
    const bool tma = !env_off("MMB_ZMAC_TMA") && tmap_encoder() && (g.ly * sizeof(cx<T>)) % 16 == 0;
    std::snprintf(buf, sizeof buf, "k_yrow<L%d> %s rows/cta=%d ctas=%lld; k_zmac<Lz%d> pencils/cta=%d tiles=%s", g.log2ly,
                  la == 2 ? "pair" : "plain", p, (nrows + p - 1) / (p ? p : 1), g.log2lz, w, tma ? "tma" : "copies");
    return buf;
}

#define MMB_BINST(T)                                                                              \
    template std::string big_describe<T>(const Geom&);                                           \
    template bool big_supported<T>(const Geom&);                                                 \
    template void prepare_big_kernels<T>(const Geom&);                                           \
    template void launch_big_yf<T>(const cx<T>*, cx<T>*, const Geom&, const cx<T>*, StepCtl*,     \
                                   const StageTable&, int, cudaStream_t, const RowMap<T>*);      \
    template void launch_big_yi<T>(const cx<T>*, cx<T>*, const Geom&, const cx<T>*, cudaStream_t, \
                                   const RowMap<T>*);                                            \
    template void launch_big_z<T>(cx<T>*, const Geom&, const cx<T>*, const T*, cudaStream_t);
#ifndef MMB_ONLY_F64
MMB_BINST(float)
#endif
#ifndef MMB_ONLY_F32
MMB_BINST(double)
#endif

} // namespace mmb
