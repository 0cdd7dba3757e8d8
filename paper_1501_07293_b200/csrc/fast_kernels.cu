// fast_kernels.cu — the fast demag path (sm_100a): three kernels per demag evaluation.
//
//   KX  (k_xf) : x-r2c of 2P consecutive rows of one (component, z) plane: two real rows
//                packed per complex four-step FFT, pruned to the nx live cells, separated
//                in shared memory and written kx-major: S[kx][c][z][y] (y fastest), so every
//                kx owns one contiguous block of 3*nz*Ly complex values.
//   KYZ (k_yz) : per kx block, entirely in shared memory: y-forward four-step FFT of the
//                3*nz live rows (ny live inputs, Ly outputs), z-forward DFT (Lz = 16, pruned),
//                real-symmetric 6-component tensor MAC, z-inverse, y-inverse (ny live
//                outputs) — written back in place. The padded spectrum never reaches HBM.
//   KXI (k_xi) : x-c2r back to the nx live cells of H_demag (SoA, x fastest).
//
// Replaces proj/src/demag.cpp:67-145 (pad, 3 forward FFTs, MAC, 3 inverse FFTs, window
// extract). 1/(Lx Ly Lz) is folded into the tensor spectrum (tensor_kernels.cu).
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <type_traits>
#include <string>

#include "fast.hpp"
#include "fft4.cuh"
#include "llg_cell.cuh"
#include "fast_common.cuh"

#ifndef MMB_YZ_KPREFETCH
#define MMB_YZ_KPREFETCH 1 // k_yz (nz > 1): load a pencil's tensor coefficients before its z-DFTs
#endif
#ifndef MMB_XS_ZC
#define MMB_XS_ZC 4 // planes per chunk of the 2-row-tile x grid
#endif

namespace mmb {

namespace {

void check_launch() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e));
}

template <int LOG2L>
constexpr int x_pairs() {
    constexpr int n2 = Split<LOG2L>::N2;
    return n2 >= 256 ? 1 : 256 / n2;
}
template <typename T, int LOG2L>
constexpr int x_smem_bytes() {
    using S = Split<LOG2L>;
    constexpr int P = x_pairs<LOG2L>();
    constexpr int ex = P * S::N2 * (S::N1 + 1);
    constexpr int zz = P * ((1 << LOG2L) + 1);
    constexpr int rr = 2 * P * (((1 << LOG2L) / 2 + 1) | 1);
    int m = ex > zz ? ex : zz;
    m = m > rr ? m : rr;
    return (m + (1 << LOG2L)) * static_cast<int>(sizeof(cx<T>)); // + twiddle table
}
template <typename T, int LOG2L>
constexpr int x_main_words() {
    return x_smem_bytes<T, LOG2L>() / static_cast<int>(sizeof(cx<T>)) - (1 << LOG2L);
}

// S row (kx, c, z) start; rows hold the ny live y values (the padded half never reaches HBM)
// ------------------------------------------------------------------ KX: x forward
template <typename T, int LOG2L>
__global__ void __launch_bounds__(x_pairs<LOG2L>() * Split<LOG2L>::N2)
    k_xf(const T* __restrict__ m, cx<T>* __restrict__ S, Geom g, const cx<T>* __restrict__ tw,
         StepCtl* ctl, StageTable st, int prologue) {
    using SP = Split<LOG2L>;
    constexpr int L = SP::L, N1 = SP::N1, N2 = SP::N2, P = x_pairs<LOG2L>();
    constexpr int XH = L == 1 ? 1 : L / 2 + 1;
    constexpr int EX = N1 + 1, ZP = L + 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw);
    cx<T>* tws = sm + x_main_words<T, LOG2L>();
    if (prologue && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0)
        step_prologue(ctl, st, prologue);
    stage_twiddles<T, LOG2L>(tws, tw);
    cp_async_wait_all();
    __syncthreads();

    const int y0 = blockIdx.x * (2 * P), z = blockIdx.y, c = blockIdx.z;
    const int nx = g.nx, ny = g.ny, nz = g.nz;
    const int tid = threadIdx.x;
    const T* plane = m + c * g.cs + static_cast<long long>(z) * ny * nx;

    // stage A: task (p, n1), n1 fastest; inputs beyond nx (and rows beyond ny) are zero
    if (tid < P * N1) {
        const int p = tid / N1, n1 = tid % N1;
        const int ya = y0 + 2 * p, yb = ya + 1;
        const T* ra = plane + static_cast<long long>(ya) * nx;
        const T* rb = plane + static_cast<long long>(yb) * nx;
        const bool va = ya < ny, vb = yb < ny;
        constexpr int NZ = L == 1 ? 1 : N2 / 2;
        cx<T> v[N2];
#pragma unroll
        for (int n2 = 0; n2 < NZ; ++n2) {
            const int x = n1 + N1 * n2;
            const bool in = x < nx;
            v[n2] = cx<T>{(in && va) ? __ldg(ra + x) : T(0), (in && vb) ? __ldg(rb + x) : T(0)};
        }
        DftP<N2, -1, NZ, N2>::run(v);
        cx<T>* ex = sm + (p * N2) * EX + n1;
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
            cx<T> w = v[k2];
            if (k2 > 0) w = cmul(w, tws[k2 * N1 + n1]);
            ex[k2 * EX] = w;
        }
    }
    __syncthreads();
    // stage B: task (p, k2), k2 fastest -> natural-order Z[k2 + N2 k1]
    {
        const int p = tid / N2, k2 = tid % N2;
        cx<T> u[N1];
        const cx<T>* ex = sm + (p * N2 + k2) * EX;
#pragma unroll
        for (int n1 = 0; n1 < N1; ++n1) u[n1] = ex[n1];
        DftP<N1, -1, N1, N1>::run(u);
        __syncthreads();
        cx<T>* zr = sm + p * ZP + k2;
#pragma unroll
        for (int k1 = 0; k1 < N1; ++k1) zr[N2 * k1] = u[k1];
    }
    __syncthreads();
    // separate the packed rows; task (k, r), r fastest -> coalesced kx-major stores
    const T half = T(0.5);
    const int ly = g.ly;
    for (int it = tid; it < XH * 2 * P; it += blockDim.x) {
        const int r = it % (2 * P), k = it / (2 * P);
        const int y = y0 + r;
        if (y >= ny) continue;
        const cx<T>* zr = sm + (r >> 1) * ZP;
        const cx<T> zk = zr[k], zm = zr[(L - k) & (L - 1)];
        const cx<T> val = (r & 1) ? cx<T>{(zk.y + zm.y) * half, (zm.x - zk.x) * half}
                                  : cx<T>{(zk.x + zm.x) * half, (zk.y - zm.y) * half};
        S[sf_row(k, c, z, nz, ny) + y] = val;
    }
}

// ------------------------------------------------------------------ KXI: x inverse
template <typename T, int LOG2L>
__global__ void __launch_bounds__(x_pairs<LOG2L>() * Split<LOG2L>::N2)
    k_xi(const cx<T>* __restrict__ S, T* __restrict__ h, Geom g, const cx<T>* __restrict__ tw) {
    using SP = Split<LOG2L>;
    constexpr int L = SP::L, N1 = SP::N1, N2 = SP::N2, P = x_pairs<LOG2L>();
    constexpr int XH = L == 1 ? 1 : L / 2 + 1;
    constexpr int EX = N1 + 1, RP = (L / 2 + 1) | 1; // odd staging pitch: conflict free
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw);
    cx<T>* tws = sm + x_main_words<T, LOG2L>();

    const int y0 = blockIdx.x * (2 * P), z = blockIdx.y, c = blockIdx.z;
    const int nx = g.nx, ny = g.ny, nz = g.nz;
    const int tid = threadIdx.x;
    stage_twiddles<T, LOG2L>(tws, tw);

    // stage the 2P half-spectrum rows with async copies (all loads in flight at once):
    // task (k, r), r fastest (coalesced reads)
    for (int it = tid; it < XH * 2 * P; it += blockDim.x) {
        const int r = it % (2 * P), k = it / (2 * P);
        const int y = y0 + r;
        if (y < ny) cp_async<sizeof(cx<T>)>(sm + r * RP + k, S + sf_row(k, c, z, nz, ny) + y);
        else sm[r * RP + k] = cx<T>{0, 0};
    }
    cp_async_wait_all();
    __syncthreads();
    // stage A on Z = A + iB (full circle from the two Hermitian halves)
    cx<T> v[N2];
    int p = 0, n1 = 0;
    const bool a_task = tid < P * N1;
    if (a_task) {
        p = tid / N1;
        n1 = tid % N1;
        const cx<T>* A = sm + (2 * p) * RP;
        const cx<T>* B = A + RP;
#pragma unroll
        for (int n2 = 0; n2 < N2; ++n2) {
            const int k = n1 + N1 * n2;
            cx<T> zv;
            if (k == 0 || 2 * k == L) {
                zv = cx<T>{A[k].x, B[k].x};
            } else if (2 * k < L) {
                const cx<T> a = A[k], b = B[k];
                zv = cx<T>{a.x - b.y, a.y + b.x};
            } else {
                const cx<T> a = A[L - k], b = B[L - k];
                zv = cx<T>{a.x + b.y, b.x - a.y};
            }
            v[n2] = zv;
        }
        DftP<N2, +1, N2, N2>::run(v);
    }
    __syncthreads();
    if (a_task) {
        cx<T>* ex = sm + (p * N2) * EX + n1;
#pragma unroll
        for (int k2 = 0; k2 < N2; ++k2) {
            cx<T> w = v[k2];
            if (k2 > 0) w = cmulc(w, tws[k2 * N1 + n1]);
            ex[k2 * EX] = w;
        }
    }
    __syncthreads();
    // stage B: natural-order outputs, only the nx live cells
    {
        const int pb = tid / N2, k2 = tid % N2;
        cx<T> u[N1];
        const cx<T>* ex = sm + (pb * N2 + k2) * EX;
#pragma unroll
        for (int q = 0; q < N1; ++q) u[q] = ex[q];
        constexpr int NO = N1 == 1 ? 1 : N1 / 2;
        DftP<N1, +1, N1, NO>::run(u);
        const int ya = y0 + 2 * pb, yb = ya + 1;
        T* ha = h + c * g.cs + (static_cast<long long>(z) * ny + ya) * nx; // component stride cs (slabs: halo)
        T* hb = ha + nx;
#pragma unroll
        for (int k1 = 0; k1 < NO; ++k1) {
            const int x = k2 + N2 * k1;
            if (x < nx) {
                if (ya < ny) ha[x] = u[k1].x;
                if (yb < ny) hb[x] = u[k1].y;
            }
        }
    }
}

// ------------------------------------------------------------------ KYZ: y, z, MAC, z^-1, y^-1
template <typename T, int LOG2L>
constexpr int yz_threads() {
    // ~384 threads; ~192 for f64 and for DFT_64 stages, so the stage-A registers fit under the
    // launch bound without spilling
#ifndef MMB_YZ_NT
#define MMB_YZ_NT 384
#endif
    constexpr int n2 = Split<LOG2L>::N2, target = (sizeof(T) == 8 || n2 >= 64) ? 192 : MMB_YZ_NT;
    return n2 >= target ? n2 : (target / n2) * n2;
}

template <typename T, int LOG2L, int ZM, bool PEER = false>
__global__ void __launch_bounds__(yz_threads<T, LOG2L>())
    k_yz(cx<T>* __restrict__ S, Geom g, const cx<T>* __restrict__ tw, const T* __restrict__ kt,
         int kxb, StepCtl* ctl, StageTable st, int prologue, const __grid_constant__ RowMap<T> rm) {
    using SP = Split<LOG2L>;
    constexpr int L = SP::L, N1 = SP::N1, N2 = SP::N2;
    constexpr int RP = fpitch<LOG2L>();
    constexpr int NT = yz_threads<T, LOG2L>();
    constexpr int RB = NT / N2; // rows per batch
    using RC = rcx<T, LOG2L>; // register complex type (packed FFMA2 arithmetic for f32)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    cx<T>* sm = reinterpret_cast<cx<T>*>(smem_raw);

    const int nz = g.nz, ny = g.ny, xh = g.xh;
    cx<T>* tws = sm + kxb * 3 * nz * RP;
    // one transaction barrier per y-forward batch of rows (the last one takes the rest): a
    // batch's stage A starts when its rows land
    constexpr int NBAR = 4;
    __shared__ __align__(8) unsigned long long bar[NBAR];
    pdl_wait();
    pdl_trigger(); // after the wait: at most one kernel ahead of the running one
    if (prologue && blockIdx.x == 0 && threadIdx.x == 0) step_prologue(ctl, st, prologue);
    const int kx0 = blockIdx.x * kxb;
    const int kxn = min(kxb, xh - kx0);
    const int rows = kxn * 3 * nz;
    const int tid = threadIdx.x;
    cx<T>* gblk = S + sf_row(kx0, 0, 0, nz, ny); // rows of this CTA are contiguous in S
    // row r of the block: in S, or in the owning rank's slab spectrum (RowMap, peer memory)
    auto grow = [&](int r) -> cx<T>* {
        if constexpr (!PEER) {
            return gblk + static_cast<long long>(r) * ny;
        } else {
            const int kxl = r / (3 * nz), rc = r - kxl * 3 * nz;
            return rm.row(kx0 + kxl, rc / nz, rc % nz, ny);
        }
    };
    // TMA bulk copies of all live input rows (ny values each) into the first ny slots of
    // their shared-memory rows, in flight together while the twiddles are staged. Rows in
    // peer memory are read with plain loads.
    const unsigned rowbytes = static_cast<unsigned>(ny * sizeof(cx<T>));
    const bool bulk = (rowbytes % 16) == 0 && (!PEER || rm.local);
    if (tid == 0) {
        for (int b = 0; b < NBAR; ++b) mbar_init(&bar[b], 1);
        if (bulk) {
            for (int b = 0; b < NBAR; ++b) {
                const int r0 = b * RB, r1 = b == NBAR - 1 ? rows : min(rows, r0 + RB);
                if (r1 > r0) mbar_expect_tx(&bar[b], rowbytes * (r1 - r0));
            }
            for (int r = 0; r < rows; ++r) bulk_g2s(sm + r * RP, grow(r), rowbytes, &bar[min(r / RB, NBAR - 1)]);
        }
    }
    stage_twiddles<T, LOG2L>(tws, tw);
    if (!bulk) {
        for (int e = tid; e < rows * ny; e += NT) sm[(e / ny) * RP + e % ny] = grow(e / ny)[e % ny];
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- y forward, batches of RB rows
    for (int rb0 = 0; rb0 < rows; rb0 += RB) {
        const int nb = min(RB, rows - rb0);
        RC v[N2];
        const int ra = rb0 + tid / N1, n1 = tid % N1;
        const bool a_task = tid < nb * N1;
        if (bulk && rb0 / RB < NBAR) mbar_wait(&bar[rb0 / RB], 0);
        if (a_task) {
            const cx<T>* src = sm + ra * RP;
            constexpr int NZ = L == 1 ? 1 : N2 / 2;
#pragma unroll
            for (int n2 = 0; n2 < NZ; ++n2) {
                const int y = n1 + N1 * n2;
                v[n2] = y < ny ? RC(src[y]) : RC{0, 0};
            }
            DftP<N2, -1, NZ, N2>::run(v);
            // twiddles before the barrier: their shared loads overlap the other warps' arrival
#pragma unroll
            for (int k2 = 1; k2 < N2; ++k2) v[k2] = cmul(v[k2], RC(tws[k2 * N1 + n1]));
        }
        __syncthreads(); // the staged input rows are overwritten in place below
        if (a_task) {
            cx<T>* dst = sm + ra * RP;
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) dst[fpad<LOG2L>(k2 * N1 + n1)] = v[k2];
        }
        __syncthreads();
        const int rbr = rb0 + tid / N2, k2 = tid % N2;
        const bool b_task = tid < nb * N2;
        RC u[N1];
        if (b_task) {
            const cx<T>* src = sm + rbr * RP;
#pragma unroll
            for (int q = 0; q < N1; ++q) u[q] = src[fpad<LOG2L>(k2 * N1 + q)];
            DftP<N1, -1, N1, N1>::run(u);
        }
        __syncthreads();
        if (b_task) {
            cx<T>* dst = sm + rbr * RP;
#pragma unroll
            for (int k1 = 0; k1 < N1; ++k1) dst[fpad<LOG2L>(k2 + N2 * k1)] = u[k1];
        }
    }
    __syncthreads();

    // ---- z forward + tensor MAC + z inverse, one pencil (kx, ky) per task
    {
        const int ly = L, yh = g.yh, zh = g.zh;
        for (int it = tid; it < kxn * ly; it += NT) {
            const int kxl = it / ly, ky = it % ly;
            const int kx = kx0 + kxl;
            const bool fy = 2 * ky > ly;
            const int kyo = fy ? ly - ky : ky;
            const T* kb = kt + (static_cast<long long>(kx) * zh * yh + kyo) * 6;
            cx<T>* base = sm + (kxl * 3 * nz) * RP + fpad<LOG2L>(ky);
            if constexpr (ZM == 0) {
                // nz == 1: MAC only
                RC a = base[0], b = base[RP], cc = base[2 * RP];
                T k6[6];
                load6<T>(kb, k6);
                if (fy) {
                    k6[1] = -k6[1];
                    k6[4] = -k6[4];
                }
                mac3(k6, a, b, cc);
                base[0] = a;
                base[RP] = b;
                base[2 * RP] = cc;
            } else {
                // 2 <= nz <= 8, Lz = 16. The pencil's 9 x 6 tensor coefficients are loaded
                // first, so their global-load latency hides behind the forward z-DFTs.
                T kk[9][6];
#if MMB_YZ_KPREFETCH
#pragma unroll
                for (int kzo = 0; kzo <= 8; ++kzo) load6<T>(kb + kzo * yh * 6, kk[kzo]);
#endif
                RC w[3][16];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
#pragma unroll
                    for (int zz = 0; zz < 8; ++zz)
                        w[c][zz] = zz < nz ? RC(base[(c * nz + zz) * RP]) : RC{0, 0};
                    DftP<16, -1, 8, 16>::run(w[c]);
                }
#pragma unroll
                for (int kzo = 0; kzo <= 8; ++kzo) {
                    T k6[6];
#if MMB_YZ_KPREFETCH
#pragma unroll
                    for (int q = 0; q < 6; ++q) k6[q] = kk[kzo][q];
#else
                    load6<T>(kb + kzo * yh * 6, k6);
#endif
                    if (fy) {
                        k6[1] = -k6[1];
                        k6[4] = -k6[4];
                    }
                    mac3(k6, w[0][kzo], w[1][kzo], w[2][kzo]);
                    if (kzo != 0 && kzo != 8) {
                        // kz = 16 - kzo: xz and yz are odd in z
                        k6[2] = -k6[2];
                        k6[4] = -k6[4];
                        mac3(k6, w[0][16 - kzo], w[1][16 - kzo], w[2][16 - kzo]);
                    }
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    DftP<16, +1, 16, 8>::run(w[c]);
#pragma unroll
                    for (int zz = 0; zz < 8; ++zz)
                        if (zz < nz) base[(c * nz + zz) * RP] = w[c][zz];
                }
            }
        }
    }
    __syncthreads();

    // ---- y inverse, batches of RB rows, ny live outputs straight to HBM
    for (int rb0 = 0; rb0 < rows; rb0 += RB) {
        const int nb = min(RB, rows - rb0);
        RC v[N2];
        const int ra = rb0 + tid / N1, n1 = tid % N1;
        const bool a_task = tid < nb * N1;
        if (a_task) {
            const cx<T>* src = sm + ra * RP;
#pragma unroll
            for (int n2 = 0; n2 < N2; ++n2) v[n2] = src[fpad<LOG2L>(n1 + N1 * n2)];
            DftP<N2, +1, N2, N2>::run(v);
#pragma unroll
            for (int k2 = 1; k2 < N2; ++k2) v[k2] = cmulc(v[k2], RC(tws[k2 * N1 + n1]));
        }
        __syncthreads();
        if (a_task) {
            cx<T>* dst = sm + ra * RP;
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) dst[fpad<LOG2L>(k2 * N1 + n1)] = v[k2];
        }
        __syncthreads();
        const int rbr = rb0 + tid / N2, k2 = tid % N2;
        if (tid < nb * N2) {
            RC u[N1];
            const cx<T>* src = sm + rbr * RP;
#pragma unroll
            for (int q = 0; q < N1; ++q) u[q] = src[fpad<LOG2L>(k2 * N1 + q)];
            constexpr int NO = N1 == 1 ? 1 : N1 / 2;
            DftP<N1, +1, N1, NO>::run(u);
            cx<T>* dst = grow(rbr);
#pragma unroll
            for (int k1 = 0; k1 < NO; ++k1) {
                const int y = k2 + N2 * k1;
                if (y < ny) dst[y] = u[k1];
            }
        }
    }
}

#ifndef MMB_XS_PAIR_STORE
#define MMB_XS_PAIR_STORE 0 // 3c: one row pair per thread, 16-byte stores (measured +0.5 us on k_xstep)
#endif
#ifndef MMB_XS_PAIR_LLG
#define MMB_XS_PAIR_LLG 1 // f32 local terms on packed cell pairs (even nx)
#endif

// ------------------------------------------------------------------ KXS: x^-1, LLG, x (fused)
// One CTA per (TR consecutive y rows, one z plane), all three components:
//   1. x-c2r of the convolved half spectra S -> H_demag tile (shared memory only),
//   2. local terms + Euler + renormalisation for the TR x nx cells (CellLLG, exact
//      reference rounding) -> M_{t+1} to HBM,
//   3. x-r2c of the new tile -> the half spectra S for the next step, in place.
// H_demag never reaches HBM and M_{t+1} is not re-read: per step the x side moves
// S in + S out + M_t + M_{t+1} instead of three separate passes.
constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }

template <int LOG2L, int PB = 128, int TSIZE = 4>
struct XS {
    using SP = Split<LOG2L>;
    // Lx = 4096 halves the tile so exchange buffer + twiddle table stay within 227 KB
    static constexpr int PBE = (LOG2L >= 12 && PB > 16) ? PB / 2 : PB;
    // Lx = 2048 (N2 = 64 = 2 N1), WIDE: one stage-A task (DFT_64 in registers) per thread, 3 x 8
    // rows per CTA, stage B in RB = 2 rounds. Lx = 4096 (N1 = N2 = 64), PAIR: every DFT_64
    // task runs on a lane pair (dft_pair, 32 values per lane); LA / LB = lanes per stage-A /
    // stage-B task. (PAIR at Lx = 2048 with 3 x 2 rows and 3 CTAs/SM measured 26 % slower than
    // WIDE: the narrow tiles re-read more neighbour rows.)
    static constexpr bool WIDE = LOG2L == 11 && PB > 16;
    static constexpr bool PAIR = LOG2L >= 11 && !WIDE;
    static constexpr int LA = PAIR ? 2 : 1, LB = (PAIR && SP::N1 == 64) ? 2 : 1;
    static constexpr int RB = WIDE ? SP::N2 / SP::N1 : 1;
    static constexpr int P = PAIR ? 3
                                  : (WIDE ? 3 * (PBE / SP::N1) : 3 * (SP::N2 >= PBE ? 1 : PBE / SP::N2));
    static constexpr int TR = 2 * P / 3;                                        // y rows per CTA
    static constexpr bool ZFAST = TR >= 4;
    static constexpr int NT0 = WIDE ? P * SP::N1 : P * SP::N2 * LB; // threads with FFT tasks
    // small-grid tiles (PB <= 16) get TM times the threads: the extra ones only take part in
    // the staging, local-term and spectrum-store loops, which otherwise run 5+ cells deep
#ifndef MMB_XS_TM_THREADS
#define MMB_XS_TM_THREADS 192
#endif
    static constexpr int TM = ((TSIZE == 4 || LOG2L <= 8) && PB <= 16 && LA == 1 && LB == 1 && NT0 < MMB_XS_TM_THREADS)
                                  ? MMB_XS_TM_THREADS / NT0 : 1; // (f64 above Lx = 256: the registers limit)
    static constexpr int NT = NT0 * TM;                                         // threads
    static_assert(P * SP::N1 * LA <= NT0 && P * SP::N2 * LB == NT0 * RB, "stage tasks");
    static_assert(TM == 1 || (LA == 1 && LB == 1), "pair shuffles need every lane");
    static constexpr int XHP = ((1 << LOG2L) / 2 + 1) | 1;            // staging pitch (odd)
    static constexpr int EX = SP::N1 + 1;
    static constexpr int ZP = (1 << LOG2L) + 1;
    static constexpr int A0 = 3 * TR * XHP, A1 = P * SP::N2 * EX, A2 = P * ZP;
    static constexpr int AREA = A0 > A1 ? (A0 > A2 ? A0 : A2) : (A1 > A2 ? A1 : A2);
    // staging layout [c][kx][TR] (the tile's TR rows of a component side by side per kx):
    // a TMA box of TR rows x BOXK kx lands as one contiguous block. NB boxes per component,
    // BOXK rounded so every box starts 128-byte aligned; KXP = kx pitch of a component.
    static constexpr int XH = (1 << LOG2L) / 2 + 1;
    static constexpr int NB = (XH + 255) / 256;
    static constexpr int BQ = 128 / cgcd(128, TR * 2 * TSIZE); // kx multiple for 128-byte boxes
    static constexpr int BOXK = ((XH + NB - 1) / NB + BQ - 1) / BQ * BQ;
    // TMA layout where stage A's 16-byte pair loads stay bank-conflict free (an odd number
    // of 16-byte units between consecutive kx: f32 tiles of 2 or 14 rows) and at Lx >= 2048
    // (measured faster despite the conflicts: 1024x1024x32 xstep 1.16 -> 1.10 ms); otherwise
    // the pairs are staged [p][kx][2] by async copies (Lx = 256 with 8-row tiles: TMA
    // 55 -> 77 us)
    static constexpr bool TMA = BOXK <= 256 && 3 * NB * BOXK * TR <= AREA && (TR * 2 * TSIZE) % 16 == 0 &&
                                (((TR * 2 * TSIZE) / 16) % 2 == 1 || LOG2L >= 11);
    static constexpr int KXP = TMA ? NB * BOXK : XH;
};
template <typename T, int LOG2L, int PB>
constexpr int xs_smem_bytes() {
    return (XS<LOG2L, PB, sizeof(T)>::AREA + (1 << LOG2L)) * static_cast<int>(sizeof(cx<T>));
}

template <typename X>
dim3 xs_grid(const Geom& g) {
    const unsigned tiles = static_cast<unsigned>((g.ny + X::TR - 1) / X::TR);
    if (X::ZFAST) return dim3(g.nz, tiles);
    const unsigned zc = static_cast<unsigned>(std::min(MMB_XS_ZC, g.nz));
    return dim3(zc * tiles, (g.nz + zc - 1) / zc);
}

template <typename T, int LOG2L, int PB>
constexpr int xs_min_blocks() {
    // two or three CTAs per SM when their shared memory fits (registers capped accordingly;
    // f64 tiles keep at most two so their DFT registers do not spill)
    constexpr int b = xs_smem_bytes<T, LOG2L, PB>() + 2048;
    return (sizeof(T) == 4 && LOG2L <= 9 && XS<LOG2L, PB, sizeof(T)>::NT <= 256 && 3 * b <= 228 * 1024)
               ? 3 : (2 * b <= 228 * 1024 ? 2 : 1);
}

// PB = 128: ~384 threads and 3 x 8 rows per CTA (large grids); PB = 16: 3 x 2 rows for
// grids whose row count would otherwise leave SMs idle.
template <typename T, int LOG2L, int PB>
__global__ void __launch_bounds__(XS<LOG2L, PB, sizeof(T)>::NT, xs_min_blocks<T, LOG2L, PB>())
    k_xstep(cx<T>* __restrict__ S, const T* __restrict__ m, T* __restrict__ mout, Geom g,
            const cx<T>* __restrict__ tw, T coeff, T kan, StepCtl* ctl, double* __restrict__ tpart,
            const __grid_constant__ CUtensorMap tmS, int use_tma) {
    using SP = Split<LOG2L>;
    using X = XS<LOG2L, PB, sizeof(T)>;
    constexpr int L = SP::L, N1 = SP::N1, N2 = SP::N2, P = X::P, TR = X::TR, NT = X::NT;
    constexpr int XH = L / 2 + 1, XHP = X::XHP, EX = X::EX, ZP = X::ZP;
    using RC = rcx<T, LOG2L>; // register complex type (packed FFMA2 arithmetic for f32, L <= 1024)
    constexpr bool TWPRE = PB <= 16; // stage-A twiddles before the barrier (small tiles)
    extern __shared__ __align__(128) unsigned char xs_smem[]; // 128 B: TMA box destinations
    cx<T>* sm = reinterpret_cast<cx<T>*>(xs_smem);
    T* hm = reinterpret_cast<T*>(xs_smem); // [3*TR][nx] tile: H_demag, then M_{t+1}
    cx<T>* tws = sm + X::AREA;

    // ZFAST (tiles of >= 4 rows): z fastest in the grid, so the CTAs of one y tile in
    // neighbouring planes run together and the +-z neighbour rows of the local terms come from
    // L2 instead of DRAM re-reads. Narrower tiles go by chunks of 4 planes, z fastest inside a
    // chunk and y next: neighbouring y tiles (their 16-byte row segments of S share 32-byte
    // sectors) still run alongside, and only chunk-boundary planes are re-read from DRAM.
    const int zcn = min(MMB_XS_ZC, g.nz);
    const int z = X::ZFAST ? blockIdx.x : blockIdx.y * zcn + blockIdx.x % zcn;
    const int y0 = (X::ZFAST ? blockIdx.y : blockIdx.x / zcn) * TR;
    const int nx = g.nx, ny = g.ny, nz = g.nz;
    const long long cs = g.cs;
    const int zg = g.z0 + z, nzg = g.nz_g;
    const int tid = threadIdx.x;
    pdl_wait();
    pdl_trigger(); // after the wait: at most one kernel ahead of the running one
    if (!X::ZFAST && z >= g.nz) { // the last chunk's missing planes
        if (tid == 0) tpart[blockIdx.y * gridDim.x + blockIdx.x] = 0.0;
        return;
    }
    const long long cur_step = ctl->cur_step;
    if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) ctl->step = cur_step + 1;

    // ---- 1a. stage the 3*TR convolved half-spectrum rows as [c][kx][TR]: rows 2p, 2p+1 (y,
    // y+1 of one component), which stage A packs into one complex sequence, sit side by side.
    // TMA (use_tma): NB boxes of TR y x BOXK kx per component, issued by one thread (rows past
    // ny and columns past Xh arrive as zeros). Otherwise one 16-byte L1-allocating async copy
    // per row pair and kx, each thread keeping one pair and walking kx with a fixed stride.
    static_assert(TR % 2 == 0, "tile rows come in pairs");
    constexpr int NPR = 3 * TR / 2, KXP = X::KXP; // row pairs, kx pitch of a component
    static_assert(NT % NPR == 0 && 3 * KXP * TR <= X::AREA, "thread count must be a multiple of the row pairs");
    // pair p's value at kx k: sm[pair_base(p) + k * KS]
    constexpr int KS = X::TMA ? TR : 2;
    const auto pair_base = [&](int p) {
        const int c = (2 * p) / TR;
        return X::TMA ? c * KXP * TR + (2 * p - c * TR) : p * 2 * XH;
    };
    constexpr int KSTEP = NT / NPR;
    const int my_p = tid % NPR, my_k0 = tid / NPR;
    const int my_c = (2 * my_p) / TR, my_yl = 2 * my_p - my_c * TR, my_y = y0 + my_yl;
    const bool live0 = my_y < ny, live1 = my_y + 1 < ny;
    const int kx_stride = 3 * nz * ny;                      // S elements between kx blocks
    const int row_off = (my_c * nz + z) * ny + my_y;        // (c, z, y) offset inside a kx block
    // one transaction barrier per component: the stage-A tasks of component c start as soon
    // as its boxes land, while the later components are still in flight
    // even ny: pairs never straddle the grid edge and start 16-byte aligned in S
    const bool vec = (ny & 1) == 0;
    __shared__ __align__(8) unsigned long long sbar[3];
    const bool tma = X::TMA && use_tma;
    if (tma) {
        if (tid == 0) {
            constexpr int E = static_cast<int>(sizeof(cx<T>)) / 8; // 8-byte map elements
#pragma unroll 1
            for (int c = 0; c < 3; ++c) {
                mbar_init(&sbar[c], 1);
                mbar_expect_tx(&sbar[c], X::NB * X::BOXK * TR * static_cast<unsigned>(sizeof(cx<T>)));
#pragma unroll 1
                for (int j = 0; j < X::NB; ++j)
                    tma_load_3d(sm + (c * KXP + j * X::BOXK) * TR, &tmS, y0 * E, c * nz + z, j * X::BOXK, &sbar[c]);
            }
        }
    } else {
        cx<T>* dst = sm + pair_base(my_p);
        for (int k = my_k0; k < XH; k += KSTEP) {
            const cx<T>* src = S + (k * kx_stride + row_off);
            cx<T>* d = dst + k * KS;
            if (live0 && vec) {
                cp_async_pair<T>(d, src);
            } else {
                if (live0) cp_async<sizeof(cx<T>)>(d, src);
                else d[0] = cx<T>{0, 0};
                if (live1) cp_async<sizeof(cx<T>)>(d + 1, src + 1);
                else d[1] = cx<T>{0, 0};
            }
        }
    }
    stage_twiddles<T, LOG2L>(tws, tw);
    cp_async_wait_all();
    __syncthreads();

    // ---- 1b. inverse stage A on Z = A + iB (rows 2p, 2p+1 of the same component); lane
    // h of a pair task takes n2 = LA m + h
    constexpr int LA = X::LA, LB = X::LB, RA = N2 / LA, RBq = N1 / LB;
    RC v[RA];
    const int ha = LA == 2 ? pair_half(tid) : 0, ta = LA == 2 ? pair_task(tid) : tid;
    const bool a_task = ta < P * N1;
    const int pa = ta / N1, n1 = ta % N1;
    if (a_task) {
        if (tma) mbar_wait(&sbar[(2 * pa) / TR], 0); // every component has stage-A tasks
        const cx<T>* AB = sm + pair_base(pa);
#pragma unroll
        for (int m = 0; m < RA; ++m) {
            const int k = n1 + N1 * (LA * m + ha);
            cx<T> a, b, zv;
            if (k == 0 || 2 * k == L) {
                ld_pair<T>(AB + k * KS, a, b);
                zv = cx<T>{a.x, b.x};
            } else if (2 * k < L) {
                ld_pair<T>(AB + k * KS, a, b);
                zv = cx<T>{a.x - b.y, a.y + b.x};
            } else {
                ld_pair<T>(AB + (L - k) * KS, a, b);
                zv = cx<T>{a.x + b.y, b.x - a.y};
            }
            v[m] = zv;
        }
        if constexpr (LA == 2) dft_pair<RA, +1, RA>(v, ha);
        else DftP<N2, +1, N2, N2>::run(v);
        // small tiles: twiddles before the barrier, their shared loads overlapping the other
        // warps' arrival (256^2 film 14.8 -> 13.3 us; the large tiles measured slower)
        if constexpr (TWPRE) {
#pragma unroll
            for (int kk = 0; kk < RA; ++kk) {
                const int k2 = kk + RA * ha;
                if (k2 > 0) v[kk] = cmulc(v[kk], RC(tws[k2 * N1 + n1]));
            }
        }
    }
    __syncthreads();
    if (a_task) {
        cx<T>* ex = sm + (pa * N2) * EX + n1;
#pragma unroll
        for (int kk = 0; kk < RA; ++kk) {
            const int k2 = kk + RA * ha;
            RC w = v[kk];
            if (!TWPRE && k2 > 0) w = cmulc(w, RC(tws[k2 * N1 + n1]));
            ex[k2 * EX] = w;
        }
    }
    __syncthreads();
    // ---- 1c. inverse stage B -> H_demag tile (the nx live cells); lane h of a pair task
    // takes n1 = LB q + h and returns k1 = q + RBq h
    const int hb_ = LB == 2 ? pair_half(tid) : 0, tb0 = LB == 2 ? pair_task(tid) : tid;
    // RB = 2 (WIDE): the tile rows of round r lie inside exchange rows already consumed
    // (round 0: its own, synchronised below; round 1: round 0's), never in round 1's
#pragma unroll 1
    for (int rnd = 0; rnd < X::RB; ++rnd) {
        const int tb = tb0 + rnd * NT;
        const bool b_task = X::TM == 1 || tb < P * N2 * LB;
        const int pb = tb / N2, k2b = tb % N2;
        RC u[RBq];
        constexpr int NO = N1 == 1 ? 1 : N1 / 2;
        if (b_task) {
            const cx<T>* ex = sm + (pb * N2 + k2b) * EX + hb_;
#pragma unroll
            for (int q = 0; q < RBq; ++q) u[q] = ex[LB * q];
            if constexpr (LB == 2) dft_pair<RBq, +1, RBq>(u, hb_);
            else DftP<N1, +1, N1, NO>::run(u);
        }
        __syncthreads(); // the tile overlays the exchange buffer
        if (b_task) {
            T* ha_row = hm + (2 * pb) * nx;
            T* hb_row = ha_row + nx;
#pragma unroll
            for (int q = 0; q < (LB == 2 ? RBq : NO); ++q) {
                const int k1 = q + RBq * hb_;
                const int x = k2b + N2 * k1;
                if (k1 < NO && x < nx) {
                    ha_row[x] = u[q].x;
                    hb_row[x] = u[q].y;
                }
            }
        }
    }

    // ---- 2. local terms + LLG on the tile's cells; M_{t+1} to HBM and to the tile
    CellLLG<T> cl;
    cl.load(ctl, coeff, kan);
    double tmax = 0.0;
    const int sy = nx, sz = nx * ny;
    // 32-bit element indices (3 cs < 2^31) off one base: one 64-bit address per load instead
    // of 64-bit index arithmetic
    const int csi = static_cast<int>(cs);
#if MMB_XS_PAIR_LLG
    if constexpr (std::is_same_v<T, float>) {
        if ((nx & 1) == 0) {
            // f32, even nx: cell pairs (i, i+1) per thread on packed FP32 (CellPairLLG, bitwise
            // CellLLG per cell). Every pair offset is even, so the centre, +-y and +-z loads,
            // the H_demag reads and the stores are 8-byte vectors; the outer x neighbours are
            // scalar loads from the same sectors. A missing neighbour is the cell's own centre
            // (adds +0 to the exchange sum), loaded from the centre's address so every load is
            // unconditional and independent of the centre load.
            // Software-pipelined: a pair's 21 loads are in flight while the previous pair
            // updates, and the first pair's before the barrier that ends the x-inverse.
            CellPairLLG pl;
            pl.load(ctl, coeff, kan);
            const int nxh = nx >> 1;
            const int hc = (TR * nx) >> 1; // float2 stride between the component tiles
            float2 rc[3], rn[3][6];
            const auto load_pair = [&](int yl_, int ip_) {
                const int j_ = y0 + yl_, i_ = 2 * ip_;
                const int f_ = z * sz + j_ * sy + i_;
                const bool xl = i_ > 0, xr = i_ + 2 < nx, ym = j_ > 0, yp = j_ + 1 < ny, zm = zg > 0,
                           zp = zg + 1 < nzg;
                const auto ld2 = [&](int o) { return __ldg(reinterpret_cast<const float2*>(m + o)); };
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int q = c * csi + f_;
                    rc[c] = ld2(q);
                    rn[c][0].x = __ldg(m + (xl ? q - 1 : q));
                    rn[c][1].y = __ldg(m + (xr ? q + 2 : q + 1));
                    rn[c][2] = ld2(ym ? q - sy : q);
                    rn[c][3] = ld2(yp ? q + sy : q);
                    rn[c][4] = ld2(zm ? q - sz : q);
                    rn[c][5] = ld2(zp ? q + sz : q);
                }
            };
            int yl = 0, ip = tid;
            while (ip >= nxh) {
                ip -= nxh;
                ++yl;
            }
            bool valid = yl < TR && y0 + yl < ny;
            if (valid) load_pair(yl, ip);
            __syncthreads(); // the H_demag tile (x-inverse) is complete
            while (valid) {
                const int j = y0 + yl, i = 2 * ip;
                const int f = z * sz + j * sy + i;
                float2 mc[3], ex[3];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    rn[c][0].y = rc[c].x; // the inner x neighbours are the pair's own centres
                    rn[c][1].x = rc[c].y;
                    mc[c] = rc[c];
                    ex[c] = CellPairLLG::exch(rc[c], rn[c]);
                }
                // the next pair's loads go out before this pair's update
                int yl2 = yl, ip2 = ip + NT;
                while (ip2 >= nxh) {
                    ip2 -= nxh;
                    ++yl2;
                }
                const bool valid2 = yl2 < TR && y0 + yl2 < ny;
                if (valid2) load_pair(yl2, ip2);
                float2* hp = reinterpret_cast<float2*>(hm + yl * nx + i);
                float2 hx = hp[0], hy = hp[hc], hz = hp[2 * hc];
                pl.heff(mc[0], hx, hy, hz, ex[0], ex[1], ex[2]);
                double t0, t1;
                bool z0b, z1b;
                pl.update(mc[0], mc[1], mc[2], hx, hy, hz, t0, t1, z0b, z1b);
                tmax = fmax(tmax, fmax(t0, t1));
                if (z0b || z1b)
                    atomicMin(&ctl->bad_key, (static_cast<unsigned long long>(cur_step) << 36) |
                                                 static_cast<unsigned long long>(
                                                     f + (z0b ? 0 : 1) + static_cast<long long>(g.z0) * sz));
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    *reinterpret_cast<float2*>(mout + (c * csi + f)) = mc[c];
                    hp[c * hc] = mc[c];
                }
                yl = yl2;
                ip = ip2;
                valid = valid2;
            }
            goto llg_done;
        }
    }
#endif
    __syncthreads(); // the H_demag tile (x-inverse) is complete
    {
    // walk the tile's cells with a fixed stride, carrying (yl, i) instead of dividing
    int yl = 0, i = tid;
    while (i >= nx) {
        i -= nx;
        ++yl;
    }
    for (; yl < TR; ) {
        const int j = y0 + yl;
        if (j >= ny) break;
        const int f = z * sz + j * sy + i;
        const unsigned mask = nbr_mask(i, j, zg, nx, ny, nzg);
        T mc[3], ex[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int q = c * csi + f;
            T nb[6];
            nb[0] = (mask & 1u) ? __ldg(m + (q - 1)) : T(0);
            nb[1] = (mask & 2u) ? __ldg(m + (q + 1)) : T(0);
            nb[2] = (mask & 4u) ? __ldg(m + (q - sy)) : T(0);
            nb[3] = (mask & 8u) ? __ldg(m + (q + sy)) : T(0);
            nb[4] = (mask & 16u) ? __ldg(m + (q - sz)) : T(0);
            nb[5] = (mask & 32u) ? __ldg(m + (q + sz)) : T(0);
            mc[c] = __ldg(m + q);
            ex[c] = exch_sum6<T>(mc[c], nb, mask);
        }
        T hx = hm[(0 * TR + yl) * nx + i], hy = hm[(1 * TR + yl) * nx + i], hz = hm[(2 * TR + yl) * nx + i];
        cl.heff(mc[0], hx, hy, hz, ex[0], ex[1], ex[2]);
        bool zero = false;
        tmax = fmax(tmax, cl.update(mc[0], mc[1], mc[2], hx, hy, hz, zero));
        if (zero)
            atomicMin(&ctl->bad_key, (static_cast<unsigned long long>(cur_step) << 36) |
                                         static_cast<unsigned long long>(f + static_cast<long long>(g.z0) * sz));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            mout[c * csi + f] = mc[c];
            hm[(c * TR + yl) * nx + i] = mc[c];
        }
        i += NT;
        while (i >= nx) {
            i -= nx;
            ++yl;
        }
    }
    }
#if MMB_XS_PAIR_LLG
llg_done:
#endif
    __syncthreads();

    // ---- 3a. forward stage A on the new tile (rows 2p, 2p+1 of one component)
    if (a_task) {
        const int ra = 2 * pa, rb = ra + 1;
        const int ya = y0 + (ra % TR), yb = ya + 1;
        const T* tra = hm + ra * nx;
        const T* trb = hm + rb * nx;
        const bool va = ya < ny, vb = yb < ny;
        constexpr int NZ = RA / 2; // x < nx <= L/2: n2 < N2 / 2
#pragma unroll
        for (int m = 0; m < NZ; ++m) {
            const int x = n1 + N1 * (LA * m + ha);
            const bool in = x < nx;
            v[m] = RC{(in && va) ? tra[x] : T(0), (in && vb) ? trb[x] : T(0)};
        }
        if constexpr (LA == 2) dft_pair<RA, -1, NZ>(v, ha);
        else DftP<N2, -1, NZ, N2>::run(v);
        if constexpr (TWPRE) {
#pragma unroll
            for (int kk = 0; kk < RA; ++kk) {
                const int k2 = kk + RA * ha;
                if (k2 > 0) v[kk] = cmul(v[kk], RC(tws[k2 * N1 + n1]));
            }
        }
    }
    __syncthreads(); // the exchange buffer overlays the tile
    if (a_task) {
        cx<T>* ex = sm + (pa * N2) * EX + n1;
#pragma unroll
        for (int kk = 0; kk < RA; ++kk) {
            const int k2 = kk + RA * ha;
            RC w = v[kk];
            if (!TWPRE && k2 > 0) w = cmul(w, RC(tws[k2 * N1 + n1]));
            ex[k2 * EX] = w;
        }
    }
    __syncthreads();
    // ---- 3b. forward stage B -> natural-order Z rows (RB rounds as in 1c)
#pragma unroll 1
    for (int rnd = 0; rnd < X::RB; ++rnd) {
        const int tb = tb0 + rnd * NT;
        const bool b_task = X::TM == 1 || tb < P * N2 * LB;
        const int pb = tb / N2, k2b = tb % N2;
        RC u[RBq];
        if (b_task) {
            const cx<T>* ex = sm + (pb * N2 + k2b) * EX + hb_;
#pragma unroll
            for (int q = 0; q < RBq; ++q) u[q] = ex[LB * q];
            if constexpr (LB == 2) dft_pair<RBq, -1, RBq>(u, hb_);
            else DftP<N1, -1, N1, N1>::run(u);
        }
        __syncthreads();
        if (b_task) {
            cx<T>* zr = sm + pb * ZP + k2b;
#pragma unroll
            for (int q = 0; q < RBq; ++q) zr[N2 * (q + RBq * hb_)] = u[q];
        }
    }
    __syncthreads();
    // ---- 3c. separate the packed rows, write the next step's half spectra (kx-major), one
    // row pair per thread as in 1a
    const T half = T(0.5);
#if MMB_XS_PAIR_STORE
    if (live0) {
        const cx<T>* zr = sm + my_p * ZP;
        for (int k = my_k0; k < XH; k += KSTEP) {
            const cx<T> zk = zr[k], zm = zr[(L - k) & (L - 1)];
            const cx<T> e{(zk.x + zm.x) * half, (zk.y - zm.y) * half};
            const cx<T> o{(zk.y + zm.y) * half, (zm.x - zk.x) * half};
            cx<T>* d = S + (k * kx_stride + row_off);
            if (vec) {
                st_pair<T>(d, e, o);
            } else {
                d[0] = e;
                if (live1) d[1] = o;
            }
        }
    }
#else
    {
        // one row per thread (odd rows take the imaginary half of their pair's Z row)
        constexpr int KS1 = NT / (3 * TR);
        const int r = tid % (3 * TR), k0 = tid / (3 * TR);
        const int c = r / TR, y = y0 + (r - c * TR);
        if (y < ny) {
            const cx<T>* zr = sm + (r >> 1) * ZP;
            const bool odd = r & 1;
            const int off = (c * nz + z) * ny + y;
            for (int k = k0; k < XH; k += KS1) {
                const cx<T> zk = zr[k], zm = zr[(L - k) & (L - 1)];
                S[k * kx_stride + off] = odd ? cx<T>{(zk.y + zm.y) * half, (zm.x - zk.x) * half}
                                             : cx<T>{(zk.x + zm.x) * half, (zk.y - zm.y) * half};
            }
        }
    }
#endif

    // ---- per-CTA torque maximum
    __shared__ double red[NT / 32];
    double t = tmax;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if ((tid & 31) == 0) red[tid >> 5] = t;
    __syncthreads();
    if (tid == 0) {
        double b = 0.0;
        for (int w = 0; w < NT / 32; ++w) b = fmax(b, red[w]);
        tpart[blockIdx.y * gridDim.x + blockIdx.x] = b;
    }
}

// Launch, with the programmatic-stream-serialization attribute (PDL; see pdl_wait) when
// `pdl`: the kernel may start launching while its predecessor in the stream drains. Measured
// to pay for multi-wave grids at one CTA per SM and to cost time on small grids, so the caller
// decides (Solver: large grids only; MMB_NO_PDL=1 disables it everywhere).
template <typename... KArgs, typename... Args>
void launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                Args... args) {
    static const bool env_off = [] {
        const char* e = std::getenv("MMB_NO_PDL");
        return e && e[0] == '1';
    }();
    const bool off = env_off || !pdl;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e));
}

template <typename K>
void set_smem(K kernel, int bytes) {
    if (bytes > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) throw std::runtime_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    }
}

#ifndef MMB_XS_PB
#define MMB_XS_PB 128 // KXS tile: 3 * (PB / N2) row pairs (XS)
#endif
#ifndef MMB_XS_PB10
#define MMB_XS_PB10 224 // Lx = 1024: 3 x 14 rows at one CTA per SM (37 tiles = exactly 2 waves
                        // at 512 x 512 x 8; 78.2 -> 74.6 us, with PDL off for this tile)
#endif
constexpr int xs_pb(int log2l) { return log2l == 10 ? MMB_XS_PB10 : MMB_XS_PB; }

#define MMB_FAST_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12)

} // namespace

template <typename T>
int fast_yz_kxb(const Geom& g, int* smem_bytes) {
    // kx per CTA: fill ~100 KB (two CTAs per SM) when possible, else one block of up to
    // the 227 KB opt-in limit.
    const int rowbytes = [&] {
        switch (g.log2ly) {
#define X(l) case l: return fpitch<l>() * static_cast<int>(sizeof(cx<T>));
            MMB_FAST_CASES(X)
#undef X
            default: return 0;
        }
    }();
    if (!rowbytes) return 0;
    const int per_kx = 3 * g.nz * rowbytes;
    const int twb = g.ly * static_cast<int>(sizeof(cx<T>));
    const int limit = 227 * 1024 - twb;
    if (per_kx > limit) return 0;
    // kx per CTA: as many as ~100 KB allows, but no more than ~2 CTAs per SM of work on large
    // grids, and on small grids enough that the columns fit one CTA wave per SM (measured:
    // 256x256 films 21.1 -> 16.8 us/step with 2 columns per CTA instead of 1)
    const int cap = std::max(1, std::min(64, (100 * 1024) / per_kx));
    int kxb = std::min(cap, std::max(1, g.xh / (2 * 148)));
    kxb = std::max(kxb, std::min(cap, (g.xh + 147) / 148));
    if (const char* e = std::getenv("MMB_YZ_KXB"); e && std::atoi(e) > 0) // tuning experiments
        kxb = std::max(1, std::min(std::atoi(e), cap));
    if (smem_bytes) *smem_bytes = kxb * per_kx + twb;
    return kxb;
}

template <typename T>
bool fast_supported(const Geom& g) {
    if (g.lx < 2 || g.ly < 2) return false;
    if (g.log2lx > 12 || g.log2ly > 12) return false;
    if (sizeof(T) == 8 && (g.log2lx > 11 || g.log2ly > 11)) return false; // DFT_64 f64 spills
    if (g.nz > 8) return false;
    if (sizeof(T) == 8 && g.nz > 1) return false; // 3 x 16 complex f64 pencils would spill
    if (g.nz > 1 && g.lz != 16) return false;
    return fast_yz_kxb<T>(g, nullptr) > 0;
}

template <typename T>
void prepare_fast_kernels(const Geom& g) {
    switch (g.log2lx) {
#define X(l) case l: set_smem(k_xf<T, l>, x_smem_bytes<T, l>()); set_smem(k_xi<T, l>, x_smem_bytes<T, l>()); \
                     if (xs_smem_bytes<T, l, xs_pb(l)>() <= 227 * 1024) set_smem(k_xstep<T, l, xs_pb(l)>, xs_smem_bytes<T, l, xs_pb(l)>()); \
                     set_smem(k_xstep<T, l, 16>, xs_smem_bytes<T, l, 16>()); break;
        MMB_FAST_CASES(X)
#undef X
        default: throw std::invalid_argument("fast path: bad Lx");
    }
    int sb = 0;
    fast_yz_kxb<T>(g, &sb);
    switch (g.log2ly) {
#define X(l) case l: set_smem(k_yz<T, l, 0>, sb); set_smem(k_yz<T, l, 0, true>, sb); \
                     if constexpr (sizeof(T) == 4) { set_smem(k_yz<T, l, 1>, sb); set_smem(k_yz<T, l, 1, true>, sb); } break;
        MMB_FAST_CASES(X)
#undef X
        default: throw std::invalid_argument("fast path: bad Ly");
    }
}

template <typename T>
void launch_fast_xf(const T* m, cx<T>* S, const Geom& g, const cx<T>* tw, StepCtl* ctl,
                    const StageTable& st, int prologue, cudaStream_t stream) {
    switch (g.log2lx) {
#define X(l) case l: { constexpr int P = x_pairs<l>(); \
        const dim3 grid((g.ny + 2 * P - 1) / (2 * P), g.nz, 3); \
        k_xf<T, l><<<grid, P * Split<l>::N2, x_smem_bytes<T, l>(), stream>>>(m, S, g, tw, ctl, st, prologue); break; }
        MMB_FAST_CASES(X)
#undef X
        default: throw std::invalid_argument("fast path: bad Lx");
    }
    check_launch();
}

template <typename T>
void launch_fast_xi(const cx<T>* S, T* h, const Geom& g, const cx<T>* tw, cudaStream_t stream) {
    switch (g.log2lx) {
#define X(l) case l: { constexpr int P = x_pairs<l>(); \
        const dim3 grid((g.ny + 2 * P - 1) / (2 * P), g.nz, 3); \
        k_xi<T, l><<<grid, P * Split<l>::N2, x_smem_bytes<T, l>(), stream>>>(S, h, g, tw); break; }
        MMB_FAST_CASES(X)
#undef X
        default: throw std::invalid_argument("fast path: bad Lx");
    }
    check_launch();
}

template <typename T>
void launch_fast_yz(cx<T>* S, const Geom& g, const cx<T>* tw, const T* kt, StepCtl* ctl,
                    const StageTable& st, int prologue, cudaStream_t stream, bool pdl, const RowMap<T>* rows) {
    RowMap<T> rm{};
    if (rows) rm = *rows;
    int sb = 0;
    const int kxb = fast_yz_kxb<T>(g, &sb);
    const unsigned grid = static_cast<unsigned>((g.xh + kxb - 1) / kxb);
    switch (g.log2ly) {
#define X(l) case l: \
        if (g.nz == 1) { if (rows) launch_pdl(pdl, k_yz<T, l, 0, true>, grid, yz_threads<T, l>(), sb, stream, S, g, tw, kt, kxb, ctl, st, prologue, rm); \
                         else launch_pdl(pdl, k_yz<T, l, 0>, grid, yz_threads<T, l>(), sb, stream, S, g, tw, kt, kxb, ctl, st, prologue, rm); } \
        else if constexpr (sizeof(T) == 4) { if (rows) launch_pdl(pdl, k_yz<T, l, 1, true>, grid, yz_threads<T, l>(), sb, stream, S, g, tw, kt, kxb, ctl, st, prologue, rm); \
                         else launch_pdl(pdl, k_yz<T, l, 1>, grid, yz_threads<T, l>(), sb, stream, S, g, tw, kt, kxb, ctl, st, prologue, rm); } \
        else throw std::invalid_argument("fast path: f64 needs nz == 1"); break;
        MMB_FAST_CASES(X)
#undef X
        default: throw std::invalid_argument("fast path: bad Ly");
    }
    check_launch();
}

template <int LOG2L>
bool xstep_small(const Geom& g) {
    return ((g.ny + XS<LOG2L, xs_pb(LOG2L)>::TR - 1) / XS<LOG2L, xs_pb(LOG2L)>::TR) * g.nz < 2 * 148;
}

template <typename T>
int fast_xstep_blocks(const Geom& g) {
    switch (g.log2lx) {
#define X(l) case l: { const dim3 gr = xstep_small<l>(g) ? xs_grid<XS<l, 16>>(g) : xs_grid<XS<l, xs_pb(l)>>(g); \
        return static_cast<int>(gr.x * gr.y); }
        MMB_FAST_CASES(X)
#undef X
        default: throw std::invalid_argument("fast path: bad Lx");
    }
}

// TMA descriptor of the kx-major half spectra S for the x tiles: 3-D (y, (c, z) row, kx) in
// 8-byte elements, box TR y x 1 row x BOXK kx. False (plain async copies instead) when the
// driver entry point is missing, MMB_XS_TMA=0, or the layout breaks TMA's 16-byte rules.
template <typename T>
bool xs_tensor_map(CUtensorMap* tm, const cx<T>* S, const Geom& g, int tr, int boxk) {
    const bool off = env_off("MMB_XS_TMA"); // read per launch (graph capture): A/B in one process
    const unsigned long long e = sizeof(cx<T>) / 8, esz = sizeof(cx<T>);
    return !off && make_tmap_3d(tm, S, g.ny * e, 3ull * g.nz, g.xh, g.ny * esz, 3ull * g.nz * g.ny * esz,
                                static_cast<unsigned>(tr * e), 1u, static_cast<unsigned>(boxk));
}

template <typename T>
void launch_fast_xstep(cx<T>* S, const T* m, T* mout, const Geom& g, const cx<T>* tw,
                       double exch_coeff, double aniso_coeff, StepCtl* ctl, double* tpart,
                       cudaStream_t stream, bool pdl) {
    const T coeff = static_cast<T>(exch_coeff), kan = static_cast<T>(aniso_coeff);
    switch (g.log2lx) {
#define X(l) case l: if (xstep_small<l>(g)) { using XA = XS<l, 16, sizeof(T)>; const dim3 grid = xs_grid<XA>(g); \
        CUtensorMap tm{}; const int ut = XA::TMA && xs_tensor_map<T>(&tm, S, g, XA::TR, XA::BOXK); \
        launch_pdl(pdl, k_xstep<T, l, 16>, grid, XA::NT, xs_smem_bytes<T, l, 16>(), stream, S, m, mout, g, tw, coeff, kan, ctl, tpart, tm, ut); \
        } else { using XB = XS<l, xs_pb(l), sizeof(T)>; \
        if (xs_smem_bytes<T, l, xs_pb(l)>() > 227 * 1024) throw std::invalid_argument("fast path: x tile exceeds shared memory"); \
        const dim3 grid = xs_grid<XB>(g); \
        CUtensorMap tm{}; const int ut = XB::TMA && xs_tensor_map<T>(&tm, S, g, XB::TR, XB::BOXK); \
        launch_pdl(pdl, k_xstep<T, l, xs_pb(l)>, grid, XB::NT, xs_smem_bytes<T, l, xs_pb(l)>(), stream, S, m, mout, g, tw, coeff, kan, ctl, tpart, tm, ut); } break;
        MMB_FAST_CASES(X)
#undef X
        default: throw std::invalid_argument("fast path: bad Lx");
    }
    check_launch();
}

// Kernel variants the geometry selects (tests assert that each production variant is covered).
template <typename T>
std::string fast_describe(const Geom& g) {
    char buf[256];
    int sb = 0;
    const int kxb = fast_yz_kxb<T>(g, &sb);
    std::string yz;
    switch (g.log2ly) {
#define X(l) case l: std::snprintf(buf, sizeof buf, "k_yz<L%d,ZM%d> kxb=%d nt=%d ctas=%d", l, g.nz == 1 ? 0 : 1, kxb, \
                                   yz_threads<T, l>(), kxb > 0 ? (g.xh + kxb - 1) / kxb : 0); yz = buf; break;
        MMB_FAST_CASES(X)
#undef X
        default: yz = "k_yz<?>";
    }
    std::string xs;
    switch (g.log2lx) {
#define X(l) case l: { const bool sm = xstep_small<l>(g); \
        using XA = XS<l, 16, sizeof(T)>; using XB = XS<l, xs_pb(l), sizeof(T)>; \
        const dim3 gr = sm ? xs_grid<XA>(g) : xs_grid<XB>(g); \
        const bool tma = (sm ? XA::TMA : XB::TMA) && !env_off("MMB_XS_TMA") && tmap_encoder() && (g.ny * sizeof(cx<T>)) % 16 == 0; \
        std::snprintf(buf, sizeof buf, "k_xstep<L%d,PB%d> tr=%d nt=%d %s grid=%ux%u staging=%s", l, sm ? 16 : xs_pb(l), \
                      sm ? XA::TR : XB::TR, sm ? XA::NT : XB::NT, \
                      (sm ? XA::PAIR : XB::PAIR) ? "pair" : ((sm ? XA::WIDE : XB::WIDE) ? "wide" : "plain"), gr.x, gr.y, \
                      tma ? "tma" : "copies"); \
        xs = buf; break; }
        MMB_FAST_CASES(X)
#undef X
        default: xs = "k_xstep<?>";
    }
    return yz + "; " + xs;
}

#define MMB_FINST(T)                                                                            \
    template std::string fast_describe<T>(const Geom&);                                        \
    template int fast_yz_kxb<T>(const Geom&, int*);                                            \
    template bool fast_supported<T>(const Geom&);                                              \
    template void prepare_fast_kernels<T>(const Geom&);                                        \
    template void launch_fast_xf<T>(const T*, cx<T>*, const Geom&, const cx<T>*, StepCtl*,      \
                                    const StageTable&, int, cudaStream_t);                     \
    template void launch_fast_xi<T>(const cx<T>*, T*, const Geom&, const cx<T>*, cudaStream_t); \
    template void launch_fast_yz<T>(cx<T>*, const Geom&, const cx<T>*, const T*, StepCtl*,         \
                                    const StageTable&, int, cudaStream_t, bool, const RowMap<T>*); \
    template int fast_xstep_blocks<T>(const Geom&);                                            \
    template void launch_fast_xstep<T>(cx<T>*, const T*, T*, const Geom&, const cx<T>*, double, \
                                       double, StepCtl*, double*, cudaStream_t, bool);
#ifndef MMB_ONLY_F64
MMB_FINST(float)
#endif
#ifndef MMB_ONLY_F32
MMB_FINST(double)
#endif

} // namespace mmb
