// llg_kernels.cu — fused local terms + explicit-Euler LLG update, reductions and the
// one-time prism-sum tensor entries. Compiled with --fmad=false: every product and sum here
// rounds separately, exactly like the reference's x86-64 (SSE2, no FMA) build, so given the
// same H_demag the local part of H_eff and the updated M agree bitwise.
#include <stdexcept>
#include <string>

#include "kernels.hpp"

namespace mmb {

namespace {

constexpr int kTileX = 32, kTileY = 8, kLlgThreads = kTileX * kTileY;
constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 592; // 4 x 148 SMs; fixed so the reduction order is deterministic

void check_launch() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Exchange sum for one component, neighbour order -x,+x,-y,+y,-z,+z with Neumann skips
// (proj/src/local_fields.cpp:27-39).
template <typename T>
__device__ __forceinline__ T exch_sum(const T* __restrict__ src, long long f, int i, int j, int k,
                                      int nx, int ny, int nz, long long sy, long long sz) {
    const T center = __ldg(src + f);
    T sum = T(0);
    if (i > 0) sum += __ldg(src + f - 1) - center;
    if (i + 1 < nx) sum += __ldg(src + f + 1) - center;
    if (j > 0) sum += __ldg(src + f - sy) - center;
    if (j + 1 < ny) sum += __ldg(src + f + sy) - center;
    if (k > 0) sum += __ldg(src + f - sz) - center;
    if (k + 1 < nz) sum += __ldg(src + f + sz) - center;
    return sum;
}

// K6: fused local terms + Euler + renormalisation, one thread per cell, 32 x 8 (x, y) tiles
// per CTA and one z plane per grid row (no integer division; x/y neighbours of a tile hit
// L1, z neighbours L2). M and H_demag are read once from HBM, M_{t+1} written once
// (ping-pong buffers).
//   H = H_demag; H += coeff * exch_sum (local_fields.cpp:39; neighbour order -x,+x,-y,+y,
//   -z,+z with Neumann skips, :27-38); Hx += (hk/ms) Mx (local_fields.hpp:28-31);
//   H += applied (local_fields.hpp:43-55)
//   T = M x H; dM = p1 T + p2 (M x T); M += dM (llg.cpp:82-93); max |T|^2 in fp64 (:89-90)
//   mag = sqrt(Mx^2 + My^2 + Mz^2); M *= T(ms)/mag (vector_field.hpp:56-76)
// MODE 1 writes H_eff instead (field assembly only). Per-CTA torque maxima go to tpart[]
// (reduced on demand), so the hot path has no same-address atomics.
template <typename T>
__device__ __forceinline__ T exch1(const T* __restrict__ p, int i, int j, int k, int nx, int ny,
                                   int nz, int sy, int sz) {
    const T center = __ldg(p);
    T sum = T(0);
    if (i > 0) sum += __ldg(p - 1) - center;
    if (i + 1 < nx) sum += __ldg(p + 1) - center;
    if (j > 0) sum += __ldg(p - sy) - center;
    if (j + 1 < ny) sum += __ldg(p + sy) - center;
    if (k > 0) sum += __ldg(p - sz) - center;
    if (k + 1 < nz) sum += __ldg(p + sz) - center;
    return sum;
}

template <typename T, int MODE>
__global__ void __launch_bounds__(kLlgThreads) k_llg(const T* __restrict__ m, const T* __restrict__ hd,
                                                     T* __restrict__ out, Geom g, T coeff, T kan,
                                                     StepCtl* ctl, double* __restrict__ tpart) {
    // component stride cs (= n on one device; a slab's buffers carry halo planes) and the
    // global plane index for the Neumann mask (slabs: the halo planes hold the neighbours')
    const long long n = g.cs;
    const int nx = g.nx, ny = g.ny, nzg = g.nz_g;
    const int sy = nx, sz = nx * ny;
    const int tx = threadIdx.x, ty = threadIdx.y, lt = ty * kTileX + tx;
    const long long cur_step = ctl->cur_step;
    if (MODE == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && lt == 0)
        ctl->step = cur_step + 1;
    const int i = blockIdx.x * kTileX + tx, j = blockIdx.y * kTileY + ty, k = blockIdx.z, kg = g.z0 + k;
    double tmax = 0.0;
    if (i < nx && j < ny) {
        const T ax = static_cast<T>(ctl->field[0]);
        const T ay = static_cast<T>(ctl->field[1]);
        const T az = static_cast<T>(ctl->field[2]);
        const int f = k * sz + j * sy + i;
        const T* px = m + f;
        const T* py = px + n;
        const T* pz = py + n;
        const T mx = __ldg(px), my = __ldg(py), mz = __ldg(pz);
        T hx = __ldg(hd + f), hy = __ldg(hd + n + f), hz = __ldg(hd + 2 * n + f);
        hx += coeff * exch1(px, i, j, kg, nx, ny, nzg, sy, sz);
        hy += coeff * exch1(py, i, j, kg, nx, ny, nzg, sy, sz);
        hz += coeff * exch1(pz, i, j, kg, nx, ny, nzg, sy, sz);
        hx += kan * mx;
        hx += ax;
        hy += ay;
        hz += az;
        if constexpr (MODE == 1) {
            out[f] = hx;
            out[n + f] = hy;
            out[2 * n + f] = hz;
        } else {
            const T p1 = static_cast<T>(ctl->p1);
            const T p2 = static_cast<T>(ctl->p2);
            const T ms = static_cast<T>(ctl->ms);
            const T tqx = my * hz - mz * hy;
            const T tqy = mz * hx - mx * hz;
            const T tqz = mx * hy - my * hx;
            const T dx = p1 * tqx + p2 * (my * tqz - mz * tqy);
            const T dy = p1 * tqy + p2 * (mz * tqx - mx * tqz);
            const T dz = p1 * tqz + p2 * (mx * tqy - my * tqx);
            tmax = double(tqx) * tqx + double(tqy) * tqy + double(tqz) * tqz;
            T nxv = mx + dx, nyv = my + dy, nzv = mz + dz;
            const T mag = sqrt(nxv * nxv + nyv * nyv + nzv * nzv);
            if (mag == T(0)) {
                atomicMin(&ctl->bad_key, (static_cast<unsigned long long>(cur_step) << 36) |
                                             static_cast<unsigned long long>(f + static_cast<long long>(g.z0) * sz));
            } else {
                const T scale = ms / mag;
                nxv *= scale;
                nyv *= scale;
                nzv *= scale;
            }
            out[f] = nxv;
            out[n + f] = nyv;
            out[2 * n + f] = nzv;
        }
    }
    if constexpr (MODE == 0) {
        __shared__ double red[kLlgThreads / 32];
        tmax = warp_max(tmax);
        if ((lt & 31) == 0) red[lt >> 5] = tmax;
        __syncthreads();
        if (lt < 32) {
            double v = lt < kLlgThreads / 32 ? red[lt] : 0.0;
            v = warp_max(v);
            if (lt == 0) tpart[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = v;
        }
    }
}

// max over the per-CTA torque partials -> ctl->torque_sq_bits
__global__ void k_torque_partials(const double* __restrict__ tpart, int nb, StepCtl* ctl) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) v = fmax(v, tpart[b]);
    __shared__ double red[8];
    v = warp_max(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
        ctl->torque_sq_bits = static_cast<unsigned long long>(__double_as_longlong(t));
    }
}

// Block-partial fp64 sums of the three components in a fixed order.
template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_sum3(const T* __restrict__ m, long long n,
                                                      long long cs, double* __restrict__ partial) {
    double s[3] = {0.0, 0.0, 0.0};
    for (long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; f < n;
         f += static_cast<long long>(gridDim.x) * blockDim.x) {
        s[0] += double(__ldg(m + f));
        s[1] += double(__ldg(m + cs + f));
        s[2] += double(__ldg(m + 2 * cs + f));
    }
    __shared__ double red[3][kRedThreads / 32];
    for (int c = 0; c < 3; ++c) {
        const double v = warp_sum(s[c]);
        if ((threadIdx.x & 31) == 0) red[c][threadIdx.x >> 5] = v;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        double t = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) t += red[threadIdx.x][w];
        partial[blockIdx.x * 3 + threadIdx.x] = t;
    }
}

// Sums nblk x NV partials in block order (one warp per value).
template <int NV>
__global__ void k_final_sum(const double* __restrict__ partial, int nblk, double* __restrict__ out) {
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (c >= NV) return;
    double s = 0.0;
    for (int b = lane; b < nblk; b += 32) s += partial[b * NV + c];
    s = warp_sum(s);
    if (lane == 0) out[c] = s;
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_torque_max(const T* __restrict__ m, const T* __restrict__ h,
                                                            long long n, long long cs, unsigned long long* out) {
    double t = 0.0;
    for (long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; f < n;
         f += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double mx = m[f], my = m[cs + f], mz = m[2 * cs + f];
        const double hx = h[f], hy = h[cs + f], hz = h[2 * cs + f];
        const double tx = my * hz - mz * hy;
        const double ty = mz * hx - mx * hz;
        const double tz = mx * hy - my * hx;
        t = fmax(t, tx * tx + ty * ty + tz * tz);
    }
    __shared__ double red[kRedThreads / 32];
    t = warp_max(t);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < kRedThreads / 32 ? red[threadIdx.x] : 0.0;
        v = warp_max(v);
        if (threadIdx.x == 0) atomicMax(out, __double_as_longlong(v));
    }
}

// proj/src/energy.cpp:39-64 local density (anisotropy + demag + Zeeman) and the
// forward-difference exchange bonds (:17-36), fp64.
template <typename T>
__global__ void __launch_bounds__(kRedThreads) k_energy(const T* __restrict__ m, const T* __restrict__ hd,
                                                        Geom g, double ku_over_ms2,
                                                        const StepCtl* ctl, double* __restrict__ partial) {
    // cells of this geometry (a slab: its nz local planes, component stride cs, global plane
    // z0 + k; the +z bond of its last plane reads the halo plane above it)
    const long long n = g.n, cs = g.cs;
    const int nx = g.nx, ny = g.ny, nzg = g.nz_g;
    const double ex = ctl->field[0], ey = ctl->field[1], ez = ctl->field[2];
    double loc = 0.0, bonds = 0.0;
    for (long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; f < n;
         f += static_cast<long long>(gridDim.x) * blockDim.x) {
        const double x = m[f], y = m[cs + f], z = m[2 * cs + f];
        const double hx = hd[f], hy = hd[cs + f], hz = hd[2 * cs + f];
        const double anis = ku_over_ms2 * (y * y + z * z);
        const double demag = -0.5 * kMu0 * (hx * x + hy * y + hz * z);
        const double zeeman = -kMu0 * (ex * x + ey * y + ez * z);
        loc += anis + demag + zeeman;
        const int i = static_cast<int>(f % nx);
        const long long r = f / nx;
        const int j = static_cast<int>(r % ny);
        const int k = g.z0 + static_cast<int>(r / ny);
        auto bond = [&](long long b) {
            const double dx = double(m[b]) - x, dy = double(m[cs + b]) - y, dz = double(m[2 * cs + b]) - z;
            return dx * dx + dy * dy + dz * dz;
        };
        if (i + 1 < nx) bonds += bond(f + 1);
        if (j + 1 < ny) bonds += bond(f + nx);
        if (k + 1 < nzg) bonds += bond(f + static_cast<long long>(nx) * ny);
    }
    __shared__ double red[2][kRedThreads / 32];
    loc = warp_sum(loc);
    bonds = warp_sum(bonds);
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = loc;
        red[1][threadIdx.x >> 5] = bonds;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        double t = 0.0;
        for (int w = 0; w < kRedThreads / 32; ++w) t += red[threadIdx.x][w];
        partial[blockIdx.x * 2 + threadIdx.x] = t;
    }
}

// The eight-corner prism sums (proj/src/demag_tensor.cpp:9-43) in fp64 at integer offset
// (I, J, K) of any sign, in the order xx, xy, xz, yy, yz, zz.
__device__ __forceinline__ void tensor_entry(int I, int J, int K, double delta, double e[6]) {
    double xx = 0, xy = 0, xz = 0, yy = 0, yz = 0, zz = 0;
#pragma unroll
    for (int i = 0; i <= 1; ++i)
#pragma unroll
        for (int j = 0; j <= 1; ++j)
#pragma unroll
            for (int k = 0; k <= 1; ++k) {
                const double sign = ((i + j + k) & 1) ? -1.0 : 1.0;
                const double x = I + i - 0.5;
                const double y = J + j - 0.5;
                const double z = K + k - 0.5;
                const double r = delta * sqrt(x * x + y * y + z * z);
                xx += sign * atan(z * y * delta / (r * x));
                yy += sign * atan(x * z * delta / (r * y));
                zz += sign * atan(y * x * delta / (r * z));
                xy += sign * log(z * delta + r);
                xz += sign * log(y * delta + r);
                yz += sign * log(x * delta + r);
            }
    const double p = 1.0 / (4.0 * 3.14159265358979323846);
    e[0] = xx * p;
    e[1] = xy * -p;
    e[2] = xz * -p;
    e[3] = yy * p;
    e[4] = yz * -p;
    e[5] = zz * p;
}

// K0: tensor_entry on the non-negative octant; other octants follow by parity.
// E is [6][nz][ny][nx].
__global__ void k_tensor_octant(double* __restrict__ E, int nx, int ny, int nz, double delta) {
    const long long cnt = static_cast<long long>(nx) * ny * nz;
    const long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= cnt) return;
    const int I = static_cast<int>(f % nx);
    const int J = static_cast<int>((f / nx) % ny);
    const int K = static_cast<int>(f / (static_cast<long long>(nx) * ny));
    double e[6];
    tensor_entry(I, J, K, delta, e);
#pragma unroll
    for (int c = 0; c < 6; ++c) E[c * cnt + f] = e[c];
}

// tensor_entry at n arbitrary offsets ijk[3n] -> out[6n] (validation suite).
__global__ void k_tensor_entries(const int* __restrict__ ijk, int n, double delta, double* __restrict__ out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    double e[6];
    tensor_entry(ijk[3 * t], ijk[3 * t + 1], ijk[3 * t + 2], delta, e);
#pragma unroll
    for (int c = 0; c < 6; ++c) out[6 * t + c] = e[c];
}

} // namespace

int reduce_blocks(long long n) {
    const long long b = (n + kRedThreads - 1) / kRedThreads;
    return static_cast<int>(b < kRedBlocks ? (b < 1 ? 1 : b) : kRedBlocks);
}

int llg_blocks(const Geom& g) {
    return ((g.nx + kTileX - 1) / kTileX) * ((g.ny + kTileY - 1) / kTileY) * g.nz;
}

// One thread spinning on the global timer: keeps the stream busy for `ns` nanoseconds so that
// the host has enqueued a timed sequence before its start event is processed (the timing then
// excludes host launch latency, as in a long run where the device runs ahead of the host).
__global__ void k_spin(unsigned long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < ns);
}

void launch_spin(unsigned long long ns, cudaStream_t stream) {
    k_spin<<<1, 1, 0, stream>>>(ns);
    check_launch();
}

void launch_torque_partials(const double* tpart, int nb, StepCtl* ctl, cudaStream_t stream) {
    k_torque_partials<<<1, 256, 0, stream>>>(tpart, nb, ctl);
    check_launch();
}

template <typename T>
void launch_llg(int mode, const T* m, const T* hd, T* out, const Geom& g, double exch_coeff,
                double aniso_coeff, StepCtl* ctl, double* tpart, cudaStream_t stream) {
    const dim3 grid((g.nx + kTileX - 1) / kTileX, (g.ny + kTileY - 1) / kTileY, g.nz);
    const dim3 block(kTileX, kTileY);
    const T coeff = static_cast<T>(exch_coeff), kan = static_cast<T>(aniso_coeff);
    if (mode == 0) k_llg<T, 0><<<grid, block, 0, stream>>>(m, hd, out, g, coeff, kan, ctl, tpart);
    else k_llg<T, 1><<<grid, block, 0, stream>>>(m, hd, out, g, coeff, kan, ctl, tpart);
    check_launch();
}

template <typename T>
void launch_sum3(const T* m, long long n, long long cs, double* partial, double* out, cudaStream_t stream) {
    const int nb = reduce_blocks(n);
    k_sum3<T><<<nb, kRedThreads, 0, stream>>>(m, n, cs, partial);
    k_final_sum<3><<<1, 96, 0, stream>>>(partial, nb, out);
    check_launch();
}

template <typename T>
void launch_torque_max(const T* m, const T* h, long long n, long long cs, unsigned long long* out_bits,
                       cudaStream_t stream) {
    cudaMemsetAsync(out_bits, 0, sizeof(unsigned long long), stream);
    k_torque_max<T><<<reduce_blocks(n), kRedThreads, 0, stream>>>(m, h, n, cs, out_bits);
    check_launch();
}

template <typename T>
void launch_energy(const T* m, const T* hd, const Geom& g, double ku_over_ms2, const StepCtl* ctl,
                   double* partial, double* out, cudaStream_t stream) {
    const int nb = reduce_blocks(g.n);
    k_energy<T><<<nb, kRedThreads, 0, stream>>>(m, hd, g, ku_over_ms2, ctl, partial);
    k_final_sum<2><<<1, 64, 0, stream>>>(partial, nb, out);
    check_launch();
}

void launch_tensor_entries(const int* ijk, int n, double delta, double* out, cudaStream_t stream) {
    if (n <= 0) return;
    k_tensor_entries<<<(n + 127) / 128, 128, 0, stream>>>(ijk, n, delta, out);
    check_launch();
}

void launch_tensor_octant(double* E, int nx, int ny, int nz, double delta, cudaStream_t stream) {
    const long long cnt = static_cast<long long>(nx) * ny * nz;
    k_tensor_octant<<<static_cast<unsigned>((cnt + 127) / 128), 128, 0, stream>>>(E, nx, ny, nz, delta);
    check_launch();
}

#define MMB_INST(T)                                                                                 \
    template void launch_llg<T>(int, const T*, const T*, T*, const Geom&, double, double, StepCtl*, \
                                double*, cudaStream_t);                                            \
    template void launch_sum3<T>(const T*, long long, long long, double*, double*, cudaStream_t);   \
    template void launch_torque_max<T>(const T*, const T*, long long, long long, unsigned long long*, \
                                       cudaStream_t);                                              \
    template void launch_energy<T>(const T*, const T*, const Geom&, double, const StepCtl*,         \
                                   double*, double*, cudaStream_t);
MMB_INST(float)
MMB_INST(double)

} // namespace mmb
