// tensor_kernels.cu — one-time spectral tensor precompute (replaces build_demag_tensor +
// spectral_prepare, proj/src/demag_tensor.cpp:45-82 and proj/src/demag.cpp:10-31).
//
// The reference stores the tensor shifted (offset o at o+n-1) on the doubled grid and takes
// six full complex FFTs. Stored wrapped instead (offset o at o mod L), every component is
// even or odd along each axis, so its spectrum is REAL and fixed by the non-negative
// octant: per axis an even component transforms by E(k) = f(0) + 2 sum_o f(o) cos(2pi k o/L)
// and an odd one by -i S(k), S(k) = 2 sum_o f(o) sin(2pi k o/L). Off-diagonals are odd in two
// axes, so their spectrum is -S_a S_b E_c (real). Evaluated in fp64 as three separable
// dense passes, scaled by 1/(Lx Ly Lz) (exact, powers of two) and narrowed to T.
#include <stdexcept>
#include <string>

#include "fast.hpp"
#include "kernels.hpp"

namespace mmb {

namespace {

void check_launch() {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch: ") + cudaGetErrorString(e));
}

// cs[j] = (cos(2 pi j / L), sin(2 pi j / L)), exact argument reduction via sincospi.
__global__ void k_cs_table(double2* cs, int L) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= L) return;
    double s, c;
    sincospi(2.0 * static_cast<double>(j) / static_cast<double>(L), &s, &c);
    cs[j] = make_double2(c, s);
}

// One output element per thread: out[k] = sum_o w(k, o) in[o] along `axis`, for each of the
// six components (blockIdx.y). odd_mask bit c set => component c is odd along this axis.
__global__ void k_axis_transform(const double* __restrict__ in, double* __restrict__ out, int d0,
                                 int d1, int d2, int axis, int L, int nout,
                                 const double2* __restrict__ cs, int odd_mask, long long csi,
                                 long long cso, int k0) {
    const int c = blockIdx.y;
    const bool odd = (odd_mask >> c) & 1;
    int od[3] = {d0, d1, d2};
    const int nin = od[axis];
    od[axis] = nout;
    const long long total = static_cast<long long>(od[0]) * od[1] * od[2];
    const long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= total) return;
    int idx[3];
    idx[0] = static_cast<int>(f % od[0]);
    idx[1] = static_cast<int>((f / od[0]) % od[1]);
    idx[2] = static_cast<int>(f / (static_cast<long long>(od[0]) * od[1]));
    const int k = idx[axis] + k0; // output frequencies [k0, k0 + nout)
    long long stride_in = 1;
    if (axis >= 1) stride_in *= d0;
    if (axis >= 2) stride_in *= d1;
    idx[axis] = 0;
    const long long base = idx[0] + static_cast<long long>(d0) * (idx[1] + static_cast<long long>(d1) * idx[2]);
    const double* src = in + c * csi + base;
    double acc = 0.0;
    if (L == 1) {
        acc = src[0];
    } else if (!odd) {
        acc = src[0];
        for (int o = 1; o < nin; ++o) {
            const int t = static_cast<int>((static_cast<long long>(k) * o) & (L - 1));
            acc += 2.0 * cs[t].x * src[o * stride_in];
        }
    } else {
        for (int o = 1; o < nin; ++o) {
            const int t = static_cast<int>((static_cast<long long>(k) * o) & (L - 1));
            acc += 2.0 * cs[t].y * src[o * stride_in];
        }
    }
    out[c * cso + f] = acc;
}

template <typename T>
__global__ void k_finalize(const double* __restrict__ spec, T* __restrict__ out, long long count,
                           double scale) {
    const long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= count) return;
    const int c = blockIdx.y;
    // xx, xy, xz, yy, yz, zz: off-diagonals carry (-i)^2 = -1 from their two odd axes.
    const double sgn = (c == 1 || c == 2 || c == 4) ? -1.0 : 1.0;
    out[c * count + f] = static_cast<T>(sgn * scale * spec[c * count + f]);
}

// Fast-path layout [kx][kz][ky][c] (the six coefficients of one frequency contiguous, ky next):
// one contiguous tensor slab per kx, three 2-vector loads per frequency in the MAC.
template <typename T>
__global__ void k_finalize_fast(const double* __restrict__ spec, T* __restrict__ out, int xh, int yh,
                                int zh, double scale) {
    const long long count = static_cast<long long>(xh) * yh * zh;
    const long long f = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (f >= count) return;
    const int c = blockIdx.y;
    const int kx = static_cast<int>(f % xh);
    const long long r = f / xh;
    const int ky = static_cast<int>(r % yh), kz = static_cast<int>(r / yh);
    const double sgn = (c == 1 || c == 2 || c == 4) ? -1.0 : 1.0;
    out[((static_cast<long long>(kx) * zh + kz) * yh + ky) * 6 + c] =
        static_cast<T>(sgn * scale * spec[c * count + f]);
}

// tw[t] = W_L^t = exp(-2 pi i t / L) for t < L, fp64 sincospi then narrowed; then
// tw[L + k2 * N1 + n1] = W_L^(n1 k2), the same values in the [k2][n1] order of the register
// four-step (fft4.cuh Split), which the kernels copy to shared memory with async bulk copies.
template <typename T>
__global__ void k_twiddles(cx<T>* tw, int L, int log2n1) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 2 * L) return;
    int e = t;
    if (t >= L) {
        const int f = t - L, n1 = f & ((1 << log2n1) - 1), k2 = f >> log2n1;
        e = n1 * k2;
    }
    double s, c;
    sincospi(2.0 * static_cast<double>(e) / static_cast<double>(L), &s, &c);
    tw[t] = cx<T>{static_cast<T>(c), static_cast<T>(-s)};
}

} // namespace

void launch_cs_table(double2* cs, int L, cudaStream_t stream) {
    k_cs_table<<<(L + 255) / 256, 256, 0, stream>>>(cs, L);
    check_launch();
}

void launch_axis_transform(const double* in, double* out, int d0, int d1, int d2, int axis, int L,
                           const double2* cs_table, int odd_mask, long long csi, long long cso,
                           cudaStream_t stream, int k0, int nk) {
    int od[3] = {d0, d1, d2};
    od[axis] = nk >= 0 ? nk : ((L == 1) ? 1 : L / 2 + 1);
    const long long total = static_cast<long long>(od[0]) * od[1] * od[2];
    const dim3 grid(static_cast<unsigned>((total + 255) / 256), 6);
    k_axis_transform<<<grid, 256, 0, stream>>>(in, out, d0, d1, d2, axis, L, od[axis], cs_table,
                                               odd_mask, csi, cso, k0);
    check_launch();
}

template <typename T>
void launch_tensor_finalize(const double* spec, T* out, long long count, double scale,
                            cudaStream_t stream) {
    const dim3 grid(static_cast<unsigned>((count + 255) / 256), 6);
    k_finalize<T><<<grid, 256, 0, stream>>>(spec, out, count, scale);
    check_launch();
}

template <typename T>
void launch_tensor_finalize_fast(const double* spec, T* out, int xh, int yh, int zh, double scale,
                                 cudaStream_t stream) {
    const long long count = static_cast<long long>(xh) * yh * zh;
    const dim3 grid(static_cast<unsigned>((count + 255) / 256), 6);
    k_finalize_fast<T><<<grid, 256, 0, stream>>>(spec, out, xh, yh, zh, scale);
    check_launch();
}

template <typename T>
void launch_twiddles(cx<T>* tw, int L, cudaStream_t stream) {
    int log2l = 0;
    while ((1 << log2l) < L) ++log2l;
    k_twiddles<T><<<(2 * L + 255) / 256, 256, 0, stream>>>(tw, L, log2l / 2);
    check_launch();
}

template void launch_tensor_finalize<float>(const double*, float*, long long, double, cudaStream_t);
template void launch_tensor_finalize<double>(const double*, double*, long long, double, cudaStream_t);
template void launch_tensor_finalize_fast<float>(const double*, float*, int, int, int, double, cudaStream_t);
template void launch_tensor_finalize_fast<double>(const double*, double*, int, int, int, double, cudaStream_t);
template void launch_twiddles<float>(cx<float>*, int, cudaStream_t);
template void launch_twiddles<double>(cx<double>*, int, cudaStream_t);

} // namespace mmb
