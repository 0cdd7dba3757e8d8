// kernels.hpp — host-side launchers for the sm_100a kernels (implemented in fft_kernels.cu,
// llg_kernels.cu and tensor_kernels.cu). All launches are asynchronous on `stream`.
#pragma once

#include <cuda_runtime.h>

#include "types.cuh"

namespace mmb {

// ---- demag convolution (fft_kernels.cu) -----------------------------------------------
// K1: x-axis r2c of the live rows of M (pairs of real rows packed as one complex row),
// writes the half spectrum rows of S. Optionally runs the step prologue (mode 1 = stepping,
// 2 = field assembly only) in block 0.
template <typename T>
void launch_x_fwd(const T* m, cx<T>* S, const Geom& g, const cx<T>* tw, StepCtl* ctl,
                  const StageTable& st, int prologue, cudaStream_t stream);
// K2/K4: y-axis forward (ny live rows -> Ly spectrum rows) / inverse (Ly -> ny live rows).
template <typename T>
void launch_y(int inverse, cx<T>* S, const Geom& g, const cx<T>* tw, cudaStream_t stream);
// nz == 1: fused y-forward, tensor MAC, y-inverse.
template <typename T>
void launch_y_mac(cx<T>* S, const Geom& g, const cx<T>* tw, const T* kspec, cudaStream_t stream);
// K3 (nz > 1): fused z-forward, tensor MAC, z-inverse per (kx, ky) pencil.
template <typename T>
void launch_z_mac(cx<T>* S, const Geom& g, const cx<T>* tw, const T* kspec, cudaStream_t stream);
// K5: x-axis c2r back to the nx live cells of H_demag.
template <typename T>
void launch_x_inv(const cx<T>* S, T* h, const Geom& g, const cx<T>* tw, cudaStream_t stream);
// Smem attribute setup for every instantiation the geometry needs (call once, outside capture).
template <typename T>
void prepare_fft_kernels(const Geom& g);

// ---- local terms + LLG update (llg_kernels.cu, compiled without FMA contraction) -------
// mode 0: H_eff = hd + exchange + anisotropy + applied; Euler; renormalise; write m_out.
// mode 1: write H_eff only (m_out receives H_eff), no state change.
// m, hd and out share the component stride g.cs; the exchange mask uses the global plane
// g.z0 + k of g.nz_g (a slab's halo planes must then hold the neighbouring planes).
template <typename T>
void launch_llg(int mode, const T* m, const T* hd, T* out, const Geom& g, double exch_coeff,
                double aniso_coeff, StepCtl* ctl, double* tpart, cudaStream_t stream);
// CTAs of launch_llg (size of its per-CTA torque partial array) and their reduction into
// ctl->torque_sq_bits.
int llg_blocks(const Geom& g);
void launch_torque_partials(const double* tpart, int nb, StepCtl* ctl, cudaStream_t stream);
// Deterministic fp64 sums of the n cells of each M component (component stride cs):
// partial[nblk*3] then out[3] (sum, not mean).
template <typename T>
void launch_sum3(const T* m, long long n, long long cs, double* partial, double* out, cudaStream_t stream);
// max over the n cells of |M x H|^2 in fp64 -> *out_bits (double bits, atomicMax); component
// stride cs of both fields.
template <typename T>
void launch_torque_max(const T* m, const T* h, long long n, long long cs, unsigned long long* out_bits,
                       cudaStream_t stream);
// Total energy (proj/src/energy.cpp:5-64) partial sums: local (anis+demag+zeeman) and
// exchange bonds, fp64, deterministic -> out[2]. Over the g.n cells of g (component stride
// g.cs; a slab's +z bonds of its last plane read the halo plane above).
template <typename T>
void launch_energy(const T* m, const T* hd, const Geom& g, double ku_over_ms2,
                   const StepCtl* ctl, double* partial, double* out, cudaStream_t stream);
int reduce_blocks(long long n);
// keep `stream` busy for ns nanoseconds (timing helper: the host enqueues the timed work meanwhile)
void launch_spin(unsigned long long ns, cudaStream_t stream);

// ---- one-time tensor precompute (tensor_kernels.cu) ------------------------------------
// K0: fp64 prism-sum entries on the non-negative octant, E[6][nz][ny][nx]
// (proj/src/demag_tensor.cpp:9-43).
void launch_tensor_octant(double* E, int nx, int ny, int nz, double delta, cudaStream_t stream);
// The same prism sums at n signed offsets ijk[3n] -> out[6n] (validation suite).
void launch_tensor_entries(const int* ijk, int n, double delta, double* out, cudaStream_t stream);
// Per-axis real cosine / sine transform of the octant (wrapped-kernel spectrum), fp64.
// in dims (d0 fastest, d1, d2); transforms axis `axis` from length n to L/2+1 (1 if L == 1).
// [k0, k0 + nk) selects a range of the output frequencies (nk < 0: all L/2+1).
void launch_axis_transform(const double* in, double* out, int d0, int d1, int d2, int axis,
                           int L, const double2* cs_table, int odd_mask_for_axis,
                           long long comp_stride_in, long long comp_stride_out,
                           cudaStream_t stream, int k0 = 0, int nk = -1);
void launch_cs_table(double2* cs, int L, cudaStream_t stream);
template <typename T>
void launch_tensor_finalize(const double* spec, T* out, long long count, double scale,
                            cudaStream_t stream);
// tw[2L]: W_L^t (t < L), then the same values in four-step [k2][n1] order (tw + L).
template <typename T>
void launch_twiddles(cx<T>* tw, int L, cudaStream_t stream);

} // namespace mmb
