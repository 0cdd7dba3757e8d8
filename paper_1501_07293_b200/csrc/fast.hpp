// fast.hpp — launchers of the fast demag path (fast_kernels.cu). Supported when
// fast_supported<T>(g): 2 <= Lx, Ly <= 4096 (2048 for f64), nz == 1 or (2 <= nz <= 8 with
// Lz = 16, f32), and one kx block of the spectrum fits in shared memory.
// Spectrum scratch layout: S[kx][c][z][y], y fastest, ny rows; tensor: [kx][kz][ky][c].
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "types.cuh"

namespace mmb {

// Rows of the y/z stage gathered from per-rank spectrum blocks instead of one contiguous column
// buffer (slab sharding, shard.cu): row (kx, c, z) of a launch (kx counted from the launch's
// first column) lives in block q = owner(z) at
//   base[q][((kb[q] + kx) * 3 + c) * nzl_q + z - z0[q]]   (rows of ny values).
// A block is a rank's own slab spectrum S_loc[kx][c][z_loc][y] (kb = that rank's global first
// column of the launch) or the receive buffer an all-to-all filled with one peer's planes of
// this rank's columns (kb = the launch's first local column). `local`: every block is in this
// GPU's memory (whole rows are then staged with TMA bulk copies); otherwise base[q] may be
// another GPU's memory (CUDA IPC peer mapping, NVLink loads/stores) and rows are plain loads.
// world == 0: rows are the contiguous local column buffer.
constexpr int kMaxRanks = 8;
template <typename T>
struct RowMap {
    cx<T>* base[kMaxRanks];
    int kb[kMaxRanks];
    int z0[kMaxRanks + 1]; // slab starts, z0[world] = nz
    int world = 0;
    int local = 0;
    __device__ __forceinline__ cx<T>* row(int kx, int c, int z, int ny) const {
        int q = 0;
        while (z >= z0[q + 1]) ++q;
        const long long nzl = z0[q + 1] - z0[q];
        return base[q] + ((static_cast<long long>(kb[q] + kx) * 3 + c) * nzl + (z - z0[q])) * ny;
    }
};

template <typename T> bool fast_supported(const Geom& g);
// the kernel variants (template parameters, tiles, grids) the geometry selects
template <typename T> std::string fast_describe(const Geom& g);
template <typename T> std::string big_describe(const Geom& g);
template <typename T> int fast_yz_kxb(const Geom& g, int* smem_bytes);
template <typename T> void prepare_fast_kernels(const Geom& g);
template <typename T>
void launch_fast_xf(const T* m, cx<T>* S, const Geom& g, const cx<T>* tw, StepCtl* ctl,
                    const StageTable& st, int prologue, cudaStream_t stream);
// KYZ; block 0 optionally runs the step prologue (schedule, sticky alpha, prefactors).
template <typename T>
void launch_fast_yz(cx<T>* S, const Geom& g, const cx<T>* tw, const T* kt, StepCtl* ctl,
                    const StageTable& st, int prologue, cudaStream_t stream, bool pdl = false,
                    const RowMap<T>* rows = nullptr);
// KXS: fused x-c2r -> local terms + LLG update (M -> mout) -> x-r2c of mout, S in place.
// Writes one torque partial per CTA (fast_xstep_blocks of them) to tpart.
template <typename T>
void launch_fast_xstep(cx<T>* S, const T* m, T* mout, const Geom& g, const cx<T>* tw,
                       double exch_coeff, double aniso_coeff, StepCtl* ctl, double* tpart,
                       cudaStream_t stream, bool pdl = false);
template <typename T> int fast_xstep_blocks(const Geom& g);
template <typename T>
void launch_fast_xi(const cx<T>* S, T* h, const Geom& g, const cx<T>* tw, cudaStream_t stream);
// Tensor spectrum [6][zh][yh][xh] (fp64) -> fast layout [xh][zh][yh][6] in T, with the
// off-diagonal sign and the 1/P scale (see launch_tensor_finalize).
template <typename T>
void launch_tensor_finalize_fast(const double* spec, T* out, int xh, int yh, int zh, double scale,
                                 cudaStream_t stream);

// ---- nz > 8 (or blocks too large for shared memory): y and z as streaming kernels around a
// padded spectrum S2[kx][c][z][Ly] (big_kernels.cu).
template <typename T> bool big_supported(const Geom& g);
template <typename T> void prepare_big_kernels(const Geom& g);
template <typename T>
void launch_big_yf(const cx<T>* S, cx<T>* S2, const Geom& g, const cx<T>* tw, StepCtl* ctl,
                   const StageTable& st, int prologue, cudaStream_t stream, const RowMap<T>* rows = nullptr);
template <typename T>
void launch_big_z(cx<T>* S2, const Geom& g, const cx<T>* tw, const T* kt, cudaStream_t stream);
template <typename T>
void launch_big_yi(const cx<T>* S2, cx<T>* S, const Geom& g, const cx<T>* tw, cudaStream_t stream,
                   const RowMap<T>* rows = nullptr);

} // namespace mmb
