// types.cuh — device-side control block and geometry shared by the kernels and the host plan.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace mmb {

constexpr int kMaxStages = 16;
constexpr double kGammaMu0 = 0.221; // proj/include/mmsim/material.hpp:11
constexpr double kMu0 = 1.256636;   // proj/include/mmsim/material.hpp:10

// Applied-field program (proj/include/mmsim/schedule.hpp:14-48), sorted and disjoint.
struct StageTable {
    int n;
    long long start[kMaxStages];
    long long end[kMaxStages];
    double field[kMaxStages][3];
    int ramp[kMaxStages];
    double field_end[kMaxStages][3];
    int has_alpha[kMaxStages];
    double alpha[kMaxStages];
};

// Per-simulation device control block. `step` is the reference's step_ (completed steps);
// the prologue of each step evaluates the schedule at `step` exactly as
// Simulation<T>::assemble_effective_field does (proj/src/llg.cpp:46-56), including the
// sticky damping override, and publishes p1/p2/field for the fused LLG kernel.
struct StepCtl {
    long long step;        // completed steps (reference step_)
    long long cur_step;    // step being assembled (published by the prologue)
    double alpha;          // current (sticky) damping
    double dt, ms;
    double p1, p2;         // IntegratorParams prefactors for cur_step
    double field[3];       // applied field at cur_step
    unsigned long long torque_sq_bits; // max |M x H|^2 of the last step (fp64 bits, >= 0)
    unsigned long long bad_key;        // (step << 36) | cell of the first zero-|M| cell, ~0 if none
};

// Geometry of the pruned padded convolution. All lengths are powers of two with
// L >= 2n - 1 (L = 1 when n = 1); Xh = Lx/2 + 1 half-spectrum columns (1 when Lx = 1).
// Spectrum scratch S is [3][nz][Ly][Xp] complex (kx fastest, ky in DIF storage order).
struct Geom {
    int nx, ny, nz;
    int lx, ly, lz;             // padded lengths
    int log2lx, log2ly, log2lz;
    int xh, xp;                 // half-spectrum length, row pitch (complex)
    int yh, zh;                 // tensor octant extents (Ly/2+1, Lz/2+1)
    long long n;                // nx*ny*nz
    long long rows;             // ny*nz (real rows per component)
    // M/H buffer addressing (slab decomposition): component stride of the M buffers in
    // elements, the global plane count and this slab's first global plane. A single-device
    // solver has cs = n, nz_g = nz, z0 = 0.
    long long cs;
    int nz_g, z0;
};

__host__ __device__ inline long long s_index(const Geom& g, int c, int z, int ky, int kx) {
    return ((static_cast<long long>(c) * g.nz + z) * g.ly + ky) * g.xp + kx;
}

// Runtime DIF storage position -> true frequency (same digit plan as common.cuh).
__device__ __forceinline__ int freq_of_pos_rt(int p, int log2l) {
    int k = 0, shift = 0, s = log2l;
    const int np = num_passes(log2l);
    for (int q = 0; q < np; ++q) {
        const int lr = pass_log2r(log2l, q);
        s -= lr;
        k += ((p >> s) & ((1 << lr) - 1)) << shift;
        shift += lr;
    }
    return k;
}

// Six tensor-spectrum coefficients (xx, xy, xz, yy, yz, zz) at true frequency (kx, ky, kz),
// reconstructed from the stored real octant by the per-axis parities of the wrapped
// kernel: xy odd in (x, y), xz odd in (x, z), yz odd in (y, z); diagonals even.
template <typename T>
struct TensorSpec {
    const T* __restrict__ k; // [6][zh][yh][xh]
    long long cs;            // component stride
    __device__ __forceinline__ void at(const Geom& g, int kx, int ky, int kz, T (&o)[6]) const {
        bool fy = false, fz = false;
        if (2 * ky > g.ly) { ky = g.ly - ky; fy = true; }
        if (2 * kz > g.lz) { kz = g.lz - kz; fz = true; }
        const long long idx = (static_cast<long long>(kz) * g.yh + ky) * g.xh + kx;
        o[0] = __ldg(k + idx);
        o[1] = __ldg(k + cs + idx);
        o[2] = __ldg(k + 2 * cs + idx);
        o[3] = __ldg(k + 3 * cs + idx);
        o[4] = __ldg(k + 4 * cs + idx);
        o[5] = __ldg(k + 5 * cs + idx);
        if (fy) o[1] = -o[1];
        if (fz) o[2] = -o[2];
        if (fy != fz) o[4] = -o[4];
    }
};

// H^ = K M^ with the symmetric real tensor (rows {xx,xy,xz},{xy,yy,yz},{xz,yz,zz},
// proj/src/demag.cpp:94-98).
// packed registers: 9 FMUL2/FFMA2 instead of 18
__device__ __forceinline__ void mac3(const float (&k)[6], pf2& a, pf2& b, pf2& c) {
    const float2 mx = a, my = b, mz = c;
    const auto bc = [](float v) { return make_float2(v, v); };
    a = fma2(bc(k[2]), mz, fma2(bc(k[1]), my, mul2(bc(k[0]), mx)));
    b = fma2(bc(k[4]), mz, fma2(bc(k[3]), my, mul2(bc(k[1]), mx)));
    c = fma2(bc(k[5]), mz, fma2(bc(k[4]), my, mul2(bc(k[2]), mx)));
}
template <typename T>
__device__ __forceinline__ void mac3(const T (&k)[6], cx<T>& a, cx<T>& b, cx<T>& c) {
    const cx<T> mx = a, my = b, mz = c;
    a = {k[0] * mx.x + k[1] * my.x + k[2] * mz.x, k[0] * mx.y + k[1] * my.y + k[2] * mz.y};
    b = {k[1] * mx.x + k[3] * my.x + k[4] * mz.x, k[1] * mx.y + k[3] * my.y + k[4] * mz.y};
    c = {k[2] * mx.x + k[4] * my.x + k[5] * mz.x, k[2] * mx.y + k[4] * my.y + k[5] * mz.y};
}

// Step prologue (one thread): schedule lookup at ctl->step, sticky alpha update,
// prefactors (proj/include/mmsim/llg.hpp:24-30), torque reset.
// mode 1: stepping (alpha update + torque reset), 2: H_eff assembly (alpha update, as
// max_torque() does, llg.cpp:141), 3: applied field only (energy(), llg.cpp:134).
__device__ __forceinline__ void step_prologue(StepCtl* ctl, const StageTable& st, int mode) {
    const long long s = ctl->step;
    double f[3] = {0.0, 0.0, 0.0};
    bool has_alpha = false;
    double alpha = 0.0;
    for (int i = 0; i < st.n; ++i) {
        if (s < st.start[i]) break;
        if (s < st.end[i]) {
            if (!st.ramp[i]) {
                f[0] = st.field[i][0];
                f[1] = st.field[i][1];
                f[2] = st.field[i][2];
            } else {
                const double fr = static_cast<double>(s - st.start[i]) /
                                  static_cast<double>(st.end[i] - st.start[i]);
                for (int c = 0; c < 3; ++c)
                    f[c] = __dadd_rn(st.field[i][c], __dmul_rn(fr, st.field_end[i][c] - st.field[i][c]));
            }
            has_alpha = st.has_alpha[i] != 0;
            alpha = st.alpha[i];
            break;
        }
    }
    if (mode != 3 && has_alpha && alpha != ctl->alpha) ctl->alpha = alpha;
    const double a = ctl->alpha;
    // explicit _rn intrinsics: no FMA contraction, so the prefactors round exactly like the
    // reference's separate multiply/add (x86-64 SSE2, no FMA)
    const double p1 = __dmul_rn(-kGammaMu0, ctl->dt) / __dadd_rn(1.0, __dmul_rn(a, a));
    ctl->p1 = p1;
    ctl->p2 = __dmul_rn(p1, a) / ctl->ms;
    ctl->field[0] = f[0];
    ctl->field[1] = f[1];
    ctl->field[2] = f[2];
    ctl->cur_step = s;
    if (mode == 1) ctl->torque_sq_bits = 0ull;
}

} // namespace mmb
