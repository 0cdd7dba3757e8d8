// fast_common.cuh — device helpers shared by the fast-path kernels: kx-major spectrum row
// addressing, Ampere async copies, Hopper/Blackwell TMA bulk copies with mbarriers, packed
// tensor loads and shared-memory twiddle staging.
#pragma once

#include "fft4.cuh"
#include "types.cuh"

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdlib>

namespace mmb {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda), or null
using TmapEncode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline TmapEncode tmap_encoder() {
    static const TmapEncode encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<TmapEncode>(nullptr);
        return reinterpret_cast<TmapEncode>(fn);
    }();
    return encode;
}
// 3-D tile map over 8-byte elements: dims innermost first, byte strides of dims 1 and 2.
// False when the layout breaks TMA's rules (16-byte base and strides) or TMA is unavailable.
inline bool make_tmap_3d(CUtensorMap* tm, const void* base, unsigned long long d0, unsigned long long d1,
                         unsigned long long d2, unsigned long long s1, unsigned long long s2, unsigned b0,
                         unsigned b1, unsigned b2) {
    const TmapEncode encode = tmap_encoder();
    if (!encode || (reinterpret_cast<unsigned long long>(base) & 15u) || (s1 & 15u) || (s2 & 15u) || (b0 * 8u) % 16u)
        return false;
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {s1, s2};
    const cuuint32_t box[3] = {b0, b1, b2};
    const cuuint32_t es[3] = {1u, 1u, 1u};
    return encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
inline bool env_off(const char* name) {
    const char* e = std::getenv(name);
    return e && e[0] == '0';
}

__device__ __forceinline__ long long sf_row(int kx, int c, int z, int nz, int ny) {
    return ((static_cast<long long>(kx) * 3 + c) * nz + z) * ny;
}

// Programmatic dependent launch: let the next kernel in the stream start launching (its CTAs
// take SMs as this grid's last wave drains), and wait for the previous kernel's completion and
// memory before touching its outputs. Both are no-ops for a launch without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

#ifndef MMB_CP16_CA
#define MMB_CP16_CA 0
#endif
// Ampere-style async global->shared copy of one element (LDGSTS), bypassing registers.
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    if constexpr (BYTES == 16 && !MMB_CP16_CA)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(s), "l"(gmem), "n"(BYTES) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// ---- TMA (cp.async.bulk) global -> shared with an mbarrier transaction count
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// TMA tile load of a 3-D box (coordinates innermost first) into shared memory, completing
// on an mbarrier's transaction count
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// two adjacent complex values of a 16-byte aligned pair (one 16-byte vector for f32)
template <typename T>
__device__ __forceinline__ void ld_pair(const cx<T>* p, cx<T>& a, cx<T>& b) {
    if constexpr (sizeof(T) == 4) {
        const float4 f = *reinterpret_cast<const float4*>(p);
        a = cx<T>{f.x, f.y};
        b = cx<T>{f.z, f.w};
    } else {
        a = p[0];
        b = p[1];
    }
}
template <typename T>
__device__ __forceinline__ void st_pair(cx<T>* p, cx<T> a, cx<T> b) {
    if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(a.x, a.y, b.x, b.y);
    } else {
        p[0] = a;
        p[1] = b;
    }
}
// async copy of a 16-byte aligned complex pair
__device__ __forceinline__ void cp_async_ca16(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
// (.ca: allocating in L1 measured 5 % faster on the k_xstep staging than .cg)
template <typename T>
__device__ __forceinline__ void cp_async_pair(cx<T>* smem, const cx<T>* gmem) {
    cp_async_ca16(smem, gmem);
    if constexpr (sizeof(T) == 8) cp_async_ca16(smem + 1, gmem + 1);
}

// six tensor coefficients stored contiguously ([..][6]): three 2-vector loads
template <typename T>
__device__ __forceinline__ void load6(const T* __restrict__ p, T (&k)[6]) {
    const cx<T>* q = reinterpret_cast<const cx<T>*>(p);
    const cx<T> a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
    k[0] = a.x;
    k[1] = a.y;
    k[2] = b.x;
    k[3] = b.y;
    k[4] = c.x;
    k[5] = c.y;
}

// Stage-A twiddles W_L^{n1*k2} staged in shared memory as [k2][n1] (unit stride across the
// n1-consecutive lanes of stage A: bank-conflict free, no global loads on the hot path).
template <typename T, int LOG2L>
__device__ __forceinline__ void stage_twiddles(cx<T>* tws, const cx<T>* __restrict__ tw) {
    // async copies of the table's [k2][n1] copy (tw[L..2L), launch_twiddles): the caller's
    // cp_async_wait_all + barrier completes them
    constexpr int L = 1 << LOG2L;
    constexpr int PER = 16 / static_cast<int>(sizeof(cx<T>));
    const cx<T>* src = tw + L;
    if (L % PER == 0 && (static_cast<unsigned>(__cvta_generic_to_shared(tws)) & 15u) == 0) {
        for (int e = threadIdx.x * PER; e < L; e += blockDim.x * PER) cp_async_ca16(tws + e, src + e);
    } else {
        for (int e = threadIdx.x; e < L; e += blockDim.x) cp_async<sizeof(cx<T>)>(tws + e, src + e);
    }
}


} // namespace mmb
