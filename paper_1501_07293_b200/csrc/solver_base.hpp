// solver_base.hpp — the polymorphic solver interface behind mmb_ctx, shared error types and
// device-buffer helpers (single-device Solver in solver.cu, slab-sharded solver in shard.cu).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstddef>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/mmb.h"

namespace mmb {

struct numerical_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// NVTX range for the host-side phases (step launches, exchanges, queries): header-only NVTX
// v3, visible to nsys / ncu range filters, no-ops when no tool is attached.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

inline void ck(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) throw std::bad_alloc();
    if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

inline int pow2_at_least(int v) {
    int l = 1;
    while (l < v) l <<= 1;
    return l;
}
inline int ilog2(int v) {
    int r = 0;
    while ((1 << r) < v) ++r;
    return r;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        n = count;
        if (count) ck(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    size_t bytes() const { return n * sizeof(T); }
};

class SolverBase {
public:
    virtual ~SolverBase() = default;
    virtual int precision() const = 0;
    virtual void set_m(const void*, const void*, const void*) = 0;
    virtual void get_m(void*, void*, void*) = 0;
    // stream-ordered host I/O (mmb_set_m_async / mmb_get_m_async); synchronous by default
    virtual void set_m_async(const void* x, const void* y, const void* z) { set_m(x, y, z); }
    virtual void get_m_async(void* x, void* y, void* z) { get_m(x, y, z); }
    virtual void step(long long n) = 0;
    virtual long long step_index() const = 0;
    virtual void average(double* out) = 0;
    virtual double energy() = 0;
    virtual double max_torque() = 0;
    virtual double last_torque_sq() = 0;
    virtual long long run(long long steps, long long cadence, double stop_torque,
                          mmb_record_fn fn, void* user) = 0;
    virtual void synchronize() = 0;
    virtual void effective_field(void*, void*, void*) = 0;
    virtual void demag_field(const void*, const void*, const void*, void*, void*, void*) = 0;
    virtual void tensor_octant(double*) = 0;
    virtual void upload_tensor_octant(const double*) = 0;
    virtual float time_steps(long long n) = 0;
    virtual int profile_step(long long n, float* ms, int maxk, std::string& names) = 0;
    virtual int launches_per_step() const = 0;
    virtual size_t device_bytes() const = 0;
    // global z range whose M this handle's set_m/get_m exchange (the whole grid except for
    // one rank of a NCCL-sharded solver)
    virtual void slab(int& z0, int& nz_local) const = 0;
    // demag path and kernel variants this handle runs (mmb_path_info)
    virtual std::string path_info() const = 0;
};


// Slab-decomposed solvers (shard.cu). `world` ranks over z-slabs; make_sharded owns one rank
// and exchanges over NCCL (nccl_id from mmb_nccl_unique_id on rank 0); make_emulated owns all
// ranks on one device and exchanges by device copies (testing the decomposition).
std::unique_ptr<SolverBase> make_sharded(const mmb_desc& d, const mmb_stage* stages, int nstages,
                                         int rank, int world, const void* nccl_id);
std::unique_ptr<SolverBase> make_emulated(const mmb_desc& d, const mmb_stage* stages, int nstages,
                                          int world);
void nccl_unique_id(void* out128);

} // namespace mmb
