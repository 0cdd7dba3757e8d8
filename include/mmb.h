/* mmb.h — C-ABI of the B200-native LLG step (libmmb.so, paper_1501_07293_b200/).
 *
 * Drop-in boundary for the reference's per-step pipeline. Every entry point mirrors one the
 * reference exposes behind mmsim::SimulationBase (proj/include/mmsim/llg.hpp:56-73) and its
 * C FFI (proj/include/mmsim.h:40-91):
 *
 *   mmb_create          <- make_simulation(spec, backend, precision)   proj/src/llg.cpp:163-168
 *                          (+ Simulation<T> ctor: build_demag_tensor + spectral_prepare,
 *                           proj/src/llg.cpp:22-38) / mmsim_sim_create proj/src/capi.cpp:145-159
 *   mmb_free            <- mmsim_sim_free                               proj/src/capi.cpp:161
 *   mmb_step            <- mmsim_sim_step / Simulation<T>::step         proj/src/capi.cpp:163-172,
 *                                                                       proj/src/llg.cpp:58-108
 *   mmb_step_index      <- mmsim_sim_step_index                         proj/src/capi.cpp:174-181
 *   mmb_average         <- mmsim_sim_average / average_unit             proj/src/capi.cpp:183-195,
 *                                                                       proj/src/llg.cpp:126-131
 *   mmb_energy          <- mmsim_sim_energy / energy                    proj/src/capi.cpp:197-206
 *   mmb_max_torque      <- mmsim_sim_max_torque / max_torque            proj/src/capi.cpp:208-217
 *   mmb_run             <- mmsim_sim_run / Simulation<T>::run           proj/src/capi.cpp:219-239,
 *                                                                       proj/src/llg.cpp:110-124
 *   mmb_set_m/mmb_get_m <- Simulation<T>::magnetization()               proj/include/mmsim/llg.hpp:98-99
 *   mmb_status_string   <- mmsim_status_string                          proj/src/capi.cpp:82-95
 *   mmb_last_error      <- mmsim_last_error (thread-local)              proj/src/capi.cpp:27,97
 *
 * Conventions follow mmsim.h: int status (MMB_OK == 0, same numeric codes as mmsim_status),
 * opaque handle, host arrays borrowed for the duration of the call only, one handle per
 * thread. Fields are SoA host arrays of nx*ny*nz elements each, x fastest
 * (proj/include/mmsim/grid.hpp:42-47), of type float (MMB_F32) or double (MMB_F64).
 * Stepping is asynchronous on the handle's CUDA stream; calls that return data synchronise.
 * A degenerate cell (|M| = 0 during renormalisation) is reported as MMB_ERROR_NUMERICAL by
 * the next synchronising call with the reference's message shape
 * ("renormalize: zero-magnitude magnetization at cell i at step s").
 */
#ifndef MMB_H
#define MMB_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum mmb_status {
    MMB_OK = 0,
    MMB_ERROR_ARGUMENT = 1,
    MMB_ERROR_CONFIG = 2,
    MMB_ERROR_NUMERICAL = 3,
    MMB_ERROR_IO = 4,
    MMB_ERROR_NOMEM = 5,
    MMB_ERROR_VALIDATION = 6,
    MMB_ERROR_INTERNAL = 7,
    MMB_ERROR_CUDA = 8 /* no usable CUDA device / driver failure (no CPU fallback exists) */
};

enum mmb_precision { MMB_F32 = 0, MMB_F64 = 1 };

typedef struct mmb_ctx mmb_ctx;

/* ProblemSpec (proj/include/mmsim/problems.hpp:15-24) flattened: grid, material, dt,
 * initial direction. */
typedef struct mmb_desc {
    int nx, ny, nz;
    double delta;                 /* cell edge, nm (cubic cells, grid.hpp:21-34) */
    double a_ex, ms, hk, alpha;   /* MaterialParams (material.hpp:13-34) */
    double dt;                    /* ns */
    double init_dir[3];           /* uniform initial direction (normalised here) */
    int precision;                /* MMB_F32 / MMB_F64 */
    int device;                   /* CUDA device ordinal */
} mmb_desc;

/* ScheduleStage (proj/include/mmsim/schedule.hpp:14-27). */
typedef struct mmb_stage {
    long long start, end;         /* [start, end) in steps */
    double field[3];
    int ramp;
    double field_end[3];
    int has_alpha;
    double alpha_override;
} mmb_stage;

const char* mmb_status_string(int status);
const char* mmb_last_error(void);
const char* mmb_version(void);
/* Frees strings returned through char** out-parameters (mmsim_string_free,
 * proj/src/capi.cpp:102). */
void mmb_string_free(char* s);

int mmb_create(const mmb_desc* desc, const mmb_stage* stages, int nstages, mmb_ctx** out);
void mmb_free(mmb_ctx* ctx);

int mmb_set_m(mmb_ctx* ctx, const void* mx, const void* my, const void* mz);
int mmb_get_m(mmb_ctx* ctx, void* mx, void* my, void* mz);
/* Stream-ordered variants for pipelined host I/O (no reference counterpart): the copies go
 * through device staging buffers on their own host->device / device->host streams, ordered
 * with the steps enqueued around them, so a loop of set_m_async, mmb_step, get_m_async keeps
 * both PCIe directions and the step in flight together. The host arrays must stay valid and
 * unchanged (set) / untouched (get) until the next mmb_synchronize (or any synchronising
 * call); get_m_async delivers the state at its position in the sequence. Sharded handles run
 * them synchronously. */
int mmb_set_m_async(mmb_ctx* ctx, const void* mx, const void* my, const void* mz);
int mmb_get_m_async(mmb_ctx* ctx, void* mx, void* my, void* mz);

int mmb_step(mmb_ctx* ctx, long long n);
int mmb_step_index(const mmb_ctx* ctx, long long* out);
int mmb_average(mmb_ctx* ctx, double out_mxyz[3]);
int mmb_energy(mmb_ctx* ctx, double* out);
int mmb_max_torque(mmb_ctx* ctx, double* out);
/* max |M x H|^2 of the most recent step (Simulation<T>::last_torque_sq_). */
int mmb_last_torque_sq(mmb_ctx* ctx, double* out);

typedef void (*mmb_record_fn)(void* user, long long step, double mx, double my, double mz);
/* Advances up to `steps` steps; records every `cadence` completed (absolute) steps; stops
 * early when sqrt(last max|MxH|^2)/ms^2 < stop_torque (stop_torque < 0: never). */
int mmb_run(mmb_ctx* ctx, long long steps, long long cadence, double stop_torque,
            mmb_record_fn record, void* user, long long* steps_done);

int mmb_synchronize(mmb_ctx* ctx);

/* ---- parity hooks (tests) ------------------------------------------------------------ */
/* H_eff at the current state and step exactly as assemble_effective_field builds it
 * (proj/src/llg.cpp:46-56; applies the sticky damping override like the reference). */
int mmb_effective_field(mmb_ctx* ctx, void* hx, void* hy, void* hz);
/* Demag field of an arbitrary host M (DemagSolver<T>::compute, proj/src/demag.cpp:53-147). */
int mmb_demag_field(mmb_ctx* ctx, const void* mx, const void* my, const void* mz, void* hx,
                    void* hy, void* hz);
/* Device-computed fp64 prism-sum entries on the non-negative octant, [6][nz][ny][nx] in the
 * order xx, xy, xz, yy, yz, zz (demag_tensor_entry, proj/src/demag_tensor.cpp:9-43). */
int mmb_tensor_octant(mmb_ctx* ctx, double* out);
/* Replace the device tensor with host-supplied octant entries (same layout), e.g. the
 * reference's own fp64 tensor, and rebuild the spectrum. */
int mmb_upload_tensor_octant(mmb_ctx* ctx, const double* entries);

/* Device self-check suite (mmsim_validate / run_validation, proj/src/capi.cpp:286-298,
 * proj/src/validate.cpp:84-189, on the device): tensor invariants from the device prism-sum
 * kernel, the spectral demag path against an O(N^2) device direct sum (up to 16^3), linearity,
 * cube and thin-film shape factors. report_out (optional, free with mmb_string_free) receives
 * one "PASS|FAIL  name: detail" line per check. MMB_ERROR_VALIDATION when any check fails. */
int mmb_validate(char** report_out);

/* ---- measurement ---------------------------------------------------------------------- */
/* Device time (CUDA events on the handle's stream) of n steps, in ms. */
int mmb_time_steps(mmb_ctx* ctx, long long n, float* ms);
/* Number of kernels one step launches, and per-kernel average device time over n eagerly
 * launched steps (names written as a ';'-separated list into names_buf). */
int mmb_profile_step(mmb_ctx* ctx, long long n, float* kernel_ms, int max_kernels, int* count,
                     char* names_buf, size_t names_len);
int mmb_launches_per_step(mmb_ctx* ctx, int* out);
/* Bytes of device memory held by the handle. */
int mmb_device_bytes(mmb_ctx* ctx, size_t* out);
/* The reference's seeded random initial state (random_unit_field, proj/src/validate.cpp:21-39:
 * std::mt19937(seed), std::uniform_real_distribution<double>(-1, 1), draws of norm < 0.1
 * rejected, ms * v / norm computed in double and cast to the precision): cells
 * [first, first + count) of that sequence into SoA host arrays. Host-side utility (no device),
 * used for the synthetic inputs of SURVEY.md §8(d). */
int mmb_random_unit_field(unsigned seed, double ms, long long first, long long count, int precision,
                          void* x, void* y, void* z);
/* The demag path and kernel variants (template parameters, tiles, grids) this handle runs,
 * as one NUL-terminated line (truncated to len - 1 bytes). Diagnostic; no reference
 * counterpart. */
int mmb_path_info(mmb_ctx* ctx, char* buf, size_t len);

/* ---- multi-GPU: z-slab decomposition ------------------------------------
 * One process per GPU. Rank 0 creates an NCCL id with mmb_nccl_unique_id and shares it (e.g.
 * via torch.distributed broadcast); every rank then calls mmb_create_sharded with its rank.
 * The handle owns the z-slab [z0, z0+nz_local) (mmb_slab): set_m/get_m exchange that slab
 * (SoA, nz_local planes); step/run/average/last_torque_sq are collective (all ranks call
 * them in the same order); <m> is the global average. Field hooks (energy, max_torque,
 * effective_field, demag_field, tensor) are single-device only. mmb_create_emulated runs all
 * `world` ranks of the same decomposition on this process's device (exchanges by device
 * copies) and exposes the whole grid — used to test the sharded pipeline on one GPU.
 * With world == 1, mmb_create_sharded returns the single-device solver (nothing to exchange).
 * MMB_SHARD_PEER=1 (environment, read at creation) replaces the NCCL all-to-all transposes by
 * y/z kernels that read and write every rank's slab spectrum in place through CUDA IPC
 * mappings (peer memory over NVLink); see DESIGN.md §6. */
int mmb_nccl_unique_id(unsigned char out[128]);
int mmb_create_sharded(const mmb_desc* desc, const mmb_stage* stages, int nstages, int rank,
                       int world, const unsigned char nccl_id[128], mmb_ctx** out);
int mmb_create_emulated(const mmb_desc* desc, const mmb_stage* stages, int nstages, int world,
                        mmb_ctx** out);
int mmb_slab(mmb_ctx* ctx, int* z0, int* nz_local);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* MMB_H */
