// shard.cu — z-slab decomposition of the LLG step over several B200s of one box
// (grids too large for one GPU, e.g. 2048x2048x64).
//
// Rank r owns the z-slab [z0, z0+nzl) of M (with one halo plane below and above) and the
// kx column range [k0, k0+ncols) of the half spectrum. One step:
//
//   KX   (prime only)  x-r2c of the slab rows         -> S_loc[kx][c][z_loc][y]   (all Xh kx)
//   A2A  forward       all-to-all transpose          -> S_col[kx_loc][c][z][y]   (all nz z)
//   KYZ / KYF,KZ,KYI   y/z FFTs + tensor MAC on the local kx columns (no communication)
//   A2A  backward                                    -> S_loc
//   HALO               M planes z0-1 and z0+nzl from the neighbour ranks
//   KXS                x-c2r -> local terms + LLG -> x-r2c of M_{t+1} (next step's S_loc)
//
// The chunk rank r sends to rank q in the forward transpose is one contiguous range of S_loc
// (kx in q's columns); it lands in q's S_col as a 2-D strided block (rows (kx, c), each the
// nzl*ny values of r's planes), placed with cudaMemcpy2DAsync. Exchanges go over NCCL
// (grouped ncclSend/ncclRecv, ncclAllReduce for <m>); the emulated variant runs every rank on
// one device with device copies instead, which makes the decomposition testable on one GPU:
// per-rank kernels are the single-device kernels on sub-grids, so the sharded fields equal
// the single-device ones bitwise.
//
// Peer mode (MMB_SHARD_PEER=1): no transposes. The y/z kernels of rank r read the rows of its
// kx columns straight from every rank's S_loc and write the results back there (RowMap: plain
// loads/stores into the peers' memory over NVLink, mapped with CUDA IPC), and the halo planes
// are copied peer to peer. Two stream-ordered barriers (a one-word ncclAllReduce) per step
// separate the phases: every rank's KXS has written its S_loc before anyone's y/z reads it,
// and every y/z write-back has landed before any KXS reads. In emulated mode the same kernels
// run with all S_loc buffers on one device.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fast.hpp"
#include "kernels.hpp"
#include "solver_base.hpp"

namespace mmb {

namespace {

void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw cuda_error(std::string(what) + ": " + ncclGetErrorString(r));
}

std::vector<std::pair<int, int>> split_range(int n, int p) {
    std::vector<std::pair<int, int>> out;
    const int base = n / p, extra = n % p;
    int s = 0;
    for (int r = 0; r < p; ++r) {
        const int e = s + base + (r < extra ? 1 : 0);
        out.emplace_back(s, e);
        s = e;
    }
    return out;
}

Geom make_geom(int nx, int ny, int nz, int lz_force) {
    Geom g{};
    g.nx = nx;
    g.ny = ny;
    g.nz = nz;
    g.lx = nx == 1 ? 1 : pow2_at_least(2 * nx - 1);
    g.ly = ny == 1 ? 1 : pow2_at_least(2 * ny - 1);
    g.lz = lz_force > 0 ? lz_force : (nz == 1 ? 1 : pow2_at_least(2 * nz - 1));
    g.log2lx = ilog2(g.lx);
    g.log2ly = ilog2(g.ly);
    g.log2lz = ilog2(g.lz);
    g.xh = g.lx == 1 ? 1 : g.lx / 2 + 1;
    g.xp = (g.xh + 15) / 16 * 16;
    g.yh = g.ly == 1 ? 1 : g.ly / 2 + 1;
    g.zh = g.lz == 1 ? 1 : g.lz / 2 + 1;
    g.n = static_cast<long long>(nx) * ny * nz;
    g.rows = static_cast<long long>(ny) * nz;
    g.cs = g.n;
    g.nz_g = nz;
    g.z0 = 0;
    return g;
}

template <typename T>
struct Rank {
    int rank = 0, z0 = 0, nzl = 0, k0 = 0, ncols = 0;
    Geom gs{}, gc{};              // slab (x phase) / column (y-z phase) geometry
    long long plane = 0;          // nx*ny
    DevBuf<T> mb[2];              // [3][nzl + 2][ny][nx], halo planes first and last
    DevBuf<cx<T>> s_loc, s_col, s2, stage;
    DevBuf<T> kspec;              // tensor slab of the local kx columns [ncols][zh][yh][6]
    DevBuf<cx<T>> twx, twy, twz;
    DevBuf<StepCtl> ctl;
    DevBuf<double> tpart, partial, red;
    int tpart_count = 0;
    T* m(int which) { return mb[which].p + plane; } // plane 0 of the slab, component 0
};

template <typename T>
class ShardSolver final : public SolverBase {
public:
    ShardSolver(const mmb_desc& d, const mmb_stage* stages, int nstages, int world, int my_rank,
                const void* nccl_id, bool emulated)
        : d_(d), world_(world), emulated_(emulated) {
        if (world < 1) throw std::invalid_argument("mmb: world size must be >= 1");
        if (d.nx < 1 || d.ny < 1 || d.nz < 1) throw std::invalid_argument("Grid: cell counts must be >= 1");
        if (!(d.delta > 0.0)) throw std::invalid_argument("Grid: cell edge length must be > 0");
        if (!(d.ms > 0.0)) throw std::invalid_argument("MaterialParams: ms must be > 0");
        if (d.a_ex < 0.0) throw std::invalid_argument("MaterialParams: a_ex must be >= 0");
        if (d.hk < 0.0) throw std::invalid_argument("MaterialParams: hk must be >= 0");
        if (!(d.alpha > 0.0)) throw std::invalid_argument("MaterialParams: alpha must be > 0");
        if (d.nz < world) throw std::invalid_argument("mmb: z-slab sharding needs nz >= world size");
        set_schedule(stages, nstages);
        ck(cudaSetDevice(d.device), "cudaSetDevice");
        ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");

        // global geometry and path (fused y/z for nz <= 8, streaming y/z otherwise)
        Geom g = make_geom(d.nx, d.ny, d.nz, 0);
        Geom gy = make_geom(d.nx, d.ny, d.nz, (d.nz >= 2 && d.nz <= 8) ? 16 : 0);
        g_ = fast_supported<T>(gy) ? gy : g;
        yz_ = fast_supported<T>(gy);
        if (!yz_ && !big_supported<T>(g_))
            throw std::invalid_argument("mmb: grid not supported by the sharded path");
        // every rank owns at least one kx column (its y/z launch runs the step prologue)
        if (g_.xh < world) throw std::invalid_argument("mmb: z-slab sharding needs Lx/2+1 >= world size");
        slabs_ = split_range(d.nz, world);
        cols_ = split_range(g_.xh, world);
        exch_coeff_ = 2.0 * d.a_ex / (kMu0 * d.ms * d.ms * d.delta * d.delta);
        aniso_coeff_ = d.hk / d.ms;

        // tensor spectrum for all kx once (fast layout [kx][kz][ky][6]), sliced per rank
        DevBuf<T> kfull;
        build_full_tensor(kfull);

        if (emulated_) {
            for (int r = 0; r < world; ++r) ranks_.push_back(make_rank(r, kfull));
        } else {
            ranks_.push_back(make_rank(my_rank, kfull));
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            nck(ncclCommInitRank(&comm_, world, id, my_rank), "ncclCommInitRank");
        }
        const char* pe = std::getenv("MMB_SHARD_PEER");
        peer_ = pe && pe[0] == '1' && world > 1;
        if (peer_) {
            if (world > kMaxRanks) throw std::invalid_argument("mmb: peer mode supports up to 8 ranks");
            setup_peers();
        }
        prepare_fast_kernels<T>(ranks_[0]->gs);
        if (yz_) prepare_fast_kernels<T>(ranks_[0]->gc);
        else prepare_big_kernels<T>(ranks_[0]->gc);

        // uniform initial state (vector_field.hpp:41-52)
        const double norm = std::sqrt(d.init_dir[0] * d.init_dir[0] + d.init_dir[1] * d.init_dir[1] +
                                      d.init_dir[2] * d.init_dir[2]);
        if (!(norm > 0.0)) throw std::invalid_argument("init_uniform: direction vector must be nonzero");
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            std::vector<T> col(static_cast<size_t>(R.nzl) * R.plane);
            for (int c = 0; c < 3; ++c) {
                std::fill(col.begin(), col.end(), static_cast<T>(d.ms * d.init_dir[c] / norm));
                ck(cudaMemcpyAsync(R.m(0) + c * R.gs.cs, col.data(), col.size() * sizeof(T),
                                   cudaMemcpyHostToDevice, stream_), "M upload");
                ck(cudaStreamSynchronize(stream_), "sync");
            }
        }
        ck(cudaStreamSynchronize(stream_), "create sync");
    }

    ~ShardSolver() override {
        if (peer_ && !emulated_) {
            // nobody frees its buffers while a peer may still read them
            try {
                barrier();
                cudaStreamSynchronize(stream_);
            } catch (...) {
            }
            for (void* p : ipc_open_)
                if (p) cudaIpcCloseMemHandle(p);
        }
        if (comm_) ncclCommDestroy(comm_);
        ranks_.clear();
        if (stream_) cudaStreamDestroy(stream_);
    }

    int precision() const override { return sizeof(T) == 8 ? MMB_F64 : MMB_F32; }

    void slab(int& z0, int& nzl) const override {
        if (emulated_) {
            z0 = 0;
            nzl = g_.nz;
        } else {
            z0 = ranks_[0]->z0;
            nzl = ranks_[0]->nzl;
        }
    }

    void set_m(const void* x, const void* y, const void* z) override {
        const void* src[3] = {x, y, z};
        const int zbase = emulated_ ? 0 : ranks_[0]->z0;
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            for (int c = 0; c < 3; ++c)
                ck(cudaMemcpyAsync(R.m(cur_) + c * R.gs.cs,
                                   static_cast<const T*>(src[c]) + (R.z0 - zbase) * R.plane,
                                   R.nzl * R.plane * sizeof(T), cudaMemcpyHostToDevice, stream_), "set_m");
        }
        s_valid_ = false;
        ck(cudaStreamSynchronize(stream_), "set_m sync");
    }

    void get_m(void* x, void* y, void* z) override {
        void* dst[3] = {x, y, z};
        const int zbase = emulated_ ? 0 : ranks_[0]->z0;
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            for (int c = 0; c < 3; ++c)
                ck(cudaMemcpyAsync(static_cast<T*>(dst[c]) + (R.z0 - zbase) * R.plane,
                                   R.m(cur_) + c * R.gs.cs, R.nzl * R.plane * sizeof(T),
                                   cudaMemcpyDeviceToHost, stream_), "get_m");
        }
        sync_and_check();
    }

    void step(long long n) override {
        if (peer_) {
            step_peer(n);
            return;
        }
        for (long long i = 0; i < n; ++i) {
            prime();
            transpose_forward();
            for (auto& rp : ranks_) {
                Rank<T>& R = *rp;
                if (yz_) {
                    launch_fast_yz<T>(R.s_col.p, R.gc, R.twy.p, R.kspec.p, R.ctl.p, st_, 1, stream_);
                } else {
                    launch_big_yf<T>(R.s_col.p, R.s2.p, R.gc, R.twy.p, R.ctl.p, st_, 1, stream_);
                    launch_big_z<T>(R.s2.p, R.gc, R.twz.p, R.kspec.p, stream_);
                    launch_big_yi<T>(R.s2.p, R.s_col.p, R.gc, R.twy.p, stream_);
                }
            }
            transpose_backward();
            halo_exchange(cur_);
            for (auto& rp : ranks_) {
                Rank<T>& R = *rp;
                launch_fast_xstep<T>(R.s_loc.p, R.m(cur_), R.m(cur_ ^ 1), R.gs, R.twx.p, exch_coeff_,
                                     aniso_coeff_, R.ctl.p, R.tpart.p, stream_);
            }
            cur_ ^= 1;
            ++step_;
        }
    }

    long long step_index() const override { return step_; }

    void average(double* out) override {
        double s[3] = {0.0, 0.0, 0.0};
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            launch_sum3<T>(R.m(cur_), R.nzl * R.plane, R.gs.cs, R.partial.p, R.red.p, stream_);
        }
        if (!emulated_) {
            Rank<T>& R = *ranks_[0];
            nck(ncclAllReduce(R.red.p, R.red.p, 3, ncclDouble, ncclSum, comm_, stream_), "ncclAllReduce");
            ck(cudaMemcpyAsync(s, R.red.p, sizeof(s), cudaMemcpyDeviceToHost, stream_), "average");
            sync_and_check();
        } else {
            for (auto& rp : ranks_) {
                double t[3];
                ck(cudaMemcpyAsync(t, rp->red.p, sizeof(t), cudaMemcpyDeviceToHost, stream_), "average");
                ck(cudaStreamSynchronize(stream_), "average sync");
                for (int c = 0; c < 3; ++c) s[c] += t[c];
            }
            sync_and_check();
        }
        const double inv = 1.0 / static_cast<double>(g_.n);
        const double inv_ms = 1.0 / d_.ms;
        for (int c = 0; c < 3; ++c) out[c] = (inv * s[c]) * inv_ms;
    }

    double last_torque_sq() override {
        double best = 0.0;
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            launch_torque_partials(R.tpart.p, R.tpart_count, R.ctl.p, stream_);
            StepCtl c;
            ck(cudaMemcpyAsync(&c, R.ctl.p, sizeof(c), cudaMemcpyDeviceToHost, stream_), "ctl");
            ck(cudaStreamSynchronize(stream_), "ctl sync");
            double v;
            std::memcpy(&v, &c.torque_sq_bits, sizeof(v));
            best = std::max(best, v);
        }
        if (!emulated_) {
            // max over ranks
            Rank<T>& R = *ranks_[0];
            ck(cudaMemcpyAsync(R.red.p, &best, sizeof(best), cudaMemcpyHostToDevice, stream_), "torque");
            nck(ncclAllReduce(R.red.p, R.red.p, 1, ncclDouble, ncclMax, comm_, stream_), "ncclAllReduce");
            ck(cudaMemcpyAsync(&best, R.red.p, sizeof(best), cudaMemcpyDeviceToHost, stream_), "torque");
            ck(cudaStreamSynchronize(stream_), "torque sync");
        }
        return best;
    }

    long long run(long long steps, long long cadence, double stop_torque, mmb_record_fn fn,
                  void* user) override {
        const double ms2 = d_.ms * d_.ms;
        long long done = 0;
        const bool stop = stop_torque >= 0.0;
        while (done < steps) {
            long long chunk = steps - done;
            if (fn && cadence > 0) chunk = std::min(chunk, cadence - (step_ % cadence));
            if (stop) chunk = 1;
            step(chunk);
            done += chunk;
            if (fn && cadence > 0 && step_ % cadence == 0) {
                double a[3];
                average(a);
                fn(user, step_, a[0], a[1], a[2]);
            }
            if (stop && std::sqrt(last_torque_sq()) / ms2 < stop_torque) break;
        }
        sync_and_check();
        return done;
    }

    void synchronize() override { sync_and_check(); }

    float time_steps(long long n) override {
        cudaEvent_t a, b;
        ck(cudaEventCreate(&a), "event");
        ck(cudaEventCreate(&b), "event");
        prime();
        ck(cudaEventRecord(a, stream_), "record");
        step(n);
        ck(cudaEventRecord(b, stream_), "record");
        ck(cudaEventSynchronize(b), "event sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        check_numerical();
        return ms;
    }

    int profile_step(long long n, float* out, int maxk, std::string& names) override {
        const float ms = time_steps(n);
        if (maxk > 0) out[0] = ms / static_cast<float>(std::max<long long>(1, n));
        names = "sharded_step";
        return 1;
    }

    int launches_per_step() const override {
        return static_cast<int>(ranks_.size()) * (yz_ ? 2 : 4);
    }

    std::string path_info() const override {
        char head[200];
        const Rank<T>& R = *ranks_[0];
        std::snprintf(head, sizeof head, "path=sharded-%s world=%d mode=%s%s n=%dx%dx%d L=%dx%dx%d prec=%s slab=%d+%d cols=%d+%d",
                      yz_ ? "yz" : "big", world_, emulated_ ? "emulated" : "nccl", peer_ ? "+peer" : "", d_.nx, d_.ny,
                      d_.nz, g_.lx, g_.ly, g_.lz, sizeof(T) == 8 ? "f64" : "f32", R.z0, R.nzl, R.k0, R.ncols);
        std::string s = head;
        s += "; " + (yz_ ? fast_describe<T>(R.gc) : big_describe<T>(R.gc));
        const std::string x = fast_describe<T>(R.gs);
        s += "; slab " + x.substr(x.find("k_xstep"));
        return s;
    }

    size_t device_bytes() const override {
        size_t b = 0;
        for (auto& rp : ranks_) {
            const Rank<T>& R = *rp;
            b += R.mb[0].bytes() + R.mb[1].bytes() + R.s_loc.bytes() + R.s_col.bytes() + R.s2.bytes() +
                 R.stage.bytes() + R.kspec.bytes() + R.twx.bytes() + R.twy.bytes() + R.twz.bytes() +
                 R.ctl.bytes() + R.tpart.bytes() + R.partial.bytes() + R.red.bytes();
        }
        return b;
    }

    // field hooks are single-device features
    double energy() override { throw std::invalid_argument("mmb: energy() is not available on a sharded handle"); }
    double max_torque() override { throw std::invalid_argument("mmb: max_torque() is not available on a sharded handle"); }
    void effective_field(void*, void*, void*) override {
        throw std::invalid_argument("mmb: effective_field() is not available on a sharded handle");
    }
    void demag_field(const void*, const void*, const void*, void*, void*, void*) override {
        throw std::invalid_argument("mmb: demag_field() is not available on a sharded handle");
    }
    void tensor_octant(double*) override {
        throw std::invalid_argument("mmb: tensor_octant() is not available on a sharded handle");
    }
    void upload_tensor_octant(const double*) override {
        throw std::invalid_argument("mmb: upload_tensor_octant() is not available on a sharded handle");
    }

private:
    // ---- peer mode -------------------------------------------------------------------------
    void step_peer(long long n) {
        for (long long i = 0; i < n; ++i) {
            prime();
            barrier(); // every rank's S_loc (KXS / prime output) is complete
            for (size_t k = 0; k < ranks_.size(); ++k) {
                Rank<T>& R = *ranks_[k];
                const RowMap<T>& rm = rowmaps_[k];
                if (R.ncols == 0) continue;
                if (yz_) {
                    launch_fast_yz<T>(R.s_loc.p, R.gc, R.twy.p, R.kspec.p, R.ctl.p, st_, 1, stream_, false, &rm);
                } else {
                    launch_big_yf<T>(R.s_loc.p, R.s2.p, R.gc, R.twy.p, R.ctl.p, st_, 1, stream_, &rm);
                    launch_big_z<T>(R.s2.p, R.gc, R.twz.p, R.kspec.p, stream_);
                    launch_big_yi<T>(R.s2.p, R.s_loc.p, R.gc, R.twy.p, stream_, &rm);
                }
            }
            barrier(); // every y/z write-back into the S_loc buffers has landed
            halo_peer(cur_);
            for (auto& rp : ranks_) {
                Rank<T>& R = *rp;
                launch_fast_xstep<T>(R.s_loc.p, R.m(cur_), R.m(cur_ ^ 1), R.gs, R.twx.p, exch_coeff_,
                                     aniso_coeff_, R.ctl.p, R.tpart.p, stream_);
            }
            cur_ ^= 1;
            ++step_;
        }
    }

    // stream-ordered barrier across ranks (nothing to do when all ranks share one stream)
    void barrier() {
        if (emulated_) return;
        nck(ncclAllReduce(bar_.p, bar_.p, 1, ncclInt32, ncclSum, comm_, stream_), "ncclAllReduce (barrier)");
    }

    // S_loc and M base pointers of every rank: local buffers in emulated mode, CUDA IPC
    // mappings of the peers' allocations otherwise (handles all-gathered over NCCL)
    void setup_peers() {
        s_loc_of_.assign(world_, nullptr);
        m_of_[0].assign(world_, nullptr);
        m_of_[1].assign(world_, nullptr);
        if (emulated_) {
            for (auto& rp : ranks_) {
                s_loc_of_[rp->rank] = rp->s_loc.p;
                m_of_[0][rp->rank] = rp->mb[0].p;
                m_of_[1][rp->rank] = rp->mb[1].p;
            }
        } else {
            Rank<T>& R = *ranks_[0];
            bar_.alloc(1);
            ck(cudaMemsetAsync(bar_.p, 0, sizeof(int), stream_), "memset");
            constexpr int H = sizeof(cudaIpcMemHandle_t);
            std::vector<unsigned char> mine(3 * H), all(static_cast<size_t>(3) * H * world_);
            void* ptrs[3] = {R.s_loc.p, R.mb[0].p, R.mb[1].p};
            for (int i = 0; i < 3; ++i) {
                cudaIpcMemHandle_t h;
                ck(cudaIpcGetMemHandle(&h, ptrs[i]), "cudaIpcGetMemHandle");
                std::memcpy(mine.data() + i * H, &h, H);
            }
            DevBuf<unsigned char> dall;
            dall.alloc(all.size());
            ck(cudaMemcpyAsync(dall.p + static_cast<size_t>(R.rank) * 3 * H, mine.data(), 3 * H, cudaMemcpyHostToDevice,
                               stream_), "ipc handles");
            nck(ncclAllGather(dall.p + static_cast<size_t>(R.rank) * 3 * H, dall.p, 3 * H, ncclUint8, comm_, stream_),
                "ncclAllGather");
            ck(cudaMemcpyAsync(all.data(), dall.p, all.size(), cudaMemcpyDeviceToHost, stream_), "ipc handles");
            ck(cudaStreamSynchronize(stream_), "ipc sync");
            for (int q = 0; q < world_; ++q) {
                void* p[3] = {ptrs[0], ptrs[1], ptrs[2]};
                if (q != R.rank) {
                    for (int i = 0; i < 3; ++i) {
                        cudaIpcMemHandle_t h;
                        std::memcpy(&h, all.data() + (static_cast<size_t>(q) * 3 + i) * H, H);
                        ck(cudaIpcOpenMemHandle(&p[i], h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
                        ipc_open_.push_back(p[i]);
                    }
                }
                s_loc_of_[q] = static_cast<cx<T>*>(p[0]);
                m_of_[0][q] = static_cast<T*>(p[1]);
                m_of_[1][q] = static_cast<T*>(p[2]);
            }
        }
        for (auto& rp : ranks_) {
            RowMap<T> rm{};
            rm.world = world_;
            rm.k0 = rp->k0;
            for (int q = 0; q < world_; ++q) {
                rm.base[q] = s_loc_of_[q];
                rm.z0[q] = slabs_[q].first;
            }
            rm.z0[world_] = d_.nz;
            rowmaps_.push_back(rm);
        }
    }

    // halo planes of M_cur copied from the neighbours' slabs (peer to peer)
    void halo_peer(int which) {
        const size_t plane = static_cast<size_t>(d_.nx) * d_.ny, pb = plane * sizeof(T);
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            for (int c = 0; c < 3; ++c) {
                T* mc = R.m(which) + c * R.gs.cs;
                if (R.rank > 0) {
                    const int q = R.rank - 1, nq = slabs_[q].second - slabs_[q].first;
                    const T* src = m_of_[which][q] + plane + c * (nq + 2) * plane + (nq - 1) * plane;
                    ck(cudaMemcpyAsync(mc - plane, src, pb, cudaMemcpyDefault, stream_), "halo (peer)");
                }
                if (R.rank + 1 < world_) {
                    const int q = R.rank + 1, nq = slabs_[q].second - slabs_[q].first;
                    const T* src = m_of_[which][q] + plane + c * (nq + 2) * plane;
                    ck(cudaMemcpyAsync(mc + R.nzl * plane, src, pb, cudaMemcpyDefault, stream_), "halo (peer)");
                }
            }
        }
    }

    void set_schedule(const mmb_stage* stages, int n) {
        if (n < 0 || (n > 0 && !stages)) throw std::invalid_argument("mmb: bad stage list");
        if (n > kMaxStages) throw std::invalid_argument("mmb: too many schedule stages (max 16)");
        std::vector<mmb_stage> s(stages, stages + n);
        std::stable_sort(s.begin(), s.end(), [](const mmb_stage& a, const mmb_stage& b) { return a.start < b.start; });
        for (size_t i = 0; i < s.size(); ++i) {
            if (s[i].end <= s[i].start) throw std::invalid_argument("FieldSchedule: stage range must be nonempty");
            if (i > 0 && s[i].start < s[i - 1].end)
                throw std::invalid_argument("FieldSchedule: stage ranges must be disjoint");
        }
        std::memset(&st_, 0, sizeof(st_));
        st_.n = n;
        for (int i = 0; i < n; ++i) {
            st_.start[i] = s[i].start;
            st_.end[i] = s[i].end;
            st_.ramp[i] = s[i].ramp;
            st_.has_alpha[i] = s[i].has_alpha;
            st_.alpha[i] = s[i].alpha_override;
            for (int c = 0; c < 3; ++c) {
                st_.field[i][c] = s[i].field[c];
                st_.field_end[i][c] = s[i].field_end[c];
            }
        }
    }

    void build_full_tensor(DevBuf<T>& out) {
        const Geom& g = g_;
        const long long c0 = g.n;
        const long long c1 = static_cast<long long>(g.xh) * g.ny * g.nz;
        const long long c2 = static_cast<long long>(g.xh) * g.yh * g.nz;
        const long long c3 = static_cast<long long>(g.xh) * g.yh * g.zh;
        DevBuf<double2> csx, csy, csz;
        csx.alloc(g.lx);
        csy.alloc(g.ly);
        csz.alloc(g.lz);
        launch_cs_table(csx.p, g.lx, stream_);
        launch_cs_table(csy.p, g.ly, stream_);
        launch_cs_table(csz.p, g.lz, stream_);
        DevBuf<double> a3;
        {
            DevBuf<double> E, a1, a2;
            E.alloc(6 * static_cast<size_t>(c0));
            launch_tensor_octant(E.p, g.nx, g.ny, g.nz, d_.delta, stream_);
            a1.alloc(6 * c1);
            launch_axis_transform(E.p, a1.p, g.nx, g.ny, g.nz, 0, g.lx, csx.p, 0x06, c0, c1, stream_);
            a2.alloc(6 * c2);
            launch_axis_transform(a1.p, a2.p, g.xh, g.ny, g.nz, 1, g.ly, csy.p, 0x12, c1, c2, stream_);
            a3.alloc(6 * c3);
            launch_axis_transform(a2.p, a3.p, g.xh, g.yh, g.nz, 2, g.lz, csz.p, 0x14, c2, c3, stream_);
            ck(cudaStreamSynchronize(stream_), "tensor sync");
        }
        out.alloc(6 * c3);
        launch_tensor_finalize_fast<T>(a3.p, out.p, g.xh, g.yh, g.zh,
                                       1.0 / (static_cast<double>(g.lx) * g.ly * g.lz), stream_);
        ck(cudaStreamSynchronize(stream_), "tensor sync");
    }

    std::unique_ptr<Rank<T>> make_rank(int r, const DevBuf<T>& kfull) {
        auto R = std::make_unique<Rank<T>>();
        R->rank = r;
        R->z0 = slabs_[r].first;
        R->nzl = slabs_[r].second - slabs_[r].first;
        R->k0 = cols_[r].first;
        R->ncols = cols_[r].second - cols_[r].first;
        R->plane = static_cast<long long>(d_.nx) * d_.ny;
        // slab geometry: local planes for rows/S, global planes for the Neumann mask
        R->gs = g_;
        R->gs.nz = R->nzl;
        R->gs.n = R->nzl * R->plane;
        R->gs.rows = static_cast<long long>(d_.ny) * R->nzl;
        R->gs.cs = (R->nzl + 2) * R->plane;
        R->gs.nz_g = d_.nz;
        R->gs.z0 = R->z0;
        // column geometry: local kx columns, all planes
        R->gc = g_;
        R->gc.xh = R->ncols;
        const size_t plane = static_cast<size_t>(R->plane);
        R->mb[0].alloc(3 * (R->nzl + 2) * plane);
        R->mb[1].alloc(3 * (R->nzl + 2) * plane);
        R->s_loc.alloc(static_cast<size_t>(g_.xh) * 3 * R->nzl * d_.ny);
        R->s_col.alloc(static_cast<size_t>(std::max(R->ncols, 1)) * 3 * d_.nz * d_.ny);
        if (!yz_) R->s2.alloc(static_cast<size_t>(std::max(R->ncols, 1)) * 3 * d_.nz * g_.ly);
        if (!emulated_) R->stage.alloc(std::max(R->s_loc.n, R->s_col.n));
        const size_t per_kx = static_cast<size_t>(g_.zh) * g_.yh * 6;
        R->kspec.alloc(std::max(R->ncols, 1) * per_kx);
        if (R->ncols > 0)
            ck(cudaMemcpyAsync(R->kspec.p, kfull.p + R->k0 * per_kx, R->ncols * per_kx * sizeof(T),
                               cudaMemcpyDeviceToDevice, stream_), "tensor slice");
        R->twx.alloc(2 * g_.lx);
        R->twy.alloc(2 * g_.ly);
        R->twz.alloc(2 * g_.lz);
        launch_twiddles<T>(R->twx.p, g_.lx, stream_);
        launch_twiddles<T>(R->twy.p, g_.ly, stream_);
        launch_twiddles<T>(R->twz.p, g_.lz, stream_);
        R->ctl.alloc(1);
        StepCtl c{};
        c.alpha = d_.alpha;
        c.dt = d_.dt;
        c.ms = d_.ms;
        c.bad_key = ~0ull;
        ck(cudaMemcpyAsync(R->ctl.p, &c, sizeof(c), cudaMemcpyHostToDevice, stream_), "ctl upload");
        R->tpart_count = fast_xstep_blocks<T>(R->gs);
        R->tpart.alloc(R->tpart_count);
        ck(cudaMemsetAsync(R->tpart.p, 0, R->tpart.bytes(), stream_), "memset");
        R->partial.alloc(3 * 1024);
        R->red.alloc(8);
        // zero the halo planes once (never read at the global ends: Neumann mask)
        ck(cudaMemsetAsync(R->mb[0].p, 0, R->mb[0].bytes(), stream_), "memset");
        ck(cudaMemsetAsync(R->mb[1].p, 0, R->mb[1].bytes(), stream_), "memset");
        ck(cudaStreamSynchronize(stream_), "rank sync");
        return R;
    }

    void prime() {
        if (s_valid_) return;
        for (auto& rp : ranks_)
            launch_fast_xf<T>(rp->m(cur_), rp->s_loc.p, rp->gs, rp->twx.p, rp->ctl.p, st_, 0, stream_);
        s_valid_ = true;
    }

    // element offsets and counts of the transposes (complex elements)
    long long loc_chunk_off(int nzl_r, int q) const { return static_cast<long long>(cols_[q].first) * 3 * nzl_r * d_.ny; }
    long long loc_chunk_cnt(int nzl_r, int q) const {
        return static_cast<long long>(cols_[q].second - cols_[q].first) * 3 * nzl_r * d_.ny;
    }

    void copy2d(cx<T>* dst, size_t dpitch, const cx<T>* src, size_t spitch, size_t width, size_t height) {
        if (width == 0 || height == 0) return;
        ck(cudaMemcpy2DAsync(dst, dpitch * sizeof(cx<T>), src, spitch * sizeof(cx<T>), width * sizeof(cx<T>),
                             height, cudaMemcpyDeviceToDevice, stream_), "cudaMemcpy2DAsync");
    }

    // S_loc (all kx, local planes) -> S_col (local kx, all planes)
    void transpose_forward() {
        const size_t ny = d_.ny, nz = d_.nz;
        if (emulated_) {
            for (auto& rp : ranks_)
                for (auto& qp : ranks_) {
                    Rank<T>& R = *rp;
                    Rank<T>& Q = *qp;
                    // R's planes for Q's columns -> Q.s_col rows (kx, c), plane offset R.z0
                    copy2d(Q.s_col.p + R.z0 * ny, nz * ny, R.s_loc.p + loc_chunk_off(R.nzl, Q.rank),
                           R.nzl * ny, R.nzl * ny, static_cast<size_t>(Q.ncols) * 3);
                }
            return;
        }
        Rank<T>& R = *ranks_[0];
        // receive every peer's chunk contiguously into `stage`, then place it
        std::vector<long long> roff(world_);
        long long off = 0;
        for (int q = 0; q < world_; ++q) {
            roff[q] = off;
            off += static_cast<long long>(R.ncols) * 3 * (slabs_[q].second - slabs_[q].first) * d_.ny;
        }
        nck(ncclGroupStart(), "ncclGroupStart");
        for (int q = 0; q < world_; ++q) {
            if (q == R.rank) continue;
            const long long sc = loc_chunk_cnt(R.nzl, q);
            if (sc) nck(ncclSend(R.s_loc.p + loc_chunk_off(R.nzl, q), 2 * sc * sizeof(T), ncclInt8, q, comm_, stream_), "ncclSend");
            const long long rc = static_cast<long long>(R.ncols) * 3 * (slabs_[q].second - slabs_[q].first) * d_.ny;
            if (rc) nck(ncclRecv(R.stage.p + roff[q], 2 * rc * sizeof(T), ncclInt8, q, comm_, stream_), "ncclRecv");
        }
        nck(ncclGroupEnd(), "ncclGroupEnd");
        for (int q = 0; q < world_; ++q) {
            const int zq = slabs_[q].first, nq = slabs_[q].second - slabs_[q].first;
            const cx<T>* src = (q == R.rank) ? R.s_loc.p + loc_chunk_off(R.nzl, q) : R.stage.p + roff[q];
            copy2d(R.s_col.p + zq * ny, nz * ny, src, nq * ny, nq * ny, static_cast<size_t>(R.ncols) * 3);
        }
    }

    // S_col -> S_loc
    void transpose_backward() {
        const size_t ny = d_.ny, nz = d_.nz;
        if (emulated_) {
            for (auto& rp : ranks_)
                for (auto& qp : ranks_) {
                    Rank<T>& R = *rp; // holds columns
                    Rank<T>& Q = *qp; // receives its planes of R's columns
                    copy2d(Q.s_loc.p + loc_chunk_off(Q.nzl, R.rank), Q.nzl * ny, R.s_col.p + Q.z0 * ny, nz * ny,
                           Q.nzl * ny, static_cast<size_t>(R.ncols) * 3);
                }
            return;
        }
        Rank<T>& R = *ranks_[0];
        // pack each peer's planes of my columns contiguously, then exchange
        std::vector<long long> soff(world_);
        long long off = 0;
        for (int q = 0; q < world_; ++q) {
            const int zq = slabs_[q].first, nq = slabs_[q].second - slabs_[q].first;
            soff[q] = off;
            if (q != R.rank)
                copy2d(R.stage.p + off, nq * ny, R.s_col.p + zq * ny, nz * ny, nq * ny, static_cast<size_t>(R.ncols) * 3);
            else
                copy2d(R.s_loc.p + loc_chunk_off(R.nzl, R.rank), R.nzl * ny, R.s_col.p + zq * ny, nz * ny,
                       R.nzl * ny, static_cast<size_t>(R.ncols) * 3);
            off += static_cast<long long>(R.ncols) * 3 * nq * d_.ny;
        }
        nck(ncclGroupStart(), "ncclGroupStart");
        for (int q = 0; q < world_; ++q) {
            if (q == R.rank) continue;
            const int nq = slabs_[q].second - slabs_[q].first;
            const long long sc = static_cast<long long>(R.ncols) * 3 * nq * d_.ny;
            if (sc) nck(ncclSend(R.stage.p + soff[q], 2 * sc * sizeof(T), ncclInt8, q, comm_, stream_), "ncclSend");
            const long long rc = loc_chunk_cnt(R.nzl, q);
            if (rc) nck(ncclRecv(R.s_loc.p + loc_chunk_off(R.nzl, q), 2 * rc * sizeof(T), ncclInt8, q, comm_, stream_),
                        "ncclRecv");
        }
        nck(ncclGroupEnd(), "ncclGroupEnd");
    }

    // halo planes of M_cur from the neighbouring slabs
    void halo_exchange(int which) {
        if (world_ == 1) return;
        const size_t pb = static_cast<size_t>(d_.nx) * d_.ny * sizeof(T);
        if (emulated_) {
            for (size_t r = 0; r < ranks_.size(); ++r) {
                Rank<T>& R = *ranks_[r];
                for (int c = 0; c < 3; ++c) {
                    T* mc = R.m(which) + c * R.gs.cs;
                    if (r > 0) {
                        Rank<T>& L = *ranks_[r - 1];
                        ck(cudaMemcpyAsync(mc - R.plane, L.m(which) + c * L.gs.cs + (L.nzl - 1) * L.plane, pb,
                                           cudaMemcpyDeviceToDevice, stream_), "halo");
                    }
                    if (r + 1 < ranks_.size()) {
                        Rank<T>& U = *ranks_[r + 1];
                        ck(cudaMemcpyAsync(mc + R.nzl * R.plane, U.m(which) + c * U.gs.cs, pb,
                                           cudaMemcpyDeviceToDevice, stream_), "halo");
                    }
                }
            }
            return;
        }
        Rank<T>& R = *ranks_[0];
        nck(ncclGroupStart(), "ncclGroupStart");
        for (int c = 0; c < 3; ++c) {
            T* mc = R.m(which) + c * R.gs.cs;
            if (R.rank > 0) {
                nck(ncclSend(mc, pb, ncclInt8, R.rank - 1, comm_, stream_), "ncclSend");
                nck(ncclRecv(mc - R.plane, pb, ncclInt8, R.rank - 1, comm_, stream_), "ncclRecv");
            }
            if (R.rank + 1 < world_) {
                nck(ncclSend(mc + (R.nzl - 1) * R.plane, pb, ncclInt8, R.rank + 1, comm_, stream_), "ncclSend");
                nck(ncclRecv(mc + R.nzl * R.plane, pb, ncclInt8, R.rank + 1, comm_, stream_), "ncclRecv");
            }
        }
        nck(ncclGroupEnd(), "ncclGroupEnd");
    }

    // The first zero-|M| cell over all ranks (keys are (step << 36) | global cell, so the
    // minimum is the reference's smallest cell of the earliest failing step). With NCCL the
    // keys are min-all-reduced first: every rank raises the same error at the same call, and
    // none is left waiting in a collective its failed peer never joins.
    void check_numerical() {
        unsigned long long key = ~0ull;
        for (auto& rp : ranks_) {
            unsigned long long k;
            if (!emulated_) {
                unsigned long long* red = reinterpret_cast<unsigned long long*>(rp->red.p + 7);
                ck(cudaMemcpyAsync(red, &rp->ctl.p->bad_key, sizeof(k), cudaMemcpyDeviceToDevice, stream_), "ctl");
                nck(ncclAllReduce(red, red, 1, ncclUint64, ncclMin, comm_, stream_), "ncclAllReduce (error word)");
                ck(cudaMemcpyAsync(&k, red, sizeof(k), cudaMemcpyDeviceToHost, stream_), "ctl");
            } else {
                ck(cudaMemcpyAsync(&k, &rp->ctl.p->bad_key, sizeof(k), cudaMemcpyDeviceToHost, stream_), "ctl");
            }
            ck(cudaStreamSynchronize(stream_), "ctl sync");
            key = std::min(key, k);
        }
        if (key == ~0ull) return;
        const long long cell = static_cast<long long>(key & ((1ull << 36) - 1));
        const long long st = static_cast<long long>(key >> 36);
        // as Solver::check_numerical: the step index returns to the failing step
        step_ = st;
        for (auto& rp : ranks_) {
            StepCtl c;
            ck(cudaMemcpyAsync(&c, rp->ctl.p, sizeof(c), cudaMemcpyDeviceToHost, stream_), "ctl");
            ck(cudaStreamSynchronize(stream_), "ctl sync");
            c.bad_key = ~0ull;
            c.step = c.cur_step = st;
            ck(cudaMemcpyAsync(rp->ctl.p, &c, sizeof(c), cudaMemcpyHostToDevice, stream_), "reset");
            ck(cudaStreamSynchronize(stream_), "reset sync");
        }
        s_valid_ = false;
        throw numerical_error("renormalize: zero-magnitude magnetization at cell " + std::to_string(cell) +
                              " at step " + std::to_string(st));
    }

    void sync_and_check() {
        ck(cudaStreamSynchronize(stream_), "sync");
        check_numerical();
    }

    mmb_desc d_;
    int world_;
    bool emulated_;
    Geom g_{};
    bool yz_ = false;
    StageTable st_{};
    std::vector<std::pair<int, int>> slabs_, cols_;
    std::vector<std::unique_ptr<Rank<T>>> ranks_;
    cudaStream_t stream_ = nullptr;
    ncclComm_t comm_ = nullptr;
    bool peer_ = false;
    std::vector<RowMap<T>> rowmaps_;        // per local rank (peer mode)
    std::vector<cx<T>*> s_loc_of_;          // every rank's S_loc (peer mode)
    std::vector<T*> m_of_[2];               // every rank's M buffers, halo planes included
    std::vector<void*> ipc_open_;
    DevBuf<int> bar_;
    int cur_ = 0;
    bool s_valid_ = false;
    long long step_ = 0;
    double exch_coeff_ = 0.0, aniso_coeff_ = 0.0;
};

} // namespace

std::unique_ptr<SolverBase> make_sharded(const mmb_desc& d, const mmb_stage* stages, int nstages,
                                         int rank, int world, const void* nccl_id) {
    if (rank < 0 || rank >= world || !nccl_id) throw std::invalid_argument("mmb: bad rank / world / NCCL id");
    if (d.precision == MMB_F64) return std::make_unique<ShardSolver<double>>(d, stages, nstages, world, rank, nccl_id, false);
    return std::make_unique<ShardSolver<float>>(d, stages, nstages, world, rank, nccl_id, false);
}

std::unique_ptr<SolverBase> make_emulated(const mmb_desc& d, const mmb_stage* stages, int nstages,
                                          int world) {
    if (d.precision == MMB_F64) return std::make_unique<ShardSolver<double>>(d, stages, nstages, world, 0, nullptr, true);
    return std::make_unique<ShardSolver<float>>(d, stages, nstages, world, 0, nullptr, true);
}

void nccl_unique_id(void* out128) {
    ncclUniqueId id;
    nck(ncclGetUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof(id));
}

} // namespace mmb
