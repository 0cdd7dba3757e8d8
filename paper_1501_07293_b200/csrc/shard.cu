// shard.cu — z-slab decomposition of the LLG step over several B200s of one box
// (grids too large for one GPU, e.g. 2048x2048x64).
//
// Rank r owns the z-slab [z0, z0+nzl) of M (with one halo plane below and above) and the
// kx column range [k0, k0+ncols) of the half spectrum. One step:
//
//   KX   (prime only)  x-r2c of the slab rows            -> S_loc[kx][c][z_loc][y]  (all Xh kx)
//   HALO               M planes z0-1 and z0+nzl from the neighbours          (comm stream)
//   per column chunk j (the rank's columns split into NCH chunks):
//     A2A forward  (j) rank q's planes of my chunk-j columns -> recv[q]       (comm stream)
//     KYZ / KYF,KZ,KYI (j) on the chunk: rows gathered through a RowMap from the receive
//                  buffers and from my own S_loc, results written back in place (main stream)
//     A2A backward (j) the results back to their owners' S_loc                (comm stream)
//   KXS                x-c2r -> local terms + LLG -> x-r2c of M_{t+1} (next step's S_loc)
//
// Chunk j+1's all-to-all runs while chunk j's y/z kernels compute, and chunk j's results go
// back while chunk j+1 computes (two streams, events between them). There are no pack or
// placement copies: a rank sends contiguous ranges of its S_loc, receives each peer's planes
// into one contiguous block per peer, and the y/z kernels read and write those blocks in place
// through the RowMap (fast.hpp); its own planes never leave S_loc.
//
// Exchanges go through a Transport: grouped ncclSend/ncclRecv between processes (one rank per
// GPU), or, with every rank in one process on one device (the emulated solver that makes the
// decomposition testable on one GPU), device copies that pair the k-th send from a to b with
// the k-th receive posted at b from a. Both run the same posting code, so the emulated tests
// cover the offsets, counts and buffer placement of the NCCL path. The per-rank kernels are
// the single-device kernels on sub-grids, so the sharded fields equal the single-device ones
// bitwise.
//
// Peer mode (MMB_SHARD_PEER=1): no all-to-all. The y/z kernels of rank r read the rows of its
// kx columns straight from every rank's S_loc and write the results back there (RowMap over
// the peers' memory, mapped with CUDA IPC: plain loads/stores over NVLink), and the halo
// planes are copied peer to peer. Two stream-ordered barriers (a one-word ncclAllReduce) per
// step separate the phases.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
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

// ---- point-to-point exchange of one group -------------------------------------------------
class Transport {
public:
    virtual ~Transport() = default;
    virtual void begin(cudaStream_t s) = 0;
    virtual void send(int from, int to, const void* buf, size_t bytes) = 0;
    virtual void recv(int at, int from, void* buf, size_t bytes) = 0;
    virtual void end() = 0;
};

// One rank per process: grouped NCCL point-to-point operations on the group's stream.
class NcclTransport final : public Transport {
public:
    explicit NcclTransport(ncclComm_t c) : comm_(c) {}
    void begin(cudaStream_t s) override {
        s_ = s;
        nck(ncclGroupStart(), "ncclGroupStart");
    }
    void send(int, int to, const void* buf, size_t bytes) override {
        if (bytes) nck(ncclSend(buf, bytes, ncclInt8, to, comm_, s_), "ncclSend");
    }
    void recv(int, int from, void* buf, size_t bytes) override {
        if (bytes) nck(ncclRecv(buf, bytes, ncclInt8, from, comm_, s_), "ncclRecv");
    }
    void end() override { nck(ncclGroupEnd(), "ncclGroupEnd"); }

private:
    ncclComm_t comm_;
    cudaStream_t s_ = nullptr;
};

// Every rank in this process (emulated): at the end of the group the k-th send from a to b
// is copied into the k-th receive posted at b from a, on the group's stream.
class LoopbackTransport final : public Transport {
public:
    void begin(cudaStream_t s) override {
        s_ = s;
        sends_.clear();
        recvs_.clear();
    }
    void send(int from, int to, const void* buf, size_t bytes) override {
        if (bytes) sends_[{from, to}].push_back({const_cast<void*>(buf), bytes});
    }
    void recv(int at, int from, void* buf, size_t bytes) override {
        if (bytes) recvs_[{from, at}].push_back({buf, bytes});
    }
    void end() override {
        if (sends_.size() != recvs_.size()) throw std::logic_error("loopback transport: unmatched peers");
        for (auto& [key, ss] : sends_) {
            auto it = recvs_.find(key);
            if (it == recvs_.end() || it->second.size() != ss.size())
                throw std::logic_error("loopback transport: unmatched send/recv");
            for (size_t i = 0; i < ss.size(); ++i) {
                if (ss[i].second != it->second[i].second) throw std::logic_error("loopback transport: size mismatch");
                ck(cudaMemcpyAsync(it->second[i].first, ss[i].first, ss[i].second, cudaMemcpyDeviceToDevice, s_),
                   "loopback copy");
            }
        }
    }

private:
    cudaStream_t s_ = nullptr;
    std::map<std::pair<int, int>, std::vector<std::pair<void*, size_t>>> sends_, recvs_;
};

template <typename T>
struct Rank {
    int rank = 0, z0 = 0, nzl = 0, k0 = 0, ncols = 0;
    Geom gs{}, gc{};              // slab (x phase) / column (y-z phase) geometry
    long long plane = 0;          // nx*ny
    DevBuf<T> mb[2];              // [3][nzl + 2][ny][nx], halo planes first and last
    DevBuf<T> hb;                 // H (field hooks), same layout as mb
    DevBuf<cx<T>> s_loc, recv, s2;
    std::vector<long long> roff;  // recv: start of peer q's block [ncols][3][nzl_q][ny]
    DevBuf<T> kspec;              // tensor slab of the local kx columns [ncols][zh][yh][6]
    DevBuf<cx<T>> twx, twy, twz;
    DevBuf<StepCtl> ctl;
    DevBuf<double> tpart, partial, red;
    int tpart_count = 0;
    T* m(int which) { return mb[which].p + plane; } // plane 0 of the slab, component 0
    T* h() { return hb.p + plane; }
};

template <typename T>
class ShardSolver final : public SolverBase {
public:
    ShardSolver(const mmb_desc& d, const mmb_stage* stages, int nstages, int world, int my_rank,
                const void* nccl_id, bool emulated)
        : d_(d), world_(world), emulated_(emulated) {
        if (world < 1) throw std::invalid_argument("mmb: world size must be >= 1");
        if (world > kMaxRanks) throw std::invalid_argument("mmb: z-slab sharding supports up to 8 ranks");
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
        ck(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "cudaStreamCreate");

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
        // column chunks of the overlapped exchange (MMB_SHARD_CHUNKS, default 4; 1 = no overlap)
        nch_ = 4;
        if (const char* e = std::getenv("MMB_SHARD_CHUNKS"); e && std::atoi(e) > 0) nch_ = std::atoi(e);
        if (world == 1) nch_ = 1;
        for (int q = 0; q < world; ++q) {
            const int nc = cols_[q].second - cols_[q].first;
            chunks_.push_back(split_range(nc, std::min(nch_, nc)));
            chunks_.back().resize(nch_, {nc, nc}); // ranks with fewer columns than chunks: empty tail
        }
        exch_coeff_ = 2.0 * d.a_ex / (kMu0 * d.ms * d.ms * d.delta * d.delta);
        aniso_coeff_ = d.hk / d.ms;
        const char* pe = std::getenv("MMB_SHARD_PEER");
        peer_ = pe && pe[0] == '1' && world > 1;

        // the prism-sum octant once; each rank's tensor spectrum only for its columns
        {
            DevBuf<double> E;
            build_octant(E);
            if (emulated_) {
                for (int r = 0; r < world; ++r) ranks_.push_back(make_rank(r, E));
            } else {
                ranks_.push_back(make_rank(my_rank, E));
            }
        }
        if (emulated_) {
            transport_ = std::make_unique<LoopbackTransport>();
        } else {
            ncclUniqueId id;
            std::memcpy(&id, nccl_id, sizeof(id));
            nck(ncclCommInitRank(&comm_, world, id, my_rank), "ncclCommInitRank");
            transport_ = std::make_unique<NcclTransport>(comm_);
        }
        if (peer_) setup_peers();
        for (int i = 0; i < 2 * nch_ + 2; ++i) {
            cudaEvent_t e;
            ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
            events_.push_back(e);
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
        if (comm_stream_) cudaStreamSynchronize(comm_stream_);
        if (stream_) cudaStreamSynchronize(stream_);
        for (auto e : events_) cudaEventDestroy(e);
        if (comm_) ncclCommDestroy(comm_);
        ranks_.clear();
        if (comm_stream_) cudaStreamDestroy(comm_stream_);
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
        upload([&](Rank<T>& R) { return R.m(cur_); }, x, y, z, "set_m");
        s_valid_ = false;
    }

    void get_m(void* x, void* y, void* z) override {
        download([&](Rank<T>& R) { return R.m(cur_); }, x, y, z, "get_m");
    }

    void step(long long n) override {
        NvtxRange r("mmb::sharded_step");
        for (long long i = 0; i < n; ++i) {
            prime();
            if (peer_) exchange_and_yz_peer(1, true);
            else exchange_and_yz(1, true);
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
        reduce_over_ranks(s, 3, ncclSum);
        sync_and_check();
        const double inv = 1.0 / static_cast<double>(g_.n);
        const double inv_ms = 1.0 / d_.ms;
        for (int c = 0; c < 3; ++c) out[c] = (inv * s[c]) * inv_ms;
    }

    double last_torque_sq() override {
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            launch_torque_partials(R.tpart.p, R.tpart_count, R.ctl.p, stream_);
            ck(cudaMemcpyAsync(R.red.p, &R.ctl.p->torque_sq_bits, sizeof(double), cudaMemcpyDeviceToDevice, stream_),
               "torque");
        }
        double best = 0.0;
        reduce_over_ranks(&best, 1, ncclMax);
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
        launch_spin(200000ull, stream_); // the host enqueues the timed steps meanwhile
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
        // per local rank: the y/z kernels of each non-empty column chunk (one launch per rank
        // in peer mode), and the x step
        int k = 0;
        for (auto& rp : ranks_) {
            if (peer_) {
                k += yz_ ? 1 : 3;
                continue;
            }
            for (int j = 0; j < nch_; ++j)
                if (chunks_[rp->rank][j].second > chunks_[rp->rank][j].first) k += yz_ ? 1 : 3;
        }
        return k + static_cast<int>(ranks_.size());
    }

    std::string path_info() const override {
        char head[240];
        const Rank<T>& R = *ranks_[0];
        std::snprintf(head, sizeof head,
                      "path=sharded-%s world=%d mode=%s n=%dx%dx%d L=%dx%dx%d prec=%s slab=%d+%d cols=%d+%d chunks=%d",
                      yz_ ? "yz" : "big", world_,
                      emulated_ ? (peer_ ? "emulated+peer" : "emulated") : (peer_ ? "nccl+peer" : "nccl"), d_.nx,
                      d_.ny, d_.nz, g_.lx, g_.ly, g_.lz, sizeof(T) == 8 ? "f64" : "f32", R.z0, R.nzl, R.k0, R.ncols,
                      peer_ ? 1 : nch_);
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
            b += R.mb[0].bytes() + R.mb[1].bytes() + R.hb.bytes() + R.s_loc.bytes() + R.recv.bytes() +
                 R.s2.bytes() + R.kspec.bytes() + R.twx.bytes() + R.twy.bytes() + R.twz.bytes() + R.ctl.bytes() +
                 R.tpart.bytes() + R.partial.bytes() + R.red.bytes();
        }
        return b;
    }

    // ---- field hooks on the slabs (collective over the ranks) --------------------------------
    // Simulation<T>::energy (llg.cpp:133-138): applied field at step_ (no alpha update), demag
    // recomputed, total_energy (energy.cpp:39-64): local densities and exchange bonds summed
    // per slab (the +z bonds of a slab's last plane read its halo), then over the ranks.
    double energy() override {
        demag_slabs(nullptr, 3, true);
        const double ms = d_.ms, ku = 0.5 * d_.hk * kMu0 * ms;
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            launch_energy<T>(R.m(cur_), R.h(), R.gs, ku / (ms * ms), R.ctl.p, R.partial.p, R.red.p, stream_);
        }
        double e[2] = {0.0, 0.0};
        reduce_over_ranks(e, 2, ncclSum);
        sync_and_check();
        return e[0] * (d_.delta * d_.delta * d_.delta) + d_.a_ex * d_.delta / (ms * ms) * e[1];
    }

    // llg.cpp:140-156: re-assemble H_eff (may apply the sticky alpha override), then the fp64
    // max of |M x H| over all cells (max over the ranks).
    double max_torque() override {
        heff_slabs();
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            launch_torque_max<T>(R.m(cur_), R.h(), R.nzl * R.plane, R.gs.cs,
                                 reinterpret_cast<unsigned long long*>(R.red.p), stream_);
        }
        double sq = 0.0;
        reduce_over_ranks(&sq, 1, ncclMax);
        sync_and_check();
        return std::sqrt(sq) / (d_.ms * d_.ms);
    }

    void effective_field(void* x, void* y, void* z) override {
        heff_slabs();
        download([&](Rank<T>& R) { return R.h(); }, x, y, z, "effective_field");
    }

    void demag_field(const void* mx, const void* my, const void* mz, void* hx, void* hy, void* hz) override {
        upload([&](Rank<T>& R) { ensure_h(R); return R.h(); }, mx, my, mz, "demag upload");
        demag_slabs([&](Rank<T>& R) { return R.h(); }, 0, false);
        download([&](Rank<T>& R) { return R.h(); }, hx, hy, hz, "demag_field");
    }

    void tensor_octant(double*) override {
        throw std::invalid_argument("mmb: tensor_octant() is not available on a sharded handle");
    }
    void upload_tensor_octant(const double*) override {
        throw std::invalid_argument("mmb: upload_tensor_octant() is not available on a sharded handle");
    }

private:
    // ---- host <-> slab copies (the handle's planes: one rank's slab, or all in emulated mode)
    template <typename F>
    void upload(F dst_of, const void* x, const void* y, const void* z, const char* what) {
        const void* src[3] = {x, y, z};
        const int zbase = emulated_ ? 0 : ranks_[0]->z0;
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            T* dst = dst_of(R);
            for (int c = 0; c < 3; ++c)
                ck(cudaMemcpyAsync(dst + c * R.gs.cs, static_cast<const T*>(src[c]) + (R.z0 - zbase) * R.plane,
                                   R.nzl * R.plane * sizeof(T), cudaMemcpyHostToDevice, stream_), what);
        }
        ck(cudaStreamSynchronize(stream_), what);
    }
    template <typename F>
    void download(F src_of, void* x, void* y, void* z, const char* what) {
        void* dst[3] = {x, y, z};
        const int zbase = emulated_ ? 0 : ranks_[0]->z0;
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            const T* src = src_of(R);
            for (int c = 0; c < 3; ++c)
                ck(cudaMemcpyAsync(static_cast<T*>(dst[c]) + (R.z0 - zbase) * R.plane, src + c * R.gs.cs,
                                   R.nzl * R.plane * sizeof(T), cudaMemcpyDeviceToHost, stream_), what);
        }
        sync_and_check();
    }

    // v[0..k) of every local rank's red buffer, then over the ranks (NCCL all-reduce on the
    // main stream, or in rank order on the host for the emulated ranks)
    void reduce_over_ranks(double* v, int k, ncclRedOp_t op) {
        for (int i = 0; i < k; ++i) v[i] = 0.0;
        if (!emulated_) {
            Rank<T>& R = *ranks_[0];
            nck(ncclAllReduce(R.red.p, R.red.p, k, ncclDouble, op, comm_, stream_), "ncclAllReduce");
            ck(cudaMemcpyAsync(v, R.red.p, k * sizeof(double), cudaMemcpyDeviceToHost, stream_), "reduce");
            ck(cudaStreamSynchronize(stream_), "reduce sync");
            return;
        }
        for (auto& rp : ranks_) {
            double t[8];
            ck(cudaMemcpyAsync(t, rp->red.p, k * sizeof(double), cudaMemcpyDeviceToHost, stream_), "reduce");
            ck(cudaStreamSynchronize(stream_), "reduce sync");
            for (int i = 0; i < k; ++i) v[i] = op == ncclMax ? std::max(v[i], t[i]) : v[i] + t[i];
        }
    }

    void ensure_h(Rank<T>& R) {
        if (!R.hb.p) {
            R.hb.alloc(R.mb[0].n);
            ck(cudaMemsetAsync(R.hb.p, 0, R.hb.bytes(), stream_), "memset");
        }
    }

    // H_demag of M (m_of(R) per rank, or M_cur with nullptr) into every rank's H slab;
    // prologue 2 / 3 as in Solver::enqueue_demag. `halo`: also refresh M_cur's halo planes
    // (the local terms and the energy's bonds read them).
    template <typename F>
    void demag_slabs(F m_of, int prologue, bool halo) {
        for (auto& rp : ranks_) ensure_h(*rp);
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            const T* m = nullptr;
            if constexpr (std::is_same_v<F, std::nullptr_t>) m = R.m(cur_);
            else m = m_of(R);
            launch_fast_xf<T>(m, R.s_loc.p, R.gs, R.twx.p, R.ctl.p, st_, 0, stream_);
        }
        if (peer_) exchange_and_yz_peer(prologue, halo);
        else exchange_and_yz(prologue, halo);
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            launch_fast_xi<T>(R.s_loc.p, R.h(), R.gs, R.twx.p, stream_);
        }
        s_valid_ = false; // S_loc held another spectrum
    }

    void heff_slabs() {
        demag_slabs(nullptr, 2, true);
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            // in place: each thread reads its own H_demag cell before writing H_eff there
            launch_llg<T>(1, R.m(cur_), R.h(), R.h(), R.gs, exch_coeff_, aniso_coeff_, R.ctl.p, R.tpart.p, stream_);
        }
    }

    // ---- the all-to-all step phase -----------------------------------------------------------
    cudaEvent_t ev(int i) { return events_[i]; }

    // Halo planes, then per column chunk: forward exchange, y/z kernels, backward exchange.
    // Exchanges on the comm stream, kernels on the main stream; returns with the main stream
    // ordered after the last backward exchange.
    void exchange_and_yz(int prologue, bool halo) {
        cudaEvent_t ready = ev(2 * nch_), done = ev(2 * nch_ + 1);
        ck(cudaEventRecord(ready, stream_), "record");
        ck(cudaStreamWaitEvent(comm_stream_, ready, 0), "wait");
        if (halo) halo_exchange(cur_, comm_stream_);
        for (int j = 0; j < nch_; ++j) {
            exchange_chunk(j, false);
            ck(cudaEventRecord(ev(j), comm_stream_), "record");
        }
        for (int j = 0; j < nch_; ++j) {
            ck(cudaStreamWaitEvent(stream_, ev(j), 0), "wait");
            for (auto& rp : ranks_) yz_chunk(*rp, j, j == 0 ? prologue : 0);
            ck(cudaEventRecord(ev(nch_ + j), stream_), "record");
        }
        for (int j = 0; j < nch_; ++j) {
            ck(cudaStreamWaitEvent(comm_stream_, ev(nch_ + j), 0), "wait");
            exchange_chunk(j, true);
        }
        ck(cudaEventRecord(done, comm_stream_), "record");
        ck(cudaStreamWaitEvent(stream_, done, 0), "wait");
    }

    // Chunk j of the all-to-all. Forward: every rank sends each peer q the contiguous S_loc
    // range of q's chunk-j columns (its planes of them) and receives each peer's planes of its
    // own chunk-j columns into that peer's receive block. Backward: the reverse.
    void exchange_chunk(int j, bool backward) {
        NvtxRange r(backward ? "mmb::a2a_backward" : "mmb::a2a_forward");
        const long long ny = d_.ny;
        transport_->begin(comm_stream_);
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            const int a = chunks_[R.rank][j].first, b = chunks_[R.rank][j].second;
            for (int q = 0; q < world_; ++q) {
                if (q == R.rank) continue;
                const int nq = slabs_[q].second - slabs_[q].first;
                // my S_loc range of q's chunk-j columns
                const int qa = chunks_[q][j].first, qb = chunks_[q][j].second;
                cx<T>* mine = R.s_loc.p + (cols_[q].first + qa) * 3 * R.nzl * ny;
                const size_t mine_bytes = static_cast<size_t>(qb - qa) * 3 * R.nzl * ny * sizeof(cx<T>);
                // q's planes of my chunk-j columns, in q's receive block
                cx<T>* theirs = R.recv.p + R.roff[q] + static_cast<long long>(a) * 3 * nq * ny;
                const size_t theirs_bytes = static_cast<size_t>(b - a) * 3 * nq * ny * sizeof(cx<T>);
                if (!backward) {
                    transport_->send(R.rank, q, mine, mine_bytes);
                    transport_->recv(R.rank, q, theirs, theirs_bytes);
                } else {
                    transport_->send(R.rank, q, theirs, theirs_bytes);
                    transport_->recv(R.rank, q, mine, mine_bytes);
                }
            }
        }
        transport_->end();
    }

    // rows of rank R's chunk-j columns: its own planes in S_loc, each peer's in its receive block
    RowMap<T> chunk_rows(Rank<T>& R, int j) {
        RowMap<T> rm{};
        const int a = chunks_[R.rank][j].first;
        rm.world = world_;
        rm.local = 1;
        for (int q = 0; q < world_; ++q) {
            rm.z0[q] = slabs_[q].first;
            if (q == R.rank) {
                rm.base[q] = R.s_loc.p;
                rm.kb[q] = R.k0 + a;
            } else {
                rm.base[q] = R.recv.p + R.roff[q];
                rm.kb[q] = a;
            }
        }
        rm.z0[world_] = d_.nz;
        return rm;
    }

    void yz_chunk(Rank<T>& R, int j, int prologue) {
        const int a = chunks_[R.rank][j].first, b = chunks_[R.rank][j].second;
        if (b <= a) return;
        Geom gc = R.gc;
        gc.xh = b - a;
        const RowMap<T> rm = chunk_rows(R, j);
        const size_t per_kx = static_cast<size_t>(g_.zh) * g_.yh * 6;
        const T* kt = R.kspec.p + a * per_kx;
        if (yz_) {
            launch_fast_yz<T>(R.s_loc.p, gc, R.twy.p, kt, R.ctl.p, st_, prologue, stream_, false, &rm);
        } else {
            cx<T>* s2 = R.s2.p + static_cast<size_t>(a) * 3 * d_.nz * g_.ly;
            launch_big_yf<T>(R.s_loc.p, s2, gc, R.twy.p, R.ctl.p, st_, prologue, stream_, &rm);
            launch_big_z<T>(s2, gc, R.twz.p, kt, stream_);
            launch_big_yi<T>(s2, R.s_loc.p, gc, R.twy.p, stream_, &rm);
        }
    }

    // halo planes of M (buffer `which`) from the neighbouring slabs
    void halo_exchange(int which, cudaStream_t s) {
        if (world_ == 1) return;
        if (peer_) {
            halo_peer(which, s);
            return;
        }
        const size_t pb = static_cast<size_t>(d_.nx) * d_.ny * sizeof(T);
        transport_->begin(s);
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            for (int c = 0; c < 3; ++c) {
                T* mc = R.m(which) + c * R.gs.cs;
                if (R.rank > 0) {
                    transport_->send(R.rank, R.rank - 1, mc, pb);
                    transport_->recv(R.rank, R.rank - 1, mc - R.plane, pb);
                }
                if (R.rank + 1 < world_) {
                    transport_->send(R.rank, R.rank + 1, mc + (R.nzl - 1) * R.plane, pb);
                    transport_->recv(R.rank, R.rank + 1, mc + R.nzl * R.plane, pb);
                }
            }
        }
        transport_->end();
    }

    // ---- peer mode -------------------------------------------------------------------------
    void exchange_and_yz_peer(int prologue, bool halo) {
        barrier(); // every rank's S_loc (KXS / prime output) is complete
        for (size_t k = 0; k < ranks_.size(); ++k) {
            Rank<T>& R = *ranks_[k];
            const RowMap<T>& rm = rowmaps_[k];
            if (yz_) {
                launch_fast_yz<T>(R.s_loc.p, R.gc, R.twy.p, R.kspec.p, R.ctl.p, st_, prologue, stream_, false, &rm);
            } else {
                launch_big_yf<T>(R.s_loc.p, R.s2.p, R.gc, R.twy.p, R.ctl.p, st_, prologue, stream_, &rm);
                launch_big_z<T>(R.s2.p, R.gc, R.twz.p, R.kspec.p, stream_);
                launch_big_yi<T>(R.s2.p, R.s_loc.p, R.gc, R.twy.p, stream_, &rm);
            }
        }
        barrier(); // every y/z write-back into the S_loc buffers has landed
        if (halo) halo_peer(cur_, stream_);
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
            rm.local = emulated_ ? 1 : 0;
            for (int q = 0; q < world_; ++q) {
                rm.base[q] = s_loc_of_[q];
                rm.kb[q] = rp->k0;
                rm.z0[q] = slabs_[q].first;
            }
            rm.z0[world_] = d_.nz;
            rowmaps_.push_back(rm);
        }
    }

    // halo planes of M copied from the neighbours' slabs (peer to peer)
    void halo_peer(int which, cudaStream_t s) {
        const size_t plane = static_cast<size_t>(d_.nx) * d_.ny, pb = plane * sizeof(T);
        for (auto& rp : ranks_) {
            Rank<T>& R = *rp;
            for (int c = 0; c < 3; ++c) {
                T* mc = R.m(which) + c * R.gs.cs;
                if (R.rank > 0) {
                    const int q = R.rank - 1, nq = slabs_[q].second - slabs_[q].first;
                    const T* src = m_of_[which][q] + plane + c * (nq + 2) * plane + (nq - 1) * plane;
                    ck(cudaMemcpyAsync(mc - plane, src, pb, cudaMemcpyDefault, s), "halo (peer)");
                }
                if (R.rank + 1 < world_) {
                    const int q = R.rank + 1, nq = slabs_[q].second - slabs_[q].first;
                    const T* src = m_of_[which][q] + plane + c * (nq + 2) * plane;
                    ck(cudaMemcpyAsync(mc + R.nzl * plane, src, pb, cudaMemcpyDefault, s), "halo (peer)");
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

    // The prism-sum octant (fp64, every offset) once; each rank's spectrum slice is built from
    // it for that rank's kx columns only (the x pass evaluates just those frequencies, so the y
    // and z passes and their fp64 temporaries shrink by the world size).
    void build_octant(DevBuf<double>& E) {
        E.alloc(6 * static_cast<size_t>(g_.n));
        launch_tensor_octant(E.p, g_.nx, g_.ny, g_.nz, d_.delta, stream_);
    }

    void build_rank_tensor(const DevBuf<double>& E, int k0, int ncols, DevBuf<T>& out) {
        const Geom& g = g_;
        const int nc = std::max(ncols, 1);
        const long long c0 = g.n;
        const long long c1 = static_cast<long long>(nc) * g.ny * g.nz;
        const long long c2 = static_cast<long long>(nc) * g.yh * g.nz;
        const long long c3 = static_cast<long long>(nc) * g.yh * g.zh;
        DevBuf<double2> csx, csy, csz;
        csx.alloc(g.lx);
        csy.alloc(g.ly);
        csz.alloc(g.lz);
        launch_cs_table(csx.p, g.lx, stream_);
        launch_cs_table(csy.p, g.ly, stream_);
        launch_cs_table(csz.p, g.lz, stream_);
        DevBuf<double> a1, a2, a3;
        a1.alloc(6 * c1);
        launch_axis_transform(E.p, a1.p, g.nx, g.ny, g.nz, 0, g.lx, csx.p, 0x06, c0, c1, stream_, k0, nc);
        a2.alloc(6 * c2);
        launch_axis_transform(a1.p, a2.p, nc, g.ny, g.nz, 1, g.ly, csy.p, 0x12, c1, c2, stream_);
        a3.alloc(6 * c3);
        launch_axis_transform(a2.p, a3.p, nc, g.yh, g.nz, 2, g.lz, csz.p, 0x14, c2, c3, stream_);
        out.alloc(6 * c3);
        launch_tensor_finalize_fast<T>(a3.p, out.p, nc, g.yh, g.zh,
                                       1.0 / (static_cast<double>(g.lx) * g.ly * g.lz), stream_);
        ck(cudaStreamSynchronize(stream_), "tensor sync");
    }

    std::unique_ptr<Rank<T>> make_rank(int r, const DevBuf<double>& E) {
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
        // receive blocks: peer q's planes of my columns [ncols][3][nzl_q][ny], q != r
        R->roff.assign(world_, 0);
        long long off = 0;
        for (int q = 0; q < world_; ++q) {
            R->roff[q] = off;
            if (q != r) off += static_cast<long long>(R->ncols) * 3 * (slabs_[q].second - slabs_[q].first) * d_.ny;
        }
        if (!peer_) R->recv.alloc(static_cast<size_t>(std::max(off, 1LL)));
        if (!yz_) R->s2.alloc(static_cast<size_t>(std::max(R->ncols, 1)) * 3 * d_.nz * g_.ly);
        build_rank_tensor(E, R->k0, R->ncols, R->kspec);
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
        ck(cudaStreamSynchronize(comm_stream_), "sync");
        ck(cudaStreamSynchronize(stream_), "sync");
        check_comm();
        check_numerical();
    }

    // an asynchronous NCCL failure (a peer died, a network error) surfaces as a CUDA-class error
    void check_comm() {
        if (!comm_) return;
        ncclResult_t st = ncclSuccess;
        nck(ncclCommGetAsyncError(comm_, &st), "ncclCommGetAsyncError");
        if (st != ncclSuccess) throw cuda_error(std::string("NCCL asynchronous error: ") + ncclGetErrorString(st));
    }

    mmb_desc d_;
    int world_;
    bool emulated_;
    Geom g_{};
    bool yz_ = false;
    StageTable st_{};
    std::vector<std::pair<int, int>> slabs_, cols_;
    int nch_ = 1;
    std::vector<std::vector<std::pair<int, int>>> chunks_; // [rank][chunk] local column range
    std::vector<std::unique_ptr<Rank<T>>> ranks_;
    std::unique_ptr<Transport> transport_;
    cudaStream_t stream_ = nullptr, comm_stream_ = nullptr;
    std::vector<cudaEvent_t> events_;
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
