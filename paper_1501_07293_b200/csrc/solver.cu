// solver.cu — host side of the B200 LLG step: device buffers, the per-step launch sequence,
// CUDA-graph replay, synchronising queries, and the mmb.h C-ABI.
//
// Mirrors mmsim::Simulation<T> (proj/include/mmsim/llg.hpp:78-115, proj/src/llg.cpp):
// same construction (material validation, uniform initial state, tensor precompute),
// same step semantics (schedule at the 0-based step before increment, sticky alpha
// override, demag -> exchange -> anisotropy -> applied accumulation, Euler update with
// fp64 torque max, renormalisation), same run() cadence/stop rules and the same error
// contract (exceptions mapped to status codes as proj/src/capi.cpp:31-58 does).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/mmb.h"
#include "fast.hpp"
#include "kernels.hpp"
#include "solver_base.hpp"
#include "validate.hpp"

namespace mmb {

// Event record that also works inside stream capture (an external event-record node), so the
// per-kernel profile can be taken from inside a replayed graph.
inline void record_event(cudaEvent_t ev, cudaStream_t s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    ck(cudaStreamIsCapturing(s, &cs), "cudaStreamIsCapturing");
    if (cs == cudaStreamCaptureStatusActive) ck(cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal), "record");
    else ck(cudaEventRecord(ev, s), "record");
}

template <typename T>
class Solver final : public SolverBase {
public:
    Solver(const mmb_desc& d, const mmb_stage* stages, int nstages) : d_(d) {
        if (d.nx < 1 || d.ny < 1 || d.nz < 1) throw std::invalid_argument("Grid: cell counts must be >= 1");
        if (!(d.delta > 0.0)) throw std::invalid_argument("Grid: cell edge length must be > 0");
        // MaterialParams::validate (proj/include/mmsim/material.hpp:17-22)
        if (!(d.ms > 0.0)) throw std::invalid_argument("MaterialParams: ms must be > 0");
        if (d.a_ex < 0.0) throw std::invalid_argument("MaterialParams: a_ex must be >= 0");
        if (d.hk < 0.0) throw std::invalid_argument("MaterialParams: hk must be >= 0");
        if (!(d.alpha > 0.0)) throw std::invalid_argument("MaterialParams: alpha must be > 0");
        set_schedule(stages, nstages);

        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw cuda_error("mmb: no CUDA device available (the B200 path has no CPU fallback)");
        if (d.device < 0 || d.device >= ndev) throw std::invalid_argument("mmb: bad device ordinal");
        ck(cudaSetDevice(d.device), "cudaSetDevice");
        ck(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");

        Geom& g = g_;
        g.nx = d.nx;
        g.ny = d.ny;
        g.nz = d.nz;
        g.lx = d.nx == 1 ? 1 : pow2_at_least(2 * d.nx - 1);
        g.ly = d.ny == 1 ? 1 : pow2_at_least(2 * d.ny - 1);
        g.lz = d.nz == 1 ? 1 : pow2_at_least(2 * d.nz - 1);
        g.log2lx = ilog2(g.lx);
        g.log2ly = ilog2(g.ly);
        g.log2lz = ilog2(g.lz);
        if (g.log2lx > 12 || g.log2ly > 12 || g.log2lz > 12)
            throw std::invalid_argument("mmb: grid axis too long (max 2048 cells per axis)");
        g.xh = g.lx == 1 ? 1 : g.lx / 2 + 1;
        g.xp = (g.xh + 15) / 16 * 16;
        g.yh = g.ly == 1 ? 1 : g.ly / 2 + 1;
        g.zh = g.lz == 1 ? 1 : g.lz / 2 + 1;
        g.n = static_cast<long long>(d.nx) * d.ny * d.nz;
        if (3 * g.n >= (1LL << 31))
            throw std::invalid_argument("mmb: more than 715M cells per device (32-bit cell indexing)");
        g.rows = static_cast<long long>(d.ny) * d.nz;
        g.cs = g.n;
        g.nz_g = g.nz;
        g.z0 = 0;

        // Path: fused y/z in shared memory (nz <= 8; z padded to Lz = 16, which gives the same
        // linear convolution as any L >= 2nz-1), streaming y/z kernels for larger blocks, or
        // the general pipeline (MMB_GENERAL_PATH=1 forces it, for parity testing).
        const char* force_general = std::getenv("MMB_GENERAL_PATH");
        const bool allow_fast = !(force_general && force_general[0] == '1');
        Geom gy = g;
        if (gy.nz >= 2 && gy.nz <= 8) {
            gy.lz = 16;
            gy.log2lz = 4;
            gy.zh = 9;
        }
        const char* force_big = std::getenv("MMB_BIG_PATH");
        const bool allow_yz = !(force_big && force_big[0] == '1');
        if (allow_fast && allow_yz && fast_supported<T>(gy)) {
            g = gy;
            fast_ = yz_ = true;
        } else if (allow_fast && big_supported<T>(g)) {
            fast_ = true;
            yz_ = false;
        }

        const size_t n = static_cast<size_t>(g.n);
        m_[0].alloc(3 * n);
        m_[1].alloc(3 * n);
        hd_.alloc(3 * n);
        heff_.alloc(3 * n);
        S_.alloc(fast_ ? static_cast<size_t>(3) * g.nz * g.ny * g.xh
                      : static_cast<size_t>(3) * g.nz * g.ly * g.xp);
        if (fast_ && !yz_) S2_.alloc(static_cast<size_t>(3) * g.nz * g.ly * g.xh);
        kspec_.alloc(static_cast<size_t>(6) * g.zh * g.yh * g.xh);
        twx_.alloc(2 * g.lx);
        twy_.alloc(2 * g.ly);
        twz_.alloc(2 * g.lz);
        partial_.alloc(3 * 1024);
        tpart_count_ = fast_ ? fast_xstep_blocks<T>(g) : llg_blocks(g);
        tpart_.alloc(std::max(llg_blocks(g), tpart_count_));
        // last_torque_sq() before the first step reduces zeros (the reference's
        // last_torque_sq_ starts at 0.0, llg.hpp)
        ck(cudaMemsetAsync(tpart_.p, 0, tpart_.bytes(), stream_), "memset");
        red_.alloc(8);
        ctl_.alloc(1);
        ck(cudaMallocHost(&ctl_host_, sizeof(StepCtl)), "cudaMallocHost");

        launch_twiddles<T>(twx_.p, g.lx, stream_);
        launch_twiddles<T>(twy_.p, g.ly, stream_);
        launch_twiddles<T>(twz_.p, g.lz, stream_);
        if (fast_) prepare_fast_kernels<T>(g_);
        else prepare_fft_kernels<T>(g_);
        if (fast_ && !yz_) prepare_big_kernels<T>(g_);
        // PDL pays on multi-wave grids (>= 1 M cells) and on SP#4-size grids (a few thousand
        // cells, launch-latency bound); on mid-size films it costs time
        pdl_ = g.n >= (1LL << 20) || g.n <= 8192;
        // ... except with the one-CTA-per-SM Lx = 1024 x tile, whose early-launched CTAs only
        // get in the way (+4 us at 512 x 512 x 8)
        if (fast_ && yz_ && g.lx == 1024) pdl_ = false;
        if (const char* e = std::getenv("MMB_PDL"); e && e[0] == '1') pdl_ = true; // tuning
        if (const char* v = std::getenv("MMB_VERBOSE"); v && v[0] == '1')
            std::fprintf(stderr, "mmb: %dx%dx%d L=%dx%dx%d path=%s\n", d.nx, d.ny, d.nz, g.lx, g.ly, g.lz,
                         yz_ ? "yz" : (fast_ ? "big" : "general"));

        // StepCtl: step 0, alpha from the material (llg.cpp:31-33).
        StepCtl c{};
        c.step = 0;
        c.cur_step = 0;
        c.alpha = d.alpha;
        c.dt = d.dt;
        c.ms = d.ms;
        c.bad_key = ~0ull;
        ck(cudaMemcpyAsync(ctl_.p, &c, sizeof(c), cudaMemcpyHostToDevice, stream_), "ctl upload");

        // Tensor entries on device (K0), then the spectrum.
        DevBuf<double> E;
        E.alloc(6 * n);
        launch_tensor_octant(E.p, g.nx, g.ny, g.nz, d.delta, stream_);
        build_spectrum(E.p);

        // init_uniform (proj/include/mmsim/vector_field.hpp:41-52)
        const double norm = std::sqrt(d.init_dir[0] * d.init_dir[0] + d.init_dir[1] * d.init_dir[1] +
                                      d.init_dir[2] * d.init_dir[2]);
        if (!(norm > 0.0)) throw std::invalid_argument("init_uniform: direction vector must be nonzero");
        std::vector<T> col(n);
        for (int c3 = 0; c3 < 3; ++c3) {
            std::fill(col.begin(), col.end(), static_cast<T>(d.ms * d.init_dir[c3] / norm));
            ck(cudaMemcpyAsync(m_[0].p + c3 * n, col.data(), n * sizeof(T), cudaMemcpyHostToDevice,
                               stream_), "M upload");
            ck(cudaStreamSynchronize(stream_), "sync");
        }
        cur_ = 0;
        exch_coeff_ = 2.0 * d.a_ex / (kMu0 * d.ms * d.ms * d.delta * d.delta); // material.hpp:27-29
        aniso_coeff_ = d.hk / d.ms;                                           // local_fields.hpp:27
        ck(cudaStreamSynchronize(stream_), "create sync");
    }

    ~Solver() override {
        for (auto& row : graphs_)
            for (auto& ge : row)
                if (ge) cudaGraphExecDestroy(ge);
        if (ctl_host_) cudaFreeHost(ctl_host_);
        if (rec_host_) cudaFreeHost(rec_host_);
        if (h2d_) {
            cudaStreamSynchronize(h2d_);
            cudaStreamSynchronize(d2h_);
            for (cudaEvent_t e : {in_ready_, in_free_, out_ready_, out_free_}) cudaEventDestroy(e);
            cudaStreamDestroy(h2d_);
            cudaStreamDestroy(d2h_);
        }
        if (stream_) cudaStreamDestroy(stream_);
    }

    int precision() const override { return sizeof(T) == 8 ? MMB_F64 : MMB_F32; }

    void set_m(const void* x, const void* y, const void* z) override {
        const size_t n = g_.n;
        const void* src[3] = {x, y, z};
        for (int c = 0; c < 3; ++c)
            ck(cudaMemcpyAsync(m_[cur_].p + c * n, src[c], n * sizeof(T), cudaMemcpyHostToDevice, stream_),
               "set_m");
        s_valid_ = false;
        // the host arrays are borrowed for the call only: one synchronisation before returning
        ck(cudaStreamSynchronize(stream_), "set_m sync");
    }

    void get_m(void* x, void* y, void* z) override {
        const size_t n = g_.n;
        void* dst[3] = {x, y, z};
        for (int c = 0; c < 3; ++c)
            ck(cudaMemcpyAsync(dst[c], m_[cur_].p + c * n, n * sizeof(T), cudaMemcpyDeviceToHost, stream_),
               "get_m");
        sync_and_check();
    }

    // n steps as graph replays: n = 32 q + binary digits of the rest, one graph of 2^b
    // consecutive steps per digit (at most q + 5 graph launches, so a short run replays at the
    // long-run rate); only the 1-step graph flips the ping-pong buffer
    // Pipelined host I/O: host <-> staging copies on their own streams, staging <-> M on the
    // main stream, events in both directions so a staging buffer is reused only after its
    // previous copy finished.
    void set_m_async(const void* x, const void* y, const void* z) override {
        ensure_io();
        const size_t n = g_.n;
        const void* src[3] = {x, y, z};
        if (in_free_rec_) ck(cudaStreamWaitEvent(h2d_, in_free_, 0), "wait");
        for (int c = 0; c < 3; ++c)
            ck(cudaMemcpyAsync(in_.p + c * n, src[c], n * sizeof(T), cudaMemcpyHostToDevice, h2d_), "set_m_async");
        ck(cudaEventRecord(in_ready_, h2d_), "record");
        ck(cudaStreamWaitEvent(stream_, in_ready_, 0), "wait");
        ck(cudaMemcpyAsync(m_[cur_].p, in_.p, 3 * n * sizeof(T), cudaMemcpyDeviceToDevice, stream_), "set_m_async");
        ck(cudaEventRecord(in_free_, stream_), "record");
        in_free_rec_ = true;
        s_valid_ = false;
    }

    void get_m_async(void* x, void* y, void* z) override {
        ensure_io();
        const size_t n = g_.n;
        void* dst[3] = {x, y, z};
        if (out_free_rec_) ck(cudaStreamWaitEvent(stream_, out_free_, 0), "wait");
        ck(cudaMemcpyAsync(out_.p, m_[cur_].p, 3 * n * sizeof(T), cudaMemcpyDeviceToDevice, stream_), "get_m_async");
        ck(cudaEventRecord(out_ready_, stream_), "record");
        ck(cudaStreamWaitEvent(d2h_, out_ready_, 0), "wait");
        for (int c = 0; c < 3; ++c)
            ck(cudaMemcpyAsync(dst[c], out_.p + c * n, n * sizeof(T), cudaMemcpyDeviceToHost, d2h_), "get_m_async");
        ck(cudaEventRecord(out_free_, d2h_), "record");
        out_free_rec_ = true;
    }

    void ensure_io() {
        if (h2d_) return;
        ck(cudaStreamCreateWithFlags(&h2d_, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking), "cudaStreamCreate");
        for (cudaEvent_t* e : {&in_ready_, &in_free_, &out_ready_, &out_free_})
            ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        in_.alloc(3 * static_cast<size_t>(g_.n));
        out_.alloc(3 * static_cast<size_t>(g_.n));
    }

    void step(long long n) override {
        NvtxRange r("mmb::step");
        if (n > 0) prime();
        for (; n >= (1LL << kMaxLog2Batch); n -= (1LL << kMaxLog2Batch)) launch_graph(kMaxLog2Batch);
        for (int b = kMaxLog2Batch - 1; b >= 0; --b)
            if (n & (1LL << b)) launch_graph(b);
    }

    void launch_graph(int b) {
        ensure_graph(b, cur_);
        ck(cudaGraphLaunch(graphs_[b][cur_], stream_), "cudaGraphLaunch");
        if (b == 0) cur_ ^= 1;
        step_ += 1LL << b;
    }

    // instantiate every graph step(n) will replay (outside any timed region)
    void prepare_graphs(long long n) {
        int cur = cur_;
        if (n >= (1LL << kMaxLog2Batch)) ensure_graph(kMaxLog2Batch, cur);
        for (int b = kMaxLog2Batch - 1; b >= 0; --b)
            if (n & (1LL << b)) {
                ensure_graph(b, cur);
                if (b == 0) cur ^= 1;
            }
    }

    long long step_index() const override { return step_; }

    void average(double* out) override {
        // average_magnetization (vector_field.hpp:86-99) / average_unit (llg.cpp:126-131)
        launch_sum3<T>(m_[cur_].p, g_.n, g_.n, partial_.p, red_.p, stream_);
        double s[3];
        ck(cudaMemcpyAsync(s, red_.p, sizeof(s), cudaMemcpyDeviceToHost, stream_), "average");
        sync_and_check();
        const double inv = 1.0 / static_cast<double>(g_.n);
        const double inv_ms = 1.0 / d_.ms;
        for (int c = 0; c < 3; ++c) out[c] = (inv * s[c]) * inv_ms;
    }

    double energy() override {
        // Simulation<T>::energy (llg.cpp:133-138): applied field at step_ (no alpha update),
        // demag recomputed, total_energy (energy.cpp:39-64).
        enqueue_demag(m_[cur_].p, hd_.p, 3);
        const double ms = d_.ms;
        const double ku = 0.5 * d_.hk * kMu0 * ms;
        launch_energy<T>(m_[cur_].p, hd_.p, g_, ku / (ms * ms), ctl_.p, partial_.p, red_.p, stream_);
        double e[2];
        ck(cudaMemcpyAsync(e, red_.p, sizeof(e), cudaMemcpyDeviceToHost, stream_), "energy");
        sync_and_check();
        return e[0] * (d_.delta * d_.delta * d_.delta) + d_.a_ex * d_.delta / (ms * ms) * e[1];
    }

    double max_torque() override {
        // llg.cpp:140-156: re-assemble H_eff (may apply the sticky alpha override).
        enqueue_heff();
        launch_torque_max<T>(m_[cur_].p, heff_.p, g_.n, g_.n,
                             reinterpret_cast<unsigned long long*>(red_.p + 4), stream_);
        double sq;
        ck(cudaMemcpyAsync(&sq, red_.p + 4, sizeof(sq), cudaMemcpyDeviceToHost, stream_), "torque");
        sync_and_check();
        return std::sqrt(sq) / (d_.ms * d_.ms);
    }

    double last_torque_sq() override {
        launch_torque_partials(tpart_.p, tpart_count_, ctl_.p, stream_);
        fetch_ctl();
        double v;
        std::memcpy(&v, &ctl_host_->torque_sq_bits, sizeof(v));
        return v;
    }

    long long run(long long steps, long long cadence, double stop_torque, mmb_record_fn fn,
                  void* user) override {
        NvtxRange r("mmb::run");
        // Simulation<T>::run (llg.cpp:110-124): record on absolute step_ % cadence == 0, stop
        // when sqrt(last_torque_sq)/ms^2 < stop_torque.
        const double ms2 = d_.ms * d_.ms;
        long long done = 0;
        const bool stop = stop_torque >= 0.0;
        if (fn && cadence > 0 && !stop) return run_streaming(steps, cadence, fn, user);
        while (done < steps) {
            // Batch graph replays up to the next record point when no per-step check is needed.
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

    // run() without a torque stop: each record's <m> sums go into a device ring right behind
    // the graph replays (no host round trip per record); the ring is copied back and delivered
    // to `fn` in order every kRing records and at the end. If a step failed, the records taken
    // before the failing step are delivered first, then the error is raised as usual.
    long long run_streaming(long long steps, long long cadence, mmb_record_fn fn, void* user) {
        constexpr int kRing = 256;
        if (!rec_.p) {
            rec_.alloc(3 * kRing);
            ck(cudaMallocHost(&rec_host_, 3 * kRing * sizeof(double)), "cudaMallocHost");
        }
        long long rsteps[kRing];
        int nrec = 0;
        const double inv = 1.0 / static_cast<double>(g_.n), inv_ms = 1.0 / d_.ms;
        auto flush = [&]() {
            if (nrec) ck(cudaMemcpyAsync(rec_host_, rec_.p, 3 * nrec * sizeof(double), cudaMemcpyDeviceToHost, stream_),
                         "records");
            ck(cudaStreamSynchronize(stream_), "sync");
            fetch_ctl();
            const unsigned long long key = ctl_host_->bad_key;
            const long long fail = key != ~0ull ? static_cast<long long>(key >> 36) : (1LL << 62);
            for (int i = 0; i < nrec && rsteps[i] <= fail; ++i) {
                const double* s = rec_host_ + 3 * i;
                fn(user, rsteps[i], (inv * s[0]) * inv_ms, (inv * s[1]) * inv_ms, (inv * s[2]) * inv_ms);
            }
            nrec = 0;
            check_numerical();
        };
        long long done = 0;
        while (done < steps) {
            const long long chunk = std::min(steps - done, cadence - (step_ % cadence));
            step(chunk);
            done += chunk;
            if (step_ % cadence == 0) {
                launch_sum3<T>(m_[cur_].p, g_.n, g_.n, partial_.p, rec_.p + 3 * nrec, stream_);
                rsteps[nrec++] = step_;
                if (nrec == kRing) flush();
            }
        }
        flush();
        return done;
    }

    void effective_field(void* x, void* y, void* z) override {
        enqueue_heff();
        copy_out(heff_.p, x, y, z);
    }

    void demag_field(const void* mx, const void* my, const void* mz, void* hx, void* hy,
                     void* hz) override {
        const size_t n = g_.n;
        const void* src[3] = {mx, my, mz};
        for (int c = 0; c < 3; ++c)
            ck(cudaMemcpyAsync(heff_.p + c * n, src[c], n * sizeof(T), cudaMemcpyHostToDevice, stream_),
               "demag upload");
        enqueue_demag(heff_.p, hd_.p, 0);
        copy_out(hd_.p, hx, hy, hz);
    }

    void tensor_octant(double* out) override {
        DevBuf<double> E;
        E.alloc(6 * static_cast<size_t>(g_.n));
        launch_tensor_octant(E.p, g_.nx, g_.ny, g_.nz, d_.delta, stream_);
        ck(cudaMemcpyAsync(out, E.p, E.bytes(), cudaMemcpyDeviceToHost, stream_), "octant");
        sync_and_check();
    }

    void upload_tensor_octant(const double* entries) override {
        DevBuf<double> E;
        E.alloc(6 * static_cast<size_t>(g_.n));
        ck(cudaMemcpyAsync(E.p, entries, E.bytes(), cudaMemcpyHostToDevice, stream_), "octant upload");
        build_spectrum(E.p);
        sync_and_check();
    }

    float time_steps(long long n) override {
        prime();
        prepare_graphs(n);
        cudaEvent_t a, b;
        ck(cudaEventCreate(&a), "event");
        ck(cudaEventCreate(&b), "event");
        // the stream is busy for 200 us before the start event, so every graph launch of the
        // timed sequence is already queued when the device reaches it (device time only)
        launch_spin(200000ull, stream_);
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

    // Per-kernel device time from inside replayed graphs: a graph of kProfSteps consecutive
    // steps with an external event-record node between consecutive kernels (the same kernels
    // and launch parameters as the production graphs, minus any programmatic-launch overlap
    // across the event nodes), replayed until n steps ran; mean per step per kernel.
    int profile_step(long long n, float* out, int maxk, std::string& names) override {
        constexpr int kProfSteps = 16; // even: the graph returns M to the same buffer
        const std::vector<std::string> kn = kernel_names();
        const int nk = static_cast<int>(kn.size());
        std::vector<cudaEvent_t> ev(static_cast<size_t>(kProfSteps) * (nk + 1));
        for (auto& e : ev) ck(cudaEventCreate(&e), "event");
        prime();
        cudaGraph_t gr;
        cudaGraphExec_t ge = nullptr;
        ck(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
        for (int i = 0; i < kProfSteps; ++i) {
            cudaEvent_t* e = ev.data() + static_cast<size_t>(i) * (nk + 1);
            record_event(e[0], stream_);
            enqueue_step_eager(cur_ ^ (i & 1), e);
        }
        ck(cudaStreamEndCapture(stream_, &gr), "end capture");
        ck(cudaGraphInstantiate(&ge, gr, 0), "graph instantiate");
        cudaGraphDestroy(gr);
        std::vector<double> acc(nk, 0.0);
        long long done = 0;
        const long long reps = std::max<long long>(1, (n + kProfSteps - 1) / kProfSteps);
        for (long long r = 0; r < reps; ++r) {
            ck(cudaGraphLaunch(ge, stream_), "cudaGraphLaunch");
            ck(cudaStreamSynchronize(stream_), "sync");
            for (int i = 0; i < kProfSteps; ++i)
                for (int k = 0; k < nk; ++k) {
                    float ms = 0.f;
                    const size_t b = static_cast<size_t>(i) * (nk + 1);
                    ck(cudaEventElapsedTime(&ms, ev[b + k], ev[b + k + 1]), "elapsed");
                    acc[k] += ms;
                }
            done += kProfSteps;
            step_ += kProfSteps;
        }
        cudaGraphExecDestroy(ge);
        for (auto& e : ev) cudaEventDestroy(e);
        names.clear();
        for (int k = 0; k < nk; ++k) {
            if (k < maxk) out[k] = static_cast<float>(acc[k] / static_cast<double>(done));
            names += kn[k];
            if (k + 1 < nk) names += ";";
        }
        check_numerical();
        return nk;
    }

    int launches_per_step() const override { return static_cast<int>(kernel_names().size()); }

    void slab(int& z0, int& nzl) const override {
        z0 = 0;
        nzl = g_.nz;
    }

    std::string path_info() const override {
        char head[160];
        std::snprintf(head, sizeof head, "path=%s n=%dx%dx%d L=%dx%dx%d prec=%s pdl=%d", yz_ ? "yz" : (fast_ ? "big" : "general"),
                      g_.nx, g_.ny, g_.nz, g_.lx, g_.ly, g_.lz, sizeof(T) == 8 ? "f64" : "f32", pdl_ ? 1 : 0);
        std::string s = head;
        if (fast_ && yz_) s += "; " + fast_describe<T>(g_);
        else if (fast_) s += "; " + big_describe<T>(g_) + "; " + fast_describe_xstep(g_);
        return s;
    }

    static std::string fast_describe_xstep(const Geom& g) {
        const std::string d = fast_describe<T>(g);
        const size_t k = d.find("k_xstep");
        return k == std::string::npos ? d : d.substr(k);
    }

    size_t device_bytes() const override {
        return m_[0].bytes() + m_[1].bytes() + hd_.bytes() + heff_.bytes() + S_.bytes() + S2_.bytes() +
               kspec_.bytes() + twx_.bytes() + twy_.bytes() + twz_.bytes() + partial_.bytes() +
               red_.bytes() + tpart_.bytes() + ctl_.bytes();
    }

private:
    void set_schedule(const mmb_stage* stages, int n) {
        // FieldSchedule ctor validation (proj/src/schedule.cpp:8-17)
        if (n < 0 || (n > 0 && !stages)) throw std::invalid_argument("mmb: bad stage list");
        if (n > kMaxStages) throw std::invalid_argument("mmb: too many schedule stages (max 16)");
        std::vector<mmb_stage> s(stages, stages + n);
        std::stable_sort(s.begin(), s.end(),
                         [](const mmb_stage& a, const mmb_stage& b) { return a.start < b.start; });
        for (size_t i = 0; i < s.size(); ++i) {
            if (s[i].end <= s[i].start)
                throw std::invalid_argument("FieldSchedule: stage range must be nonempty");
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

    void build_spectrum(const double* E) {
        const Geom& g = g_;
        DevBuf<double2> csx, csy, csz;
        csx.alloc(g.lx);
        csy.alloc(g.ly);
        csz.alloc(g.lz);
        launch_cs_table(csx.p, g.lx, stream_);
        launch_cs_table(csy.p, g.ly, stream_);
        launch_cs_table(csz.p, g.lz, stream_);
        const long long c0 = g.n;
        const long long c1 = static_cast<long long>(g.xh) * g.ny * g.nz;
        const long long c2 = static_cast<long long>(g.xh) * g.yh * g.nz;
        const long long c3 = static_cast<long long>(g.xh) * g.yh * g.zh;
        DevBuf<double> a1, a2, a3;
        a1.alloc(6 * c1);
        launch_axis_transform(E, a1.p, g.nx, g.ny, g.nz, 0, g.lx, csx.p, 0x06, c0, c1, stream_);
        a2.alloc(6 * c2);
        launch_axis_transform(a1.p, a2.p, g.xh, g.ny, g.nz, 1, g.ly, csy.p, 0x12, c1, c2, stream_);
        a3.alloc(6 * c3);
        launch_axis_transform(a2.p, a3.p, g.xh, g.yh, g.nz, 2, g.lz, csz.p, 0x14, c2, c3, stream_);
        const double scale = 1.0 / (static_cast<double>(g.lx) * g.ly * g.lz);
        if (fast_) launch_tensor_finalize_fast<T>(a3.p, kspec_.p, g.xh, g.yh, g.zh, scale, stream_);
        else launch_tensor_finalize<T>(a3.p, kspec_.p, c3, scale, stream_);
        ck(cudaStreamSynchronize(stream_), "spectrum sync");
    }

    std::vector<std::string> kernel_names() const {
        if (fast_ && yz_) return {"yz", "xstep"};
        if (fast_) return {"y_fwd", "z_mac", "y_inv", "xstep"};
        if (g_.nz == 1) return {"x_fwd", "y_mac", "x_inv", "llg"};
        return {"x_fwd", "y_fwd", "z_mac", "y_inv", "x_inv", "llg"};
    }

    // Demag of m into h; prologue: 0 none, 1 stepping, 2 assembly, 3 applied field only.
    void enqueue_demag(const T* m, T* h, int prologue, cudaEvent_t* ev = nullptr) {
        int k = 1;
        auto mark = [&]() {
            if (ev) record_event(ev[k++], stream_);
        };
        if (fast_) {
            // S is reused as scratch: it no longer holds the x spectrum of the current M
            s_valid_ = false;
            launch_fast_xf<T>(m, S_.p, g_, twx_.p, ctl_.p, st_, prologue, stream_);
            mark();
            enqueue_yz(0, ev ? &k : nullptr, ev);
            launch_fast_xi<T>(S_.p, h, g_, twx_.p, stream_);
            mark();
            return;
        }
        launch_x_fwd<T>(m, S_.p, g_, twx_.p, ctl_.p, st_, prologue, stream_);
        mark();
        if (g_.nz == 1) {
            launch_y_mac<T>(S_.p, g_, twy_.p, kspec_.p, stream_);
            mark();
        } else {
            launch_y<T>(0, S_.p, g_, twy_.p, stream_);
            mark();
            launch_z_mac<T>(S_.p, g_, twz_.p, kspec_.p, stream_);
            mark();
            launch_y<T>(1, S_.p, g_, twy_.p, stream_);
            mark();
        }
        launch_x_inv<T>(S_.p, h, g_, twx_.p, stream_);
        mark();
    }

    // Fast path: the step starts from S = x spectrum of M_cur (kept valid across steps by the
    // fused KXS); prime() recomputes it after anything else touched M or S.
    void prime() {
        if (!fast_ || s_valid_) return;
        launch_fast_xf<T>(m_[cur_].p, S_.p, g_, twx_.p, ctl_.p, st_, 0, stream_);
        s_valid_ = true;
    }

    // y/z part of the fast path on S (fused KYZ, or KYF/KZ/KYI through S2); `k` indexes
    // the profiling events.
    void enqueue_yz(int prologue, int* k, cudaEvent_t* ev) {
        auto mark = [&]() {
            if (ev && k) record_event(ev[(*k)++], stream_);
        };
        if (yz_) {
            launch_fast_yz<T>(S_.p, g_, twy_.p, kspec_.p, ctl_.p, st_, prologue, stream_, pdl_);
            mark();
            return;
        }
        launch_big_yf<T>(S_.p, S2_.p, g_, twy_.p, ctl_.p, st_, prologue, stream_);
        mark();
        launch_big_z<T>(S2_.p, g_, twz_.p, kspec_.p, stream_);
        mark();
        launch_big_yi<T>(S2_.p, S_.p, g_, twy_.p, stream_);
        mark();
    }

    void enqueue_step_eager(int cur, cudaEvent_t* ev = nullptr) {
        if (fast_) {
            int k = 1;
            enqueue_yz(1, &k, ev);
            launch_fast_xstep<T>(S_.p, m_[cur].p, m_[cur ^ 1].p, g_, twx_.p, exch_coeff_, aniso_coeff_,
                                 ctl_.p, tpart_.p, stream_, pdl_);
            if (ev) record_event(ev[k], stream_);
            return;
        }
        enqueue_demag(m_[cur].p, hd_.p, 1, ev);
        launch_llg<T>(0, m_[cur].p, hd_.p, m_[cur ^ 1].p, g_, exch_coeff_, aniso_coeff_, ctl_.p, tpart_.p, stream_);
        if (ev) record_event(ev[kernel_names().size()], stream_);
    }

    void enqueue_heff() {
        enqueue_demag(m_[cur_].p, hd_.p, 2);
        launch_llg<T>(1, m_[cur_].p, hd_.p, heff_.p, g_, exch_coeff_, aniso_coeff_, ctl_.p, tpart_.p, stream_);
    }

    // graph of 2^b consecutive steps starting from buffer `cur`
    void ensure_graph(int b, int cur) {
        if (graphs_[b][cur]) return;
        cudaGraph_t gr;
        ck(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "begin capture");
        for (int i = 0; i < (1 << b); ++i) enqueue_step_eager(cur ^ (i & 1));
        ck(cudaStreamEndCapture(stream_, &gr), "end capture");
        ck(cudaGraphInstantiate(&graphs_[b][cur], gr, 0), "graph instantiate");
        cudaGraphDestroy(gr);
    }

    void copy_out(const T* src, void* x, void* y, void* z) {
        const size_t n = g_.n;
        void* dst[3] = {x, y, z};
        for (int c = 0; c < 3; ++c)
            ck(cudaMemcpyAsync(dst[c], src + c * n, n * sizeof(T), cudaMemcpyDeviceToHost, stream_), "copy out");
        sync_and_check();
    }

    void fetch_ctl() {
        ck(cudaMemcpyAsync(ctl_host_, ctl_.p, sizeof(StepCtl), cudaMemcpyDeviceToHost, stream_), "ctl");
        ck(cudaStreamSynchronize(stream_), "ctl sync");
    }

    void check_numerical() {
        fetch_ctl();
        const unsigned long long key = ctl_host_->bad_key;
        if (key != ~0ull) {
            const long long cell = static_cast<long long>(key & ((1ull << 36) - 1));
            const long long st = static_cast<long long>(key >> 36);
            // The reference's step() throws before ++step_ (llg.cpp:102-107): the step index
            // returns to the failing step (steps queued after it ran on a degenerate state; M
            // is unspecified after a numerical failure, as in the reference). Reset the error
            // word so the handle can report later failures.
            step_ = st;
            StepCtl* c = ctl_host_;
            c->bad_key = ~0ull;
            c->step = st;
            c->cur_step = st;
            ck(cudaMemcpyAsync(ctl_.p, c, sizeof(StepCtl), cudaMemcpyHostToDevice, stream_), "reset");
            ck(cudaStreamSynchronize(stream_), "reset sync");
            s_valid_ = false;
            throw numerical_error("renormalize: zero-magnitude magnetization at cell " +
                                  std::to_string(cell) + " at step " + std::to_string(st));
        }
    }

    void sync_and_check() {
        ck(cudaStreamSynchronize(stream_), "sync");
        if (h2d_) {
            ck(cudaStreamSynchronize(h2d_), "sync");
            ck(cudaStreamSynchronize(d2h_), "sync");
        }
        check_numerical();
    }

    mmb_desc d_;
    Geom g_{};
    StageTable st_{};
    cudaStream_t stream_ = nullptr;
    DevBuf<T> m_[2], hd_, heff_;
    // pipelined host I/O (set_m_async / get_m_async): copy streams, staging buffers, events
    cudaStream_t h2d_ = nullptr, d2h_ = nullptr;
    DevBuf<T> in_, out_;
    cudaEvent_t in_ready_ = nullptr, in_free_ = nullptr, out_ready_ = nullptr, out_free_ = nullptr;
    bool in_free_rec_ = false, out_free_rec_ = false;
    DevBuf<cx<T>> S_, S2_, twx_, twy_, twz_;
    DevBuf<T> kspec_;
    DevBuf<double> partial_, red_, tpart_, rec_;
    double* rec_host_ = nullptr;
    DevBuf<StepCtl> ctl_;
    StepCtl* ctl_host_ = nullptr;
    static constexpr int kMaxLog2Batch = 5; // graphs of 1, 2, 4, 8, 16 and 32 steps
    cudaGraphExec_t graphs_[kMaxLog2Batch + 1][2] = {};
    // programmatic dependent launch between the per-step kernels: pays on large grids only
    bool pdl_ = false;
    int cur_ = 0;
    bool fast_ = false;
    bool yz_ = false;       // fast path with the fused shared-memory y/z kernel
    bool s_valid_ = false;  // fast path: S holds the x spectrum of m_[cur_]
    int tpart_count_ = 0;
    long long step_ = 0;
    double exch_coeff_ = 0.0, aniso_coeff_ = 0.0;
};

} // namespace mmb

// ------------------------------------------------------------------------------ C-ABI
struct mmb_ctx {
    std::unique_ptr<mmb::SolverBase> s;
};

namespace {

thread_local std::string t_last_error;

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const mmb::numerical_error& e) {
        t_last_error = e.what();
        return MMB_ERROR_NUMERICAL;
    } catch (const std::invalid_argument& e) {
        t_last_error = e.what();
        return MMB_ERROR_ARGUMENT;
    } catch (const std::bad_alloc&) {
        t_last_error = "out of memory";
        return MMB_ERROR_NOMEM;
    } catch (const mmb::cuda_error& e) {
        t_last_error = e.what();
        return MMB_ERROR_CUDA;
    } catch (const std::exception& e) {
        t_last_error = e.what();
        return MMB_ERROR_INTERNAL;
    } catch (...) {
        t_last_error = "unknown error";
        return MMB_ERROR_INTERNAL;
    }
}

int bad(const char* what) {
    t_last_error = std::string(what) + ": NULL or invalid argument";
    return MMB_ERROR_ARGUMENT;
}

} // namespace

extern "C" {

const char* mmb_status_string(int status) {
    switch (status) {
        case MMB_OK: return "ok";
        case MMB_ERROR_ARGUMENT: return "invalid argument";
        case MMB_ERROR_CONFIG: return "configuration error";
        case MMB_ERROR_NUMERICAL: return "numerical failure";
        case MMB_ERROR_IO: return "i/o error";
        case MMB_ERROR_NOMEM: return "out of memory";
        case MMB_ERROR_VALIDATION: return "validation failure";
        case MMB_ERROR_INTERNAL: return "internal error";
        case MMB_ERROR_CUDA: return "cuda error";
        default: return "unknown status";
    }
}

const char* mmb_last_error(void) { return t_last_error.c_str(); }

void mmb_string_free(char* s) { delete[] s; }

int mmb_validate(char** report_out) {
    return guarded([&] {
        bool ok = false;
        const std::string report = mmb::run_device_validation(ok);
        if (report_out) {
            char* out = new char[report.size() + 1];
            std::memcpy(out, report.c_str(), report.size() + 1);
            *report_out = out;
        }
        if (!ok) {
            t_last_error = "validation suite reported failing checks";
            return static_cast<int>(MMB_ERROR_VALIDATION);
        }
        return static_cast<int>(MMB_OK);
    });
}
const char* mmb_version(void) { return "0.1.0-b200"; }

int mmb_create(const mmb_desc* desc, const mmb_stage* stages, int nstages, mmb_ctx** out) {
    if (!desc || !out) return bad("mmb_create");
    *out = nullptr;
    return guarded([&] {
        auto h = std::make_unique<mmb_ctx>();
        if (desc->precision == MMB_F64) h->s = std::make_unique<mmb::Solver<double>>(*desc, stages, nstages);
        else if (desc->precision == MMB_F32) h->s = std::make_unique<mmb::Solver<float>>(*desc, stages, nstages);
        else throw std::invalid_argument("unknown precision (expected MMB_F32 or MMB_F64)");
        *out = h.release();
        return MMB_OK;
    });
}

void mmb_free(mmb_ctx* ctx) { delete ctx; }

int mmb_set_m(mmb_ctx* ctx, const void* x, const void* y, const void* z) {
    if (!ctx || !x || !y || !z) return bad("mmb_set_m");
    return guarded([&] { ctx->s->set_m(x, y, z); return MMB_OK; });
}

int mmb_get_m(mmb_ctx* ctx, void* x, void* y, void* z) {
    if (!ctx || !x || !y || !z) return bad("mmb_get_m");
    return guarded([&] { ctx->s->get_m(x, y, z); return MMB_OK; });
}

int mmb_set_m_async(mmb_ctx* ctx, const void* x, const void* y, const void* z) {
    if (!ctx || !x || !y || !z) return bad("mmb_set_m_async");
    return guarded([&] { ctx->s->set_m_async(x, y, z); return MMB_OK; });
}

int mmb_get_m_async(mmb_ctx* ctx, void* x, void* y, void* z) {
    if (!ctx || !x || !y || !z) return bad("mmb_get_m_async");
    return guarded([&] { ctx->s->get_m_async(x, y, z); return MMB_OK; });
}

int mmb_step(mmb_ctx* ctx, long long n) {
    if (!ctx || n < 0) {
        t_last_error = "mmb_step: bad handle or negative count";
        return MMB_ERROR_ARGUMENT;
    }
    return guarded([&] { ctx->s->step(n); return MMB_OK; });
}

int mmb_step_index(const mmb_ctx* ctx, long long* out) {
    if (!ctx || !out) return bad("mmb_step_index");
    *out = ctx->s->step_index();
    return MMB_OK;
}

int mmb_average(mmb_ctx* ctx, double out[3]) {
    if (!ctx || !out) return bad("mmb_average");
    return guarded([&] { ctx->s->average(out); return MMB_OK; });
}

int mmb_energy(mmb_ctx* ctx, double* out) {
    if (!ctx || !out) return bad("mmb_energy");
    return guarded([&] { *out = ctx->s->energy(); return MMB_OK; });
}

int mmb_max_torque(mmb_ctx* ctx, double* out) {
    if (!ctx || !out) return bad("mmb_max_torque");
    return guarded([&] { *out = ctx->s->max_torque(); return MMB_OK; });
}

int mmb_last_torque_sq(mmb_ctx* ctx, double* out) {
    if (!ctx || !out) return bad("mmb_last_torque_sq");
    return guarded([&] { *out = ctx->s->last_torque_sq(); return MMB_OK; });
}

int mmb_run(mmb_ctx* ctx, long long steps, long long cadence, double stop_torque,
            mmb_record_fn record, void* user, long long* steps_done) {
    if (!ctx || steps < 0) return bad("mmb_run");
    return guarded([&] {
        const long long d = ctx->s->run(steps, cadence, stop_torque, record, user);
        if (steps_done) *steps_done = d;
        return MMB_OK;
    });
}

int mmb_synchronize(mmb_ctx* ctx) {
    if (!ctx) return bad("mmb_synchronize");
    return guarded([&] { ctx->s->synchronize(); return MMB_OK; });
}

int mmb_effective_field(mmb_ctx* ctx, void* hx, void* hy, void* hz) {
    if (!ctx || !hx || !hy || !hz) return bad("mmb_effective_field");
    return guarded([&] { ctx->s->effective_field(hx, hy, hz); return MMB_OK; });
}

int mmb_demag_field(mmb_ctx* ctx, const void* mx, const void* my, const void* mz, void* hx,
                    void* hy, void* hz) {
    if (!ctx || !mx || !my || !mz || !hx || !hy || !hz) return bad("mmb_demag_field");
    return guarded([&] { ctx->s->demag_field(mx, my, mz, hx, hy, hz); return MMB_OK; });
}

int mmb_tensor_octant(mmb_ctx* ctx, double* out) {
    if (!ctx || !out) return bad("mmb_tensor_octant");
    return guarded([&] { ctx->s->tensor_octant(out); return MMB_OK; });
}

int mmb_upload_tensor_octant(mmb_ctx* ctx, const double* entries) {
    if (!ctx || !entries) return bad("mmb_upload_tensor_octant");
    return guarded([&] { ctx->s->upload_tensor_octant(entries); return MMB_OK; });
}

int mmb_time_steps(mmb_ctx* ctx, long long n, float* ms) {
    if (!ctx || !ms || n < 0) return bad("mmb_time_steps");
    return guarded([&] { *ms = ctx->s->time_steps(n); return MMB_OK; });
}

int mmb_profile_step(mmb_ctx* ctx, long long n, float* kernel_ms, int max_kernels, int* count,
                     char* names_buf, size_t names_len) {
    if (!ctx || !kernel_ms || !count || n < 1) return bad("mmb_profile_step");
    return guarded([&] {
        std::string names;
        *count = ctx->s->profile_step(n, kernel_ms, max_kernels, names);
        if (names_buf && names_len) {
            const size_t k = std::min(names.size(), names_len - 1);
            std::memcpy(names_buf, names.data(), k);
            names_buf[k] = 0;
        }
        return MMB_OK;
    });
}

int mmb_launches_per_step(mmb_ctx* ctx, int* out) {
    if (!ctx || !out) return bad("mmb_launches_per_step");
    *out = ctx->s->launches_per_step();
    return MMB_OK;
}

int mmb_nccl_unique_id(unsigned char out[128]) {
    if (!out) return bad("mmb_nccl_unique_id");
    return guarded([&] { mmb::nccl_unique_id(out); return MMB_OK; });
}

int mmb_create_sharded(const mmb_desc* desc, const mmb_stage* stages, int nstages, int rank,
                       int world, const unsigned char nccl_id[128], mmb_ctx** out) {
    if (!desc || !out || !nccl_id) return bad("mmb_create_sharded");
    *out = nullptr;
    return guarded([&] {
        auto h = std::make_unique<mmb_ctx>();
        // one rank owns the whole grid: no exchange is needed, so the single-device solver
        // runs it (MMB_FORCE_SHARDED=1 keeps the NCCL slab pipeline, for testing it)
        const char* force = std::getenv("MMB_FORCE_SHARDED");
        if (world == 1 && rank == 0 && !(force && force[0] == '1')) {
            if (desc->precision == MMB_F64) h->s = std::make_unique<mmb::Solver<double>>(*desc, stages, nstages);
            else if (desc->precision == MMB_F32) h->s = std::make_unique<mmb::Solver<float>>(*desc, stages, nstages);
            else throw std::invalid_argument("unknown precision (expected MMB_F32 or MMB_F64)");
        } else {
            h->s = mmb::make_sharded(*desc, stages, nstages, rank, world, nccl_id);
        }
        *out = h.release();
        return MMB_OK;
    });
}

int mmb_create_emulated(const mmb_desc* desc, const mmb_stage* stages, int nstages, int world,
                        mmb_ctx** out) {
    if (!desc || !out) return bad("mmb_create_emulated");
    *out = nullptr;
    return guarded([&] {
        auto h = std::make_unique<mmb_ctx>();
        h->s = mmb::make_emulated(*desc, stages, nstages, world);
        *out = h.release();
        return MMB_OK;
    });
}

int mmb_slab(mmb_ctx* ctx, int* z0, int* nz_local) {
    if (!ctx || !z0 || !nz_local) return bad("mmb_slab");
    ctx->s->slab(*z0, *nz_local);
    return MMB_OK;
}

int mmb_random_unit_field(unsigned seed, double ms, long long first, long long count, int precision,
                          void* x, void* y, void* z) {
    if (!x || !y || !z || first < 0 || count < 0 || (precision != MMB_F32 && precision != MMB_F64))
        return bad("mmb_random_unit_field");
    return guarded([&] {
        // proj/src/validate.cpp:21-39: mt19937(seed), U(-1, 1) from libstdc++, rejection of
        // norm < 0.1, ms * v / norm in double, then cast to T. Cells before `first` are drawn
        // and dropped (a slab of the same global field).
        std::mt19937 rng(seed);
        std::uniform_real_distribution<double> dist(-1.0, 1.0);
        for (long long i = 0; i < first + count; ++i) {
            double a, b, c, norm;
            do {
                a = dist(rng);
                b = dist(rng);
                c = dist(rng);
                norm = std::sqrt(a * a + b * b + c * c);
            } while (norm < 0.1);
            if (i < first) continue;
            const long long k = i - first;
            if (precision == MMB_F64) {
                static_cast<double*>(x)[k] = ms * a / norm;
                static_cast<double*>(y)[k] = ms * b / norm;
                static_cast<double*>(z)[k] = ms * c / norm;
            } else {
                static_cast<float*>(x)[k] = static_cast<float>(ms * a / norm);
                static_cast<float*>(y)[k] = static_cast<float>(ms * b / norm);
                static_cast<float*>(z)[k] = static_cast<float>(ms * c / norm);
            }
        }
        return MMB_OK;
    });
}

int mmb_path_info(mmb_ctx* ctx, char* buf, size_t len) {
    if (!ctx || !buf || len == 0) return bad("mmb_path_info");
    return guarded([&] {
        const std::string s = ctx->s->path_info();
        const size_t k = std::min(s.size(), len - 1);
        std::memcpy(buf, s.data(), k);
        buf[k] = 0;
        return MMB_OK;
    });
}

int mmb_device_bytes(mmb_ctx* ctx, size_t* out) {
    if (!ctx || !out) return bad("mmb_device_bytes");
    *out = ctx->s->device_bytes();
    return MMB_OK;
}

} // extern "C"
