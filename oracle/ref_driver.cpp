// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (links the reference build; never the product).
//
// A small C surface over the reference's C++ API so the Python parity tests and bench.py's
// CPU arm can drive the UNMODIFIED reference code (compiled in place from
// /root/reference/proj/src with the FFTW shim) through ctypes. The reference's own C FFI
// (proj/include/mmsim.h) has no set/get-M or field hooks, so this wraps the C++ classes the
// reference tests use directly:
//   Simulation<T> + magnetization()      proj/include/mmsim/llg.hpp:78-115
//   demag_field_fft / demag_field_direct proj/src/demag.cpp:149-190
//   add_exchange/anisotropy/uniform      proj/src/local_fields.cpp:5-42, local_fields.hpp:25-55
//   demag_tensor_entry / build tensor    proj/src/demag_tensor.cpp:9-82
//   random_unit_field (validate.cpp:21-39, copied generator contract: mt19937 + U(-1,1))
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>

#include "mmsim/demag.hpp"
#include "mmsim/demag_tensor.hpp"
#include "mmsim/errors.hpp"
#include "mmsim/llg.hpp"
#include "mmsim/local_fields.hpp"
#include "mmsim/problems.hpp"

using namespace mmsim;

namespace {

thread_local std::string g_err;

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const numerical_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

struct RefSim {
    int precision = 1; // 0 = f32, 1 = f64
    std::unique_ptr<SimulationBase> sim;
};

template <typename T>
VectorField<T>& mag(RefSim* s) {
    return static_cast<Simulation<T>*>(s->sim.get())->magnetization();
}

template <typename T>
void copy_in(VectorField<T>& f, const void* x, const void* y, const void* z) {
    const std::size_t n = f.size();
    std::memcpy(f.x.data(), x, n * sizeof(T));
    std::memcpy(f.y.data(), y, n * sizeof(T));
    std::memcpy(f.z.data(), z, n * sizeof(T));
}

template <typename T>
void copy_out(const VectorField<T>& f, void* x, void* y, void* z) {
    const std::size_t n = f.size();
    std::memcpy(x, f.x.data(), n * sizeof(T));
    std::memcpy(y, f.y.data(), n * sizeof(T));
    std::memcpy(z, f.z.data(), n * sizeof(T));
}

} // namespace

// Flat problem description shared with the Python side (oracle/ref.py mirrors it).
struct ref_problem {
    int nx, ny, nz;
    double delta;
    double a_ex, ms, hk, alpha;
    double dt;
    double init_x, init_y, init_z;
    int nstages;
    const long long* start;
    const long long* end;
    const double* field;     // 3 per stage
    const int* ramp;
    const double* field_end; // 3 per stage
    const int* has_alpha;
    const double* alpha_override;
};

ProblemSpec to_spec(const ref_problem* p) {
    ProblemSpec s;
    s.name = "custom";
    s.grid = Grid(p->nx, p->ny, p->nz, p->delta);
    s.material.a_ex = p->a_ex;
    s.material.ms = p->ms;
    s.material.hk = p->hk;
    s.material.alpha = p->alpha;
    s.initial_direction = {p->init_x, p->init_y, p->init_z};
    s.dt = p->dt;
    std::vector<ScheduleStage> stages;
    for (int i = 0; i < p->nstages; ++i) {
        ScheduleStage st;
        st.start = p->start[i];
        st.end = p->end[i];
        st.field = {p->field[3 * i], p->field[3 * i + 1], p->field[3 * i + 2]};
        st.ramp = p->ramp[i] != 0;
        st.field_end = {p->field_end[3 * i], p->field_end[3 * i + 1], p->field_end[3 * i + 2]};
        if (p->has_alpha[i]) st.alpha_override = p->alpha_override[i];
        stages.push_back(st);
    }
    s.schedule = FieldSchedule(stages);
    return s;
}

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_sim_create(const ref_problem* p, int precision, int backend, void** out) {
    *out = nullptr;
    return guard([&] {
        auto s = std::make_unique<RefSim>();
        s->precision = precision;
        s->sim = make_simulation(to_spec(p), backend ? Backend::parallel : Backend::serial,
                                 precision ? Precision::f64 : Precision::f32);
        *out = s.release();
    });
}

void ref_sim_free(void* h) { delete static_cast<RefSim*>(h); }

int ref_sim_set_m(void* h, const void* x, const void* y, const void* z) {
    auto* s = static_cast<RefSim*>(h);
    return guard([&] {
        if (s->precision) copy_in(mag<double>(s), x, y, z);
        else copy_in(mag<float>(s), x, y, z);
    });
}

int ref_sim_get_m(void* h, void* x, void* y, void* z) {
    auto* s = static_cast<RefSim*>(h);
    return guard([&] {
        if (s->precision) copy_out(mag<double>(s), x, y, z);
        else copy_out(mag<float>(s), x, y, z);
    });
}

int ref_sim_step(void* h, long long n) {
    auto* s = static_cast<RefSim*>(h);
    return guard([&] { for (long long i = 0; i < n; ++i) s->sim->step(); });
}

long long ref_sim_step_index(void* h) { return static_cast<RefSim*>(h)->sim->step_index(); }

int ref_sim_average(void* h, double* out) {
    auto* s = static_cast<RefSim*>(h);
    return guard([&] {
        const Vec3 a = s->sim->average_unit();
        out[0] = a.x;
        out[1] = a.y;
        out[2] = a.z;
    });
}

int ref_sim_energy(void* h, double* out) {
    auto* s = static_cast<RefSim*>(h);
    return guard([&] { *out = s->sim->energy(); });
}

int ref_sim_max_torque(void* h, double* out) {
    auto* s = static_cast<RefSim*>(h);
    return guard([&] { *out = s->sim->max_torque(); });
}

typedef void (*ref_record_fn)(void* user, long long step, double mx, double my, double mz);

int ref_sim_run(void* h, long long steps, long long cadence, double stop_torque,
                ref_record_fn record, void* user, long long* done) {
    auto* s = static_cast<RefSim*>(h);
    return guard([&] {
        RunOptions opts;
        opts.steps = steps;
        opts.cadence = cadence;
        if (stop_torque >= 0.0) opts.stop_torque = stop_torque;
        if (record)
            opts.sink = [record, user](const TrajectoryRecord& r) {
                record(user, r.step, r.mx, r.my, r.mz);
            };
        const long long d = s->sim->run(opts);
        if (done) *done = d;
    });
}

} // extern "C"

// H_eff exactly as Simulation<T>::assemble_effective_field builds it (llg.cpp:52-55):
// demag, += exchange, += anisotropy, += applied. `parts` selects terms (bit0 demag,
// bit1 exchange, bit2 anisotropy, bit3 applied) so tests can isolate each one.
template <typename T>
static void heff_impl(const ref_problem* p, const double* applied, int parts, const void* mx,
                      const void* my, const void* mz, void* hx, void* hy, void* hz) {
    const ProblemSpec spec = to_spec(p);
    VectorField<T> m(spec.grid), h(spec.grid);
    copy_in(m, mx, my, mz);
    if (parts & 1) {
        const auto spectral = spectral_prepare(build_demag_tensor<T>(spec.grid));
        h = demag_field_fft(m, spectral);
    }
    if (parts & 2) add_exchange_field(m, spec.material, spec.grid, Backend::serial, h);
    if (parts & 4) add_anisotropy_field(m, spec.material, Backend::serial, h);
    if (parts & 8) add_uniform_field(Vec3{applied[0], applied[1], applied[2]}, Backend::serial, h);
    copy_out(h, hx, hy, hz);
}

extern "C" {

int ref_heff(const ref_problem* p, int precision, const double* applied, int parts,
             const void* mx, const void* my, const void* mz, void* hx, void* hy, void* hz) {
    return guard([&] {
        if (precision) heff_impl<double>(p, applied, parts, mx, my, mz, hx, hy, hz);
        else heff_impl<float>(p, applied, parts, mx, my, mz, hx, hy, hz);
    });
}

// O(N^2) direct dipolar sum (demag.cpp:160-190), f64.
int ref_demag_direct(const ref_problem* p, const double* mx, const double* my, const double* mz,
                     double* hx, double* hy, double* hz) {
    return guard([&] {
        const ProblemSpec spec = to_spec(p);
        VectorField<double> m(spec.grid);
        copy_in(m, mx, my, mz);
        const auto t = build_demag_tensor<double>(spec.grid);
        const auto h = demag_field_direct(m, t);
        copy_out(h, hx, hy, hz);
    });
}

int ref_tensor_entry(int I, int J, int K, double delta, double* out6) {
    return guard([&] {
        const TensorEntry e = demag_tensor_entry(I, J, K, delta);
        out6[0] = e.xx;
        out6[1] = e.xy;
        out6[2] = e.xz;
        out6[3] = e.yy;
        out6[4] = e.yz;
        out6[5] = e.zz;
    });
}

// Shifted-storage tensor on the doubled grid (demag_tensor.cpp:45-82), f64, 6 arrays of
// 2nx*2ny*2nz in the order xx, xy, xz, yy, yz, zz.
int ref_build_tensor(int nx, int ny, int nz, double delta, double* out) {
    return guard([&] {
        const auto t = build_demag_tensor<double>(Grid(nx, ny, nz, delta));
        const std::size_t c = t.doubled_count();
        const std::vector<double>* comps[6] = {&t.kxx, &t.kxy, &t.kxz, &t.kyy, &t.kyz, &t.kzz};
        for (int i = 0; i < 6; ++i) std::memcpy(out + i * c, comps[i]->data(), c * sizeof(double));
    });
}

// The reference's seeded random start (validate.cpp:21-39; same in the tests), f64 output.
void ref_random_unit_field(long long n, double ms, unsigned seed, double* x, double* y, double* z) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (long long i = 0; i < n; ++i) {
        double a, b, c, norm;
        do {
            a = dist(rng);
            b = dist(rng);
            c = dist(rng);
            norm = std::sqrt(a * a + b * b + c * c);
        } while (norm < 0.1);
        x[i] = ms * a / norm;
        y[i] = ms * b / norm;
        z[i] = ms * c / norm;
    }
}

} // extern "C"
