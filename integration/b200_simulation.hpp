// integration/b200_simulation.hpp — the reference-side binding a maintainer adds to mmsim to
// select the B200 path: a mmsim::SimulationBase (proj/include/mmsim/llg.hpp:56-73)
// implemented over the C-ABI in include/mmb.h. Header-only; compile it inside the
// reference tree (needs proj/include on the include path) and link libmmb.so.
//
// make_simulation (proj/src/llg.cpp:163-168) then gains one branch:
//     if (backend == Backend::b200) return std::make_unique<B200Simulation>(spec, precision);
// after `b200` is added to `enum class Backend` (proj/include/mmsim/backend.hpp:17) and to
// backend_from_string / to_string (proj/src/backend.cpp:10-19). MMB_BACKEND_VALUE is the
// enumerator this adapter reports (integration/b200_backend.cpp sets it to the b200 value).
//
// step() is synchronous, like the reference's (callers such as run_benchmark time it with a
// wall clock); run() streams the whole batch asynchronously and synchronises only at the
// cadence records.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "mmb.h"
#include "mmsim/errors.hpp"
#include "mmsim/llg.hpp"

#ifndef MMB_BACKEND_VALUE
#define MMB_BACKEND_VALUE (::mmsim::Backend::parallel)
#endif

namespace mmsim {

class B200Simulation final : public SimulationBase {
public:
    B200Simulation(const ProblemSpec& spec, Precision precision, int device = 0)
        : spec_(spec), precision_(precision) {
        spec_.material.validate();
        mmb_desc d{};
        d.nx = spec.grid.nx;
        d.ny = spec.grid.ny;
        d.nz = spec.grid.nz;
        d.delta = spec.grid.delta;
        d.a_ex = spec.material.a_ex;
        d.ms = spec.material.ms;
        d.hk = spec.material.hk;
        d.alpha = spec.material.alpha;
        d.dt = spec.dt;
        d.init_dir[0] = spec.initial_direction.x;
        d.init_dir[1] = spec.initial_direction.y;
        d.init_dir[2] = spec.initial_direction.z;
        d.precision = precision == Precision::f64 ? MMB_F64 : MMB_F32;
        d.device = device;
        std::vector<mmb_stage> st;
        for (const ScheduleStage& s : spec.schedule.stages()) {
            mmb_stage m{};
            m.start = s.start;
            m.end = s.end;
            m.field[0] = s.field.x;
            m.field[1] = s.field.y;
            m.field[2] = s.field.z;
            m.ramp = s.ramp ? 1 : 0;
            m.field_end[0] = s.field_end.x;
            m.field_end[1] = s.field_end.y;
            m.field_end[2] = s.field_end.z;
            m.has_alpha = s.alpha_override ? 1 : 0;
            m.alpha_override = s.alpha_override.value_or(0.0);
            st.push_back(m);
        }
        check(mmb_create(&d, st.data(), static_cast<int>(st.size()), &ctx_));
    }
    ~B200Simulation() override { mmb_free(ctx_); }
    B200Simulation(const B200Simulation&) = delete;
    B200Simulation& operator=(const B200Simulation&) = delete;

    void step() override {
        check(mmb_step(ctx_, 1));
        check(mmb_synchronize(ctx_));
    }

    std::int64_t run(const RunOptions& opts) override {
        long long done = 0;
        const double stop = opts.stop_torque ? *opts.stop_torque : -1.0;
        if (opts.sink) {
            check(mmb_run(ctx_, opts.steps, opts.cadence, stop, &B200Simulation::trampoline,
                          const_cast<TrajectorySink*>(&opts.sink), &done));
        } else {
            check(mmb_run(ctx_, opts.steps, opts.cadence, stop, nullptr, nullptr, &done));
        }
        return done;
    }

    std::int64_t step_index() const override {
        long long s = 0;
        check(mmb_step_index(ctx_, &s));
        return s;
    }
    Vec3 average_unit() const override {
        double a[3];
        check(mmb_average(ctx_, a));
        return {a[0], a[1], a[2]};
    }
    double energy() override {
        double e = 0.0;
        check(mmb_energy(ctx_, &e));
        return e;
    }
    double max_torque() override {
        double t = 0.0;
        check(mmb_max_torque(ctx_, &t));
        return t;
    }
    const ProblemSpec& spec() const override { return spec_; }
    Backend backend() const override { return MMB_BACKEND_VALUE; }
    Precision precision() const override { return precision_; }

    // Simulation<T>::magnetization() equivalents (host SoA copies).
    template <typename T>
    void get_magnetization(VectorField<T>& m) const {
        check(mmb_get_m(ctx_, m.x.data(), m.y.data(), m.z.data()));
    }
    template <typename T>
    void set_magnetization(const VectorField<T>& m) {
        check(mmb_set_m(ctx_, m.x.data(), m.y.data(), m.z.data()));
    }

private:
    static void trampoline(void* user, long long step, double mx, double my, double mz) {
        (*static_cast<TrajectorySink*>(user))(TrajectoryRecord{step, mx, my, mz});
    }
    // mmb status -> the exception types the reference's guarded() maps to the same codes
    // (proj/src/capi.cpp:31-58).
    static void check(int rc) {
        if (rc == MMB_OK) return;
        const std::string msg = mmb_last_error();
        switch (rc) {
            case MMB_ERROR_NUMERICAL: throw numerical_error(msg);
            case MMB_ERROR_CONFIG: throw config_error(msg);
            case MMB_ERROR_ARGUMENT: throw std::invalid_argument(msg);
            case MMB_ERROR_NOMEM: throw std::bad_alloc();
            default: throw std::runtime_error(msg);
        }
    }

    ProblemSpec spec_;
    Precision precision_;
    mmb_ctx* ctx_ = nullptr;
};

} // namespace mmsim
