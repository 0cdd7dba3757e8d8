// Compile-and-link check of the reference-side adapter against the reference headers and
// libmmb.so (built by tests/test_capi.py when /root/reference is present). Run on a GPU box
// it also steps a small problem through mmsim::SimulationBase.
#include <cstdio>
#include <memory>

#include "b200_simulation.hpp"
#include "mmsim/problems.hpp"

int main() {
    try {
        mmsim::ProblemSpec spec = mmsim::standard_problem_3_benchmark(8);
        std::unique_ptr<mmsim::SimulationBase> sim =
            std::make_unique<mmsim::B200Simulation>(spec, mmsim::Precision::f64);
        mmsim::RunOptions opts;
        opts.steps = 10;
        opts.cadence = 5;
        int records = 0;
        opts.sink = [&](const mmsim::TrajectoryRecord&) { ++records; };
        const auto done = sim->run(opts);
        const mmsim::Vec3 a = sim->average_unit();
        std::printf("steps %lld records %d <m> %.6f %.6f %.6f\n", static_cast<long long>(done),
                    records, a.x, a.y, a.z);
        return (done == 10 && records == 2) ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("adapter: %s\n", e.what());
        return 2;
    }
}
