// validate.cu — the `validate` self-check suite on the device, mirroring
// run_validation (proj/src/validate.cpp:84-189): demag tensor invariants (trace, parity and
// permutation symmetry) evaluated by the device prism-sum kernel, the spectral demag path of
// libmmb against an O(N^2) direct dipolar sum computed on the device (the counterpart of
// demag_field_direct, proj/src/demag.cpp:160-190), linearity, and the cube / thin-film shape
// factors. Random fields follow random_unit_field (proj/src/validate.cpp:21-39: mt19937,
// uniform(-1, 1), reject |v| < 0.1, scale to ms), so the inputs match the reference suite's.
// No CPU arithmetic stands in for a device result: the host only draws inputs and compares.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/mmb.h"
#include "kernels.hpp"
#include "solver_base.hpp"
#include "validate.hpp"

namespace mmb {
namespace {

// H = sum_s K(t - s) M_s over every source cell, fp64 accumulation, K from the octant table
// E[6][nz][ny][nx] with the parity of the off-diagonal entries (xy odd in x and y, xz in x
// and z, yz in y and z). One thread per target cell; for the <= 16^3 validation grids.
template <typename T>
__global__ void k_demag_direct(const T* __restrict__ m, int nx, int ny, int nz,
                               const double* __restrict__ E, T* __restrict__ h) {
    const long long n = static_cast<long long>(nx) * ny * nz;
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int ti = static_cast<int>(t % nx), tj = static_cast<int>((t / nx) % ny),
              tk = static_cast<int>(t / (static_cast<long long>(nx) * ny));
    double hx = 0.0, hy = 0.0, hz = 0.0;
    for (int sk = 0; sk < nz; ++sk)
        for (int sj = 0; sj < ny; ++sj)
            for (int si = 0; si < nx; ++si) {
                const int di = ti - si, dj = tj - sj, dk = tk - sk;
                const long long o = (static_cast<long long>(abs(dk)) * ny + abs(dj)) * nx + abs(di);
                const double fx = di < 0 ? -1.0 : 1.0, fy = dj < 0 ? -1.0 : 1.0, fz = dk < 0 ? -1.0 : 1.0;
                const double kxx = E[o], kxy = fx * fy * E[n + o], kxz = fx * fz * E[2 * n + o];
                const double kyy = E[3 * n + o], kyz = fy * fz * E[4 * n + o], kzz = E[5 * n + o];
                const long long s = (static_cast<long long>(sk) * ny + sj) * nx + si;
                const double mx = m[s], my = m[n + s], mz = m[2 * n + s];
                hx += kxx * mx + kxy * my + kxz * mz;
                hy += kxy * mx + kyy * my + kyz * mz;
                hz += kxz * mx + kyz * my + kzz * mz;
            }
    h[t] = static_cast<T>(hx);
    h[n + t] = static_cast<T>(hy);
    h[2 * n + t] = static_cast<T>(hz);
}

struct Grid3 {
    int nx, ny, nz;
    double delta;
    long long n() const { return static_cast<long long>(nx) * ny * nz; }
};

template <typename T>
std::vector<T> random_unit_field(const Grid3& g, double ms, unsigned seed) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    const long long n = g.n();
    std::vector<T> m(3 * n);
    for (long long i = 0; i < n; ++i) {
        double x, y, z, norm;
        do {
            x = dist(rng);
            y = dist(rng);
            z = dist(rng);
            norm = std::sqrt(x * x + y * y + z * z);
        } while (norm < 0.1);
        m[i] = static_cast<T>(ms * x / norm);
        m[n + i] = static_cast<T>(ms * y / norm);
        m[2 * n + i] = static_cast<T>(ms * z / norm);
    }
    return m;
}

template <typename T>
double max_relative_error(const std::vector<T>& a, const std::vector<T>& b) {
    double diff = 0.0, ref = 0.0;
    for (size_t i = 0; i < a.size(); ++i) {
        diff = std::max(diff, std::abs(double(a[i]) - double(b[i])));
        ref = std::max(ref, std::abs(double(b[i])));
    }
    return ref > 0.0 ? diff / ref : diff;
}

void status(int rc) {
    if (rc != MMB_OK) throw std::runtime_error(std::string("validate: ") + mmb_last_error());
}

// Spectral demag of m through the product path (mmb_create + mmb_demag_field).
template <typename T>
std::vector<T> demag_fft(const Grid3& g, const std::vector<T>& m, double ms) {
    mmb_desc d{};
    d.nx = g.nx;
    d.ny = g.ny;
    d.nz = g.nz;
    d.delta = g.delta;
    d.a_ex = 1.0e7;
    d.ms = ms;
    d.hk = 0.0;
    d.alpha = 0.5;
    d.dt = 1e-5;
    d.init_dir[0] = 1.0;
    d.precision = sizeof(T) == 8 ? MMB_F64 : MMB_F32;
    mmb_ctx* ctx = nullptr;
    status(mmb_create(&d, nullptr, 0, &ctx));
    const long long n = g.n();
    std::vector<T> h(3 * n);
    const int rc = mmb_demag_field(ctx, m.data(), m.data() + n, m.data() + 2 * n, h.data(), h.data() + n,
                                   h.data() + 2 * n);
    mmb_free(ctx);
    status(rc);
    return h;
}

// The same field by the device direct sum over the device-computed octant.
template <typename T>
std::vector<T> demag_direct(const Grid3& g, const std::vector<T>& m) {
    const long long n = g.n();
    DevBuf<double> E;
    DevBuf<T> dm, dh;
    E.alloc(6 * n);
    dm.alloc(3 * n);
    dh.alloc(3 * n);
    launch_tensor_octant(E.p, g.nx, g.ny, g.nz, g.delta, nullptr);
    ck(cudaMemcpy(dm.p, m.data(), 3 * n * sizeof(T), cudaMemcpyHostToDevice), "copy");
    k_demag_direct<T><<<static_cast<unsigned>((n + 127) / 128), 128>>>(dm.p, g.nx, g.ny, g.nz, E.p, dh.p);
    ck(cudaGetLastError(), "k_demag_direct");
    std::vector<T> h(3 * n);
    ck(cudaMemcpy(h.data(), dh.p, 3 * n * sizeof(T), cudaMemcpyDeviceToHost), "copy");
    return h;
}

std::vector<std::array<double, 6>> entries(const std::vector<std::array<int, 3>>& off, double delta) {
    const int n = static_cast<int>(off.size());
    DevBuf<int> d_ijk;
    DevBuf<double> d_out;
    d_ijk.alloc(3 * n);
    d_out.alloc(6 * n);
    ck(cudaMemcpy(d_ijk.p, off.data(), 3 * n * sizeof(int), cudaMemcpyHostToDevice), "copy");
    launch_tensor_entries(d_ijk.p, n, delta, d_out.p, nullptr);
    std::vector<std::array<double, 6>> out(n);
    ck(cudaMemcpy(out.data(), d_out.p, 6 * n * sizeof(double), cudaMemcpyDeviceToHost), "copy");
    return out;
}

struct Reporter {
    std::vector<std::string> lines;
    bool ok = true;
    void check(const std::string& name, bool passed, const std::string& detail) {
        lines.push_back(std::string(passed ? "PASS" : "FAIL") + "  " + name + ": " + detail);
        ok = ok && passed;
    }
    void check_le(const std::string& name, double value, double bound) {
        std::ostringstream os;
        os << value << " (bound " << bound << ")";
        check(name, value <= bound, os.str());
    }
};

template <typename T>
void fft_vs_direct(Reporter& rep, const Grid3& g, double tol, const char* label) {
    const double ms = 800.0;
    const auto m = random_unit_field<T>(g, ms, 20240u + static_cast<unsigned>(g.nx));
    std::ostringstream name;
    name << "fft-vs-direct " << label << " " << g.nx << "x" << g.ny << "x" << g.nz;
    rep.check_le(name.str(), max_relative_error(demag_fft<T>(g, m, ms), demag_direct<T>(g, m)), tol);
}

} // namespace

std::string run_device_validation(bool& all_passed) {
    Reporter rep;
    // ---- tensor invariants (validate.cpp:87-130), entries from the device kernel
    {
        const auto e0 = entries({{{0, 0, 0}}}, 1.0)[0];
        rep.check_le("tensor trace at zero offset (+1)", std::abs(e0[0] + e0[3] + e0[5] + 1.0), 1e-12);
        rep.check_le("tensor kxy at zero offset", std::abs(e0[1]), 1e-12);
    }
    {
        std::mt19937 rng(7u);
        std::uniform_int_distribution<int> di(-7, 7), dk(-3, 3);
        std::vector<std::array<int, 3>> off;
        while (off.size() < 50 * 6) {
            const int I = di(rng), J = di(rng), K = dk(rng);
            if (I == 0 && J == 0 && K == 0) continue;
            // e, flip-x, flip-y, flip-z, swap x<->y, swap x<->z
            off.push_back({I, J, K});
            off.push_back({-I, J, K});
            off.push_back({I, -J, K});
            off.push_back({I, J, -K});
            off.push_back({J, I, K});
            off.push_back({K, J, I});
        }
        const auto v = entries(off, 1.0);
        double trace = 0.0, parity = 0.0, perm = 0.0;
        for (size_t s = 0; s < off.size(); s += 6) {
            const auto &e = v[s], &fi = v[s + 1], &fj = v[s + 2], &fk = v[s + 3], &pxy = v[s + 4], &pxz = v[s + 5];
            trace = std::max(trace, std::abs(e[0] + e[3] + e[5]));
            parity = std::max({parity, std::abs(fi[0] - e[0]), std::abs(fj[0] - e[0]), std::abs(fk[0] - e[0]),
                               std::abs(fi[1] + e[1]), std::abs(fj[1] + e[1]), std::abs(fk[1] - e[1]),
                               std::abs(fi[2] + e[2]), std::abs(fj[2] - e[2]), std::abs(fk[2] + e[2]),
                               std::abs(fi[4] - e[4]), std::abs(fj[4] + e[4]), std::abs(fk[4] + e[4])});
            perm = std::max({perm, std::abs(e[3] - pxy[0]), std::abs(e[5] - pxz[0])});
        }
        rep.check_le("tensor trace at 50 nonzero offsets", trace, 1e-12);
        rep.check_le("tensor parity symmetry", parity, 1e-12);
        rep.check_le("tensor permutation symmetry", perm, 1e-12);
    }

    // ---- spectral path against the device direct sum (validate.cpp:133-136), plus the
    // largest grids the O(N^2) sum is meant for (16^3)
    fft_vs_direct<double>(rep, {4, 4, 2, 1.0}, 1e-10, "f64");
    fft_vs_direct<double>(rep, {8, 8, 4, 1.0}, 1e-10, "f64");
    fft_vs_direct<double>(rep, {5, 3, 2, 1.0}, 1e-10, "f64");
    fft_vs_direct<float>(rep, {8, 8, 4, 1.0}, 1e-4, "f32");
    fft_vs_direct<double>(rep, {16, 16, 16, 1.0}, 1e-10, "f64");
    fft_vs_direct<float>(rep, {16, 16, 16, 1.0}, 1e-4, "f32");
    fft_vs_direct<double>(rep, {33, 17, 1, 3.0}, 1e-10, "f64");

    // ---- linearity (validate.cpp:139-161)
    {
        const Grid3 g{6, 5, 3, 1.0};
        const auto m1 = random_unit_field<double>(g, 1.0, 11u);
        const auto m2 = random_unit_field<double>(g, 1.0, 12u);
        const double a = 2.5, b = -0.75;
        std::vector<double> combo(m1.size());
        for (size_t i = 0; i < combo.size(); ++i) combo[i] = a * m1[i] + b * m2[i];
        const auto h1 = demag_fft<double>(g, m1, 1.0), h2 = demag_fft<double>(g, m2, 1.0);
        const auto hc = demag_fft<double>(g, combo, 1.0);
        std::vector<double> expect(hc.size());
        for (size_t i = 0; i < expect.size(); ++i) expect[i] = a * h1[i] + b * h2[i];
        rep.check_le("fft linearity", max_relative_error(hc, expect), 1e-10);
    }

    // ---- shape factors (validate.cpp:164-185)
    {
        const double ms = 800.0;
        const Grid3 cube{8, 8, 8, 1.0};
        const long long n = cube.n();
        std::vector<double> m(3 * n, 0.0);
        std::fill(m.begin(), m.begin() + n, ms);
        const auto h = demag_fft<double>(cube, m, ms);
        double sx = 0.0;
        for (long long i = 0; i < n; ++i) sx += h[i];
        const double avg = sx / static_cast<double>(n);
        rep.check_le("cube shape factor (avg Hx vs -ms/3)", std::abs(avg + ms / 3.0) / (ms / 3.0), 0.02);
    }
    {
        const double ms = 800.0;
        const Grid3 film{64, 64, 1, 1.0};
        const long long n = film.n();
        std::vector<double> m(3 * n, 0.0);
        std::fill(m.begin() + 2 * n, m.end(), ms);
        const auto h = demag_fft<double>(film, m, ms);
        const double hz = h[2 * n + 32 * film.nx + 32];
        std::ostringstream os;
        os << "Hz = " << hz << " (want within [-ms, -0.95 ms], ms = " << ms << ")";
        rep.check("thin-film central demag factor", hz >= -ms && hz <= -0.95 * ms, os.str());
    }

    std::string out;
    for (const auto& l : rep.lines) out += l + "\n";
    out += rep.ok ? "all checks passed\n" : "VALIDATION FAILED\n";
    all_passed = rep.ok;
    return out;
}

} // namespace mmb
