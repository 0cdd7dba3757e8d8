// oracle/fftw_shim/fftw_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Single-threaded CPU implementation of the FFTW3 entry points the reference uses
// (proj/src/fft.cpp:18-40). The reference's FFTW is unpinned and absent from this image;
// this restates FFTW's published contract: unnormalised c2c 3-D DFT, row-major n0 x n1 x n2
// with n2 fastest, sign -1 forward / +1 backward, arbitrary lengths (the reference-native
// SP#4 grid needs 332 = 4*83 and 84 = 4*3*7).
//
// Algorithm: mixed-radix Stockham autosort per axis (radix 4 and 2, then odd factors with a
// symmetric O(p^2/4) butterfly that pairs inputs q, p-q and outputs r, p-r), twiddles
// computed in long double and rounded once, every axis processed in batches of 16
// interleaved lines (split re/im arrays) so the inner loops vectorise. Accuracy ~1e-16
// relative; pinned by the reference's own spectral_prepare / fft-vs-direct-sum unit tests
// (oracle `make check`) and by tests/test_oracle.py against numpy.fft.
#include "fftw3.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstring>
#include <vector>

namespace {

constexpr long double kTwoPi = 6.283185307179586476925286766559005768L;
constexpr int kBatch = 16;

template <typename T>
struct Pass {
    int radix = 1;
    int ns = 1;               // product of the radices before this pass
    std::vector<T> twr, twi;  // W_{ns*radix}^{m}, m in [0, ns*radix)
    std::vector<T> cr, sr;    // cos / sign*sin (2 pi m / radix), m in [0, radix)
};

template <typename T>
void unit_root(long long m, long long n, int sign, T& re, T& im) {
    const long long r = ((m % n) + n) % n;
    const long double a = kTwoPi * static_cast<long double>(r) / static_cast<long double>(n);
    re = static_cast<T>(std::cos(a));
    im = static_cast<T>(sign * std::sin(a));
}

template <typename T>
struct Axis {
    int n = 1;
    int sign = -1;
    std::vector<Pass<T>> passes;

    void init(int len, int sgn) {
        n = len;
        sign = sgn;
        passes.clear();
        int rest = len;
        std::vector<int> radices;
        while (rest % 4 == 0) { radices.push_back(4); rest /= 4; }
        while (rest % 2 == 0) { radices.push_back(2); rest /= 2; }
        for (int p = 3; rest > 1; p += 2) {
            while (rest % p == 0) { radices.push_back(p); rest /= p; }
            if (static_cast<long long>(p) * p > rest && rest > 1) { radices.push_back(rest); rest = 1; }
        }
        int ns = 1;
        for (int r : radices) {
            Pass<T> ps;
            ps.radix = r;
            ps.ns = ns;
            ps.twr.resize(static_cast<std::size_t>(ns) * r);
            ps.twi.resize(static_cast<std::size_t>(ns) * r);
            for (int m = 0; m < ns * r; ++m) unit_root<T>(m, ns * r, sign, ps.twr[m], ps.twi[m]);
            ps.cr.resize(r);
            ps.sr.resize(r);
            for (int m = 0; m < r; ++m) unit_root<T>(m, r, sign, ps.cr[m], ps.sr[m]);
            passes.push_back(std::move(ps));
            ns *= r;
        }
    }

    // Transforms B <= kBatch interleaved lines held as split arrays: element q of line b at
    // [q*kBatch + b]. Ping-pongs with the scratch arrays; the result ends in (re, im).
    void run(T* re, T* im, T* tre, T* tim, int B) const {
        if (n == 1) return;
        T *ir = re, *ii = im, *orr = tre, *oi = tim;
        std::vector<T> vr, vi;
        for (const Pass<T>& ps : passes) {
            const int R = ps.radix, Ns = ps.ns, stride = n / R;
            vr.assign(static_cast<std::size_t>(R) * kBatch, T(0));
            vi.assign(static_cast<std::size_t>(R) * kBatch, T(0));
            for (int j = 0; j < stride; ++j) {
                const int k = j % Ns;
                const int dst = (j / Ns) * Ns * R + k;
                for (int q = 0; q < R; ++q) {
                    const T wr = ps.twr[static_cast<std::size_t>(q) * k];
                    const T wi = ps.twi[static_cast<std::size_t>(q) * k];
                    const T* sr = ir + static_cast<std::size_t>(j + q * stride) * kBatch;
                    const T* si = ii + static_cast<std::size_t>(j + q * stride) * kBatch;
                    T* dr = vr.data() + q * kBatch;
                    T* di = vi.data() + q * kBatch;
                    for (int b = 0; b < B; ++b) {
                        dr[b] = sr[b] * wr - si[b] * wi;
                        di[b] = sr[b] * wi + si[b] * wr;
                    }
                }
                auto out_r = [&](int r) { return orr + static_cast<std::size_t>(dst + r * Ns) * kBatch; };
                auto out_i = [&](int r) { return oi + static_cast<std::size_t>(dst + r * Ns) * kBatch; };
                if (R == 2) {
                    T *o0r = out_r(0), *o0i = out_i(0), *o1r = out_r(1), *o1i = out_i(1);
                    for (int b = 0; b < B; ++b) {
                        const T ar = vr[b], ai = vi[b], br = vr[kBatch + b], bi = vi[kBatch + b];
                        o0r[b] = ar + br;
                        o0i[b] = ai + bi;
                        o1r[b] = ar - br;
                        o1i[b] = ai - bi;
                    }
                } else if (R == 4) {
                    const T s = static_cast<T>(sign);
                    T *o0r = out_r(0), *o0i = out_i(0), *o1r = out_r(1), *o1i = out_i(1);
                    T *o2r = out_r(2), *o2i = out_i(2), *o3r = out_r(3), *o3i = out_i(3);
                    for (int b = 0; b < B; ++b) {
                        const T x0r = vr[b], x0i = vi[b];
                        const T x1r = vr[kBatch + b], x1i = vi[kBatch + b];
                        const T x2r = vr[2 * kBatch + b], x2i = vi[2 * kBatch + b];
                        const T x3r = vr[3 * kBatch + b], x3i = vi[3 * kBatch + b];
                        const T a0r = x0r + x2r, a0i = x0i + x2i, a1r = x0r - x2r, a1i = x0i - x2i;
                        const T a2r = x1r + x3r, a2i = x1i + x3i, dr = x1r - x3r, di = x1i - x3i;
                        const T a3r = -s * di, a3i = s * dr; // sign * i * d
                        o0r[b] = a0r + a2r;
                        o0i[b] = a0i + a2i;
                        o1r[b] = a1r + a3r;
                        o1i[b] = a1i + a3i;
                        o2r[b] = a0r - a2r;
                        o2i[b] = a0i - a2i;
                        o3r[b] = a1r - a3r;
                        o3i[b] = a1i - a3i;
                    }
                } else {
                    // Odd radix: X[r] = x0 + sum_{q<=h} [(x_q + x_{R-q}) c_qr + (x_q - x_{R-q}) i s_qr],
                    // X[R-r] differs only in the sign of the sine part.
                    const int h = (R - 1) / 2;
                    T spr[kBatch], spi[kBatch], smr[kBatch], smi[kBatch];
                    T x0r[kBatch], x0i[kBatch];
                    for (int b = 0; b < B; ++b) {
                        x0r[b] = vr[b];
                        x0i[b] = vi[b];
                    }
                    // DC
                    {
                        T* o = out_r(0);
                        T* oo = out_i(0);
                        for (int b = 0; b < B; ++b) { o[b] = x0r[b]; oo[b] = x0i[b]; }
                        for (int q = 1; q < R; ++q)
                            for (int b = 0; b < B; ++b) {
                                o[b] += vr[q * kBatch + b];
                                oo[b] += vi[q * kBatch + b];
                            }
                    }
                    for (int r = 1; r <= h; ++r) {
                        T ar[kBatch], ai[kBatch], br[kBatch], bi[kBatch];
                        for (int b = 0; b < B; ++b) {
                            ar[b] = x0r[b];
                            ai[b] = x0i[b];
                            br[b] = 0;
                            bi[b] = 0;
                        }
                        int idx = 0;
                        for (int q = 1; q <= h; ++q) {
                            idx += r;
                            if (idx >= R) idx -= R;
                            const T c = ps.cr[idx], s = ps.sr[idx];
                            const T* pr = vr.data() + q * kBatch;
                            const T* pi = vi.data() + q * kBatch;
                            const T* mr = vr.data() + (R - q) * kBatch;
                            const T* mi = vi.data() + (R - q) * kBatch;
                            for (int b = 0; b < B; ++b) {
                                spr[b] = pr[b] + mr[b];
                                spi[b] = pi[b] + mi[b];
                                smr[b] = pr[b] - mr[b];
                                smi[b] = pi[b] - mi[b];
                                ar[b] += spr[b] * c;
                                ai[b] += spi[b] * c;
                                // i*s*(smr + i smi) = (-s smi, s smr)
                                br[b] -= smi[b] * s;
                                bi[b] += smr[b] * s;
                            }
                        }
                        T *o1r = out_r(r), *o1i = out_i(r), *o2r = out_r(R - r), *o2i = out_i(R - r);
                        for (int b = 0; b < B; ++b) {
                            o1r[b] = ar[b] + br[b];
                            o1i[b] = ai[b] + bi[b];
                            o2r[b] = ar[b] - br[b];
                            o2i[b] = ai[b] - bi[b];
                        }
                    }
                }
            }
            std::swap(ir, orr);
            std::swap(ii, oi);
        }
        if (ir != re) {
            std::memcpy(re, ir, sizeof(T) * static_cast<std::size_t>(n) * kBatch);
            std::memcpy(im, ii, sizeof(T) * static_cast<std::size_t>(n) * kBatch);
        }
    }
};

template <typename T>
struct Plan3 {
    int n[3] = {1, 1, 1};
    Axis<T> axis[3];

    void transform(std::complex<T>* data) const {
        const std::size_t n0 = n[0], n1 = n[1], n2 = n[2];
        // Per axis: length, element stride, line count, and line offset function.
        for (int a = 2; a >= 0; --a) {
            const std::size_t len = n[a];
            if (len == 1) continue;
            const std::size_t stride = (a == 2) ? 1 : (a == 1 ? n2 : n1 * n2);
            const std::size_t lines = (n0 * n1 * n2) / len;
            auto line_off = [&](std::size_t l) -> std::size_t {
                if (a == 2) return l * n2;
                if (a == 1) return (l / n2) * n1 * n2 + (l % n2);
                return l;
            };
            std::vector<T> re(len * kBatch), im(len * kBatch), tre(len * kBatch), tim(len * kBatch);
            for (std::size_t l0 = 0; l0 < lines; l0 += kBatch) {
                const int B = static_cast<int>(std::min<std::size_t>(kBatch, lines - l0));
                std::size_t off[kBatch];
                for (int b = 0; b < B; ++b) off[b] = line_off(l0 + b);
                for (std::size_t q = 0; q < len; ++q)
                    for (int b = 0; b < B; ++b) {
                        const std::complex<T> v = data[off[b] + q * stride];
                        re[q * kBatch + b] = v.real();
                        im[q * kBatch + b] = v.imag();
                    }
                axis[a].run(re.data(), im.data(), tre.data(), tim.data(), B);
                for (std::size_t q = 0; q < len; ++q)
                    for (int b = 0; b < B; ++b)
                        data[off[b] + q * stride] = std::complex<T>(re[q * kBatch + b], im[q * kBatch + b]);
            }
        }
    }
};

template <typename T>
Plan3<T>* make_plan(int n0, int n1, int n2, int sign) {
    if (n0 < 1 || n1 < 1 || n2 < 1 || (sign != -1 && sign != 1)) return nullptr;
    auto* p = new Plan3<T>();
    p->n[0] = n0;
    p->n[1] = n1;
    p->n[2] = n2;
    p->axis[0].init(n0, sign);
    p->axis[1].init(n1, sign);
    p->axis[2].init(n2, sign);
    return p;
}

template <typename T>
void execute(const Plan3<T>* p, std::complex<T>* in, std::complex<T>* out) {
    const std::size_t count = static_cast<std::size_t>(p->n[0]) * p->n[1] * p->n[2];
    if (in != out) std::memcpy(out, in, sizeof(std::complex<T>) * count);
    p->transform(out);
}

} // namespace

struct mmb_shim_plan_d : Plan3<double> {};
struct mmb_shim_plan_f : Plan3<float> {};

extern "C" {

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex*, fftw_complex*, int sign,
                           unsigned) {
    Plan3<double>* p = make_plan<double>(n0, n1, n2, sign);
    return static_cast<fftw_plan>(static_cast<void*>(p));
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    execute(static_cast<const Plan3<double>*>(static_cast<const void*>(p)),
            reinterpret_cast<std::complex<double>*>(in),
            reinterpret_cast<std::complex<double>*>(out));
}

void fftw_destroy_plan(fftw_plan p) { delete static_cast<Plan3<double>*>(static_cast<void*>(p)); }

fftwf_plan fftwf_plan_dft_3d(int n0, int n1, int n2, fftwf_complex*, fftwf_complex*, int sign,
                             unsigned) {
    Plan3<float>* p = make_plan<float>(n0, n1, n2, sign);
    return static_cast<fftwf_plan>(static_cast<void*>(p));
}

void fftwf_execute_dft(const fftwf_plan p, fftwf_complex* in, fftwf_complex* out) {
    execute(static_cast<const Plan3<float>*>(static_cast<const void*>(p)),
            reinterpret_cast<std::complex<float>*>(in),
            reinterpret_cast<std::complex<float>*>(out));
}

void fftwf_destroy_plan(fftwf_plan p) { delete static_cast<Plan3<float>*>(static_cast<void*>(p)); }

} // extern "C"
