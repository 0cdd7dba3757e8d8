"""CPU tests: pin the oracle before trusting it.

* the reference itself (compiled in place with the FFTW shim, oracle/_ref) passes its own
  unit-test suite (proj/tests/*.cpp through oracle/doctest_mini);
* the NumPy restatement (oracle/mmsim_oracle.py) reproduces the compiled reference on the
  same seeded inputs: local terms bitwise, demag to FFT round-off, whole steps;
* both reproduce the committed golden vectors (tests/golden/, made by make_golden.py) and
  the reference's known-answer cases (tensor self term, hand Euler step, Neumann line).
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import mmsim_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _cases():
    d = np.load(os.path.join(GOLD, "fields_small.npz"))
    for idx, row in enumerate(d["cases"]):
        nx, ny, nz = int(row[0]), int(row[1]), int(row[2])
        delta, a_ex, ms, hk, alpha = row[3:8]
        applied = tuple(row[8:11])
        yield idx, (nx, ny, nz, delta, a_ex, ms, hk, alpha, applied), d


def test_reference_unit_suite_passes_with_shim():
    exe = os.path.join(os.path.dirname(HERE), "oracle", "_ref", "mmsim_ref_tests")
    if not os.path.exists(exe):
        pytest.skip("reference test binary not built (needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, cwd=os.path.dirname(exe), timeout=600)
    assert r.returncode == 0, r.stdout[-2000:]
    assert "0 failed" in r.stdout


def test_tensor_known_answers():
    # proj/tests/test_demag_tensor.cpp:54-69: self term -1/3 diagonal, zero off-diagonal
    for delta in (1.0, 3.0):
        xx, xy, xz, yy, yz, zz = (float(v) for v in O.tensor_entry(0, 0, 0, delta))
        for v in (xx, yy, zz):
            assert abs(v + 1.0 / 3.0) <= 1e-12
        for v in (xy, xz, yz):
            assert abs(v) <= 1e-12
    # traceless far field (:71-77)
    e = [float(v) for v in O.tensor_entry(3, 1, 2, 1.0)]
    assert abs(e[0] + e[3] + e[5]) <= 1e-12


def test_tensor_matches_reference(refsolver):
    rng = np.random.default_rng(99)
    for _ in range(40):
        I, J, K = (int(v) for v in rng.integers(-9, 10, 3))
        a = refsolver.tensor_entry(I, J, K, 2.5)
        b = [float(v) for v in O.tensor_entry(I, J, K, 2.5)]
        assert np.max(np.abs(np.array(a) - np.array(b))) <= 1e-13
    t_ref = refsolver.build_tensor(4, 3, 2, 1.5)
    t_np = O.build_tensor(O.Grid(4, 3, 2, 1.5))
    assert np.max(np.abs(t_ref - t_np)) <= 1e-13


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_restatement_matches_reference_fields(refsolver, prec):
    dt = np.float64 if prec == "f64" else np.float32
    for idx, (nx, ny, nz, delta, a_ex, ms, hk, alpha, applied), d in _cases():
        g = O.Grid(nx, ny, nz, delta)
        mat = O.Material(a_ex, ms, hk, alpha)
        m = d[f"c{idx}_{prec}_m0"]
        P = refsolver.Problem(nx, ny, nz, delta, a_ex, ms, hk, alpha, 5e-6)
        # local terms: bitwise
        h_loc = np.zeros_like(m)
        O.add_exchange_field(m, mat, g, h_loc)
        O.add_anisotropy_field(m, mat, h_loc)
        O.add_uniform_field(applied, h_loc)
        assert np.array_equal(h_loc, refsolver.heff(P, m, applied, parts=14))
        # full H_eff vs golden (made by the reference)
        h = O.effective_field(m, mat, g, applied)
        tol = 1e-13 if prec == "f64" else 1e-6
        assert O.max_relative_error(h, d[f"c{idx}_{prec}_heff"]) <= tol, (idx, prec)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_restatement_steps_match_golden(prec):
    dt = np.float64 if prec == "f64" else np.float32
    for idx, (nx, ny, nz, delta, a_ex, ms, hk, alpha, applied), d in _cases():
        sim = O.Simulation(O.Grid(nx, ny, nz, delta), O.Material(a_ex, ms, hk, alpha), 5e-6,
                           [O.Stage(0, 1_000_000, applied)], dtype=dt)
        sim.m = d[f"c{idx}_{prec}_m0"].copy()
        for _ in range(10):
            sim.step()
        tol = 1e-12 if prec == "f64" else 1e-5
        assert O.max_relative_error(sim.m, d[f"c{idx}_{prec}_m10"]) <= tol, (idx, prec)
        assert np.max(np.abs(np.array(sim.average_unit()) - d[f"c{idx}_{prec}_avg10"])) <= tol


def test_restatement_direct_sum_equals_fft():
    # proj/tests/test_demag_field.cpp:150-162 (1e-10 f64) on the restatement itself
    seed = 1000
    for shp, delta in [((2, 2, 2), 1.0), ((3, 3, 3), 2.0), ((4, 4, 2), 1.0), ((5, 3, 2), 3.0),
                       ((7, 1, 1), 1.0), ((1, 6, 2), 1.0), ((8, 8, 4), 1.0)]:
        g = O.Grid(*shp, delta)
        rng = np.random.default_rng(seed)
        seed += 1
        m = rng.uniform(-800, 800, (3,) + g.shape)
        assert O.max_relative_error(O.demag_field_fft(m, g), O.demag_field_direct(m, g)) <= 1e-10


def test_hand_euler_step():
    # proj/tests/test_llg.cpp:76-95
    ms, h, dt, alpha = 800.0, 40.0, 2e-5, 0.5
    sim = O.Simulation(O.Grid(1, 1, 1, 1.0), O.Material(0.0, ms, 0.0, alpha), dt,
                       [O.Stage(0, 1_000_000, (ms / 3.0, 0.0, h))])
    sim.step()
    p1, p2 = O.integrator_params(dt, alpha, ms)
    vy, vz = p1 * (-ms * h), p2 * (-ms * ms * h)
    norm = np.sqrt(ms * ms + vy * vy + vz * vz)
    got = sim.m.ravel()
    np.testing.assert_allclose(got, [ms * ms / norm, ms * vy / norm, ms * vz / norm], rtol=1e-12)


def test_exchange_neumann_line():
    # proj/tests/test_local_fields.cpp:46-65
    g = O.Grid(3, 1, 1, 2.0)
    mat = O.Material(1.3e7, 800.0, 0.0, 0.5)
    m = np.zeros((3, 1, 1, 3))
    m[0, 0, 0, 1] = 13.5
    h = np.zeros_like(m)
    O.add_exchange_field(m, mat, g, h)
    c = mat.exchange_coefficient(2.0)
    np.testing.assert_allclose(h[0].ravel(), [c * 13.5, -2 * c * 13.5, c * 13.5], rtol=1e-14)


def test_sp4_fixture_and_schedule():
    # proj/tests/test_local_fields.cpp:141-170
    g, mat, dt, stages, steps, cad = O.standard_problem_4()
    assert O.schedule_at(stages, 1000) == ((100.0, 100.0, 100.0), None)
    f, a = O.schedule_at(stages, 5000)
    assert abs(f[0] - 50.0) < 1e-12 and a is None
    f, a = O.schedule_at(stages, 60000)
    assert f == (-19.576, 3.422, 0.0) and a == 0.02
    assert O.schedule_at(stages, 6000)[0][0] == 0.0
    rows = np.loadtxt(os.path.join(GOLD, "sp4_field1_reference.tsv"))
    assert rows.shape == (150, 4) and rows[0, 0] == 1000 and rows[-1, 0] == 150000
