"""GPU parity of the PRODUCTION kernel variants against the compiled reference (oracle/_ref).

Every BASELINE config runs a kernel variant chosen by its geometry (the x-tile height and
thread shape of k_xstep, the lane-pair DFT_64 stages at L >= 2048, the y/z kernel of the
padded length). Each case below is the benchmarked grid itself or a reduced grid that forces
the same variant; the test first asserts the variant (mmb_path_info), then compares with the
reference `Simulation<T>` (proj/src/llg.cpp:58-108, proj/src/demag.cpp:53-147,
proj/src/local_fields.cpp:5-42, proj/include/mmsim/vector_field.hpp:56-83) started from the
reference generator's random state (proj/src/validate.cpp:21-39):

* H_demag of that state (north-star gate: <= 1e-12 f64 / 1e-5 f32, reference metric
  max|a-b|/max|b|, proj/src/validate.cpp:41-53);
* the first step's update dM = M_1 - M_0 through the fused x-inverse + local terms + Euler +
  renormalise + x-forward kernel. dM is ~1e-1 of |M|, so this isolates the fused update from
  the state both sides share: its error is the H_eff error of the step, not the f32 rounding of
  M itself;
* M, <m> and max_torque after three steps, through a schedule that ramps the field and sets
  the sticky damping override at step 2;
* H_eff re-assembled at the reference's state after the steps.

Film relaxation (BASELINE configs[1]): 20 000 steps from the reference generator's random
state at cadence 100, <m>(t) against trajectories produced by the compiled reference
(tests/golden/make_golden.py film). Acceptance criterion 6 (proj/tests/acceptance.cpp:307-336)
runs on the B200 path with its energies compared to the reference's.
"""
import json
import os

import numpy as np
import pytest

from paper_1501_07293_b200 import RunOptions

from .helpers import b200, ref_problem, rel, spec

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
OUT = os.path.join(os.path.dirname(HERE), "gpurun_out")

# north-star field gate, and the gates of the step comparisons (measured on B200: see
# profiles/parity_production_r2.json for the observed values of every case)
TOL_H = {"f64": 1e-12, "f32": 1e-5}
# dM in f32 carries the rounding of M itself (ulp(ms) ~ 6e-5 at ms = 800-1000 against |dM| of
# a few ms): observed up to 1.5e-5 (256^2 film), 3.3e-6 elsewhere
TOL_DM = {"f64": 1e-11, "f32": 1e-4}
TOL_M3 = {"f64": 1e-12, "f32": 2e-6}

SCHED = [(0, 2, (10.0, -20.0, 5.0)), (2, 10, (0.0, 50.0, 0.0), True, (40.0, 0.0, 0.0), 0.1)]

# id: (nx, ny, nz, delta, a_ex, ms, hk, alpha, dt), precision, substrings of path_info
CASES = {
    # BASELINE configs[2], the headline: 3 x 14-row x tile at one CTA per SM, last y tile partial
    "512x512x8_f32": ((512, 512, 8, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5), "f32",
                      ["path=yz", "k_yz<L10,ZM1>", "k_xstep<L10,PB224> tr=14"]),
    # BASELINE configs[1]: Ly = 512 y/z kernel, small x tile
    "film256_f32": ((256, 256, 1, 3.0, 1.3e7, 800.0, 0.0, 0.5, 5e-6), "f32", ["path=yz", "k_yz<L9,ZM0>"]),
    "film256_f64": ((256, 256, 1, 3.0, 1.3e7, 800.0, 0.0, 0.5, 5e-6), "f64", ["path=yz", "k_yz<L9,ZM0>"]),
    # the PB = 128 x tile (3 x 8 rows) at Lx = 512
    "pb128_200x300x8_f32": ((200, 300, 8, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5), "f32",
                            ["path=yz", "k_xstep<L9,PB128> tr=8"]),
    # Lx = 2048 WIDE x tile (one DFT_64 task per thread, stage B in two rounds)
    "wide_600x300x8_f32": ((600, 300, 8, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5), "f32",
                           ["path=yz", "k_xstep<L11,PB128>", "wide"]),
    # Lx = 2048 small-grid x tile on lane pairs (dft_pair)
    "pair_700x20x1_f32": ((700, 20, 1, 2.0, 1.3e7, 800.0, 30.0, 0.5, 5e-6), "f32",
                          ["path=yz", "k_xstep<L11,PB16>", "pair"]),
    "pair_700x20x1_f64": ((700, 20, 1, 2.0, 1.3e7, 800.0, 30.0, 0.5, 5e-6), "f64",
                          ["path=yz", "k_xstep<L11,PB16>", "pair"]),
    # streaming y/z path (configs[3] and [4]): Ly = 2048 / 4096 y rows on lane pairs
    "yrow2048_40x600x9_f32": ((40, 600, 9, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5), "f32",
                              ["path=big", "k_yrow<L11> pair"]),
    "yrow4096_24x1100x9_f32": ((24, 1100, 9, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5), "f32",
                               ["path=big", "k_yrow<L12> pair"]),
    # Lx = 4096 x tiles (configs[4] on one GPU), small grid and >= 296-tile grid
    "x4096_1100x24x9_f32": ((1100, 24, 9, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5), "f32",
                            ["path=big", "k_xstep<L12,PB16>", "pair"]),
    "x4096_1100x24x25_f32": ((1100, 24, 25, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5), "f32",
                             ["path=big", "k_xstep<L12,PB128>", "pair"]),
    # Lx = 2048 WIDE tile behind the streaming y/z path (configs[3] x side), and f64 big path
    "bigwide_1024x300x12_f32": ((1024, 300, 12, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5), "f32",
                                ["path=big", "k_xstep<L11,PB128>", "wide"]),
    "big_f64_100x300x12": ((100, 300, 12, 1.0, 1.3e7, 800.0, 30.0, 0.5, 5e-6), "f64",
                           ["path=big", "k_yrow<L10>"]),
}

_observed = {}


@pytest.fixture(scope="module", autouse=True)
def _record_observed():
    yield
    if _observed:
        os.makedirs(OUT, exist_ok=True)
        path = os.path.join(OUT, "parity_production.json")
        old = {}
        if os.path.exists(path):
            with open(path) as f:
                old = json.load(f)
        old.update(_observed)
        with open(path, "w") as f:
            json.dump(old, f, indent=1, sort_keys=True)


def _spec(p, stages=()):
    nx, ny, nz, delta, a_ex, ms, hk, alpha, dt = p
    return spec(nx, ny, nz, delta, a_ex, ms, hk, alpha, dt, list(stages))


@pytest.mark.parametrize("case", list(CASES))
def test_production_variant_matches_reference(refsolver, case, monkeypatch):
    for v in ("MMB_GENERAL_PATH", "MMB_BIG_PATH"):
        monkeypatch.delenv(v, raising=False)
    p, prec, want_path = CASES[case]
    nx, ny, nz, delta, a_ex, ms = p[:6]
    dt = np.float64 if prec == "f64" else np.float32
    sp = _spec(p, SCHED)
    sim = b200(sp, prec)
    info = sim.path_info()
    for w in want_path:
        assert w in info, f"{case}: expected variant {w!r} in {info!r}"
    big = nx * ny * nz >= 100_000
    r = refsolver.RefSimulation(ref_problem(refsolver, sp), prec, backend="parallel" if big else "serial")
    m0 = refsolver.random_unit_field(nx, ny, nz, ms, 20240 + nx, dt)
    obs = {"path": info}

    # H_demag of the random state (the y/z kernel of this geometry)
    h_ref = refsolver.heff(ref_problem(refsolver, sp), m0, parts=1)
    h_b = sim.demag_field(m0)
    obs["h_demag"] = rel(h_b, h_ref)
    if prec == "f64":
        # The reference evaluates the prism sums at negative offsets separately, so its tensor
        # is symmetric only up to the far-field cancellation error of each entry; on grids of
        # 1e5+ cells that asymmetry alone moves its field by up to ~1e-10 relative (8.4e-11 at
        # 100x300x12, measured on the CPU: reference vs the reference with its own tensor
        # symmetrized). The B200 spectrum is exactly symmetric, so the 1e-12 gate is taken
        # against the reference's convolution of its own tensor symmetrized, and against the
        # reference itself up to that measured asymmetry.
        from .test_parity_gpu import _symmetrized_reference_field
        sym = _symmetrized_reference_field(refsolver.build_tensor(nx, ny, nz, delta), m0, nx, ny, nz)
        obs["h_demag_vs_symmetrized_ref"] = rel(h_b, sym)
        obs["ref_tensor_asymmetry"] = rel(sym, h_ref)

    # one fused step: the update dM
    sim.set_magnetization(m0)
    r.set_m(m0)
    sim.step(1)
    r.step(1)
    m1, m1r = sim.magnetization().astype(np.float64), r.get_m().astype(np.float64)
    obs["dm_step1"] = rel(m1 - m0, m1r - m0)
    obs["m_step1"] = rel(m1, m1r)

    # two more steps, across the ramp stage with the sticky alpha override
    sim.step(2)
    r.step(2)
    assert sim.step_index() == r.step_index() == 3
    obs["m_step3"] = rel(sim.magnetization(), r.get_m())
    obs["avg_step3"] = float(np.max(np.abs(np.array(sim.average_unit()) - np.array(r.average_unit()))))
    tq_b, tq_r = sim.max_torque(), r.max_torque()
    obs["max_torque_rel"] = abs(tq_b - tq_r) / tq_r
    # H_eff at the reference's state, same step (applied field of the ramp at step 3)
    sim.set_magnetization(r.get_m())
    obs["heff_step3"] = rel(sim.effective_field(),
                            refsolver.heff(ref_problem(refsolver, sp), r.get_m(), sp.schedule.at(3)[0]))
    _observed[case] = obs

    if prec == "f64":
        assert obs["h_demag_vs_symmetrized_ref"] <= TOL_H[prec], obs
        assert obs["h_demag"] <= max(TOL_H[prec], obs["ref_tensor_asymmetry"] + TOL_H[prec]), obs
    else:
        assert obs["h_demag"] <= TOL_H[prec], obs
    assert obs["heff_step3"] <= TOL_H[prec], obs
    assert obs["dm_step1"] <= TOL_DM[prec], obs
    assert obs["m_step3"] <= TOL_M3[prec], obs
    assert obs["avg_step3"] <= TOL_M3[prec], obs
    assert obs["max_torque_rel"] <= (1e-9 if prec == "f64" else 1e-4), obs


# ---------------------------------------------------------------- film relaxation
def _load(name):
    p = os.path.join(GOLD, name)
    if not os.path.exists(p):
        pytest.skip(f"golden {name} not generated (tests/golden/make_golden.py)")
    return np.loadtxt(p, comments="#")


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_film256_relaxation_trajectory_matches_reference(refsolver, prec):
    """BASELINE configs[1]: the 256x256x1 film relaxing from the reference generator's random
    state, <m>(t) every 100 steps for 20 000 steps against the compiled reference's run
    (north-star trajectory gate: 1e-6 f64, 1e-3 f32)."""
    want = _load(f"traj_film256_{prec}.tsv")
    p = CASES[f"film256_{prec}"][0]
    sim = b200(_spec(p), prec)
    assert "k_yz<L9,ZM0>" in sim.path_info()
    sim.set_magnetization(refsolver.random_unit_field(256, 256, 1, 800.0, 20240 + 256,
                                                      np.float64 if prec == "f64" else np.float32))
    recs = []
    assert sim.run(RunOptions(steps=20000, cadence=100, sink=recs.append)) == 20000
    got = np.array([[rr.step, rr.mx, rr.my, rr.mz] for rr in recs])
    assert got.shape == want.shape and np.array_equal(got[:, 0], want[:, 0])
    dev = float(np.max(np.abs(got[:, 1:] - want[:, 1:])))
    _observed[f"film256_{prec}_traj"] = {"max_abs_dev": dev, "records": len(recs),
                                         "final": [float(v) for v in got[-1, 1:]]}
    assert dev <= (1e-6 if prec == "f64" else 1e-3)


# ---------------------------------------------------------------- acceptance criterion 6
def test_criterion6_relaxation_reaches_minimum_energy():
    """proj/tests/acceptance.cpp:307-336 on the B200 path: SP#3 16^3 f64 from uniform +x,
    energy sampled after each of 200 bursts of 100 steps, never rising (after step 500) by more
    than 1e-6 relative, final max torque < 1e-3; energies and <m> against the compiled
    reference's samples (tests/golden/crit6_sp3_16_f64.tsv)."""
    want = _load("crit6_sp3_16_f64.tsv")
    sim = b200(spec(16, 16, 16, 1.0, 1e7, 1000.0, 100.0, 0.5, 1e-5), "f64")
    rows = [(0, sim.energy()) + tuple(sim.average_unit())]
    for _ in range(200):
        sim.run(RunOptions(steps=100))
        rows.append((sim.step_index(), sim.energy()) + tuple(sim.average_unit()))
    assert sim.step_index() == 20000
    for (s0, e0, *_), (s1, e1, *_) in zip(rows, rows[1:]):
        if s0 < 500:
            continue
        assert e1 <= e0 + 1e-6 * abs(e0), f"energy rose between steps {s0} and {s1}: {e0} -> {e1}"
    torque = sim.max_torque()
    assert torque < 1e-3
    got = np.array(rows)
    assert np.array_equal(got[:, 0], want[:, 0])
    e_dev = float(np.max(np.abs(got[:, 1] - want[:, 1]) / np.abs(want[:, 1])))
    m_dev = float(np.max(np.abs(got[:, 2:] - want[:, 2:])))
    _observed["crit6"] = {"energy_rel_dev": e_dev, "m_dev": m_dev, "final_torque": torque}
    assert e_dev <= 1e-9 and m_dev <= 1e-9
