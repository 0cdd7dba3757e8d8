"""CPU checks of the measurement harness (bench.py): the canonical algorithmic bytes of
SURVEY.md §8(d), the per-kernel byte split the roofline uses, and the reference arm's
behaviour where the reference cannot run (2048x2048x64: ~181 GB of host memory)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_canonical_bytes_match_survey():
    # 512x512x8 f32 = 787.8 MB/step; 1024^2x32 = 12.52 GB; 2048^2x64 = 100.0 GB
    b, k = bench.algorithmic_bytes(512, 512, 8, 4)
    assert b == 787_833_048
    assert abs(bench.algorithmic_bytes(1024, 1024, 32, 4)[0] - 12.52e9) < 0.01e9
    assert abs(bench.algorithmic_bytes(2048, 2048, 64, 4)[0] - 100.0e9) < 0.05e9
    # the fused kernels' compulsory bytes
    assert k["yz"] == 157_704_408
    assert k["xstep"] == 151_191_552


def test_reference_arm_reports_unavailable_for_the_sharded_config():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                        "2048x2048x64_f32"], capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and "181 GB" in line["unavailable"]


def test_canonical_stage_split_sums_to_the_step():
    # the fused kernels' canonical stage bytes (roofline.canonical_stages) partition B_alg
    for g in [(512, 512, 8), (256, 256, 1), (128, 32, 1), (1024, 1024, 32), (2048, 2048, 64)]:
        b, k = bench.algorithmic_bytes(*g, 4)
        c = k["canonical"]
        assert c["yz"] + c["xstep"] == b
        assert c["y_fwd"] + c["z_mac"] + c["y_inv"] == c["yz"]
