"""The committed ncu traffic figure is tied to the sweep's current source:
bench.py reports it only while the SHA-256 of fdw_kernels.cuh up to the end
of the 3D TMA sweep matches the capture (CPU only)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import pytest  # noqa: E402


def test_traffic_matches_current_sweep_source():
    with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
        d = json.load(f)
    if d["sweep_source_sha256"] != bench.sweep_source_sha():
        assert bench.traffic_for("C4")[0] is None  # reported as stale, never as an old number
        pytest.skip("the sweep changed since the committed ncu capture: re-run tools/ncu_dev.sh")
    tr, src = bench.traffic_for("C4")
    # 17 B/pt floor (1-byte damping index) <= measured <= 20 B/pt model
    assert 17 * 142_725_457 <= tr <= 20 * 142_725_457, (tr, src)
