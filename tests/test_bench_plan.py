"""bench.py's run plan on CPU: which workload each N runs, 2D replicas, and
when the timing rule needs an L2 flush (no GPU, no library calls)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

L2 = 126 * 2**20


def test_default_workloads():
    assert bench.workload_cfg("auto", 1)[0] == "C4"
    name, cfg = bench.workload_cfg("auto", 8)
    assert name == "C5" and cfg.fixed_steps == 500
    assert cfg.bbox[1] == 20.0 * (200 * 8 - 10 - 1)  # 200 extended planes per GPU
    name, cfg = bench.workload_cfg("C4w", 2)
    assert name == "C4w" and cfg.ndim == 3


def test_2d_runs_replicas_3d_shards():
    assert bench.replicated(bench.workload_cfg("C2", 4)[1], 4)
    assert not bench.replicated(bench.workload_cfg("C2", 1)[1], 1)
    assert not bench.replicated(bench.workload_cfg("C4", 4)[1], 4)


def test_l2_flush_rule():
    assert bench.l2_flush_needed(421 * 1841, L2)          # C1/C2: 12 MB working set
    assert not bench.l2_flush_needed(142_725_457, L2)     # C4: 2.3 GB
    assert not bench.l2_flush_needed(131_544_200, L2)     # C5 per GPU
