"""bench.py at N > 1 without torchrun (one process, a host thread per rank),
emulated on this box's one GPU with --devices 0,0: the default C5 weak-scaling
workload and the C4 strong-scaling split run end to end through the slab
decomposition, and the line carries the transport and a passing parity check
(a reduced grid over the same ranks, bit-exact against one domain)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload,scaling", [("auto", "weak"), ("C4", "strong")])
def test_bench_two_ranks_emulated(workload, scaling):
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--devices", "0,0", "--steps", "1",
                        "--warmup", "1", "--no-e2e", "--no-cpu", "--workload", workload],
                       cwd=ROOT, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == scaling
    assert line["config"]["workload"] == ("C5" if workload == "auto" else "C4")
    assert line["parity"]["ok"] and line["parity"]["field_bit_exact"] and line["parity"]["seismogram_bit_exact"], \
        line["parity"]
    assert "host-ordered" in line["transport"]
    assert line["value"] > 0 and line["gpu_launches"] > 0
