"""The reference's whole C4 forward on this host's cores (oracle/_ref: the
reference's setup chain and Solver<float>::forward, Backend::Parallel, all
threads), timed like the reference times it (kernel_seconds,
kernel.hpp:253-261), and checked against the committed full-length fixture
(the same bits as the build container's run and as the GPU).  One JSON line.
Run next to `bench.py` on the GPU box for "CPU time in the same run"."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_2201_05278_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
cfg = configs.CONFIGS[name]()
t0 = time.time()
r = O.RefRun(cfg, np.float32)
setup = time.time() - t0
res = r.forward()
seis = res["seismogram"].reshape(r.n_steps + 1, r.n_rec)
meta = json.loads(str(np.load(os.path.join(ROOT, "tests", "golden", f"full_{name.lower()}.npz"))["meta"]))
pts = int(np.prod(r.extended))
print(json.dumps({
    "config": name, "n_steps": r.n_steps, "kernel_seconds": round(res["seconds"], 2), "setup_seconds": round(setup, 2),
    "gpts": round(pts * r.n_steps / res["seconds"] / 1e9, 4), "threads": int(O.rlib().ref_max_threads()),
    "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ") if os.path.exists("/proc/cpuinfo") else None,
    "matches_fixture": hashlib.sha256(np.ascontiguousarray(seis).tobytes()).hexdigest() == meta["sha_seismogram"]
    and hashlib.sha256(np.ascontiguousarray(res["final"]).tobytes()).hexdigest() == meta["sha_final"],
}), flush=True)
