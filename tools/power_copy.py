"""Data-dependent power of a pure HBM stream (development helper): a device
copy of 2 GiB of zeros vs the same bytes holding a developed-looking
wavefield (smooth random fp32), back to back for ~3 s each, with nvidia-smi
power/clock samples.  Tells whether the HBM/fabric path or the SM side carries
the extra power the developed wavefield costs the sweep."""
import json
import subprocess
import time

import torch

N = 512 * 1024 * 1024  # floats (2 GiB)


def run(name, a):
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "100"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 0
    e0.record()
    t = time.time()
    while time.time() - t < 3.0:
        for _ in range(20):
            b.copy_(a)
        iters += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    p.terminate()
    out, _ = p.communicate()
    rows = [tuple(float(x) for x in l.split(",")) for l in out.strip().splitlines() if l.strip()]
    rows = rows[5:-2] if len(rows) > 10 else rows
    mhz = sorted(r[0] for r in rows)
    pw = sorted(r[1] for r in rows)
    ms = e0.elapsed_time(e1) / iters
    print(json.dumps(dict(case=name, gbs=round(2 * N * 4 / (ms * 1e-3) / 1e9, 1),
                          sm_mhz=mhz[len(mhz) // 2], power_w=pw[len(pw) // 2], n=len(rows))), flush=True)


def main():
    z = torch.zeros(N, device="cuda")
    run("zeros", z)
    g = torch.randn(N, device="cuda") * 1e-3
    run("random_fp32", g)
    # smooth field: low-order bits random, high bits correlated (like a wavefield)
    x = torch.linspace(0, 200, N, device="cuda")
    s = torch.sin(x) * 1e-2 + torch.randn(N, device="cuda") * 1e-5
    run("smooth_fp32", s)
    run("zeros_again", z)


if __name__ == "__main__":
    main()
