"""Per-step cost of the multi-GPU (peer) step path, measured on ONE GPU.

A middle rank of a C5 weak-scaling decomposition (200 extended planes x 811 x
811, SO8; world 3, rank 1: neighbours on both sides, as every inner GPU of an
8-GPU run) is stepped with emulated neighbours (fdw_peer_loopback): its sweep
runs the boundary Z segments first, waits for the neighbours' epoch in its
boundary CTAs, stores the 2 x R halo planes (to scratch on this GPU instead
of NVLink) and publishes; the health check reduces through the sync blocks.
The baseline is the same 200-plane grid as ONE single-GPU domain with rank
1's own velocity / eta ("single_same_medium": same eta-skipping, same work);
"single" is C5 at N=1 (its damped top / bottom planes stream more eta).
Variants of the peer path (env knobs read at Solver creation) isolate the
boundary-segment rotation, the release fences, the halo stores and PDL.  Both run
graph-captured with programmatic dependent launch, no sources / receivers on
either (rank 1 of C5 owns none), on the same box, interleaved.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2201_05278_b200 import DampingField, Solver, configs, make_material_model  # noqa: E402

N = int(os.environ.get("STEPS", "500"))
REPS = int(os.environ.get("REPS", "3"))


def solver(w, slab=None):
    return Solver(w.grid, make_material_model(w.velocity), DampingField(eta=w.eta), w.spec, w.axis, w.coeffs,
                  slab=slab)


def main():
    w1 = configs.build_workload(configs.weak3d(1), np.float32)
    w3 = configs.build_workload(configs.weak3d(3), np.float32, rank=1, world=3)
    pts = int(np.prod(w1.grid.extended_shape))
    stream = torch.cuda.Stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    variants = {"single": {}, "single_same_medium": {}, "peer_middle_rank": {}, "peer_no_segrot": {"FDW_DBG_NO_SEGROT": "1"},
                "peer_fence_all": {"FDW_DBG_FENCE_ALL": "1"}, "peer_fence_sc": {"FDW_DBG_FENCE_SC": "1"}, "peer_no_halo_store": {"FDW_DBG_NO_HALO_STORE": "1"},
                "peer_no_pdl": {"FDW_NO_PDL": "1"}}
    only = os.environ.get("CASES")
    res = {k: [] for k in variants if not only or k in only.split(",") or k.startswith("single")}
    lay = {}
    for rep in range(REPS):
        for name in res:
            os.environ.update(variants[name])
            if name == "single":
                s = solver(w1)
            elif name == "single_same_medium":  # rank 1's velocity / eta as one 200-plane domain
                s = Solver(w1.grid, make_material_model(w3.velocity), DampingField(eta=w3.eta), w1.spec, w1.axis,
                           w1.coeffs)
            else:
                s = solver(w3, w3.slab)
            for k in variants[name]:
                os.environ.pop(k, None)
            if name.startswith("peer"):
                s.peer_loopback()
            s.set_stream(stream.cuda_stream)
            lay[name] = s.layout()
            # a developed (non-zero) state: random levels, then 100 warm steps
            rng = np.random.default_rng(5)
            s.previous_level()[...] = rng.standard_normal(s.previous_level().shape).astype(np.float32) * 1e-3
            s.current_level()[...] = rng.standard_normal(s.current_level().shape).astype(np.float32) * 1e-3
            s.refresh_boundary()
            s._host_view = False
            s.advance_raw(100)
            torch.cuda.synchronize()
            ev0.record(stream)
            s.advance_raw(N)
            ev1.record(stream)
            torch.cuda.synchronize()
            res[name].append(ev0.elapsed_time(ev1) / N * 1e3)
            s.close()
    best = {k: min(v) for k, v in res.items()}
    out = {"steps": N, "points": pts, "us_per_step": {k: round(v, 2) for k, v in best.items()},
           "reps": {k: [round(x, 2) for x in v] for k, v in res.items()},
           "overhead_us_vs_same_medium": {k: round(v - best["single_same_medium"], 2) for k, v in best.items()
                                          if k.startswith("peer")},
           "efficiency_without_nvlink": round(best["single_same_medium"] / best.get("peer_middle_rank", float("nan")),
                                              4),
           "layout": lay}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
