"""The real reference's CPU path beside the C port the bench's reference arm uses, on the same
config-5 face sample (one-off measurement for DESIGN.md / profiles):

  * port:      oracle C restatement of HaloExchange.run over all host threads (OpenMP) — what
               ``bench.py --impl reference`` times;
  * reference: the unmodified reference (baseline/_ref, pure Python + Numba) HaloExchange.run,
               one exchange object per (orientation, segment / half) class built outside the
               timer, faces spread over a process pool of os.cpu_count() workers (SURVEY §8d:
               threads do not scale, the Numba kernel holds the GIL); and on one core.

    python tools/reference_cpu.py [faces per role] > profiles/r02_reference_cpu.json
"""

from __future__ import annotations

import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

JOBS = []      # (role, normal, side, segment, source) — inherited by forked workers
_EX = {}


def _ref():
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    import trihalo

    return trihalo


def _run_chunk(idx):
    R = _ref()
    t = 0.0
    n_vals = 0
    for i in idx:
        role, normal, side, seg, src = JOBS[i]
        key = (role, normal, side, seg)
        ex = _EX.get(key)
        if ex is None:
            cfg = R.FaceConfig("xyz"[normal], ("negative", "positive")[side], seg, 9, 3, 59)
            ex = _EX[key] = R.HaloExchange(cfg, "order3", role)
            o = np.empty(ex.target_region.cell_count * 59)
            ex.run(src, o)  # warm (Numba JIT / cache load) outside the timer
        out = np.empty(ex.target_region.cell_count * 59)
        t0 = time.perf_counter()
        ex.run(src, out)
        t += time.perf_counter() - t0
        n_vals += out.size
    return t, n_vals


def main() -> None:
    import bench
    import workloads as W
    from oracle import exchange as OE
    from oracle import geometry as OG

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    wl = W.describe_multi(1)
    rng = np.random.default_rng(777)
    exs, srcs, outs = [], [], []
    for role in ("interpolate", "restrict"):
        for f in np.sort(rng.choice(wl.spec.n_faces, n, replace=False)):
            seg = int(wl.segment[f]) if role == "interpolate" else 0
            src = bench.c5_host_source(wl, f, role, rng)
            JOBS.append((role, int(wl.normal[f]), int(wl.side[f]), seg, src))
            cfg = OG.FaceCfg("xyz"[int(wl.normal[f])], ("negative", "positive")[int(wl.side[f])], seg, 9, 3, 59)
            ex = OE.exchange_for(cfg, "order3", role)
            exs.append(ex)
            srcs.append(src)
            outs.append(np.empty(ex.n_out))
    nth = bench.cpu_threads()
    OE.run_many(exs, srcs, outs, nth)
    t = time.perf_counter()
    reps = 5
    for _ in range(reps):
        OE.run_many(exs, srcs, outs, nth)
    port = reps * sum(o.size for o in outs) / (time.perf_counter() - t)
    OE.run_many(exs, srcs, outs, 1)
    t = time.perf_counter()
    OE.run_many(exs, srcs, outs, 1)
    port1 = sum(o.size for o in outs) / (time.perf_counter() - t)
    res = {"sample": f"{n} interpolation + {n} restriction faces of config 5 (order3, p=9, k=3, u=59)",
           "host_threads": nth, "port_values_per_s": port, "port_1core_values_per_s": port1}
    try:
        _ref()
        workers = os.cpu_count() or 1
        chunks = [list(range(i, len(JOBS), workers)) for i in range(workers)]
        with mp.get_context("fork").Pool(workers) as pool:
            pool.map(_run_chunk, chunks)  # warm every worker's exchanges and JIT
            t = time.perf_counter()
            parts = pool.map(_run_chunk, chunks)
            wall = time.perf_counter() - t
        vals = sum(v for _, v in parts)
        res["reference_pool_workers"] = workers
        res["reference_pool_values_per_s"] = vals / wall
        t1, v1 = _run_chunk(list(range(0, len(JOBS), 4)))
        t1, v1 = _run_chunk(list(range(0, len(JOBS), 4)))
        res["reference_1core_values_per_s"] = v1 / t1
        res["port_over_reference_pool"] = port / res["reference_pool_values_per_s"]
    except Exception as exc:  # noqa: BLE001
        res["reference_error"] = repr(exc)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
