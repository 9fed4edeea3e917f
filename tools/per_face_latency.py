"""Per-face drop-in latency: harness.run_bench (HaloExchange.run with HOST arrays, the call a
reference user makes) on the B200 path, beside the reference's own run_bench on one host core
when the reference is installed (baseline/_ref, Numba).  p = 9, k = 3, u = 59, every scheme and
role (restriction: half "inner", run_bench's default, and the full face).

    python tools/per_face_latency.py > profiles/r02_per_face_latency.json
"""

from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SCHEMES = ("tensor_linear", "matrix_linear", "order2", "order3")


def main() -> None:
    import torch

    import paper_2504_15814_b200 as th

    ref = None
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "trihalo")):
        sys.path.insert(0, ref_dir)
        try:
            import trihalo as ref  # the unmodified reference (pure Python + Numba)
        except Exception as exc:  # noqa: BLE001
            print(f"reference not importable: {exc}", file=sys.stderr)
            ref = None
    rows = []
    for scheme in SCHEMES:
        for role, half in (("interpolate", None), ("restrict", "inner"), ("restrict", None)):
            cfg = th.FaceConfig("x", "negative", 4, 9, 3, 59)
            r = th.run_bench(scheme, role, cfg, repetitions=200, half=half)
            row = {"scheme": scheme, "role": role, "half": half, "b200_us": round(r.mean_ns / 1e3, 1)}
            if ref is not None:
                rcfg = ref.FaceConfig("x", "negative", 4, 9, 3, 59)
                t = time.perf_counter()
                rr = ref.run_bench(scheme, role, rcfg, repetitions=20, half=half)
                row["reference_us"] = round(rr.mean_ns / 1e3, 1)
                row["reference_wall_s"] = round(time.perf_counter() - t, 1)
                row["speedup"] = round(row["reference_us"] / row["b200_us"], 2)
            rows.append(row)
            print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps({"what": "mean wall time of one HaloExchange.run with host numpy arrays (harness.run_bench), "
                              "p=9 k=3 u=59, face x/negative segment 4",
                      "b200": "H2D (page-locked staging) + finiteness kernel + apply kernel + D2H of result and "
                              "flag, one synchronisation",
                      "reference": "unmodified reference run_bench on one host core (Numba kernel)" if ref else None,
                      "gpu": torch.cuda.get_device_name(0), "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
