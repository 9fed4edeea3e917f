"""Generate golden fixtures from the REAL reference package (run in the build
container, where /root/reference exists; the outputs are committed).

    python tests/golden/make_golden.py

Writes, next to this script:
  operators.npz  canonical CSR arrays of reference operators
                 (OperatorCache.get, taylor.py:252-308) for small (p, k) and
                 the p=9 restriction operators
  maps.npz       HaloExchange gather/scatter CELL maps (_gather[::u] // u,
                 schemes.py:147-151) for every orientation x segment / half at
                 the bench shapes p=9 and p=17 (k=3) and at p=4, k=3 / p=5, k=2
  exchange.npz   HaloExchange.run outputs (schemes.py:185-202) for seeded
                 random sources: every scheme x role x half x orientation at
                 small p, and sampled faces at p=9 / p=17 (u=2).  Sources are
                 regenerated from their seeds with numpy PCG64
                 standard_normal, so only seeds and outputs are stored.
  golden_p1k1.txt the reference's own dump golden (pkg/tests/test_csr.py:185-194)
"""

from __future__ import annotations

import itertools
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from trihalo import csr, schemes, taylor  # noqa: E402
from trihalo.geometry import FaceConfig  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
FACES = list(itertools.product(("x", "y", "z"), ("negative", "positive")))


def op_key(scheme, role, p, k):
    return f"{scheme}|{role}|{p}|{k}"


def make_operators(cache):
    out = {}
    cases = [(p, k) for p in range(1, 7) for k in range(1, 4) if k <= p] + [(9, 3)]
    for scheme in ("matrix_linear", "order2", "order3"):
        for role in ("interpolate", "restrict"):
            for p, k in cases:
                ok, _ = schemes.scheme_feasible(scheme, role, p, k)
                if not ok:
                    continue
                if p == 9 and role == "interpolate" and scheme != "matrix_linear":
                    continue  # large; covered through exchange outputs instead
                op = cache.get(csr.OperatorKey(role, scheme, p, k))
                key = op_key(scheme, role, p, k)
                out[key + "|ro"] = op.row_offsets.astype(np.int32)
                out[key + "|ci"] = op.col_indices.astype(np.int32)
                out[key + "|v"] = op.values
                out[key + "|cond"] = np.array([op.max_condition])
    return out


def make_maps(cache):
    out = {}
    for p, k in ((4, 3), (5, 2), (9, 3), (17, 3)):
        for normal, side in FACES:
            for seg in range(9):
                cfg = FaceConfig(normal, side, seg, p, k, 1)
                ex = schemes.HaloExchange(cfg, "matrix_linear", "interpolate", cache=cache)
                key = f"interp|{p}|{k}|{normal}|{side}|{seg}"
                out[key + "|g"] = ex._gather.astype(np.int32)
                out[key + "|s"] = ex._scatter.astype(np.int32)
            for half in (None, "inner", "outer"):
                cfg = FaceConfig(normal, side, 0, p, k, 1)
                ex = schemes.HaloExchange(cfg, "matrix_linear", "restrict", half=half, cache=cache)
                key = f"restrict|{p}|{k}|{normal}|{side}|{half}"
                out[key + "|g"] = ex._gather.astype(np.int32)
                out[key + "|s"] = ex._scatter.astype(np.int32)
    return out


def make_exchanges(cache):
    out = {}
    seed = 1000
    small = [(4, 3, 3), (5, 2, 2), (3, 3, 2), (6, 3, 2), (1, 1, 2), (2, 2, 3)]
    for (p, k, u), scheme in itertools.product(small, schemes.SCHEMES):
        for normal, side in FACES:
            for role, half in (("interpolate", None), ("restrict", None), ("restrict", "inner"),
                               ("restrict", "outer")):
                ok, _ = schemes.scheme_feasible(scheme, role, p, k)
                if not ok:
                    continue
                segs = (0, 4, 8, seed % 9) if role == "interpolate" else (0,)
                for seg in sorted(set(segs)):
                    cfg = FaceConfig(normal, side, seg, p, k, u)
                    ex = schemes.HaloExchange(cfg, scheme, role, half=half, cache=cache)
                    n_src = ex.source_region.cell_count * u
                    src = np.random.default_rng(seed).standard_normal(n_src)
                    o = np.zeros(ex.target_region.cell_count * u)
                    ex.run(src, o)
                    key = f"{scheme}|{role}|{half}|{p}|{k}|{u}|{normal}|{side}|{seg}"
                    out[key + "|seed"] = np.array([seed])
                    out[key + "|out"] = o
                    seed += 1
    # bench shapes, sampled faces, u=2
    rng = np.random.default_rng(7)
    for p in (9, 17):
        for scheme in schemes.SCHEMES:
            for role, half in (("interpolate", None), ("restrict", None)):
                for _ in range(2):
                    normal, side = FACES[int(rng.integers(0, 6))]
                    seg = int(rng.integers(0, 9))
                    cfg = FaceConfig(normal, side, seg, p, 3, 2)
                    ex = schemes.HaloExchange(cfg, scheme, role, half=half, cache=cache)
                    src = np.random.default_rng(seed).standard_normal(ex.source_region.cell_count * 2)
                    o = np.zeros(ex.target_region.cell_count * 2)
                    ex.run(src, o)
                    key = f"{scheme}|{role}|{half}|{p}|3|2|{normal}|{side}|{seg}"
                    out[key + "|seed"] = np.array([seed])
                    out[key + "|out"] = o
                    seed += 1
    return out


def main():
    cache = taylor.OperatorCache()
    np.savez_compressed(os.path.join(HERE, "operators.npz"), **make_operators(cache))
    np.savez_compressed(os.path.join(HERE, "maps.npz"), **make_maps(cache))
    np.savez_compressed(os.path.join(HERE, "exchange.npz"), **make_exchanges(cache))
    from trihalo.linear import _collapse

    with open(os.path.join(HERE, "golden_p1k1.txt"), "w") as fh:
        fh.write(csr.dumps_operator(_collapse(1, 1, "interpolate")))
    for name in ("operators.npz", "maps.npz", "exchange.npz", "golden_p1k1.txt"):
        print(name, os.path.getsize(os.path.join(HERE, name)))


if __name__ == "__main__":
    main()
