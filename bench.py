"""Benchmark of the B200 halo interpolation / restriction path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of every (role, scheme) of BASELINE.json's config over all
of its faces, inputs resident in HBM.  Default: config 5 (configs[4]), the
largest configuration that fits one B200: p=9, k=3, u=59, 32,768 coarse
patches (52.2 GB pool), 196,608 faces, order3 interpolation + restriction of
every face, fine patches read from the pool by index lists; under torchrun
the patches are block-partitioned over the ranks and cross faces exchange
source boxes / results over NCCL.  --config 1..4 run the other BASELINE
configs.  Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine ghost-cell values/s (interp+restrict, fp64) and % of HBM roofline"
PEAK_NORTH_STAR = 8000.0  # GB/s, BASELINE.json north_star's roofline denominator


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--fine-layout", choices=("random", "siblings"), default="random",
                    help="config 5 diagnosis: the nine fine patches of a face uniform over the pool (default) "
                         "or consecutive ids")
    ap.add_argument("--straddle", type=float, default=0.0,
                    help="config 5: fraction of faces with one fine patch drawn from the whole pool (A/B, tests)")
    ap.add_argument("--scale", type=float, default=1.0, help="shrink patch / face counts (tuning runs only)")
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--graph", action="store_true",
                    help="configs 1-4: capture the timed steps in one CUDA graph (launch-bound small batches)")
    ap.add_argument("--passes", default=None,
                    help="configs 1-4: override the (role:scheme,...) passes, e.g. interpolate:matrix_linear,"
                         "restrict:matrix_linear (extra measurements; the default is BASELINE's)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-chunks", type=int, default=64, help="pipeline chunks of the e2e leg")
    ap.add_argument("--cpu-sample", type=int, default=512, help="faces per pass in the CPU reference arm's sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sustained", action="store_true", help="skip the sustained-copy yardstick (config 5)")
    ap.add_argument("--no-same-level", action="store_true", help="skip the same-level halo fill leg")
    ap.add_argument("--overlap", action="store_true", help="A/B: interpolation passes on a side stream (diagnosis)")
    ap.add_argument("--reverse-passes", action="store_true", help="run the step's passes in reverse order (diagnosis)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 20 ms; only samples taken inside the
    timed region (mark() .. stop()) are reported (the nearest one before it if the region is
    shorter than the sampling interval)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None
        self.t_mark = None

    def _rows(self):
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) == 6 and parts[0].isdigit():
                    rows.append(parts)
        return rows

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        deadline = time.time() + 5.0  # nvidia-smi needs a moment before its first sample
        while time.time() < deadline and not self._rows():
            time.sleep(0.02)

    def mark(self):
        """Start of the timed region."""
        self.n_before = len(self._rows()) if self.proc is not None else 0

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.03)  # let the sample covering the end of the region land
        self.proc.terminate()
        self.proc.wait()
        rows = self._rows()
        os.unlink(self.path)
        start = getattr(self, "n_before", 0)
        inside = rows[start:] if len(rows) > start else rows[-1:]
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        reasons = sorted({names[i] for r in inside for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(float(r[0]) for r in inside), "sm_max_mhz": float(inside[0][1]),
                "reasons": reasons, "samples": len(inside)}


def sustained_copy(dev, index: int, seconds: float = 2.0):
    """The copy yardstick of MEASURED_PEAKS.json (b.copy_(a) over 1 Gi bf16 elements, read + write
    bytes) run back to back for `seconds` on this box, right after the timed sweeps: what a plain
    copy sustains under the same power cap the sweep runs into (the peak itself is a best-of-10
    burst).  Reported beside the roofline, never used as its denominator."""
    import torch

    try:
        a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
        b = torch.empty_like(a)
    except RuntimeError as exc:  # out of memory beside a large workload
        return {"error": str(exc).splitlines()[0]}
    a.zero_()
    nbytes = 2 * a.numel() * a.element_size()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(10):
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    n = max(30, int(seconds * best * 1e9 / nbytes))
    sampler = ClockSampler(index)
    sampler.start()
    for _ in range(n // 3):  # a third of the run to reach the sustained state
        b.copy_(a)
    torch.cuda.synchronize()
    sampler.mark()
    e0.record()
    for _ in range(n - n // 3):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    clocks = sampler.stop()
    gbs = (n - n // 3) * nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9
    del a, b
    return {"GBps": round(gbs, 1), "burst_GBps": round(best, 1), "seconds": round(e0.elapsed_time(e1) / 1e3, 2),
            "clocks": clocks, "how": "b.copy_(a), 1 Gi bf16 elements, back to back; read + write bytes"}


# ---------------------------------------------------------------------------
# algorithmic bytes / flops per face (distinct support cells + output)
# ---------------------------------------------------------------------------

def unit_costs(role, scheme, p, k, u, selectors):
    """Per-face (bytes, flops) averaged over the faces' segments / halves, from the
    operator's exported rows (the reference CSR structure)."""
    from paper_2504_15814_b200.operators import HostOperator

    h = HostOperator(role, scheme, p, k)
    cache = {}
    b_tot = f_tot = 0.0
    for sel in selectors:
        if sel not in cache:
            c = h.csr(segment=int(sel)) if role == "interpolate" else h.csr(half=sel)
            support = np.unique(c.col_indices).size
            cache[sel] = ((support + c.n_rows) * u * 8.0, 2.0 * c.nnz * u)
        b, f = cache[sel]
        b_tot += b
        f_tot += f
    n = max(1, len(selectors))
    return b_tot / n, f_tot / n, h.info.device_bytes if hasattr(h.info, "device_bytes") else 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def ours_config(s, world, wl=None):
    """Config dict of configs 1-4, shared by both arms."""
    return {"workload": f"config{s.config}: {s.name}", "p": s.p, "k": s.k, "u": s.u, "coarse_patches": s.n_patches,
            "faces": s.n_faces, "passes": [f"{r}:{sc}" for r, sc in s.passes],
            "layout": "coarse pool (p+2k)^3 AoS + per-face fine restriction slabs (world layout)",
            "l2": "inputs >> 126 MB L2 (no flush needed)",
            "parallelism": f"weak: {world} independent shard(s)"}


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2504_15814_b200 as th
    import workloads as W

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    wl = W.build(args.config, rank=rank, scale=args.scale)
    s = wl.spec
    if args.passes:
        s.passes = [tuple(x.split(":")) for x in args.passes.split(",")]
    p, k, u = s.p, s.k, s.u
    passes = []
    cache = th.operators.DEFAULT_CACHE
    for role, scheme in (reversed(s.passes) if args.reverse_passes else s.passes):
        op = cache.device_operator(role, scheme, p, k)
        if role == "interpolate":
            rec, src, ids = W.interp_records(wl), wl.pool, wl.interp_ids
            n_tgt = k * p * p
            sel = wl.faces.segment[ids]
        else:
            rec, src, ids = W.restrict_records(wl), wl.fine, wl.restrict_ids
            n_tgt = k * p * p
            sel = [None] * ids.size
        batch = th.FaceBatch(op, rec, u)
        out = torch.empty(ids.size * n_tgt * u, dtype=torch.float64, device=dev)
        b, f, _ = unit_costs(role, scheme, p, k, u, sel)
        passes.append(dict(role=role, scheme=scheme, batch=batch, src=src, out=out, n=ids.size,
                           values=ids.size * n_tgt * u, bytes=b * ids.size + op.info.device_bytes,
                           flops=f * ids.size))
    stream = torch.cuda.current_stream()
    side = torch.cuda.Stream(device=dev) if args.overlap else None

    def step(evs=None):
        if side is not None:  # A/B: interpolation passes on a side stream beside the restrictions
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                for ps in passes:
                    if ps["role"] == "interpolate":
                        ps["batch"].launch(ps["src"], ps["out"], stream=side.cuda_stream)
            for ps in passes:
                if ps["role"] != "interpolate":
                    ps["batch"].launch(ps["src"], ps["out"])
            stream.wait_stream(side)
            return
        for i, ps in enumerate(passes):
            if evs is not None:
                evs[i].record(stream)
            ps["batch"].launch(ps["src"], ps["out"])
        if evs is not None:
            evs[-1].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.05)
    ev_all = [[torch.cuda.Event(enable_timing=True) for _ in range(len(passes) + 1)] for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    graph = None
    if args.graph:  # the K timed steps as one CUDA graph: no host launch gaps between passes
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            for kk in range(args.steps):
                step()
        torch.cuda.synchronize()
        graph.replay()  # warm replay
        torch.cuda.synchronize()
    sampler.mark()
    t0.record(stream)
    if graph is not None:
        graph.replay()
    else:
        for kk in range(args.steps):
            step(ev_all[kk])
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    total_ms = t0.elapsed_time(t1)
    if graph is not None:  # per-pass events from ungraphed steps (the graph has no event nodes)
        for kk in range(args.steps):
            step(ev_all[kk])
        torch.cuda.synchronize()
    if side is not None:  # no per-pass events in the overlapped step: one serial step per pass row
        ev_all = ev_all[:1]
        step(None)
        torch.cuda.synchronize()
        side_, side = side, None
        step(ev_all[0])
        side = side_
        torch.cuda.synchronize()
    per_pass_ms = [statistics.mean(ev[i].elapsed_time(ev[i + 1]) for ev in ev_all) for i in range(len(passes))]
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    values_per_step = sum(ps["values"] for ps in passes)
    value = values_per_step * world / (ms_per_step / 1e3)
    peak, peak_kind = peaks()
    pass_rows = []
    for ps, ms in zip(passes, per_pass_ms):
        gbs = ps["bytes"] / (ms / 1e3) / 1e9
        pass_rows.append({"role": ps["role"], "scheme": ps["scheme"], "faces": ps["n"], "ms": round(ms, 4),
                          "alg_bytes": int(ps["bytes"]), "alg_GBps": round(gbs, 1), "frac_hbm": round(gbs / peak, 3),
                          "frac_8tbs": round(gbs / PEAK_NORTH_STAR, 3),
                          "csr_equiv_TFLOPs": round(ps["flops"] / (ms / 1e3) / 1e12, 2)})
    dom = max(range(len(passes)), key=lambda i: per_pass_ms[i])
    result = {
        "metric": METRIC, "value": value, "unit": "values/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded field (BASELINE config text) sampled at cell centres + 1e-6 N(0,1), generated in HBM",
        "config": {**ours_config(s, world, wl),
                   **({"overlap": "interpolation passes on a side stream"} if args.overlap else {})},
        "roofline": {"bound": "hbm", "kernel": f"{passes[dom]['role']}:{passes[dom]['scheme']}",
                     "achieved": pass_rows[dom]["alg_GBps"], "peak": peak, "unit": "GB/s",
                     "frac": round(pass_rows[dom]["alg_GBps"] / peak, 4),
                     "frac_8tbs": round(pass_rows[dom]["alg_GBps"] / PEAK_NORTH_STAR, 4), "traffic": None,
                     "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy)"},
        "passes": pass_rows,
        "gpu_launches": args.steps * len(passes),
        "clocks": clocks,
    }
    # measured DRAM traffic of the dominant kernel (ncu --set full, committed under profiles/)
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get(f"config{s.config}", {})
        ent = tr.get(f"{passes[dom]['role']}:{passes[dom]['scheme']}")
        if isinstance(ent, dict):  # bytes of one measured launch over its face count, scaled to this launch
            result["roofline"]["traffic"] = round(ent["bytes"] * s.n_faces / ent["faces"])
            result["roofline"]["traffic_source"] = (f"profiles/traffic.json (dram__bytes_read.sum + dram__bytes_write.sum, "
                                                    f"measured on {ent['faces']} faces, scaled per face)")
    except (OSError, ValueError):
        pass
    step_bytes = sum(ps["bytes"] for ps in passes)
    result["step_alg_GBps"] = round(step_bytes / (ms_per_step / 1e3) / 1e9, 1)
    result["step_frac_hbm"] = round(step_bytes / (ms_per_step / 1e3) / 1e9 / peak, 4)
    result["nonfinite_flag"] = any(ps["batch"].nonfinite() for ps in passes)
    if not args.no_e2e:
        result["e2e"] = run_e2e(args, wl, passes, dev, world)
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"], result["parity"] = cpu_baseline(args, wl, passes)
    if not args.no_same_level:  # last: it rewrites the pool's halos
        result["same_level"] = same_level_leg(wl, dev, peak)
    return result


def same_level_leg(wl, dev, peak, reps=20):
    """Same-level halo fill (th_copy_faces) over the workload's patch pool:
    all six faces of every patch from a random same-level neighbour, bit-exactness of a
    sample checked against the copy, k x p x p cells x u read + written per face."""
    import numpy as np
    import torch

    import paper_2504_15814_b200 as th

    s = wl.spec
    p, k, u = s.p, s.k, s.u
    n = wl.pool.numel() // ((p + 2 * k) ** 3 * u)
    rng = np.random.default_rng(100 + s.config)
    dst = np.repeat(np.arange(n), 6)
    nrm, sid = np.tile(np.repeat(np.arange(3), 2), n), np.tile(np.arange(2), 3 * n)
    src = (dst + rng.integers(1, max(n, 2), dst.size)) % max(n, 2) if n > 1 else dst
    rec = th.pool_same_level_faces(p, k, u, src, dst, nrm, sid)
    rec_d = torch.from_numpy(rec.view(np.uint8).ravel().copy()).to(dev)
    pool = wl.pool
    for _ in range(3):
        th.copy_faces(pool, pool, rec_d, k, p, u)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        th.copy_faces(pool, pool, rec_d, k, p, u)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byts = 2 * dst.size * k * p * p * u * 8
    # sample: face 0's halo box equals its neighbour's interior box
    E = p + 2 * k
    v = pool.view(n, E, E, E, u)
    r0 = rec[0]
    ax = 2 - int(r0["normal"])
    a = [slice(k, k + p)] * 3
    b = list(a)
    a[ax] = slice(p, p + k) if r0["side"] == 0 else slice(k, 2 * k)
    b[ax] = slice(0, k) if r0["side"] == 0 else slice(p + k, p + 2 * k)
    ok = bool(torch.equal(v[(int(src[0]), *a)], v[(int(dst[0]), *b)]))
    gbs = byts / (ms / 1e3) / 1e9
    return {"faces": int(dst.size), "ms": round(ms, 4), "alg_bytes": int(byts), "alg_GBps": round(gbs, 1),
            "frac_hbm": round(gbs / peak, 3), "sample_bit_exact": ok, "launches": reps}


# ---------------------------------------------------------------------------
# config 5 (default): the largest BASELINE configuration that fits one B200
# ---------------------------------------------------------------------------

def c5_config(spec, world, straddle=0.0):
    """The config dict of both arms (ours and --impl reference)."""
    return {"workload": f"config5: {spec.name}", "p": spec.p, "k": spec.k, "u": spec.u,
            "coarse_patches": spec.n_patches, "faces": spec.n_faces,
            "passes": ["interpolate:order3", "restrict:order3"],
            "fine_sources": "the nine fine patches of every face read from the patch pool by index lists",
            "cross_faces": "10% of faces: fine patches on a partner rank (uniform); at N=1 all faces are local",
            **({"straddle": straddle} if straddle else {}),
            "parallelism": f"{world} rank(s), block-partitioned patches, NCCL P2P for cross faces",
            "l2": "pool 52.2 GB >> 126 MB L2 (no flush needed)"}


def c5_jobs(wl, faces_by_role):
    """Oracle jobs (exchange, source, output) for {role: face ids}; patches regenerated."""
    import workloads as W
    from oracle import exchange as OE
    from oracle import geometry as OG

    s = wl.spec
    need = set()
    for role, ids in faces_by_role.items():
        for f in ids:
            need.update([int(wl.coarse[f])] if role == "interpolate" else [int(x) for x in wl.fine[f]])
    need = np.array(sorted(need), dtype=np.int64)
    vals = W.patch_values(wl, need)
    patches = {int(g): vals[i] for i, g in enumerate(need)}
    jobs = []
    for role, ids in faces_by_role.items():
        for f in ids:
            seg = int(wl.segment[f]) if role == "interpolate" else 0
            cfg = OG.FaceCfg("xyz"[int(wl.normal[f])], ("negative", "positive")[int(wl.side[f])], seg, s.p, s.k, s.u)
            ex = OE.exchange_for(cfg, "order3", role)
            jobs.append((role, int(f), ex, W.face_source(wl, f, role, patches), np.empty(ex.n_out)))
    return jobs


def c5_parity(wl, plan, sweep, per, world, n_sample=16):
    """Oracle check of sampled output slots on EVERY rank: local faces, faces computed from
    received source boxes (staged) and faces whose results arrived from a peer; the worst
    error is reduced to rank 0."""
    import torch

    from oracle import exchange as OE

    rng = np.random.default_rng(5 + plan.rank)
    pick = {}
    counts = {"local": 0, "staged": 0, "received": 0}
    for role, rp in plan.items():
        groups = [("local", 0, rp.local.size), ("staged", rp.local.size, rp.local.size + rp.staged.size),
                  ("received", rp.local.size + rp.staged.size, rp.n_out)]
        for name, a, b in groups:
            if b > a:
                j = rng.choice(np.arange(a, b), min(n_sample, b - a), replace=False)
                pick.setdefault(role, []).extend(j.tolist())
                counts[name] += j.size
    order = {role: rp.out_order() for role, rp in plan.items()}
    jobs = c5_jobs(wl, {role: [order[role][j] for j in js] for role, js in pick.items()})
    st = OE.run_many([j[2] for j in jobs], [j[3] for j in jobs], [j[4] for j in jobs], cpu_threads())
    assert (st == 0).all()
    worst = 0.0
    it = iter(jobs)
    for role, js in pick.items():
        for j in js:
            _, _, _, _, want = next(it)
            got = sweep.out[role][j * per:(j + 1) * per].cpu().numpy()
            worst = max(worst, float(np.abs(got - want).max() / np.abs(want).max()))
    n = sum(counts.values())
    if world > 1:
        t = torch.tensor([worst, -float(n)] + [-float(counts[c]) for c in counts], dtype=torch.float64,
                         device=sweep.out["interpolate"].device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)  # max of worst; -max(-n) = min
        t2 = torch.tensor([float(n)] + [float(counts[c]) for c in counts], dtype=torch.float64, device=t.device)
        torch.distributed.all_reduce(t2)
        worst = float(t[0])
        n = int(t2[0])
        counts = {c: int(v) for c, v in zip(counts, t2[1:].tolist())}
    return {"sample_faces": n, "by_kind": counts, "ranks": world, "max_rel_err": worst, "tol": 1e-12,
            "ok": worst <= 1e-12}


def c5_cpu_baseline(wl, n_per_role=128, budget_s=12.0):
    """Oracle C port (reference HaloExchange.run restated) on the host cores over a sample of
    config-5 faces, repeated to fill ~budget_s of CPU time."""
    from oracle import exchange as OE

    rng = np.random.default_rng(12345)
    nf = wl.spec.n_faces
    ids = {r: np.sort(rng.choice(nf, n_per_role, replace=False)) for r in ("interpolate", "restrict")}
    jobs = c5_jobs(wl, ids)
    nth = cpu_threads()
    exs, srcs, outs = [j[2] for j in jobs], [j[3] for j in jobs], [j[4] for j in jobs]
    OE.run_many(exs, srcs, outs, nth)  # warm
    reps, t_all = 0, 0.0
    while t_all < budget_s and reps < 1000:
        t = time.perf_counter()
        st = OE.run_many(exs, srcs, outs, nth)
        t_all += time.perf_counter() - t
        reps += 1
    assert (st == 0).all()
    values = reps * sum(o.size for o in outs)
    return {"value": values / t_all, "unit": "values/s", "cores": nth, "kind": "port",
            "sample": f"{n_per_role} interpolation + {n_per_role} restriction faces of config 5 (order3), "
                      f"x {reps} repetitions = {t_all:.1f} s; oracle C restatement of HaloExchange.run "
                      f"(reference schemes.py:185-202) over {nth} OpenMP threads"}


def alg_bytes_c5(p, k, u, segments_i, n_restrict):
    """Algorithmic bytes (distinct support cells + output) of the faces of a launch."""
    b_i, f_i, _ = unit_costs("interpolate", "order3", p, k, u, list(range(9)))
    per_seg_i = {}
    from paper_2504_15814_b200.operators import HostOperator

    h = HostOperator("interpolate", "order3", p, k)
    for sgm in range(9):
        c = h.csr(segment=sgm)
        per_seg_i[sgm] = ((np.unique(c.col_indices).size + c.n_rows) * u * 8.0, 2.0 * c.nnz * u)
    b_r, f_r, _ = unit_costs("restrict", "order3", p, k, u, [None])
    bi = sum(per_seg_i[int(x)][0] for x in segments_i)
    fi = sum(per_seg_i[int(x)][1] for x in segments_i)
    return bi, fi, b_r * n_restrict, f_r * n_restrict


def run_multi(args, rank, world, local_rank):
    """Config 5: 32,768 coarse patches block-partitioned over the ranks, 196,608 faces,
    order3 interpolation + restriction of every face, fine patches drawn from the pool
    by index lists; 10% of faces have their fine patches on another rank (their source
    boxes or results cross NVLink in one grouped NCCL send/recv step, overlapped with
    local faces).  Strong scaling: the job is fixed, ranks split it."""
    import torch

    import paper_2504_15814_b200 as th
    import workloads as W
    from paper_2504_15814_b200.multigpu import NcclTransport, Support, make_rank_sweep, plan_sweep

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    t_setup = time.perf_counter()
    wl = W.describe_multi(world, scale=args.scale, straddle=args.straddle, fine_layout=args.fine_layout)
    s = wl.spec
    p, k, u = s.p, s.k, s.u
    ops = {role: th.operators.DEFAULT_CACHE.device_operator(role, "order3", p, k)
           for role in ("interpolate", "restrict")}
    support = Support.from_operators(ops["interpolate"], ops["restrict"], p, k)
    plan = plan_sweep(wl.part, wl.coarse, wl.fine, wl.segment, rank, wl.normal, wl.side, support=support)
    wl = W.build_multi(world, rank, scale=args.scale, src_elems=plan.src_elems(p, k, u), straddle=args.straddle,
                       fine_layout=args.fine_layout)
    lo = int(wl.part.bounds[rank])
    per = k * p * p * u
    if world > 1:
        torch.distributed.barrier()  # every rank is set up before the first P2P
    transport = NcclTransport(dev)
    sweep, comp = make_rank_sweep(plan, ops, support, p, k, u, wl.src, transport, wl.coarse, wl.fine, wl.normal,
                                  wl.side, wl.segment, lo)
    t_setup = time.perf_counter() - t_setup
    for _ in range(max(3, args.warmup)):
        sweep.run(comp)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.05)
    stream = torch.cuda.current_stream()
    keys = list(comp.batches)
    ev_steps = [{kk: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for kk in keys}
                for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    sampler.mark()
    t0.record(stream)
    for kk in range(args.steps):
        comp.events = ev_steps[kk]
        sweep.run(comp)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    comp.events = None
    nonfinite = comp.nonfinite()
    ms = t0.elapsed_time(t1) / args.steps
    launch_ms = {kk: statistics.mean(ev[kk][0].elapsed_time(ev[kk][1]) for ev in ev_steps) for kk in keys}
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    values = 2 * s.n_faces * per
    peak, peak_kind = peaks()
    rows = []
    from paper_2504_15814_b200.multigpu import batch_ids

    for (role, kind) in keys:
        ids = batch_ids(plan, role, kind)
        if role == "interpolate":
            byts, flops, _, _ = alg_bytes_c5(p, k, u, wl.segment[ids], 0)
        else:
            _, _, byts, flops = alg_bytes_c5(p, k, u, [], ids.size)
        byts += ops[role].info.device_bytes
        m_ = launch_ms[(role, kind)]
        gbs = byts / (m_ / 1e3) / 1e9
        rows.append({"role": role, "kind": kind, "faces": int(ids.size), "ms": round(m_, 4), "alg_bytes": int(byts),
                     "alg_GBps": round(gbs, 1), "frac_hbm": round(gbs / peak, 4),
                     "frac_8tbs": round(gbs / PEAK_NORTH_STAR, 4),
                     "csr_equiv_TFLOPs": round(flops / (m_ / 1e3) / 1e12, 2)})
    dom = max(range(len(rows)), key=lambda i: rows[i]["ms"])
    step_bytes = sum(r["alg_bytes"] for r in rows)
    res = {
        "metric": METRIC, "value": values / (ms / 1e3), "unit": "values/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: cubic polynomial field per unknown + 1e-6 N(0,1) noise, generated in HBM (seeded per "
                "64-patch group, partition-independent); fine patches drawn from the pool by index lists",
        "config": {**c5_config(s, world, args.straddle),
                   **({"fine_layout": args.fine_layout} if args.fine_layout != "random" else {})},
        "roofline": {"bound": "hbm", "kernel": f"{rows[dom]['role']}:order3 ({rows[dom]['kind']} faces)",
                     "achieved": rows[dom]["alg_GBps"], "peak": peak, "unit": "GB/s", "frac": rows[dom]["frac_hbm"],
                     "frac_8tbs": rows[dom]["frac_8tbs"], "traffic": None,
                     "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy); frac_8tbs against the "
                                  f"north star's 8 TB/s"},
        "passes": rows,
        "step_alg_GBps": round(step_bytes / (ms / 1e3) / 1e9, 1),
        "step_frac_hbm": round(step_bytes / (ms / 1e3) / 1e9 / peak, 4),
        "step_frac_8tbs": round(step_bytes / (ms / 1e3) / 1e9 / PEAK_NORTH_STAR, 4),
        "exchange": {"src_boxes_sent": int(sum(b.size for b in plan.src_send)),
                     "src_bytes_sent": int(plan.n_src_send_cells * u * 8),
                     "results_sent": {r: rp.n_send for r, rp in plan.items()},
                     "staged_faces": {r: int(rp.staged.size) for r, rp in plan.items()},
                     "rank": rank},
        "gpu_launches": args.steps * (comp.launches + (1 if sweep.pack is not None else 0)
                                      + (1 if sweep.unpack is not None else 0)),
        "nonfinite_flag": nonfinite,
        "clocks": clocks,
        "setup_s": round(t_setup, 1),
    }
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            tr = json.load(fh).get("config5", {})
        ent = tr.get(f"{rows[dom]['role']}:order3")
        if isinstance(ent, dict):
            res["roofline"]["traffic"] = round(ent["bytes"] * rows[dom]["faces"] / ent["faces"])
            res["roofline"]["traffic_source"] = ("profiles/traffic.json (dram__bytes_read.sum + dram__bytes_write.sum "
                                                 f"of one ncu --set full launch over {ent['faces']} faces, per face)")
    except (OSError, ValueError):
        pass
    if not args.no_sustained:
        sc = sustained_copy(dev, local_rank)
        res["roofline"]["sustained_copy"] = sc
        if "GBps" in sc:
            res["roofline"]["frac_sustained_copy"] = round(rows[dom]["alg_GBps"] / sc["GBps"], 4)
    if not args.no_e2e:
        res["e2e"] = run_c5_e2e(args, wl, plan, sweep, comp, ops, p, k, u, lo, dev, world)
    res["parity"] = c5_parity(wl, plan, sweep, per, world)
    if rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"] = c5_cpu_baseline(wl)
    return res


def run_c5_e2e(args, wl, plan, sweep, comp, ops, p, k, u, lo, dev, world):
    """Config 5 end to end through the C ABI with HOST buffers.

    The host holds this rank's patch pool compactly: per patch only the cells face work reads
    (the six face slabs, 2,160 of 3,375 cells at p = 9; halo edges and corners and the patch
    centre are never read), 33 GB instead of 52 GB, in memory page-locked with cudaHostRegister.
    Every step, in 16 chunks of patches: upload the chunk (th_memcpy_async into a ring of three
    staging buffers), scatter it into the device pool (th_pool_blocks), interpolate the local
    faces whose coarse patch is in the chunk, restrict the local faces whose last fine patch just
    arrived (faces ordered by their largest fine patch id), and read those results back into
    page-locked host memory (th_memcpy_async) -- upload, kernels and read-back overlap on three
    streams.  Faces that cross ranks (N > 1) go through the sweep's exchange after the upload."""
    import torch

    try:
        st = _c5_e2e_setup(wl, plan, sweep, ops, p, k, u, lo, dev, n_chunks=args.e2e_chunks)
        err = None
    except Exception as exc:  # noqa: BLE001 -- reported in the JSON line
        st, err = None, f"{type(exc).__name__}: {exc}"
    if world > 1:  # every rank set up, or none runs the leg (no rank left waiting in a collective)
        ok = torch.tensor([0.0 if err else 1.0], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
        if float(ok.item()) < 1.0 and err is None:
            err = "another rank could not set up the e2e leg"
    if err:
        if st is not None:
            st["release"]()
        return {"error": err}
    return _c5_e2e_run(args, wl, plan, sweep, comp, p, k, u, dev, world, st)


def _c5_e2e_setup(wl, plan, sweep, ops, p, k, u, lo, dev, n_chunks=16):
    import torch

    import paper_2504_15814_b200 as th
    from paper_2504_15814_b200 import _native

    lib = _native.load()
    pool = wl.pool
    E = p + 2 * k
    patch = E ** 3 * u
    per = k * p * p * u
    n_local = plan.n_local
    blocks = th.faces.pool_face_blocks(p, k, u)
    bsz = blocks[:, 1].astype(np.int64) * blocks[:, 3]
    boff = np.concatenate([[0], np.cumsum(bsz)[:-1]]).astype(np.int64)
    ce = int(bsz.sum())
    d_blocks = torch.from_numpy(blocks.ravel().copy()).to(dev)
    d_boff = torch.from_numpy(boff).to(dev)
    cb = [(n_local * c) // n_chunks for c in range(n_chunks + 1)]
    max_chunk = max(cb[c + 1] - cb[c] for c in range(n_chunks))
    staging = [torch.empty(max(1, max_chunk * ce), dtype=torch.float64, device=dev) for _ in range(3)]
    rp_i, rp_r = plan["interpolate"], plan["restrict"]
    nr = rp_r.local.size
    rout = torch.empty(max(1, nr * per), dtype=torch.float64, device=dev)  # e2e restriction results
    host_compact = np.empty(max(1, n_local * ce), dtype=np.float64)
    host_i = np.empty(max(1, rp_i.n_out * per), dtype=np.float64)
    host_r = np.empty(max(1, nr * per), dtype=np.float64)
    host_rx = np.empty(max(1, (rp_r.n_out - nr) * per), dtype=np.float64)  # staged + received (N > 1)
    reg = torch._C._cudart
    registered = []
    for a in (host_compact, host_i, host_r, host_rx):
        rc = reg.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
        if int(rc) != 0:
            raise RuntimeError(f"cudaHostRegister failed: {rc}")
        registered.append(a)
    cur = torch.cuda.current_stream(dev).cuda_stream
    for c in range(n_chunks):  # host copy of the compact pool (setup, not timed)
        a, b = cb[c], cb[c + 1]
        if b > a:
            _native.check(lib.th_pool_blocks(pool[a * patch:].data_ptr(), staging[0].data_ptr(), b - a, patch, E * u,
                                             d_blocks.data_ptr(), d_boff.data_ptr(), len(blocks), ce, 1, cur))
            _native.check(lib.th_memcpy_async(host_compact.ctypes.data + a * ce * 8, staging[0].data_ptr(),
                                              (b - a) * ce * 8, 1, cur))
            torch.cuda.synchronize()
    # interpolation: local faces are in coarse-patch order, chunk c's faces a contiguous range
    cut = np.searchsorted(wl.coarse[rp_i.local] - lo, cb)
    chunk_i = []
    for c in range(n_chunks):
        a, b = int(cut[c]), int(cut[c + 1])
        ids = rp_i.local[a:b]
        rec = th.pool_interp_faces(p, k, u, wl.coarse[ids] - lo, wl.normal[ids], wl.side[ids], wl.segment[ids],
                                   dst_offsets=np.arange(a, b, dtype=np.int64) * per) if b > a else None
        chunk_i.append((th.FaceBatch(ops["interpolate"], rec, u) if rec is not None else None, a, b))
    # restriction: local faces ordered by the chunk their last fine patch arrives in
    need = np.searchsorted(cb, wl.fine[rp_r.local].max(axis=1) - lo, side="right") - 1
    order = np.argsort(need, kind="stable")
    rcut = np.searchsorted(need[order], np.arange(n_chunks + 1))
    chunk_r = []
    for c in range(n_chunks):
        a, b = int(rcut[c]), int(rcut[c + 1])
        ids = rp_r.local[order[a:b]]
        rec = th.pool_restrict_faces(p, k, u, wl.fine[ids] - lo, wl.normal[ids], wl.side[ids],
                                     dst_offsets=np.arange(a, b, dtype=np.int64) * per) if b > a else None
        chunk_r.append((th.FaceBatch(ops["restrict"], rec, u) if rec is not None else None, a, b))

    def release():
        for a in registered:
            reg.cudaHostUnregister(a.ctypes.data)

    return dict(lib=lib, pool=pool, E=E, patch=patch, per=per, n_local=n_local, blocks=blocks, d_blocks=d_blocks,
                d_boff=d_boff, ce=ce, cb=cb, staging=staging, rp_i=rp_i, rp_r=rp_r, nr=nr, rout=rout,
                host_compact=host_compact, host_i=host_i, host_r=host_r, host_rx=host_rx, chunk_i=chunk_i,
                chunk_r=chunk_r,
                order=order, n_chunks=n_chunks, release=release)


def _c5_e2e_run(args, wl, plan, sweep, comp, p, k, u, dev, world, st):
    import torch

    from paper_2504_15814_b200 import _native

    lib, pool, E, patch, per, n_local = st["lib"], st["pool"], st["E"], st["patch"], st["per"], st["n_local"]
    blocks, d_blocks, d_boff, ce, cb = st["blocks"], st["d_blocks"], st["d_boff"], st["ce"], st["cb"]
    staging, rp_i, rp_r, nr, rout = st["staging"], st["rp_i"], st["rp_r"], st["nr"], st["rout"]
    host_compact, host_i, host_r, host_rx = st["host_compact"], st["host_i"], st["host_r"], st["host_rx"]
    chunk_i, chunk_r, order, n_chunks = st["chunk_i"], st["chunk_r"], st["order"], st["n_chunks"]
    s_in, s_run, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def d2h(host, dev_buf, a, b):
        if b > a:
            _native.check(lib.th_memcpy_async(host.ctypes.data + a * per * 8, dev_buf[a * per:].data_ptr(),
                                              (b - a) * per * 8, 1, s_out.cuda_stream))

    def run_done():
        e = torch.cuda.Event()
        e.record(s_run)
        s_out.wait_event(e)

    trace = [] if os.environ.get("TH_E2E_TRACE") else None  # diagnosis: per-chunk stream timeline

    def tr(stream, what, c):
        if trace is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            trace.append((what, c, e))

    def e2e_step():
        unpacked = [None] * n_chunks
        if trace is not None:
            trace.clear()
            tr(s_in, "t0", -1)
        for c in range(n_chunks):
            a, b = cb[c], cb[c + 1]
            st = staging[c % 3]
            if c >= 3:
                s_in.wait_event(unpacked[c - 3])  # the staging buffer is free again
            if b > a:
                _native.check(lib.th_memcpy_async(st.data_ptr(), host_compact.ctypes.data + a * ce * 8,
                                                  (b - a) * ce * 8, 0, s_in.cuda_stream))
            tr(s_in, "h2d", c)
            ev = torch.cuda.Event()
            ev.record(s_in)
            s_run.wait_event(ev)
            if b > a:
                _native.check(lib.th_pool_blocks(pool[a * patch:].data_ptr(), st.data_ptr(), b - a, patch, E * u,
                                                 d_blocks.data_ptr(), d_boff.data_ptr(), len(blocks), ce, 0,
                                                 s_run.cuda_stream))
            unpacked[c] = torch.cuda.Event()
            unpacked[c].record(s_run)
            batch, ia, ib = chunk_i[c]
            if batch is not None:
                batch.launch(wl.src, sweep.out["interpolate"], stream=s_run.cuda_stream)
                run_done()  # interpolation results leave while the chunk's restriction runs
                d2h(host_i, sweep.out["interpolate"], ia, ib)
                tr(s_out, "d2h_i", c)
            batch, ra, rb = chunk_r[c]
            if batch is not None:
                batch.launch(wl.src, rout, stream=s_run.cuda_stream)
                tr(s_run, "run", c)
                run_done()
                d2h(host_r, rout, ra, rb)
                tr(s_out, "d2h_r", c)
        with torch.cuda.stream(s_run):  # faces that cross ranks (none at N = 1)
            sweep.pre(comp)
            sweep.post(comp)
            run_done()
        d2h(host_i, sweep.out["interpolate"], rp_i.local.size, rp_i.n_out)
        if rp_r.n_out > nr:
            _native.check(lib.th_memcpy_async(host_rx.ctypes.data, sweep.out["restrict"][nr * per:].data_ptr(),
                                              (rp_r.n_out - nr) * per * 8, 1, s_out.cuda_stream))

    e2e_step()
    torch.cuda.synchronize()
    times = []
    for _ in range(max(1, args.e2e_steps)):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        e2e_step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t)
    if trace:
        t0e = trace[0][2]
        for what, c, e in trace[1:]:
            if c % 8 == 7 or c == n_chunks - 1:
                print(f"e2e trace chunk {c:3d} {what:6s} {t0e.elapsed_time(e):8.1f} ms", file=sys.stderr)
    t_step = statistics.median(times)
    if world > 1:
        tt = torch.tensor([t_step], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_step = float(tt.item())
    # the host results equal the device-resident sweep's (windows of 64 faces)
    agree = True
    oi = sweep.out["interpolate"]
    for a in (0, rp_i.local.size // 2, max(0, rp_i.local.size - 64)):
        b = min(rp_i.local.size, a + 64)
        agree &= bool(np.array_equal(host_i[a * per:b * per], oi[a * per:b * per].cpu().numpy()))
    orr = sweep.out["restrict"]
    for j in (0, nr // 2, max(0, nr - 1)):
        if nr:
            slot = int(order[j])  # e2e position j holds local restriction face order[j]
            agree &= bool(np.array_equal(host_r[j * per:(j + 1) * per], orr[slot * per:(slot + 1) * per].cpu().numpy()))
    st["release"]()
    values = 2 * wl.spec.n_faces * per
    return {"value": values / t_step, "unit": "values/s",
            "h2d_bytes_per_step": int(n_local * ce * 8),
            "d2h_bytes_per_step": int((rp_i.n_out + nr + sum(r.size for r in rp_r.recv) + rp_r.staged.size) * per * 8),
            "ms_per_step": round(t_step * 1e3, 1), "steps": len(times), "matches_device_run": agree,
            "how": f"per step, {n_chunks} chunks of patches: the compact host pool (only the six face slabs of every "
                   "patch that face work reads, 2,160 of 3,375 cells; host memory page-locked with "
                   "cudaHostRegister) -> staging ring (th_memcpy_async) -> device pool (th_pool_blocks); "
                   "interpolation of the faces whose coarse patch arrived, restriction of the faces whose last "
                   "fine patch arrived (th_apply_faces), results -> page-locked host memory (th_memcpy_async); "
                   "upload, kernels and read-back overlap on three streams; wall clock with device sync, max "
                   "over ranks"}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(args, wl, passes):
    """Oracle port (C restatement of the reference HaloExchange.run) on a sample of
    this workload's faces, on the host cores; also a parity check of our outputs."""
    import torch

    import workloads as W
    from oracle import exchange as OE
    from oracle import geometry as OG

    s = wl.spec
    p, k, u = s.p, s.k, s.u
    rng = np.random.default_rng(12345)
    nth = cpu_threads()
    jobs = []
    fc = wl.faces
    sample_i = rng.choice(wl.interp_ids, min(args.cpu_sample, wl.interp_ids.size), replace=False) \
        if wl.interp_ids.size else np.zeros(0, dtype=np.int64)
    sample_r = rng.choice(np.arange(wl.restrict_ids.size), min(args.cpu_sample, wl.restrict_ids.size),
                          replace=False) if wl.restrict_ids.size else np.zeros(0, dtype=np.int64)
    per_r = 2 * k * 9 * p * p * u
    tgt = k * p * p * u
    src_i = W.interp_source_boxes(wl, sample_i).cpu().numpy() if sample_i.size else None
    worst = 0.0
    values = 0
    for ps in passes:
        outs_dev = ps["out"]
        if ps["role"] == "interpolate":
            pos = {f: i for i, f in enumerate(wl.interp_ids)}
            for j, f in enumerate(sample_i):
                cfg = OG.FaceCfg("xyz"[fc.normal[f]], ("negative", "positive")[fc.side[f]], int(fc.segment[f]), p, k, u)
                ex = OE.exchange_for(cfg, ps["scheme"], "interpolate")
                got = outs_dev[pos[f] * tgt:(pos[f] + 1) * tgt].cpu().numpy()
                jobs.append((ex, src_i[j], np.empty(ex.n_out), got))
        else:
            for j in sample_r:
                f = wl.restrict_ids[j]
                cfg = OG.FaceCfg("xyz"[fc.normal[f]], ("negative", "positive")[fc.side[f]], 0, p, k, u)
                ex = OE.exchange_for(cfg, ps["scheme"], "restrict")
                src = wl.fine[j * per_r:(j + 1) * per_r].cpu().numpy()
                got = outs_dev[j * tgt:(j + 1) * tgt].cpu().numpy()
                jobs.append((ex, src, np.empty(ex.n_out), got))
    t = time.perf_counter()
    status = OE.run_many([j[0] for j in jobs], [j[1] for j in jobs], [j[2] for j in jobs], nth)
    dt = time.perf_counter() - t
    assert (status == 0).all()
    for ex, src, want, got in jobs:
        values += want.size
        worst = max(worst, float(np.abs(got - want).max() / np.abs(want).max()))
    base = {"value": values / dt, "unit": "values/s", "cores": nth, "kind": "port",
            "sample": f"{len(jobs)} face-passes ({sample_i.size} interp faces x interp passes + {sample_r.size} "
                      f"restrict faces x restrict passes) of this workload; oracle C restatement of "
                      f"HaloExchange.run over {nth} OpenMP threads; {dt:.2f} s"}
    parity = {"sample_face_passes": len(jobs), "max_rel_err": worst, "tol": 1e-12, "ok": worst <= 1e-12}
    return base, parity


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU path (oracle port; the reference is Python
# and cannot travel to the GPU box) on the host cores, same config and metric
# ---------------------------------------------------------------------------

def c5_host_source(wl, f, role, rng):
    """Host (numpy) world-layout source buffer of config-5 face f for one role: the field at
    the pool cells it reads (coarse patch box, or the nine fine patches' blocks) + fresh noise.
    The CPU reference arm builds its inputs with this (it must not need a GPU)."""
    s = wl.spec
    p, k, u, m, H = s.p, s.k, s.u, wl.m, wl.H
    n, sd = int(wl.normal[f]), int(wl.side[f])
    t1, t2 = [d for d in range(3) if d != n]

    def block(pid, lo3, ext):
        pos = np.array([pid % m, (pid // m) % m, pid // (m * m)], dtype=np.float64)
        ax = [np.arange(lo3[d], lo3[d] + ext[d]) - k + 0.5 for d in range(3)]
        zz, yy, xx = np.meshgrid(ax[2], ax[1], ax[0], indexing="ij")
        xyz = (pos * p + np.stack([xx.ravel(), yy.ravel(), zz.ravel()], axis=1)) * H
        v = wl.fld.eval_numpy(xyz) + 1e-6 * rng.standard_normal((xyz.shape[0], u))
        return v.reshape(ext[2], ext[1], ext[0], u)

    if role == "interpolate":
        lo3, ext = [k, k, k], [p, p, p]
        lo3[n], ext[n] = (p if sd == 0 else 0), 2 * k
        return np.ascontiguousarray(block(int(wl.coarse[f]), lo3, ext).reshape(-1))
    ext = [3 * p, 3 * p, 3 * p]
    ext[n] = 2 * k
    box = np.zeros((ext[2], ext[1], ext[0], u))
    for b in range(9):
        lo3, e = [k, k, k], [p, p, p]
        lo3[n], e[n] = (0 if sd == 0 else p), 2 * k
        off = [0, 0, 0]
        off[t1], off[t2] = (b % 3) * p, (b // 3) * p
        box[off[2]:off[2] + e[2], off[1]:off[1] + e[1], off[0]:off[0] + e[0]] = block(int(wl.fine[f, b]), lo3, e)
    return box.reshape(-1)


def run_reference(args):
    import workloads as W
    from oracle import exchange as OE
    from oracle import geometry as OG

    rng = np.random.default_rng(777)
    nth = cpu_threads()
    jobs = []
    if args.config == 5:
        wl = W.describe_multi(args.gpus, scale=args.scale, straddle=args.straddle)
        s = wl.spec
        p, k, u = s.p, s.k, s.u
        n_sample = min(args.cpu_sample, s.n_faces)
        for role in ("interpolate", "restrict"):
            for f in np.sort(rng.choice(s.n_faces, n_sample, replace=False)):
                seg = int(wl.segment[f]) if role == "interpolate" else 0
                cfg = OG.FaceCfg("xyz"[int(wl.normal[f])], ("negative", "positive")[int(wl.side[f])], seg, p, k, u)
                ex = OE.exchange_for(cfg, "order3", role)
                jobs.append((ex, c5_host_source(wl, f, role, rng), np.empty(ex.n_out)))
        config = c5_config(s, args.gpus, args.straddle)
        passes = ("interpolate:order3", "restrict:order3")
    else:
        wl = W.describe(args.config)
        s = wl.spec
        p, k, u = s.p, s.k, s.u
        n_sample = min(args.cpu_sample, s.n_faces)
        fc = wl.faces
        for role, scheme in s.passes:
            ids = wl.interp_ids if role == "interpolate" else wl.restrict_ids
            pick = np.sort(rng.choice(ids, min(n_sample, ids.size), replace=False))
            for f in pick:
                seg = int(fc.segment[f]) if role == "interpolate" else 0
                cfg = OG.FaceCfg("xyz"[fc.normal[f]], ("negative", "positive")[fc.side[f]], seg, p, k, u)
                ex = OE.exchange_for(cfg, scheme, role)
                jobs.append((ex, W.host_sources(wl, int(f), role, rng), np.empty(ex.n_out)))
        config = ours_config(s, args.gpus, wl)
        passes = tuple(f"{r}:{sc}" for r, sc in s.passes)
    exs, srcs, outs = zip(*jobs)

    def step():
        st = OE.run_many(exs, srcs, outs, nth)
        assert (st == 0).all()

    for _ in range(max(1, args.warmup)):
        step()
    t = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t) / args.steps
    values = sum(o.size for o in outs)
    value = values / dt
    sample = (f"{len(jobs)} face-passes per step ({n_sample} faces per pass: {', '.join(passes)}) drawn from "
              f"config{s.config}; oracle C restatement of HaloExchange.run (reference schemes.py:185-202) over "
              f"{nth} OpenMP threads; values/s of the sample = the job's rate (faces are independent)")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "values/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.config == 5 else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (same field and face generators, host numpy)", "config": config,
            "cpu_baseline": {"value": value, "unit": "values/s", "cores": nth, "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "values/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    res = run_multi(args, rank, world, local_rank) if args.config == 5 else run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
