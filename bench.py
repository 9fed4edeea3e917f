"""Benchmark of the B200 halo interpolation / restriction path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one pass of every (role, scheme) of BASELINE.json's config over all
of its faces, inputs resident in HBM.  Default: config 2 (configs[1]): p=9,
k=3, u=59, 1,024 coarse patches, 4,096 faces; tensor_linear + order2
interpolation and tensor_linear + order2 restriction (full coarse face) of
every face.  Prints ONE JSON line (rank 0).  See DESIGN.md §Measurement.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0, help="shrink patch / face counts (tuning runs only)")
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-chunks", type=int, default=16, help="pipeline chunks of the e2e leg")
    ap.add_argument("--cpu-sample", type=int, default=256, help="faces in the CPU baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
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

def run_ours(args, rank, world, local_rank):
    import torch

    import paper_2504_15814_b200 as th
    import workloads as W

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    wl = W.build(args.config, rank=rank, scale=args.scale)
    s = wl.spec
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
                        ps["batch"].launch(ps["src"], ps["out"], stream=side.cuda_stream, check_flag=False)
            for ps in passes:
                if ps["role"] != "interpolate":
                    ps["batch"].launch(ps["src"], ps["out"], check_flag=False)
            stream.wait_stream(side)
            return
        for i, ps in enumerate(passes):
            if evs is not None:
                evs[i].record(stream)
            ps["batch"].launch(ps["src"], ps["out"], check_flag=False)
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
    sampler.mark()
    t0.record(stream)
    for kk in range(args.steps):
        step(ev_all[kk])
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    total_ms = t0.elapsed_time(t1)
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
                          "fp64_TFLOPs": round(ps["flops"] / (ms / 1e3) / 1e12, 2)})
    dom = max(range(len(passes)), key=lambda i: per_pass_ms[i])
    result = {
        "metric": METRIC, "value": value, "unit": "values/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded field (BASELINE config text) sampled at cell centres + 1e-6 N(0,1), generated in HBM",
        "config": {"workload": f"config{s.config}: {s.name}", "p": p, "k": k, "u": u, "coarse_patches": s.n_patches,
                   "faces": s.n_faces, "passes": [f"{r}:{sc}" for r, sc in s.passes],
                   "layout": "coarse pool (p+2k)^3 AoS + per-face fine restriction slabs (world layout)",
                   "l2": f"inputs {(wl.pool.numel() + (wl.fine.numel() if wl.fine is not None else 0)) * 8 / 1e9:.1f} GB"
                         " >> 126 MB L2 (no flush needed)",
                   "parallelism": f"weak: {world} independent shard(s)",
                   **({"overlap": "interpolation passes on a side stream"} if args.overlap else {})},
        "roofline": {"bound": "hbm", "kernel": f"{passes[dom]['role']}:{passes[dom]['scheme']}",
                     "achieved": pass_rows[dom]["alg_GBps"], "peak": peak, "unit": "GB/s",
                     "frac": round(pass_rows[dom]["alg_GBps"] / peak, 4), "traffic": None,
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


def run_multi(args, rank, world, local_rank):
    """Config 5: 32,768 coarse patches block-partitioned over the ranks, 196,608 faces,
    order3 interpolation + restriction of every face, fine patches drawn from the pool
    by index lists, 10% of faces with their fine patches on another rank (results of
    those cross NVLink in one grouped NCCL send/recv step, overlapped with local faces).
    Strong scaling: the job is fixed, ranks split it."""
    import torch

    import paper_2504_15814_b200 as th
    import workloads as W
    from paper_2504_15814_b200.multigpu import GpuCompute, Sweep, plan_sweep

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    wl = W.build_multi(world, rank, scale=args.scale)
    s = wl.spec
    p, k, u = s.p, s.k, s.u
    plans = plan_sweep(wl.part, wl.coarse, wl.fine, wl.segment, rank)
    per = k * p * p * u
    lo = int(wl.part.bounds[rank])
    ops = {role: th.operators.DEFAULT_CACHE.device_operator(role, "order3", p, k) for role in plans}

    def make_records(role, ids):
        if role == "interpolate":
            return th.pool_interp_faces(p, k, u, wl.coarse[ids] - lo, wl.normal[ids], wl.side[ids], wl.segment[ids])
        return th.pool_restrict_faces(p, k, u, wl.fine[ids] - lo, wl.normal[ids], wl.side[ids])

    comp = GpuCompute(plans, make_records, ops, {"interpolate": wl.pool, "restrict": wl.pool}, u)
    sweep = Sweep(plans, per, dev, torch.float64)
    for _ in range(max(3, args.warmup)):
        sweep.run(comp)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.05)
    stream = torch.cuda.current_stream()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    sampler.mark()
    t0.record(stream)
    for _ in range(args.steps):
        sweep.run(comp)
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    n_faces = s.n_faces
    values = 2 * n_faces * per
    b_i, f_i, _ = unit_costs("interpolate", "order3", p, k, u, list(range(9)))
    b_r, f_r, _ = unit_costs("restrict", "order3", p, k, u, [None])
    step_bytes = n_faces * (b_i + b_r) / world
    peak, peak_kind = peaks()
    cross = {r: int(sum(x.size for x in pl.send)) for r, pl in plans.items()}
    res = {
        "metric": METRIC, "value": values / (ms / 1e3), "unit": "values/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic cubic field + 1e-6 noise in HBM; fine patches drawn from the pool by index lists",
        "config": {"workload": f"config5: {s.name}", "p": p, "k": k, "u": u, "coarse_patches": s.n_patches,
                   "faces": n_faces, "passes": ["interpolate:order3", "restrict:order3"],
                   "parallelism": f"{world} ranks, block-partitioned patches, NCCL P2P for cross faces",
                   "cross_faces_sent_rank0": cross},
        "roofline": {"bound": "hbm", "kernel": "interpolate+restrict:order3 (whole sweep, per rank)",
                     "achieved": round(step_bytes / (ms / 1e3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(step_bytes / (ms / 1e3) / 1e9 / peak, 4), "traffic": None,
                     "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy)"},
        "gpu_launches": args.steps * comp.launches,
        "clocks": clocks,
    }
    if rank == 0 and not args.no_cpu:
        res["parity"] = multi_parity(wl, plans, sweep, per)
    return res


def multi_parity(wl, plans, sweep, per, n_sample=24):
    """Oracle check of a sample of faces computed and kept on this rank."""
    from oracle import exchange as OE
    from oracle import geometry as OG

    s = wl.spec
    p, k, u = s.p, s.k, s.u
    E = p + 2 * k
    lo = int(wl.part.bounds[0])
    pool = wl.pool.view(-1, E, E, E, u)
    rng = np.random.default_rng(5)
    worst = 0.0
    for role, plan in plans.items():
        pick = rng.choice(plan.local.size, min(n_sample, plan.local.size), replace=False)
        for j in pick:
            f = int(plan.local[j])
            n, sd = int(wl.normal[f]), int(wl.side[f])
            t1, t2 = [d for d in range(3) if d != n]
            if role == "interpolate":
                lo3, ext = [k, k, k], [p, p, p]
                lo3[n], ext[n] = (p if sd == 0 else 0), 2 * k
                c = int(wl.coarse[f]) - lo
                src = pool[c, lo3[2]:lo3[2] + ext[2], lo3[1]:lo3[1] + ext[1], lo3[0]:lo3[0] + ext[0]].cpu().numpy().reshape(-1)
                seg = int(wl.segment[f])
            else:
                ext = [3 * p, 3 * p, 3 * p]
                ext[n] = 2 * k
                world_box = np.zeros((ext[2], ext[1], ext[0], u))
                for b in range(9):
                    lo3, e = [k, k, k], [p, p, p]
                    lo3[n], e[n] = (0 if sd == 0 else p), 2 * k
                    blk = pool[int(wl.fine[f, b]) - lo, lo3[2]:lo3[2] + e[2], lo3[1]:lo3[1] + e[1],
                               lo3[0]:lo3[0] + e[0]].cpu().numpy()
                    off = [0, 0, 0]
                    off[t1], off[t2] = (b % 3) * p, (b // 3) * p
                    world_box[off[2]:off[2] + e[2], off[1]:off[1] + e[1], off[0]:off[0] + e[0]] = blk
                src = world_box.reshape(-1)
                seg = 0
            cfg = OG.FaceCfg("xyz"[n], ("negative", "positive")[sd], seg, p, k, u)
            ex = OE.exchange_for(cfg, "order3", role)
            want = np.empty(ex.n_out)
            ex.run(src, want)
            got = sweep.out[role][j * per:(j + 1) * per].cpu().numpy()
            worst = max(worst, float(np.abs(got - want).max() / np.abs(want).max()))
    return {"sample_faces": 2 * n_sample, "max_rel_err": worst, "tol": 1e-12, "ok": worst <= 1e-12}


def run_e2e(args, wl, passes, dev, world):
    """Same metric through the C ABI with HOST buffers: every step ships each face's
    reference source buffer (pinned host, world layout) to HBM, applies all passes and
    copies the results back, chunked over 3 streams so PCIe overlaps the kernels.  Only
    the normal layers the operators read are shipped (th_operator_support_layers:
    3 of the 6 source layers for linear / order2), one strided cudaMemcpy2D/3DAsync per
    (chunk, orientation) group via th_copy_box_layers."""
    import ctypes

    import torch

    import paper_2504_15814_b200 as th
    import workloads as W
    from paper_2504_15814_b200 import _native

    lib = _native.load()
    s = wl.spec
    p, k, u = s.p, s.k, s.u
    fc = wl.faces
    orient = fc.normal * 2 + fc.side
    ord_i = wl.interp_ids[np.argsort(orient[wl.interp_ids], kind="stable")]
    ord_r = wl.restrict_ids[np.argsort(orient[wl.restrict_ids], kind="stable")]
    n_i, n_r = ord_i.size, ord_r.size
    per_i, per_r = 2 * k * p * p * u, 2 * k * 9 * p * p * u
    tgt = k * p * p * u
    # host copies of the per-face reference source buffers, in orientation order
    h_i = torch.empty(max(1, n_i * per_i), dtype=torch.float64, pin_memory=True)
    for a in range(0, n_i, 1024):
        b = min(n_i, a + 1024)
        h_i[a * per_i:b * per_i].copy_(W.interp_source_boxes(wl, ord_i[a:b]).reshape(-1))
    h_r = torch.empty(max(1, n_r * per_r), dtype=torch.float64, pin_memory=True)
    if n_r:
        pos = {f: j for j, f in enumerate(wl.restrict_ids)}
        fine = wl.fine.view(n_r, per_r)
        for a in range(0, n_r, 512):
            b = min(n_r, a + 512)
            idx = torch.as_tensor([pos[f] for f in ord_r[a:b]], device=fine.device)
            h_r[a * per_r:b * per_r].copy_(fine.index_select(0, idx).reshape(-1))
    d_i = torch.empty(max(1, n_i * per_i), dtype=torch.float64, device=dev)
    d_r = torch.empty(max(1, n_r * per_r), dtype=torch.float64, device=dev)
    # normal layers each role's operators read (union over the passes)
    layers = {}
    for ps in passes:
        lo, cnt = ps["batch"].op.support_layers()
        a, b = layers.get(ps["role"], (lo, lo + cnt))
        layers[ps["role"]] = (min(a, lo), max(b, lo + cnt))
    n_chunks = max(1, args.e2e_chunks)
    outs_d = [torch.empty(ps["out"].numel(), dtype=torch.float64, device=dev) for ps in passes]
    outs_h = [torch.empty(ps["out"].numel(), dtype=torch.float64, pin_memory=True) for ps in passes]
    chunks = []
    h2d = 0
    for c in range(n_chunks):
        ia, ib = n_i * c // n_chunks, n_i * (c + 1) // n_chunks
        ra, rb = n_r * c // n_chunks, n_r * (c + 1) // n_chunks
        copies = []
        for role, order, a0, b0, per, host, devb, t_ext in (
                ("interpolate", ord_i, ia, ib, per_i, h_i, d_i, p), ("restrict", ord_r, ra, rb, per_r, h_r, d_r, 3 * p)):
            if role not in layers or b0 <= a0:
                continue
            lo, hi = layers[role]
            o = orient[order[a0:b0]]
            cuts = np.flatnonzero(np.diff(o)) + 1
            for g0, g1 in zip(np.r_[0, cuts], np.r_[cuts, o.size]):
                nrm, side = int(o[g0]) // 2, int(o[g0]) % 2
                wlo = lo if side == 0 else 2 * k - hi
                off = int(a0 + g0) * per * 8
                copies.append((int(host.data_ptr() + off), int(devb.data_ptr() + off), int(g1 - g0), nrm, 2 * k,
                               t_ext, int(wlo), int(hi - lo)))
                h2d += int(g1 - g0) * (hi - lo) * t_ext * t_ext * u * 8
        batches = []
        for ps in passes:
            op = ps["batch"].op
            if ps["role"] == "interpolate":
                ids = ord_i[ia:ib]
                rec = th.slab_faces("interpolate", p, k, u, fc.normal[ids], fc.side[ids], segments=fc.segment[ids],
                                    src_offsets=np.arange(ia, ib) * per_i, dst_offsets=np.arange(ia, ib) * tgt)
                lo_, hi_ = ia, ib
            else:
                ids = ord_r[ra:rb]
                rec = th.slab_faces("restrict", p, k, u, fc.normal[ids], fc.side[ids],
                                    src_offsets=np.arange(ra, rb) * per_r, dst_offsets=np.arange(ra, rb) * tgt)
                lo_, hi_ = ra, rb
            batches.append((th.FaceBatch(op, rec, u) if hi_ > lo_ else None, lo_, hi_))
        chunks.append(dict(copies=copies, batches=batches))
    s_in, s_run, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_step():
        for ch in chunks:
            for (hs, ds, n, nrm, n_ext, t_ext, wlo, cnt) in ch["copies"]:
                _native.check(lib.th_copy_box_layers(hs, ds, n, nrm, n_ext, t_ext, u, wlo, cnt, 0, s_in.cuda_stream))
            e_in = torch.cuda.Event()
            e_in.record(s_in)
            s_run.wait_event(e_in)
            with torch.cuda.stream(s_run):
                for ps, od, (batch, lo_, hi_) in zip(passes, outs_d, ch["batches"]):
                    if batch is not None:
                        batch.launch(d_i if ps["role"] == "interpolate" else d_r, od, check_flag=False)
                e_run = torch.cuda.Event()
                e_run.record(s_run)
            s_out.wait_event(e_run)
            with torch.cuda.stream(s_out):
                for od, oh, (batch, lo_, hi_) in zip(outs_d, outs_h, ch["batches"]):
                    if hi_ > lo_:
                        oh[lo_ * tgt:hi_ * tgt].copy_(od[lo_ * tgt:hi_ * tgt], non_blocking=True)

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
    t_step = statistics.median(times)
    if world > 1:
        tt = torch.tensor([t_step], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_step = float(tt.item())
    # the e2e results must equal the device-resident run's (same faces, orientation order)
    agree = True
    for ps, oh in zip(passes, outs_h):
        order = ord_i if ps["role"] == "interpolate" else ord_r
        ids = wl.interp_ids if ps["role"] == "interpolate" else wl.restrict_ids
        pos = {f: j for j, f in enumerate(ids)}
        j = np.array([pos[f] for f in order[:64]])
        ref = ps["out"].view(-1, tgt)[torch.as_tensor(j, device=ps["out"].device)].cpu()
        agree &= bool(torch.equal(ref.reshape(-1), oh[: 64 * tgt]))
    values = sum(ps["values"] for ps in passes) * world
    return {"value": values / t_step, "unit": "values/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(sum(ps["out"].numel() for ps in passes) * 8),
            "ms_per_step": round(t_step * 1e3, 2), "matches_device_run": agree,
            "how": "pinned host buffers of the per-face reference source layouts -> only the operators' normal "
                   "support layers shipped (th_copy_box_layers, strided 2D/3D async copies) -> th_apply_faces -> "
                   "pinned host outputs; 16 chunks pipelined over copy/compute/copy streams; wall clock with "
                   "device sync"}


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

def run_reference(args):
    import workloads as W
    from oracle import exchange as OE
    from oracle import geometry as OG

    wl = W.describe(args.config)
    s = wl.spec
    p, k, u = s.p, s.k, s.u
    rng = np.random.default_rng(777)
    nth = cpu_threads()
    n_sample = min(args.cpu_sample, s.n_faces)
    fc = wl.faces
    jobs = []
    for role, scheme in s.passes:
        ids = wl.interp_ids if role == "interpolate" else wl.restrict_ids
        pick = np.sort(rng.choice(ids, min(n_sample, ids.size), replace=False))
        for f in pick:
            seg = int(fc.segment[f]) if role == "interpolate" else 0
            cfg = OG.FaceCfg("xyz"[fc.normal[f]], ("negative", "positive")[fc.side[f]], seg, p, k, u)
            ex = OE.exchange_for(cfg, scheme, role)
            jobs.append((ex, W.host_sources(wl, int(f), role, rng), np.empty(ex.n_out)))
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
    sample = (f"{len(jobs)} face-passes per step ({n_sample} faces per pass) drawn from config{s.config}; "
              f"oracle C restatement of HaloExchange.run (reference schemes.py:185-202) over {nth} OpenMP threads")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "values/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (same generator, host numpy)",
            "config": {"workload": f"config{s.config}: {s.name}", "p": p, "k": k, "u": u,
                       "passes": [f"{r}:{sc}" for r, sc in s.passes]},
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
