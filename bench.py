#!/usr/bin/env python
"""Benchmark of the gDist hot path on B200 (BASELINE.json metric).

Workload (config 2 / 3 of BASELINE.json): two interlocked rings of
2500 x 1500 quads = 7,500,000 triangles each.  One step on rank r is one
frame f of the 1000-frame rotation sequence (scenes.ring_frame_transforms):
refit(A_f), refit(B_f), exact min-distance query.  Frames are sharded
f = step * N + rank, so per-GPU work is fixed as N grows (weak scaling, no
collective in the loop).  `value` = whole-job milliseconds per min-distance
query (refits included): max-over-ranks device time of the K steps / (K N).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--impl reference` times the reference's own CPU path on the box's host cores:
the unmodified reference package (pure Python + numpy) installed into
baseline/_ref (git-ignored, shipped by gpurun), driven through its public API
on the same frames with all host threads, bounded steps; the oracle port
(oracle/, a numpy restatement) stands in only if baseline/_ref is absent.

`--gpus N` without a torchrun environment (WORLD_SIZE unset) launches the N
ranks itself (torch.distributed.run, one process per GPU, 127.0.0.1); under
torchrun it never re-launches.  Extra keys of the line: the max query of the
same frames (`max_query_ms`, its own roofline), refit + min + max per frame
(config 3), and for N > 1 the single query split over the N ranks
(`split`, max over ranks).  `--dry-run` exercises the launcher, the process
group, the max-over-ranks reduction and the result all-gather without a GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "ms per min/max distance query, 2×7.5M-tri rings; frames/s at 1/2/4/8 GPUs"
PAPER_MS = 0.38  # rings min query, 2 x 7.5M, RTX 4090


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--nu", type=int, default=2500)
    ap.add_argument("--nv", type=int, default=1500)
    ap.add_argument("--kind", choices=["min", "max"], default="min")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=150.0, help="seconds for CPU legs")
    ap.add_argument("--profile-only", action="store_true", help="a short run for ncu (no baselines)")
    ap.add_argument("--no-max", action="store_true", help="skip the max-query keys")
    ap.add_argument("--dry-run", action="store_true", help="launcher / collective plumbing only (no GPU work)")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs (1, 4, 5)")
    return ap.parse_args()


def self_launch(args) -> int:
    """`--gpus N` outside torchrun: start the N ranks (one process per GPU)
    with torch.distributed.run on 127.0.0.1; rank 0 prints the line."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(args.gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=str(REPO)).returncode


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_dry(args):
    """The N > 1 plumbing without GPU work: process group (NCCL when every
    rank has a GPU, else gloo), barrier, a max-over-ranks reduction of a
    per-rank "time" and the frame-result all-gather of parallel.run_frames;
    rank 0 prints one line."""
    import torch
    import torch.distributed as dist

    from paper_2411_11244_b200 import parallel

    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n_frames = 4 * world + 1
    res = parallel.run_frames(n_frames, lambda f: (float(f) * 0.5, f, 2 * f))
    ok = bool(np.all(res[:, 0] == np.arange(n_frames) * 0.5) and np.all(res[:, 2] == 2 * np.arange(n_frames)))
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": world, "max_over_ranks": float(t.item()),
                          "frames_gathered": n_frames, "gather_ok": ok}))
    if world > 1:
        dist.destroy_process_group()
    return ok


def workload_name(args):
    return (f"rings 2 x {args.nu * args.nv * 2} tris (configs 2/3): a step is one frame f = step * N + rank of the "
            f"1000-frame rotation sequence = refit A + refit B + {args.kind} distance query")


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region, in
    process through NVML (a sample every ~0.5 ms; nvidia-smi as fallback)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, reasons_mask)
        self._stop = threading.Event()
        self._t = None
        self._h = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _sample(self):
        if self._nv is not None:
            nv = self._nv
            sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            self.rows.append((float(sm), float(self._max), int(mask)))
            return
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                              "clocks_event_reasons.active", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=5)
        if out.returncode == 0 and out.stdout.strip():
            a = [x.strip() for x in out.stdout.strip().split(",")]
            self.rows.append((float(a[0]), float(a[1]), int(a[2], 16)))

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                pass
            self._stop.wait(0.0005 if self._nv is not None else 0.1)

    def __enter__(self):
        # the launching thread holds the GIL between its ctypes calls: a short
        # switch interval lets the sampler run every ~0.5 ms during the region
        self._switch = sys.getswitchinterval()
        sys.setswitchinterval(1e-4)
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        sys.setswitchinterval(self._switch)
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for r in self.rows for name, bit in self.REASONS.items() if r[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml" if self._nv is not None else "nvidia-smi"}


def query_bytes(res, depth_a, depth_b):
    """Algorithmic bytes of one query: per iteration
    front_in*12 + front_in*(2^ka + 2^kb)*24 + front_out*12; narrow phase
    leaf_pairs*(12 + 2*8) + narrow_pairs*72."""
    da = db = 0
    total = 0
    expand = 0
    leaf_pairs = 0
    for s in res.iterations:
        ka, kb = min(s.k, depth_a - da), min(s.k, depth_b - db)
        b = s.front_in * 12 + s.front_in * ((1 << ka) + (1 << kb)) * 24 + s.front_out * 12
        expand += b
        if s.front_out == 0 and s.k == max(depth_a - da, depth_b - db):
            leaf_pairs = (s.front_in << (ka + kb)) - s.culled
        da += ka
        db += kb
    narrow = leaf_pairs * (12 + 16) + res.narrow_pairs * 72
    total = expand + narrow
    return {"expand_bytes": expand, "narrow_bytes": narrow, "total_bytes": total, "leaf_pairs": leaf_pairs,
            "narrow_flops": res.narrow_pairs * (2100 if res.kind == "min" else 72)}


def traverse_roofline(res, phases, bvh_a, bvh_b, kind):
    """Roofline of k_traverse (the dominant kernel): SURVEY 8(d) algorithmic
    bytes of this query / its CUDA-event time, against the measured HBM peak;
    traffic = ncu DRAM bytes of one launch (profiles/kernel_traffic.json)."""
    qb = query_bytes(res, bvh_a.depth, bvh_b.depth)
    hbm, _, src = peaks()
    expand_ms = phases["expand"]
    achieved = qb["expand_bytes"] / (expand_ms * 1e-3) / 1e9 if expand_ms > 0 else None
    traffic = None
    tf = REPO / "profiles" / "kernel_traffic.json"
    if tf.exists():
        per = json.loads(tf.read_text())["per_launch_dram_bytes"]
        traffic = per.get(f"k_traverse_{kind}", per.get("k_traverse" if kind == "min" else "k_traverse_max"))
    return {"bound": "hbm", "kernel": f"k_traverse_{kind} (all expansion iterations of one query, one launch)",
            "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": (achieved / hbm) if achieved else None,
            "traffic": traffic, "peak_source": src, "algorithmic_bytes": qb["expand_bytes"], "kernel_ms": expand_ms,
            "note": "algorithmic bytes (SURVEY 8d) count every box load; most hit L2 (traffic = ncu DRAM bytes "
                    "of one launch, profiles/kernel_traffic.json)"}


def measure_query(md, _lib, a, b, ta, tb, kind, cfg, reps=5):
    """One query of a config: median device ms over `reps` launches (CUDA
    events; a chunked query -- several traversal rounds -- is timed through
    its collect, host gaps between rounds included), the answer, and the
    k_traverse roofline from a profiled run (single-round queries)."""
    import ctypes as C

    import torch

    pq = md.PreparedQuery(a, b, ta, tb, cfg, kind)
    r = pq.run()
    rounds = int(pq.res.rounds)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(reps):
        torch.cuda.synchronize()
        s.record()
        pq.launch()
        if rounds > 1:
            pq.collect()
        e.record()
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
    if rounds == 1:
        pq.collect()
    out = {"query_ms": round(float(np.median(ms)), 6), "distance": r.distance,
           "witness": [r.witness.tri_a, r.witness.tri_b] if r.witness else None, "rounds": rounds,
           "expanded_pairs": r.expanded_pairs, "narrow_pairs": r.narrow_pairs, "band_pairs": r.band_pairs,
           "peak_front": r.peak_front}
    if rounds == 1:
        L = _lib.lib()
        L.gd_set_profiling(1)
        pq.launch()
        res = pq.collect()
        ph = (C.c_float * 5)()
        L.gd_query_phase_ms(ph, 5)
        L.gd_set_profiling(0)
        phases = {"init": ph[0], "expand": ph[1], "narrow": ph[2], "exact": ph[3], "final": ph[4]}
        out["phases_ms"] = {k: round(v, 6) for k, v in phases.items()}
        rl = traverse_roofline(res, phases, ta, tb, kind)
        rl["traffic"] = None  # the committed ncu DRAM capture is of the rings workload only
        out["roofline"] = rl
        # the narrow phase against the FP32 CUDA-core peak (per
        # tested triangle pair ~2100 flop for min, 72 for max; nominal peak)
        flop = res.narrow_pairs * (2100 if kind == "min" else 72)
        if phases["narrow"] > 0:
            tf = flop / (phases["narrow"] * 1e-3) / 1e12
            out["narrow_fp32"] = {"bound": "fp32", "achieved": round(tf, 3), "peak": FP32_PEAK_TFLOPS,
                                  "unit": "TFLOP/s", "frac": round(tf / FP32_PEAK_TFLOPS, 4),
                                  "peak_source": "nominal (148 SM x 128 lanes x 2 x 1.965 GHz)",
                                  "flop": int(flop), "narrow_ms": round(phases["narrow"], 6)}
    else:
        out["roofline"] = None
        out["roofline_note"] = "chunked traversal (the front outgrew the arena): per-round phases not timed"
    return out


def configs_section(md, _lib):
    """BASELINE.json's other configs on this GPU (rank 0, N = 1), each
    query with its own device time, answer and k_traverse roofline:
    config 1 (tori 2 x 10K, min + max, with the unmodified reference on the
    host cores: time and distance / witness parity), config 4 (nested
    shells 2 x 2M, min + max; no front cap), config 5 (rings 100K -> 30M
    total triangles, min + max; the 8-GPU split of config 5 needs the 8-GPU
    box, see the split keys of an N > 1 run)."""
    import torch

    out = {}
    t0 = time.perf_counter()
    # config 1
    a, b = md.gen_scene("interlocked-rings", {"nu": 100, "nv": 50})
    ta, tb = md.build_f12(a), md.build_f12(b)
    ref = load_reference()
    c1 = {}
    for kind in ("min", "max"):
        rec = measure_query(md, _lib, a, b, ta, tb, kind, md.EngineConfig())
        if ref is not None:
            A, B = ref.TriangleMesh(a.vertices, a.triangles), ref.TriangleMesh(b.vertices, b.triangles)
            RA, RB = ref.build_f12(A), ref.build_f12(B)
            run = ref.run_min_query if kind == "min" else ref.run_max_query
            times, rr = [], None
            for _ in range(3):
                t1 = time.perf_counter()
                rr = run(A, B, RA, RB, ref.EngineConfig(threads=os.cpu_count() or 1))
                times.append((time.perf_counter() - t1) * 1e3)
            rec["reference"] = {"ms": round(min(times), 3), "threads": os.cpu_count(), "kind": "reference",
                                "sample": "the whole config-1 query, unmodified reference package (baseline/_ref), "
                                          "best of 3",
                                "distance_equal": rr.distance == rec["distance"],
                                "witness_equal": [rr.witness.tri_a, rr.witness.tri_b] == rec["witness"]}
        c1[kind] = rec
    out["config1_tori_2x10K"] = c1
    # config 4
    a, b = md.gen_scene("nested-shells", {"lat": 1001, "lon": 1000, "r_inner": 0.8, "r_outer": 0.81})
    ta, tb = md.build_f12(a), md.build_f12(b)
    cfg4 = md.EngineConfig(front_hard_cap=1 << 40)
    out["config4_nested_shells_2x2M"] = {kind: measure_query(md, _lib, a, b, ta, tb, kind, cfg4, reps=3)
                                         for kind in ("min", "max")}
    del ta, tb
    torch.cuda.empty_cache()
    # config 5
    c5 = {}
    for nu, nv in [(250, 100), (500, 150), (1000, 250), (1500, 500), (2500, 1000), (5000, 1500)]:
        tz, tbase = md.ring_pair_base(nu, nv)
        A, B = md.build_f12(tz), md.build_f12(tbase)
        xa, xb = md.ring_frame_transforms(0)
        a, b = md.apply_transform(tz, xa), md.apply_transform(tbase, xb)
        md.refit(A, a)
        md.refit(B, b)
        cfg = md.EngineConfig(front_hard_cap=1 << 28)
        c5[f"{2 * tz.n_triangles}"] = {kind: measure_query(md, _lib, a, b, A, B, kind, cfg) for kind in ("min", "max")}
        del A, B
        torch.cuda.empty_cache()
    out["config5_rings_sweep_total_tris"] = c5
    out["wall_s"] = round(time.perf_counter() - t0, 2)
    out["note"] = "device ms per query (CUDA events, median); rooflines as the headline's (k_traverse algorithmic bytes)"
    return out


def frame_graph_section(md, bvh_a, bvh_b, prepared, W, K, cfg, stream, dist, red_dev, seq):
    """Config 3 through its public API, run_sequence_minmax: each frame
    (refit A + refit B + min + max + the two record copies) is one CUDA graph
    replay (FrameGraph); two graphs alternate on two streams so frame f + 1's
    refits overlap frame f's narrow / exact phases.  Device ms per frame =
    CUDA events on the calling stream around the whole K-frame call (the call
    joins its streams into it), max over ranks; e2e = the host wall clock of
    the same call (transforms in, every frame's records read back); plus one
    graph replayed back to back without the overlap."""
    import torch

    a0, b0, _ = prepared[0]
    fg = md.FrameGraph(a0, b0, bvh_a, bvh_b, ("min", "max"), cfg)
    try:
        for i in range(W):
            a, b, _ = prepared[i]
            fg.run(a, b)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for i in range(W, W + K):
            a, b, _ = prepared[i]
            fg.launch(a, b)
        e.record(stream)
        torch.cuda.synchronize()
        single_ms = s.elapsed_time(e) / K
    finally:
        fg.close()
    tz, tb, xfs = seq  # the base meshes and the timed frames' transforms
    md.run_sequence_minmax(tz, tb, bvh_a, bvh_b, xfs[:2], ("min", "max"), cfg)  # its two graphs, captured once
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    t0 = time.perf_counter()
    out = md.run_sequence_minmax(tz, tb, bvh_a, bvh_b, xfs, ("min", "max"), cfg)
    e.record(stream)
    torch.cuda.synchronize()
    host_ms = (time.perf_counter() - t0) * 1e3 / K
    dev_ms = s.elapsed_time(e) / K
    from paper_2411_11244_b200.parallel import release_frame_graphs

    release_frame_graphs()
    # the job's last frame through the plain API: the same answers
    a, b = md.apply_transform(tz, xfs[-1][0]), md.apply_transform(tb, xfs[-1][1])
    md.refit(bvh_a, a)
    md.refit(bvh_b, b)
    ref = (md.run_min_query(a, b, bvh_a, bvh_b, cfg), md.run_max_query(a, b, bvh_a, bvh_b, cfg))
    if dist:
        t = torch.tensor([dev_ms, host_ms, single_ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms, host_ms, single_ms = float(t[0].item()), float(t[1].item()), float(t[2].item())
    return {"frame_min_max_graph_ms": round(dev_ms, 6), "frame_min_max_graph_e2e_ms": round(host_ms, 6),
            "frame_min_max_graph_single_ms": round(single_ms, 6),
            "frame_min_max_graph_note": "config 3 through run_sequence_minmax: per frame one CUDA graph replay "
                                        "(refit A + refit B + min + max + record copies), two graphs alternating "
                                        "on two streams so frame f+1's refits overlap frame f's narrow / exact "
                                        "phases; device ms = CUDA events around the whole call / K, e2e = its host "
                                        "wall clock (records read back per frame); _single_ms: one graph "
                                        "replayed back to back",
            "frame_graph_answers_equal": bool(ref[0].distance == out["min"][-1][0]
                                              and ref[1].distance == out["max"][-1][0])}


def max_section(md, _lib, bvh_a, bvh_b, prepared, W, K, cfg, stream, dist, red_dev, seq):
    """The max query of the same frames: its own time and roofline, and the
    whole config-3 frame (refit A + refit B + min + max) back to back on the
    device (CUDA events on the launching stream, max over ranks)."""
    import ctypes as C

    import torch

    plans = [md.PreparedQuery(a, b, bvh_a, bvh_b, cfg, "max") for a, b, _ in prepared]
    for i in range(W):
        a, b, pq = prepared[i]
        bvh_a._device_refit(a)
        bvh_b._device_refit(b)
        plans[i].launch()
        plans[i].collect()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(K)]
    if dist:
        dist.barrier()
    for j, i in enumerate(range(W, W + K)):
        a, b, pq = prepared[i]
        ev[j][0].record(stream)
        bvh_a._device_refit(a)
        bvh_b._device_refit(b)
        ev[j][1].record(stream)
        pq.launch()
        ev[j][2].record(stream)
        plans[i].launch()
        ev[j][3].record(stream)
    torch.cuda.synchronize()
    max_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in ev]))
    seq_frame_ms = float(np.mean([e[0].elapsed_time(e[3]) for e in ev]))
    # the same frames with the two queries as one group (md.launch_group):
    # traversals back to back, the two narrow / exact chains side by side
    # (a group's queries need distinct workspaces: two private plans, bound
    # to each frame's moved meshes)
    a0, b0, _ = prepared[0]
    gmin = md.PreparedQuery(a0, b0, bvh_a, bvh_b, cfg, "min", private_workspace=True)
    gmax = md.PreparedQuery(a0, b0, bvh_a, bvh_b, cfg, "max", private_workspace=True)
    gev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(K)]
    for j, i in enumerate(list(range(W)) + list(range(W, W + K))):
        a, b, pq = prepared[i]
        if j >= W:
            gev[j - W][0].record(stream)
        bvh_a._device_refit(a)
        bvh_b._device_refit(b)
        gmin.bind(a, b)
        gmax.bind(a, b)
        md.launch_group([gmin, gmax])
        if j >= W:
            gev[j - W][1].record(stream)
    torch.cuda.synchronize()
    frame_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in gev]))
    # the last frame's grouped answers equal its separate ones
    gres = (gmin.collect(), gmax.collect())
    sres = []
    for pq in (prepared[-1][2], plans[-1]):  # the boxes describe the last frame
        pq.launch()
        sres.append(pq.collect())
    group_equal = all(g.distance == r.distance and (g.witness.tri_a, g.witness.tri_b) == (r.witness.tri_a, r.witness.tri_b)
                      for g, r in zip(gres, sres))
    del gmin, gmax
    if dist:
        t = torch.tensor([max_ms, frame_ms, seq_frame_ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        max_ms, frame_ms, seq_frame_ms = float(t[0].item()), float(t[1].item()), float(t[2].item())
    # answers and the profiled phases of the last frame's max query
    L = _lib.lib()
    a, b, _ = prepared[-1]
    bvh_a._device_refit(a)
    bvh_b._device_refit(b)
    L.gd_set_profiling(1)
    plans[-1].launch()
    res = plans[-1].collect()
    ph = (C.c_float * 5)()
    L.gd_query_phase_ms(ph, 5)
    L.gd_set_profiling(0)
    phases = {"init": ph[0], "expand": ph[1], "narrow": ph[2], "exact": ph[3], "final": ph[4]}
    graph = frame_graph_section(md, bvh_a, bvh_b, prepared, W, K, cfg, stream, dist, red_dev, seq)
    return {**graph, "max_query_ms": round(max_ms, 6), "max_phases_ms": {k: round(v, 6) for k, v in phases.items()},
            "max_distance": res.distance, "max_witness": [res.witness.tri_a, res.witness.tri_b],
            "max_roofline": traverse_roofline(res, phases, bvh_a, bvh_b, "max"),
            "frame_min_max_ms": round(frame_ms, 6),
            "frame_min_max_sequential_ms": round(seq_frame_ms, 6),
            "frame_min_max_group_answers_equal": bool(group_equal),
            "frame_min_max_note": "config 3 per frame: refit A + refit B + min + max as one query group (traversals "
                                  "back to back, the two narrow / exact chains side by side on forked streams); "
                                  "_sequential_ms: the two queries back to back on one stream"}, res


def split_section(md, tz, tb, bvh_a, bvh_b, cfg, kind, dist, red_dev, backend, frame=7, reps=5):
    """One query (frame `frame`, every rank the same) split over the N ranks
    (parallel.run_split_query): ownership by ancestor-pair hash, exact parts
    combined in one all-gather; the three bound exchanges (none, CUDA IPC
    peer atomics inside the kernels, all-reduce between traversal rounds).  Time = max over ranks of the mean wall time per collective
    query (the all-gather's synchronisation included), beside the same query
    on one GPU (rank 0's plain query)."""
    import torch

    from paper_2411_11244_b200 import parallel

    xa, xb = md.ring_frame_transforms(frame)
    a, b = md.apply_transform(tz, xa), md.apply_transform(tb, xb)
    md.refit(bvh_a, a)
    md.refit(bvh_b, b)
    run = md.run_min_query if kind == "min" else md.run_max_query
    single = run(a, b, bvh_a, bvh_b, cfg)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        run(a, b, bvh_a, bvh_b, cfg)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    out = {"frame": frame, "single_gpu_query_ms": round(float(np.median(ts)), 6), "modes": {}}
    modes = [("rank-local bound", "none"), ("bound shared over CUDA IPC (peer atomics, the default)", "ipc"),
             ("bound all-reduced between one-sweep traversal rounds", "allreduce")]
    for name, share in modes:
        try:
            for _ in range(2):
                r = parallel.run_split_query(a, b, bvh_a, bvh_b, kind, cfg, bound_exchange=share)
            assert r.distance == single.distance, (r.distance, single.distance)
            times = []
            for _ in range(reps):
                dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = parallel.run_split_query(a, b, bvh_a, bvh_b, kind, cfg, bound_exchange=share)
                times.append((time.perf_counter() - t0) * 1e3)
            mine = torch.tensor([float(np.median(times)), float(r.expanded_pairs)], device=red_dev)
            allv = [torch.zeros_like(mine) for _ in range(dist.get_world_size())]
            dist.all_gather(allv, mine)
            ms = max(float(v[0]) for v in allv)
            work = [float(v[1]) for v in allv]
            out["modes"][name] = {"ms": round(ms, 6), "expanded_pairs_per_rank": work,
                                  "busiest_rank_share_of_single": round(max(work) / max(1, single.expanded_pairs), 4),
                                  "distance_equal_to_single_gpu": bool(r.distance == single.distance)}
        except Exception as exc:  # report, never hide
            out["modes"][name] = {"error": repr(exc)}
    parallel.release_split_plans()
    out["note"] = ("the traversal's top levels (above the split level) are replicated on every rank; they are "
                   "latency bound (fronts < 25K entries), so the split pays only on large queries")
    out["backend"] = backend
    return {"split": out}


FP32_PEAK_TFLOPS = 74.4


def peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1965.0, "fallback"


# ---------------------------------------------------------------------------
def run_ours(args):
    import torch

    import paper_2411_11244_b200 as md
    from paper_2411_11244_b200 import _lib

    world, rank, local = dist_env()
    # one process per GPU over NCCL; more ranks than visible GPUs (a
    # functional check of the N > 1 path on one device) falls back to gloo
    n_dev = torch.cuda.device_count()
    if n_dev == 0:
        # the product path is the CUDA one; there is no CPU fallback to time
        raise SystemExit("bench.py: no CUDA device visible (the reference arm is --impl reference)")
    backend = "nccl" if world <= n_dev else "gloo"
    local = local % n_dev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    red_dev = dev if backend == "nccl" else torch.device("cpu")  # device of the max-over-ranks reductions
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    t0 = time.time()
    tz, tb = md.ring_pair_base(args.nu, args.nv)
    bvh_a, bvh_b = md.build_f12(tz), md.build_f12(tb)
    setup_s = time.time() - t0
    cfg = md.EngineConfig(front_hard_cap=1 << 27)
    K, W, N = args.steps, args.warmup, world

    def frame_meshes(f):
        xa, xb = md.ring_frame_transforms(f % 1000)
        return md.apply_transform(tz, xa), md.apply_transform(tb, xb)

    # prepared queries per frame (device views resolved outside the timing)
    frames = [(s * N + rank) for s in range(W + K)]
    prepared = []
    for f in frames:
        a, b = frame_meshes(f)
        md.refit(bvh_a, a)
        md.refit(bvh_b, b)
        prepared.append((a, b, md.PreparedQuery(a, b, bvh_a, bvh_b, cfg, args.kind)))
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(W + K)]

    def step(i):
        a, b, pq = prepared[i]
        e0, e1, e2 = ev[i]
        e0.record(stream)
        bvh_a._device_refit(a)
        bvh_b._device_refit(b)
        e1.record(stream)
        pq.launch()
        e2.record(stream)

    # pipelined frames (the timed `value`): the refit of frame i runs on a
    # second stream once frame i-1's traversal has read the boxes, so it
    # overlaps frame i-1's narrow and exact phases (gd_query_async_ev)
    rstream = torch.cuda.Stream()
    trav = [torch.cuda.Event() for _ in range(W + K)]
    refd = [torch.cuda.Event() for _ in range(W + K)]

    def pipe_step(i, first):
        a, b, pq = prepared[i]
        with torch.cuda.stream(rstream):
            if not first:
                rstream.wait_event(trav[i - 1])
            bvh_a._device_refit(a)
            bvh_b._device_refit(b)
            refd[i].record(rstream)
        stream.wait_event(refd[i])
        pq.launch(traversal_done=trav[i])

    def pipe_pass(lo, hi, start_ev=None, end_ev=None):
        if start_ev is not None:
            start_ev.record(stream)
        rstream.wait_stream(stream)
        for i in range(lo, hi):
            pipe_step(i, i == lo)
        stream.wait_stream(rstream)
        if end_ev is not None:
            end_ev.record(stream)

    for i in range(W):
        step(i)
        prepared[i][2].collect()
    pipe_pass(0, W)
    torch.cuda.synchronize()
    launches0 = _lib.lib().gd_launch_count()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_start, s_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        pipe_pass(W, W + K, start, end)
        torch.cuda.synchronize()
        launches = _lib.lib().gd_launch_count() - launches0
        # the same frames one after another (per-phase breakdown)
        s_start.record(stream)
        for i in range(W, W + K):
            step(i)
        s_end.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    region_ms = start.elapsed_time(end)
    serial_ms = s_start.elapsed_time(s_end)
    refit_ms = [ev[i][0].elapsed_time(ev[i][1]) for i in range(W, W + K)]
    query_ms = [ev[i][1].elapsed_time(ev[i][2]) for i in range(W, W + K)]
    # results of every timed query (read after the region)
    results = []
    for i in range(W, W + K):
        a, b, pq = prepared[i]
        # re-run to read back stats (the timed launches share one workspace)
        bvh_a._device_refit(a)
        bvh_b._device_refit(b)
        pq.launch()
        results.append(pq.collect())
    if dist:
        t = torch.tensor([region_ms, serial_ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        region_ms, serial_ms = float(t[0].item()), float(t[1].item())

    # phase breakdown + roofline on one extra (untimed) query of the last frame
    L = _lib.lib()
    L.gd_set_profiling(1)
    a, b, pq = prepared[-1]
    bvh_a._device_refit(a)
    bvh_b._device_refit(b)
    pq.launch()
    res = pq.collect()
    import ctypes as C

    ph = (C.c_float * 5)()
    L.gd_query_phase_ms(ph, 5)
    L.gd_set_profiling(0)
    phases = {"init": ph[0], "expand": ph[1], "narrow": ph[2], "exact": ph[3], "final": ph[4]}
    roofline = traverse_roofline(res, phases, bvh_a, bvh_b, args.kind)

    # the max query of the same frames (config 3 is min + max per frame)
    max_keys, max_res = {}, None
    if not args.no_max and args.kind == "min" and not args.profile_only:
        max_keys, max_res = max_section(md, _lib, bvh_a, bvh_b, prepared, W, K, cfg, stream, dist, red_dev,
                                        (tz, tb, [md.ring_frame_transforms(f % 1000)
                                                  for f in range(W * N, (W + K) * N)]))
    # one query split over the N ranks, max over ranks
    split_keys = {}
    if N > 1 and not args.profile_only:
        split_keys = split_section(md, tz, tb, bvh_a, bvh_b, cfg, args.kind, dist, red_dev, backend)

    # e2e through the public API: run_sequence over this job's frames (host
    # transforms in, every frame's (distance, tri_a, tri_b) back on the host;
    # refits pipelined against the previous frame's narrow / exact phases,
    # one result read-back per frame, one all-gather at the end)
    seq_w = [md.ring_frame_transforms(f % 1000) for f in range(0, W * N)]
    seq = [md.ring_frame_transforms(f % 1000) for f in range(W * N, (W + K) * N)]
    md.run_sequence(tz, tb, bvh_a, bvh_b, seq_w, args.kind, cfg)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t1 = time.perf_counter()
    seq_res = md.run_sequence(tz, tb, bvh_a, bvh_b, seq, args.kind, cfg)
    e2e_wall_ms = (time.perf_counter() - t1) * 1e3
    for j, i in enumerate(range(W, W + K)):
        assert seq_res[j * N + rank][0] == results[i - W].distance
    if dist:
        t = torch.tensor([e2e_wall_ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_wall_ms = float(t.item())
    e2e_step_ms = e2e_wall_ms / K  # per step of one rank; whole job divides by N below

    value = region_ms / (K * N)
    clocks = clk.summary()
    out = None
    if rank == 0:
        out = {
            "metric": METRIC,
            "value": round(value, 6),
            "unit": "ms/query",
            "n_gpus": N,
            "steps": K,
            "warmup": W,
            "ms_per_step": round(region_ms / K, 6),
            "ms_per_step_unpipelined": round(serial_ms / K, 6),
            "higher_is_better": False,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32 traversal + f64 exact pass",
            "data": "synthetic (interlocked tori, rotation sequence frames)",
            "config": {"workload": workload_name(args),
                       "execution": "frames pipelined: the refit of frame f+1 runs on a second stream and overlaps "
                                    "frame f's narrow / exact phases",
                       "nu": args.nu, "nv": args.nv, "kind": args.kind, "precision": 64,
                       "parallelism": f"frames sharded over {N} rank(s), no data-path collective; one all-gather "
                                      f"of per-frame results ({backend})" if N > 1 else "1 GPU",
                       "l2": "inputs larger than L2 (2 x 200 MB node boxes rewritten by each step's refits)"},
            "query_ms": round(float(np.mean(query_ms)), 6),
            "paper_query_ms_rtx4090": PAPER_MS,
            "query_vs_paper": round(float(np.mean(query_ms)) / PAPER_MS, 4),
            "query_ms_min": round(float(np.min(query_ms)), 6),
            "refit_ms": round(float(np.mean(refit_ms)), 6),
            "frames_per_s": round(1000.0 / value, 3),
            "phases_ms": {k: round(v, 6) for k, v in phases.items()},
            "distance": results[-1].distance,
            "witness": [results[-1].witness.tri_a, results[-1].witness.tri_b],
            "iterations": len(res.iterations),
            "expanded_pairs": res.expanded_pairs,
            "narrow_pairs": res.narrow_pairs,
            "band_pairs": res.band_pairs,
            "peak_front": res.peak_front,
            "roofline": roofline,
            "e2e": {"value": round(e2e_step_ms / N, 6), "unit": "ms/query", "h2d_bytes_per_step": 2 * 96,
                    "d2h_bytes_per_step": C.sizeof(_lib.GdResult) + 64 * C.sizeof(_lib.GdIterStat),
                    "note": "public API, host wall clock: run_sequence over the job's K*N frames (apply_transform x2 "
                            "+ refit x2 + min query per frame, refits pipelined, result record + stats read back per "
                            "frame, one all-gather); frame transforms are host inputs"},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "setup_s": round(setup_s, 2),
            **max_keys,
            **split_keys,
        }
    if dist:
        dist.barrier()
    return out, (tz, tb, bvh_a, bvh_b, frames[W:], results, max_res)


# ---------------------------------------------------------------------------
# CPU legs: the UNMODIFIED reference package (pure Python + numpy, pip-installed
# into baseline/_ref, which gpurun ships to the box) through its own public API;
# the oracle port (oracle/, test infrastructure) only when baseline/_ref is absent.
def load_reference():
    src = REPO / "baseline" / "_ref"
    if not (src / "meshdist" / "__init__.py").exists():
        return None
    sys.path.insert(0, str(src))
    import meshdist

    assert Path(meshdist.__file__).resolve().is_relative_to(src.resolve()), meshdist.__file__
    return meshdist


class CpuLeg:
    """One step of the reference path on the host: apply_transform + refit of
    both meshes for frame f, then run_min_query / run_max_query.  The tree
    topology comes from our exact-pairing build (bit-equal to the reference's
    greedy, tests/test_abi_host.py); the reference's own O(n^2) pairing cannot
    build 7.5M triangles (hard part 1)."""

    def __init__(self, md, tz, tbm, bvh_a, bvh_b, kind, workers):
        self.md, self.kind, self.workers = md, kind, workers
        self.ref = load_reference()
        self.kind_label = "reference" if self.ref is not None else "port"
        if self.ref is not None:
            R = self.ref
            self.A0 = R.TriangleMesh(tz.vertices, tz.triangles)
            self.B0 = R.TriangleMesh(tbm.vertices, tbm.triangles)

            def tree(b):
                n = b.n_nodes
                return R.F12Bvh(np.empty((n, 3)), np.empty((n, 3)), np.asarray(b.leaf_tris).copy(),
                                np.asarray(b.prim_order).copy(), int(b.depth))

            self.ta, self.tb = tree(bvh_a), tree(bvh_b)
            # front_hard_cap raised as in the GPU run: at the default 2^24 the
            # reference raises FrontOverflowError on this workload (query.py:375)
            self.cfg = R.EngineConfig(threads=workers, front_hard_cap=1 << 27)
        else:
            from oracle import meshdist_oracle as oracle

            self.oracle = oracle
            self.tz, self.tbm = tz, tbm

            def tree(b):
                return oracle.Tree(np.empty((b.n_nodes, 3)), np.empty((b.n_nodes, 3)), np.asarray(b.leaf_tris),
                                   np.asarray(b.prim_order), b.depth)

            self.ta, self.tb = tree(bvh_a), tree(bvh_b)

    def describe(self):
        if self.ref is not None:
            return f"unmodified reference package (baseline/_ref, numpy, EngineConfig(threads={self.workers}))"
        return f"oracle port of the reference (oracle/, numpy, {self.workers} threads)"

    def frame(self, f, kind=None):
        """(distance, tri_a, tri_b) of frame f's query (default: the leg's kind)."""
        kind = kind or self.kind
        xa, xb = self.md.ring_frame_transforms(f % 1000)
        if self.ref is not None:
            R = self.ref
            a = R.apply_transform(self.A0, R.RigidTransform(xa.rotation, xa.translation))
            b = R.apply_transform(self.B0, R.RigidTransform(xb.rotation, xb.translation))
            R.refit(self.ta, a)
            R.refit(self.tb, b)
            run = R.run_min_query if kind == "min" else R.run_max_query
            r = run(a, b, self.ta, self.tb, self.cfg)
            self.last = (a, b)
            return r.distance, r.witness.tri_a, r.witness.tri_b
        o = self.oracle
        va = o.transform_vertices(self.tz.vertices, xa.rotation, xa.translation)
        vb = o.transform_vertices(self.tbm.vertices, xb.rotation, xb.translation)
        o.fill_boxes(self.ta, va, self.tz.triangles)
        o.fill_boxes(self.tb, vb, self.tbm.triangles)
        pa = o.triangle_points(va, self.tz.triangles)
        pb = o.triangle_points(vb, self.tbm.triangles)
        r = o.run_query(self.ta, self.tb, pa, pb, kind, o.Config(workers=self.workers, front_hard_cap=1 << 27))
        self.last = (pa, pb)
        return r.distance, r.tri_a, r.tri_b

    def pair_distance(self, kind, ta, tb):
        """The reference's own arithmetic on one triangle pair of the last
        frame (bounds.py batch_tri_tri_*): classifies a witness tie."""
        if self.ref is not None:
            from meshdist import bounds as rb

            a, b = self.last
            pa, pb = a.triangle_points()[[ta]], b.triangle_points()[[tb]]
            return float((rb.batch_tri_tri_min if kind == "min" else rb.batch_tri_tri_max)(pa, pb)[0][0])
        pa, pb = self.last
        return float((self.oracle.tri_tri_min if kind == "min" else self.oracle.tri_tri_max)(
            pa[[ta]], pb[[tb]])[0][0])


class _Topology:
    def __init__(self, leaf_tris, prim_order):
        self.leaf_tris, self.prim_order = leaf_tris, prim_order
        self.n_nodes = 2 * len(leaf_tris) - 1
        self.depth = len(leaf_tris).bit_length() - 1


def host_topology(mesh):
    """build_f12's topology (bvh.py:267-289) on the host, for the reference
    arm's untimed setup: the oracle's Morton order + surface areas and its
    O(n log n) C restatement of the greedy pairing (oracle/pairing.c,
    bit-equal to the reference's greedy, tests/test_oracle_golden.py) -- no
    product code on this arm."""
    from oracle import meshdist_oracle as oracle

    V, T = mesh.vertices, mesh.triangles
    _, order = oracle.morton_order(V, T)
    P = V[T]
    n = len(T)
    sa = oracle.pair_surface_areas(order, P.min(axis=1), P.max(axis=1))
    return _Topology(oracle.leaves_from_pairs(order, oracle.greedy_pairs_fast(sa, n), n), order)


def cpu_baseline(args, ctx, budget):
    """The reference on the box's host cores, same frame as the GPU's last
    timed step (SURVEY.md 8(d) protocol, bounded): threads = all cores, best
    of up to 3 (one warm-up excluded when the budget allows), and threads = 1
    once; the GPU's answer checked against it -- distance, witness (equal, or
    a documented tie: the reference arithmetic on the GPU's pair gives the
    same distance) -- and the max query of the same frame likewise."""
    import paper_2411_11244_b200 as md

    tz, tbm, bvh_a, bvh_b, frames, results, max_res = ctx
    f = frames[-1]
    workers = os.cpu_count() or 1
    leg = CpuLeg(md, tz, tbm, bvh_a, bvh_b, args.kind, workers)
    t_start = time.perf_counter()
    times, out = [], None
    while len(times) < 3:
        t0 = time.perf_counter()
        out = leg.frame(f)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget / 3:
            break
    gpu = results[-1]

    def classify(kind, ref, g):
        d, ta, tb = ref
        if (g.witness.tri_a, g.witness.tri_b) == (ta, tb):
            return "equal"
        same = leg.pair_distance(kind, g.witness.tri_a, g.witness.tri_b) == d
        return "tie (reference arithmetic on the GPU pair gives the same distance)" if same else "MISMATCH"

    rec = {"value": round(min(times) * 1e3, 3), "unit": "ms/query", "cores": workers, "kind": leg.kind_label,
           "sample": f"frame f={f} of the same workload: refit A+B + {args.kind} query, {leg.describe()}; "
                     f"best of {len(times)}",
           "runs_ms": [round(t * 1e3, 1) for t in times], "cpu_model": cpu_model(), "nproc": workers,
           "distance_equal_to_gpu": bool(out[0] == gpu.distance),
           "witness": classify(args.kind, out, gpu), "witness_ref": [out[1], out[2]],
           "witness_gpu": [gpu.witness.tri_a, gpu.witness.tri_b]}
    # one thread (the reference's default EngineConfig(threads=1), query.py:57-58)
    if time.perf_counter() - t_start < budget:
        leg1 = CpuLeg(md, tz, tbm, bvh_a, bvh_b, args.kind, 1)
        t0 = time.perf_counter()
        o1 = leg1.frame(f)
        rec["threads_1_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
        rec["threads_1_distance_equal"] = bool(o1[0] == out[0])
    # the max query of the same frame, full scale
    if max_res is not None and time.perf_counter() - t_start < 2 * budget:
        t0 = time.perf_counter()
        om = leg.frame(f, "max")
        rec["max_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
        rec["max_distance_equal_to_gpu"] = bool(om[0] == max_res.distance)
        rec["max_witness"] = classify("max", om, max_res)
    return rec


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return None
    import paper_2411_11244_b200 as md

    tz, tbm = md.ring_pair_base(args.nu, args.nv)
    # tree topology on the host (untimed setup, no device work on this arm)
    bvh_a, bvh_b = host_topology(tz), host_topology(tbm)
    workers = os.cpu_count() or 1
    leg = CpuLeg(md, tz, tbm, bvh_a, bvh_b, args.kind, workers)
    N = args.gpus
    W = min(args.warmup, 1)
    times = []
    t_start = time.perf_counter()
    s = 0
    while s < W + args.steps:
        f = s * N
        t0 = time.perf_counter()
        leg.frame(f)
        dt = time.perf_counter() - t0
        if s >= W:
            times.append(dt)
        s += 1
        if time.perf_counter() - t_start > args.cpu_budget and times:
            break
    value = float(np.mean(times)) * 1e3
    extra = {}
    if args.kind == "min" and not args.no_max and time.perf_counter() - t_start < 1.5 * args.cpu_budget:
        # the max query of one frame (config 3 is min + max per frame)
        t0 = time.perf_counter()
        leg.frame(0, "max")
        extra["max_ms_per_query"] = round((time.perf_counter() - t0) * 1e3, 3)
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "ms/query",
        "n_gpus": N,
        "steps": len(times),
        "warmup": W,
        "ms_per_step": round(value, 3),
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (interlocked tori, rotation sequence frames)",
        "config": {"workload": workload_name(args),
                   "execution": "frames one after another on the host (the reference's stock, synchronous path)",
                   "nu": args.nu, "nv": args.nv, "kind": args.kind, "precision": 64},
        "cpu_baseline": {"value": round(value, 3), "unit": "ms/query", "cores": workers, "kind": leg.kind_label,
                         "sample": f"{len(times)} frame steps (bounded to {args.cpu_budget:.0f} s) of the same "
                                   f"workload, {leg.describe()}", "cpu_model": cpu_model()},
        "e2e": {"value": round(value, 3), "unit": "ms/query", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "topology": "tree topology from the oracle's C restatement of the reference's greedy pairing "
                    "(oracle/pairing.c; the reference's own O(n^2) pairing cannot build 7.5M triangles), untimed",
        **extra,
    }


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.dry_run:
        sys.exit(0 if run_dry(args) else 1)
    if args.impl == "reference":
        out = run_reference(args)
        if out is not None:
            print(json.dumps(out))
        return
    out, ctx = run_ours(args)
    world, rank, _ = dist_env()
    if rank == 0 and out is not None:
        if not args.no_cpu_baseline and not args.profile_only and world == 1:
            try:
                out["cpu_baseline"] = cpu_baseline(args, ctx, args.cpu_budget)
            except Exception as exc:  # report, never hide
                out["cpu_baseline"] = {"value": None, "error": repr(exc)}
        if not args.no_configs and not args.profile_only and world == 1:
            try:
                import paper_2411_11244_b200 as md
                from paper_2411_11244_b200 import _lib

                out["configs"] = configs_section(md, _lib)
            except Exception as exc:  # report, never hide
                out["configs"] = {"error": repr(exc)}
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
