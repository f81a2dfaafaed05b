#!/usr/bin/env python
"""Benchmark of the B200 point-cloud -> elevation-map update path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C4] [--impl b200|reference]

A step is one map update (relief_map_integrate semantics) with one synthetic frame of the
workload (default C4: 128-ring LiDAR, 1,000,064 points, into a 1000x1000 @0.04 m map with the
default pipeline incl. ray-cast cleanup, drift compensation, overlap clearance, normals and
geometric traversability). Frames are rendered by the library's scene simulator (bit-identical
to the reference simulator); the map evolves across steps as in a real mission. Both arms cycle
the same number of distinct frames (N_FRAMES) with the same stamps.

Legs of the b200 arm (one JSON line from rank 0):
  value      points/s with the frame already resident in HBM (relief_gpu_map_integrate_device),
             device time from CUDA events recorded on the library's own stream, L2 flushed
             (256 MiB write) before every step, summed over exactly K steps, max over ranks.
  e2e        the same metric through the drop-in C ABI relief_map_integrate with the frame in
             pinned host memory: host->device copy of the points and the device->host read of
             the scan statistics inside the timed region (host clock around the synchronous call).
  e2e_pageable  the same with the frame in ordinary (pageable) numpy memory.
  configs    every BASELINE config (C1, C2, C3, headline, C4, C5) through the same legs, with the
             reference CPU path timed beside each (N=1).
  roofline   the dominant kernel's algorithmic bytes / its event-timed duration vs measured HBM
             copy bandwidth (MEASURED_PEAKS.json); traffic from the committed ncu capture.
  cpu_baseline  the reference (oracle/_ref, reliefmap compiled in place) timed on this host's
             cores in its parallel mode on a bounded sample of the same workload (rank 0, N=1).
N>1 (torchrun): the configured split of ONE frame across the GPUs ("point
batches sharded across 1/2/4/8 GPUs"): every rank keeps a map replica and ingests / ray-casts its
batch of the frame; the exchanges run inside the library over NCCL (relief_gpu_group_*). `value`
is the frame's points / the slowest rank's device time (strong scaling); rank 0 re-runs the same
frames on a single-GPU map and checks every layer bit for bit (parity_hash_ok). Independent maps
per GPU (replicas, weak scaling) are reported under `replicas`.

--impl reference: rank 0 alone times the reference's CPU implementation (oracle/_ref, parallel
mode, all host threads up to its 16-thread cap) through its own C API on the same workload.
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import statistics
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "points/sec integrated and per-frame map-update ms (1/2/4/8 B200) vs CPU ref"
REF_LIB = ROOT / "oracle" / "_ref" / "librelief_ref.so"
L2_FLUSH_BYTES = 256 << 20
DEVSTATS_BYTES = 128  # DevStats read back per scan (device_map.hpp)
N_FRAMES = 8          # distinct frames cycled by both arms
# gates that cannot fire: the configuration the information-form group mode requires
PRE_FRAMES = 40  # steady-state leg: frames integrated before its warm-up (untimed)
UNGATED = "update.mahalanobis_threshold = 1e12\nupdate.wall_count_threshold = 1073741824\n"
CONFIG_NAMES = ("C1", "C2", "C3", "headline", "C4", "C5")
LAYERS = ("elevation", "variance", "last_update", "upper_bound", "upper_bound_valid", "traversability",
          "normal_x", "normal_y", "normal_z", "valid")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled DURING the timed region.

    NVML polled from a thread every ~1 ms (the timed region is tens of ms, too short for
    nvidia-smi -lms); reasons are the B200_PROFILING.md set."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, device: int, period_s: float = 0.001):
        self.device = device
        self.period = period_s
        self.samples, self.reasons_seen = [], set()
        self.max_mhz = None
        self.stop = threading.Event()
        self.handle = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            props = torch.cuda.get_device_properties(device)
            bus = (f"{int(getattr(props, 'pci_domain_id', 0)):08X}:{int(props.pci_bus_id):02X}:"
                   f"{int(getattr(props, 'pci_device_id', 0)):02X}.0")
            try:
                self.handle = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.handle = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.nv = pynvml
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # no NVML: report no samples rather than guess
            log(f"clock sampler disabled: {e}")

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)))
                mask = get_reasons(self.handle)
                for name, bit in self.REASONS.items():
                    if mask & bit:
                        self.reasons_seen.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.handle is not None:
            self.thread = threading.Thread(target=self._run, daemon=True)
            self.thread.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.handle is not None:
            self.thread.join(timeout=1)

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons_seen),
                "samples": len(self.samples), "source": "NVML, 1 ms polling during the timed steps"}


# ------------------------------------------------------------- workloads
def workload(name):
    from paper_2204_12876_b200 import workloads as wl
    return wl.ALL["C3" if name == "C5" else name]()


def render_frames(lib, w, cfg_path, n_frames, ref=None):
    """Distinct frames (cycled if more steps are needed). ref: use the reference's renderer."""
    import paper_2204_12876_b200 as pk
    frames = []
    for f in range(n_frames):
        calls = []
        for c in w.calls(f):
            if ref is None:
                xyz = pk.sim_render(lib, cfg_path, c.pose, c.time, c.seed, c.scan_index)
            else:
                xyz = ref_render(ref, cfg_path, c.pose, c.time, c.seed, c.scan_index)
            calls.append((np.ascontiguousarray(xyz), c))
        frames.append(calls)
    return frames


def ref_render(ref, cfg_path, pose, t, seed, idx, cap=1 << 21):
    DP = ctypes.POINTER(ctypes.c_double)
    ref.ref_render_scan.restype = ctypes.c_int64
    ref.ref_render_scan.argtypes = [ctypes.c_char_p, DP, ctypes.c_double, ctypes.c_uint64,
                                    ctypes.c_uint64, DP, ctypes.c_int64]
    pose = np.ascontiguousarray(pose, dtype=np.float64)
    buf = np.empty(cap * 3)
    n = ref.ref_render_scan(str(cfg_path).encode(), pose.ctypes.data_as(DP), t, seed, idx,
                            buf.ctypes.data_as(DP), cap)
    if n > cap:
        return ref_render(ref, cfg_path, pose, t, seed, idx, cap=int(n))
    return buf[: 3 * n].reshape(n, 3).copy()


def config_dict(w, name, pts, calls, n_frames, world):
    """The `config` object -- identical in both arms (it names the workload, not the impl)."""
    from paper_2204_12876_b200 import workloads as wl
    d = {"workload": f"{w.name}: {w.description}", "points_per_frame": int(pts),
         "map": f"{w.width}x{w.height}@{w.resolution}m", "calls_per_frame": int(calls),
         "distinct_frames": int(n_frames),
         "parallelism": ("1 GPU" if world == 1 else
                         f"one frame split over {world} GPUs (point batches, NCCL exchanges)"),
         "l2": "flushed before every timed step (256 MiB write, then a 256 MiB read)"}
    if name == "C5":
        d["workload"] = f"C5: C3 frame + post-processing chain {wl.C5_CHAIN} on the 500x500 map"
    return d


# -------------------------------------------------------- reference (CPU)
def ref_library():
    import paper_2204_12876_b200 as pk
    ref = pk.load_library(REF_LIB, gpu_api=False)
    I, DP = ctypes.c_int, ctypes.POINTER(ctypes.c_double)
    ref.ref_smooth_chain.restype = I
    ref.ref_smooth_chain.argtypes = [DP, ctypes.POINTER(ctypes.c_uint8), I, I, ctypes.POINTER(I),
                                     ctypes.POINTER(I), DP, I, DP, ctypes.POINTER(ctypes.c_uint8)]
    return ref


def ref_chain(ref, m, steps):
    """The reference's smoothChain (postprocess.cpp:166-197) on the map's masked elevation."""
    elev = m.layer("elevation")
    valid = np.ascontiguousarray(m.layer("valid") != 0, dtype=np.uint8)
    H, W = elev.shape
    kinds = (ctypes.c_int * len(steps))(*[s[0] for s in steps])
    radii = (ctypes.c_int * len(steps))(*[s[1] for s in steps])
    sig = (ctypes.c_double * len(steps))(*[float(s[2]) for s in steps])
    vo, ko = np.empty_like(elev), np.empty_like(valid)
    DP, U8 = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint8)
    t0 = time.perf_counter()
    ref.ref_smooth_chain(np.ascontiguousarray(elev).ctypes.data_as(DP), valid.ctypes.data_as(U8), W, H,
                         kinds, radii, sig, len(steps), vo.ctypes.data_as(DP), ko.ctypes.data_as(U8))
    return time.perf_counter() - t0


def time_reference(name, steps, warmup, mode="par", n_frames=N_FRAMES):
    """Times oracle/_ref (the reference compiled in place) through its own C API. Returns
    (points/s, per-step seconds, points per frame, calls per frame, frames used)."""
    import paper_2204_12876_b200 as pk
    from paper_2204_12876_b200 import workloads as wl
    w = workload(name)
    ref = ref_library()
    d = Path(tempfile.mkdtemp())
    cfgp = d / "ref.config"
    cfgp.write_text(w.config_text)
    cfg = pk.Config.load(ref, cfgp)
    cfg.set_mode(mode)
    m = pk.ReliefMap.create(ref, w.resolution, w.width, w.height)
    nf = min(steps + warmup, n_frames)
    frames = render_frames(None, w, cfgp, nf, ref=ref)
    times, pts = [], 0
    for s in range(warmup + steps):
        calls = frames[s % nf]
        t0 = time.perf_counter()
        for xyz, c in calls:
            m.integrate(xyz, c.pose, 0.1 * s, cfg)
        dt = time.perf_counter() - t0
        if name == "C5":
            dt += ref_chain(ref, m, wl.C5_CHAIN)
        if s >= warmup:
            times.append(dt)
            pts += sum(len(x) for x, _ in calls)
    return pts / sum(times), times, sum(len(x) for x, _ in frames[0]), len(frames[0]), nf


def cpu_threads_used(mode):
    return 1 if mode == "det" else min(os.cpu_count() or 1, 16)


def run_reference(args, world):
    """--impl reference: same workload / metric / config as the b200 arm; rank 0 only."""
    w = workload(args.workload)
    v, times, pts, calls, nf = time_reference(args.workload, args.steps, args.warmup)
    cores = cpu_threads_used("par")
    sample = (f"{args.steps} frames of {args.workload} ({pts} pts each) after {args.warmup} warm-up "
              f"frames, {nf} distinct frames cycled, reliefmap reference (oracle/_ref) par mode via "
              f"its C API, {cores} threads")
    out = {"metric": METRIC, "value": v, "unit": "points/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": statistics.mean(times) * 1e3, "higher_is_better": True,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (reference renderer, same frames as the b200 arm)",
           "config": config_dict(w, args.workload, pts, calls, nf, world),
           "impl": "reference",
           "impl_detail": {"library": "oracle/_ref/librelief_ref.so (reference compiled in place)",
                           "mode": "par (parallelFor)", "threads": cores, "host_cpus": os.cpu_count()},
           "cpu_baseline": {"value": v, "unit": "points/s", "cores": cores, "kind": "reference",
                            "sample": sample},
           "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if not args.no_configs:
        cfgs = {}
        for name in CONFIG_NAMES:
            cv, ct, cpts, ccalls, cnf = time_reference(name, args.config_ref_steps, 1)
            cfgs[name] = {"value": cv, "unit": "points/s", "ms_per_frame": statistics.median(ct) * 1e3,
                          "points_per_frame": cpts, "calls_per_frame": ccalls,
                          "sample": f"{args.config_ref_steps} frames after 1 warm-up, {cores} threads"}
        out["configs"] = cfgs
    return out


# ------------------------------------------------------------- b200 arm
class Device:
    """Per-rank device context: L2 flush buffers, barrier, max-over-ranks."""

    def __init__(self, local_rank, dist):
        import torch
        self.torch, self.dist, self.dev = torch, dist, f"cuda:{local_rank}"
        self.flush_buf = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=self.dev)
        self.sweep = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=self.dev)

    def flush_l2(self):
        """Write a buffer larger than L2, then read another one so the flush's dirty lines are
        written back here, outside the timed region, instead of during the next timed step."""
        self.flush_buf.zero_()
        self.sweep.sum()
        self.torch.cuda.synchronize()

    def barrier(self):
        self.torch.cuda.synchronize()
        if self.dist is not None:
            self.dist.barrier()

    def max(self, v):
        from paper_2204_12876_b200 import multigpu as mg
        return mg.max_over_ranks(v, self.dist)


def load_frames(lib, name, n_frames, local_rank):
    import torch
    import paper_2204_12876_b200 as pk
    w = workload(name)
    tmp = Path(tempfile.mkdtemp())
    cfgp = tmp / "w.config"
    cfgp.write_text(w.config_text)
    cfg = pk.Config.load(lib, cfgp)
    frames = render_frames(lib, w, cfgp, n_frames)
    dev = [[(torch.from_numpy(x).to(f"cuda:{local_rank}").contiguous(), c) for x, c in fr] for fr in frames]
    torch.cuda.synchronize()
    pin = [[(torch.from_numpy(x).pin_memory().numpy(), c) for x, c in fr] for fr in frames]
    return w, cfg, frames, dev, pin


def roofline(dom, kmean, visits, w, pts, calls):
    """Algorithmic bytes of the dominant kernel group / its event-timed duration."""
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    cells = w.width * w.height
    by = {
        "ingest": 24 * pts + 40 * pts + 5 * pts,               # xyz in; map-frame xyz+var out; key+flag
        "drift": 2 * 18 * cells * calls,                       # elev/ub/valid/ubv read+write
        "sort": 2 * 2 * 8 * pts + 16 * pts,                    # 2 passes (key,val) in+out; payload out
        "fusion": 16 * pts + 132 * cells * calls // 8,         # payload in; touched cell state r/w
        "rays": 25 * pts + visits,                             # endpoint + flag per ray, 1 B per visit
        "cells": 132 * cells * calls,                          # persistent state read + written
    }
    idx = ["ingest", "drift", "sort", "fusion", "rays", "cells"].index(dom)
    dur = kmean[1 + idx]
    ach = by[dom] / dur / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(dom)
    ceiling = None
    cf = ROOT / "profiles" / "l2_visit_ceiling.json"
    if cf.exists():
        ceiling = json.loads(cf.read_text()).get("u8_1MB_probes_per_s")
    return {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
            "frac": ach / peak, "traffic": traffic, "algorithmic_bytes": int(by[dom]),
            "duration_us": dur * 1e6, "dda_visits_per_frame": int(visits),
            "visits_per_s": visits / dur if dom == "rays" else None,
            "l2_random_probe_ceiling_per_s": ceiling,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)" if peaks else "fallback 6.65 TB/s"}


def single_gpu_legs(lib, D, name, steps, warmup, local_rank, want_roofline=True, want_stream=False,
                    n_frames=N_FRAMES, clocks=None):
    """value / wall / e2e (pinned, pageable) / phase split of one workload on one GPU."""
    import torch
    import paper_2204_12876_b200 as pk
    from paper_2204_12876_b200 import workloads as wl
    nf = min(steps + warmup, n_frames)
    w, cfg, frames, dev_frames, pin_frames = load_frames(lib, name, nf, local_rank)
    pts = sum(len(x) for x, _ in frames[0])
    calls = len(frames[0])
    chain = name == "C5"
    cells = w.width * w.height
    d_vals = torch.empty(cells, dtype=torch.float64, device=D.dev)
    d_ok = torch.empty(cells, dtype=torch.uint8, device=D.dev)

    def run_device(m, s):
        """(device seconds, wall seconds inside the library calls, wall seconds of the Python
        calls) of one step. The library's in-call time is its own clock around the C call
        (ScanStats.total_seconds); the Python time adds the ctypes marshalling."""
        dev = wall = pywall = 0.0
        for t, c in dev_frames[s % nf]:
            t0 = time.perf_counter()
            st = m.integrate_device(t.data_ptr(), t.shape[0], c.pose, 0.1 * s, cfg)
            pywall += time.perf_counter() - t0
            wall += st.total_seconds
            dev += m.kernel_seconds()[7]  # device time, events at the frame ends only
        if chain:
            t0 = time.perf_counter()
            dev += m.smooth_chain_device("elevation", wl.C5_CHAIN, d_vals.data_ptr(), d_ok.data_ptr())
            wall += time.perf_counter() - t0
            pywall += time.perf_counter() - t0
        return dev, wall, pywall

    # value: device-resident input
    m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height, device=local_rank)
    for s in range(warmup):
        run_device(m, s)
    D.barrier()
    dev_t, wall_t, pywall_t, launches = [], [], [], 0
    cm = clocks if clocks is not None else _Null()
    with cm:
        for s in range(warmup, warmup + steps):
            D.flush_l2()
            dv, wv, pv = run_device(m, s)
            dev_t.append(dv)
            wall_t.append(wv)
            pywall_t.append(pv)
            launches += m.last_launches() * calls
    D.barrier()
    dev_total = D.max(sum(dev_t))
    out = {"value": pts * steps / dev_total, "unit": "points/s", "ms_per_frame": dev_total / steps * 1e3,
           "wall_ms_per_frame": statistics.mean(wall_t) * 1e3,
           "host_overhead_us_per_call": (statistics.mean(wall_t) - statistics.mean(dev_t)) / calls * 1e6,
           "python_call_us_per_call": (statistics.mean(pywall_t) - statistics.mean(wall_t)) / calls * 1e6,
           "points_per_frame": pts, "calls_per_frame": calls, "gpu_launches": int(launches),
           "graphs": {"instantiated": m.graph_stats()[0], "updated": m.graph_stats()[1]},
           "frame_device_ms": [round(x * 1e3, 4) for x in dev_t]}
    if chain:
        out["ms_per_frame_incl_post"] = out["ms_per_frame"]
    # phase split (separate pass with phase events on: they end the programmatic overlap)
    if want_roofline:
        m.set_phase_timing(True)
        diag = max(3, min(steps, 6))
        ksum = np.zeros(8)
        for s in range(warmup + steps, warmup + steps + diag):
            D.flush_l2()
            for t, c in dev_frames[s % nf]:
                m.integrate_device(t.data_ptr(), t.shape[0], c.pose, 0.1 * s, cfg)
                ksum += m.kernel_seconds()
        m.set_phase_timing(False)
        kmean = ksum / diag
        names = ["ingest", "drift", "sort", "fusion", "rays", "cells"]
        shares = dict(zip(names, kmean[1:7]))
        dom = max(shares, key=shares.get)
        out["kernel_ms"] = {n: float(v) * 1e3 for n, v in zip(names, kmean[1:7])}
        out["roofline"] = roofline(dom, kmean, m.last_visits() * calls, w, pts, calls)
    if chain:
        ct = [m.smooth_chain_device("elevation", wl.C5_CHAIN, d_vals.data_ptr(), d_ok.data_ptr())
              for _ in range(5)]
        out["post_chain_ms"] = statistics.median(ct[1:]) * 1e3
    m.close()

    # steady state: the same timed protocol on a map that has already integrated PRE_FRAMES frames
    # (untimed), as a mapper that has been running for a few seconds; pass 1's jumps clear most of
    # the rays' cells only once the map's bounds have settled
    if want_stream:
        m4 = pk.ReliefMap.create(lib, w.resolution, w.width, w.height, device=local_rank)
        for s in range(PRE_FRAMES + warmup):
            run_device(m4, s)
        D.barrier()
        st_t = []
        for s in range(PRE_FRAMES + warmup, PRE_FRAMES + warmup + steps):
            D.flush_l2()
            st_t.append(run_device(m4, s)[0])
        D.barrier()
        st_total = D.max(sum(st_t))
        out["steady_state"] = {"value": pts * steps / st_total, "unit": "points/s",
                               "ms_per_frame": st_total / steps * 1e3, "pre_frames": PRE_FRAMES,
                               "note": f"same steps / warm-up / L2 flush as value, on a map that integrated "
                                       f"{PRE_FRAMES} earlier frames of the same sequence (untimed)"}
        m4.close()

    # e2e: drop-in C ABI, pinned host input (and pageable)
    def e2e(frames_src, label):
        m2 = pk.ReliefMap.create(lib, w.resolution, w.width, w.height, device=local_rank)
        for s in range(warmup):
            for x, c in frames_src[s % nf]:
                m2.integrate(x, c.pose, 0.1 * s, cfg)
                if chain:  # (the first chain call allocates its scratch)
                    m2.smooth_chain_device("elevation", wl.C5_CHAIN, d_vals.data_ptr(), d_ok.data_ptr())
        D.barrier()
        tt, copy = [], 0.0
        for s in range(warmup, warmup + steps):
            D.flush_l2()
            t0 = time.perf_counter()
            for x, c in frames_src[s % nf]:
                m2.integrate(x, c.pose, 0.1 * s, cfg)  # H2D + kernels + stats D2H, synchronous
                if chain:
                    m2.smooth_chain_device("elevation", wl.C5_CHAIN, d_vals.data_ptr(), d_ok.data_ptr())
            tt.append(time.perf_counter() - t0)
            copy += m2.kernel_seconds()[0] * calls
        D.barrier()
        tot = D.max(sum(tt))
        m2.close()
        return {"value": pts * steps / tot, "unit": "points/s", "h2d_bytes_per_step": 24 * pts,
                "d2h_bytes_per_step": DEVSTATS_BYTES * calls, "ms_per_step": tot / steps * 1e3,
                "h2d_copy_ms_per_step": copy / steps * 1e3, "api": label}

    out["e2e"] = e2e(pin_frames, "relief_map_integrate (drop-in C ABI, synchronous), pinned host input")
    out["e2e_pageable"] = e2e(frames, "relief_map_integrate, pageable (numpy) host input")

    if want_stream:  # the additive async API, 3 frames in flight
        m3 = pk.ReliefMap.create(lib, w.resolution, w.width, w.height, device=local_rank)
        for s in range(warmup):
            for x, c in pin_frames[s % nf]:
                m3.integrate(x, c.pose, 0.1 * s, cfg)
        D.barrier()
        t0 = time.perf_counter()
        pending = 0
        for s in range(warmup, warmup + steps):
            for x, c in pin_frames[s % nf]:
                m3.integrate_async(x, c.pose, 0.1 * s, cfg)
                pending += 1
                if pending == 3:
                    m3.wait()
                    pending -= 1
        while pending:
            m3.wait()
            pending -= 1
        tot = D.max(time.perf_counter() - t0)
        out["e2e_streaming"] = {"value": pts * steps / tot, "unit": "points/s", "h2d_bytes_per_step": 24 * pts,
                                "d2h_bytes_per_step": DEVSTATS_BYTES * calls, "ms_per_step": tot / steps * 1e3,
                                "api": "relief_gpu_map_integrate_async + relief_gpu_map_wait, pinned host input, "
                                       "3 frames in flight; no per-step L2 flush"}
        m3.close()
    return w, out, nf


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        pass


def layer_digest(m) -> str:
    h = hashlib.sha256()
    for name in LAYERS:
        h.update(np.ascontiguousarray(m.layer(name)).tobytes())
    return h.hexdigest()


def sharded_legs(lib, D, args, rank, world, local_rank, dist):
    """N>1: the configured split of one frame over the group (NCCL inside the library)."""
    import torch
    import paper_2204_12876_b200 as pk
    from paper_2204_12876_b200 import multigpu as mg
    steps, warmup = args.steps, args.warmup
    nf = min(steps + warmup, N_FRAMES)
    w, cfg, frames, dev_frames, pin_frames = load_frames(lib, args.workload, nf, local_rank)
    if len(frames[0]) != 1:
        raise RuntimeError("the sharded bench takes one integrate call per frame")
    n_total = len(frames[0][0][0])
    lo, hi = pk.group_bounds(lib, n_total, world, rank)
    my_dev = [fr[0][0][lo:hi].contiguous() for fr in dev_frames]
    my_pin = [np.ascontiguousarray(fr[0][0][lo:hi]) for fr in pin_frames]
    torch.cuda.synchronize()

    m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height, device=local_rank)
    grp = mg.create_nccl_group(lib, m, dist)
    for s in range(warmup):
        grp.integrate_device(my_dev[s % nf].data_ptr(), hi - lo, n_total, frames[s % nf][0][1].pose, 0.1 * s, cfg)
    D.barrier()
    dev_t, launches = [], 0
    with ClockSampler(local_rank) as clocks:
        for s in range(warmup, warmup + steps):
            D.flush_l2()
            grp.integrate_device(my_dev[s % nf].data_ptr(), hi - lo, n_total, frames[s % nf][0][1].pose,
                                 0.1 * s, cfg)
            dev_t.append(m.kernel_seconds()[7])
            launches += m.last_launches()
    D.barrier()
    dev_total = D.max(sum(dev_t))
    digest = layer_digest(m)
    digests = [None] * world
    dist.all_gather_object(digests, digest)

    # e2e: host batches (pinned), group call synchronous on every rank
    m2 = pk.ReliefMap.create(lib, w.resolution, w.width, w.height, device=local_rank)
    grp2 = mg.create_nccl_group(lib, m2, dist)
    for s in range(warmup):
        grp2.integrate(my_pin[s % nf], n_total, frames[s % nf][0][1].pose, 0.1 * s, cfg)
    D.barrier()
    tt = []
    for s in range(warmup, warmup + steps):
        D.flush_l2()
        t0 = time.perf_counter()
        grp2.integrate(my_pin[s % nf], n_total, frames[s % nf][0][1].pose, 0.1 * s, cfg)
        tt.append(time.perf_counter() - t0)
    D.barrier()
    e2e_total = D.max(sum(tt))
    grp2.close()
    m2.close()

    # information-form group frames (relief_gpu_group_set_fusion): the same split with ungated
    # fusion -- per-cell partial sums all-reduced instead of the records gathered and the whole
    # frame sorted and folded on every rank; needs a config whose gates cannot fire
    import tempfile
    from pathlib import Path
    up = Path(tempfile.mkdtemp()) / "ungated.config"
    up.write_text(w.config_text + UNGATED)
    cfg_u = pk.Config.load(lib, up)
    m3 = pk.ReliefMap.create(lib, w.resolution, w.width, w.height, device=local_rank)
    grp3 = mg.create_nccl_group(lib, m3, dist)
    grp3.set_fusion(pk.Group.INFORMATION)
    for s in range(warmup):
        grp3.integrate_device(my_dev[s % nf].data_ptr(), hi - lo, n_total, frames[s % nf][0][1].pose, 0.1 * s,
                              cfg_u)
    D.barrier()
    info_t = []
    for s in range(warmup, warmup + steps):
        D.flush_l2()
        grp3.integrate_device(my_dev[s % nf].data_ptr(), hi - lo, n_total, frames[s % nf][0][1].pose, 0.1 * s,
                              cfg_u)
        info_t.append(m3.kernel_seconds()[7])
    D.barrier()
    info_total = D.max(sum(info_t))
    info_digests = [None] * world
    dist.all_gather_object(info_digests, layer_digest(m3))
    info_elev = m3.layers()["elevation"] if rank == 0 else None
    grp3.close()
    m3.close()

    # replicas: an independent map per GPU (weak scaling)
    _, rep, _ = single_gpu_legs(lib, D, args.workload, steps, warmup, local_rank, want_roofline=False)
    rep_max_ms = D.max(rep["ms_per_frame"])

    parity = None
    if rank == 0:  # the same frames on one GPU, one map: bit-identical layers expected
        ms = pk.ReliefMap.create(lib, w.resolution, w.width, w.height, device=local_rank)
        for s in range(warmup + steps):
            t, c = dev_frames[s % nf][0]
            ms.integrate_device(t.data_ptr(), t.shape[0], c.pose, 0.1 * s, cfg)
        want = layer_digest(ms)
        mu = pk.ReliefMap.create(lib, w.resolution, w.width, w.height, device=local_rank)
        for s in range(warmup + steps):  # the ungated sequential fold on one GPU
            t, c = dev_frames[s % nf][0]
            mu.integrate_device(t.data_ptr(), t.shape[0], c.pose, 0.1 * s, cfg_u)
        ue = mu.layers()["elevation"]
        fin = np.isfinite(ue) & np.isfinite(info_elev)
        same_mask = bool((np.isnan(ue) == np.isnan(info_elev)).all())
        rel = float((np.abs(info_elev[fin] - ue[fin]) / np.maximum(1.0, np.abs(ue[fin]))).max()) if fin.any() else 0.0
        mu.close()
        parity = {"parity_hash_ok": all(d == want for d in digests),
                  "replicas_consistent": len(set(digests)) == 1,
                  "layer_sha256": want[:16],
                  "check": "sha256 of all 10 layers after the warm-up + timed frames, every rank vs a "
                           "single-GPU map fed the whole frames",
                  "information_form": {
                      "value": n_total * steps / info_total, "unit": "points/s",
                      "ms_per_step": info_total / steps * 1e3,
                      "replicas_consistent": len(set(info_digests)) == 1,
                      "elevation_max_rel_diff_vs_sequential": rel, "valid_mask_equal": same_mask,
                      "parity_ok": same_mask and rel <= 1e-9 and len(set(info_digests)) == 1,
                      "config": "workload config + " + UNGATED.replace(chr(10), "; ").strip("; "),
                      "api": "relief_gpu_group_set_fusion(RELIEF_GPU_GROUP_INFORMATION), device batches"}}
    grp.close()
    m.close()
    out = {"value": n_total * steps / dev_total, "ms_per_step": dev_total / steps * 1e3,
           "points_per_frame": n_total, "gpu_launches": int(launches), "clocks": clocks.summary(),
           "e2e": {"value": n_total * steps / e2e_total, "unit": "points/s", "h2d_bytes_per_step": 24 * n_total,
                   "d2h_bytes_per_step": DEVSTATS_BYTES * world, "ms_per_step": e2e_total / steps * 1e3,
                   "api": "relief_gpu_group_integrate (NCCL group), each rank's batch from pinned host memory"},
           "replicas": {"value": world * pts_rate(rep), "unit": "points/s", "scaling": "weak",
                        "ms_per_frame_max_rank": rep_max_ms,
                        "note": "independent map + frame stream per GPU; sum of per-rank rates"},
           "nccl_version": lib.relief_gpu_nccl_version()}
    if parity is not None:
        out.update(parity)
    return w, out, nf


def pts_rate(leg):
    return leg["points_per_frame"] / (leg["ms_per_frame"] * 1e-3)


def run_b200(args, rank, world, local_rank):
    import torch
    import paper_2204_12876_b200 as pk

    lib = pk.load_library()
    if lib.relief_gpu_device_count() <= local_rank:
        raise RuntimeError(f"rank {rank}: CUDA device {local_rank} not visible (no CPU fallback)")
    torch.cuda.set_device(local_rank)
    dist = None
    # RB_BENCH_GROUP=1: the N > 1 legs (group frames over NCCL) even on one rank -- a smoke run of
    # that code path on a single GPU (torchrun --nproc-per-node 1)
    group = world > 1 or os.environ.get("RB_BENCH_GROUP") == "1"
    if group:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    D = Device(local_rank, dist)

    if group:
        w, main, nf = sharded_legs(lib, D, args, rank, world, local_rank, dist)
        result = None
        if rank == 0:
            result = {
                "metric": METRIC, "value": main["value"], "unit": "points/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (library scene simulator, bit-identical to the reference renderer)",
                "config": config_dict(w, args.workload, main["points_per_frame"], 1, nf, world),
                "e2e": main["e2e"], "gpu_launches": main["gpu_launches"], "clocks": main["clocks"],
                "replicas": main["replicas"], "parity_hash_ok": main.get("parity_hash_ok"),
                "information_form": main.get("information_form"),
                "replicas_consistent": main.get("replicas_consistent"),
                "parity_check": main.get("check"), "layer_sha256": main.get("layer_sha256"),
                "nccl_version": main["nccl_version"], "cpu_baseline": None,
                "timing": "device time per frame from CUDA events on each rank's library stream "
                          "(ingest -> exchanges -> cell phases), max over ranks",
            }
        dist.destroy_process_group()
        return result

    # ---------------- N = 1
    clocks = ClockSampler(local_rank)
    w, main, nf = single_gpu_legs(lib, D, args.workload, args.steps, args.warmup, local_rank,
                                  want_stream=True, clocks=clocks)
    configs = {}
    if not args.no_configs:
        for name in CONFIG_NAMES:
            if name == args.workload:
                leg = {k: v for k, v in main.items() if k not in ("frame_device_ms",)}
            else:
                _, leg, _ = single_gpu_legs(lib, D, name, args.config_steps, 3, local_rank)
                leg.pop("frame_device_ms", None)
            configs[name] = leg
    cpu = None
    if not args.no_cpu_baseline and REF_LIB.exists():
        v, times, pts_r, _, cnf = time_reference(args.workload, args.cpu_frames, 1)
        cpu = {"value": v, "unit": "points/s", "cores": cpu_threads_used("par"), "kind": "reference",
               "sample": f"{args.cpu_frames} frames of {args.workload} ({pts_r} pts each) after 1 "
                         f"warm-up frame, reliefmap reference (oracle/_ref) par mode via its C API",
               "ms_per_frame": statistics.median(times) * 1e3, "host_cpus": os.cpu_count()}
        for name, leg in configs.items():
            cv, ct, _, _, _ = time_reference(name, args.config_ref_steps, 1)
            leg["cpu_baseline"] = {"value": cv, "ms_per_frame": statistics.median(ct) * 1e3,
                                   "kind": "reference", "cores": cpu_threads_used("par")}
            leg["speedup_e2e_vs_reference"] = leg["e2e"]["value"] / cv
            leg["speedup_device_vs_reference"] = leg["value"] / cv
    return {
        "metric": METRIC, "value": main["value"], "unit": "points/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": main["ms_per_frame"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (library scene simulator, bit-identical to the reference renderer)",
        "config": config_dict(w, args.workload, main["points_per_frame"], main["calls_per_frame"], nf, 1),
        "wall_ms_per_step": main["wall_ms_per_frame"],
        "host_overhead_us_per_call": main["host_overhead_us_per_call"],
        "python_call_us_per_call": main["python_call_us_per_call"],
        "host_overhead_note": "wall time inside the library's synchronous call (its own clock) minus the "
                              "frame's device time; python_call_us_per_call is the ctypes marshalling of the "
                              "bench driver on top",
        "kernel_ms": main.get("kernel_ms"),
        "phase_split_note": "kernel_ms / roofline.duration_us come from a separate pass with phase events "
                            "on (they end the programmatic overlap at the phase boundaries); value and "
                            "ms_per_step are timed without them",
        "e2e": main["e2e"], "e2e_pageable": main["e2e_pageable"], "e2e_streaming": main.get("e2e_streaming"),
        "steady_state": main.get("steady_state"),
        "gpu_launches": main["gpu_launches"], "roofline": main.get("roofline"),
        "cpu_baseline": cpu, "clocks": clocks.summary(), "configs": configs,
    }


# ---------------------------------------------------------------- main
def main():
    import faulthandler
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="C4", choices=["C1", "C2", "C3", "C4", "headline"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-frames", type=int, default=3)
    ap.add_argument("--config-steps", type=int, default=10)
    ap.add_argument("--config-ref-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        if not REF_LIB.exists():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/librelief_ref.so not built"}))
            return
        print(json.dumps(run_reference(args, world)), flush=True)
        return

    res = run_b200(args, rank, world, local_rank)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
